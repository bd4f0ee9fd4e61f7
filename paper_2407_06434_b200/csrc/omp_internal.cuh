// Internal declarations shared by the library's translation units (not part of the ABI).
#pragma once

#include <cuda.h>
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdlib.h>

#include "omp_b200.h"

namespace ompb {

// per-signal running state; finished signals hold an ompSigStatus_t (>= 0)
constexpr int32_t SIG_RUNNING = -1;
// selection codes besides an atom index
constexpr int32_t SEL_DEGENERATE = -1;   // maximum correlation is 0 (exhausted residual)
constexpr int32_t SEL_NAN = -2;          // a correlation was not finite
constexpr int32_t SEL_OVERFLOW = -3;     // screen partial: more in-window entries than TOPK slots
// factor-append pivot threshold: ||a||^2 - ||z||^2 <= TAU_F * ||a||^2 -> DEGENERATE
constexpr float TAU_F = 1e-5f;

constexpr int K_TILE = 64;     // K padding of every plane (a 128-byte bf16 TMA/UMMA row)
constexpr int N_TILE = 256;    // atom padding (UMMA N of the correlation kernel)
constexpr int MAX_S = 512;
#ifndef OMP_TOPK
#define OMP_TOPK 4
#endif
constexpr int TOPK = OMP_TOPK;   // screening candidates kept per (signal, 128-atom half tile)
constexpr int SCREEN_GROUP = 128;   // atoms per screen partial (half of the 256-atom UMMA tile)

// Programmatic dependent launch between the screen and the update of the screened path: each kernel
// lets the next one launch early (griddepcontrol.launch_dependents) and the next one waits for the
// previous grid's completion (griddepcontrol.wait) before reading its output, so only launch latency
// and prologues overlap.  OMP_B200_PDL=0 turns the launch attribute off (A/B; same results).
// edge: 1 = update -> next screen (the screen's prologue overlaps the update's tail),
//       2 = screen -> update (the update's launch overlaps the screen's tail)
inline bool pdl_enabled(int edge) {
  static int on = -1;
  if (on < 0) {
    const char* e = getenv("OMP_B200_PDL");
    on = e ? atoi(e) : 1;   // measured: edge 1 gains 1-5 % (c2, c3, c5), edge 2 loses 2-10 %
  }
  return (on & edge) != 0;
}

// The screen's candidate window per signal, in absolute units:
//   W_b = ca (||r_b|| + d_b) + cd d_b + cr ||r_b||,   d_b = ||r_b - bf16(r_b)|| (measured when the
// residual's bf16 plane is written; 0 without a bf16 plane).  bf16 screen: ca = 2.5 (E_a + K 2^-23
// (1 + E_a)) with E_a = max_n ||bf16(a_n / ||a_n||) - a_n / ||a_n||||, cd = 2.5, cr = 2.5 c0' (the FP32
// re-evaluation); 3xTF32 screen: ca = cd = 0, cr = the static window 2.5 (c0 + c0').  Stored per live
// row in rslot (the screen's and the refine's threshold is max - W_b).
struct WinCoef {
  float ca, cd, cr;
};

// screening-GEMM operand kinds
constexpr int KIND_BF16 = 0;
constexpr int KIND_3XTF32 = 1;

inline int64_t round_up(int64_t a, int64_t b) { return (a + b - 1) / b * b; }

// A row-major K-major operand: element (row, k) of plane p at plane[p] + row * ld + k.
// bf16 kind: plane[0] = bf16 values.  3xtf32 kind: plane[0] = tf32 hi, plane[1] = lo (fp32).
// fp32 (SIMT): plane[0] = fp32 values.
struct Operand {
  const void* plane[2];
  int64_t rows;
  int64_t ld;      // row stride in elements (multiple of K_TILE)
};

// ---- K1: correlation C[b, n] = sum_k R[b, k] * At[n, k] ----
// Row counts: R.rows is the buffer's capacity; `live_rows` (device, may be null) is the number of
// live rows at the top of the buffer when the kernel runs (live-set compaction).
// FP32 SIMT GEMM (round-to-nearest, sequential K): C written for rows < live rows, n < ncols
cudaError_t launch_corr_simt(const Operand& R, const Operand& At, int64_t K, float* C, int64_t ldc,
                             int64_t ncols, const int32_t* live_rows, cudaStream_t st);
// split-K form: K in slabs of kchunk, partials (slabs x rows x ldc floats of `work`) summed in slab
// order by a second kernel; 2 launches
int64_t corr_simt_splitk_slabs(int64_t K, int64_t kchunk);
cudaError_t launch_corr_simt_splitk(const Operand& R, const Operand& At, int64_t K, float* C, int64_t ldc,
                                    int64_t ncols, int64_t kchunk, float* work, cudaStream_t st);
// C = sum of nz slab partials (slab z at work + z zstride), in slab order
cudaError_t launch_sum_slabs(const float* work, int64_t nz, int64_t zstride, int64_t rows, int64_t cols, int64_t ld,
                             float* C, int64_t ldc, cudaStream_t st);
// tcgen05 GEMM C = R A^T on RAW operand planes, split-K in slabs of kslab (a multiple of the kind's
// K block), partials summed in slab order (2 launches); 3xTF32 for an FP32-grade result
cudaError_t launch_corr_tc_splitk(int kind, const Operand& R, const Operand& At, int64_t K, float* C, int64_t ldc,
                                  int64_t ncols, int64_t kslab, float* work, cudaStream_t st);
// tcgen05 screening GEMM on normalised atoms; C~ stored times ||a_n|| (diagnostics / numerics tests)
cudaError_t launch_corr_tc(int kind, const Operand& R, const Operand& At, int64_t K, float* C, int64_t ldc,
                           int64_t ncols, const float* norm, cudaStream_t st);
// tcgen05 screening GEMM, epilogue -> per (row, 128-atom group) the first TOPK entries (|c~_n|, n) within
// window * rslot[row] of the group's maximum, in index order; unused slots (-1, -1); overflow flagged
cudaError_t launch_corr_tc_topk(int kind, const Operand& R, const Operand& At, int64_t K, const int32_t* live_rows,
                                const float* rslot, float window, float2* part, cudaStream_t st);

// ---- K2 ----
// a3 over a materialised FP32 C (row slot[b]): n*_b = lowest n maximising |C[row,n]| * inv_norm[n]; c* = C[row,n*]
cudaError_t launch_select(const float* C, int64_t ldc, int64_t B, int64_t N, const float* inv_norm,
                          const int32_t* status, const int32_t* slot, int32_t* nstar, float* cstar,
                          cudaStream_t st);
// ---- setup / init ----
// K0: atoms -> FP32 copy At (Np x Mp), ||a_n||, 1/||a_n||, and the screen planes of the NORMALISED
// atoms a_n / ||a_n|| (optional bf16 plane / tf32 hi-lo planes)
// ea2_max (bf16 plane only): max over atoms of ||bf16(a_n / ||a_n||) - a_n / ||a_n||||^2 in FP64, as the
// bits of a non-negative double (atomicMax on unsigned long long); zero it before the launch
cudaError_t launch_prepare_atoms(const float* A, int64_t M, int64_t N, int64_t lda, int64_t Mp, int64_t Np,
                                 float* At, void* At_bf16, float* At_hi, float* At_lo, float* norm,
                                 float* inv_norm, int* bad_zero, int* bad_nonfinite,
                                 unsigned long long* ea2_max, cudaStream_t st);
// row-major fp32 matrix -> padded planes (fp32 copy, optional bf16, optional hi/lo)
cudaError_t launch_make_planes(const float* R, int64_t B, int64_t ldr, int64_t M, int64_t Mp, float* R32,
                               void* Rb, float* R_hi, float* R_lo, cudaStream_t st);
// a1: batch init; running signals take live-set slots (atomic counter *live0) and their r_0 = y
// planes go to row slot[b]; rslot[slot] = the window W_b of r_0 = y (WinCoef).  live0 == nullptr: no
// compaction, row b (slot and rslot may then be null).
cudaError_t launch_batch_init(const float* Y, int64_t B, int64_t ldy, int64_t M, int64_t Mp, int32_t S,
                              float eps, float* R32, void* Rb, float* R_hi, float* R_lo, float* X, int64_t ldx,
                              int32_t* support, int64_t lds, float* resid, int32_t* n_iter, int32_t* status,
                              int32_t* slot, int32_t* live0, float* rslot, cudaStream_t st,
                              double* ynorm2 = nullptr, WinCoef win = WinCoef{0.f, 0.f, 0.f});
// projection path: exact ||y - A_S x|| per signal after the last iteration
cudaError_t launch_final_resid(const float* Y, int64_t B, int64_t ldy, int64_t M, const float* At, int64_t Mp,
                               const float* X, int64_t ldx, const int32_t* support, int64_t lds,
                               const int32_t* n_iter, const int32_t* status, float* resid, cudaStream_t st);

// ---- a3 + a4 + a5 fused per signal (k_update.cu) ----
struct UpdateLaunch {
  int32_t k, S;
  float eps;
  int64_t B, N, M, Mp;
  const float2* part;      // screen partials (tensor-core modes) or nullptr (then nstar/cstar are used)
  int groups;              // screen partial groups per row (Np / SCREEN_GROUP)
  const float* rslot_in;   // the window W of each row of this iteration's buffer (refine threshold)
  WinCoef win;             // the next window's coefficients
  const int32_t* nstar;
  const float* cstar;
  const float* At;
  const float* inv_norm;
  const float* G;
  int64_t ldg;
  const float* Y;
  int64_t ldy;
  float* F;
  int64_t ldf;             // multiple of 4 (16-byte aligned packed-F rows)
  float* U;
  int64_t ldu;
  float* X;
  int64_t ldx;
  int32_t* support;
  int64_t lds;
  const float* R32in;      // residual planes read at row slot[b] (this iteration's buffer)
  float* R32;              // residual planes written at the signal's new slot (next iteration's buffer)
  void* Rb;
  float* Rhi;
  float* Rlo;
  float* rslot_out;        // window W per new slot (the next screen's and refine's threshold)
  int32_t* slot;           // signal -> row of the current buffer; updated to the new slot
  int32_t* live_next;      // atomic slot counter of the next buffer
  float* resid;
  int32_t* n_iter;
  int32_t* status;
  size_t l2_persist_bytes;  // > 0: launch with a persisting L2 access-policy window over At
  // projection path (algorithm v0): non-null selects it.  Then At := G, Y := P0 = A^T Y (ldy = Np),
  // M := N, Mp := Np, R32in / R32 := the projection rows, part = nstar = nullptr
  const double* ynorm2 = nullptr;
  const float* At_res = nullptr;   // the fp32 atom rows, Mp_res apart, and y (ldy_res): exact ||r|| near eps
  int64_t Mp_res = 0, M_res = 0;
  const float* Y_res = nullptr;
  int64_t ldy_res = 0;
};
cudaError_t launch_update(const UpdateLaunch& L, cudaStream_t st);
// ---- small-batch path: all S iterations in one persistent cooperative kernel (k_small.cu) ----
constexpr int SMALL_MAX_B = 64;            // largest batch the persistent kernel takes
constexpr int SMALL_MAX_CTAS_PER_SM = 8;   // pbest holds SMALL_MAX_B x (SMs x this) partials
bool small_path_supported(int64_t B, int64_t Mp, int32_t S);
// L as for launch_update (k, part, nstar, cstar, R32in, Rb/Rhi/Rlo, rslot_out, slot, live_next unused);
// L.R32 = the residual rows at row b, initialised by launch_batch_init with live0 = nullptr.
// pbest: SMALL_MAX_B x SMs x SMALL_MAX_CTAS_PER_SM float4; bar: one counter, zero at launch.
cudaError_t launch_small(const UpdateLaunch& L, float4* pbest, unsigned int* bar, cudaStream_t st);
cudaError_t launch_densify(const float* X, int64_t ldx, const int32_t* support, int64_t lds,
                           const int32_t* n_iter, int64_t B, int32_t S, int64_t N, float* Xd,
                           int64_t ldxd, cudaStream_t st);

}  // namespace ompb
