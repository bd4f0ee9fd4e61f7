// Internal declarations shared by the library's translation units (not part of the ABI).
#pragma once

#include <cuda.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include "omp_b200.h"

namespace ompb {

// per-signal running state; finished signals hold an ompSigStatus_t (>= 0)
constexpr int32_t SIG_RUNNING = -1;
// K2 -> K3 selection codes besides an atom index
constexpr int32_t SEL_DEGENERATE = -1;   // maximum correlation is 0 (exhausted residual)
constexpr int32_t SEL_NAN = -2;          // a correlation was not finite
// factor-append pivot threshold: ||a||^2 - ||z||^2 <= TAU_F * ||a||^2 -> DEGENERATE
constexpr float TAU_F = 1e-5f;

constexpr int K_TILE = 32;     // K padding of every plane (one 128-byte TMA/UMMA row)
constexpr int N_TILE = 256;    // atom padding (UMMA N of the correlation kernel)
constexpr int MAX_S = 512;

inline int64_t round_up(int64_t a, int64_t b) { return (a + b - 1) / b * b; }

// Row-major fp32 planes: element (row, k) at base[row * ld + k].
struct Planes {
  const float* hi;
  const float* lo;
  int64_t rows;
  int64_t ld;     // row stride in floats (multiple of K_TILE)
};

// Correlation C[b, n] = sum_k R[b, k] * At[n, k], R and At K-major.
//   mode OMP_CORR_FP32_SIMT : FP32 FFMA on R = hi + lo, At = hi + lo (exact sums)
//   mode OMP_CORR_3XTF32    : tcgen05 kind::tf32, Ahi'Rhi + Ahi'Rlo + Alo'Rhi
// rows of C >= R.rows are not written; columns n in [0, At.rows) are written.
cudaError_t launch_corr_simt(const Planes& R, const Planes& At, int64_t K, float* C, int64_t ldc,
                             cudaStream_t st);
// returns cudaErrorNotSupported if the tensor-core kernel cannot be used for this shape
cudaError_t launch_corr_tc(const Planes& R, const Planes& At, int64_t K, float* C, int64_t ldc,
                           cudaStream_t st);

// K0: atoms -> FP32 copy At (Np x Mp), hi/lo planes, 1/||a_n||; bad_col = min offending column
cudaError_t launch_prepare_atoms(const float* A, int64_t M, int64_t N, int64_t lda, int64_t Mp,
                                 int64_t Np, float* At, float* At_hi, float* At_lo, float* inv_norm,
                                 int* bad_zero, int* bad_nonfinite, cudaStream_t st);
// plain row-major planes of an arbitrary row-major fp32 matrix (for ompCorrelate)
cudaError_t launch_split_rows(const float* R, int64_t B, int64_t ldr, int64_t M, int64_t Mp,
                              float* R_hi, float* R_lo, cudaStream_t st);
// a1: batch init
cudaError_t launch_batch_init(const float* Y, int64_t B, int64_t ldy, int64_t M, int64_t Mp,
                              int32_t S, float eps, float* R_hi, float* R_lo, float* X, int64_t ldx,
                              int32_t* support, int64_t lds, float* resid, int32_t* n_iter,
                              int32_t* status, cudaStream_t st);
// a3 (K2): n*_b = lowest n maximising |C[b,n]| * inv_norm[n]
cudaError_t launch_select(const float* C, int64_t ldc, int64_t B, int64_t N, const float* inv_norm,
                          const int32_t* status, int32_t* nstar, cudaStream_t st);
// a4 (K3): inverse-Cholesky factor append + coefficients
cudaError_t launch_factor_append(int32_t k, int64_t B, const int32_t* nstar, const float* G,
                                 int64_t ldg, const float* P0, int64_t ldp, float* F, int64_t ldf,
                                 float* u, int64_t ldu, float* X, int64_t ldx, int32_t* support,
                                 int64_t lds, int32_t* status, cudaStream_t st);
// a5 (K4): residual gather + norm + eps mask + planes
cudaError_t launch_residual(int32_t k, int32_t S, float eps, int64_t B, const float* Y, int64_t ldy,
                            int64_t M, int64_t Mp, const float* At, const float* X, int64_t ldx,
                            const int32_t* support, int64_t lds, float* R_hi, float* R_lo,
                            float* resid, int32_t* n_iter, int32_t* status, cudaStream_t st);
cudaError_t launch_densify(const float* X, int64_t ldx, const int32_t* support, int64_t lds,
                           const int32_t* n_iter, int64_t B, int32_t S, int64_t N, float* Xd,
                           int64_t ldxd, cudaStream_t st);

}  // namespace ompb
