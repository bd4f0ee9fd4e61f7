// Device code shared by the per-iteration update kernel (k_update.cu) and the small-batch
// persistent kernel (k_small.cu): the exact FP32 correlation dot, and the per-signal tail of one
// OMP iteration once the atom n* and its correlation c* are known:
//
//  a4  inverse-Cholesky factor append, the paper's algorithm-v0 update:
//        w = A_k^T a_{n*} = [A^T A]_{n*, S_k}
//        z = F_k^T w,  gamma = 1/sqrt(||a_{n*}||^2 - ||z||^2)
//        F_{k+1} = [[F_k, -gamma F_k z], [0, gamma]]                               (Eq. 8)
//        u = F^T A^T y grows by u_new = gamma <r_k, a_{n*}> = gamma c*  (q = A_{k+1} f is orthogonal
//            to span A_k, so q^T y = q^T r_k; pin P9)
//        x = F_{k+1} u   (matrix-vector products only, Eq. 11)
//      F is upper triangular, packed by columns (column j = F[0..j, j] at offset j(j+1)/2), the
//      paper's packed representation.
//
//  a5  residual r_b = y_b - sum_{j<=k} x_j a_{s_j} from gathered atom rows of A^T,
//      ||r_b||, the eps test, and the operand planes of the next screen.
//
// Both kernels run the same instructions in the same order for a signal, so a signal's result does
// not depend on which kernel (i.e. which batch size) processed it.
#pragma once

#include <cuda_bf16.h>
#include <math.h>

#include "omp_internal.cuh"

// optional timeline hook (k_small.cu defines it for its diagnostic trace; a no-op elsewhere)
#ifndef OMP_TAIL_TRACE
#define OMP_TAIL_TRACE(p)
#endif

namespace ompb {

// OMP_V8 = 1: 256-bit atom-row loads in the gather and the chunk-pair ownership that goes with them.
// Off: the probe's 256-bit gather is 2.5 % (c4) / 6 % (c5) faster than its 128-bit one, but in the
// update it lost (c4 -5 %, c5 B = 10^5 -4 %, c3 -5 %, c2 +0.8 %; profiles/r02/ab/ab_v8_r02ad.txt)
#ifndef OMP_V8
#define OMP_V8 0
#endif
// does a CTA of T threads own, per thread, exactly the chunks lane l of warp 0 sums for ||r||^2, in
// that order (so it may sum them in registers)?  Only one-warp CTAs, with the matching ownership.
template <int T, int CH>
__host__ __device__ constexpr bool update_rreg() {
  return T == 32 && (OMP_V8 == 0 || CH % 2 == 0);
}

struct UpdateArgs {
  int32_t k, S;
  int32_t fsm;          // k_update: the packed F_k is staged in shared memory
  float eps;
  int64_t N, M, Mp;
  // selection inputs
  const float2* part;   // screen partials (REFINE)
  int groups;           // screen partial groups per row (Np / SCREEN_GROUP)
  int candcap;          // capacity of the refine's kept-entry list (k_update)
  const float* rslot_in;  // window W of each row of the current buffer (REFINE)
  WinCoef win;          // coefficients of the next window (written to rslot_out)
  const int32_t* nstar; // preselected (SIMT mode)
  const float* cstar;
  // dictionary
  const float* At;      // fp32 atom rows (Np x Mp)
  const float* inv_norm;
  const float* G;       // Gram matrix, row stride ldg
  int64_t ldg;
  // per-signal state
  const float* Y;
  int64_t ldy;
  float* F;
  int64_t ldf;
  float* U;
  int64_t ldu;
  float* X;
  int64_t ldx;
  int32_t* support;
  int64_t lds;
  const float* R32in;   // current residual rows (row = slot)
  float* R32;           // next residual planes (row = new slot)
  __nv_bfloat16* Rb;
  float* Rhi;
  float* Rlo;
  float* rslot_out;
  int32_t* slot;
  int32_t* live_next;   // nullptr: no live-set compaction, the signal keeps row b
  float* resid;
  int32_t* n_iter;
  int32_t* status;
  const double* ynorm2; // projection path: ||y_b||^2 (the residual norm comes from u, reading R22)
  // projection path: the dictionary itself, for the exact residual norm near the eps threshold
  const float* At_res;
  int64_t Mp_res, M_res;
  const float* Y_res;
  int64_t ldy_res;
};

struct Cand {
  float w;
  int n;
  float c;
};

__device__ __forceinline__ bool cand_better(const Cand& a, const Cand& b) {   // is a better than b
  return a.w > b.w || (a.w == b.w && a.n < b.n);
}

__device__ __forceinline__ float tf32_rna_u(float x) {
  uint32_t r;
  asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(r) : "f"(x));
  return __uint_as_float(r & 0xFFFFE000u);
}

__device__ __forceinline__ uint32_t smem_addr(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

// L2 policies: the 64 MB (c4) fp32 atom table is re-read by every signal and should stay in L2;
// y, the residual planes and the factors are streamed once per iteration.
__device__ __forceinline__ uint64_t policy_evict_last() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(p));
  return p;
}
__device__ __forceinline__ uint64_t policy_evict_first() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
  return p;
}
__device__ __forceinline__ float4 ldg_policy(const float4* ptr, uint64_t pol) {
  float4 v;
  asm volatile("ld.global.nc.L1::no_allocate.L2::cache_hint.v4.f32 {%0, %1, %2, %3}, [%4], %5;"
               : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w) : "l"(ptr), "l"(pol));
  return v;
}
// 256-bit load (LDG.E.256 on sm_100a): two adjacent float4 chunks
__device__ __forceinline__ void ldg8_policy(const float* ptr, uint64_t pol, float4& lo, float4& hi) {
  asm volatile("ld.global.nc.L1::no_allocate.L2::cache_hint.v8.f32 {%0, %1, %2, %3, %4, %5, %6, %7}, [%8], %9;"
               : "=f"(lo.x), "=f"(lo.y), "=f"(lo.z), "=f"(lo.w), "=f"(hi.x), "=f"(hi.y), "=f"(hi.z), "=f"(hi.w)
               : "l"(ptr), "l"(pol));
}
__device__ __forceinline__ void stg_policy(float4* ptr, float4 v, uint64_t pol) {
  asm volatile("st.global.L1::no_allocate.L2::cache_hint.v4.f32 [%0], {%1, %2, %3, %4}, %5;"
               ::"l"(ptr), "f"(v.x), "f"(v.y), "f"(v.z), "f"(v.w), "l"(pol) : "memory");
}
__device__ __forceinline__ void stg_policy(uint2* ptr, uint2 v, uint64_t pol) {
  asm volatile("st.global.L1::no_allocate.L2::cache_hint.v2.u32 [%0], {%1, %2}, %3;"
               ::"l"(ptr), "r"(v.x), "r"(v.y), "l"(pol) : "memory");
}

__device__ __forceinline__ void cp_async4(void* dst, const void* src) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"(smem_addr(dst)), "l"(src) : "memory");
}
__device__ __forceinline__ void cp_async16(void* dst, const void* src) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(smem_addr(dst)), "l"(src) : "memory");
}

template <int T>
__device__ __forceinline__ double block_sum_d(double v) {
  __shared__ double redd[T / 32];
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  __syncthreads();
  if ((threadIdx.x & 31) == 0) redd[threadIdx.x >> 5] = v;
  __syncthreads();
  double r = 0.0;
#pragma unroll
  for (int w = 0; w < T / 32; ++w) r += redd[w];
  return r;
}

// one float4 chunk into a partial sum, in the fixed order w, z, y, x
__device__ __forceinline__ float fma4(const float4 r, const float4 a, float s) {
  return fmaf(r.x, a.x, fmaf(r.y, a.y, fmaf(r.z, a.z, fmaf(r.w, a.w, s))));
}

// The exact FP32 correlation c = <r, a_n> of one warp, in one fixed order: lane l owns the float4
// chunks q = l + 32 i; chunk i goes to partial sum i mod 4 while a whole group of four exists, the
// rest to partial 0; then (s0 + s1) + (s2 + s3) and an xor tree over the lanes.  The selection in both
// update paths uses this order (warp_dot and warp_dot_regs below), so they agree bit for bit.
__device__ __forceinline__ float warp_dot(const float4* __restrict__ r4, const float4* __restrict__ a4, int q4,
                                          int lane) {
  // four float4 loads in flight per lane, four partial sums
  float s0 = 0.f, s1 = 0.f, s2 = 0.f, s3 = 0.f;
  int q = lane;
  for (; q + 96 < q4; q += 128) {
    const float4 a0 = __ldg(a4 + q), a1 = __ldg(a4 + q + 32), a2 = __ldg(a4 + q + 64), a3 = __ldg(a4 + q + 96);
    const float4 r0 = r4[q], r1 = r4[q + 32], r2 = r4[q + 64], r3 = r4[q + 96];
    s0 = fma4(r0, a0, s0);
    s1 = fma4(r1, a1, s1);
    s2 = fma4(r2, a2, s2);
    s3 = fma4(r3, a3, s3);
  }
  for (; q < q4; q += 32) s0 = fma4(r4[q], __ldg(a4 + q), s0);
  float acc = (s0 + s1) + (s2 + s3);
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
  return acc;
}

// two such dots (rows a4, b4 against the same r4) with their loads in flight together; each result is
// bit for bit warp_dot's
__device__ __forceinline__ float2 warp_dot2(const float4* __restrict__ r4, const float4* __restrict__ a4,
                                           const float4* __restrict__ b4, int q4, int lane) {
  float s0 = 0.f, s1 = 0.f, s2 = 0.f, s3 = 0.f, t0 = 0.f, t1 = 0.f, t2 = 0.f, t3 = 0.f;
  int q = lane;
  for (; q + 96 < q4; q += 128) {
    const float4 a0 = __ldg(a4 + q), a1 = __ldg(a4 + q + 32), a2 = __ldg(a4 + q + 64), a3 = __ldg(a4 + q + 96);
    const float4 b0 = __ldg(b4 + q), b1 = __ldg(b4 + q + 32), b2 = __ldg(b4 + q + 64), b3 = __ldg(b4 + q + 96);
    const float4 r0 = r4[q], r1 = r4[q + 32], r2 = r4[q + 64], r3 = r4[q + 96];
    s0 = fma4(r0, a0, s0);
    s1 = fma4(r1, a1, s1);
    s2 = fma4(r2, a2, s2);
    s3 = fma4(r3, a3, s3);
    t0 = fma4(r0, b0, t0);
    t1 = fma4(r1, b1, t1);
    t2 = fma4(r2, b2, t2);
    t3 = fma4(r3, b3, t3);
  }
  for (; q < q4; q += 32) {
    const float4 r = r4[q];
    s0 = fma4(r, __ldg(a4 + q), s0);
    t0 = fma4(r, __ldg(b4 + q), t0);
  }
  float x = (s0 + s1) + (s2 + s3), y = (t0 + t1) + (t2 + t3);
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    x += __shfl_xor_sync(0xffffffffu, x, o);
    y += __shfl_xor_sync(0xffffffffu, y, o);
  }
  return make_float2(x, y);
}

// the same dot with the atom's chunks held in registers (areg[i] = chunk lane + 32 i, KC >= chunks)
template <int KC>
__device__ __forceinline__ float warp_dot_regs(const float4* __restrict__ r4, const float4 (&areg)[KC], int q4,
                                               int lane) {
  static_assert(KC % 4 == 0, "KC: groups of four chunks");
  float s0 = 0.f, s1 = 0.f, s2 = 0.f, s3 = 0.f;
#pragma unroll
  for (int i = 0; i < KC; i += 4) {
    const int q = lane + 32 * i;
    if (q + 96 < q4) {
      s0 = fma4(r4[q], areg[i], s0);
      s1 = fma4(r4[q + 32], areg[i + 1], s1);
      s2 = fma4(r4[q + 64], areg[i + 2], s2);
      s3 = fma4(r4[q + 96], areg[i + 3], s3);
    } else {
#pragma unroll
      for (int t = 0; t < 4; ++t)
        if (q + 32 * t < q4) s0 = fma4(r4[q + 32 * t], areg[i + t], s0);
    }
  }
  float acc = (s0 + s1) + (s2 + s3);
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
  return acc;
}

// Per-signal scratch in shared memory for the tail (Sp >= k + 1 entries each).
struct TailSmem {
  float *w, *z, *u, *xs;
  int* ss;
  uint32_t* ro;   // atom row offsets (float4 units) for the gather
  float* red;     // T / 32 floats
  float* pr;      // Mp / 4 floats: per-chunk partials of ||r||^2 (and, with a bf16 plane, Mp / 4 more:
                  // per-chunk partials of ||r - bf16(r)||^2)
  int* bcast;     // one int
};

// a4 + a5 for signal b at iteration k with the selected atom n >= 0 and c* = <r_k, a_n>.
// V0 (the projection path, paper's algorithm v0): the caller passes At := G,
// Y := P0 = A^T Y, M := N, Mp := Np, so the "residual" this computes is the projection vector
// p_{k+1} = A^T r_{k+1} = P0 - sum_j x_j G[s_j, :]; ||r_{k+1}|| = sqrt(||y||^2 - ||u||^2) (reading R22).
// P: atom rows in flight per thread in the gather, ZC: columns per warp in z = F^T w (the
// per-iteration kernel hides latency with 8 CTAs per SM and uses 2 / 2; the persistent small-batch
// kernel has one CTA per signal on the critical path and uses more).  Neither changes the order of
// any floating-point operation, only how far loads and reductions run ahead.
// Preconditions: sm.ss[0..k) = support, sm.u[0..k) = u, visible to every thread.  Every exit is
// uniform over the CTA.  Fb: the packed F_k (global memory, prefetched into L1, or a shared-memory
// copy); Fs_append (nullable): a shared-memory copy that receives the new column as well.  On
// return sm.ss[k] = n* and sm.u[k] = u_new, so a persistent caller's copies stay current.
// rows_sm (nullable): a shared-memory copy of the support's atom rows (row j at rows_sm + j q4,
// j <= k; row k may still be landing by cp.async, waited for here) that the gather reads instead
// of A^T in global memory -- the same values, so the same result.
// FZN: the row sweep keeps FZN (8, or 16 in the one-CTA-per-SM variant) column loads in flight (F_k in
// L1 / L2); FZN = 0: F_k in shared memory, where 4 do,
// and the smaller code keeps more of the kernel in the instruction cache (same FMA order either way).
// ZLANE (only with F_k in shared memory, FZN = 0): z = F^T w thread per column instead of warp per
// column -- the same bits (see the z loop); pays where it frees warps of a small CTA (T <= 64: c5 at 10^4 /
// 10^5 signals +4 %, c2 +5.7 %) and costs the 48-register T = 128 variant spills (c3 -2.7 %).
// ZR: rows of a column whose loads the warp-per-column z keeps in flight (4; 8 in the one-CTA-per-SM
// variant, where F_k of a large S is read from L2 one column group at a time).
template <int T, int CH, int P = 2, int ZC = 2, bool V0 = false, int FZN = 8, bool ZLANE = false, int ZR = 4>
__device__ __forceinline__ void append_residual(const UpdateArgs& a, const int64_t b, const int k, const int n,
                                                const float cst, const TailSmem& sm, const float* Fb,
                                                float* Fs_append, const float4* rows_sm = nullptr,
                                                unsigned long long* trace_t0 = nullptr) {
#ifdef OMP_UPDATE_TRACE
  unsigned long long& upd_t0_ = *trace_t0;   // the caller's phase timer (diagnostic build only)
#endif
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int q4 = (int)(a.Mp >> 2);
  float* w = sm.w;
  float* z = sm.z;
  float* u = sm.u;
  float* xs = sm.xs;
  int* ss = sm.ss;
  uint32_t* ro = sm.ro;

  // ---- a4: factor append --------------------------------------------------------------------------
  const float* grow = a.G + (int64_t)n * a.ldg;
  const float d = grow[n];              // ||a_{n*}||^2 (issued with the w loads, used after z)
  bool dup = false;
  for (int j = tid; j < k; j += T) {
    const int s = ss[j];
    ro[j] = (uint32_t)s * (uint32_t)q4;
    dup |= (s == n);
    w[j] = grow[s];                     // [A^T A]_{n*, s_j}
  }
  if (__syncthreads_or(dup)) {          // re-selection (reading R6)
    if (tid == 0) a.status[b] = OMP_SIG_DEGENERATE;
    return;
  }
  OMP_TAIL_TRACE(0);
  // z_j = F[:, j] . w  (column dots: lane l sums i = l, l + 32, ... <= j, then an xor tree; a warp
  // takes ZC columns at a time so their loads and shuffle reductions overlap -- ZC changes only the
  // interleaving, not any column's arithmetic)
  constexpr int NW = T / 32;
  if constexpr (ZLANE && FZN == 0) {
    // F_k in shared memory: thread per column, the same arithmetic without a shuffle.  Thread j forms the
    // 32 lane partials p_l = sum_{i = l, l+32, ... <= j} F[i, j] w_i (the same FMA chains, from 0) and adds
    // them in the xor tree's pairing: level o pairs the partials of lanes l and l ^ o (o = 16, 8, 4, 2, 1),
    // which is the adjacent-pair tree over the leaves in bit-reversed order.  IEEE addition is
    // commutative, so z_j is bit for bit the warp-per-column result (tests/test_tree_order.py emulates
    // both).  About a third of the instructions and no shuffle latency chain; reads are conflict-free
    // (the column offsets j(j+1)/2 of 32 consecutive j fall in 32 distinct banks).
    for (int j = tid; j < k; j += T) {
      const float* colj = Fb + (int64_t)j * (j + 1) / 2;
      float p[32];                      // p[r] = partial of lane brev5(r)
#pragma unroll
      for (int r = 0; r < 32; ++r) p[r] = 0.f;
      for (int i0 = 0; i0 <= j; i0 += 32) {
#pragma unroll
        for (int r = 0; r < 32; ++r) {
          const int i = i0 + (int)(__brev((unsigned)r) >> 27);
          if (i <= j) p[r] = fmaf(colj[i], w[i], p[r]);
        }
      }
#pragma unroll
      for (int h = 1; h < 32; h <<= 1)  // adjacent pairs, then pairs of pairs, ...
#pragma unroll
        for (int r = 0; r < 32; r += 2 * h) p[r] = p[r] + p[r + h];
      z[j] = p[0];
    }
  } else
  for (int j0 = ZC * warp; j0 < k; j0 += ZC * NW) {
    const float* col[ZC];
    float acc_z[ZC];
#pragma unroll
    for (int c = 0; c < ZC; ++c) {
      col[c] = Fb + (int64_t)(j0 + c) * (j0 + c + 1) / 2;
      acc_z[c] = 0.f;
    }
    const int jl = min(j0 + ZC, k) - 1;   // last column of the group
    int i = lane;
    // long columns (F_k of a large S lives in L2): ZR rows' loads in flight, FMAs in the same order
    for (; i + 32 * (ZR - 1) <= jl; i += 32 * ZR) {
      float cv[ZR][ZC], wv[ZR];
#pragma unroll
      for (int q = 0; q < ZR; ++q) {
        const int ii = i + 32 * q;
        wv[q] = w[ii];
#pragma unroll
        for (int c = 0; c < ZC; ++c) cv[q][c] = (ii <= j0 + c && j0 + c < k) ? col[c][ii] : 0.f;
      }
#pragma unroll
      for (int q = 0; q < ZR; ++q)
#pragma unroll
        for (int c = 0; c < ZC; ++c)
          if (i + 32 * q <= j0 + c && j0 + c < k) acc_z[c] = fmaf(cv[q][c], wv[q], acc_z[c]);
    }
    for (; i <= jl; i += 32) {
      const float wi = w[i];
#pragma unroll
      for (int c = 0; c < ZC; ++c)
        if (i <= j0 + c && j0 + c < k) acc_z[c] = fmaf(col[c][i], wi, acc_z[c]);
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1)
#pragma unroll
      for (int c = 0; c < ZC; ++c) acc_z[c] += __shfl_xor_sync(0xffffffffu, acc_z[c], o);
    if (lane == 0)
#pragma unroll
      for (int c = 0; c < ZC; ++c)
        if (j0 + c < k) z[j0 + c] = acc_z[c];
  }
  __syncthreads();
  OMP_TAIL_TRACE(1);
  // ||z||^2 in one order whatever T is: warp 0's lane l sums z_j^2 for j = l, l + 32, ... ascending,
  // then the xor tree; one barrier broadcasts it.  So a signal's result does not depend on the
  // kernel's block size.
  if (warp == 0) {
    float v = 0.f;
    for (int j = lane; j < k; j += 32) v = fmaf(z[j], z[j], v);
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    if (lane == 0) sm.red[0] = v;
  }
  __syncthreads();
  const float zz = sm.red[0];

  OMP_TAIL_TRACE(2);
  const float delta = d - zz;
  if (!(delta > TAU_F * d)) {           // rank deficiency (reading R6); also catches NaN
    if (tid == 0) a.status[b] = OMP_SIG_DEGENERATE;
    return;
  }
  const float gamma = 1.0f / sqrtf(delta);
  const float unew = gamma * cst;       // gamma <r_k, a_{n*}>
  // v = F_k z and t = F_k u in one pass over F (thread per row; lanes of a warp share column j)
  float* newcol = a.F + b * a.ldf + (int64_t)k * (k + 1) / 2;
  for (int i = tid; i < k; i += T) {
    // four independent partial sums so four column loads are in flight per thread
    float v0 = 0.f, v1 = 0.f, v2 = 0.f, v3 = 0.f, t0 = 0.f, t1 = 0.f, t2 = 0.f, t3 = 0.f;
    int j = i & ~31;
    int o = j * (j + 1) / 2 + i;                  // offset of F[i, j] in the packed columns
    // FZN column loads in flight (F_k of a large S lives in L2, not L1), the FMAs in the same order
    // (column j always goes to partial j mod 4, whatever the blocking)
    if constexpr (FZN > 0) for (; j + FZN <= k; j += FZN) {
      float f[FZN > 0 ? FZN : 1];
#pragma unroll
      for (int q = 0; q < FZN; ++q) {
        f[q] = (j + q >= i) ? Fb[o] : 0.f;
        o += j + q + 1;
      }
#pragma unroll
      for (int g = 0; g < FZN; g += 4) {
        v0 = fmaf(f[g], z[j + g], v0);
        t0 = fmaf(f[g], u[j + g], t0);
        v1 = fmaf(f[g + 1], z[j + g + 1], v1);
        t1 = fmaf(f[g + 1], u[j + g + 1], t1);
        v2 = fmaf(f[g + 2], z[j + g + 2], v2);
        t2 = fmaf(f[g + 2], u[j + g + 2], t2);
        v3 = fmaf(f[g + 3], z[j + g + 3], v3);
        t3 = fmaf(f[g + 3], u[j + g + 3], t3);
      }
    }
    for (; j + 4 <= k; j += 4) {
      const int o1 = o + j + 1, o2 = o1 + j + 2, o3 = o2 + j + 3;
      const float f0 = (j >= i) ? Fb[o] : 0.f;
      const float f1 = (j + 1 >= i) ? Fb[o1] : 0.f;
      const float f2 = (j + 2 >= i) ? Fb[o2] : 0.f;
      const float f3 = (j + 3 >= i) ? Fb[o3] : 0.f;
      o = o3 + j + 4;
      v0 = fmaf(f0, z[j], v0);
      t0 = fmaf(f0, u[j], t0);
      v1 = fmaf(f1, z[j + 1], v1);
      t1 = fmaf(f1, u[j + 1], t1);
      v2 = fmaf(f2, z[j + 2], v2);
      t2 = fmaf(f2, u[j + 2], t2);
      v3 = fmaf(f3, z[j + 3], v3);
      t3 = fmaf(f3, u[j + 3], t3);
    }
    for (; j < k; ++j) {
      const float f = (j >= i) ? Fb[o] : 0.f;
      o += j + 1;
      v0 = fmaf(f, z[j], v0);
      t0 = fmaf(f, u[j], t0);
    }
    const float v = (v0 + v1) + (v2 + v3);
    const float t = (t0 + t1) + (t2 + t3);
    newcol[i] = -gamma * v;                       // -gamma F_k z
    if (Fs_append) Fs_append[(int64_t)k * (k + 1) / 2 + i] = -gamma * v;
    const float xi = fmaf(-gamma * v, unew, t);   // x_i = (F_k u)_i + f_i u_new
    a.X[b * a.ldx + i] = xi;
    xs[i] = xi;
  }
  if (tid == 0) {
    newcol[k] = gamma;
    if (Fs_append) Fs_append[(int64_t)k * (k + 1) / 2 + k] = gamma;
    u[k] = unew;
    const float xk = gamma * unew;
    a.X[b * a.ldx + k] = xk;
    xs[k] = xk;
    ss[k] = n;
    ro[k] = (uint32_t)n * (uint32_t)q4;
    a.U[b * a.ldu + k] = unew;
    a.support[b * a.lds + k] = n;
  }
  if (rows_sm) asm volatile("cp.async.wait_all;" ::: "memory");   // row k of the cache
  __syncthreads();
  OMP_TAIL_TRACE(3);

  // ---- a5: residual r = y - A_S x, ||r||, eps test, next screening operand ------------------------
  // L2-bandwidth bound gather: per group of P rows, every thread issues its P x CH float4 loads before
  // the FMAs (with T * CH == Mp / 4, the benchmark shapes, no load is predicated off).
  const int kk = k + 1;
  const uint64_t keep = policy_evict_last(), stream = policy_evict_first();
  // r = y - sum_j x_j a_{s_j}, in one of two orders fixed by the row width (so every kernel and block
  // size computes a signal the same way):
  //   Mp <= 1024: acc starts at y and takes fmaf(-x_j, a_j, acc), j ascending -- y's loads go out with
  //     the first rows', no round trip of their own after the gather (c5: +5 %, c2 / c3: +1 %);
  //   wider rows: acc = sum_j x_j a_j, j ascending, then r = y - acc (y loaded after the gather: holding
  //     it through the gather costs the wide-row kernels registers, c4: -3 %; profiles/r02/ab)
  // A compile-time choice: both kernels' (T, CH) maps give T x CH = the power of two >= Mp / 4 (>= 32),
  // so T x CH <= 256 <=> Mp <= 1024 in k_update and k_small alike.
  constexpr bool yfirst = T * CH <= 256;
  // Chunk ownership: with OMP_V8 and an even CH (V8) thread t owns the float4 chunk PAIRS t, t + T, ...
  // (one 256-bit load per pair and row), else the chunks t, t + T, ...; qidx(c) = the float4 chunk of slot c.
  // Nothing elementwise depends on it.  ||r||^2 sums its per-chunk partials in ONE order for every
  // kernel and block size: lane l of warp 0 takes chunks l, l + 32, ... ascending (OMP_V8: chunks
  // 2(l + 32 i) + e, i ascending, e = 0, 1), then the xor tree.  A one-warp CTA owns exactly
  // lane l's chunks in that order when V8 (or OMP_V8 = 0) holds, and sums them in registers (RREG).
  constexpr bool V8 = (OMP_V8 != 0) && (CH % 2 == 0);
  constexpr bool RREG = update_rreg<T, CH>();
  auto qidx = [&](int c) -> int { return V8 ? 2 * (tid + (c >> 1) * T) + (c & 1) : tid + c * T; };
  const float* y = a.Y + b * a.ldy;
  const bool yvec = ((reinterpret_cast<uintptr_t>(a.Y) & 15) == 0) && (a.ldy % 4 == 0);
  auto load_y = [&](int c) {
    const int q = qidx(c);
    const int64_t m = (int64_t)q << 2;
    float4 v;
    if (yvec && m + 3 < a.M) {
      v = ldg_policy(reinterpret_cast<const float4*>(y + m), stream);
    } else {
      v.x = m < a.M ? y[m] : 0.f;
      v.y = m + 1 < a.M ? y[m + 1] : 0.f;
      v.z = m + 2 < a.M ? y[m + 2] : 0.f;
      v.w = m + 3 < a.M ? y[m + 3] : 0.f;
    }
    return v;
  };
  float4 acc[CH];
  {
#pragma unroll
    for (int c = 0; c < CH; ++c) {
      const int q = qidx(c);
      if (q >= q4 || !yfirst) {
        acc[c] = make_float4(0.f, 0.f, 0.f, 0.f);
      } else {
        acc[c] = load_y(c);
      }
    }
  }
  const float4* A4 = reinterpret_cast<const float4*>(a.At) + tid;
  {
    // chunk c of this thread exists for every row (T * CH == q4 at the benchmark shapes: no predicate)
    bool has[CH];
#pragma unroll
    for (int c = 0; c < CH; ++c) has[c] = (T * CH == q4) || (qidx(c) < q4);
    // fold (-)x_j times row j into acc, j ascending; rows come P at a time (loads before FMAs)
    const bool full = (T * CH == q4);
    auto fold = [&](const float x, const float4 (&v)[CH]) {
#pragma unroll
      for (int c = 0; c < CH; ++c) {
        if (full || has[c]) {
          acc[c].x = fmaf(x, v[c].x, acc[c].x);
          acc[c].y = fmaf(x, v[c].y, acc[c].y);
          acc[c].z = fmaf(x, v[c].z, acc[c].z);
          acc[c].w = fmaf(x, v[c].w, acc[c].w);
        }
      }
    };
    auto gather = [&](auto load_row) {
      int j = 0;
      for (; j + P <= kk; j += P) {
        float4 v[P][CH];
#pragma unroll
        for (int p = 0; p < P; ++p) load_row(j + p, v[p]);
#pragma unroll
        for (int p = 0; p < P; ++p) fold(yfirst ? -xs[j + p] : xs[j + p], v[p]);
      }
      for (; j < kk; ++j) {
        float4 v[CH];
        load_row(j, v);
        fold(yfirst ? -xs[j] : xs[j], v);
      }
    };
    if (rows_sm) {
      gather([&](int j, float4 (&v)[CH]) {
        const float4* r = rows_sm + (size_t)j * q4;
#pragma unroll
        for (int c = 0; c < CH; ++c) v[c] = has[c] ? r[qidx(c)] : make_float4(0.f, 0.f, 0.f, 0.f);
      });
    } else if (full) {           // every chunk exists: unpredicated loads (measured: the predicated form
                                 // alone doubled the c4 update's time)
      if constexpr (V8) {
        gather([&](int j, float4 (&v)[CH]) {
          const float* r = a.At + ((size_t)ro[j] << 2) + (size_t)tid * 8;
#pragma unroll
          for (int c = 0; c < CH; c += 2) ldg8_policy(r + (size_t)(c >> 1) * T * 8, keep, v[c], v[c + 1]);
        });
      } else {
        gather([&](int j, float4 (&v)[CH]) {
          const float4* r = A4 + ro[j];
#pragma unroll
          for (int c = 0; c < CH; ++c) v[c] = ldg_policy(r + c * T, keep);
        });
      }
    } else {
      gather([&](int j, float4 (&v)[CH]) {
        const float4* r = reinterpret_cast<const float4*>(a.At) + ro[j];
#pragma unroll
        for (int c = 0; c < CH; ++c) v[c] = has[c] ? ldg_policy(r + qidx(c), keep) : make_float4(0.f, 0.f, 0.f, 0.f);
      });
    }
  }
  OMP_TAIL_TRACE(4);
#pragma unroll
  for (int c = 0; c < CH; ++c) {
    const int q = qidx(c);
    if (q < q4) {
      if (!yfirst) {
        const float4 yv = load_y(c);
        acc[c] = make_float4(yv.x - acc[c].x, yv.y - acc[c].y, yv.z - acc[c].z, yv.w - acc[c].w);
      }
      // acc[c] = r
      // ||r||^2: one partial per float4 chunk, summed below in an order that does not depend on T
      // (RREG: the one warp owns its chunks in the summation order -- it sums them itself, below)
      if constexpr (!V0 && !RREG) {
        sm.pr[q] = fmaf(acc[c].x, acc[c].x, fmaf(acc[c].y, acc[c].y, fmaf(acc[c].z, acc[c].z, acc[c].w * acc[c].w)));
        if (a.Rb) {   // the bf16 plane's rounding error, for the next window (exact differences)
          const float4 e = make_float4(acc[c].x - __bfloat162float(__float2bfloat16_rn(acc[c].x)),
                                       acc[c].y - __bfloat162float(__float2bfloat16_rn(acc[c].y)),
                                       acc[c].z - __bfloat162float(__float2bfloat16_rn(acc[c].z)),
                                       acc[c].w - __bfloat162float(__float2bfloat16_rn(acc[c].w)));
          sm.pr[q4 + q] = fmaf(e.x, e.x, fmaf(e.y, e.y, fmaf(e.z, e.z, e.w * e.w)));
        }
      }
    }
  }
  float rr;
  float dn2 = 0.f;                      // ||r - bf16(r)||^2 (bf16 plane only; warp 0)
  if constexpr (V0) {
    // ||r_{k+1}||^2 = ||y||^2 - ||u_{k+1}||^2 (q_j orthonormal, u_j = q_j^T y, pin P9),
    // in FP64.  The u_j carry FP32 errors, so where this estimate is within 1e-5 ||y||^2 of eps^2 the
    // eps decision is taken on the exact ||y - A_S x|| instead (k+1 atom rows, reading R22).
    double uu = 0.0;
    for (int j = tid; j <= k; j += T) uu += (double)u[j] * (double)u[j];
    uu = block_sum_d<T>(uu);
    const double yy = a.ynorm2[b];
    double r2 = fmax(yy - uu, 0.0);
    const double e2 = (double)a.eps * (double)a.eps;
    if (a.eps >= 0.f && fabs(r2 - e2) <= 1e-5 * yy) {
      const float* yr = a.Y_res + b * a.ldy_res;
      double pr = 0.0;
      for (int64_t m = tid; m < a.M_res; m += T) {
        float accm = 0.f;
        for (int j = 0; j <= k; ++j) accm = fmaf(xs[j], a.At_res[(int64_t)ss[j] * a.Mp_res + m], accm);
        const float r = yr[m] - accm;
        pr += (double)r * (double)r;
      }
      r2 = block_sum_d<T>(pr);
    }
    rr = (float)r2;
  } else if constexpr (RREG) {
    // the same order from registers: lane l's chunks, in the summation order, are its acc[0], acc[1], ...
    rr = 0.f;
    float dd = 0.f;
#pragma unroll
    for (int c = 0; c < CH; ++c) {
      if (qidx(c) < q4) {
        const float4 r = acc[c];
        rr += fmaf(r.x, r.x, fmaf(r.y, r.y, fmaf(r.z, r.z, r.w * r.w)));
        if (a.Rb) {
          const float4 e = make_float4(r.x - __bfloat162float(__float2bfloat16_rn(r.x)),
                                       r.y - __bfloat162float(__float2bfloat16_rn(r.y)),
                                       r.z - __bfloat162float(__float2bfloat16_rn(r.z)),
                                       r.w - __bfloat162float(__float2bfloat16_rn(r.w)));
          dd += fmaf(e.x, e.x, fmaf(e.y, e.y, fmaf(e.z, e.z, e.w * e.w)));
        }
      }
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) rr += __shfl_xor_sync(0xffffffffu, rr, o);
    if (a.Rb) {
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) dd += __shfl_xor_sync(0xffffffffu, dd, o);
    }
    dn2 = dd;
  } else {
    __syncthreads();
    rr = 0.f;
    float dd = 0.f;
    if (warp == 0) {                    // lane l: its chunks in the summation order, then the xor tree
      if constexpr (OMP_V8 != 0) {
        for (int q = 2 * lane; q < q4; q += 64) {
          rr += sm.pr[q];
          if (q + 1 < q4) rr += sm.pr[q + 1];
        }
      } else {
        for (int q = lane; q < q4; q += 32) rr += sm.pr[q];
      }
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) rr += __shfl_xor_sync(0xffffffffu, rr, o);
      if (a.Rb) {
        if constexpr (OMP_V8 != 0) {
          for (int q = 2 * lane; q < q4; q += 64) {
            dd += sm.pr[q4 + q];
            if (q + 1 < q4) dd += sm.pr[q4 + q + 1];
          }
        } else {
          for (int q = lane; q < q4; q += 32) dd += sm.pr[q4 + q];
        }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) dd += __shfl_xor_sync(0xffffffffu, dd, o);
      }
    }
    dn2 = dd;
  }
  OMP_TAIL_TRACE(5);
  if (tid == 0) {
    const float rn = sqrtf(rr);
    a.resid[b] = rn;
    a.n_iter[b] = kk;
    int ns = -1;
    if (a.eps >= 0.f && rn <= a.eps) a.status[b] = OMP_SIG_EPS;
    else if (kk == a.S) a.status[b] = OMP_SIG_MAXITER;
    else if (a.live_next) {
      ns = atomicAdd(a.live_next, 1);                                  // next live-set slot
      // the next screen's window: d = ||r - bf16(r)|| rounded up (its FP32 sum of
      // squares is off by < 2^-17 relative: the 1 + 2^-10 margin covers it)
      const float dn = a.Rb ? sqrtf(dn2) * (1.f + 0x1p-10f) : 0.f;
      a.rslot_out[ns] = fmaf(a.win.ca, rn + dn, fmaf(a.win.cd, dn, a.win.cr * rn));
    } else {
      ns = (int)b;                                                     // no compaction: row b
    }
    if (a.slot) a.slot[b] = ns;
    *sm.bcast = ns;
  }
  __syncthreads();
  const int ns = *sm.bcast;
  if (ns < 0) return;                   // finished: no planes for the next screen
  const int64_t ro_out = (int64_t)ns * a.Mp;
#pragma unroll
  for (int c = 0; c < CH; ++c) {
    const int q = qidx(c);
    if (q < q4) {
      const float4 r = acc[c];
      if (a.R32) stg_policy(reinterpret_cast<float4*>(a.R32 + ro_out) + q, r, stream);
      if (a.Rb) {
        __nv_bfloat162 p0 = __floats2bfloat162_rn(r.x, r.y), p1 = __floats2bfloat162_rn(r.z, r.w);
        uint2 pk;
        pk.x = *reinterpret_cast<uint32_t*>(&p0);
        pk.y = *reinterpret_cast<uint32_t*>(&p1);
        stg_policy(reinterpret_cast<uint2*>(a.Rb + ro_out) + q, pk, stream);
      }
      if (a.Rhi) {
        const float4 h = make_float4(tf32_rna_u(r.x), tf32_rna_u(r.y), tf32_rna_u(r.z), tf32_rna_u(r.w));
        reinterpret_cast<float4*>(a.Rhi + ro_out)[q] = h;
        reinterpret_cast<float4*>(a.Rlo + ro_out)[q] = make_float4(r.x - h.x, r.y - h.y, r.z - h.z, r.w - h.w);
      }
    }
  }
}

}  // namespace ompb
