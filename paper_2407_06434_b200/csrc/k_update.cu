// K3: inverse-Cholesky factor append + coefficients, and
// K4 (a5): residual gather r = y - A_S x, ||r||, eps mask, TF32 hi/lo planes of r.
//
// K3 follows the paper's algorithm-v0 factor update:
//   w = A_k^T a_{n*} = [A^T A]_{n*, S_k}    (Gram entries)
//   z = F_k^T w,  gamma = 1/sqrt(||a_{n*}||^2 - ||z||^2)
//   F_{k+1} = [[F_k, -gamma F_k z], [0, gamma]]                               (Eq. 8)
//   u = F^T A^T y grows by u_new = f^T A_{k+1}^T y = gamma a_{n*}^T r_k = gamma c*
//     (the new basis vector q = A_{k+1} f is orthogonal to span A_k, so q^T y = q^T r_k; pin P9)
//   x = F_{k+1} u  (matrix-vector products only, Eq. 11)
// F is upper triangular and packed by columns (column j = F[0..j, j] at offset j(j+1)/2),
// the paper's packed representation applied to the factor, so the
// leading block is a contiguous prefix and appending a column is a contiguous write.
// Every live signal is at the same k (= iteration), so k is a kernel argument.
#include <cuda_bf16.h>
#include <math.h>

#include "omp_internal.cuh"

namespace ompb {

__device__ __forceinline__ float tf32_rna_u(float x) {
  uint32_t r;
  asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(r) : "f"(x));
  return __uint_as_float(r & 0xFFFFE000u);
}

template <int T>
__device__ __forceinline__ float block_sum(float v, float* red) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  __syncthreads();
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = v;
  __syncthreads();
  float r = 0.f;
#pragma unroll
  for (int w = 0; w < T / 32; ++w) r += red[w];
  return r;
}

template <int T>
__global__ void __launch_bounds__(T) k3_factor_append(
    int32_t k, const int32_t* __restrict__ nstar, const float* __restrict__ cstar, const float* __restrict__ G,
    int64_t ldg, float* __restrict__ F, int64_t ldf,
    float* __restrict__ U, int64_t ldu, float* __restrict__ X, int64_t ldx,
    int32_t* __restrict__ support, int64_t lds, int32_t* __restrict__ status) {
  const int64_t b = blockIdx.x;
  if (status[b] != SIG_RUNNING) return;
  const int n = nstar[b];
  if (n < 0) {   // exhausted residual or non-finite correlations (K2)
    if (threadIdx.x == 0) status[b] = (n == SEL_NAN) ? OMP_SIG_NAN : OMP_SIG_DEGENERATE;
    return;
  }
  __shared__ float w[MAX_S], z[MAX_S], u[MAX_S];
  __shared__ float red[T / 32];
  const float* grow = G + (int64_t)n * ldg;
  bool dup = false;
  for (int j = threadIdx.x; j < k; j += T) {
    const int s = support[b * lds + j];
    dup |= (s == n);
    w[j] = grow[s];                     // [A^T A]_{n*, s_j}
    u[j] = U[b * ldu + j];
  }
  if (__syncthreads_or(dup)) {          // re-selection (reading R6)
    if (threadIdx.x == 0) status[b] = OMP_SIG_DEGENERATE;
    return;
  }
  float* Fb = F + b * ldf;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  // z_j = F[:, j] . w  (column dot, one warp per column, coalesced)
  for (int j = warp; j < k; j += T / 32) {
    const float* col = Fb + (int64_t)j * (j + 1) / 2;
    float acc = 0.f;
    for (int i = lane; i <= j; i += 32) acc = fmaf(col[i], w[i], acc);
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
    if (lane == 0) z[j] = acc;
  }
  __syncthreads();
  float zz = 0.f;
  for (int j = threadIdx.x; j < k; j += T) zz = fmaf(z[j], z[j], zz);
  zz = block_sum<T>(zz, red);
  const float d = grow[n];              // ||a_{n*}||^2
  const float delta = d - zz;
  if (!(delta > TAU_F * d)) {           // rank deficiency (reading R6); also catches NaN
    if (threadIdx.x == 0) status[b] = OMP_SIG_DEGENERATE;
    return;
  }
  const float gamma = 1.0f / sqrtf(delta);
  const float unew = gamma * cstar[b];  // gamma <r_k, a_{n*}>
  // v = F_k z and t = F_k u in one pass over F (thread per row, coalesced per column)
  float* newcol = Fb + (int64_t)k * (k + 1) / 2;
  for (int i = threadIdx.x; i < k; i += T) {
    float v = 0.f, t = 0.f;
    // lanes of a warp walk the same column j together (i & ~31 = warp's first row)
    for (int j = i & ~31; j < k; ++j) {
      const float f = (j >= i) ? Fb[(int64_t)j * (j + 1) / 2 + i] : 0.f;
      v = fmaf(f, z[j], v);
      t = fmaf(f, u[j], t);
    }
    newcol[i] = -gamma * v;                       // -gamma F_k z
    X[b * ldx + i] = fmaf(-gamma * v, unew, t);   // x_i = (F_k u)_i + f_i u_new
  }
  if (threadIdx.x == 0) {
    newcol[k] = gamma;
    X[b * ldx + k] = gamma * unew;
    U[b * ldu + k] = unew;
    support[b * lds + k] = n;
  }
}

cudaError_t launch_factor_append(int32_t k, int64_t B, const int32_t* nstar, const float* cstar, const float* G,
                                 int64_t ldg, float* F, int64_t ldf, float* u, int64_t ldu, float* X, int64_t ldx,
                                 int32_t* support, int64_t lds, int32_t* status, cudaStream_t st) {
  if (B == 0) return cudaSuccess;
  k3_factor_append<128><<<(unsigned)B, 128, 0, st>>>(k, nstar, cstar, G, ldg, F, ldf, u, ldu, X, ldx, support, lds,
                                                     status);
  return cudaGetLastError();
}

// ---------------------------------------------------------------------------------------
// K4: r_b = y_b - sum_{j<=k} x_j a_{s_j}, gathered atom rows of A^T.
// Thread t owns CH float4 chunks of r (m = 4(t + c T)); atoms are streamed in the outer
// loop so the CH loads of one atom row are independent (memory-level parallelism).
// ---------------------------------------------------------------------------------------
template <int T, int CH>
__global__ void __launch_bounds__(T) k4_residual(
    int32_t k, int32_t S, float eps, const float* __restrict__ Y, int64_t ldy, int64_t M, int64_t Mp,
    const float* __restrict__ At, const float* __restrict__ X, int64_t ldx,
    const int32_t* __restrict__ support, int64_t lds, float* __restrict__ R32, __nv_bfloat16* __restrict__ Rb,
    float* __restrict__ R_hi, float* __restrict__ R_lo, float* __restrict__ resid, int32_t* __restrict__ n_iter,
    int32_t* __restrict__ status, bool yvec) {
  const int64_t b = blockIdx.x;
  if (status[b] != SIG_RUNNING) return;
  __shared__ float xs[MAX_S];
  __shared__ int ss[MAX_S];
  __shared__ float red[T / 32];
  const int kk = k + 1;
  for (int j = threadIdx.x; j < kk; j += T) {
    xs[j] = X[b * ldx + j];
    ss[j] = support[b * lds + j];
  }
  __syncthreads();
  const int64_t q4 = Mp >> 2;   // float4 chunks per row
  float4 acc[CH];
#pragma unroll
  for (int c = 0; c < CH; ++c) acc[c] = make_float4(0.f, 0.f, 0.f, 0.f);
  const float4* A4 = reinterpret_cast<const float4*>(At);
#pragma unroll 2
  for (int j = 0; j < kk; ++j) {
    const float xj = xs[j];
    const float4* row = A4 + (int64_t)ss[j] * q4;
#pragma unroll
    for (int c = 0; c < CH; ++c) {
      const int64_t q = threadIdx.x + (int64_t)c * T;
      if (q < q4) {
        const float4 a = __ldg(row + q);
        acc[c].x = fmaf(xj, a.x, acc[c].x);
        acc[c].y = fmaf(xj, a.y, acc[c].y);
        acc[c].z = fmaf(xj, a.z, acc[c].z);
        acc[c].w = fmaf(xj, a.w, acc[c].w);
      }
    }
  }
  const float* y = Y + b * ldy;
  float part = 0.f;
  float4* R4 = reinterpret_cast<float4*>(R32 + b * Mp);
#pragma unroll
  for (int c = 0; c < CH; ++c) {
    const int64_t q = threadIdx.x + (int64_t)c * T;
    if (q < q4) {
      const int64_t m = q << 2;
      float4 yv;
      if (yvec && m + 3 < M) {
        yv = __ldcs(reinterpret_cast<const float4*>(y + m));
      } else {
        yv.x = m < M ? y[m] : 0.f;
        yv.y = m + 1 < M ? y[m + 1] : 0.f;
        yv.z = m + 2 < M ? y[m + 2] : 0.f;
        yv.w = m + 3 < M ? y[m + 3] : 0.f;
      }
      float4 r = make_float4(yv.x - acc[c].x, yv.y - acc[c].y, yv.z - acc[c].z, yv.w - acc[c].w);
      part = fmaf(r.x, r.x, fmaf(r.y, r.y, fmaf(r.z, r.z, fmaf(r.w, r.w, part))));
      R4[q] = r;
      if (Rb) {
        __nv_bfloat162 p0 = __floats2bfloat162_rn(r.x, r.y), p1 = __floats2bfloat162_rn(r.z, r.w);
        uint2 pk;
        pk.x = *reinterpret_cast<uint32_t*>(&p0);
        pk.y = *reinterpret_cast<uint32_t*>(&p1);
        reinterpret_cast<uint2*>(Rb + b * Mp)[q] = pk;
      }
      if (R_hi) {
        const float4 h = make_float4(tf32_rna_u(r.x), tf32_rna_u(r.y), tf32_rna_u(r.z), tf32_rna_u(r.w));
        reinterpret_cast<float4*>(R_hi + b * Mp)[q] = h;
        reinterpret_cast<float4*>(R_lo + b * Mp)[q] = make_float4(r.x - h.x, r.y - h.y, r.z - h.z, r.w - h.w);
      }
    }
  }
  const float rr = block_sum<T>(part, red);
  if (threadIdx.x == 0) {
    const float rn = sqrtf(rr);
    resid[b] = rn;
    n_iter[b] = kk;
    if (eps >= 0.f && rn <= eps) status[b] = OMP_SIG_EPS;
    else if (kk == S) status[b] = OMP_SIG_MAXITER;
  }
}

template <int T, int CH>
static void launch_k4(int32_t k, int32_t S, float eps, int64_t B, const float* Y, int64_t ldy, int64_t M,
                      int64_t Mp, const float* At, const float* X, int64_t ldx, const int32_t* support,
                      int64_t lds, float* R32, void* Rb, float* R_hi, float* R_lo, float* resid, int32_t* n_iter,
                      int32_t* status, bool yvec, cudaStream_t st) {
  k4_residual<T, CH><<<(unsigned)B, T, 0, st>>>(k, S, eps, Y, ldy, M, Mp, At, X, ldx, support, lds, R32,
                                                (__nv_bfloat16*)Rb, R_hi, R_lo, resid, n_iter, status, yvec);
}

cudaError_t launch_residual(int32_t k, int32_t S, float eps, int64_t B, const float* Y, int64_t ldy,
                            int64_t M, int64_t Mp, const float* At, const float* X, int64_t ldx,
                            const int32_t* support, int64_t lds, float* R32, void* Rb, float* R_hi, float* R_lo,
                            float* resid, int32_t* n_iter, int32_t* status, cudaStream_t st) {
  if (B == 0) return cudaSuccess;
  const bool yvec = ((reinterpret_cast<uintptr_t>(Y) & 15) == 0) && (ldy % 4 == 0);
  const int64_t q4 = Mp / 4;
  if (q4 <= 32)
    launch_k4<32, 1>(k, S, eps, B, Y, ldy, M, Mp, At, X, ldx, support, lds, R32, Rb, R_hi, R_lo, resid, n_iter, status, yvec, st);
  else if (q4 <= 128)
    launch_k4<128, 1>(k, S, eps, B, Y, ldy, M, Mp, At, X, ldx, support, lds, R32, Rb, R_hi, R_lo, resid, n_iter, status, yvec, st);
  else if (q4 <= 256)
    launch_k4<128, 2>(k, S, eps, B, Y, ldy, M, Mp, At, X, ldx, support, lds, R32, Rb, R_hi, R_lo, resid, n_iter, status, yvec, st);
  else if (q4 <= 512)
    launch_k4<128, 4>(k, S, eps, B, Y, ldy, M, Mp, At, X, ldx, support, lds, R32, Rb, R_hi, R_lo, resid, n_iter, status, yvec, st);
  else if (q4 <= 1024)
    launch_k4<128, 8>(k, S, eps, B, Y, ldy, M, Mp, At, X, ldx, support, lds, R32, Rb, R_hi, R_lo, resid, n_iter, status, yvec, st);
  else if (q4 <= 2048)
    launch_k4<256, 8>(k, S, eps, B, Y, ldy, M, Mp, At, X, ldx, support, lds, R32, Rb, R_hi, R_lo, resid, n_iter, status, yvec, st);
  else
    return cudaErrorNotSupported;   // M > 8192
  return cudaGetLastError();
}

}  // namespace ompb
