// K0 (dictionary setup), batch init (a1), densify (a6) and the TF32 hi/lo split.
//
// TF32 split (3xTF32): hi = rna_tf32(x) keeps the 11 leading
// significand bits, lo = x - hi is exact in FP32, so hi + lo == x bit for bit and the
// tensor-core products Ahi'Rhi + Ahi'Rlo + Alo'Rhi reproduce an FP32-accurate dot.
#include <math.h>

#include "omp_internal.cuh"

namespace ompb {

__device__ __forceinline__ float tf32_rna(float x) {
  uint32_t r;
  asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(r) : "f"(x));
  return __uint_as_float(r & 0xFFFFE000u);
}

__device__ __forceinline__ double block_sum_double(double v, double* red) {
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  const int w = threadIdx.x >> 5, l = threadIdx.x & 31, nw = blockDim.x >> 5;
  __syncthreads();
  if (l == 0) red[w] = v;
  __syncthreads();
  v = (threadIdx.x < nw) ? red[threadIdx.x] : 0.0;
  if (w == 0)
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  if (threadIdx.x == 0) red[0] = v;
  __syncthreads();
  return red[0];
}

// One CTA per (padded) atom n: copy a_n into row n of At (Np x Mp, zero padded), split it,
// and compute ||a_n|| in FP64 (PAPER.md:46 denominator; App. A).
__global__ void k0_prepare_atoms(const float* __restrict__ A, int64_t M, int64_t N, int64_t lda,
                                 int64_t Mp, float* __restrict__ At, float* __restrict__ At_hi,
                                 float* __restrict__ At_lo, float* __restrict__ inv_norm,
                                 int* bad_zero, int* bad_nonfinite) {
  __shared__ double red[32];
  const int64_t n = blockIdx.x;
  double ss = 0.0;
  bool finite = true;
  for (int64_t m = threadIdx.x; m < Mp; m += blockDim.x) {
    float v = 0.f;
    if (n < N && m < M) {
      v = A[n * lda + m];
      finite &= isfinite(v);
      ss += (double)v * (double)v;
    }
    const float h = tf32_rna(v);
    At[n * Mp + m] = v;
    At_hi[n * Mp + m] = h;
    At_lo[n * Mp + m] = v - h;
  }
  const int any_bad = __syncthreads_or(!finite);
  ss = block_sum_double(ss, red);
  if (threadIdx.x == 0) {
    if (n < N) {
      if (any_bad) atomicMin(bad_nonfinite, (int)n);
      else if (ss == 0.0) atomicMin(bad_zero, (int)n);
      inv_norm[n] = (ss > 0.0 && !any_bad) ? (float)(1.0 / sqrt(ss)) : 0.f;
    } else {
      inv_norm[n] = 0.f;   // padded atoms never win the argmax
    }
  }
}

cudaError_t launch_prepare_atoms(const float* A, int64_t M, int64_t N, int64_t lda, int64_t Mp,
                                 int64_t Np, float* At, float* At_hi, float* At_lo, float* inv_norm,
                                 int* bad_zero, int* bad_nonfinite, cudaStream_t st) {
  k0_prepare_atoms<<<(unsigned)Np, 128, 0, st>>>(A, M, N, lda, Mp, At, At_hi, At_lo, inv_norm,
                                                 bad_zero, bad_nonfinite);
  return cudaGetLastError();
}

__global__ void k_split_rows(const float* __restrict__ R, int64_t ldr, int64_t M, int64_t Mp,
                             float* __restrict__ R_hi, float* __restrict__ R_lo) {
  const int64_t b = blockIdx.x;
  for (int64_t m = threadIdx.x; m < Mp; m += blockDim.x) {
    const float v = m < M ? R[b * ldr + m] : 0.f;
    const float h = tf32_rna(v);
    R_hi[b * Mp + m] = h;
    R_lo[b * Mp + m] = v - h;
  }
}

cudaError_t launch_split_rows(const float* R, int64_t B, int64_t ldr, int64_t M, int64_t Mp,
                              float* R_hi, float* R_lo, cudaStream_t st) {
  if (B == 0) return cudaSuccess;
  k_split_rows<<<(unsigned)B, 128, 0, st>>>(R, ldr, M, Mp, R_hi, R_lo);
  return cudaGetLastError();
}

// a1: x_0 = 0, r_0 = y; eps is tested on r_0 (reading R2);
// support = -1, n_iter = 0.  One CTA per signal.
__global__ void k_batch_init(const float* __restrict__ Y, int64_t ldy, int64_t M, int64_t Mp,
                             int32_t S, float eps, float* __restrict__ R_hi, float* __restrict__ R_lo,
                             float* __restrict__ X, int64_t ldx, int32_t* __restrict__ support,
                             int64_t lds, float* __restrict__ resid, int32_t* __restrict__ n_iter,
                             int32_t* __restrict__ status) {
  __shared__ double red[32];
  const int64_t b = blockIdx.x;
  const float* y = Y + b * ldy;
  float part = 0.f;
  for (int64_t m = threadIdx.x; m < Mp; m += blockDim.x) {
    const float v = m < M ? y[m] : 0.f;
    part = fmaf(v, v, part);
    const float h = tf32_rna(v);
    R_hi[b * Mp + m] = h;
    R_lo[b * Mp + m] = v - h;
  }
  for (int j = threadIdx.x; j < S; j += blockDim.x) {
    X[b * ldx + j] = 0.f;
    support[b * lds + j] = -1;
  }
  const double ss = block_sum_double((double)part, red);
  if (threadIdx.x == 0) {
    const float rn = (float)sqrt(ss);
    n_iter[b] = 0;
    if (!isfinite(ss)) {
      status[b] = OMP_SIG_NAN;
      resid[b] = nanf("");
    } else {
      resid[b] = rn;
      status[b] = (eps >= 0.f && rn <= eps) ? OMP_SIG_EPS : SIG_RUNNING;
    }
  }
}

cudaError_t launch_batch_init(const float* Y, int64_t B, int64_t ldy, int64_t M, int64_t Mp,
                              int32_t S, float eps, float* R_hi, float* R_lo, float* X, int64_t ldx,
                              int32_t* support, int64_t lds, float* resid, int32_t* n_iter,
                              int32_t* status, cudaStream_t st) {
  if (B == 0) return cudaSuccess;
  k_batch_init<<<(unsigned)B, 128, 0, st>>>(Y, ldy, M, Mp, S, eps, R_hi, R_lo, X, ldx, support,
                                            lds, resid, n_iter, status);
  return cudaGetLastError();
}

__global__ void k_densify(const float* __restrict__ X, int64_t ldx, const int32_t* __restrict__ support,
                          int64_t lds, const int32_t* __restrict__ n_iter, int64_t N,
                          float* __restrict__ Xd, int64_t ldxd) {
  const int64_t b = blockIdx.x;
  for (int64_t n = threadIdx.x; n < N; n += blockDim.x) Xd[b * ldxd + n] = 0.f;
  __syncthreads();
  const int k = n_iter[b];
  for (int j = threadIdx.x; j < k; j += blockDim.x) {
    const int s = support[b * lds + j];
    if (s >= 0 && s < N) Xd[b * ldxd + s] = X[b * ldx + j];
  }
}

cudaError_t launch_densify(const float* X, int64_t ldx, const int32_t* support, int64_t lds,
                           const int32_t* n_iter, int64_t B, int32_t S, int64_t N, float* Xd,
                           int64_t ldxd, cudaStream_t st) {
  (void)S;
  if (B == 0) return cudaSuccess;
  k_densify<<<(unsigned)B, 256, 0, st>>>(X, ldx, support, lds, n_iter, N, Xd, ldxd);
  return cudaGetLastError();
}

}  // namespace ompb
