// K0 (dictionary setup), batch init (a1), densify (a6) and the operand planes of K1.
//
// Planes written for every row (atom of A^T, or residual of a signal), padded to Mp with zeros:
//   fp32 copy           (gather in K4, exact re-evaluation in the refine kernel, SIMT GEMM)
//   bf16  = RN(x)       (BF16 tcgen05 screen)
//   tf32 hi = RNA(x), lo = x - hi (exact in FP32)   (3xTF32 tcgen05 screen)
#include <cuda_bf16.h>
#include <math.h>

#include "omp_internal.cuh"

namespace ompb {

__device__ __forceinline__ float tf32_rna(float x) {
  uint32_t r;
  asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(r) : "f"(x));
  return __uint_as_float(r & 0xFFFFE000u);
}

__device__ __forceinline__ void put_planes(int64_t off, float v, float* __restrict__ P32,
                                           __nv_bfloat16* __restrict__ Pb, float* __restrict__ Phi,
                                           float* __restrict__ Plo) {
  if (P32) P32[off] = v;
  if (Pb) Pb[off] = __float2bfloat16_rn(v);
  if (Phi) {
    const float h = tf32_rna(v);
    Phi[off] = h;
    Plo[off] = v - h;
  }
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

// One CTA per (padded) atom n: ||a_n|| in FP64 (PAPER.md:46 denominator; App. A), then
// row n of the FP32 copy (raw a_n, used by the exact re-evaluation, the gather and the Gram matrix)
// and of the screen planes of the NORMALISED atom a_n / ||a_n|| (the screen's correlations are then
// already the normalised |<r, a_n>| / ||a_n|| of PAPER.md:46, App. A "invariant to column norm").
__global__ void k0_prepare_atoms(const float* __restrict__ A, int64_t M, int64_t N, int64_t lda, int64_t Mp,
                                 float* __restrict__ At, __nv_bfloat16* __restrict__ Ab, float* __restrict__ Ahi,
                                 float* __restrict__ Alo, float* __restrict__ norm, float* __restrict__ inv_norm,
                                 int* bad_zero, int* bad_nonfinite, unsigned long long* ea2_max) {
  __shared__ double red[32];
  const int64_t n = blockIdx.x;
  double ss = 0.0;
  bool finite = true;
  if (n < N)
    for (int64_t m = threadIdx.x; m < M; m += blockDim.x) {
      const float v = A[n * lda + m];
      finite &= isfinite(v);
      ss += (double)v * (double)v;
    }
  const int any_bad = __syncthreads_or(!finite);
  ss = block_sum_double(ss, red);
  const bool ok = n < N && ss > 0.0 && !any_bad;
  const float inv = ok ? (float)(1.0 / sqrt(ss)) : 0.f;
  // E_a: ||bf16(a_n * (1/||a_n||)) - a_n / ||a_n|||| in FP64, the screen's atom error
  const double rs = ok ? 1.0 / sqrt(ss) : 0.0;
  double e2 = 0.0;
  for (int64_t m = threadIdx.x; m < Mp; m += blockDim.x) {
    const float v = (n < N && m < M) ? A[n * lda + m] : 0.f;
    At[n * Mp + m] = v;
    put_planes(n * Mp + m, v * inv, nullptr, Ab, Ahi, Alo);
    if (Ab) {
      const double d = (double)__bfloat162float(__float2bfloat16_rn(v * inv)) - (double)v * rs;
      e2 += d * d;
    }
  }
  if (Ab && ea2_max) {
    e2 = block_sum_double(e2, red);
    if (threadIdx.x == 0 && n < N) atomicMax(ea2_max, (unsigned long long)__double_as_longlong(e2));
  }
  if (threadIdx.x == 0) {
    if (n < N) {
      if (any_bad) atomicMin(bad_nonfinite, (int)n);
      else if (ss == 0.0) atomicMin(bad_zero, (int)n);
    }
    inv_norm[n] = inv;                 // padded atoms: 0, they never win the argmax
    norm[n] = ok ? (float)sqrt(ss) : 0.f;
  }
}

cudaError_t launch_prepare_atoms(const float* A, int64_t M, int64_t N, int64_t lda, int64_t Mp, int64_t Np,
                                 float* At, void* At_bf16, float* At_hi, float* At_lo, float* norm,
                                 float* inv_norm, int* bad_zero, int* bad_nonfinite, unsigned long long* ea2_max,
                                 cudaStream_t st) {
  k0_prepare_atoms<<<(unsigned)Np, 128, 0, st>>>(A, M, N, lda, Mp, At, (__nv_bfloat16*)At_bf16, At_hi, At_lo,
                                                 norm, inv_norm, bad_zero, bad_nonfinite, ea2_max);
  return cudaGetLastError();
}

__global__ void k_make_planes(const float* __restrict__ R, int64_t ldr, int64_t M, int64_t Mp,
                              float* __restrict__ R32, __nv_bfloat16* __restrict__ Rb, float* __restrict__ Rhi,
                              float* __restrict__ Rlo) {
  const int64_t b = blockIdx.x;
  for (int64_t m = threadIdx.x; m < Mp; m += blockDim.x)
    put_planes(b * Mp + m, m < M ? R[b * ldr + m] : 0.f, R32, Rb, Rhi, Rlo);
}

cudaError_t launch_make_planes(const float* R, int64_t B, int64_t ldr, int64_t M, int64_t Mp, float* R32,
                               void* Rb, float* R_hi, float* R_lo, cudaStream_t st) {
  if (B == 0) return cudaSuccess;
  k_make_planes<<<(unsigned)B, 128, 0, st>>>(R, ldr, M, Mp, R32, (__nv_bfloat16*)Rb, R_hi, R_lo);
  return cudaGetLastError();
}

// a1: x_0 = 0, r_0 = y; eps is tested on r_0 (reading R2);
// support = -1, n_iter = 0.  One CTA per signal.  A signal that is still running takes the next
// slot of the live set (atomic counter live0): its planes go to that row, so the first correlation
// only covers running signals (live-set compaction).
__global__ void k_batch_init(const float* __restrict__ Y, int64_t ldy, int64_t M, int64_t Mp, int32_t S, float eps,
                             float* __restrict__ R32, __nv_bfloat16* __restrict__ Rb, float* __restrict__ Rhi,
                             float* __restrict__ Rlo, float* __restrict__ X, int64_t ldx,
                             int32_t* __restrict__ support, int64_t lds, float* __restrict__ resid,
                             int32_t* __restrict__ n_iter, int32_t* __restrict__ status, int32_t* __restrict__ slot,
                             int32_t* __restrict__ live0, float* __restrict__ rslot, double* __restrict__ ynorm2,
                             WinCoef win) {
  __shared__ double red[32];
  __shared__ int s_slot;
  const int64_t b = blockIdx.x;
  const float* y = Y + b * ldy;
  float part = 0.f, dpart = 0.f;
  for (int64_t m = threadIdx.x; m < M; m += blockDim.x) {
    const float v = y[m];
    part = fmaf(v, v, part);
    if (Rb) {                 // the bf16 plane's rounding error (exact difference), for the window
      const float d = v - __bfloat162float(__float2bfloat16_rn(v));
      dpart = fmaf(d, d, dpart);
    }
  }
  for (int j = threadIdx.x; j < S; j += blockDim.x) {
    X[b * ldx + j] = 0.f;
    support[b * lds + j] = -1;
  }
  const double ss = block_sum_double((double)part, red);
  const double dd = (Rb && live0) ? block_sum_double((double)dpart, red) : 0.0;
  if (threadIdx.x == 0) {
    const float rn = (float)sqrt(ss);
    if (ynorm2) ynorm2[b] = ss;
    n_iter[b] = 0;
    int st;
    if (!isfinite(ss)) {
      st = OMP_SIG_NAN;
      resid[b] = nanf("");
    } else {
      resid[b] = rn;
      st = (eps >= 0.f && rn <= eps) ? OMP_SIG_EPS : SIG_RUNNING;
    }
    status[b] = st;
    s_slot = -1;
    if (st == SIG_RUNNING) {
      if (live0) {
        s_slot = atomicAdd(live0, 1);
        // the first screen's window W_b; d rounded up over its FP32 partial sums
        const float dn = (float)sqrt(dd) * (1.f + 0x1p-10f);
        rslot[s_slot] = fmaf(win.ca, rn + dn, fmaf(win.cd, dn, win.cr * rn));
      } else {
        s_slot = (int)b;                  // small-batch path: no compaction
      }
    }
    if (slot) slot[b] = s_slot;
  }
  __syncthreads();
  const int sl = s_slot;
  if (sl < 0) return;
  for (int64_t m = threadIdx.x; m < Mp; m += blockDim.x)
    put_planes((int64_t)sl * Mp + m, m < M ? y[m] : 0.f, R32, Rb, Rhi, Rlo);
}

cudaError_t launch_batch_init(const float* Y, int64_t B, int64_t ldy, int64_t M, int64_t Mp, int32_t S,
                              float eps, float* R32, void* Rb, float* R_hi, float* R_lo, float* X, int64_t ldx,
                              int32_t* support, int64_t lds, float* resid, int32_t* n_iter, int32_t* status,
                              int32_t* slot, int32_t* live0, float* rslot, cudaStream_t st, double* ynorm2,
                              WinCoef win) {
  if (B == 0) return cudaSuccess;
  k_batch_init<<<(unsigned)B, 128, 0, st>>>(Y, ldy, M, Mp, S, eps, R32, (__nv_bfloat16*)Rb, R_hi, R_lo, X, ldx,
                                            support, lds, resid, n_iter, status, slot, live0, rslot, ynorm2, win);
  return cudaGetLastError();
}

// Projection path, after the last iteration: the exact ||y_b - A_S x_b|| from gathered
// atom rows, replacing the sqrt(||y||^2 - ||u||^2) the iterations used for the eps test (reading R22).
__global__ void __launch_bounds__(256) k_final_resid(const float* __restrict__ Y, int64_t ldy, int64_t M,
                                                     const float* __restrict__ At, int64_t Mp,
                                                     const float* __restrict__ X, int64_t ldx,
                                                     const int32_t* __restrict__ support, int64_t lds,
                                                     const int32_t* __restrict__ n_iter,
                                                     const int32_t* __restrict__ status, float* __restrict__ resid) {
  __shared__ double red[32];
  __shared__ float xs[MAX_S];
  __shared__ int64_t rows[MAX_S];
  const int64_t b = blockIdx.x;
  const int k = n_iter[b];
  if (k == 0 || status[b] == OMP_SIG_NAN) return;   // ||r|| = ||y|| (init) or NaN
  for (int j = threadIdx.x; j < k; j += blockDim.x) {
    xs[j] = X[b * ldx + j];
    rows[j] = (int64_t)support[b * lds + j] * Mp;
  }
  __syncthreads();
  const float* y = Y + b * ldy;
  double part = 0.0;
  // float4 columns of the gathered rows, four rows' loads in flight per step
  for (int64_t m0 = (int64_t)threadIdx.x * 4; m0 < M; m0 += (int64_t)blockDim.x * 4) {
    float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
    int j = 0;
    for (; j + 4 <= k; j += 4) {
      float4 v[4];
#pragma unroll
      for (int q = 0; q < 4; ++q) v[q] = __ldg(reinterpret_cast<const float4*>(At + rows[j + q] + m0));
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        const float x = xs[j + q];
        acc.x = fmaf(x, v[q].x, acc.x);
        acc.y = fmaf(x, v[q].y, acc.y);
        acc.z = fmaf(x, v[q].z, acc.z);
        acc.w = fmaf(x, v[q].w, acc.w);
      }
    }
    for (; j < k; ++j) {
      const float4 v = __ldg(reinterpret_cast<const float4*>(At + rows[j] + m0));
      const float x = xs[j];
      acc.x = fmaf(x, v.x, acc.x);
      acc.y = fmaf(x, v.y, acc.y);
      acc.z = fmaf(x, v.z, acc.z);
      acc.w = fmaf(x, v.w, acc.w);
    }
    const float a4[4] = {acc.x, acc.y, acc.z, acc.w};
#pragma unroll
    for (int q = 0; q < 4; ++q)
      if (m0 + q < M) {
        const float r = y[m0 + q] - a4[q];
        part += (double)r * (double)r;
      }
  }
  const double ss = block_sum_double(part, red);
  if (threadIdx.x == 0) resid[b] = (float)sqrt(ss);
}

cudaError_t launch_final_resid(const float* Y, int64_t B, int64_t ldy, int64_t M, const float* At, int64_t Mp,
                               const float* X, int64_t ldx, const int32_t* support, int64_t lds,
                               const int32_t* n_iter, const int32_t* status, float* resid, cudaStream_t st) {
  if (B == 0) return cudaSuccess;
  k_final_resid<<<(unsigned)B, 256, 0, st>>>(Y, ldy, M, At, Mp, X, ldx, support, lds, n_iter, status, resid);
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
