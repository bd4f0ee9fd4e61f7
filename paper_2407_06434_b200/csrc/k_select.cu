// K2: fused normalisation + argmax over one correlation row,
//   n*_b = lowest n maximising |C[b,n]| / ||a_n||            (Sec. 3.4)
// in a single pass: no |C| temporary, float4 streaming loads of C, warp
// shuffles, ties to the lowest index (reading R4).  HBM-bound: 4N bytes per live signal.
#include "omp_internal.cuh"

namespace ompb {

struct Best {
  float v;
  int i;
};

__device__ __forceinline__ Best better(Best a, Best b) {
  return (b.v > a.v || (b.v == a.v && b.i < a.i)) ? b : a;
}

template <int THREADS>
__global__ void __launch_bounds__(THREADS) k2_select(const float* __restrict__ C, int64_t ldc, int64_t N,
                                                     const float* __restrict__ inv_norm,
                                                     const int32_t* __restrict__ status,
                                                     const int32_t* __restrict__ slot,
                                                     int32_t* __restrict__ nstar, float* __restrict__ cstar,
                                                     bool vec) {
  const int64_t b = blockIdx.x;
  if (status[b] != SIG_RUNNING) return;
  const float* c = C + (int64_t)slot[b] * ldc;   // the signal's row in the live set
  Best best{-1.f, 0x7fffffff};
  bool nan_seen = false;
  if (vec) {
    const int64_t n4 = N >> 2;
    const float4* c4 = reinterpret_cast<const float4*>(c);
    const float4* w4 = reinterpret_cast<const float4*>(inv_norm);
#pragma unroll 4
    for (int64_t q = threadIdx.x; q < n4; q += THREADS) {
      const float4 x = __ldcs(c4 + q);
      const float4 w = __ldg(w4 + q);
      const int n = (int)(q << 2);
      nan_seen |= isnan(x.x) | isnan(x.y) | isnan(x.z) | isnan(x.w);
      const float v0 = fabsf(x.x) * w.x, v1 = fabsf(x.y) * w.y;
      const float v2 = fabsf(x.z) * w.z, v3 = fabsf(x.w) * w.w;
      if (v0 > best.v) best = {v0, n};
      if (v1 > best.v) best = {v1, n + 1};
      if (v2 > best.v) best = {v2, n + 2};
      if (v3 > best.v) best = {v3, n + 3};
    }
    for (int64_t n = (n4 << 2) + threadIdx.x; n < N; n += THREADS) {
      const float x = c[n];
      nan_seen |= isnan(x);
      const float v = fabsf(x) * inv_norm[n];
      if (v > best.v) best = {v, (int)n};
    }
  } else {
    for (int64_t n = threadIdx.x; n < N; n += THREADS) {
      const float x = c[n];
      nan_seen |= isnan(x);
      const float v = fabsf(x) * inv_norm[n];
      if (v > best.v) best = {v, (int)n};
    }
  }
  // warp then block reduction, lowest index on equal values
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    Best other{__shfl_xor_sync(0xffffffffu, best.v, o), __shfl_xor_sync(0xffffffffu, best.i, o)};
    best = better(best, other);
  }
  __shared__ Best red[THREADS / 32];
  const int any_nan = __syncthreads_or(nan_seen);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = best;
  __syncthreads();
  if (threadIdx.x == 0) {
    Best r = red[0];
#pragma unroll
    for (int w = 1; w < THREADS / 32; ++w) r = better(r, red[w]);
    nstar[b] = any_nan ? SEL_NAN : (r.v > 0.f ? r.i : SEL_DEGENERATE);
    cstar[b] = (!any_nan && r.v > 0.f) ? c[r.i] : 0.f;   // signed <r, a_{n*}>
  }
}

cudaError_t launch_select(const float* C, int64_t ldc, int64_t B, int64_t N, const float* inv_norm,
                          const int32_t* status, const int32_t* slot, int32_t* nstar, float* cstar,
                          cudaStream_t st) {
  if (B == 0) return cudaSuccess;
  const bool vec = ((reinterpret_cast<uintptr_t>(C) & 15) == 0) && (ldc % 4 == 0) &&
                   ((reinterpret_cast<uintptr_t>(inv_norm) & 15) == 0);
  if (N >= 2048)
    k2_select<256><<<(unsigned)B, 256, 0, st>>>(C, ldc, N, inv_norm, status, slot, nstar, cstar, vec);
  else
    k2_select<128><<<(unsigned)B, 128, 0, st>>>(C, ldc, N, inv_norm, status, slot, nstar, cstar, vec);
  return cudaGetLastError();
}

}  // namespace ompb
