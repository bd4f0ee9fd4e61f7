// K2 after the tensor-core screen: exact selection
//     n*_b = lowest n maximising |<r_b, a_n>| / ||a_n||
//
// The screening GEMM (k_corr_tc.cu) gives c~_n with |c~_n - c_n| <= c0 ||a_n|| ||r_b|| (rigorous
// bound from the operand rounding and the truncating accumulator).  In normalised
// units v_n = |c_n| / ||a_n|| the error is at most c0 ||r_b||, uniformly over n, so the exact
// argmax lies in  { n : v~_n >= max v~ - window ||r_b|| },  window = 2 (c0 + c0'), c0' bounding
// the FP32 re-evaluation below.  The screen's epilogue kept the top-TOPK of every 256-atom tile;
// a tile whose TOPK-th entry is still inside the window is re-evaluated in full, and an
// overfull candidate list falls back to all N atoms, so the candidate set always contains the
// exact argmax.  Every candidate is re-evaluated as an FP32 dot of the fp32 residual and the
// fp32 atom (fixed summation order), and the winner's signed c* = <r_b, a_{n*}> is handed to
// the factor append (u_new = gamma c*, pin P9).
#include <math.h>

#include "omp_internal.cuh"

namespace ompb {

constexpr int RF_THREADS = 128;
constexpr int RF_CAP = 512;

struct Cand {
  float w;
  int n;
  float c;
};

__device__ __forceinline__ bool cand_better(const Cand& a, const Cand& b) {   // is a better than b
  return a.w > b.w || (a.w == b.w && a.n < b.n);
}

// lanes of one warp: c = sum_m r[m] a_n[m] in a fixed order (lane-strided float4, xor tree)
__device__ __forceinline__ float warp_dot(const float4* __restrict__ r4, const float4* __restrict__ a4, int q4,
                                          int lane) {
  float acc = 0.f;
  for (int q = lane; q < q4; q += 32) {
    const float4 a = __ldg(a4 + q);
    const float4 r = r4[q];
    acc = fmaf(r.x, a.x, acc);
    acc = fmaf(r.y, a.y, acc);
    acc = fmaf(r.z, a.z, acc);
    acc = fmaf(r.w, a.w, acc);
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
  return acc;
}

__global__ void __launch_bounds__(RF_THREADS) k2_refine(const float2* __restrict__ part, int tiles_n, int64_t N,
                                                        int64_t Mp, const float* __restrict__ R32,
                                                        const float* __restrict__ At,
                                                        const float* __restrict__ inv_norm,
                                                        const float* __restrict__ resid, float window,
                                                        const int32_t* __restrict__ status,
                                                        int32_t* __restrict__ nstar, float* __restrict__ cstar) {
  extern __shared__ float4 rsm[];                 // the fp32 residual row (Mp floats)
  __shared__ int cand[RF_CAP];
  __shared__ int ncand;
  __shared__ float red_v[RF_THREADS / 32];
  __shared__ Cand red_c[RF_THREADS / 32];
  const int64_t b = blockIdx.x;
  if (status[b] != SIG_RUNNING) return;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const float rn = resid[b];
  if (rn == 0.f) {                                // r = 0 exactly: every correlation is 0
    if (tid == 0) { nstar[b] = SEL_DEGENERATE; cstar[b] = 0.f; }
    return;
  }
  const float2* P = part + b * (int64_t)tiles_n * TOPK;
  const int E = tiles_n * TOPK;
  // 1) max screened value and NaN flag
  float vmax = -1.f;
  bool nan_seen = false;
  for (int e = tid; e < E; e += RF_THREADS) {
    const float2 p = P[e];
    nan_seen |= (__float_as_int(p.y) == SEL_NAN) | isnan(p.x);
    vmax = fmaxf(vmax, p.x);
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) vmax = fmaxf(vmax, __shfl_xor_sync(0xffffffffu, vmax, o));
  if (lane == 0) red_v[warp] = vmax;
  if (tid == 0) ncand = 0;
  const int any_nan = __syncthreads_or(nan_seen);
  if (any_nan || !isfinite(rn)) {
    if (tid == 0) { nstar[b] = SEL_NAN; cstar[b] = 0.f; }
    return;
  }
  vmax = red_v[0];
#pragma unroll
  for (int w = 1; w < RF_THREADS / 32; ++w) vmax = fmaxf(vmax, red_v[w]);
  const float thr = vmax - window * rn;
  // 2) candidates: entries inside the window; tiles whose last kept entry is inside -> whole tile
  bool full = false;
  for (int t = tid; t < tiles_n; t += RF_THREADS) {
    const bool overflow = P[t * TOPK + TOPK - 1].x >= thr;
    if (overflow) {
      const int n0 = t * N_TILE;
      const int cnt = (int)min((int64_t)N_TILE, N - n0);
      if (cnt > 0) {
        const int at = atomicAdd(&ncand, cnt);
        if (at + cnt > RF_CAP) full = true;
        else
          for (int i = 0; i < cnt; ++i) cand[at + i] = n0 + i;
      }
    } else {
      for (int j = 0; j < TOPK; ++j) {
        const float2 p = P[t * TOPK + j];
        const int n = __float_as_int(p.y);
        if (p.x >= thr && n >= 0 && n < N) {
          const int at = atomicAdd(&ncand, 1);
          if (at >= RF_CAP) full = true;
          else cand[at] = n;
        }
      }
    }
  }
  // 3) the residual row into shared memory
  const int q4 = (int)(Mp >> 2);
  const float4* r4g = reinterpret_cast<const float4*>(R32 + b * Mp);
  for (int q = tid; q < q4; q += RF_THREADS) rsm[q] = r4g[q];
  full = __syncthreads_or(full);
  // 4) exact FP32 re-evaluation, one warp per candidate
  Cand best{-1.f, 0x7fffffff, 0.f};
  const int count = full ? (int)N : min(ncand, RF_CAP);
  for (int j = warp; j < count; j += RF_THREADS / 32) {
    const int n = full ? j : cand[j];
    const float c = warp_dot(rsm, reinterpret_cast<const float4*>(At + (int64_t)n * Mp), q4, lane);
    const Cand cd{fabsf(c) * inv_norm[n], n, c};
    if (cand_better(cd, best)) best = cd;
  }
  if (lane == 0) red_c[warp] = best;
  __syncthreads();
  if (tid == 0) {
    Cand r = red_c[0];
#pragma unroll
    for (int w = 1; w < RF_THREADS / 32; ++w)
      if (cand_better(red_c[w], r)) r = red_c[w];
    const bool ok = r.w > 0.f && r.n < N;
    nstar[b] = ok ? r.n : SEL_DEGENERATE;
    cstar[b] = ok ? r.c : 0.f;
  }
}

cudaError_t launch_refine(const float2* part, int tiles_n, int64_t B, int64_t N, int64_t Mp,
                          const float* R32, const float* At, const float* inv_norm, const float* resid,
                          float window, const int32_t* status, int32_t* nstar, float* cstar, cudaStream_t st) {
  if (B == 0) return cudaSuccess;
  const size_t smem = (size_t)Mp * sizeof(float);
  if (smem > 48 * 1024) {
    cudaError_t e = cudaFuncSetAttribute(k2_refine, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
  }
  k2_refine<<<(unsigned)B, RF_THREADS, smem, st>>>(part, tiles_n, N, Mp, R32, At, inv_norm, resid, window, status,
                                                   nstar, cstar);
  return cudaGetLastError();
}

}  // namespace ompb
