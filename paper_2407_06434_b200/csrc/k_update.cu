// The per-signal update of one OMP iteration, fused in one CTA per signal:
//
//  a3  (REFINE = true, tensor-core modes) exact selection after the screen:
//        n*_b = lowest n maximising |<r_b, a_n>| / ||a_n||
//      The screen (k_corr_tc.cu) bounds |c~_n - c_n| <= c0 ||a_n|| ||r_b||, i.e. c0 ||r_b|| in
//      normalised units for every n, so the exact argmax lies in
//        { n : v~_n >= max v~ - window ||r_b|| },  window = 2 (c0 + c0')   (c0' bounds this FP32 dot).
//      The screen kept, per 128-atom group, its entries within the window of the group max (up to 4,
//      in index order; more are flagged as an overflow, and such a group is re-evaluated in full when
//      its maximum is inside the global window); an overfull candidate list falls back to all N atoms.  Every candidate is re-evaluated as an
//      FP32 dot of the fp32 residual and the fp32 atom in a fixed order.  (REFINE = false: n*, c*
//      come from the standalone argmax over a materialised FP32 C, k_select.cu.)
//
//  a4  inverse-Cholesky factor append, the paper's algorithm-v0 update:
//        w = A_k^T a_{n*} = [A^T A]_{n*, S_k}
//        z = F_k^T w,  gamma = 1/sqrt(||a_{n*}||^2 - ||z||^2)
//        F_{k+1} = [[F_k, -gamma F_k z], [0, gamma]]                               (Eq. 8)
//        u = F^T A^T y grows by u_new = gamma <r_k, a_{n*}> = gamma c*  (q = A_{k+1} f is orthogonal
//            to span A_k, so q^T y = q^T r_k; pin P9)
//        x = F_{k+1} u   (matrix-vector products only, Eq. 11)
//      F is upper triangular, packed by columns (column j = F[0..j, j] at offset j(j+1)/2), the
//      paper's packed representation: the leading block is a contiguous prefix,
//      staged into shared memory by one cp.async.bulk at kernel start, so F leaves HBM once per
//      iteration and both passes over it run from shared memory.
//
//  a5  residual r_b = y_b - sum_{j<=k} x_j a_{s_j} from gathered atom rows of A^T,
//      ||r_b||, the eps test, and the operand planes of the next screen.
//
// Every live signal is at the same k (= iteration), so k is a kernel argument.  Finished signals
// return at once (capture-and-continue).
#include <cuda_bf16.h>
#include <math.h>
#include <stdlib.h>

#include "omp_internal.cuh"

namespace ompb {

constexpr int RF_CAP = 512;   // explicit candidate list capacity (beyond: all N atoms)

struct UpdateArgs {
  int32_t k, S;
  float eps;
  int64_t N, M, Mp;
  // selection inputs
  const float2* part;   // screen partials (REFINE)
  int groups;           // screen partial groups per row (Np / SCREEN_GROUP)
  float window;
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
  int32_t* live_next;
  float* resid;
  int32_t* n_iter;
  int32_t* status;
  int f_stage;          // 1: stage F_k in shared memory (else read F from global)
  int region_floats;    // floats of the aliased residual-row / F / gather-ring region
  int ring_slots;       // > 0: bulk-async gather through this many atom-row slots (else LDG gather)
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
__device__ __forceinline__ void stg_policy(float4* ptr, float4 v, uint64_t pol) {
  asm volatile("st.global.L1::no_allocate.L2::cache_hint.v4.f32 [%0], {%1, %2, %3, %4}, %5;"
               ::"l"(ptr), "f"(v.x), "f"(v.y), "f"(v.z), "f"(v.w), "l"(pol) : "memory");
}
__device__ __forceinline__ void stg_policy(uint2* ptr, uint2 v, uint64_t pol) {
  asm volatile("st.global.L1::no_allocate.L2::cache_hint.v2.u32 [%0], {%1, %2}, %3;"
               ::"l"(ptr), "r"(v.x), "r"(v.y), "l"(pol) : "memory");
}

__device__ __forceinline__ void mbar_wait_parity(uint64_t* bar, uint32_t parity) {
  uint32_t ok = 0;
  do {
    asm volatile("{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
                 "selp.u32 %0, 1, 0, p;\n\t}" : "=r"(ok) : "r"(smem_addr(bar)), "r"(parity) : "memory");
  } while (!ok);
}

// one contiguous atom row global -> shared through the bulk-copy (TMA) engine, completing on `bar`
__device__ __forceinline__ void bulk_row(void* dst, const void* src, uint32_t bytes, uint64_t* bar, uint64_t pol) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_addr(bar)), "r"(bytes) : "memory");
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], %4;"
      ::"r"(smem_addr(dst)), "l"(src), "r"(bytes), "r"(smem_addr(bar)), "l"(pol) : "memory");
}

constexpr int MAX_RING = 16;

__device__ __forceinline__ void cp_async4(void* dst, const void* src) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"(smem_addr(dst)), "l"(src) : "memory");
}
__device__ __forceinline__ void cp_async16(void* dst, const void* src) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(smem_addr(dst)), "l"(src) : "memory");
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

// lanes of one warp: c = sum_m r[m] a_n[m] in a fixed order (lane-strided float4, xor tree)
__device__ __forceinline__ float warp_dot(const float4* __restrict__ r4, const float4* __restrict__ a4, int q4,
                                          int lane) {
  // four float4 loads in flight per lane, four partial sums (fixed order: deterministic)
  float s0 = 0.f, s1 = 0.f, s2 = 0.f, s3 = 0.f;
  int q = lane;
  for (; q + 96 < q4; q += 128) {
    const float4 a0 = __ldg(a4 + q), a1 = __ldg(a4 + q + 32), a2 = __ldg(a4 + q + 64), a3 = __ldg(a4 + q + 96);
    const float4 r0 = r4[q], r1 = r4[q + 32], r2 = r4[q + 64], r3 = r4[q + 96];
    s0 = fmaf(r0.x, a0.x, fmaf(r0.y, a0.y, fmaf(r0.z, a0.z, fmaf(r0.w, a0.w, s0))));
    s1 = fmaf(r1.x, a1.x, fmaf(r1.y, a1.y, fmaf(r1.z, a1.z, fmaf(r1.w, a1.w, s1))));
    s2 = fmaf(r2.x, a2.x, fmaf(r2.y, a2.y, fmaf(r2.z, a2.z, fmaf(r2.w, a2.w, s2))));
    s3 = fmaf(r3.x, a3.x, fmaf(r3.y, a3.y, fmaf(r3.z, a3.z, fmaf(r3.w, a3.w, s3))));
  }
  for (; q < q4; q += 32) {
    const float4 a = __ldg(a4 + q);
    const float4 r = r4[q];
    s0 = fmaf(r.x, a.x, fmaf(r.y, a.y, fmaf(r.z, a.z, fmaf(r.w, a.w, s0))));
  }
  float acc = (s0 + s1) + (s2 + s3);
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
  return acc;
}

// MINB: resident CTAs per SM the register budget must allow.  The kernel is latency-bound on its L2
// gather and needs >= 8 CTAs of 128 threads per SM (measured: 2x slower at fewer, flat above).
template <bool REFINE, int T, int CH, int MINB = 1024 / T>
__global__ void __launch_bounds__(T, MINB) k_update(const UpdateArgs a) {
  const int64_t b = blockIdx.x;
  if (a.status[b] != SIG_RUNNING) return;
  const int k = a.k;
  const int q4 = (int)(a.Mp >> 2);
  const int Sp = (k + 4) & ~3;          // >= k + 1, multiple of 4
  const int cur_slot = a.slot[b];       // this signal's row in the current live set
  // dynamic shared memory (sizes in launch_update):
  //   [region X: the fp32 residual row (refine) then the packed F_k prefix (append), aliased]
  //   [w, z, u, xs: Sp floats each] [ss: Sp ints] [cand: RF_CAP ints (refine)]
  extern __shared__ __align__(16) uint8_t dsm[];
  float4* rsm = reinterpret_cast<float4*>(dsm);
  float* Fs = reinterpret_cast<float*>(dsm);
  float* w = reinterpret_cast<float*>(dsm + (size_t)a.region_floats * 4);
  float* z = w + Sp;
  float* u = z + Sp;
  float* xs = u + Sp;
  int* ss = reinterpret_cast<int*>(xs + Sp);
  uint32_t* ro = reinterpret_cast<uint32_t*>(ss + Sp);   // atom row offsets (float4 units) for the gather
  int* cand = reinterpret_cast<int*>(ro + Sp);
  __shared__ float red[T / 32];
  __shared__ Cand red_c[T / 32];
  __shared__ int ncand;
  __shared__ int sel_n;
  __shared__ float sel_c;
  __shared__ __align__(8) uint64_t fbar;
  __shared__ __align__(8) uint64_t rfull[MAX_RING], rempty[MAX_RING];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const float* Fg = a.F + b * a.ldf;
  const uint32_t fbytes = (uint32_t)((((int64_t)k * (k + 1) / 2) + 3) / 4 * 16);
  const bool staged = a.f_stage && fbytes > 0;
  bool issued = false;
  if (tid == 0) {
    ncand = 0;
    if (staged) {
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_addr(&fbar)) : "memory");
      asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
  }

  // ---- issue every load that does not depend on the selection (one round trip instead of a chain):
  // support and u of the current factor and (REFINE) the residual row -> shared memory by cp.async;
  // F_k -> L1 (both passes of the append read it); y -> L2 (the residual phase reads it)
  for (int j = tid; j < k; j += T) {
    cp_async4(&ss[j], a.support + b * a.lds + j);
    cp_async4(&u[j], a.U + b * a.ldu + j);
  }
  if constexpr (REFINE) {
    const float4* r4g = reinterpret_cast<const float4*>(a.R32in + (int64_t)cur_slot * a.Mp);
    for (int q = tid; q < q4; q += T) cp_async16(&rsm[q], r4g + q);
  }
  asm volatile("cp.async.commit_group;" ::: "memory");
  if (!staged) {
    const char* fp = reinterpret_cast<const char*>(Fg);
    for (uint32_t o = (uint32_t)tid * 128u; o < fbytes; o += (uint32_t)T * 128u)
      asm volatile("prefetch.global.L1 [%0];" ::"l"(fp + o));
  }
  {
    const char* yp = reinterpret_cast<const char*>(a.Y + b * a.ldy);
    for (int64_t o = (int64_t)tid * 128; o < a.M * 4; o += (int64_t)T * 128)
      asm volatile("prefetch.global.L2 [%0];" ::"l"(yp + o));
  }

  // ---- a3: selection ------------------------------------------------------------------------------
  if constexpr (REFINE) {
    const float rn = a.resid[b];
    const float2* P = a.part + (int64_t)cur_slot * a.groups * TOPK;
    const int E = a.groups * TOPK;
    float vmax = -1.f;
    for (int e = tid; e < E; e += T) vmax = fmaxf(vmax, P[e].x);
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) vmax = fmaxf(vmax, __shfl_xor_sync(0xffffffffu, vmax, o));
    if (lane == 0) red[warp] = vmax;
    __syncthreads();
    vmax = red[0];
#pragma unroll
    for (int i = 1; i < T / 32; ++i) vmax = fmaxf(vmax, red[i]);
    // every finite, nonzero residual leaves >= 1 entry per group (the group maximum itself); no entry
    // at all means the screened correlations were NaN.  (No CTA may exit with a cp.async in flight.)
    if (!(vmax >= 0.f) || !isfinite(rn) || rn == 0.f) asm volatile("cp.async.wait_all;" ::: "memory");
    if (!(vmax >= 0.f) || !isfinite(rn)) {
      if (tid == 0) a.status[b] = OMP_SIG_NAN;
      return;
    }
    if (rn == 0.f) {                                   // r = 0 exactly: every correlation is 0
      if (tid == 0) a.status[b] = OMP_SIG_DEGENERATE;
      return;
    }
    const float thr = vmax - a.window * rn;
    bool full = false;
    for (int t = tid; t < a.groups; t += T) {
      const float2 last = P[t * TOPK + TOPK - 1];
      const int nl = __float_as_int(last.y);
      if (nl == SEL_OVERFLOW && last.x >= thr) {         // more in-window entries than kept: all of it
        const int n0 = t * SCREEN_GROUP;
        const int cnt = (int)min((int64_t)SCREEN_GROUP, a.N - n0);
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
          if (p.x >= thr && n >= 0 && n < a.N) {
            const int at = atomicAdd(&ncand, 1);
            if (at >= RF_CAP) full = true;
            else cand[at] = n;
          }
        }
      }
    }
    asm volatile("cp.async.wait_all;" ::: "memory");   // residual row (and ss, u) landed
    full = __syncthreads_or(full);
    Cand best{-1.f, 0x7fffffff, 0.f};
    bool nan_c = false;
    const int count = full ? (int)a.N : min(ncand, RF_CAP);
    for (int j = warp; j < count; j += T / 32) {
      const int n = full ? j : cand[j];
      const float c = warp_dot(rsm, reinterpret_cast<const float4*>(a.At + (int64_t)n * a.Mp), q4, lane);
      nan_c |= isnan(c);
      const Cand cd{fabsf(c) * a.inv_norm[n], n, c};
      if (cand_better(cd, best)) best = cd;
    }
    if (lane == 0) red_c[warp] = best;
    const int any_nan = __syncthreads_or(nan_c);      // residual row no longer needed past here
    if (tid == 0) {
      Cand r = red_c[0];
#pragma unroll
      for (int i = 1; i < T / 32; ++i)
        if (cand_better(red_c[i], r)) r = red_c[i];
      const bool ok = r.w > 0.f && r.n < a.N;
      sel_n = any_nan ? SEL_NAN : (ok ? r.n : SEL_DEGENERATE);
      sel_c = ok ? r.c : 0.f;
    }
  } else {
    if (tid == 0) {
      sel_n = a.nstar[b];
      sel_c = a.cstar[b];
    }
  }
  // stage F_k (the contiguous packed prefix) over the freed residual-row region, asynchronously;
  // it lands while the support, the Gram entries and u are gathered below
  if (tid == 0 && staged && sel_n >= 0) {
    // order the generic-proxy reads of the residual row before the async-proxy overwrite
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_addr(&fbar)), "r"(fbytes)
                 : "memory");
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                 ::"r"(smem_addr(Fs)), "l"(Fg), "r"(fbytes), "r"(smem_addr(&fbar))
                 : "memory");
  }
  asm volatile("cp.async.wait_all;" ::: "memory");     // ss, u (SIMT path: first wait)
  __syncthreads();
  const int n = sel_n;
  const float cst = sel_c;
  if (n < 0) {
    if (tid == 0) a.status[b] = (n == SEL_NAN) ? OMP_SIG_NAN : OMP_SIG_DEGENERATE;
    return;
  }
  issued = staged;
  auto wait_f = [&]() {
    if (!issued) return;
    uint32_t ok = 0;
    do {
      asm volatile("{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], 0;\n\t"
                   "selp.u32 %0, 1, 0, p;\n\t}" : "=r"(ok) : "r"(smem_addr(&fbar)) : "memory");
    } while (!ok);
  };

  // ---- a4: factor append --------------------------------------------------------------------------
  const float* grow = a.G + (int64_t)n * a.ldg;
  bool dup = false;
  for (int j = tid; j < k; j += T) {
    const int s = ss[j];
    ro[j] = (uint32_t)s * (uint32_t)q4;
    dup |= (s == n);
    w[j] = grow[s];                     // [A^T A]_{n*, s_j}
  }
  if (__syncthreads_or(dup)) {          // re-selection (reading R6); let the F copy land first
    wait_f();
    if (tid == 0) a.status[b] = OMP_SIG_DEGENERATE;
    return;
  }
  wait_f();
  const float* Fb = staged ? Fs : Fg;
  // z_j = F[:, j] . w  (column dots; a warp takes two columns at a time so their loads and
  // shuffle reductions overlap)
  constexpr int NW = T / 32;
  for (int j0 = 2 * warp; j0 < k; j0 += 2 * NW) {
    const int j1 = j0 + 1;
    const float* c0 = Fb + (int64_t)j0 * (j0 + 1) / 2;
    const float* c1 = Fb + (int64_t)j1 * (j1 + 1) / 2;
    float a0 = 0.f, a1 = 0.f;
    for (int i = lane; i <= j1; i += 32) {
      if (i <= j0) a0 = fmaf(c0[i], w[i], a0);
      if (j1 < k) a1 = fmaf(c1[i], w[i], a1);
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      a0 += __shfl_xor_sync(0xffffffffu, a0, o);
      a1 += __shfl_xor_sync(0xffffffffu, a1, o);
    }
    if (lane == 0) {
      z[j0] = a0;
      if (j1 < k) z[j1] = a1;
    }
  }
  __syncthreads();
  float zz = 0.f;
  for (int j = tid; j < k; j += T) zz = fmaf(z[j], z[j], zz);
  zz = block_sum<T>(zz, red);
  const float d = grow[n];              // ||a_{n*}||^2
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
    for (; j + 4 <= k; j += 4) {
      const float f0 = (j >= i) ? Fb[(int64_t)j * (j + 1) / 2 + i] : 0.f;
      const float f1 = (j + 1 >= i) ? Fb[(int64_t)(j + 1) * (j + 2) / 2 + i] : 0.f;
      const float f2 = (j + 2 >= i) ? Fb[(int64_t)(j + 2) * (j + 3) / 2 + i] : 0.f;
      const float f3 = (j + 3 >= i) ? Fb[(int64_t)(j + 3) * (j + 4) / 2 + i] : 0.f;
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
      const float f = (j >= i) ? Fb[(int64_t)j * (j + 1) / 2 + i] : 0.f;
      v0 = fmaf(f, z[j], v0);
      t0 = fmaf(f, u[j], t0);
    }
    const float v = (v0 + v1) + (v2 + v3);
    const float t = (t0 + t1) + (t2 + t3);
    newcol[i] = -gamma * v;                       // -gamma F_k z
    const float xi = fmaf(-gamma * v, unew, t);   // x_i = (F_k u)_i + f_i u_new
    a.X[b * a.ldx + i] = xi;
    xs[i] = xi;
  }
  if (tid == 0) {
    newcol[k] = gamma;
    const float xk = gamma * unew;
    a.X[b * a.ldx + k] = xk;
    xs[k] = xk;
    ss[k] = n;
    ro[k] = (uint32_t)n * (uint32_t)q4;
    a.U[b * a.ldu + k] = unew;
    a.support[b * a.lds + k] = n;
  }
  __syncthreads();

  // ---- a5: residual r = y - A_S x, ||r||, eps test, next screening operand ------------------------
  // L2-bandwidth bound gather: per atom pair, every thread issues its 2 x CH float4 loads before the
  // FMAs; with T * CH == Mp / 4 (the benchmark shapes) no load is predicated.
  const int kk = k + 1;
  const uint64_t keep = policy_evict_last(), stream = policy_evict_first();
  float4 acc[CH];
#pragma unroll
  for (int c = 0; c < CH; ++c) acc[c] = make_float4(0.f, 0.f, 0.f, 0.f);
  const float4* A4 = reinterpret_cast<const float4*>(a.At) + tid;
  if (a.ring_slots > 0) {
    // Bulk-async gather: thread 0 streams whole atom rows (Mp floats, contiguous) into a ring of
    // shared-memory slots with cp.async.bulk (evict_last L2 policy); every thread folds x_j times its
    // float4 chunks of row j out of shared memory.  In-flight bytes are bounded by the ring, not by
    // the register file.  The ring aliases the F / residual-row region, free at this point.
    const int NS = a.ring_slots;
    const uint32_t rowb = (uint32_t)(a.Mp * 4);
    float4* ring = reinterpret_cast<float4*>(dsm);
    if (tid == 0) {
      for (int s = 0; s < NS; ++s) {
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_addr(&rfull[s])) : "memory");
        asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_addr(&rempty[s])), "r"(T / 32) : "memory");
      }
      asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");   // generic reads of F -> async writes
      for (int j = 0; j < NS && j < kk; ++j) bulk_row(ring + (size_t)j * q4, A4 - tid + ro[j], rowb, &rfull[j], keep);
    }
    __syncthreads();
    for (int j = 0; j < kk; ++j) {
      const int s = j % NS;
      const uint32_t par = (uint32_t)((j / NS) & 1);
      mbar_wait_parity(&rfull[s], par);
      const float xj = xs[j];
      const float4* row = ring + (size_t)s * q4 + tid;
#pragma unroll
      for (int c = 0; c < CH; ++c) {
        if (T * CH == q4 || tid + c * T < q4) {
          const float4 v = row[c * T];
          acc[c].x = fmaf(xj, v.x, acc[c].x);
          acc[c].y = fmaf(xj, v.y, acc[c].y);
          acc[c].z = fmaf(xj, v.z, acc[c].z);
          acc[c].w = fmaf(xj, v.w, acc[c].w);
        }
      }
      __syncwarp();
      if (lane == 0) asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_addr(&rempty[s])) : "memory");
      if (tid == 0 && j + NS < kk) {
        mbar_wait_parity(&rempty[s], par);          // every warp has read slot s
        bulk_row(ring + (size_t)s * q4, A4 - tid + ro[j + NS], rowb, &rfull[s], keep);
      }
    }
  } else if (T * CH == q4) {
    int j = 0;
    for (; j + 2 <= kk; j += 2) {
      const float4* r0 = A4 + ro[j];
      const float4* r1 = A4 + ro[j + 1];
      float4 v0[CH], v1[CH];
#pragma unroll
      for (int c = 0; c < CH; ++c) v0[c] = ldg_policy(r0 + c * T, keep);
#pragma unroll
      for (int c = 0; c < CH; ++c) v1[c] = ldg_policy(r1 + c * T, keep);
      const float x0 = xs[j], x1 = xs[j + 1];
#pragma unroll
      for (int c = 0; c < CH; ++c) {
        acc[c].x = fmaf(x1, v1[c].x, fmaf(x0, v0[c].x, acc[c].x));
        acc[c].y = fmaf(x1, v1[c].y, fmaf(x0, v0[c].y, acc[c].y));
        acc[c].z = fmaf(x1, v1[c].z, fmaf(x0, v0[c].z, acc[c].z));
        acc[c].w = fmaf(x1, v1[c].w, fmaf(x0, v0[c].w, acc[c].w));
      }
    }
    if (j < kk) {
      const float4* r0 = A4 + ro[j];
      const float x0 = xs[j];
#pragma unroll
      for (int c = 0; c < CH; ++c) {
        const float4 v = ldg_policy(r0 + c * T, keep);
        acc[c].x = fmaf(x0, v.x, acc[c].x);
        acc[c].y = fmaf(x0, v.y, acc[c].y);
        acc[c].z = fmaf(x0, v.z, acc[c].z);
        acc[c].w = fmaf(x0, v.w, acc[c].w);
      }
    }
  } else {
    for (int j = 0; j < kk; ++j) {
      const float4* r0 = A4 + ro[j];
      const float x0 = xs[j];
#pragma unroll
      for (int c = 0; c < CH; ++c) {
        if (tid + c * T < q4) {
          const float4 v = ldg_policy(r0 + c * T, keep);
          acc[c].x = fmaf(x0, v.x, acc[c].x);
          acc[c].y = fmaf(x0, v.y, acc[c].y);
          acc[c].z = fmaf(x0, v.z, acc[c].z);
          acc[c].w = fmaf(x0, v.w, acc[c].w);
        }
      }
    }
  }
  const float* y = a.Y + b * a.ldy;
  const bool yvec = ((reinterpret_cast<uintptr_t>(a.Y) & 15) == 0) && (a.ldy % 4 == 0);
  float part = 0.f;
#pragma unroll
  for (int c = 0; c < CH; ++c) {
    const int q = tid + c * T;
    if (q < q4) {
      const int64_t m = (int64_t)q << 2;
      float4 yv;
      if (yvec && m + 3 < a.M) {
        yv = ldg_policy(reinterpret_cast<const float4*>(y + m), stream);
      } else {
        yv.x = m < a.M ? y[m] : 0.f;
        yv.y = m + 1 < a.M ? y[m + 1] : 0.f;
        yv.z = m + 2 < a.M ? y[m + 2] : 0.f;
        yv.w = m + 3 < a.M ? y[m + 3] : 0.f;
      }
      acc[c] = make_float4(yv.x - acc[c].x, yv.y - acc[c].y, yv.z - acc[c].z, yv.w - acc[c].w);   // r
      part = fmaf(acc[c].x, acc[c].x, fmaf(acc[c].y, acc[c].y, fmaf(acc[c].z, acc[c].z, fmaf(acc[c].w, acc[c].w, part))));
    }
  }
  const float rr = block_sum<T>(part, red);
  if (tid == 0) {
    const float rn = sqrtf(rr);
    a.resid[b] = rn;
    a.n_iter[b] = kk;
    int ns = -1;
    if (a.eps >= 0.f && rn <= a.eps) a.status[b] = OMP_SIG_EPS;
    else if (kk == a.S) a.status[b] = OMP_SIG_MAXITER;
    else {
      ns = atomicAdd(a.live_next, 1);                                  // next live-set slot
      a.rslot_out[ns] = rn;
    }
    a.slot[b] = ns;
    sel_n = ns;
  }
  __syncthreads();
  const int ns = sel_n;
  if (ns < 0) return;                   // finished: no planes for the next screen
  const int64_t ro_out = (int64_t)ns * a.Mp;
#pragma unroll
  for (int c = 0; c < CH; ++c) {
    const int q = tid + c * T;
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

template <bool REFINE, int T, int CH, int MINB = 1024 / T>
static cudaError_t launch_t(const UpdateArgs& a, int64_t B, size_t smem, size_t persist, cudaStream_t st) {
  auto kern = k_update<REFINE, T, CH, MINB>;
  // static + dynamic shared memory may exceed the 48 KB default: opt in once per variant
  static bool opted = false;
  if (!opted) {
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, 160 * 1024);
    if (e != cudaSuccess) return e;
    opted = true;
  }
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3((unsigned)B);
  cfg.blockDim = dim3(T);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  if (persist > 0) {
    // keep the fp32 atom table (re-read by every signal's gather) in the persisting L2 carve-out;
    // a launch attribute, so the caller's stream is left untouched
    attr[0].id = cudaLaunchAttributeAccessPolicyWindow;
    attr[0].val.accessPolicyWindow.base_ptr = const_cast<float*>(a.At);
    attr[0].val.accessPolicyWindow.num_bytes = persist;
    attr[0].val.accessPolicyWindow.hitRatio = 1.0f;
    attr[0].val.accessPolicyWindow.hitProp = cudaAccessPropertyPersisting;
    attr[0].val.accessPolicyWindow.missProp = cudaAccessPropertyStreaming;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
  }
  return cudaLaunchKernelEx(&cfg, kern, a);
}

template <bool REFINE>
static cudaError_t launch_r(const UpdateArgs& a, int64_t B, size_t smem, size_t persist, cudaStream_t st) {
  const int64_t q4 = a.Mp / 4;   // float4 chunks per row; T * CH == q4 at powers of two
  static int wide = -1;          // OMP_B200_UPDATE_WIDE=1: 256 threads per signal at M = 1025..2048
  if (wide < 0) {
    const char* env = getenv("OMP_B200_UPDATE_WIDE");
    wide = (env && env[0] == '1') ? 1 : 0;
  }
  if (wide && q4 > 256 && q4 <= 512) return launch_t<REFINE, 256, 2>(a, B, smem, persist, st);
  if (q4 <= 32) return launch_t<REFINE, 32, 1>(a, B, smem, persist, st);
  if (q4 <= 64) return launch_t<REFINE, 64, 1>(a, B, smem, persist, st);
  if (q4 <= 128) return launch_t<REFINE, 128, 1>(a, B, smem, persist, st);
  if (q4 <= 256) return launch_t<REFINE, 128, 2>(a, B, smem, persist, st);
  if (q4 <= 512) {
    static int minb = -1;          // OMP_B200_UPDATE_MINB: register budget for 10 or 12 CTAs per SM
    if (minb < 0) {
      const char* env = getenv("OMP_B200_UPDATE_MINB");
      minb = env ? atoi(env) : 0;
    }
    if (minb == 10) return launch_t<REFINE, 128, 4, 10>(a, B, smem, persist, st);
    if (minb == 12) return launch_t<REFINE, 128, 4, 12>(a, B, smem, persist, st);
    return launch_t<REFINE, 128, 4>(a, B, smem, persist, st);
  }
  if (q4 <= 1024) return launch_t<REFINE, 256, 4>(a, B, smem, persist, st);
  if (q4 <= 2048) return launch_t<REFINE, 256, 8>(a, B, smem, persist, st);
  return cudaErrorNotSupported;   // M > 8192
}

cudaError_t launch_update(const UpdateLaunch& L, cudaStream_t st) {
  if (L.B == 0) return cudaSuccess;
  UpdateArgs a;
  a.k = L.k; a.S = L.S; a.eps = L.eps; a.N = L.N; a.M = L.M; a.Mp = L.Mp;
  a.part = L.part; a.groups = L.groups; a.window = L.window; a.nstar = L.nstar; a.cstar = L.cstar;
  a.At = L.At; a.inv_norm = L.inv_norm; a.G = L.G; a.ldg = L.ldg;
  a.Y = L.Y; a.ldy = L.ldy; a.F = L.F; a.ldf = L.ldf; a.U = L.U; a.ldu = L.ldu; a.X = L.X; a.ldx = L.ldx;
  a.support = L.support; a.lds = L.lds; a.R32in = L.R32in; a.R32 = L.R32; a.Rb = (__nv_bfloat16*)L.Rb;
  a.Rhi = L.Rhi; a.Rlo = L.Rlo; a.rslot_out = L.rslot_out; a.slot = L.slot; a.live_next = L.live_next;
  a.resid = L.resid; a.n_iter = L.n_iter; a.status = L.status;
  // one region holds the residual row (refine) and then F_k (append); F is staged when it fits
  const int64_t fk = ((int64_t)L.k * (L.k + 1) / 2 + 3) / 4 * 4;
  const bool refine = L.part != nullptr;
  const int64_t rowf = refine ? L.Mp : 0;
  // F_k staging in shared memory (OMP_B200_F_STAGE=1) costs occupancy; by default F_k is prefetched
  // into L1 at kernel start instead
  static int fstage_env = -1;
  if (fstage_env < 0) {
    const char* env = getenv("OMP_B200_F_STAGE");
    fstage_env = (env && env[0] == '1') ? 1 : 0;
  }
  a.f_stage = (fstage_env && fk * 4 <= (int64_t)64 * 1024 && L.ldf % 4 == 0) ? 1 : 0;
  int64_t region = (a.f_stage && fk > rowf) ? fk : rowf;
  // gather ring: OMP_B200_RING_KB (default 48) of atom-row slots, 2..MAX_RING slots; 0 -> LDG gather
  static int ring_kb = -1;
  if (ring_kb < 0) {
    const char* env = getenv("OMP_B200_RING_KB");
    ring_kb = env ? atoi(env) : 0;   // measured slower than the LDG gather at c4
  }
  const int64_t rowf_all = L.Mp;
  int slots = (int)(((int64_t)ring_kb * 1024 / 4) / rowf_all);
  if (slots > MAX_RING) slots = MAX_RING;
  if (slots < 2 || (int64_t)L.Mp * 4 % 16 != 0) slots = 0;
  a.ring_slots = slots;
  if (slots * rowf_all > region) region = slots * rowf_all;
  a.region_floats = (int)region;
  const int64_t Sp = (L.k + 4) & ~3;
  const size_t smem = (size_t)a.region_floats * 4 + (size_t)Sp * 6 * 4 + (refine ? RF_CAP * 4 : 0);
  return refine ? launch_r<true>(a, L.B, smem, L.l2_persist_bytes, st)
                : launch_r<false>(a, L.B, smem, L.l2_persist_bytes, st);
}

}  // namespace ompb
