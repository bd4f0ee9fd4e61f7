// The per-signal update of one OMP iteration, fused in one CTA per signal:
//
//  a3  (REFINE = true, tensor-core modes) exact selection after the screen:
//        n*_b = lowest n maximising |<r_b, a_n>| / ||a_n||
//      The screen (k_corr_tc.cu) bounds |c~_n - c_n| <= c0 ||a_n|| ||r_b||, i.e. c0 ||r_b|| in
//      normalised units for every n, so the exact argmax lies in
//        { n : v~_n >= max v~ - window ||r_b|| },  window = 2 (c0 + c0')   (c0' bounds this FP32 dot).
//      The screen kept, per 128-atom group, its entries within the window of the group max (up to 4,
//      in index order; more are flagged as an overflow, and such a group is re-evaluated in full when
//      its maximum is inside the global window); an overfull candidate list falls back to all N atoms.
//      Every candidate is re-evaluated as an FP32 dot of the fp32 residual and the fp32 atom in a fixed
//      order (warp_dot, update_core.cuh).  (REFINE = false: n*, c* come from the standalone argmax over
//      a materialised FP32 C, k_select.cu.)
//
//  a4 + a5  factor append and residual: append_residual (update_core.cuh).
//
// Every live signal is at the same k (= iteration), so k is a kernel argument.  Finished signals
// return at once (capture-and-continue).
#include <math.h>

#include <atomic>
#include <stdlib.h>

#ifdef OMP_UPDATE_TRACE
// diagnostic build only (-DOMP_UPDATE_TRACE, scripts/trace_update.py): per-phase clock64 deltas of
// thread 0, summed over every CTA of the launch at iteration g_upd_trace_k
__device__ int g_upd_trace_k = -1;
__device__ unsigned long long g_upd_clk[16];
// the SM clock inside the traced launch: (clock64, globaltimer) of the first and the last CTA at their
// start and end (each pair measures its own SM over the CTA's lifetime)
__device__ unsigned long long g_upd_freq[8];
__device__ __forceinline__ void upd_freq_mark(int slot) {
  unsigned long long t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  g_upd_freq[2 * slot] = clock64();
  g_upd_freq[2 * slot + 1] = t;
}
#define UPD_TRACE(p)                                                                   \
  do {                                                                                 \
    if (threadIdx.x == 0 && a.k == g_upd_trace_k) {                                    \
      const unsigned long long t_ = clock64();                                         \
      atomicAdd(&g_upd_clk[(p)], t_ - upd_t0_);                                        \
      upd_t0_ = t_;                                                                    \
    }                                                                                  \
  } while (0)
#define OMP_TAIL_TRACE(p) UPD_TRACE(4 + (p))
#else
#define UPD_TRACE(p)
#endif
#include "update_core.cuh"

namespace ompb {

#ifndef OMP_RF_CAP
#define OMP_RF_CAP 512
#endif
constexpr int RF_CAP = OMP_RF_CAP;   // largest kept-entry list (beyond: all N atoms); a launch sizes its list
                                     // min(RF_CAP, groups x TOPK), so it overflows only when N > 16 384
constexpr int GRP_CAP = 64;          // overflowing 128-atom groups re-evaluated whole (beyond: all N)
constexpr int64_t kFsmMaxBytes = 8192;   // largest packed F_k staged in shared memory
// columns per warp in z = F^T w (interleaving only: no column's arithmetic changes; measured: 4 or 8
// cost registers and lose at c4 and at c5 B = 10^5)
constexpr int kZC = 2;
// one-warp CTAs (T = 32) take OMP_ZC32 columns per round: their single warp walks all k columns, so more
// of them in flight hides more of the shuffle trees' latency (same arithmetic per column).  Measured
// (profiles/r02/ab/ab_zc_r02o.txt): 4 columns vs 2, c5 B = 10^5 +3.2 %, B = 10^4 +4.4 %; 3: +1.3 / +2.3 %;
// round 1: 8 lost (spills)
#ifndef OMP_ZC32
#define OMP_ZC32 4
#endif
// with F_k in shared memory, CTAs of <= OMP_ZLANE_TMAX threads sum z = F^T w thread per column (the same
// bits; update_core.cuh).  Measured (profiles/r02/ab/ab_zlane_r02r.txt): c5 B = 10^5 / 10^4 (T = 32)
// +4 / +3.7 %, c2 (T = 64) +5.7 %; T = 128 lost (c3 -2.7 %, c5 B = 10^3 -3 %: register spills)
#ifndef OMP_ZLANE_TMAX
#define OMP_ZLANE_TMAX 64
#endif

// SEL: how n* is found -- SEL_GIVEN (nstar/cstar from k_select), SEL_SCREEN (refine the screen's
// candidates), SEL_PROJ (projection path: exact argmax over the projection row p = A^T r_k)
constexpr int SEL_GIVEN = 0, SEL_SCREEN = 1, SEL_PROJ = 2;
constexpr int SEL_SCREEN_FSM = 3;   // SEL_SCREEN with the packed F_k staged in shared memory

// P: atom rows in flight per thread in the gather (2 at 8 CTAs per SM; more when the batch leaves
// the SMs nearly empty and one CTA's memory parallelism is all a signal gets)
// Resident threads per SM the register budget must allow: 1280 = 10 CTAs of 128 threads (51
// registers).  The kernel is latency-bound on its L2 gather; measured at c4 (A/B builds on one box):
// 6 CTAs 5.09 ms, 7: 4.82, 8: 4.66, 10: 4.52, 12: 4.53 ms per launch, despite the spills it costs.
#ifndef OMP_UPDATE_CTAS
#define OMP_UPDATE_CTAS 1280
#endif
// float4 loads in flight per thread in the gather (P x CH, at least 2 rows): narrow rows (CH = 1, 2)
// take more rows per round trip
#ifndef OMP_UPDATE_PCH
#define OMP_UPDATE_PCH 2
#endif
// bytes of the first dynamic shared-memory region: the staged fp32 residual row (refine: Mp floats; it
// doubles as the tail's ||r||^2 chunk partials), or just those partials (Mp / 4 floats); none for one-warp
// CTAs, which sum ||r||^2 in registers (append_residual) and read the row from global memory
#ifndef OMP_RG
#define OMP_RG 1
#endif
template <int T, int CH>
__host__ __device__ constexpr size_t update_region0(bool refine, int64_t Mp) {
  // (one-warp CTAs that do not own their summation-order chunks keep the chunk partials: 2 Mp / 4 floats)
  return (T == 32 && OMP_RG) ? (update_rreg<T, CH>() ? 0 : (size_t)Mp * 2) : (refine ? (size_t)Mp * 4 : (size_t)Mp);
}

template <int SEL, int T, int CH, int MINB = (OMP_UPDATE_CTAS / T < 32 ? OMP_UPDATE_CTAS / T : 32), int P = 2>
__global__ void __launch_bounds__(T, MINB) k_update(const UpdateArgs a) {
  constexpr bool REFINE = (SEL == SEL_SCREEN || SEL == SEL_SCREEN_FSM);
  constexpr bool FSM = (SEL == SEL_SCREEN_FSM);   // compile-time, so F's address space is known
  const int64_t b = blockIdx.x;
  // PDL (screened path): wait for the screen's completion, then let the next screen launch early
  asm volatile("griddepcontrol.wait;" ::: "memory");
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
#ifdef OMP_UPDATE_TRACE
  const bool freq_cta = threadIdx.x == 0 && a.k == g_upd_trace_k && (b == 0 || b == gridDim.x - 1);
  if (freq_cta) upd_freq_mark(b == 0 ? 0 : 2);
#endif
  // the status and this signal's row in the current live set, loaded together (one round trip; the
  // slot of a finished signal is never used)
  const int status_b = a.status[b];
  const int cur_slot = a.slot ? a.slot[b] : (int)b;
  if (status_b != SIG_RUNNING) return;
#ifdef OMP_UPDATE_TRACE
  unsigned long long upd_t0_ = clock64();
#endif
  const int k = a.k;
  const int q4 = (int)(a.Mp >> 2);
  const int Sp = (k + 4) & ~3;          // >= k + 1, multiple of 4
  // dynamic shared memory (sizes in launch_update / launch_t):
  //   [update_region0: the fp32 residual row (refine): Mp floats; else Mp / 4 floats; one-warp CTAs: none,
  //    or the 2 Mp / 4 chunk partials of ||r||^2 where they cannot be summed in registers]
  //   [w, z, u, xs: Sp floats each]
  //   [ss, ro: Sp ints each] [cand: a.candcap ints (refine)] [F_k packed (fsm)]
  extern __shared__ __align__(16) uint8_t dsm[];
  // one-warp CTAs (RG) keep no residual row in shared memory: the refine reads it from global memory
  // (prefetched into L1 at the start) and the tail sums ||r||^2 in registers, so the 32 CTAs per SM
  // also fit at the last iterations of c5 (with the row staged, k >= 37 left 23..31)
  constexpr bool RG = (T == 32) && OMP_RG;
  float4* rsm = reinterpret_cast<float4*>(dsm);
  // (the first region doubles as the tail's ||r||^2 chunk partials, Mp / 4 floats, after the refine)
  float* w = reinterpret_cast<float*>(dsm + update_region0<T, CH>(REFINE, a.Mp));
  float* z = w + Sp;
  float* u = z + Sp;
  float* xs = u + Sp;
  int* ss = reinterpret_cast<int*>(xs + Sp);
  uint32_t* ro = reinterpret_cast<uint32_t*>(ss + Sp);
  int* cand = reinterpret_cast<int*>(ro + Sp);
  __shared__ float red[T / 32];
  __shared__ Cand red_c[T / 32];
  __shared__ int ncand;
  __shared__ int ngrp;                 // overflowing screen groups inside the window (re-evaluated whole)
  __shared__ int grp[GRP_CAP];
  __shared__ int sel_n;
  __shared__ float sel_c;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  if (tid == 0) {
    ncand = 0;
    ngrp = 0;
  }

  // ---- issue every load that does not depend on the selection (one round trip instead of a chain):
  // support and u of the current factor and (REFINE) the residual row -> shared memory by cp.async;
  // F_k -> L1 (both passes of the append read it)
  for (int j = tid; j < k; j += T) {
    cp_async4(&ss[j], a.support + b * a.lds + j);
    cp_async4(&u[j], a.U + b * a.ldu + j);
  }
  const float4* r4g = reinterpret_cast<const float4*>(a.R32in + (int64_t)cur_slot * a.Mp);
  if constexpr (REFINE && !RG) {
    for (int q = tid; q < q4; q += T) cp_async16(&rsm[q], r4g + q);
  } else if constexpr (REFINE) {
    for (uint32_t o = (uint32_t)tid * 128u; o < (uint32_t)a.Mp * 4u; o += (uint32_t)T * 128u)
      asm volatile("prefetch.global.L1 [%0];" ::"l"(reinterpret_cast<const char*>(r4g) + o));
  }
  const float4* rrow = RG ? r4g : rsm;   // the residual row the refine's dots read
  // a small packed F_k (fsm: decided at launch) goes to shared memory too: the column dots z = F^T w
  // and the row sweeps F z, F u then read shared memory instead of dependent L2 round trips
  float* Fs = reinterpret_cast<float*>(cand + (REFINE ? a.candcap : 0));
  if constexpr (FSM) {
    const int f4 = (k * (k + 1) / 2 + 3) >> 2;          // within the row: ldf >= S(S+1)/2 rounded to 4
    const float4* fg = reinterpret_cast<const float4*>(a.F + b * a.ldf);
    for (int q = tid; q < f4; q += T) cp_async16(reinterpret_cast<float4*>(Fs) + q, fg + q);
  }
  asm volatile("cp.async.commit_group;" ::: "memory");
#ifndef OMP_NO_FPF
  if constexpr (!FSM) {
    const char* fp = reinterpret_cast<const char*>(a.F + b * a.ldf);
    // (only while F_k fits L1 comfortably; a large one is read from L2 with loads in flight instead)
#ifndef OMP_FPF_MAX
#define OMP_FPF_MAX (64 * 1024)
#endif
    const uint32_t fbytes = (uint32_t)min((int64_t)k * (k + 1) / 2 * 4, (int64_t)OMP_FPF_MAX);
    for (uint32_t o = (uint32_t)tid * 128u; o < fbytes; o += (uint32_t)T * 128u)
      asm volatile("prefetch.global.L1 [%0];" ::"l"(fp + o));
  }
#endif
  // (no L2 prefetch of y: measured at c4, its lines are evicted before the residual phase reads them
  // -- 0.84 GB of extra DRAM reads per launch for 0.8 GB of y, and 1.2 % slower; profiles/r02/ab_dram;
  // nor a shared-memory copy: 8 % slower at c4, 3 % at c5 -- the L1 it takes from the F_k prefetch --
  // for 1 % at c2 / c3, profiles/r02/ab/ab_ystage_r02g.txt.  The gather's accumulator starts at y.)

  // ---- a3: selection ------------------------------------------------------------------------------
  if constexpr (REFINE) {
    const float rn = a.resid[b];
    const float2* Pt = a.part + (int64_t)cur_slot * a.groups * TOPK;
    const int E = a.groups * TOPK;
    float vmax = -1.f;
    for (int e = tid; e < E; e += T) vmax = fmaxf(vmax, Pt[e].x);
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
    const float thr = vmax - a.rslot_in[cur_slot];       // the window W of this signal
    bool full = false;
    for (int t = tid; t < a.groups; t += T) {
      const float2 last = Pt[t * TOPK + TOPK - 1];
      const int nl = __float_as_int(last.y);
      if (nl == SEL_OVERFLOW && last.x >= thr) {         // more in-window entries than kept: all of it
        if ((int64_t)t * SCREEN_GROUP < a.N) {
          const int at = atomicAdd(&ngrp, 1);
          if (at >= GRP_CAP) full = true;
          else grp[at] = t;
        }
      } else {
        for (int j = 0; j < TOPK; ++j) {
          const float2 p = Pt[t * TOPK + j];
          const int n = __float_as_int(p.y);
          if (p.x >= thr && n >= 0 && n < a.N) {
            const int at = atomicAdd(&ncand, 1);
            if (at >= a.candcap) full = true;
            else cand[at] = n;
          }
        }
      }
    }
    UPD_TRACE(0);
    asm volatile("cp.async.wait_all;" ::: "memory");   // residual row (and ss, u) landed
    full = __syncthreads_or(full);
    UPD_TRACE(1);
#ifdef OMP_UPDATE_TRACE
    if (tid == 0 && a.k == g_upd_trace_k) {   // candidate statistics: sum, > 16, > 128, full fallback
      const int nc = min(ncand, a.candcap) + min(ngrp, GRP_CAP) * SCREEN_GROUP;
      atomicAdd(&g_upd_clk[12], (unsigned long long)nc);
      if (nc > 16) atomicAdd(&g_upd_clk[13], 1ull);
      if (ngrp > 0) atomicAdd(&g_upd_clk[14], 1ull);
      if (full) atomicAdd(&g_upd_clk[3], 1ull);
    }
#endif
    Cand best{-1.f, 0x7fffffff, 0.f};
    bool nan_c = false;
    // the kept entries, then every atom of each overflowing group (no atom is in both); more than the
    // lists hold: all N atoms
    const int nind = min(ncand, a.candcap), ng = min(ngrp, GRP_CAP);
    const int count = full ? (int)a.N : nind + ng * SCREEN_GROUP;
    // candidate j of the list (-1 past the end or on the last group's padding)
    auto cand_at = [&](int j) -> int {
      if (j >= count) return -1;
      if (full) return j;
      if (j < nind) return cand[j];
      const int n = grp[(j - nind) / SCREEN_GROUP] * SCREEN_GROUP + (j - nind) % SCREEN_GROUP;
      return n < a.N ? n : -1;
    };
    auto consider = [&](int n, float c) {
      nan_c |= isnan(c);
      const Cand cd{fabsf(c) * a.inv_norm[n], n, c};
      if (cand_better(cd, best)) best = cd;
    };
    // rows of <= 1024 floats: two candidates per warp at a time, their row loads in flight together (each
    // dot in warp_dot's order; the best is order-independent).  Measured (profiles/r02/ab/ab_dot2_r02q.txt):
    // c3 +1.5 %, c2 / c5 +-0; at c4 (8 KB rows) -1 %, so wider rows keep one at a time.
    constexpr int NWR = T / 32;
    constexpr int PAIR = (T * CH <= 256) ? 2 : 1;
    for (int j = warp; j < count; j += PAIR * NWR) {
      if constexpr (PAIR == 1) {
        const int n = cand_at(j);
        if (n >= 0) consider(n, warp_dot(rrow, reinterpret_cast<const float4*>(a.At + (int64_t)n * a.Mp), q4, lane));
        continue;
      }
      const int n1 = cand_at(j), n2 = cand_at(j + NWR);
      if (n1 >= 0 && n2 >= 0) {
        const float2 c = warp_dot2(rrow, reinterpret_cast<const float4*>(a.At + (int64_t)n1 * a.Mp),
                                   reinterpret_cast<const float4*>(a.At + (int64_t)n2 * a.Mp), q4, lane);
        consider(n1, c.x);
        consider(n2, c.y);
      } else if (n1 >= 0 || n2 >= 0) {
        const int n = n1 >= 0 ? n1 : n2;
        consider(n, warp_dot(rrow, reinterpret_cast<const float4*>(a.At + (int64_t)n * a.Mp), q4, lane));
      }
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
  } else if constexpr (SEL == SEL_PROJ) {
    // exact argmax over the projections p_n = <r_k, a_n> (FP32): lowest index on ties
    const float rn = a.resid[b];
    const float* prow = a.R32in + (int64_t)cur_slot * a.Mp;
    Cand best{-1.f, 0x7fffffff, 0.f};
    bool nan_c = false;
    for (int64_t n = tid; n < a.N; n += T) {
      const float c = prow[n];
      nan_c |= isnan(c);
      const Cand cd{fabsf(c) * a.inv_norm[n], (int)n, c};
      if (cand_better(cd, best)) best = cd;
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      const Cand oth{__shfl_xor_sync(0xffffffffu, best.w, o), __shfl_xor_sync(0xffffffffu, best.n, o),
                     __shfl_xor_sync(0xffffffffu, best.c, o)};
      if (cand_better(oth, best)) best = oth;
    }
    if (lane == 0) red_c[warp] = best;
    const int any_nan = __syncthreads_or(nan_c);
    if (tid == 0) {
      Cand r = red_c[0];
#pragma unroll
      for (int i = 1; i < T / 32; ++i)
        if (cand_better(red_c[i], r)) r = red_c[i];
      const bool ok = r.w > 0.f && r.n < a.N;
      // (the u-based ||r|| is not used here: it can cancel to 0 while r is not; max |p| decides)
      if (!isfinite(rn) || any_nan) sel_n = SEL_NAN;
      else if (!ok) sel_n = SEL_DEGENERATE;
      else sel_n = r.n;
      sel_c = ok ? r.c : 0.f;
    }
  } else {
    if (tid == 0) {
      sel_n = a.nstar[b];
      sel_c = a.cstar[b];
    }
  }
  asm volatile("cp.async.wait_all;" ::: "memory");     // ss, u (SIMT path: first wait)
  __syncthreads();
  UPD_TRACE(2);
  const int n = sel_n;
  if (n < 0) {
    if (tid == 0) a.status[b] = (n == SEL_NAN) ? OMP_SIG_NAN : OMP_SIG_DEGENERATE;
    return;
  }
  const TailSmem sm{w, z, u, xs, ss, ro, red, reinterpret_cast<float*>(dsm), &sel_n};
  // the append's load depth: one CTA per SM (MINB = 1: a few signals, F_k of a large S in L2) keeps 4 z
  // columns x 8 rows and 16 sweep columns in flight; otherwise occupancy hides the latency
  constexpr int ZCK = (T == 32) ? OMP_ZC32 : (MINB == 1 ? 4 : kZC);
#ifndef OMP_FEW_ZR
#define OMP_FEW_ZR 8
#endif
#ifndef OMP_FEW_FZN
#define OMP_FEW_FZN 16
#endif
  constexpr int ZRK = (MINB == 1) ? OMP_FEW_ZR : 4;
  constexpr int FZN = FSM ? 0 : (MINB == 1 ? OMP_FEW_FZN : 8);
#ifdef OMP_UPDATE_TRACE
  append_residual<T, CH, P, ZCK, SEL == SEL_PROJ, FZN, FSM && (T <= OMP_ZLANE_TMAX), ZRK>(a, b, k, n, sel_c, sm, FSM ? Fs : a.F + b * a.ldf, nullptr, nullptr,
                                                        &upd_t0_);
  UPD_TRACE(11);
  if (threadIdx.x == 0 && a.k == g_upd_trace_k) atomicAdd(&g_upd_clk[15], 1ull);
  if (freq_cta) upd_freq_mark(b == 0 ? 1 : 3);
#else
  append_residual<T, CH, P, ZCK, SEL == SEL_PROJ, FZN, FSM && (T <= OMP_ZLANE_TMAX), ZRK>(a, b, k, n, sel_c, sm, FSM ? Fs : a.F + b * a.ldf, nullptr);
#endif
}

template <int SEL, int T, int CH, int MINB = (OMP_UPDATE_CTAS / T < 32 ? OMP_UPDATE_CTAS / T : 32), int P = 2>
static cudaError_t launch_t(const UpdateArgs& a, int64_t B, size_t smem_rest, size_t persist, cudaStream_t st) {
  auto kern = k_update<SEL, T, CH, MINB, P>;
  const size_t smem = smem_rest + update_region0<T, CH>(SEL == SEL_SCREEN || SEL == SEL_SCREEN_FSM, a.Mp);
  // static + dynamic shared memory may exceed the 48 KB default: opt in once per variant
  // (a function attribute is per device: one opt-in per device this process launches on)
  static std::atomic<uint64_t> opted{0};
  {
    int dev_ = 0;
    if (cudaGetDevice(&dev_) != cudaSuccess) return cudaGetLastError();
    const uint64_t bit = 1ull << (dev_ & 63);
    if (!(opted.load(std::memory_order_acquire) & bit)) {
      cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, 160 * 1024);
      if (e != cudaSuccess) return e;
      opted.fetch_or(bit, std::memory_order_acq_rel);
    }
  }
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3((unsigned)B);
  cfg.blockDim = dim3(T);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute attr[2];
  if ((SEL == SEL_SCREEN || SEL == SEL_SCREEN_FSM) && pdl_enabled(2)) {
    attr[cfg.numAttrs].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[cfg.numAttrs].val.programmaticStreamSerializationAllowed = 1;
    cfg.numAttrs++;
  }
  if (persist > 0) {
    // keep the fp32 atom table (re-read by every signal's gather) in the persisting L2 carve-out;
    // a launch attribute, so the caller's stream is left untouched
    cudaLaunchAttribute& w = attr[cfg.numAttrs++];
    w.id = cudaLaunchAttributeAccessPolicyWindow;
    w.val.accessPolicyWindow.base_ptr = const_cast<float*>(a.At);
    w.val.accessPolicyWindow.num_bytes = persist;
    w.val.accessPolicyWindow.hitRatio = 1.0f;
    w.val.accessPolicyWindow.hitProp = cudaAccessPropertyPersisting;
    w.val.accessPolicyWindow.missProp = cudaAccessPropertyStreaming;
  }
  cfg.attrs = attr;
  return cudaLaunchKernelEx(&cfg, kern, a);
}

// (T, CH) for the row width; "few" = at most 2 CTAs per SM in the whole launch; "mid" = the whole launch
// resident at once with at most 8 CTAs per SM: the per-signal chain sets the launch time, so each thread
// keeps 8 float4 chunks (8 / CH rows) in flight in the gather instead of 2 rows.  Measured (graph path,
// profiles/r02/ab/ab_mid_r02m.txt): c2 +2.8 %, M = 1024 at B = 10^3 +2.7 %, t2m1024 at B = 10^3 +6.6 %,
// but c5 at B = 10^3 (T = 128, CH = 1) -1.2 %, which therefore keeps 2.  OMP_B200_MID=0: off (A/B)
#ifndef OMP_FEW_TMAX
#define OMP_FEW_TMAX 512
#endif
template <int SEL, int T, int CH>
static cudaError_t launch_tc(const UpdateArgs& a, int64_t B, size_t smem, size_t persist, bool few, bool mid,
                             cudaStream_t st) {
  constexpr int Q = T * CH;
  if (few && (SEL != SEL_SCREEN_FSM || Q >= 512)) {
    // at most 2 CTAs per SM: wider CTAs (up to 512 threads, one float4 chunk each while the row allows)
    // so the append's column dots and row sweeps of a large S run on more warps.  Measured
    // (profiles/r02/ab/ab_few_r02v.txt, ab_few2_r02w.txt): t2m2048 (S = 512) 2.04x, t2m1024 +29 %, c4 at
    // B = 100 +31 %; with F_k still in shared memory and rows of <= 1024 floats the wide CTA lost (c3 at
    // B = 200: -8 %), so there it keeps (T, CH).
    constexpr int TF = Q < OMP_FEW_TMAX ? Q : OMP_FEW_TMAX;
    constexpr int CHF = Q / TF;
    return launch_t<SEL, TF, CHF, 1, (16 / CHF > 2 ? 16 / CHF : 2)>(a, B, smem, persist, st);
  }
  if (few) return launch_t<SEL, T, CH, 1, (16 / CH > 2 ? 16 / CH : 2)>(a, B, smem, persist, st);
  if constexpr ((T <= 64 && CH <= 2) || (T == 128 && CH == 2))
    if (mid) return launch_t<SEL, T, CH, 8, (8 / CH > 2 ? 8 / CH : 2)>(a, B, smem, persist, st);
  constexpr int MINB = (OMP_UPDATE_CTAS / T < 32 ? OMP_UPDATE_CTAS / T : 32);
#ifndef OMP_P32
#define OMP_P32 2
#endif
  constexpr int P = (T == 32 && CH == 4) ? OMP_P32 : (OMP_UPDATE_PCH / CH > 2 ? OMP_UPDATE_PCH / CH : 2);
  return launch_t<SEL, T, CH, MINB, P>(a, B, smem, persist, st);
}

template <int SEL>
static cudaError_t launch_r(const UpdateArgs& a, int64_t B, size_t smem, size_t persist, cudaStream_t st) {
  // float4 chunks per row -> (T, CH), T * CH == q4 at powers of two.  No floating-point result
  // depends on T (the tail's reductions run in T-independent orders), so the map may depend on the
  // batch size and differ from k_small.cu's: a signal's result is the same whichever kernel and block
  // size processed it.
  static int sms = 0;
  if (!sms) {
    int dev = 0;
    if (cudaGetDevice(&dev) != cudaSuccess || cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess)
      sms = 148;
  }
  const bool few = B <= 2 * (int64_t)sms;
  static int mid_env = -1;
  if (mid_env < 0) {
    const char* e = getenv("OMP_B200_MID");
    mid_env = (e && e[0] == '0') ? 0 : 1;
  }
  static int64_t mid_maxb = -1;       // OMP_B200_MID_MAXB: the largest batch that takes "mid" (A/B)
  if (mid_maxb < 0) {
    const char* e = getenv("OMP_B200_MID_MAXB");
    mid_maxb = e ? atoll(e) : 8 * (int64_t)sms;
  }
  const bool mid = mid_env && B <= mid_maxb;
  const int64_t q4 = a.Mp / 4;
  // Large batches of narrow rows (many waves: throughput) take one warp per signal and 32 signals per
  // SM; smaller batches keep the wider CTAs, whose shorter per-signal chain sets the launch time when
  // the whole batch is resident at once.  Measured (c5, M = 512): T = 32 vs 128 +14 % at B = 10^4,
  // +24 % at 10^5, but -24 % at B = 10^3 and -30 % at 100; c3 (M = 1024, B = 10^4, eps stops): T = 64
  // vs 128 -11 % -- hence only M <= 512 and B >= 8192.
  const bool wide_batch = B >= 8192;
  if (q4 <= 32) return launch_tc<SEL, 32, 1>(a, B, smem, persist, few, mid, st);
  if (q4 <= 64) return wide_batch ? launch_tc<SEL, 32, 2>(a, B, smem, persist, few, mid, st)
                                  : launch_tc<SEL, 64, 1>(a, B, smem, persist, few, mid, st);
  if (q4 <= 128) return wide_batch ? launch_tc<SEL, 32, 4>(a, B, smem, persist, few, mid, st)
                                   : launch_tc<SEL, 128, 1>(a, B, smem, persist, few, mid, st);
#ifndef OMP_Q256_T
#define OMP_Q256_T 128
#endif
  if (q4 <= 256) return launch_tc<SEL, OMP_Q256_T, 256 / OMP_Q256_T>(a, B, smem, persist, few, mid, st);
  if (q4 <= 512) return launch_tc<SEL, 128, 4>(a, B, smem, persist, few, mid, st);
  if (q4 <= 1024) return launch_tc<SEL, 256, 4>(a, B, smem, persist, few, mid, st);
  if (q4 <= 2048) return launch_tc<SEL, 256, 8>(a, B, smem, persist, few, mid, st);
  return cudaErrorNotSupported;   // M > 8192
}

cudaError_t launch_update(const UpdateLaunch& L, cudaStream_t st) {
  if (L.B == 0) return cudaSuccess;
  UpdateArgs a;
  a.k = L.k; a.S = L.S; a.eps = L.eps; a.N = L.N; a.M = L.M; a.Mp = L.Mp;
  a.part = L.part; a.groups = L.groups; a.rslot_in = L.rslot_in; a.win = L.win; a.nstar = L.nstar; a.cstar = L.cstar;
  a.At = L.At; a.inv_norm = L.inv_norm; a.G = L.G; a.ldg = L.ldg;
  a.Y = L.Y; a.ldy = L.ldy; a.F = L.F; a.ldf = L.ldf; a.U = L.U; a.ldu = L.ldu; a.X = L.X; a.ldx = L.ldx;
  a.support = L.support; a.lds = L.lds; a.R32in = L.R32in; a.R32 = L.R32; a.Rb = (__nv_bfloat16*)L.Rb;
  a.Rhi = L.Rhi; a.Rlo = L.Rlo; a.rslot_out = L.rslot_out; a.slot = L.slot; a.live_next = L.live_next;
  a.resid = L.resid; a.n_iter = L.n_iter; a.status = L.status; a.ynorm2 = L.ynorm2;
  a.At_res = L.At_res; a.Mp_res = L.Mp_res; a.M_res = L.M_res; a.Y_res = L.Y_res; a.ldy_res = L.ldy_res;
  const bool refine = L.part != nullptr;
  const int64_t Sp = (L.k + 4) & ~3;
  // F_k staged in shared memory while it is small and the batch is latency-bound (< 8192 signals);
  // the big batches keep their occupancy (measured: c2, c5 B <= 10^3)
  const int64_t fk = ((int64_t)L.k * (L.k + 1) / 2 + 3) & ~3;
  // (large batches: only up to M = 1024 -- c5 B = 10^4 +2..5 %, c3 B = 3 x 10^4 +1 %; at c4 it cost 0.5 %)
#ifndef OMP_FSM_MP_MAX
#define OMP_FSM_MP_MAX 1024
#endif
  a.fsm = (refine && fk * 4 <= kFsmMaxBytes && (L.B < 8192 || L.Mp <= OMP_FSM_MP_MAX)) ? 1 : 0;
  // the kept entries of one signal are at most groups x TOPK: a list that size never overflows
  a.candcap = refine ? (int)min((int64_t)RF_CAP, (int64_t)L.groups * TOPK) : 0;
  // (without the first region, whose size depends on the block size: update_region0)
  const size_t smem = (size_t)Sp * 6 * 4 + (size_t)a.candcap * 4 + (a.fsm ? (size_t)fk * 4 : 0);
  if (refine) return a.fsm ? launch_r<SEL_SCREEN_FSM>(a, L.B, smem, L.l2_persist_bytes, st)
                           : launch_r<SEL_SCREEN>(a, L.B, smem, L.l2_persist_bytes, st);
  if (L.ynorm2) return launch_r<SEL_PROJ>(a, L.B, smem, L.l2_persist_bytes, st);
  return launch_r<SEL_GIVEN>(a, L.B, smem, L.l2_persist_bytes, st);
}

}  // namespace ompb

#ifdef OMP_UPDATE_TRACE
extern "C" int omp_debug_update_trace(int k, unsigned long long* host16) {
  // host16 == nullptr: arm the trace for iteration k (clears the sums); else read them back
  if (!host16) {
    unsigned long long z[16] = {};
    cudaError_t e = cudaMemcpyToSymbol(g_upd_clk, z, sizeof(z));
    if (e == cudaSuccess) e = cudaMemcpyToSymbol(g_upd_trace_k, &k, sizeof(int));
    return (int)e;
  }
  return (int)cudaMemcpyFromSymbol(host16, g_upd_clk, sizeof(unsigned long long) * 16);
}

extern "C" int omp_debug_update_freq(unsigned long long* host8) {
  return (int)cudaMemcpyFromSymbol(host8, g_upd_freq, sizeof(unsigned long long) * 8);
}
#endif
