// Small-batch path (PAPER.md:243 on per-call overhead at small batch sizes):
// ONE persistent cooperative kernel runs all S iterations of a small batch, with two grid barriers
// per iteration instead of two kernel launches.
//
//   phase A  every warp of the grid owns a strided set of atoms; it holds atom n's fp32 row in
//            registers and computes the exact FP32 correlation c_bn = <r_b, a_n> (warp_dot_regs: the
//            same instructions in the same order as the refine of the screened path) with each live
//            signal's residual row, staged in shared memory.  Per (signal, CTA) it keeps the best
//            (|c| / ||a_n||, lowest n) and a NaN flag -> pbest[b][cta].
//   barrier
//   phase B  CTA b (b < B, stride G) reduces pbest[b][*] to n*_b, c*_b and runs the
//            factor append + residual of update_core.cuh (a4, a5) for signal b.
//   barrier
//
// No screen is needed: at this batch size the exact FP32 correlation over all N atoms costs about
// what the screen would.  Since phase A evaluates every atom with the refine's arithmetic, n* is the
// exact FP32 argmax that the screen + refine path also finds (the screen's window is rigorous), and
// the append/residual code is shared, a signal's result is bitwise the same on both paths.
//
// Coherence: per-signal state (F, u, x, support, ||r||) is only touched by the CTA that owns the
// signal (b mod G), so it never crosses SMs.  Data that does (residual rows, statuses, partials)
// is written before a barrier and read after it with ld.global.cg (L2), never from L1.
#include <math.h>

#include <atomic>
#include <stdlib.h>

#include "omp_internal.cuh"
// diagnostic timeline of the shared tail (CTA 0, clock64 at 6 points per iteration)
__device__ unsigned long long g_tail_clk[ompb::MAX_S * 8];
#define OMP_TAIL_TRACE(p)                                                      \
  do {                                                                         \
    if (blockIdx.x == 0 && threadIdx.x == 0) g_tail_clk[k * 8 + (p)] = clock64(); \
  } while (0)
#include "update_core.cuh"

namespace ompb {


// diagnostic timeline (OMP_B200_SMALL_TRACE=1): globaltimer of CTA 0 at 7 points per iteration
__device__ unsigned long long g_small_trace[MAX_S * 8];
__device__ unsigned long long g_small_clk[MAX_S * 8];
__device__ __forceinline__ void trace_pt(int on, int k, int p) {
  if (on && blockIdx.x == 0 && threadIdx.x == 0) {
    unsigned long long t;
    asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
    g_small_trace[k * 8 + p] = t;
    g_small_clk[k * 8 + p] = clock64();
  }
}

constexpr int SMALL_PB = 4;   // partial loads in flight per thread in the selection

struct SmallArgs {
  UpdateArgs a;            // k is set per iteration; R32 = the residual rows (row b), slot/live_next null
  int64_t B;
  float4* pbest;           // B x G: (w, n, c, nan) per (signal, CTA)
  unsigned int* bar;       // grid barrier counter (zero at launch)
  int ja;                  // > 0: each warp keeps its (<= ja) atoms in shared memory for the whole run
  int rows;                // 1: the owned signal's support rows are cached in shared memory
  int trace;
};

__device__ __forceinline__ void grid_barrier(unsigned int* bar, unsigned int target) {
  __syncthreads();
  if (threadIdx.x == 0) {
    // release: this CTA's writes (ordered before by bar.sync) are visible to whoever acquires the
    // count; cheaper than a full membar.gl + relaxed atomic
    asm volatile("red.release.gpu.global.add.u32 [%0], 1;" ::"l"(bar) : "memory");
    unsigned int v;
    do {
      asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(bar) : "memory");
    } while (v < target);
  }
  __syncthreads();
}

template <int T, int CH, int KC>
__global__ void __launch_bounds__(T, 1) k_small(const SmallArgs s) {
  constexpr int NW = T / 32;
  const int G = gridDim.x, cta = blockIdx.x;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  UpdateArgs a = s.a;
  const int64_t B = s.B;
  const int q4 = (int)(a.Mp >> 2);
  const int Sp = (a.S + 3) & ~3;
  const int64_t fsz = ((int64_t)a.S * (a.S + 1) / 2 + 3) & ~3;
  // dynamic shared memory: [residual rows: B x Mp floats] [atom cache: NW x ja x Mp floats]
  //   [support-row cache: S x Mp floats, if rows] [F of the owned signal: fsz floats]
  //   [w, z, u, xs: Sp floats] [ss, ro: Sp ints]
  // The owned signal's F, support and u stay in shared memory for the whole run (B <= G: a CTA owns
  // at most one signal); every new column also goes to global memory (ompGetFactor).
  extern __shared__ __align__(16) uint8_t dsm[];
  float4* rs = reinterpret_cast<float4*>(dsm);
  float4* atoms = reinterpret_cast<float4*>(dsm + (size_t)B * a.Mp * 4);   // [warp][j][q4]
  float4* rows_sm = atoms + (size_t)NW * s.ja * q4;
  float* Fsm = reinterpret_cast<float*>(rows_sm) + (s.rows ? (size_t)a.S * a.Mp : 0);
  float* w = Fsm + fsz;
  float* z = w + Sp;
  float* u = z + Sp;
  float* xs = u + Sp;
  int* ss = reinterpret_cast<int*>(xs + Sp);
  uint32_t* ro = reinterpret_cast<uint32_t*>(ss + Sp);
  __shared__ float red[NW];
  __shared__ Cand wb[NW][SMALL_MAX_B];
  __shared__ int wn[NW][SMALL_MAX_B];
  __shared__ int lb[SMALL_MAX_B];
  __shared__ int nlive_s;
  __shared__ int sel_n;
  __shared__ float sel_c;
  __shared__ float rn_s;
  __shared__ Cand red_c[NW];
  __shared__ int red_nan[NW];
  const TailSmem sm{w, z, u, xs, ss, ro, red, reinterpret_cast<float*>(rs), &sel_n};   // (rs is free in the tail)
  const int64_t b = cta;                 // the signal this CTA owns (if b < B)
  unsigned int epoch = 0;
  const int64_t gstride = (int64_t)G * NW;
  // the dictionary is fixed: each warp's atoms (n = cta NW + warp + j G NW) are loaded once
  for (int j = 0; j < s.ja; ++j) {
    const int64_t n = (int64_t)cta * NW + warp + j * gstride;
    if (n < a.N) {
      const float4* a4 = reinterpret_cast<const float4*>(a.At + n * a.Mp);
      for (int q = lane; q < q4; q += 32) atoms[((size_t)warp * s.ja + j) * q4 + q] = __ldg(a4 + q);
    }
  }

  for (int k = 0; k < a.S; ++k) {
    a.k = k;
    trace_pt(s.trace, k, 0);
    // ---- live signals (every CTA derives the same list from the statuses); all B residual rows are
    // staged at once (cp.async.cg: L2 -> shared, never a stale L1 line), overlapping the status reads
    for (int i = 0; i < B; ++i) {
      const float4* src = reinterpret_cast<const float4*>(a.R32 + (int64_t)i * a.Mp);
      for (int q = tid; q < q4; q += T) cp_async16(&rs[(size_t)i * q4 + q], src + q);
    }
    asm volatile("cp.async.commit_group;" ::: "memory");
    if (tid == 0) {
      int nl = 0;
      for (int i = 0; i < B; ++i)
        if (__ldcg(a.status + i) == SIG_RUNNING) lb[nl++] = i;
      nlive_s = nl;
    }
    for (int e = tid; e < NW * SMALL_MAX_B; e += T) {
      wb[e / SMALL_MAX_B][e % SMALL_MAX_B] = Cand{-1.f, 0x7fffffff, 0.f};
      wn[e / SMALL_MAX_B][e % SMALL_MAX_B] = 0;
    }
    asm volatile("cp.async.wait_all;" ::: "memory");
    __syncthreads();
    const int nlive = nlive_s;
    if (nlive == 0) break;                       // uniform over the grid
    trace_pt(s.trace, k, 1);

    // ---- phase A: exact correlations, atoms strided over the warps of the grid ----
    int ja_i = 0;
    for (int64_t n = (int64_t)cta * NW + warp; n < a.N; n += gstride, ++ja_i) {
      float4 areg[KC];
      if (ja_i < s.ja) {
        const float4* a4 = atoms + ((size_t)warp * s.ja + ja_i) * q4;
#pragma unroll
        for (int i = 0; i < KC; ++i) {
          const int q = lane + 32 * i;
          areg[i] = q < q4 ? a4[q] : make_float4(0.f, 0.f, 0.f, 0.f);
        }
      } else {
        const float4* a4 = reinterpret_cast<const float4*>(a.At + n * a.Mp);
#pragma unroll
        for (int i = 0; i < KC; ++i) {
          const int q = lane + 32 * i;
          areg[i] = q < q4 ? __ldg(a4 + q) : make_float4(0.f, 0.f, 0.f, 0.f);
        }
      }
      const float inv = __ldg(a.inv_norm + n);
      auto take = [&](int i, float c) {
        if (lane == 0) {
          const Cand cd{fabsf(c) * inv, (int)n, c};
          if (isnan(c)) wn[warp][i] = 1;
          if (cand_better(cd, wb[warp][i])) wb[warp][i] = cd;
        }
      };
      int i = 0;
      for (; i + 2 <= nlive; i += 2) {   // two independent dot chains in flight
        const float c0 = warp_dot_regs<KC>(rs + (size_t)lb[i] * q4, areg, q4, lane);
        const float c1 = warp_dot_regs<KC>(rs + (size_t)lb[i + 1] * q4, areg, q4, lane);
        take(i, c0);
        take(i + 1, c1);
      }
      if (i < nlive) take(i, warp_dot_regs<KC>(rs + (size_t)lb[i] * q4, areg, q4, lane));
    }
    __syncthreads();
    for (int i = tid; i < nlive; i += T) {
      Cand r = wb[0][i];
      int nan = wn[0][i];
#pragma unroll
      for (int v = 1; v < NW; ++v) {
        if (cand_better(wb[v][i], r)) r = wb[v][i];
        nan |= wn[v][i];
      }
      s.pbest[(int64_t)lb[i] * G + cta] = make_float4(r.w, __int_as_float(r.n), r.c, __int_as_float(nan));
    }
    trace_pt(s.trace, k, 2);
    grid_barrier(s.bar, (++epoch) * (unsigned)G);
    trace_pt(s.trace, k, 3);

    // ---- phase B: selection + append + residual of the signal this CTA owns ----
    if (b < B && __ldcg(a.status + b) == SIG_RUNNING) {   // uniform over the CTA
      if (tid == 0) rn_s = a.resid[b];                     // in flight with the partials
      {
        const char* yp = reinterpret_cast<const char*>(a.Y + b * a.ldy);
        for (int64_t o = (int64_t)tid * 128; o < a.M * 4; o += (int64_t)T * 128)
          asm volatile("prefetch.global.L2 [%0];" ::"l"(yp + o));
      }
      Cand best{-1.f, 0x7fffffff, 0.f};
      int nan = 0;
      // every partial load in flight before any is consumed (G <= SMALL_PB * T per pass)
      for (int g0 = 0; g0 < G; g0 += SMALL_PB * T) {
        float4 pv[SMALL_PB];
#pragma unroll
        for (int i = 0; i < SMALL_PB; ++i) {
          const int g = g0 + i * T + tid;
          pv[i] = g < G ? __ldcg(s.pbest + b * G + g) : make_float4(-1.f, __int_as_float(0x7fffffff), 0.f, 0.f);
        }
#pragma unroll
        for (int i = 0; i < SMALL_PB; ++i) {
          const Cand cd{pv[i].x, __float_as_int(pv[i].y), pv[i].z};
          nan |= __float_as_int(pv[i].w);
          if (cand_better(cd, best)) best = cd;
        }
      }
      trace_pt(s.trace, k, 7);
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) {
        const Cand oth{__shfl_xor_sync(0xffffffffu, best.w, o), __shfl_xor_sync(0xffffffffu, best.n, o),
                       __shfl_xor_sync(0xffffffffu, best.c, o)};
        if (cand_better(oth, best)) best = oth;
        nan |= __shfl_xor_sync(0xffffffffu, nan, o);
      }
      if (lane == 0) {
        red_c[warp] = best;
        red_nan[warp] = nan;
      }
      __syncthreads();
      if (tid == 0) {
        Cand r = red_c[0];
        int any_nan = red_nan[0];
#pragma unroll
        for (int v = 1; v < NW; ++v) {
          if (cand_better(red_c[v], r)) r = red_c[v];
          any_nan |= red_nan[v];
        }
        // the screened path's order of tests (k_update.cu): non-finite ||r|| -> NaN; r = 0 ->
        // degenerate; a NaN correlation -> NaN; no positive correlation -> degenerate
        const float rn = rn_s;
        if (!isfinite(rn)) sel_n = SEL_NAN;
        else if (rn == 0.f) sel_n = SEL_DEGENERATE;
        else {
          const bool ok = r.w > 0.f && r.n < a.N;
          sel_n = any_nan ? SEL_NAN : (ok ? r.n : SEL_DEGENERATE);
        }
        sel_c = r.c;
      }
      __syncthreads();
      trace_pt(s.trace, k, 4);
      const int n = sel_n;
      if (n < 0) {
        if (tid == 0) a.status[b] = (n == SEL_NAN) ? OMP_SIG_NAN : OMP_SIG_DEGENERATE;
      } else {
        if (s.rows) {   // the new support row joins the cache (lands while the append runs)
          const float4* src = reinterpret_cast<const float4*>(a.At + (int64_t)n * a.Mp);
          for (int q = tid; q < q4; q += T) cp_async16(rows_sm + (size_t)k * q4 + q, src + q);
          asm volatile("cp.async.commit_group;" ::: "memory");
        }
        // one CTA per signal on the critical path: F_k (and, if cached, the support rows) from shared
        // memory; 8 rows in flight, 8 z columns per warp
        append_residual<T, CH, 8, 8, false, 0>(a, b, k, n, sel_c, sm, Fsm, Fsm,
                                                                  s.rows ? rows_sm : nullptr);
      }
      __syncthreads();
      trace_pt(s.trace, k, 5);
    }
    grid_barrier(s.bar, (++epoch) * (unsigned)G);
    trace_pt(s.trace, k, 6);
  }
}

template <int T, int CH, int KC>
static cudaError_t launch_s(SmallArgs s, size_t smem0, int ctas_per_sm, cudaStream_t st) {
  auto kern = k_small<T, CH, KC>;
  constexpr size_t kMaxSmem = 200 * 1024;
  // (a function attribute is per device: one opt-in per device this process launches on)
  static std::atomic<uint64_t> opted{0};
  {
    int dev_ = 0;
    if (cudaGetDevice(&dev_) != cudaSuccess) return cudaGetLastError();
    const uint64_t bit = 1ull << (dev_ & 63);
    if (!(opted.load(std::memory_order_acquire) & bit)) {
      cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kMaxSmem);
      if (e != cudaSuccess) return e;
      opted.fetch_or(bit, std::memory_order_acq_rel);
    }
  }
  int dev = 0, sms = 0, occ = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e == cudaSuccess) e = cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  if (e != cudaSuccess) return e;
  // grid = SMs x per_sm co-resident CTAs.  Shared-memory caches, in order of value: the owned
  // signal's support rows (the gather then reads shared memory instead of L2: a single SM's L2
  // bandwidth bounds it otherwise), and each warp's atoms (phase A).  Take the first configuration
  // that fits, preferring caches over CTAs per SM.
  size_t smem = smem0;
  int ja = 0, rows = 0, per_sm = 0;
  const size_t rows_bytes = (size_t)s.a.S * s.a.Mp * 4;
  bool found = false;
  for (int cfg_i = 0; cfg_i < 4 && !found; ++cfg_i) {
    const int want_rows = cfg_i < 2, want_atoms = (cfg_i % 2) == 0;
    for (int ps = ctas_per_sm; ps >= 1 && !found; --ps) {
      const int64_t G = (int64_t)sms * ps;
      const int64_t jneed = (s.a.N + G * (T / 32) - 1) / (G * (T / 32));
      const size_t need = smem0 + (want_rows ? rows_bytes : 0) +
                          (want_atoms ? (size_t)(T / 32) * jneed * s.a.Mp * 4 : 0);
      if (need > kMaxSmem) continue;
      e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kern, T, need);
      if (e != cudaSuccess) return e;
      if (occ >= ps) {
        found = true;
        smem = need;
        per_sm = ps;
        ja = want_atoms ? (int)jneed : 0;
        rows = want_rows;
      }
    }
  }
  if (!found) return cudaErrorNotSupported;
  if (per_sm < 1) return cudaErrorNotSupported;
  if ((int64_t)sms * per_sm < s.B) return cudaErrorNotSupported;   // a CTA owns at most one signal
  s.ja = ja;
  s.rows = rows;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3((unsigned)(sms * per_sm));
  cfg.blockDim = dim3(T);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeCooperative;   // all CTAs co-resident: the grid barrier is safe
  attr[0].val.cooperative = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, kern, s);
}

int64_t small_path_smem(int64_t B, int64_t Mp, int32_t S) {
  return B * Mp * 4 + ((((int64_t)S * (S + 1) / 2) + 3) & ~3) * 4 + (int64_t)((S + 3) & ~3) * 6 * 4;
}

bool small_path_supported(int64_t B, int64_t Mp, int32_t S) {
  return B >= 1 && B <= SMALL_MAX_B && Mp <= 2048 && small_path_smem(B, Mp, S) <= 190 * 1024;
}

cudaError_t launch_small(const UpdateLaunch& L, float4* pbest, unsigned int* bar, cudaStream_t st) {
  if (!small_path_supported(L.B, L.Mp, L.S)) return cudaErrorNotSupported;
  SmallArgs s;
  UpdateArgs& a = s.a;
  a.k = 0; a.S = L.S; a.fsm = 0; a.eps = L.eps; a.N = L.N; a.M = L.M; a.Mp = L.Mp;
  a.part = nullptr; a.groups = 0; a.candcap = 0; a.rslot_in = nullptr; a.win = WinCoef{0.f, 0.f, 0.f}; a.nstar = nullptr;
  a.cstar = nullptr;
  a.At = L.At; a.inv_norm = L.inv_norm; a.G = L.G; a.ldg = L.ldg;
  a.Y = L.Y; a.ldy = L.ldy; a.F = L.F; a.ldf = L.ldf; a.U = L.U; a.ldu = L.ldu; a.X = L.X; a.ldx = L.ldx;
  a.support = L.support; a.lds = L.lds; a.R32in = L.R32; a.R32 = L.R32;
  a.Rb = nullptr; a.Rhi = nullptr; a.Rlo = nullptr; a.rslot_out = nullptr; a.slot = nullptr; a.live_next = nullptr;
  a.resid = L.resid; a.n_iter = L.n_iter; a.status = L.status; a.ynorm2 = nullptr;
  a.At_res = nullptr; a.Mp_res = 0; a.M_res = 0; a.Y_res = nullptr; a.ldy_res = 0;
  s.B = L.B;
  s.pbest = pbest;
  s.bar = bar;
  static int trace = -1;
  if (trace < 0) {
    const char* env = getenv("OMP_B200_SMALL_TRACE");
    trace = (env && env[0] == '1') ? 1 : 0;
  }
  s.trace = trace;
  const size_t smem = (size_t)small_path_smem(L.B, L.Mp, L.S);
  static int per_sm = -1;   // OMP_B200_SMALL_CTAS_PER_SM: CTAs per SM of the persistent grid (default 2)
  if (per_sm < 0) {
    const char* env = getenv("OMP_B200_SMALL_CTAS_PER_SM");
    per_sm = env ? atoi(env) : 2;
    if (per_sm < 1) per_sm = 1;
    if (per_sm > SMALL_MAX_CTAS_PER_SM) per_sm = SMALL_MAX_CTAS_PER_SM;
  }
  // (T, CH) per Mp: the tail's results do not depend on T (T-independent reduction orders), so the
  // small-batch path agrees bit for bit with the per-iteration kernel whatever block size each uses
  const int64_t q4 = L.Mp / 4;
  if (q4 <= 32) return launch_s<32, 1, 4>(s, smem, per_sm, st);
  if (q4 <= 64) return launch_s<64, 1, 4>(s, smem, per_sm, st);
  if (q4 <= 128) return launch_s<128, 1, 4>(s, smem, per_sm, st);
  if (q4 <= 256) return launch_s<128, 2, 8>(s, smem, per_sm, st);
  if (q4 <= 512) return launch_s<128, 4, 16>(s, smem, per_sm, st);
  return cudaErrorNotSupported;
}

}  // namespace ompb

// diagnostic: copy the last traced launch's timeline (S x 8 u64, ns) to host memory
extern "C" int omp_debug_tail_clk(unsigned long long* host, int S) {
  return (int)cudaMemcpyFromSymbol(host, g_tail_clk, sizeof(unsigned long long) * 8 * (size_t)S);
}
extern "C" int omp_debug_small_clk(unsigned long long* host, int S) {
  return (int)cudaMemcpyFromSymbol(host, ompb::g_small_clk, sizeof(unsigned long long) * 8 * (size_t)S);
}
extern "C" int omp_debug_small_trace(unsigned long long* host, int S) {
  return (int)cudaMemcpyFromSymbol(host, ompb::g_small_trace, sizeof(unsigned long long) * 8 * (size_t)S);
}
