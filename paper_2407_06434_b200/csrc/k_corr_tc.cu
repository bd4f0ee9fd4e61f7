// K1: the correlation C = A^T R as ONE batched GEMM (PAPER.md:204-212,
// "a single call to gemm") on the 5th-generation tensor cores, used as a SCREEN:
//   KIND_BF16  : C~ = bf16(A)' bf16(R)                       (kind::f16, 1 MMA per K step)
//   KIND_3XTF32: C~ = Ahi'Rhi + Ahi'Rlo + Alo'Rhi            (kind::tf32, 3 MMAs per K step)
// Measured on B200 (scripts/diag_accum.py): the tensor-core FP32 accumulator
// truncates, so even 3xTF32 drifts by ~1e-5 relative at K = 2048 — above the 1e-5 near-tie
// budget.  The kernel therefore does not decide the argmax; its epilogue emits, per signal and
// 256-atom tile, the top-4 candidates of |c~_n| / ||a_n||, and the refine kernel (k_refine.cu)
// re-evaluates every atom inside the rigorous error window c0 ||r|| in exact FP32.
// Blackwell-native structure:
//   * operands staged by TMA (cp.async.bulk.tensor, 128-byte swizzle) into an mbarrier ring;
//   * one elected thread issues tcgen05.mma into TMEM accumulators (UMMA M = 128 signals per
//     CTA, N = 256 atoms); two accumulators (2 x 256 of the 512 TMEM columns) so the epilogue of
//     tile i overlaps the MMAs of tile i+1; tcgen05.commit -> mbarrier hand-offs only;
//   * persistent grid (one CTA / CTA pair per SM), static tile schedule rasterised in groups of
//     GM row-blocks so concurrently running tiles share A and R slabs in L2;
//   * CG = 2: cta_group::2 pairs two SMs on a 256 x 256 tile (each CTA stages its 128 signal
//     rows and half of the atoms; the leader issues the MMA), halving per-SM operand traffic.
// Epilogues: MODE_STORE writes C~ (ompCorrelate, numerics tests); MODE_TOPK writes partials.
#include <cuda.h>
#include <cuda_bf16.h>
#include <stdio.h>
#include <stdlib.h>

#include "omp_internal.cuh"

namespace ompb {
namespace tc {

constexpr int BM = 128;       // signal rows per CTA (UMMA M per CTA)
constexpr int BN = 256;       // atoms per tile (UMMA N)
constexpr int GM = 16;        // row-blocks per raster group
// Epilogue warps EW: 8 (two per TMEM lane group, 128 columns each) or 16 (four per lane group, 64
// columns each, the two warps of a 128-atom partial group merging their in-window lists through shared
// memory).  At small K a tile's MMAs are short and 8 warps' epilogue is not hidden behind the next
// tile's (c5, K = 512: tensor pipe 50 % busy); at K = 2048 the 16 warps cost the MMA-bound screen 2 %.
// The launch picks 16 below K = OMP_EPI16_KMAX (measured, profiles/r02/ab/ab_epi16_r02ag.txt).
#ifndef OMP_EPI16_KMAX
#define OMP_EPI16_KMAX 1536
#endif
__host__ __device__ constexpr int epi_threads(int ew) { return 32 * ew; }
__host__ __device__ constexpr int num_threads(int ew) { return 128 + 32 * ew; }
// shared memory of the 16-warp epilogue: pair exchange (max, count) and each thread's kept entries
__host__ __device__ constexpr uint32_t epi_smem(int ew) {
  return ew == 16 ? (2u * 4u * 2u * 32u * 8u + 16u * 32u * TOPK * 8u) : 0u;
}
constexpr int MODE_STORE = 0, MODE_TOPK = 1;

// Operand kinds.  Every stage holds one 128-byte-wide K slab of each plane.
template <int KIND>
struct Kind;
template <>
struct Kind<KIND_BF16> {
  static constexpr int ELEM = 2, BK = 64, UK = 16, NPLANES = 1;
  static constexpr uint32_t FMT = 1;   // BF16
};
template <>
struct Kind<KIND_3XTF32> {
  static constexpr int ELEM = 4, BK = 32, UK = 8, NPLANES = 2;   // hi, lo
  static constexpr uint32_t FMT = 2;   // TF32
};

template <int KIND, int CG>
struct Cfg {
  using K_ = Kind<KIND>;
  static constexpr int BN_CTA = BN / CG;
  static constexpr uint32_t R_BYTES = BM * K_::BK * K_::ELEM;        // one plane of the R tile
  static constexpr uint32_t A_BYTES = BN_CTA * K_::BK * K_::ELEM;    // one plane of the A tile
  static constexpr uint32_t STAGE_BYTES = K_::NPLANES * (R_BYTES + A_BYTES);
  static constexpr int STAGES = (int)((200u * 1024u) / STAGE_BYTES) < 8 ? (int)((200u * 1024u) / STAGE_BYTES) : 8;
  static constexpr uint32_t SMEM = STAGES * STAGE_BYTES + 1024 /*align*/ + 256 /*barriers*/;   // + epi_smem(EW)
  static constexpr uint32_t IDESC = (1u << 4)                            // D = F32
                                    | (K_::FMT << 7) | (K_::FMT << 10)   // A, B formats
                                    | ((uint32_t)(BN >> 3) << 17)        // N
                                    | ((uint32_t)((BM * CG) >> 4) << 24);  // M
};

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}

__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  const uint32_t a = smem_u32(bar);
  uint32_t ok = 0;
  do {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
        "selp.u32 %0, 1, 0, p;\n\t}"
        : "=r"(ok)
        : "r"(a), "r"(parity)
        : "memory");
  } while (!ok);
}

__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
               : "memory");
}

// arrive on the barrier at the same offset in CTA rank 0 of the cluster (own CTA when CG = 1)
__device__ __forceinline__ void mbar_arrive_cta0(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cluster.b64 _, [%0];" ::"r"(smem_u32(bar) & 0xFEFFFFFFu)
               : "memory");
}

// 2-D TMA tile load with an L2 cache policy (A tiles: evict_last, they are re-read by every row block;
// residual tiles: evict_normal, they are re-read across the N tiles of their raster group)
template <int CG>
__device__ __forceinline__ void tma_load_2d(const CUtensorMap* map, uint64_t* bar, void* dst, int k, int row,
                                            uint64_t policy) {
  if constexpr (CG == 1) {
    asm volatile(
        "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint"
        " [%0], [%1, {%2, %3}], [%4], %5;"
        ::"r"(smem_u32(dst)), "l"(map), "r"(k), "r"(row), "r"(smem_u32(bar)), "l"(policy)
        : "memory");
  } else {
    asm volatile(
        "cp.async.bulk.tensor.2d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint"
        " [%0], [%1, {%2, %3}], [%4], %5;"
        ::"r"(smem_u32(dst)), "l"(map), "r"(k), "r"(row), "r"(smem_u32(bar) & 0xFEFFFFFFu), "l"(policy)
        : "memory");
  }
}

__device__ __forceinline__ uint64_t l2_policy(bool keep) {
  uint64_t p;
  if (keep) asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(p));
  else asm volatile("createpolicy.fractional.L2::evict_normal.b64 %0, 1.0;" : "=l"(p));
  return p;
}

// K-major, 128-byte-swizzled UMMA shared-memory descriptor (8-row x 128 B atoms, SBO = 1024 B)
__device__ __forceinline__ uint64_t desc_sw128(uint32_t addr) {
  return (uint64_t)((addr >> 4) & 0x3FFFu) | ((uint64_t)1 << 16) | ((uint64_t)(1024 >> 4) << 32) |
         ((uint64_t)1 << 46) | ((uint64_t)2 << 61);
}

template <int KIND, int CG>
__device__ __forceinline__ void mma(uint32_t tmem_d, uint64_t a, uint64_t b, uint32_t idesc, uint32_t acc) {
#define OMPB_MMA(KINDSTR, CGSTR)                                                   \
  asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"                   \
               "tcgen05.mma.cta_group::" CGSTR ".kind::" KINDSTR " [%0], %1, %2, %3, p;\n\t}" \
               ::"r"(tmem_d), "l"(a), "l"(b), "r"(idesc), "r"(acc) : "memory")
  if constexpr (KIND == KIND_BF16) {
    if constexpr (CG == 1) OMPB_MMA("f16", "1"); else OMPB_MMA("f16", "2");
  } else {
    if constexpr (CG == 1) OMPB_MMA("tf32", "1"); else OMPB_MMA("tf32", "2");
  }
#undef OMPB_MMA
}

template <int CG>
__device__ __forceinline__ void mma_commit(uint64_t* bar) {
  if constexpr (CG == 1) {
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];"
                 ::"r"(smem_u32(bar)) : "memory");
  } else {
    const uint16_t mask = 0x3;
    asm volatile(
        "tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;"
        ::"r"(smem_u32(bar)), "h"(mask) : "memory");
  }
}

__device__ __forceinline__ void fence_before() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void fence_after() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }

__device__ __forceinline__ void tmem_ld32(uint32_t taddr, float (&v)[32]) {
  uint32_t r[32];
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0, %1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, "
      "%13, %14, %15, %16, %17, %18, %19, %20, %21, %22, %23, %24, %25, %26, %27, %28, %29, %30, %31}, [%32];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
        "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15]),
        "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]),
        "=r"(r[24]), "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
      : "r"(taddr));
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
  for (int i = 0; i < 32; ++i) v[i] = __uint_as_float(r[i]);
}

// 64 columns in one load (one wait for twice the data: the epilogue's pass A is two of these per warp)
__device__ __forceinline__ void tmem_ld64(uint32_t taddr, float (&v)[64]) {
  uint32_t r[64];
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x64.b32 {%0, %1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, %14, %15, %16, %17, %18, %19, %20, %21, %22, %23, %24, %25, %26, %27, %28, %29, %30, %31, %32, %33, %34, %35, %36, %37, %38, %39, %40, %41, %42, %43, %44, %45, %46, %47, %48, %49, %50, %51, %52, %53, %54, %55, %56, %57, %58, %59, %60, %61, %62, %63}, [%64];\n\t"
      "tcgen05.wait::ld.sync.aligned;"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]), "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15]), "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]), "=r"(r[24]), "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31]), "=r"(r[32]), "=r"(r[33]), "=r"(r[34]), "=r"(r[35]), "=r"(r[36]), "=r"(r[37]), "=r"(r[38]), "=r"(r[39]), "=r"(r[40]), "=r"(r[41]), "=r"(r[42]), "=r"(r[43]), "=r"(r[44]), "=r"(r[45]), "=r"(r[46]), "=r"(r[47]), "=r"(r[48]), "=r"(r[49]), "=r"(r[50]), "=r"(r[51]), "=r"(r[52]), "=r"(r[53]), "=r"(r[54]), "=r"(r[55]), "=r"(r[56]), "=r"(r[57]), "=r"(r[58]), "=r"(r[59]), "=r"(r[60]), "=r"(r[61]), "=r"(r[62]), "=r"(r[63])
      : "r"(taddr)
      : "memory");
#pragma unroll
  for (int i = 0; i < 64; ++i) v[i] = __uint_as_float(r[i]);
}

__device__ __forceinline__ uint32_t cluster_rank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}

__device__ __forceinline__ void cluster_sync() {
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}

struct TileSched {
  int tiles_m, tiles_n;
  __device__ void coords(int t, int& tm, int& tn) const {
    const int per_group = GM * tiles_n;
    const int g = t / per_group;
    const int first = g * GM;
    const int gm = min(GM, tiles_m - first);
    const int local = t - g * per_group;
    tm = first + local % gm;
    tn = local / gm;
  }
};

struct EpiArgs {
  float* C;                 // MODE_STORE
  int64_t ldc;
  int64_t ncols;            // columns < ncols are stored
  const float* norm;        // MODE_STORE: ||a_n|| (the screen runs on normalised atoms)
  float2* part;             // MODE_TOPK: rows x (2 tiles_n) x TOPK {value, index bits}
  const int32_t* live_rows; // rows < *live_rows are live (live-set compaction); null: all rows
  const float* rslot;       // MODE_TOPK: ||r|| of the residual in each row
  float window;             // MODE_TOPK: screening window / ||r||
  int kslab;                // MODE_STORE split-K: K blocks per slab (0: one slab); slab z -> C + z zstride
  int64_t zstride;
};

struct Maps {
  CUtensorMap r[2];         // R planes (bf16: r[0]; 3xtf32: hi, lo)
  CUtensorMap a[2];         // A^T planes
};

template <int KIND, int CG, int MODE, int EW>
__global__ void __launch_bounds__(num_threads(EW), 1)
k1_corr_tc(const __grid_constant__ Maps maps, int rows, int num_kb, int tiles_m, int tiles_n, EpiArgs ep) {
  using C_ = Cfg<KIND, CG>;
  using K_ = Kind<KIND>;
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + C_::STAGES * C_::STAGE_BYTES);
  uint64_t* empty = full + C_::STAGES;
  uint64_t* tfull = empty + C_::STAGES;
  uint64_t* tempty = tfull + 2;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + 2);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint32_t rank = (CG == 2) ? cluster_rank() : 0u;
  const bool leader = rank == 0;
  const int cluster_id = blockIdx.x / CG, num_clusters = gridDim.x / CG;

  // programmatic dependent launch: the next kernel (the update) may start launching now; it waits
  // for this grid's completion itself (griddepcontrol.wait) before touching anything this writes
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  // the TMA descriptors (kernel parameters) are fetched now, under the prologue, not at the first load
  if (threadIdx.x == 0) {
#pragma unroll
    for (int p = 0; p < K_::NPLANES; ++p) {
      asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&maps.r[p])) : "memory");
      asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&maps.a[p])) : "memory");
    }
  }

  if (threadIdx.x == 0) {
    for (int s = 0; s < C_::STAGES; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    for (int a = 0; a < 2; ++a) {
      mbar_init(&tfull[a], 1);
      mbar_init(&tempty[a], epi_threads(EW) * CG);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 2) {
    if constexpr (CG == 1) {
      asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(smem_u32(tmem_slot)));
      asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    } else {
      asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(smem_u32(tmem_slot)));
      asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;");
    }
  }
  fence_before();
  // (the CTA barrier after the cluster barrier also orders the TMEM address tcgen05.alloc wrote to
  // shared memory for compute-sanitizer's racecheck, which does not model barrier.cluster)
  if constexpr (CG == 2) cluster_sync();
  __syncthreads();
  fence_after();
  const uint32_t tmem_base = *tmem_slot;

  // everything above (barriers, TMEM) overlaps the previous kernel's tail under PDL; the operands and
  // the live count are that kernel's output
  asm volatile("griddepcontrol.wait;" ::: "memory");
  // live-set compaction: the live rows are the first *live_rows rows of the buffer; the grid was sized
  // for the buffer's capacity and the clusters without a live tile have nothing to do
  if (ep.live_rows) {
    const int lr = *ep.live_rows;
    if (lr < rows) rows = lr;
    tiles_m = (rows + BM * CG - 1) / (BM * CG);
  }
  // split-K (MODE_STORE): the work items are (slab z, tile); slab z covers K blocks [z kslab, ...)
  const int kslab = ep.kslab > 0 ? ep.kslab : num_kb;
  const int nz = (num_kb + kslab - 1) / kslab;
  const int tiles_mn = tiles_m * tiles_n;
  const int num_tiles = tiles_mn * nz;
  const TileSched sched{tiles_m, tiles_n};

  if (warp == 0) {
    // ===================== TMA producer (one thread per CTA) =====================
    if (lane == 0) {
      int stage = 0;
      uint32_t phase = 0;
      const uint64_t keep = l2_policy(true), normal = l2_policy(false);
      for (int t = cluster_id; t < num_tiles; t += num_clusters) {
        const int z = t / tiles_mn;
        int tm, tn;
        sched.coords(t - z * tiles_mn, tm, tn);
        const int row0 = tm * BM * CG + (int)rank * BM;
        const int atom0 = tn * BN + (int)rank * C_::BN_CTA;
        const int kb0 = z * kslab, kb1 = min(num_kb, kb0 + kslab);
        for (int kb = kb0; kb < kb1; ++kb) {
          mbar_wait(&empty[stage], phase ^ 1);
          uint8_t* st = smem + stage * C_::STAGE_BYTES;
          if (leader) mbar_expect_tx(&full[stage], C_::STAGE_BYTES * CG);
#pragma unroll
          for (int p = 0; p < K_::NPLANES; ++p) {
            tma_load_2d<CG>(&maps.r[p], &full[stage], st + p * C_::R_BYTES, kb * K_::BK, row0, normal);
            tma_load_2d<CG>(&maps.a[p], &full[stage], st + K_::NPLANES * C_::R_BYTES + p * C_::A_BYTES,
                            kb * K_::BK, atom0, keep);
          }
          if (++stage == C_::STAGES) { stage = 0; phase ^= 1; }
        }
      }
    }
  } else if (warp == 1) {
    // ===================== MMA issuer (leader CTA, one thread) =====================
    if (leader && lane == 0) {
      int stage = 0;
      uint32_t phase = 0;
      int it = 0;
      for (int t = cluster_id; t < num_tiles; t += num_clusters, ++it) {
        const int a = it & 1;
        const uint32_t aphase = (it >> 1) & 1;
        mbar_wait(&tempty[a], aphase ^ 1);
        fence_after();
        const uint32_t d = tmem_base + (uint32_t)(a * BN);
        const int z = t / tiles_mn;
        const int kb0 = z * kslab, kb1 = min(num_kb, kb0 + kslab);
        for (int kb = kb0; kb < kb1; ++kb) {
          mbar_wait(&full[stage], phase);
          fence_after();
          const uint32_t base = smem_u32(smem + stage * C_::STAGE_BYTES);
          const uint64_t dr0 = desc_sw128(base);
          const uint64_t da0 = desc_sw128(base + K_::NPLANES * C_::R_BYTES);
#pragma unroll
          for (int kk = 0; kk < K_::BK / K_::UK; ++kk) {
            const uint64_t off = (uint64_t)((kk * K_::UK * K_::ELEM) >> 4);   // +32 B per K step
            if constexpr (KIND == KIND_BF16) {
              mma<KIND, CG>(d, dr0 + off, da0 + off, C_::IDESC, (kb != kb0 || kk != 0));
            } else {
              const uint64_t dr1 = desc_sw128(base + C_::R_BYTES);
              const uint64_t da1 = desc_sw128(base + 2 * C_::R_BYTES + C_::A_BYTES);
              mma<KIND, CG>(d, dr0 + off, da0 + off, C_::IDESC, (kb != kb0 || kk != 0));   // Rhi Ahi
              mma<KIND, CG>(d, dr1 + off, da0 + off, C_::IDESC, 1u);                // Rlo Ahi
              mma<KIND, CG>(d, dr0 + off, da1 + off, C_::IDESC, 1u);                // Rhi Alo
            }
          }
          mma_commit<CG>(&empty[stage]);          // slot free once these MMAs have read it
          if (++stage == C_::STAGES) { stage = 0; phase ^= 1; }
        }
        mma_commit<CG>(&tfull[a]);                // accumulator a complete
      }
    }
  } else if (warp >= 4) {
    // ===================== epilogue: TMEM -> registers -> global =====================
    // Warp w reads TMEM lane group (w % 4) (hardware rule: warp i owns lanes 32 (i % 4) .. +31) and the
    // column part (w - 4) / 4 of the 256-atom tile: CB = 128 (8 warps) or 64 (16 warps) atoms.
    const int ew = warp - 4, lg = ew & 3, part = ew >> 2;
    constexpr int HB = BN / (EW / 4);                      // accumulator columns per epilogue warp
    constexpr int CB = HB;
    const int half = part * CB / SCREEN_GROUP;            // the 128-atom partial group of this part
    const int sub = (part * CB / (SCREEN_GROUP / 2)) & 1;  // 16 warps: its lower / upper 64 atoms
    // 16 warps: [group half][lane group][sub][lane] maxima and counts, [epilogue warp][lane][TOPK] entries
    float* xm = reinterpret_cast<float*>(tmem_slot + 4);
    int* xc = reinterpret_cast<int*>(xm + 2 * 4 * 2 * 32);
    float2* ent = reinterpret_cast<float2*>(xc + 2 * 4 * 2 * 32) + ((size_t)ew * 32 + lane) * TOPK;
    const int xi = ((half * 4 + lg) * 2) * 32 + lane;      // + sub * 32: this warp's slot
    int it = 0;
    for (int t = cluster_id; t < num_tiles; t += num_clusters, ++it) {
      const int z = t / tiles_mn;
      int tm, tn;
      sched.coords(t - z * tiles_mn, tm, tn);
      const int a = it & 1;
      const uint32_t aphase = (it >> 1) & 1;
      const int row = tm * BM * CG + (int)rank * BM + lg * 32 + lane;
      // this row's window, loaded before waiting for the accumulator (its round trip overlaps the MMAs)
      float rs = 0.f;
      if constexpr (MODE == MODE_TOPK) {
        if (row < rows) rs = __ldg(ep.rslot + row);
      }
      mbar_wait(&tfull[a], aphase);
      fence_after();
      const uint32_t taddr = tmem_base + ((uint32_t)(lg * 32) << 16) + (uint32_t)(a * BN + part * HB);
      const int64_t colh = (int64_t)tn * BN + part * HB;
      bool live = row < rows;
      if constexpr (MODE == MODE_STORE) {
#pragma unroll 1
        for (int c = 0; c < HB / 32; ++c) {
          float v[32];
          tmem_ld32(taddr + (uint32_t)(c * 32), v);
          const int64_t col0 = colh + c * 32;
          if (live) {
            float* dst = ep.C + (int64_t)z * ep.zstride + (int64_t)row * ep.ldc + col0;
            if (ep.norm) {
#pragma unroll
              for (int q = 0; q < 32; ++q)    // undo the normalisation: C = A^T R
                if (col0 + q < ep.ncols) dst[q] = v[q] * __ldg(ep.norm + col0 + q);
            } else {
#pragma unroll
              for (int q = 0; q < 32; ++q)    // raw operands (split-K partials)
                if (col0 + q < ep.ncols) dst[q] = v[q];
            }
          }
        }
      } else {
        // The exact selection needs every atom within W = window ||r_b|| of the GLOBAL maximum of
        // |c~_n| (the screen runs on normalised atoms, so c~ is already |<r, a_n>| / ||a_n||); the
        // global maximum is >= this half tile's, so the entries within W of the half-tile maximum
        // are a superset.  Pass A: chunk maxima (one FMNMX per value).  Pass B: re-read the chunks
        // reaching max - W and emit their in-window entries in index order (predicated stores; at
        // most TOPK, an overflow is flagged in the last slot with the half-tile maximum).
        float W = 0.f;
        if (live) W = ep.window * rs;
        float cm[HB / 32];
        float tmax = 0.f;
#pragma unroll
        for (int c = 0; c < HB / 32; c += 2) {
          float v[64];
          tmem_ld64(taddr + (uint32_t)(c * 32), v);
#pragma unroll
          for (int h = 0; h < 2; ++h) {
            float m = 0.f;
#pragma unroll
            for (int q = 0; q < 32; ++q) m = fmaxf(m, fabsf(v[32 * h + q]));
            cm[c + h] = m;
            tmax = fmaxf(tmax, m);
          }
        }
        float2* dst = ep.part + ((int64_t)row * (2 * tiles_n) + 2 * tn + half) * TOPK;
        if constexpr (EW == 16) {
          // The two warps of this 128-atom group (sub = 0: atoms 0..63, 1: 64..127) exchange their maxima
          // (named barrier 1 + half * 4 + lg, 64 threads), take the in-window entries of their own 64
          // atoms, exchange the counts, and store the group's list in index order: the lower warp's
          // entries first, then the upper's, -1 padding, and with more than TOPK the overflow flag
          // (group maximum) in the last slot -- exactly the 8-warp epilogue's list for the group.
          const int bar_id = 1 + half * 4 + lg;
          xm[xi + sub * 32] = tmax;
          asm volatile("bar.sync %0, 64;" ::"r"(bar_id) : "memory");
          tmax = fmaxf(tmax, xm[xi + (sub ^ 1) * 32]);
          const float thr = tmax - W;
          int cnt = 0;
#pragma unroll
          for (int c = 0; c < HB / 32; ++c) {
            const bool need = live && cm[c] >= thr;
            if (!__any_sync(0xffffffffu, need)) continue;       // warp-uniform: tcgen05.ld is .aligned
            float v[32];
            tmem_ld32(taddr + (uint32_t)(c * 32), v);
            if (need) {
#pragma unroll
              for (int q = 0; q < 32; ++q) {
                const float s = fabsf(v[q]);
                if (s >= thr) {
                  if (cnt < TOPK) ent[cnt] = make_float2(s, __int_as_float((int)colh + c * 32 + q));
                  ++cnt;
                }
              }
            }
          }
          xc[xi + sub * 32] = cnt;
          asm volatile("bar.sync %0, 64;" ::"r"(bar_id) : "memory");
          const int other = xc[xi + (sub ^ 1) * 32];
          const int total = cnt + other, base = sub ? other : 0;
          if (live) {
            for (int i = 0; i < cnt && base + i < TOPK; ++i)
              if (!(total > TOPK && base + i == TOPK - 1)) dst[base + i] = ent[i];
            if (sub) {
              for (int j = total; j < TOPK; ++j) dst[j] = make_float2(-1.f, __int_as_float(-1));
              if (total > TOPK) dst[TOPK - 1] = make_float2(tmax, __int_as_float(SEL_OVERFLOW));
            }
          }
          fence_before();
          mbar_arrive_cta0(&tempty[a]);
          continue;
        }
        const float thr = tmax - W;
        int cnt = 0;
#pragma unroll
        for (int c = 0; c < HB / 32; ++c) {
          const bool need = live && cm[c] >= thr;
          if (!__any_sync(0xffffffffu, need)) continue;       // warp-uniform: tcgen05.ld is .aligned
          float v[32];
          tmem_ld32(taddr + (uint32_t)(c * 32), v);
          if (need) {
#pragma unroll
            for (int q = 0; q < 32; ++q) {
              const float s = fabsf(v[q]);
              if (s >= thr) {
                if (cnt < TOPK) dst[cnt] = make_float2(s, __int_as_float((int)colh + c * 32 + q));
                ++cnt;
              }
            }
          }
        }
        if (live) {
          for (int j = cnt; j < TOPK; ++j) dst[j] = make_float2(-1.f, __int_as_float(-1));
          if (cnt > TOPK) dst[TOPK - 1] = make_float2(tmax, __int_as_float(SEL_OVERFLOW));
        }
      }
      fence_before();
      mbar_arrive_cta0(&tempty[a]);
    }
  }

  // teardown (reconverge the single-lane role loops before the aligned barriers)
  __syncwarp();
  fence_before();
  if constexpr (CG == 2) cluster_sync(); else __syncthreads();
  fence_after();
  if (warp == 2) {
    if constexpr (CG == 1)
      asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tmem_base));
    else
      asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, 512;" ::"r"(tmem_base));
  }
}

// ------------------------------------------------------------------------------------------
// host side
// ------------------------------------------------------------------------------------------
typedef CUresult (*EncodeTiledFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                  const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                  CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

static EncodeTiledFn encode_fn() {
  static EncodeTiledFn fn = nullptr;
  if (!fn) {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<EncodeTiledFn>(p);
  }
  return fn;
}

template <int KIND>
static bool make_map(CUtensorMap* m, const void* base, int64_t rows, int64_t ld_elems, int64_t K, int box_rows) {
  using K_ = Kind<KIND>;
  EncodeTiledFn f = encode_fn();
  if (!f) return false;
  cuuint64_t dims[2] = {(cuuint64_t)K, (cuuint64_t)rows};
  cuuint64_t strides[1] = {(cuuint64_t)(ld_elems * K_::ELEM)};
  cuuint32_t box[2] = {(cuuint32_t)K_::BK, (cuuint32_t)box_rows};
  cuuint32_t estr[2] = {1, 1};
  const CUtensorMapDataType dt = KIND == KIND_BF16 ? CU_TENSOR_MAP_DATA_TYPE_BFLOAT16 : CU_TENSOR_MAP_DATA_TYPE_FLOAT32;
  return f(m, dt, 2, const_cast<void*>(base), dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
           CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) ==
         CUDA_SUCCESS;
}

static int num_sms() {
  int dev = 0, n = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
  return n > 0 ? n : 148;
}

template <int KIND, int CG, int MODE, int EW>
static cudaError_t launch_ew(const Operand& R, const Operand& At, int64_t K, const EpiArgs& ep, cudaStream_t st) {
  using C_ = Cfg<KIND, CG>;
  using K_ = Kind<KIND>;
  if (R.rows == 0) return cudaSuccess;
  if (K % K_::BK != 0 || At.rows % BN != 0 || R.rows > INT32_MAX) return cudaErrorNotSupported;
  Maps maps;
  for (int p = 0; p < K_::NPLANES; ++p) {
    if (!make_map<KIND>(&maps.r[p], R.plane[p], R.rows, R.ld, K, BM) ||
        !make_map<KIND>(&maps.a[p], At.plane[p], At.rows, At.ld, K, C_::BN_CTA))
      return cudaErrorNotSupported;
  }
  if (K_::NPLANES == 1) {
    maps.r[1] = maps.r[0];
    maps.a[1] = maps.a[0];
  }
  auto kern = k1_corr_tc<KIND, CG, MODE, EW>;
  const uint32_t smem = C_::SMEM + epi_smem(EW);
  cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  const int tiles_m = (int)((R.rows + BM * CG - 1) / (BM * CG));
  const int tiles_n = (int)(At.rows / BN);
  const int nkb = (int)(K / K_::BK);
  const int nz = ep.kslab > 0 ? (nkb + ep.kslab - 1) / ep.kslab : 1;
  const int tiles = tiles_m * tiles_n * nz;
  const int max_clusters = num_sms() / CG;
  const int clusters = tiles < max_clusters ? tiles : max_clusters;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3((unsigned)(clusters * CG));
  cfg.blockDim = dim3(num_threads(EW));
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute attr[2];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = CG;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  attr[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[1].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = (MODE == MODE_TOPK && pdl_enabled(1)) ? 2 : 1;
  return cudaLaunchKernelEx(&cfg, kern, maps, (int)R.rows, (int)(K / K_::BK), tiles_m, tiles_n, ep);
}

template <int KIND, int CG, int MODE>
static cudaError_t launch(const Operand& R, const Operand& At, int64_t K, const EpiArgs& ep, cudaStream_t st) {
  static int64_t kmax = -1;   // OMP_B200_EPI16_KMAX overrides the crossover (A/B)
  if (kmax < 0) {
    const char* e = getenv("OMP_B200_EPI16_KMAX");
    kmax = e ? atoll(e) : OMP_EPI16_KMAX;
  }
  return K < kmax ? launch_ew<KIND, CG, MODE, 16>(R, At, K, ep, st) : launch_ew<KIND, CG, MODE, 8>(R, At, K, ep, st);
}

template <int MODE>
static cudaError_t dispatch(int kind, const Operand& R, const Operand& At, int64_t K, const EpiArgs& ep,
                           cudaStream_t st) {
  static int cg = 0;
  if (!cg) {
    const char* env = getenv("OMP_B200_CTA_GROUP");
    cg = (env && env[0] == '1') ? 1 : 2;
  }
  if (kind == KIND_BF16)
    return cg == 1 ? launch<KIND_BF16, 1, MODE>(R, At, K, ep, st) : launch<KIND_BF16, 2, MODE>(R, At, K, ep, st);
  if (kind == KIND_3XTF32)
    return cg == 1 ? launch<KIND_3XTF32, 1, MODE>(R, At, K, ep, st) : launch<KIND_3XTF32, 2, MODE>(R, At, K, ep, st);
  return cudaErrorInvalidValue;
}

}  // namespace tc

cudaError_t launch_corr_tc(int kind, const Operand& R, const Operand& At, int64_t K, float* C, int64_t ldc,
                           int64_t ncols, const float* norm, cudaStream_t st) {
  tc::EpiArgs ep{C, ldc, ncols, norm, nullptr, nullptr, nullptr, 0.f, 0, 0};   // all rows, no compaction
  return tc::dispatch<tc::MODE_STORE>(kind, R, At, K, ep, st);
}

cudaError_t launch_corr_tc_splitk(int kind, const Operand& R, const Operand& At, int64_t K, float* C, int64_t ldc,
                                  int64_t ncols, int64_t kslab, float* work, cudaStream_t st) {
  const int64_t bk = kind == KIND_BF16 ? tc::Kind<KIND_BF16>::BK : tc::Kind<KIND_3XTF32>::BK;
  if (kslab % bk != 0 || R.rows == 0) return R.rows == 0 ? cudaSuccess : cudaErrorInvalidValue;
  const int64_t nz = (K + kslab - 1) / kslab;
  tc::EpiArgs ep{work, ldc, ncols, nullptr, nullptr, nullptr, nullptr, 0.f, (int)(kslab / bk), R.rows * ldc};
  cudaError_t e = tc::dispatch<tc::MODE_STORE>(kind, R, At, K, ep, st);
  if (e != cudaSuccess) return e;
  return launch_sum_slabs(work, nz, R.rows * ldc, R.rows, ncols, ldc, C, ldc, st);
}

cudaError_t launch_corr_tc_topk(int kind, const Operand& R, const Operand& At, int64_t K, const int32_t* live_rows,
                                const float* rslot, float window, float2* part, cudaStream_t st) {
  tc::EpiArgs ep{nullptr, 0, At.rows, nullptr, part, live_rows, rslot, window, 0, 0};
  return tc::dispatch<tc::MODE_TOPK>(kind, R, At, K, ep, st);
}

}  // namespace ompb
