// K1-SIMT: the correlation C = A^T R ("a single call to gemm") as an FP32
// FFMA tiled GEMM.  Fallback / cross-check for the tcgen05 path (BASELINE.json north_star
// "with FP32 SIMT as fallback").  Plain FP32 on the fp32 planes: round-to-nearest FFMA,
// sequential over K, so its error does not drift with K like the truncating tensor-core
// accumulator does.
//   C[b, n] = sum_k R[b, k] * At[n, k]   (both K-major)
// Tile 128 (signals) x 128 (atoms) x 16, 256 threads, 8 x 8 outputs per thread.
#include "omp_internal.cuh"

namespace ompb {

constexpr int SB = 128, SN = 128, SK = 16, SPAD = 4;

// Double-buffered: the next K-slab's operands are loaded into registers while the current slab is
// multiplied out of shared memory; one barrier per slab.  Every output is still the sequential FMA
// chain over k = 0, 1, ..., K-1, so the summation order (and the result) is that of the plain kernel.
__global__ void __launch_bounds__(256, 2) k1_corr_simt(const float* __restrict__ Rm, int64_t ldr, int64_t B,
                                                       const float* __restrict__ Am, int64_t lda, int64_t NA,
                                                       int64_t K, float* __restrict__ C, int64_t ldc, int64_t ncols,
                                                       const int32_t* __restrict__ live_rows, int64_t kchunk,
                                                       int64_t zstride) {
  if (live_rows) {                      // live-set compaction: only the first *live_rows rows are live
    const int64_t lr = *live_rows;
    if (lr < B) B = lr;
    if ((int64_t)blockIdx.y * SB >= B) return;
  }
  __shared__ __align__(16) float As[2][SK][SB + SPAD];   // R tile, transposed: As[k][row]
  __shared__ __align__(16) float Bs[2][SK][SN + SPAD];   // At tile, transposed: Bs[k][atom]
  const int tid = threadIdx.x;
  const int tx = tid & 15, ty = tid >> 4;
  const int64_t b0 = (int64_t)blockIdx.y * SB, n0 = (int64_t)blockIdx.x * SN;
  // split-K: slab z covers k in [z kchunk, min(K, (z+1) kchunk)) and writes its partial at C + z zstride
  const int64_t kb = (int64_t)blockIdx.z * kchunk;
  const int64_t ke = kb + kchunk < K ? kb + kchunk : K;
  C += (int64_t)blockIdx.z * zstride;
  Rm += kb;
  Am += kb;
  K = ke - kb;
  float acc[8][8];
#pragma unroll
  for (int i = 0; i < 8; ++i)
#pragma unroll
    for (int j = 0; j < 8; ++j) acc[i][j] = 0.f;

  float4 ra[2], rb[2];
  auto load = [&](int64_t k0) {
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      const int idx = tid + h * 256;       // 512 float4 per operand tile
      const int row = idx >> 2, kq = idx & 3;
      ra[h] = (b0 + row < B) ? *reinterpret_cast<const float4*>(Rm + (b0 + row) * ldr + k0 + kq * 4)
                             : make_float4(0.f, 0.f, 0.f, 0.f);
      rb[h] = (n0 + row < NA) ? __ldg(reinterpret_cast<const float4*>(Am + (n0 + row) * lda + k0 + kq * 4))
                              : make_float4(0.f, 0.f, 0.f, 0.f);
    }
  };
  auto store = [&](int buf) {
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      const int idx = tid + h * 256;
      const int row = idx >> 2, kq = idx & 3;
      As[buf][kq * 4 + 0][row] = ra[h].x;
      As[buf][kq * 4 + 1][row] = ra[h].y;
      As[buf][kq * 4 + 2][row] = ra[h].z;
      As[buf][kq * 4 + 3][row] = ra[h].w;
      Bs[buf][kq * 4 + 0][row] = rb[h].x;
      Bs[buf][kq * 4 + 1][row] = rb[h].y;
      Bs[buf][kq * 4 + 2][row] = rb[h].z;
      Bs[buf][kq * 4 + 3][row] = rb[h].w;
    }
  };
  load(0);
  store(0);
  __syncthreads();
  int buf = 0;
  for (int64_t k0 = 0; k0 < K; k0 += SK) {
    const bool more = k0 + SK < K;
    if (more) load(k0 + SK);              // global loads in flight during this slab's FMAs
#pragma unroll
    for (int kk = 0; kk < SK; ++kk) {
      float a[8], bb[8];
      const float4 a0 = *reinterpret_cast<const float4*>(&As[buf][kk][ty * 4]);
      const float4 a1 = *reinterpret_cast<const float4*>(&As[buf][kk][64 + ty * 4]);
      const float4 c0 = *reinterpret_cast<const float4*>(&Bs[buf][kk][tx * 4]);
      const float4 c1 = *reinterpret_cast<const float4*>(&Bs[buf][kk][64 + tx * 4]);
      a[0] = a0.x; a[1] = a0.y; a[2] = a0.z; a[3] = a0.w;
      a[4] = a1.x; a[5] = a1.y; a[6] = a1.z; a[7] = a1.w;
      bb[0] = c0.x; bb[1] = c0.y; bb[2] = c0.z; bb[3] = c0.w;
      bb[4] = c1.x; bb[5] = c1.y; bb[6] = c1.z; bb[7] = c1.w;
#pragma unroll
      for (int i = 0; i < 8; ++i)
#pragma unroll
        for (int j = 0; j < 8; ++j) acc[i][j] = fmaf(a[i], bb[j], acc[i][j]);
    }
    if (more) {
      store(buf ^ 1);                     // the other buffer: nobody reads it during this slab
      __syncthreads();
      buf ^= 1;
    }
  }
#pragma unroll
  for (int i = 0; i < 8; ++i) {
    const int64_t row = b0 + (i < 4 ? ty * 4 + i : 64 + ty * 4 + (i - 4));
    if (row >= B) continue;
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      const int64_t col = n0 + (j < 4 ? tx * 4 + j : 64 + tx * 4 + (j - 4));
      if (col < ncols) C[row * ldc + col] = acc[i][j];
    }
  }
}

cudaError_t launch_corr_simt(const Operand& R, const Operand& At, int64_t K, float* C, int64_t ldc,
                             int64_t ncols, const int32_t* live_rows, cudaStream_t st) {
  if (R.rows == 0) return cudaSuccess;
  if (K % SK != 0 || R.ld % 4 != 0 || At.ld % 4 != 0) return cudaErrorInvalidValue;
  if (ncols > At.rows) ncols = At.rows;
  dim3 grid((unsigned)((ncols + SN - 1) / SN), (unsigned)((R.rows + SB - 1) / SB));
  if (grid.y > 65535) return cudaErrorInvalidConfiguration;
  k1_corr_simt<<<grid, 256, 0, st>>>((const float*)R.plane[0], R.ld, R.rows, (const float*)At.plane[0], At.ld,
                                     At.rows, K, C, ldc, ncols, live_rows, K, 0);
  return cudaGetLastError();
}

// C = sum over K slabs of kchunk, the slabs' partials summed in slab order (deterministic, and
// independent of the batch size): fills the GPU when the output grid alone is small (P0 of the
// projection path on tall dictionaries: few output tiles, long K).
__global__ void k_sum_slabs(const float* __restrict__ part, int64_t nz, int64_t zstride, int64_t rows, int64_t cols,
                            int64_t ld, float* __restrict__ C, int64_t ldc) {
  const int64_t total = rows * cols;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < total; i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t r = i / cols, c = i - r * cols;
    float s = part[r * ld + c];
    for (int64_t z = 1; z < nz; ++z) s += part[z * zstride + r * ld + c];
    C[r * ldc + c] = s;
  }
}

int64_t corr_simt_splitk_slabs(int64_t K, int64_t kchunk) { return (K + kchunk - 1) / kchunk; }

cudaError_t launch_corr_simt_splitk(const Operand& R, const Operand& At, int64_t K, float* C, int64_t ldc,
                                    int64_t ncols, int64_t kchunk, float* work, cudaStream_t st) {
  if (R.rows == 0) return cudaSuccess;
  if (K % SK != 0 || kchunk % SK != 0 || R.ld % 4 != 0 || At.ld % 4 != 0) return cudaErrorInvalidValue;
  if (ncols > At.rows) ncols = At.rows;
  const int64_t nz = corr_simt_splitk_slabs(K, kchunk);
  const int64_t zstride = R.rows * ldc;
  dim3 grid((unsigned)((ncols + SN - 1) / SN), (unsigned)((R.rows + SB - 1) / SB), (unsigned)nz);
  if (grid.y > 65535 || nz > 65535) return cudaErrorInvalidConfiguration;
  k1_corr_simt<<<grid, 256, 0, st>>>((const float*)R.plane[0], R.ld, R.rows, (const float*)At.plane[0], At.ld,
                                     At.rows, K, work, ldc, ncols, nullptr, kchunk, zstride);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return e;
  return launch_sum_slabs(work, nz, zstride, R.rows, ncols, ldc, C, ldc, st);
}

cudaError_t launch_sum_slabs(const float* work, int64_t nz, int64_t zstride, int64_t rows, int64_t cols, int64_t ld,
                             float* C, int64_t ldc, cudaStream_t st) {
  if (rows == 0) return cudaSuccess;
  k_sum_slabs<<<1184, 256, 0, st>>>(work, nz, zstride, rows, cols, ld, C, ldc);
  return cudaGetLastError();
}

}  // namespace ompb
