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

__global__ void __launch_bounds__(256) k1_corr_simt(const float* __restrict__ Rm, int64_t ldr, int64_t B,
                                                    const float* __restrict__ Am, int64_t lda, int64_t NA,
                                                    int64_t K, float* __restrict__ C, int64_t ldc, int64_t ncols,
                                                    const int32_t* __restrict__ live_rows) {
  if (live_rows) {                      // live-set compaction: only the first *live_rows rows are live
    const int64_t lr = *live_rows;
    if (lr < B) B = lr;
    if ((int64_t)blockIdx.y * SB >= B) return;
  }
  __shared__ float As[SK][SB + SPAD];   // R tile, transposed: As[k][row]
  __shared__ float Bs[SK][SN + SPAD];   // At tile, transposed: Bs[k][atom]
  const int tid = threadIdx.x;
  const int tx = tid & 15, ty = tid >> 4;
  const int64_t b0 = (int64_t)blockIdx.y * SB, n0 = (int64_t)blockIdx.x * SN;
  float acc[8][8];
#pragma unroll
  for (int i = 0; i < 8; ++i)
#pragma unroll
    for (int j = 0; j < 8; ++j) acc[i][j] = 0.f;

  for (int64_t k0 = 0; k0 < K; k0 += SK) {
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      const int idx = tid + h * 256;       // 512 float4 per operand tile
      const int row = idx >> 2, kq = idx & 3;
      float4 r = make_float4(0.f, 0.f, 0.f, 0.f);
      if (b0 + row < B) r = *reinterpret_cast<const float4*>(Rm + (b0 + row) * ldr + k0 + kq * 4);
      As[kq * 4 + 0][row] = r.x;
      As[kq * 4 + 1][row] = r.y;
      As[kq * 4 + 2][row] = r.z;
      As[kq * 4 + 3][row] = r.w;
      float4 t = make_float4(0.f, 0.f, 0.f, 0.f);
      if (n0 + row < NA) t = *reinterpret_cast<const float4*>(Am + (n0 + row) * lda + k0 + kq * 4);
      Bs[kq * 4 + 0][row] = t.x;
      Bs[kq * 4 + 1][row] = t.y;
      Bs[kq * 4 + 2][row] = t.z;
      Bs[kq * 4 + 3][row] = t.w;
    }
    __syncthreads();
#pragma unroll
    for (int kk = 0; kk < SK; ++kk) {
      float a[8], bb[8];
      const float4 a0 = *reinterpret_cast<const float4*>(&As[kk][ty * 4]);
      const float4 a1 = *reinterpret_cast<const float4*>(&As[kk][64 + ty * 4]);
      const float4 c0 = *reinterpret_cast<const float4*>(&Bs[kk][tx * 4]);
      const float4 c1 = *reinterpret_cast<const float4*>(&Bs[kk][64 + tx * 4]);
      a[0] = a0.x; a[1] = a0.y; a[2] = a0.z; a[3] = a0.w;
      a[4] = a1.x; a[5] = a1.y; a[6] = a1.z; a[7] = a1.w;
      bb[0] = c0.x; bb[1] = c0.y; bb[2] = c0.z; bb[3] = c0.w;
      bb[4] = c1.x; bb[5] = c1.y; bb[6] = c1.z; bb[7] = c1.w;
#pragma unroll
      for (int i = 0; i < 8; ++i)
#pragma unroll
        for (int j = 0; j < 8; ++j) acc[i][j] = fmaf(a[i], bb[j], acc[i][j]);
    }
    __syncthreads();
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
                                     At.rows, K, C, ldc, ncols, live_rows);
  return cudaGetLastError();
}

}  // namespace ompb
