// L2 read-bandwidth probe for the roofline of the update kernel.
//
// The update kernel's dominant traffic is a gather of whole fp32 atom rows (Mp floats) of an
// L2-resident table (the 64 MB A^T at c4), re-read by every signal.  MEASURED_PEAKS.json holds only
// HBM and tensor peaks, so this probe measures the L2 roof on the box itself:
//   stream   every SM reads an L2-resident buffer front to back, float4, 4 loads in flight per thread
//   gather   the update kernel's access pattern: CTAs of 128 threads, each folding `rows` random rows
//            of the table (L2::evict_last, L1::no_allocate), P rows in flight per thread
//   hbm      the stream kernel over a buffer 8x larger than L2 (cross-check vs MEASURED_PEAKS)
// Each line reports bytes / CUDA-event time and the SM clock measured inside the kernel
// (clock64 vs globaltimer on CTA 0), as JSON.
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o l2_probe scripts/l2_probe.cu && ./l2_probe
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <string>
#include <vector>

#include <cuda_runtime.h>

#define CK(x)                                                                            \
  do {                                                                                   \
    cudaError_t e_ = (x);                                                                \
    if (e_ != cudaSuccess) {                                                             \
      fprintf(stderr, "%s:%d %s: %s\n", __FILE__, __LINE__, #x, cudaGetErrorString(e_)); \
      exit(1);                                                                           \
    }                                                                                    \
  } while (0)

__device__ __forceinline__ uint64_t policy_evict_last() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(p));
  return p;
}
__device__ __forceinline__ float4 ldg_keep(const float4* ptr, uint64_t pol) {
  float4 v;
  asm volatile("ld.global.nc.L1::no_allocate.L2::cache_hint.v4.f32 {%0, %1, %2, %3}, [%4], %5;"
               : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w) : "l"(ptr), "l"(pol));
  return v;
}
__device__ __forceinline__ uint64_t gtimer() {
  uint64_t t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}

struct Clk {
  unsigned long long c0, c1, t0, t1;
};

__global__ void __launch_bounds__(256) k_stream(const float4* __restrict__ buf, int64_t n4, int passes, float* out,
                                                Clk* clk) {
  const uint64_t pol = policy_evict_last();
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    clk->c0 = clock64();
    clk->t0 = gtimer();
  }
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  float4 s0 = make_float4(0, 0, 0, 0), s1 = s0, s2 = s0, s3 = s0;
  for (int pass = 0; pass < passes; ++pass) {
  int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  for (; i + 3 * stride < n4; i += 4 * stride) {
    const float4 a = ldg_keep(buf + i, pol), b = ldg_keep(buf + i + stride, pol);
    const float4 c = ldg_keep(buf + i + 2 * stride, pol), d = ldg_keep(buf + i + 3 * stride, pol);
    s0.x += a.x; s0.y += a.y; s0.z += a.z; s0.w += a.w;
    s1.x += b.x; s1.y += b.y; s1.z += b.z; s1.w += b.w;
    s2.x += c.x; s2.y += c.y; s2.z += c.z; s2.w += c.w;
    s3.x += d.x; s3.y += d.y; s3.z += d.z; s3.w += d.w;
  }
  for (; i < n4; i += stride) {
    const float4 a = ldg_keep(buf + i, pol);
    s0.x += a.x; s0.y += a.y; s0.z += a.z; s0.w += a.w;
  }
  }
  const float r = s0.x + s0.y + s0.z + s0.w + s1.x + s1.y + s1.z + s1.w + s2.x + s2.y + s2.z + s2.w + s3.x +
                  s3.y + s3.z + s3.w;
  if (r == 1234.5f) out[0] = r;   // keep the loads
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    clk->c1 = clock64();
    clk->t1 = gtimer();
  }
}

// CTA = one "signal": fold `rows` random table rows (q4 float4 each) into a register row, P rows in
// flight, every thread CH float4 of each row (T * CH == q4), as in k_update's gather.
template <int T, int CH, int P>
__global__ void __launch_bounds__(T, 1024 / T) k_gather(const float4* __restrict__ table, const uint32_t* __restrict__ idx,
                                                        int rows, float* out, Clk* clk) {
  const uint64_t pol = policy_evict_last();
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    clk->c0 = clock64();
    clk->t0 = gtimer();
  }
  const int q4 = T * CH;
  const uint32_t* id = idx + (int64_t)blockIdx.x * rows;
  float4 acc[CH];
#pragma unroll
  for (int c = 0; c < CH; ++c) acc[c] = make_float4(0, 0, 0, 0);
  int j = 0;
  for (; j + P <= rows; j += P) {
    float4 v[P][CH];
#pragma unroll
    for (int p = 0; p < P; ++p) {
      const float4* r = table + (int64_t)id[j + p] * q4 + threadIdx.x;
#pragma unroll
      for (int c = 0; c < CH; ++c) v[p][c] = ldg_keep(r + c * T, pol);
    }
#pragma unroll
    for (int p = 0; p < P; ++p)
#pragma unroll
      for (int c = 0; c < CH; ++c) {
        acc[c].x = fmaf(0.5f, v[p][c].x, acc[c].x);
        acc[c].y = fmaf(0.5f, v[p][c].y, acc[c].y);
        acc[c].z = fmaf(0.5f, v[p][c].z, acc[c].z);
        acc[c].w = fmaf(0.5f, v[p][c].w, acc[c].w);
      }
  }
  for (; j < rows; ++j) {
    const float4* r = table + (int64_t)id[j] * q4 + threadIdx.x;
#pragma unroll
    for (int c = 0; c < CH; ++c) {
      const float4 v = ldg_keep(r + c * T, pol);
      acc[c].x += v.x; acc[c].y += v.y; acc[c].z += v.z; acc[c].w += v.w;
    }
  }
  float r = 0.f;
#pragma unroll
  for (int c = 0; c < CH; ++c) r += acc[c].x + acc[c].y + acc[c].z + acc[c].w;
  if (r == 1234.5f) out[blockIdx.x] = r;
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    clk->c1 = clock64();
    clk->t1 = gtimer();
  }
}

// the same gather with 256-bit loads (ld.global.v8.f32, LDG.E.256 on sm_100a): CH8 float8 chunks per
// thread and row (T * CH8 * 8 == row length)
__device__ __forceinline__ void ldg8_keep(const float* ptr, uint64_t pol, float (&v)[8]) {
  asm volatile("ld.global.nc.L1::no_allocate.L2::cache_hint.v8.f32 {%0, %1, %2, %3, %4, %5, %6, %7}, [%8], %9;"
               : "=f"(v[0]), "=f"(v[1]), "=f"(v[2]), "=f"(v[3]), "=f"(v[4]), "=f"(v[5]), "=f"(v[6]), "=f"(v[7])
               : "l"(ptr), "l"(pol));
}
template <int T, int CH8, int P>
__global__ void __launch_bounds__(T, 1024 / T) k_gather8(const float* __restrict__ table, const uint32_t* __restrict__ idx,
                                                         int rows, float* out, Clk* clk) {
  const uint64_t pol = policy_evict_last();
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    clk->c0 = clock64();
    clk->t0 = gtimer();
  }
  const int row_len = T * CH8 * 8;
  const uint32_t* id = idx + (int64_t)blockIdx.x * rows;
  float acc[CH8][8];
#pragma unroll
  for (int c = 0; c < CH8; ++c)
#pragma unroll
    for (int e = 0; e < 8; ++e) acc[c][e] = 0.f;
  int j = 0;
  for (; j + P <= rows; j += P) {
    float v[P][CH8][8];
#pragma unroll
    for (int p = 0; p < P; ++p) {
      const float* r = table + (int64_t)id[j + p] * row_len + threadIdx.x * 8;
#pragma unroll
      for (int c = 0; c < CH8; ++c) ldg8_keep(r + c * T * 8, pol, v[p][c]);
    }
#pragma unroll
    for (int p = 0; p < P; ++p)
#pragma unroll
      for (int c = 0; c < CH8; ++c)
#pragma unroll
        for (int e = 0; e < 8; ++e) acc[c][e] = fmaf(0.5f, v[p][c][e], acc[c][e]);
  }
  float r = 0.f;
#pragma unroll
  for (int c = 0; c < CH8; ++c)
#pragma unroll
    for (int e = 0; e < 8; ++e) r += acc[c][e];
  if (r == 1234.5f) out[blockIdx.x] = r;
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    clk->c1 = clock64();
    clk->t1 = gtimer();
  }
}

template <typename F>
static void timed(const char* name, double bytes, int reps, F launch, Clk* dclk) {
  cudaEvent_t a, b;
  CK(cudaEventCreate(&a));
  CK(cudaEventCreate(&b));
  for (int i = 0; i < 3; ++i) launch();   // warm (and fill L2)
  CK(cudaDeviceSynchronize());
  std::vector<float> ms;
  double mhz = 0;
  for (int r = 0; r < reps; ++r) {
    CK(cudaEventRecord(a));
    launch();
    CK(cudaEventRecord(b));
    CK(cudaEventSynchronize(b));
    float t;
    CK(cudaEventElapsedTime(&t, a, b));
    ms.push_back(t);
    Clk h;
    CK(cudaMemcpy(&h, dclk, sizeof(Clk), cudaMemcpyDeviceToHost));
    if (h.t1 > h.t0) mhz += (double)(h.c1 - h.c0) / (double)(h.t1 - h.t0) * 1e3;
  }
  float best = ms[0], sum = 0;
  for (float t : ms) {
    best = t < best ? t : best;
    sum += t;
  }
  printf("{\"probe\": \"%s\", \"bytes\": %.0f, \"best_ms\": %.5f, \"mean_ms\": %.5f, \"best_gbs\": %.1f, "
         "\"mean_gbs\": %.1f, \"sm_mhz_in_kernel\": %.0f}\n",
         name, bytes, best, sum / reps, bytes / best / 1e6, bytes / (sum / reps) / 1e6, mhz / reps);
  fflush(stdout);
}

int main(int argc, char** argv) {
  int dev = 0, sms = 0;
  CK(cudaSetDevice(dev));
  CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
  const int reps = argc > 1 ? atoi(argv[1]) : 20;
  float* out;
  Clk* clk;
  CK(cudaMalloc(&out, 1 << 24));
  CK(cudaMalloc(&clk, sizeof(Clk)));

  // table sizes: the c4 atom table (8192 x 2048 fp32 = 64 MB) and the c5 one (2048 x 512 = 4 MB)
  const int64_t big = (int64_t)1 << 30;   // 1 GiB for the HBM cross-check
  float4* buf;
  CK(cudaMalloc(&buf, big));
  CK(cudaMemset(buf, 0, big));

  const bool only_v8 = argc > 2 && std::string(argv[2]) == "v8";   // just the 128- vs 256-bit gather
  for (int64_t mb : {4, 32, 64, 96}) {
    if (only_v8) break;
    const int64_t bytes = mb << 20;
    char name[64];
    snprintf(name, sizeof name, "stream_l2_%lldMB", (long long)mb);
    const int passes = (int)((2048ll << 20) / bytes);   // 2 GB of L2 reads per launch
    timed(name, (double)bytes * passes, reps, [&] {
      k_stream<<<sms * 8, 256>>>(buf, bytes / 16, passes, out, clk);
    }, clk);
  }
  if (!only_v8)
    timed("stream_hbm_1GB", (double)big, reps, [&] { k_stream<<<sms * 8, 256>>>(buf, big / 16, 1, out, clk); }, clk);

  // gather: c4 shape (rows of 2048 floats from 8192), 65 rows per CTA, 12500 CTAs ~ one c4 launch at k = 64
  const int nsig = 12500, rows = 65;
  std::vector<uint32_t> h((size_t)nsig * rows);
  uint64_t s = 88172645463325252ull;
  for (auto& v : h) {
    s ^= s << 13; s ^= s >> 7; s ^= s << 17;
    v = (uint32_t)(s % 8192);
  }
  uint32_t* idx;
  CK(cudaMalloc(&idx, h.size() * 4));
  CK(cudaMemcpy(idx, h.data(), h.size() * 4, cudaMemcpyHostToDevice));
  const double gb = (double)nsig * rows * 2048 * 4;
  timed("gather_c4_T128_CH4_P2", gb, reps, [&] { k_gather<128, 4, 2><<<nsig, 128>>>(buf, idx, rows, out, clk); }, clk);
  const float* fbuf = reinterpret_cast<const float*>(buf);
  timed("gather8_c4_T128_CH2_P2", gb, reps, [&] { k_gather8<128, 2, 2><<<nsig, 128>>>(fbuf, idx, rows, out, clk); }, clk);
  timed("gather8_c4_T128_CH2_P4", gb, reps, [&] { k_gather8<128, 2, 4><<<nsig, 128>>>(fbuf, idx, rows, out, clk); }, clk);
  timed("gather8_c4_T256_CH1_P4", gb, reps, [&] { k_gather8<256, 1, 4><<<nsig, 256>>>(fbuf, idx, rows, out, clk); }, clk);
  if (only_v8) {
    for (auto& v : h) v %= 2048;
    CK(cudaMemcpy(idx, h.data(), h.size() * 4, cudaMemcpyHostToDevice));
    const double g5v = (double)nsig * rows * 512 * 4;
    timed("gather_c5_T128_CH1_P2", g5v, reps, [&] { k_gather<128, 1, 2><<<nsig, 128>>>(buf, idx, rows, out, clk); }, clk);
    timed("gather_c5_T32_CH4_P2", g5v, reps, [&] { k_gather<32, 4, 2><<<nsig, 32>>>(buf, idx, rows, out, clk); }, clk);
    timed("gather8_c5_T32_CH2_P2", g5v, reps, [&] { k_gather8<32, 2, 2><<<nsig, 32>>>(fbuf, idx, rows, out, clk); }, clk);
    timed("gather8_c5_T64_CH1_P4", g5v, reps, [&] { k_gather8<64, 1, 4><<<nsig, 64>>>(fbuf, idx, rows, out, clk); }, clk);
    return 0;
  }
  timed("gather_c4_T128_CH4_P4", gb, reps, [&] { k_gather<128, 4, 4><<<nsig, 128>>>(buf, idx, rows, out, clk); }, clk);
  timed("gather_c4_T256_CH2_P4", gb, reps, [&] { k_gather<256, 2, 4><<<nsig, 256>>>(buf, idx, rows, out, clk); }, clk);
  timed("gather_c4_T512_CH1_P8", gb, reps, [&] { k_gather<512, 1, 8><<<nsig, 512>>>(buf, idx, rows, out, clk); }, clk);
  // sustained: the c4 gather back to back for ~4 s (the power-capped clock a long bench step sees)
  timed("gather_c4_T128_CH4_P2_sustained", gb * 12000, 1, [&] {
    for (int i = 0; i < 12000; ++i) k_gather<128, 4, 2><<<nsig, 128>>>(buf, idx, rows, out, clk);
  }, clk);
  timed("stream_l2_64MB_sustained", (double)(2048ll << 20) * 1500, 1, [&] {
    for (int i = 0; i < 1500; ++i) k_stream<<<sms * 8, 256>>>(buf, (64ll << 20) / 16, 32, out, clk);
  }, clk);
  // c5 shape: rows of 512 floats from 2048 (4 MB table)
  for (auto& v : h) v %= 2048;
  CK(cudaMemcpy(idx, h.data(), h.size() * 4, cudaMemcpyHostToDevice));
  const double g5 = (double)nsig * rows * 512 * 4;
  timed("gather_c5_T128_CH1_P2", g5, reps, [&] { k_gather<128, 1, 2><<<nsig, 128>>>(buf, idx, rows, out, clk); }, clk);
  timed("gather_c5_T128_CH1_P8", g5, reps, [&] { k_gather<128, 1, 8><<<nsig, 128>>>(buf, idx, rows, out, clk); }, clk);
  return 0;
}
