// Memory-system microbenchmarks for the SpMM design (B200, sm_100a).
//
// Measures, with CUDA events after warm-up:
//   1. HBM streaming copy (float4), the roofline denominator cross-check;
//   2. random row gathers of W-byte rows from an R-row buffer, indices streamed
//      from HBM (the SpMM access pattern: X panel rows gathered through L2);
//   3. FP32 FMA peak (eMA compute-bound nodes).
// Output: one line per measurement, "name value unit".
#include <cstdio>
#include <cstdint>
#include <cstdlib>
#include <vector>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t err_ = (x); if (err_ != cudaSuccess) { \
  fprintf(stderr, "CUDA %s at %s:%d\n", cudaGetErrorString(err_), __FILE__, __LINE__); exit(1);} } while (0)

__global__ void copy_k(const float4* __restrict__ a, float4* __restrict__ b, size_t n4) {
  size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x;
  size_t stride = (size_t)gridDim.x * blockDim.x;
  for (; i < n4; i += stride) b[i] = a[i];
}

// Each group of G=W/16 lanes gathers one W-byte row per index; a warp walks
// 32/G indices per iteration.  Mirrors the SpMM inner loop.
template <int W>
__global__ void gather_k(const float4* __restrict__ rows, const int* __restrict__ idx,
                         size_t nidx, float4* __restrict__ out) {
  constexpr int G = W / 16;
  constexpr int PER_WARP = 32 / G;
  const int lane = threadIdx.x & 31;
  const int sub = lane / G, part = lane % G;
  size_t warp = (blockIdx.x * (size_t)blockDim.x + threadIdx.x) >> 5;
  size_t nwarps = ((size_t)gridDim.x * blockDim.x) >> 5;
  float4 acc = make_float4(0, 0, 0, 0);
  for (size_t base = warp * 32 * 4; base < nidx; base += nwarps * 32 * 4) {
#pragma unroll
    for (int u = 0; u < 4 * G; ++u) {
      size_t e = base + u * PER_WARP + sub;
      if (e < nidx) {
        int r = __ldg(idx + e);
        float4 v = __ldg(rows + (size_t)r * G + part);
        acc.x += v.x; acc.y += v.y; acc.z += v.z; acc.w += v.w;
      }
    }
  }
  if (acc.x == -1.f) out[0] = acc;
}

__global__ void fma_k(float* out, int iters) {
  float a0 = threadIdx.x, a1 = a0 + 1, a2 = a0 + 2, a3 = a0 + 3, a4 = a0 + 4, a5 = a0 + 5, a6 = a0 + 6, a7 = a0 + 7;
  const float b = 0.999f, c = 0.001f;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int j = 0; j < 16; ++j) {
      a0 = fmaf(a0, b, c); a1 = fmaf(a1, b, c); a2 = fmaf(a2, b, c); a3 = fmaf(a3, b, c);
      a4 = fmaf(a4, b, c); a5 = fmaf(a5, b, c); a6 = fmaf(a6, b, c); a7 = fmaf(a7, b, c);
    }
  }
  float s = a0 + a1 + a2 + a3 + a4 + a5 + a6 + a7;
  if (s == 12345.f) out[0] = s;
}

static float time_ms(cudaEvent_t s, cudaEvent_t e) { float ms; CK(cudaEventElapsedTime(&ms, s, e)); return ms; }

int main() {
  cudaDeviceProp p; CK(cudaGetDeviceProperties(&p, 0));
  printf("device %s sms %d l2_bytes %d smem_per_sm %zu mem_bytes %zu\n", p.name, p.multiProcessorCount,
         p.l2CacheSize, p.sharedMemPerMultiprocessor, p.totalGlobalMem);
  const int sms = p.multiProcessorCount;
  cudaEvent_t s, e; CK(cudaEventCreate(&s)); CK(cudaEventCreate(&e));

  // 1. HBM copy, 2 GiB each way
  size_t n4 = (size_t)1 << 27;  // 2 GiB of float4
  float4 *a, *b; CK(cudaMalloc(&a, n4 * 16)); CK(cudaMalloc(&b, n4 * 16));
  CK(cudaMemset(a, 0, n4 * 16));
  for (int w = 0; w < 3; ++w) copy_k<<<sms * 8, 512>>>(a, b, n4);
  float best = 1e9;
  for (int r = 0; r < 5; ++r) {
    CK(cudaEventRecord(s)); copy_k<<<sms * 8, 512>>>(a, b, n4); CK(cudaEventRecord(e)); CK(cudaEventSynchronize(e));
    best = std::min(best, time_ms(s, e));
  }
  printf("hbm_copy %.1f GB/s\n", 2.0 * n4 * 16 / best / 1e6);

  // 2. gathers: indices uniform random over R rows
  size_t nidx = (size_t)200 << 20;  // 200M indices (800 MB, streamed from HBM)
  std::vector<int> h(nidx);
  int* didx; CK(cudaMalloc(&didx, nidx * 4));
  float4* out; CK(cudaMalloc(&out, 64));
  for (size_t rows_mb : {4, 16, 32, 64, 96, 128, 512}) {
    for (int W : {32, 64, 128}) {
      size_t R = (rows_mb << 20) / W;
      uint64_t x = 88172645463325252ull;
      for (size_t i = 0; i < nidx; ++i) { x ^= x << 13; x ^= x >> 7; x ^= x << 17; h[i] = (int)(x % R); }
      CK(cudaMemcpy(didx, h.data(), nidx * 4, cudaMemcpyHostToDevice));
      auto launch = [&]() {
        if (W == 32) gather_k<32><<<sms * 16, 256>>>(a, didx, nidx, out);
        else if (W == 64) gather_k<64><<<sms * 16, 256>>>(a, didx, nidx, out);
        else gather_k<128><<<sms * 16, 256>>>(a, didx, nidx, out);
      };
      for (int w = 0; w < 2; ++w) launch();
      CK(cudaGetLastError());
      float bt = 1e9;
      for (int r = 0; r < 3; ++r) {
        CK(cudaEventRecord(s)); launch(); CK(cudaEventRecord(e)); CK(cudaEventSynchronize(e));
        bt = std::min(bt, time_ms(s, e));
      }
      printf("gather rows_mb=%zu W=%d gathered %.1f GB/s idx %.1f GB/s  (%.3f ms)\n", rows_mb, W,
             (double)nidx * W / bt / 1e6, (double)nidx * 4 / bt / 1e6, bt);
    }
  }

  // 3. FP32 FMA
  float* f; CK(cudaMalloc(&f, 4));
  int iters = 4096;
  fma_k<<<sms * 8, 256>>>(f, iters);
  CK(cudaEventRecord(s)); fma_k<<<sms * 8, 256>>>(f, iters); CK(cudaEventRecord(e)); CK(cudaEventSynchronize(e));
  double flops = 2.0 * 8 * 16 * (double)iters * sms * 8 * 256;
  printf("fp32_fma %.1f TFLOP/s\n", flops / time_ms(s, e) / 1e9);
  return 0;
}
