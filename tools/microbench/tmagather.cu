// tmagather.cu -- can the TMA engine gather SpMM rows faster than the LSU?
//
// The rooted SpMM gathers one 128 B panel row per neighbour; ncu puts its
// L1/TEX pipe at ~78% and the gathered rate at ~10.5-14 TB/s, and halving
// the footprint (gather_scale_probe.py) gains only ~11%.  This compares,
// for R random 128 B rows (footprint 32-128 MB) indexed by a streamed index
// array:
//   ldg   : 8 lanes x float4 per row, 8 rows in flight per lane group, fp32
//           sums in registers (the spmm_rooted pattern);
//   bulk  : cp.async.bulk (SASS UBLKCP) of each row into shared memory, 32
//           rows per warp stage on an mbarrier transaction count, double
//           buffered, then the warp sums the staged rows from shared memory.
// Prints "name footprint_MB TB/s_gathered".
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <vector>

#define CK(x)                                                                                        \
  do {                                                                                               \
    cudaError_t e_ = (x);                                                                            \
    if (e_ != cudaSuccess) {                                                                         \
      fprintf(stderr, "CUDA %s at %s:%d\n", cudaGetErrorString(e_), __FILE__, __LINE__);            \
      exit(1);                                                                                       \
    }                                                                                                \
  } while (0)

__global__ void __launch_bounds__(256, 4) gather_ldg(const float4* __restrict__ rows, const int* __restrict__ idx,
                                                     int64_t nidx, float* __restrict__ out) {
  const int lane = threadIdx.x & 31, g = lane >> 3, l = lane & 7;
  const int64_t warp = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  float4 acc = make_float4(0, 0, 0, 0);
  for (int64_t base = warp * 32; base < nidx; base += nw * 32) {  // 32 rows per warp step, 8 per group
    float4 v[8];
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      const int64_t e = base + g * 8 + j;
      const int r = e < nidx ? __ldg(idx + e) : 0;
      v[j] = __ldg(rows + (int64_t)r * 8 + l);
    }
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      acc.x += v[j].x; acc.y += v[j].y; acc.z += v[j].z; acc.w += v[j].w;
    }
  }
  if (acc.x == -1.f) out[0] = acc.y;
}

__device__ __forceinline__ uint32_t s32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

template <int STAGES>
__global__ void __launch_bounds__(256, 2) gather_bulk(const float4* __restrict__ rows, const int* __restrict__ idx,
                                                      int64_t nidx, float* __restrict__ out) {
  extern __shared__ __align__(128) float4 sm[];
  __shared__ __align__(8) uint64_t bar[8][STAGES];
  const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
  const int64_t warp = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  float4* mine = sm + (int64_t)wib * STAGES * 32 * 8;  // STAGES x 32 rows x 8 float4
  if (lane < STAGES)
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(s32(&bar[wib][lane])) : "memory");
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  __syncwarp();
  float4 acc = make_float4(0, 0, 0, 0);
  auto issue = [&](int64_t base, int st) {
    if (lane == 0)
      asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(s32(&bar[wib][st])), "r"(32 * 128)
                   : "memory");
    __syncwarp();
    const int64_t e = base + lane;
    const int r = e < nidx ? __ldg(idx + e) : 0;
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], 128, [%2];" ::"r"(
                     s32(mine + (st * 32 + lane) * 8)),
                 "l"(rows + (int64_t)r * 8), "r"(s32(&bar[wib][st]))
                 : "memory");
  };
  uint32_t phase[STAGES];
#pragma unroll
  for (int s = 0; s < STAGES; ++s) phase[s] = 0;
  int64_t base = warp * 32;
#pragma unroll
  for (int s = 0; s < STAGES; ++s)
    if (base + s * nw * 32 < nidx) issue(base + s * nw * 32, s);
  for (int it = 0; base < nidx; base += nw * 32, ++it) {
    const int st = it % STAGES;
    asm volatile(
        "{\n.reg .pred P1;\nW_%=:\nmbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n@!P1 bra W_%=;\n}\n" ::"r"(
            s32(&bar[wib][st])),
        "r"(phase[st])
        : "memory");
    phase[st] ^= 1u;
    // lane = (row group g, float4 l): sum 32 rows' 8 float4s
    const float4* buf = mine + st * 32 * 8;
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      const float4 v = buf[(j * 4 + (lane >> 3)) * 8 + (lane & 7)];
      acc.x += v.x; acc.y += v.y; acc.z += v.z; acc.w += v.w;
    }
    __syncwarp();
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    const int64_t nb = base + (int64_t)STAGES * nw * 32;
    if (nb < nidx) issue(nb, st);
  }
  if (acc.x == -1.f) out[0] = acc.y;
}

int main() {
  int sms = 0;
  CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
  const int64_t nidx = 64ll << 20;
  int* didx;
  float* dout;
  CK(cudaMalloc(&didx, nidx * 4));
  CK(cudaMalloc(&dout, 64));
  for (int mb : {32, 64, 128}) {
    const int64_t R = ((int64_t)mb << 20) / 128;
    std::vector<int> h(nidx);
    uint64_t x = 88172645463325252ull;
    for (auto& v : h) {
      x ^= x << 13; x ^= x >> 7; x ^= x << 17;
      v = (int)(x % R);
    }
    CK(cudaMemcpy(didx, h.data(), nidx * 4, cudaMemcpyHostToDevice));
    float4* drows;
    CK(cudaMalloc(&drows, R * 128));
    CK(cudaMemset(drows, 0, R * 128));
    cudaEvent_t a, b;
    CK(cudaEventCreate(&a));
    CK(cudaEventCreate(&b));
    auto timeit = [&](const char* name, auto launch) {
      launch();
      CK(cudaDeviceSynchronize());
      float best = 1e30f;
      for (int rep = 0; rep < 5; ++rep) {
        CK(cudaEventRecord(a));
        launch();
        CK(cudaEventRecord(b));
        CK(cudaEventSynchronize(b));
        float ms;
        CK(cudaEventElapsedTime(&ms, a, b));
        best = ms < best ? ms : best;
      }
      printf("%s %d MB %.2f TB/s (%.3f ms)\n", name, mb, nidx * 128.0 / (best * 1e-3) / 1e12, best);
    };
    timeit("ldg", [&] { gather_ldg<<<sms * 4, 256>>>(drows, didx, nidx, dout); });
    for (int st : {2, 4}) {
      const size_t smem = (size_t)8 * st * 32 * 128;
      if (st == 2) {
        CK(cudaFuncSetAttribute(gather_bulk<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
        timeit("bulk2", [&] { gather_bulk<2><<<sms * 2, 256, smem>>>(drows, didx, nidx, dout); });
      } else {
        CK(cudaFuncSetAttribute(gather_bulk<4>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
        timeit("bulk4", [&] { gather_bulk<4><<<sms * 1, 256, smem>>>(drows, didx, nidx, dout); });
      }
    }
    CK(cudaGetLastError());
    CK(cudaFree(drows));
  }
  return 0;
}
