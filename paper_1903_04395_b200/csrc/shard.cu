// shard.cu -- vertex sharding support: row partition and the
// all-gather transports used by the sharded SpMM (engine.cu).
// The collective itself is supplied by the caller (C ABI callback): PyTorch
// torch.distributed (NCCL) on device pointers in production, gloo on host
// buffers in tests.  (Calling NCCL directly from this statically-linked
// runtime failed with cross-runtime stream errors; torch owns NCCL here.)

#include <algorithm>
#include <cstdlib>
#include <cstring>
#include <string>
#include <vector>

#include "engine.hpp"

namespace tcg {

// Contiguous row ranges balancing SpMM work (nnz of the owned rows) and eMA
// work (owned rows): weight(v) = deg(v) + average degree.
std::vector<int64_t> shard_bounds(int32_t n, const int64_t* row_ptr, int world) {
  if (world < 1) throw invalid_argument("world size must be >= 1");
  std::vector<int64_t> b(static_cast<size_t>(world) + 1, n);
  b[0] = 0;
  const int64_t nnz = row_ptr[n];
  const double avg = n > 0 ? static_cast<double>(nnz) / n : 0.0;
  const double total = static_cast<double>(nnz) + avg * n;
  int r = 1;
  double acc = 0.0;
  for (int32_t v = 0; v < n && r < world; ++v) {
    acc += static_cast<double>(row_ptr[v + 1] - row_ptr[v]) + avg;
    while (r < world && acc >= total * r / world) b[r++] = v + 1;
  }
  for (; r < world; ++r) b[r] = n;
  return b;
}

namespace {

// Device transport: the callback receives DEVICE pointers after the engine
// stream is synchronized and returns once recv is filled (e.g. PyTorch
// torch.distributed.all_gather_into_tensor over NCCL on NVLink/NVSwitch).
struct DeviceTransport : Transport {
  tcg_allgather_fn fn;
  void* user;
  DeviceTransport(tcg_allgather_fn f, void* u) : fn(f), user(u) {}
  void allgather(const void* d_send, size_t bytes, void* d_recv, cudaStream_t s) override {
    if (cudaStreamSynchronize(s) != cudaSuccess) throw cuda_error("device transport: stream sync failed");
    if (fn(user, d_send, bytes, d_recv) != 0) throw cuda_error("device transport: allgather callback failed");
  }
};

struct HostTransport : Transport {
  tcg_allgather_fn fn;
  void* user;
  std::vector<char> send, recv;
  int world = 1;
  HostTransport(tcg_allgather_fn f, void* u) : fn(f), user(u) {}
  void allgather(const void* d_send, size_t bytes, void* d_recv, cudaStream_t s) override {
    // Both copies go on the engine stream (non-blocking, so the legacy stream
    // would not order against it) and are waited for: a pageable H2D may
    // return before its DMA lands.
    send.resize(bytes);
    if (cudaMemcpyAsync(send.data(), d_send, bytes, cudaMemcpyDeviceToHost, s) != cudaSuccess ||
        cudaStreamSynchronize(s) != cudaSuccess)
      throw cuda_error("host transport: D2H failed");
    recv.resize(bytes * static_cast<size_t>(world));
    if (fn(user, send.data(), bytes, recv.data()) != 0) throw cuda_error("host transport: allgather callback failed");
    if (cudaMemcpyAsync(d_recv, recv.data(), recv.size(), cudaMemcpyHostToDevice, s) != cudaSuccess ||
        cudaStreamSynchronize(s) != cudaSuccess)
      throw cuda_error("host transport: H2D failed");
  }
};

}  // namespace

std::unique_ptr<Transport> make_device_transport(tcg_allgather_fn fn, void* user) {
  return std::make_unique<DeviceTransport>(fn, user);
}

std::unique_ptr<Transport> make_host_transport(tcg_allgather_fn fn, void* user) {
  return std::make_unique<HostTransport>(fn, user);
}

void set_host_transport_world(Transport* t, int world) {
  if (auto* h = dynamic_cast<HostTransport*>(t)) h->world = world;
}

}  // namespace tcg

