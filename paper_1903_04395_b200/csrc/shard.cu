// shard.cu -- vertex sharding support: row partition and the
// all-gather transports used by the sharded SpMM (engine.cu).
//   * NcclTransport (production): the library owns an NCCL communicator
//     (libnccl resolved with dlopen at run time -- the process's already
//     loaded NCCL, e.g. PyTorch's, else TCG_NCCL_LIB / libnccl.so.2 -- so
//     libtcg.so never links a second NCCL), and all-gathers are enqueued
//     ASYNCHRONOUSLY on a communication stream: the sharded rooted SpMM
//     prefetches group g+1's panel over NVLink/NVSwitch while group g's
//     gathers run (engine.cu rooted_spmm).
//   * DeviceTransport / HostTransport: a caller-supplied callback
//     (torch.distributed on device pointers; gloo on host buffers in tests).

#include <dlfcn.h>
#include <nccl.h>

#include <algorithm>
#include <condition_variable>
#include <mutex>
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

// ---------------------------------------------------------------- NCCL
struct NcclApi {
  void* h = nullptr;
  ncclResult_t (*GetUniqueId)(ncclUniqueId*) = nullptr;
  ncclResult_t (*CommInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
  ncclResult_t (*AllGather)(const void*, void*, size_t, ncclDataType_t, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
  const char* (*GetErrorString)(ncclResult_t) = nullptr;
  ncclResult_t (*GetVersion)(int*) = nullptr;
};

const NcclApi& nccl() {
  static NcclApi api = [] {
    NcclApi a;
    // the NCCL already in the process (PyTorch's) first, then TCG_NCCL_LIB, then the soname
    a.h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_NOLOAD);
    if (!a.h)
      if (const char* p = std::getenv("TCG_NCCL_LIB")) a.h = dlopen(p, RTLD_NOW | RTLD_LOCAL);
    if (!a.h) a.h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_LOCAL);
    if (!a.h) return a;
    auto sym = [&](const char* n) { return dlsym(a.h, n); };
    a.GetUniqueId = reinterpret_cast<decltype(a.GetUniqueId)>(sym("ncclGetUniqueId"));
    a.CommInitRank = reinterpret_cast<decltype(a.CommInitRank)>(sym("ncclCommInitRank"));
    a.AllGather = reinterpret_cast<decltype(a.AllGather)>(sym("ncclAllGather"));
    a.CommDestroy = reinterpret_cast<decltype(a.CommDestroy)>(sym("ncclCommDestroy"));
    a.GetErrorString = reinterpret_cast<decltype(a.GetErrorString)>(sym("ncclGetErrorString"));
    a.GetVersion = reinterpret_cast<decltype(a.GetVersion)>(sym("ncclGetVersion"));
    return a;
  }();
  if (!api.h || !api.GetUniqueId || !api.CommInitRank || !api.AllGather || !api.CommDestroy)
    throw cuda_error("NCCL not available (set TCG_NCCL_LIB to libnccl.so.2)");
  return api;
}

void nccl_check(ncclResult_t r, const char* what) {
  if (r != ncclSuccess)
    throw cuda_error(std::string(what) + ": " + (nccl().GetErrorString ? nccl().GetErrorString(r) : "nccl error"));
}

struct NcclTransport : Transport {
  ncclComm_t comm = nullptr;
  int world = 1;
  NcclTransport(int rank, int w, const uint8_t* id_bytes) : world(w) {
    ncclUniqueId id;
    static_assert(sizeof(id) == TCG_NCCL_ID_BYTES, "ncclUniqueId size");
    std::memcpy(&id, id_bytes, sizeof(id));
    nccl_check(nccl().CommInitRank(&comm, w, id, rank), "ncclCommInitRank");
  }
  ~NcclTransport() override {
    if (comm) nccl().CommDestroy(comm);
  }
  bool async() const override { return true; }
  // enqueued on s: recv is complete in stream order (no host sync)
  void allgather(const void* d_send, size_t bytes, void* d_recv, cudaStream_t s) override {
    nccl_check(nccl().AllGather(d_send, d_recv, bytes, ncclChar, comm, s), "ncclAllGather");
  }
};

// ----------------------------------------------------------- loopback
// In-process ranks (one engine per rank, several engines per GPU allowed)
// exchanging panels by device-to-device copies: the async transport contract
// of NcclTransport (everything enqueued on the caller's stream, ordered by
// events) without NCCL, so the pipelined sharded SpMM can be run and checked
// with world > 1 on ONE GPU.  Host barriers only order the ENQUEUES of the
// ranks' copies; no kernel ever waits on another rank.
struct LoopbackHub {
  int world;
  std::mutex m;
  std::condition_variable cv;
  int arrived = 0;
  uint64_t gen = 0;
  std::vector<const void*> send;
  std::vector<cudaEvent_t> ready, done;
  explicit LoopbackHub(int w) : world(w), send(w), ready(w), done(w) {}
  void barrier() {
    std::unique_lock<std::mutex> lk(m);
    const uint64_t g = gen;
    if (++arrived == world) {
      arrived = 0;
      ++gen;
      cv.notify_all();
    } else {
      cv.wait(lk, [&] { return gen != g; });
    }
  }
};

struct LoopbackTransport : Transport {
  std::shared_ptr<LoopbackHub> hub;
  int rank;
  cudaEvent_t ev_ready = nullptr, ev_done = nullptr;
  LoopbackTransport(std::shared_ptr<LoopbackHub> h, int r) : hub(std::move(h)), rank(r) {
    if (cudaEventCreateWithFlags(&ev_ready, cudaEventDisableTiming) != cudaSuccess ||
        cudaEventCreateWithFlags(&ev_done, cudaEventDisableTiming) != cudaSuccess)
      throw cuda_error("loopback transport: event creation failed");
  }
  ~LoopbackTransport() override {
    if (ev_ready) cudaEventDestroy(ev_ready);
    if (ev_done) cudaEventDestroy(ev_done);
  }
  bool async() const override { return true; }
  void allgather(const void* d_send, size_t bytes, void* d_recv, cudaStream_t s) override {
    auto ok = [](cudaError_t e) {
      if (e != cudaSuccess) throw cuda_error(std::string("loopback transport: ") + cudaGetErrorString(e));
    };
    ok(cudaEventRecord(ev_ready, s));  // this rank's panel, in stream order
    hub->send[rank] = d_send;
    hub->ready[rank] = ev_ready;
    hub->done[rank] = ev_done;
    hub->barrier();
    for (int r = 0; r < hub->world; ++r) {
      ok(cudaStreamWaitEvent(s, hub->ready[r], 0));
      ok(cudaMemcpyAsync(static_cast<char*>(d_recv) + static_cast<size_t>(r) * bytes, hub->send[r], bytes,
                         cudaMemcpyDeviceToDevice, s));
    }
    ok(cudaEventRecord(ev_done, s));
    hub->barrier();
    for (int r = 0; r < hub->world; ++r)  // peers have read this rank's panel before it moves on
      if (r != rank) ok(cudaStreamWaitEvent(s, hub->done[r], 0));
    hub->barrier();  // every wait enqueued before any event is re-recorded
  }
};

}  // namespace

std::shared_ptr<void> make_loopback_hub(int world) {
  if (world < 1) throw invalid_argument("world size must be >= 1");
  return std::make_shared<LoopbackHub>(world);
}

std::unique_ptr<Transport> make_loopback_transport(const std::shared_ptr<void>& hub, int rank) {
  auto h = std::static_pointer_cast<LoopbackHub>(hub);
  if (rank < 0 || rank >= h->world) throw invalid_argument("bad loopback rank");
  return std::make_unique<LoopbackTransport>(h, rank);
}

int loopback_world(const std::shared_ptr<void>& hub) { return std::static_pointer_cast<LoopbackHub>(hub)->world; }

void nccl_unique_id(uint8_t* out) {
  ncclUniqueId id;
  nccl_check(nccl().GetUniqueId(&id), "ncclGetUniqueId");
  std::memcpy(out, &id, sizeof(id));
}

int nccl_version() {
  int v = 0;
  if (nccl().GetVersion) nccl().GetVersion(&v);
  return v;
}

std::unique_ptr<Transport> make_nccl_transport(int rank, int world, const uint8_t* id) {
  return std::make_unique<NcclTransport>(rank, world, id);
}

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

