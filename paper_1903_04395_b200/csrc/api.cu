// api.cu -- the extern "C" boundary (include/tcg.h).  Every entry point
// catches the host library's exception classes and maps them to the status
// codes documented in tcg.h (mirroring the reference's exception types,
// SURVEY 8(b)); no C++ exception crosses the ABI.
#include <cstring>
#include <memory>
#include <thread>
#include <cmath>
#include <exception>
#include <string>

#include "../../include/tcg.h"
#include "engine.hpp"

struct tcg_graph {
  tcg::Csr csr;
};
struct tcg_ctx {
  std::unique_ptr<tcg::Engine> eng;
  // multi-device context (tcg_create_multi): one engine per further device;
  // graph / template go to every engine, colorings are spread over them
  std::vector<std::unique_ptr<tcg::Engine>> peers;
};

namespace {
thread_local std::string g_err;

template <typename F>
int guarded(F&& f) {
  try {
    f();
    return TCG_OK;
  } catch (const tcg::parse_error& e) {
    g_err = e.what();
    return TCG_EPARSE;
  } catch (const tcg::invalid_argument& e) {
    g_err = e.what();
    return TCG_EINVAL;
  } catch (const tcg::resource_error& e) {
    g_err = e.what();
    return TCG_ERESOURCE;
  } catch (const tcg::nonfinite_error& e) {
    g_err = e.what();
    return TCG_ENONFINITE;
  } catch (const tcg::cuda_error& e) {
    g_err = e.what();
    return TCG_ECUDA;
  } catch (const tcg::logic_error& e) {
    g_err = e.what();
    return TCG_ELOGIC;
  } catch (const std::bad_alloc&) {
    g_err = "host allocation failed";
    return TCG_ERESOURCE;
  } catch (const std::exception& e) {
    g_err = e.what();
    return TCG_ELOGIC;
  }
}

void need(const void* p, const char* what) {
  if (!p) throw tcg::invalid_argument(std::string(what) + " is NULL");
}

// f(engine, index) on every engine of the context, one host thread per
// device (each engine sets its own device); the first failure is rethrown
template <typename F>
void for_all(tcg_ctx* ctx, F&& f) {
  if (ctx->peers.empty()) {
    f(*ctx->eng, 0);
    return;
  }
  const size_t nd = ctx->peers.size() + 1;
  std::vector<std::exception_ptr> err(nd);
  std::vector<std::thread> th;
  for (size_t d = 0; d < nd; ++d)
    th.emplace_back([&, d] {
      try {
        f(d == 0 ? *ctx->eng : *ctx->peers[d - 1], static_cast<int>(d));
      } catch (...) {
        err[d] = std::current_exception();
      }
    });
  for (auto& t : th) t.join();
  for (auto& e : err)
    if (e) std::rethrow_exception(e);
}

// colorings [0, count) split into contiguous per-device chunks
std::vector<int> chunks_of(int count, size_t nd) {
  std::vector<int> b(nd + 1);
  for (size_t d = 0; d <= nd; ++d) b[d] = static_cast<int>(static_cast<int64_t>(count) * d / nd);
  return b;
}

void fill_plan(const tcg::Plan& p, tcg_plan* out) {
  std::memset(out, 0, sizeof(*out));
  out->k = p.k;
  out->root = p.root;
  out->num_nodes = p.num_nodes;
  for (int i = 0; i < p.num_nodes; ++i) {
    out->size[i] = p.size[i];
    out->node_root[i] = p.node_root[i];
    out->active_child[i] = p.active[i];
    out->passive_child[i] = p.passive[i];
    out->parent[i] = p.parent[i];
    out->dp_order[i] = p.dp_order[i];
  }
}
}  // namespace

extern "C" {

const char* tcg_last_error(void) { return g_err.c_str(); }

const char* tcg_version(void) {
  return "treecount-b200 0.2 (sm_100a; fp32 128 B panel tables, rooted-color compression, fp64 accumulation/root)";
}

// ------------------------------------------------------------------ graph
int tcg_graph_from_edges(const int32_t* edges, int64_t m, int32_t n_hint, tcg_graph** out) {
  return guarded([&] {
    need(out, "out");
    if (m < 0) throw tcg::invalid_argument("negative edge count");
    if (m > 0) need(edges, "edges");
    auto g = std::make_unique<tcg_graph>();
    g->csr = tcg::csr_from_edges(edges, m, n_hint);
    *out = g.release();
  });
}

int tcg_graph_from_csr(int32_t n, const int64_t* row_ptr, const int32_t* col, tcg_graph** out) {
  return guarded([&] {
    need(out, "out");
    need(row_ptr, "row_ptr");
    if (n < 0) throw tcg::invalid_argument("negative vertex count");
    if (row_ptr[n] > 0) need(col, "col");
    auto g = std::make_unique<tcg_graph>();
    g->csr = tcg::csr_adopt(n, row_ptr, col);
    *out = g.release();
  });
}

int tcg_generate_rmat(int scale, int64_t edges, double a, double b, double c, double d,
                      uint64_t seed, tcg_graph** out) {
  return guarded([&] {
    need(out, "out");
    auto g = std::make_unique<tcg_graph>();
    g->csr = tcg::generate_rmat(scale, edges, a, b, c, d, seed);
    *out = g.release();
  });
}

int tcg_generate_erdos_renyi(int32_t n, double p, uint64_t seed, tcg_graph** out) {
  return guarded([&] {
    need(out, "out");
    auto g = std::make_unique<tcg_graph>();
    g->csr = tcg::generate_erdos_renyi(n, p, seed);
    *out = g.release();
  });
}

int tcg_graph_info(const tcg_graph* g, int32_t* n, int64_t* m, int64_t* nnz, int32_t* max_degree) {
  return guarded([&] {
    need(g, "graph");
    if (n) *n = g->csr.n;
    if (m) *m = g->csr.nnz() / 2;
    if (nnz) *nnz = g->csr.nnz();
    if (max_degree) *max_degree = g->csr.max_degree();
  });
}

const int64_t* tcg_graph_row_ptr(const tcg_graph* g) { return g ? g->csr.row_ptr.data() : nullptr; }
const int32_t* tcg_graph_col(const tcg_graph* g) { return g ? g->csr.col.data() : nullptr; }
void tcg_graph_destroy(tcg_graph* g) { delete g; }

// --------------------------------------------------------------- template
int tcg_partition(int k, const int32_t* edges, int root, tcg_plan* out) {
  return guarded([&] {
    need(out, "out");
    if (k > 1) need(edges, "edges");
    fill_plan(tcg::partition(tcg::make_template(k, edges, root)), out);
  });
}

int tcg_automorphisms(int k, const int32_t* edges, uint64_t* out) {
  return guarded([&] {
    need(out, "out");
    if (k > 1) need(edges, "edges");
    *out = tcg::automorphism_count(tcg::make_template(k, edges, -1));
  });
}

int tcg_split_table(int k, int parent_size, int active_size, int32_t* ai, int32_t* pi,
                    int32_t* gp, int32_t* ga) {
  return guarded([&] {
    if (k < 1 || k > tcg::kMaxK) throw tcg::invalid_argument("color count k must be in [1, 20]");
    tcg::SplitTable st = tcg::build_split_table(k, parent_size, active_size);
    const size_t bytes = st.active_index.size() * sizeof(int32_t);
    if (ai) std::memcpy(ai, st.active_index.data(), bytes);
    if (pi) std::memcpy(pi, st.passive_index.data(), bytes);
    if (gp) std::memcpy(gp, st.grouped_parent.data(), bytes);
    if (ga) std::memcpy(ga, st.grouped_active.data(), bytes);
  });
}

int64_t tcg_color_index_of(int k, const int32_t* colors, int h) {
  int64_t r = -1;
  const int st = guarded([&] {
    if (k < 1 || k > tcg::kMaxK) throw tcg::invalid_argument("color count k must be in [1, 20]");
    int c[tcg::kMaxK];
    for (int i = 0; i < h; ++i) {
      c[i] = colors[i];
      if (c[i] >= k || (i && c[i] <= c[i - 1]) || c[i] < 0)
        throw tcg::invalid_argument("color set must be strictly increasing in [0, k)");
    }
    r = tcg::index_of(c, h);
  });
  return st == TCG_OK ? r : -1;
}

int tcg_color_set_of(int k, int64_t index, int h, int32_t* colors) {
  return guarded([&] {
    if (k < 1 || k > tcg::kMaxK) throw tcg::invalid_argument("color count k must be in [1, 20]");
    if (h < 0 || h > k || index < 0 || index >= tcg::binom()(k, h))
      throw tcg::invalid_argument("color set index out of range");
    int c[tcg::kMaxK];
    tcg::set_of(k, index, h, c);
    for (int i = 0; i < h; ++i) colors[i] = c[i];
  });
}

int64_t tcg_estimate_bytes(const tcg_plan* plan, int64_t n) {
  if (!plan) return -1;
  tcg::Plan p;
  p.k = plan->k;
  p.num_nodes = plan->num_nodes;
  p.size.assign(plan->size, plan->size + plan->num_nodes);
  p.active.assign(plan->active_child, plan->active_child + plan->num_nodes);
  p.passive.assign(plan->passive_child, plan->passive_child + plan->num_nodes);
  p.dp_order.assign(plan->dp_order, plan->dp_order + plan->num_nodes);
  return tcg::estimate_bytes(p, n);
}

double tcg_colorful_probability(int k) { return tcg::colorful_probability(k); }

int tcg_rooted_layout(int k, int s, int32_t* info, int32_t* perm, int32_t* slot_col) {
  return guarded([&] {
    need(info, "info");
    const tcg::RootedLayout L = tcg::build_rooted_layout(k, s);
    info[0] = L.zw;
    info[1] = L.groups;
    info[2] = L.full_cols;
    info[3] = L.store_cols;
    if (perm) std::copy(L.perm.begin(), L.perm.end(), perm);
    if (slot_col) std::copy(L.slot_col.begin(), L.slot_col.end(), slot_col);
  });
}

int tcg_rtv_task_layout(int k, int s, int a, int V, int64_t* info) {
  return guarded([&] {
    need(info, "info");
    tcg::rtv_task_layout_check(k, s, a, V, info);
  });
}

// ----------------------------------------------------------------- engine
int tcg_create(const tcg_config* cfg, tcg_ctx** out) {
  return guarded([&] {
    need(out, "out");
    tcg_config c{};
    if (cfg) c = *cfg;
    auto ctx = std::make_unique<tcg_ctx>();
    ctx->eng = std::make_unique<tcg::Engine>(c);
    *out = ctx.release();
  });
}

int tcg_create_multi(const tcg_config* cfg, const int* device_ids, int ndev, tcg_ctx** out) {
  return guarded([&] {
    need(out, "out");
    need(device_ids, "device_ids");
    if (ndev < 1) throw tcg::invalid_argument("ndev must be >= 1");
    tcg_config c{};
    if (cfg) c = *cfg;
    auto ctx = std::make_unique<tcg_ctx>();
    c.device = device_ids[0];
    ctx->eng = std::make_unique<tcg::Engine>(c);
    for (int d = 1; d < ndev; ++d) {
      c.device = device_ids[d];
      ctx->peers.push_back(std::make_unique<tcg::Engine>(c));
    }
    *out = ctx.release();
  });
}

int tcg_device_count_of(const tcg_ctx* ctx) { return ctx ? static_cast<int>(ctx->peers.size()) + 1 : 0; }

void tcg_destroy(tcg_ctx* ctx) { delete ctx; }

int tcg_set_graph(tcg_ctx* ctx, int32_t n, const int64_t* row_ptr, const int32_t* col) {
  return guarded([&] {
    need(ctx, "ctx");
    need(row_ptr, "row_ptr");
    // the reference's Graph invariants are the caller's contract here (as for
    // a treecount::Graph); row_ptr is checked on the host, ids / order / loops
    // on the device after the upload (O(nnz) there, no host copy)
    if (n < 0 || row_ptr[0] != 0) throw tcg::parse_error("bad CSR row_ptr");
    for (int32_t v = 0; v < n; ++v)
      if (row_ptr[v + 1] < row_ptr[v]) throw tcg::parse_error("CSR row_ptr not monotone");
    if (row_ptr[n] > 0) need(col, "col");
    if (ctx->eng->sharded()) ctx->eng->set_graph(tcg::csr_adopt(n, row_ptr, col, /*check_symmetry=*/false));
    else for_all(ctx, [&](tcg::Engine& e, int) { e.set_graph_ptrs(n, row_ptr, col, /*validate=*/true); });
  });
}

int tcg_set_graph_handle(tcg_ctx* ctx, const tcg_graph* g) {
  return guarded([&] {
    need(ctx, "ctx");
    need(g, "graph");
    for_all(ctx, [&](tcg::Engine& e, int) { e.set_graph(g->csr); });
  });
}

int tcg_set_template(tcg_ctx* ctx, int k, const int32_t* edges, int root) {
  return guarded([&] {
    need(ctx, "ctx");
    if (k > 1) need(edges, "edges");
    for_all(ctx, [&](tcg::Engine& e, int) { e.set_template(k, edges, root); });
  });
}

int tcg_required_device_bytes(tcg_ctx* ctx, int64_t* bytes) {
  return guarded([&] {
    need(ctx, "ctx");
    need(bytes, "bytes");
    *bytes = ctx->eng->required_bytes();
  });
}

int tcg_get_plan(tcg_ctx* ctx, tcg_plan* out, uint64_t* aut) {
  return guarded([&] {
    need(ctx, "ctx");
    if (out) fill_plan(ctx->eng->plan(), out);
    if (aut) *aut = ctx->eng->aut();
  });
}

int tcg_coloring(tcg_ctx* ctx, uint64_t seed, uint8_t* colors) {
  return guarded([&] {
    need(ctx, "ctx");
    need(colors, "colors");
    ctx->eng->coloring(seed, colors);
  });
}

int tcg_run_coloring(tcg_ctx* ctx, uint64_t seed, const uint8_t* colors, double* rooted_total,
                     double* per_vertex, tcg_node_stats* stats) {
  return guarded([&] {
    need(ctx, "ctx");
    need(rooted_total, "rooted_total");
    *rooted_total = ctx->eng->run_coloring(seed, colors, per_vertex, stats);
  });
}

int tcg_estimate(tcg_ctx* ctx, uint64_t seed, int iterations, double* rooted_totals,
                 double* estimate, double* stderr_of_mean, double* per_vertex_estimate) {
  return guarded([&] {
    need(ctx, "ctx");
    need(rooted_totals, "rooted_totals");
    need(estimate, "estimate");
    need(stderr_of_mean, "stderr_of_mean");
    if (ctx->peers.empty()) {
      ctx->eng->estimate(seed, iterations, rooted_totals, estimate, stderr_of_mean, per_vertex_estimate);
      return;
    }
    // colorings seed + i spread over the devices in contiguous chunks; totals
    // land in i order, the estimator arithmetic is the reference's
    if (iterations < 1) throw tcg::invalid_argument("iterations must be >= 1");
    const size_t nd = ctx->peers.size() + 1;
    const std::vector<int> b = chunks_of(iterations, nd);
    const int32_t n = ctx->eng->n_global();
    std::vector<std::vector<double>> pv(nd);
    for_all(ctx, [&](tcg::Engine& e, int d) {
      const int cnt = b[d + 1] - b[d];
      if (cnt == 0) return;
      double est = 0, se = 0;
      if (per_vertex_estimate) pv[d].assign(static_cast<size_t>(std::max(n, 0)), 0.0);
      e.estimate(seed + static_cast<uint64_t>(b[d]), cnt, rooted_totals + b[d], &est, &se,
                 per_vertex_estimate ? pv[d].data() : nullptr);
    });
    double mean = 0.0;  // estimator.hpp:80-91
    for (int i = 0; i < iterations; ++i) mean += rooted_totals[i];
    mean /= static_cast<double>(iterations);
    double var = 0.0;
    for (int i = 0; i < iterations; ++i) var += (rooted_totals[i] - mean) * (rooted_totals[i] - mean);
    const double scale = 1.0 / (static_cast<double>(ctx->eng->aut()) * tcg::colorful_probability(ctx->eng->plan().k));
    *estimate = mean * scale;
    *stderr_of_mean = iterations > 1 ? std::sqrt(var / (static_cast<double>(iterations) *
                                                        static_cast<double>(iterations - 1))) * scale : 0.0;
    if (per_vertex_estimate)
      for (int32_t v = 0; v < n; ++v) {
        double s = 0.0;  // device (= coloring) order
        for (size_t d = 0; d < nd; ++d)
          if (!pv[d].empty()) s += pv[d][v] * (b[d + 1] - b[d]);
        per_vertex_estimate[v] = s / iterations;
      }
  });
}

int tcg_node_table(tcg_ctx* ctx, int node_id, int which, double* out) {
  return guarded([&] {
    need(ctx, "ctx");
    need(out, "out");
    ctx->eng->node_table(node_id, which, out);
  });
}

int tcg_spmm(tcg_ctx* ctx, const float* x, int cols, float* y) {
  return guarded([&] {
    need(ctx, "ctx");
    need(x, "x");
    need(y, "y");
    ctx->eng->spmm_host(x, cols, y);
  });
}

int tcg_set_graph_edges(tcg_ctx* ctx, const int32_t* edges, int64_t m, int32_t n_hint) {
  return guarded([&] {
    need(ctx, "ctx");
    if (m > 0) need(edges, "edges");
    for_all(ctx, [&](tcg::Engine& e, int) { e.set_graph_edges(edges, m, n_hint); });
  });
}

int tcg_get_graph_csr(tcg_ctx* ctx, int32_t* n, int64_t* nnz, int64_t* row_ptr, int32_t* col) {
  return guarded([&] {
    need(ctx, "ctx");
    ctx->eng->graph_csr(n, nnz, row_ptr, col);
  });
}

int tcg_spmm_rooted(tcg_ctx* ctx, int k, int s, int pair, const uint8_t* colors, const float* x, float* y) {
  return guarded([&] {
    need(ctx, "ctx");
    need(colors, "colors");
    need(x, "x");
    need(y, "y");
    ctx->eng->spmm_rooted_host(k, s, pair != 0, colors, x, y);
  });
}

int tcg_set_rejection_limit(tcg_ctx* ctx, uint64_t limit) {
  return guarded([&] {
    need(ctx, "ctx");
    for_all(ctx, [&](tcg::Engine& e, int) { e.set_rejection_limit(limit); });
  });
}

int tcg_time_colorings(tcg_ctx* ctx, uint64_t seed, int count, int per_kernel, double* totals,
                       tcg_timing* out) {
  return guarded([&] {
    need(ctx, "ctx");
    need(out, "out");
    if (ctx->peers.empty()) {
      ctx->eng->time_colorings(seed, count, per_kernel != 0, totals, out);
      return;
    }
    // devices time their chunks concurrently: total = the slowest device
    if (count < 1) throw tcg::invalid_argument("count must be >= 1");
    const size_t nd = ctx->peers.size() + 1;
    const std::vector<int> b = chunks_of(count, nd);
    std::vector<tcg_timing> t(nd);
    std::vector<double> tot(static_cast<size_t>(count));
    for_all(ctx, [&](tcg::Engine& e, int d) {
      if (b[d + 1] > b[d])
        e.time_colorings(seed + static_cast<uint64_t>(b[d]), b[d + 1] - b[d], per_kernel != 0, tot.data() + b[d], &t[d]);
    });
    tcg_timing r{};
    for (const auto& x : t) {
      r.total_ms = std::max(r.total_ms, x.total_ms);
      r.spmm_ms = std::max(r.spmm_ms, x.spmm_ms);
      r.ema_ms = std::max(r.ema_ms, x.ema_ms);
      r.spmm_launches += x.spmm_launches;
      r.ema_launches += x.ema_launches;
      r.launches += x.launches;
      r.spmm_alg_bytes += x.spmm_alg_bytes;
      r.hist_alg_bytes += x.hist_alg_bytes;
      r.ema_alg_bytes += x.ema_alg_bytes;
      r.ema_flops += x.ema_flops;
      r.spmm_gathered_bytes += x.spmm_gathered_bytes;
    }
    *out = r;
    if (totals) std::copy(tot.begin(), tot.end(), totals);
  });
}

int tcg_shard_bounds(int32_t n, const int64_t* row_ptr, int world, int64_t* bounds) {
  return guarded([&] {
    need(row_ptr, "row_ptr");
    need(bounds, "bounds");
    const auto b = tcg::shard_bounds(n, row_ptr, world);
    std::copy(b.begin(), b.end(), bounds);
  });
}

int tcg_set_shard_device(tcg_ctx* ctx, int rank, int world, tcg_allgather_fn fn, void* user) {
  return guarded([&] {
    need(ctx, "ctx");
    if (!ctx->peers.empty()) throw tcg::invalid_argument("a multi-device context spreads colorings; shard with one context per rank");
    if (!fn) throw tcg::invalid_argument("allgather callback is NULL");
    ctx->eng->set_shard(rank, world, tcg::make_device_transport(fn, user));
  });
}

int tcg_nccl_unique_id(uint8_t id[TCG_NCCL_ID_BYTES]) {
  return guarded([&] {
    need(id, "id");
    tcg::nccl_unique_id(id);
  });
}

int tcg_set_shard_nccl(tcg_ctx* ctx, int rank, int world, const uint8_t id[TCG_NCCL_ID_BYTES]) {
  return guarded([&] {
    need(ctx, "ctx");
    if (!ctx->peers.empty()) throw tcg::invalid_argument("a multi-device context spreads colorings; shard with one context per rank");
    need(id, "id");
    if (world < 1 || rank < 0 || rank >= world) throw tcg::invalid_argument("bad shard rank/world");
    cudaSetDevice(ctx->eng->device());
    ctx->eng->set_shard(rank, world, tcg::make_nccl_transport(rank, world, id));
  });
}

struct tcg_loopback {
  std::shared_ptr<void> hub;
};

int tcg_loopback_create(int world, tcg_loopback** out) {
  return guarded([&] {
    need(out, "out");
    auto l = std::make_unique<tcg_loopback>();
    l->hub = tcg::make_loopback_hub(world);
    *out = l.release();
  });
}

void tcg_loopback_destroy(tcg_loopback* hub) { delete hub; }

int tcg_set_shard_loopback(tcg_ctx* ctx, int rank, tcg_loopback* hub) {
  return guarded([&] {
    need(ctx, "ctx");
    need(hub, "hub");
    if (!ctx->peers.empty()) throw tcg::invalid_argument("a multi-device context spreads colorings; shard with one context per rank");
    const int world = tcg::loopback_world(hub->hub);
    if (rank < 0 || rank >= world) throw tcg::invalid_argument("bad shard rank/world");
    cudaSetDevice(ctx->eng->device());
    ctx->eng->set_shard(rank, world, tcg::make_loopback_transport(hub->hub, rank));
  });
}

int tcg_set_shard_host(tcg_ctx* ctx, int rank, int world, tcg_allgather_fn fn, void* user) {
  return guarded([&] {
    need(ctx, "ctx");
    if (!ctx->peers.empty()) throw tcg::invalid_argument("a multi-device context spreads colorings; shard with one context per rank");
    if (!fn) throw tcg::invalid_argument("allgather callback is NULL");
    auto t = tcg::make_host_transport(fn, user);
    tcg::set_host_transport_world(t.get(), world);
    ctx->eng->set_shard(rank, world, std::move(t));
  });
}

int64_t tcg_kernel_launches(const tcg_ctx* ctx) {
  if (!ctx) return -1;
  int64_t s = ctx->eng->launches();
  for (const auto& p : ctx->peers) s += p->launches();
  return s;
}

}  // extern "C"
