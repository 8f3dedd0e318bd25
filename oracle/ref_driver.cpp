// ref_driver.cpp -- C-ABI shim over the UNMODIFIED reference headers.
//
// TEST / BASELINE INFRASTRUCTURE ONLY.  Compiled by oracle/Makefile from the
// reference sources where they lie (/root/reference/proj/include), with the
// reference's own flags (-std=c++20 -O3, no -march; proj/CMakeLists.txt:6-8,18)
// into oracle/_ref/libtcref.so.  Used (1) to pin the C restatement
// (tc_oracle.c) and generate tests/golden fixtures, and (2) as the CPU
// baseline / `bench.py --impl reference` arm.  Nothing here is product code.
#include <chrono>
#include <cstdint>
#include <cstring>
#include <exception>
#include <memory>
#include <vector>

#include "treecount/count_table.hpp"
#include "treecount/engines.hpp"
#include "treecount/estimator.hpp"
#include "treecount/la_kernels.hpp"
#include "treecount/synthgen.hpp"

using namespace treecount;

namespace {
TemplateTree make_tree(int k, const int32_t* edges, int root) {
  if (k == 1) return single_vertex_template();
  std::vector<std::pair<int, int>> e;
  for (int i = 0; i < k - 1; ++i) e.emplace_back(edges[2 * i], edges[2 * i + 1]);
  return make_template(std::move(e), root);
}
double now_s() {
  return std::chrono::duration<double>(std::chrono::steady_clock::now().time_since_epoch()).count();
}
}  // namespace

extern "C" {

void ref_random_coloring(int32_t n, int k, uint64_t seed, uint8_t* out) {
  Graph g;
  g.n = n;
  Coloring c = random_coloring(g, k, seed);
  std::memcpy(out, c.color.data(), static_cast<size_t>(n));
}

void ref_mt_first(uint64_t seed, int count, uint64_t* out) {
  Rng r(seed);
  for (int i = 0; i < count; ++i) out[i] = r.next_u64();
}

void* ref_graph_from_edges(const int32_t* edges, int64_t m, int32_t n_hint) {
  try {
    std::vector<std::pair<vertex_t, vertex_t>> e(static_cast<size_t>(m));
    for (int64_t i = 0; i < m; ++i) e[i] = {edges[2 * i], edges[2 * i + 1]};
    return new Graph(from_edges(std::move(e), n_hint));
  } catch (const std::exception&) {
    return nullptr;
  }
}

void* ref_generate_rmat(int scale, int64_t edges, double a, double b, double c, double d,
                        uint64_t seed) {
  try {
    RmatSpec s;
    s.scale = scale; s.edges = edges; s.a = a; s.b = b; s.c = c; s.d = d; s.seed = seed;
    return new Graph(generate_rmat(s));
  } catch (const std::exception&) {
    return nullptr;
  }
}

void* ref_generate_erdos_renyi(int32_t n, double p, uint64_t seed) {
  try {
    return new Graph(generate_erdos_renyi(n, p, seed));
  } catch (const std::exception&) {
    return nullptr;
  }
}

// Wrap an existing symmetric sorted CSR (e.g. built by the product's host
// code) as a reference Graph, so the reference engine runs on identical input.
void* ref_graph_from_csr(int32_t n, const int64_t* row_ptr, const int32_t* col) {
  auto* g = new Graph();
  g->n = n;
  g->m = row_ptr[n] / 2;
  g->adj.assign(static_cast<size_t>(n), {});
  for (int32_t v = 0; v < n; ++v) g->adj[v].assign(col + row_ptr[v], col + row_ptr[v + 1]);
  g->csc_col_ptr.assign(row_ptr, row_ptr + n + 1);
  g->csc_rows.assign(col, col + row_ptr[n]);
  return g;
}

void ref_graph_info(const void* gp, int32_t* n, int64_t* nnz) {
  const Graph* g = static_cast<const Graph*>(gp);
  *n = g->n;
  *nnz = static_cast<int64_t>(g->csc_rows.size());
}

void ref_graph_csr(const void* gp, int64_t* row_ptr, int32_t* col) {
  const Graph* g = static_cast<const Graph*>(gp);
  std::memcpy(row_ptr, g->csc_col_ptr.data(), g->csc_col_ptr.size() * sizeof(int64_t));
  std::memcpy(col, g->csc_rows.data(), g->csc_rows.size() * sizeof(int32_t));
}

void ref_graph_free(void* gp) { delete static_cast<Graph*>(gp); }

// Plan: per node id: size, root, active_child, passive_child; plus dp_order.
int ref_plan(int k, const int32_t* edges, int root, int* size, int* node_root, int* active,
             int* passive, int* dp_order, int* full_root) {
  try {
    TemplateTree t = make_tree(k, edges, root);
    PartitionPlan plan = partition(t);
    for (const PlanNode& nd : plan.nodes) {
      size[nd.id] = nd.size;
      node_root[nd.id] = nd.root;
      active[nd.id] = nd.active_child;
      passive[nd.id] = nd.passive_child;
    }
    for (size_t i = 0; i < plan.dp_order.size(); ++i) dp_order[i] = plan.dp_order[i];
    *full_root = t.root;
    return static_cast<int>(plan.nodes.size());
  } catch (const std::exception&) {
    return -1;
  }
}

int ref_split_table(int k, int parent, int active, int32_t* ai, int32_t* pi, int32_t* gp,
                    int32_t* ga) {
  try {
    ColorIndexer idx(k);
    SplitTable st = build_split_table(parent, active, idx);
    std::memcpy(ai, st.active_index.data(), st.active_index.size() * 4);
    std::memcpy(pi, st.passive_index.data(), st.passive_index.size() * 4);
    std::memcpy(gp, st.grouped_parent.data(), st.grouped_parent.size() * 4);
    std::memcpy(ga, st.grouped_active.data(), st.grouped_active.size() * 4);
    return 0;
  } catch (const std::exception&) {
    return -1;
  }
}

uint64_t ref_automorphisms(int k, const int32_t* edges) {
  try {
    return automorphism_count(make_tree(k, edges, -1));
  } catch (const std::exception&) {
    return 0;
  }
}

int64_t ref_estimate_bytes(int k, const int32_t* edges, int root, int64_t n) {
  try {
    return estimate_bytes(partition(make_tree(k, edges, root)), n, k);
  } catch (const std::exception&) {
    return -1;
  }
}

// run_iteration(EngineKind::vectorized, ..., keep_full_table) on a given coloring.
int ref_run_iteration(const void* gp, int k, const int32_t* edges, int root,
                      const uint8_t* colors, int workers, int batch, double* total,
                      double* per_vertex, double* seconds) {
  try {
    const Graph& g = *static_cast<const Graph*>(gp);
    TemplateTree t = make_tree(k, edges, root);
    PartitionPlan plan = partition(t);
    ColorIndexer idx(k);
    Coloring c;
    c.color.assign(colors, colors + g.n);
    EngineConfig cfg;
    cfg.workers = workers;
    cfg.batch = batch;
    cfg.keep_full_table = per_vertex != nullptr;
    const double t0 = now_s();
    IterationResult r = run_iteration(EngineKind::vectorized, g, plan, c, idx, cfg);
    if (seconds) *seconds = now_s() - t0;
    *total = r.rooted_total;
    if (per_vertex)
      for (vertex_t i = 0; i < g.n; ++i) per_vertex[i] = r.full_table->at(i, 0);
    return 0;
  } catch (const std::exception&) {
    return -1;
  }
}

int ref_estimate(const void* gp, int k, const int32_t* edges, int root, int iterations,
                 uint64_t seed, int workers, double* totals, double* estimate_out,
                 double* stderr_out, uint64_t* aut, double* seconds) {
  try {
    const Graph& g = *static_cast<const Graph*>(gp);
    EngineConfig cfg;
    cfg.workers = workers;
    const double t0 = now_s();
    EstimateResult r =
        estimate(g, make_tree(k, edges, root), EngineKind::vectorized, iterations, seed, cfg);
    if (seconds) *seconds = now_s() - t0;
    for (int i = 0; i < iterations; ++i) totals[i] = r.rooted_totals[i];
    *estimate_out = r.estimate;
    *stderr_out = r.stderr_of_mean;
    *aut = r.aut;
    return 0;
  } catch (const std::exception&) {
    return -1;
  }
}

// Bounded-sample timing of one vectorized coloring for the CPU baseline.
// Replays engines.hpp:224-268 through the reference's own public kernels
// (load_batch / spmm_csc / ema) and WorkerPool: for every internal node the
// first `max_batches` Z=16 SpMM batches over ALL rows and the first
// `max_pairs` eMA column pairs over ALL rows are timed, then extrapolated
// linearly to the node's full batch / pair count.  Random coloring and leaf
// init are timed in full.  out[0] = extrapolated s/coloring, out[1] = SpMM s,
// out[2] = eMA s, out[3] = measured wall seconds of the sample itself.
int ref_time_sampled(const void* gp, int k, const int32_t* edges, int root, uint64_t seed,
                     int workers, int max_batches, int max_pairs, double* out) {
  try {
    const Graph& g = *static_cast<const Graph*>(gp);
    TemplateTree t = make_tree(k, edges, root);
    PartitionPlan plan = partition(t);
    ColorIndexer idx(k);
    WorkerPool pool(workers);
    const int Z = 16;
    const double wall0 = now_s();
    double spmm_s = 0, ema_s = 0, misc_s = 0;

    double t0 = now_s();
    Coloring col = random_coloring(g, k, seed);
    CountTable leaf = init_leaf_table(col, k, Layout::column_major);
    misc_s += now_s() - t0;
    t0 = now_s();
    for (int rep = 1; rep < k; ++rep) leaf = init_leaf_table(col, k, Layout::column_major);
    misc_s += now_s() - t0;

    for (int id : plan.dp_order) {
      const PlanNode& nd = plan.node(id);
      if (nd.is_leaf()) continue;
      const int64_t cp = idx.num_sets(plan.node(nd.passive_child).size);
      const int64_t cs = idx.num_sets(nd.size);
      const int64_t pairs = cs * idx.binom(nd.size, plan.node(nd.active_child).size);
      // SpMM: stage + neighbour-sum batches, exactly vectorized_node's loop body
      {
        CountTable passive(g.n, Z, Layout::column_major);
        for (int z = 0; z < Z; ++z)
          for (vertex_t i = 0; i < g.n; ++i) passive.at(i, z) = leaf.at(i, (z + i) % k);
        const int64_t nbatch = (cp + Z - 1) / Z;
        const int64_t timed = std::min<int64_t>(nbatch, max_batches);
        double s = 0, cols_timed = 0;
        for (int64_t b = 0; b < timed; ++b) {
          const int zc = static_cast<int>(std::min<int64_t>(Z, cp - b * Z));
          const double b0 = now_s();
          RowBatch staged(g.n, zc);
          pool.for_range(static_cast<size_t>(g.n), [&](size_t lo, size_t hi, int) {
            load_batch(passive, 0, zc, staged, static_cast<vertex_t>(lo), static_cast<vertex_t>(hi));
          });
          ColumnBlock block{&passive, 0, zc};
          pool.for_range(static_cast<size_t>(g.n), [&](size_t lo, size_t hi, int) {
            spmm_csc(g, staged, block, static_cast<vertex_t>(lo), static_cast<vertex_t>(hi));
          });
          s += now_s() - b0;
          cols_timed += zc;
        }
        // full batches cost the measured average; scale by columns for the tail
        spmm_s += s / cols_timed * static_cast<double>(cp);
      }
      // eMA: one pool dispatch per (I_p, partner) pair (engines.hpp:252-268)
      {
        const int64_t timed = std::min<int64_t>(pairs, max_pairs);
        const int ncol = static_cast<int>(timed);
        CountTable out(g.n, ncol, Layout::column_major), act(g.n, ncol, Layout::column_major),
            pas(g.n, ncol, Layout::column_major);
        for (int z = 0; z < ncol; ++z)
          for (vertex_t i = 0; i < g.n; ++i) {
            act.at(i, z) = 1.0 + ((i + z) & 7);
            pas.at(i, z) = 2.0 + ((i ^ z) & 3);
          }
        const double e0 = now_s();
        for (int q = 0; q < ncol; ++q) {
          std::span<double> cs_ = out.column(q);
          std::span<const double> ca = act.column(q);
          std::span<const double> cpv = pas.column(q);
          pool.for_range(static_cast<size_t>(g.n), [&](size_t lo, size_t hi, int) {
            ema(cs_, ca, cpv, lo, hi);
          });
        }
        ema_s += (now_s() - e0) / static_cast<double>(timed) * static_cast<double>(pairs);
      }
    }
    out[0] = spmm_s + ema_s + misc_s;
    out[1] = spmm_s;
    out[2] = ema_s;
    out[3] = now_s() - wall0;
    return 0;
  } catch (const std::exception&) {
    return -1;
  }
}

}  // extern "C"
