// ref_driver.cpp -- C-ABI shim over the UNMODIFIED reference headers.
//
// TEST / BASELINE INFRASTRUCTURE ONLY.  Compiled by oracle/Makefile from the
// reference sources where they lie (/root/reference/proj/include), with the
// reference's own flags (-std=c++20 -O3, no -march; proj/CMakeLists.txt:6-8,18)
// into oracle/_ref/libtcref.so.  Used (1) to pin the C restatement
// (tc_oracle.c) and generate tests/golden fixtures, and (2) as the CPU
// baseline / `bench.py --impl reference` arm.  Nothing here is product code.
#include <algorithm>
#include <chrono>
#include <cstdint>
#include <cstring>
#include <exception>
#include <memory>
#include <optional>
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

// run_iteration(EngineKind::vectorized, ...) with the per-node NodeStats::seconds
// (engines.hpp:53-61,106-132): node_seconds[num_nodes] by plan node id.
int ref_run_iteration_stats(const void* gp, int k, const int32_t* edges, int root, uint64_t seed,
                            int workers, int batch, double* total, double* seconds,
                            double* node_seconds, int* num_nodes) {
  try {
    const Graph& g = *static_cast<const Graph*>(gp);
    TemplateTree t = make_tree(k, edges, root);
    PartitionPlan plan = partition(t);
    ColorIndexer idx(k);
    EngineConfig cfg;
    cfg.workers = workers;
    cfg.batch = batch;
    const double t0 = now_s();
    Coloring c = random_coloring(g, k, seed);
    IterationResult r = run_iteration(EngineKind::vectorized, g, plan, c, idx, cfg);
    if (seconds) *seconds = now_s() - t0;
    *total = r.rooted_total;
    *num_nodes = static_cast<int>(r.per_node.size());
    if (node_seconds)
      for (size_t i = 0; i < r.per_node.size(); ++i) node_seconds[i] = r.per_node[i].seconds;
    return 0;
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
//
// The reference engine's per-coloring cost is a sum of identical units
// (engines.hpp:224-268): every SpMM batch is load_batch + spmm_csc over the
// whole graph for zc <= Z=16 columns, and every eMA column pair is one
// pool-dispatched ema() over n rows.  So the sample times, through the
// reference's own kernels and WorkerPool, `reps` full-graph batches of Z=16
// and of 1 column, and `pairs` ema() dispatches, plus random_coloring and one
// init_leaf_table in full; the coloring is then
//   sum_nodes [ sum_batches t(zc) ] + pairs_total * t_pair + t_color + k * t_leaf
// with t(zc) interpolated linearly between t(1) and t(16).
// out[0] = estimated s/coloring, [1] SpMM s, [2] eMA s, [3] wall s of the
// sample, [4] t(16), [5] t(1), [6] t_pair, [7] t_color + k*t_leaf.
int ref_time_sampled(const void* gp, int k, const int32_t* edges, int root, uint64_t seed,
                     int workers, int reps, int pairs_sample, double* out) {
  try {
    const Graph& g = *static_cast<const Graph*>(gp);
    TemplateTree t = make_tree(k, edges, root);
    PartitionPlan plan = partition(t);
    ColorIndexer idx(k);
    WorkerPool pool(workers);
    const int Z = 16;
    const double wall0 = now_s();

    double t0 = now_s();
    Coloring col = random_coloring(g, k, seed);
    const double t_color = now_s() - t0;
    t0 = now_s();
    CountTable leaf = init_leaf_table(col, k, Layout::column_major);
    const double t_leaf = now_s() - t0;

    auto time_batch = [&](int zc) {
      CountTable passive(g.n, zc, Layout::column_major);
      for (int z = 0; z < zc; ++z)
        for (vertex_t i = 0; i < g.n; ++i) passive.at(i, z) = leaf.at(i, (z + i) % k);
      double best = 1e30;
      for (int r = 0; r < std::max(1, reps); ++r) {
        const double b0 = now_s();
        RowBatch staged(g.n, zc);
        pool.for_range(static_cast<size_t>(g.n), [&](size_t lo, size_t hi, int) {
          load_batch(passive, 0, zc, staged, static_cast<vertex_t>(lo), static_cast<vertex_t>(hi));
        });
        ColumnBlock block{&passive, 0, zc};
        pool.for_range(static_cast<size_t>(g.n), [&](size_t lo, size_t hi, int) {
          spmm_csc(g, staged, block, static_cast<vertex_t>(lo), static_cast<vertex_t>(hi));
        });
        best = std::min(best, now_s() - b0);
      }
      return best;
    };
    const double t16 = time_batch(Z);
    const double t1 = time_batch(1);
    auto t_of = [&](int zc) { return t1 + (t16 - t1) * (zc - 1) / (Z - 1); };

    double t_pair = 0;
    {
      const int ncol = std::max(1, pairs_sample);
      CountTable out_t(g.n, ncol, Layout::column_major), act(g.n, ncol, Layout::column_major),
          pas(g.n, 1, Layout::column_major);
      for (vertex_t i = 0; i < g.n; ++i) {
        pas.at(i, 0) = 2.0 + (i & 3);
        for (int z = 0; z < ncol; ++z) act.at(i, z) = 1.0 + ((i + z) & 7);
      }
      const double e0 = now_s();
      std::span<const double> cpv = pas.column(0);  // one passive column, several partners
      for (int q = 0; q < ncol; ++q) {
        std::span<double> cs_ = out_t.column(q);
        std::span<const double> ca = act.column(q);
        pool.for_range(static_cast<size_t>(g.n), [&](size_t lo, size_t hi, int) {
          ema(cs_, ca, cpv, lo, hi);
        });
      }
      t_pair = (now_s() - e0) / ncol;
    }

    double spmm_s = 0, ema_s = 0;
    for (int id : plan.dp_order) {
      const PlanNode& nd = plan.node(id);
      if (nd.is_leaf()) continue;
      const int64_t cp = idx.num_sets(plan.node(nd.passive_child).size);
      const int64_t cs = idx.num_sets(nd.size);
      const int64_t npairs = cs * idx.binom(nd.size, plan.node(nd.active_child).size);
      for (int64_t c0 = 0; c0 < cp; c0 += Z) spmm_s += t_of(static_cast<int>(std::min<int64_t>(Z, cp - c0)));
      ema_s += t_pair * static_cast<double>(npairs);
    }
    const double misc = t_color + k * t_leaf;
    out[0] = spmm_s + ema_s + misc;
    out[1] = spmm_s;
    out[2] = ema_s;
    out[3] = now_s() - wall0;
    out[4] = t16;
    out[5] = t1;
    out[6] = t_pair;
    out[7] = misc;
    return 0;
  } catch (const std::exception&) {
    return -1;
  }
}

// ---------------------------------------------------------------------------
// One coloring of the reference vectorized engine, replayed in K bounded steps.
//
// IterationRun::run (engines.hpp:106-132) with vectorized_node
// (engines.hpp:224-246) and accumulate_grouped (252-268) is a fixed sequence of
// pool-dispatched units over the reference's own public pieces:
// random_coloring (estimator.hpp:66), init_leaf_table per leaf, the zeroed
// output CountTable per internal node, one load_batch + spmm_csc pass per
// batch of <= Z passive columns, one ema() per grouped split (column pair),
// the release of the children, and the sequential root sum.  The stepper
// executes exactly that sequence, in that order, with the same WorkerPool
// slicing -- so the result is bit-identical to run_iteration (tests pin it) --
// but lets the caller time it in K slices of about equal estimated cost, so a
// full coloring of cfg3 (minutes on the host) is measured IN FULL across
// bench.py's K steps instead of being extrapolated from a sample.
struct RefStepper {
  const Graph* g = nullptr;
  int k = 0;
  uint64_t seed = 0;
  PartitionPlan plan;
  ColorIndexer idx{1};
  std::vector<SplitTable> splits;
  std::unique_ptr<WorkerPool> pool;
  int Z = 16;
  Coloring col;
  std::vector<std::optional<CountTable>> tables;
  enum Kind { COLOR, LEAF, ALLOC, SPMM, EMA, FREE, ROOT };
  struct Unit { Kind kind; int node; int a, b; double cost; };
  std::vector<Unit> units;
  std::vector<size_t> cuts;  // step i runs units [cuts[i], cuts[i+1])
  size_t next = 0;
  std::vector<double> node_sec, node_spmm, node_ema;
  double total = 0, color_sec = 0;
};

void* ref_step_begin(const void* gp, int k, const int32_t* edges, int root, uint64_t seed,
                     int workers, int batch, int steps) {
  try {
    auto st = std::make_unique<RefStepper>();
    st->g = static_cast<const Graph*>(gp);
    st->k = k;
    st->seed = seed;
    st->plan = partition(make_tree(k, edges, root));
    st->idx = ColorIndexer(k);
    st->splits = build_plan_splits(st->plan, st->idx);  // estimate(): once, before the colorings
    st->pool = std::make_unique<WorkerPool>(workers);
    st->Z = std::max(1, batch);
    st->tables.resize(st->plan.nodes.size());
    const double n = st->g->n, nnz = static_cast<double>(st->g->csc_col_ptr[st->g->n]);
    auto& u = st->units;
    u.push_back({RefStepper::COLOR, -1, 0, 0, 4 * n});
    for (int id : st->plan.dp_order) {
      const PlanNode& nd = st->plan.node(id);
      if (nd.is_leaf()) {
        u.push_back({RefStepper::LEAF, id, 0, 0, 8 * n * k});
        continue;
      }
      const SplitTable& sp = st->splits[static_cast<size_t>(id)];
      u.push_back({RefStepper::ALLOC, id, 0, 0, 8 * n * sp.parent_cols});
      for (int32_t c0 = 0; c0 < sp.passive_cols; c0 += st->Z) {
        const int zc = static_cast<int>(std::min<int32_t>(st->Z, sp.passive_cols - c0));
        u.push_back({RefStepper::SPMM, id, c0, zc, 8 * nnz * zc + 16 * n * zc});
      }
      for (int32_t ip = 0; ip < sp.passive_cols; ++ip)
        u.push_back({RefStepper::EMA, id, ip, 0, 32 * n * sp.partners_per_passive});
      u.push_back({RefStepper::FREE, id, 0, 0, 0});
    }
    u.push_back({RefStepper::ROOT, st->plan.full_node(), 0, 0, 8 * n});
    double tot = 0;
    for (auto& x : u) tot += x.cost;
    steps = std::max(1, steps);
    st->cuts.assign(static_cast<size_t>(steps) + 1, u.size());
    st->cuts[0] = 0;
    double cum = 0;
    size_t j = 0;
    for (int i = 1; i < steps; ++i) {
      const double target = tot * i / steps;
      while (j < u.size() && cum + u[j].cost * 0.5 < target) cum += u[j++].cost;
      st->cuts[static_cast<size_t>(i)] = j;
    }
    st->node_sec.assign(st->plan.nodes.size(), 0.0);
    st->node_spmm.assign(st->plan.nodes.size(), 0.0);
    st->node_ema.assign(st->plan.nodes.size(), 0.0);
    return st.release();
  } catch (const std::exception&) {
    return nullptr;
  }
}

static void ref_step_unit(RefStepper& s, const RefStepper::Unit& x) {
  const Graph& g = *s.g;
  WorkerPool& pool = *s.pool;
  const double t0 = now_s();
  switch (x.kind) {
    case RefStepper::COLOR:
      s.col = random_coloring(g, s.k, s.seed);
      break;
    case RefStepper::LEAF:
      s.tables[static_cast<size_t>(x.node)] = init_leaf_table(s.col, s.k, Layout::column_major);
      break;
    case RefStepper::ALLOC:
      s.tables[static_cast<size_t>(x.node)] =
          CountTable(g.n, s.splits[static_cast<size_t>(x.node)].parent_cols, Layout::column_major);
      break;
    case RefStepper::SPMM: {
      const PlanNode& nd = s.plan.node(x.node);
      CountTable& passive = *s.tables[static_cast<size_t>(nd.passive_child)];
      RowBatch staged(g.n, x.b);
      pool.for_range(static_cast<size_t>(g.n), [&](size_t lo, size_t hi, int) {
        load_batch(passive, x.a, x.b, staged, static_cast<vertex_t>(lo), static_cast<vertex_t>(hi));
      });
      ColumnBlock block{&passive, x.a, x.b};
      pool.for_range(static_cast<size_t>(g.n), [&](size_t lo, size_t hi, int) {
        spmm_csc(g, staged, block, static_cast<vertex_t>(lo), static_cast<vertex_t>(hi));
      });
      break;
    }
    case RefStepper::EMA: {
      const PlanNode& nd = s.plan.node(x.node);
      const SplitTable& st = s.splits[static_cast<size_t>(x.node)];
      const CountTable& active = *s.tables[static_cast<size_t>(nd.active_child)];
      const CountTable& passive = *s.tables[static_cast<size_t>(nd.passive_child)];
      CountTable& out = *s.tables[static_cast<size_t>(x.node)];
      std::span<const double> col_p = passive.column(x.a);
      const size_t base = static_cast<size_t>(x.a) * static_cast<size_t>(st.partners_per_passive);
      for (int q = 0; q < st.partners_per_passive; ++q) {
        std::span<double> col_s = out.column(st.grouped_parent[base + q]);
        std::span<const double> col_a = active.column(st.grouped_active[base + q]);
        pool.for_range(static_cast<size_t>(g.n), [&](size_t lo, size_t hi, int) { ema(col_s, col_a, col_p, lo, hi); });
      }
      break;
    }
    case RefStepper::FREE: {
      const PlanNode& nd = s.plan.node(x.node);
      s.tables[static_cast<size_t>(nd.active_child)].reset();
      s.tables[static_cast<size_t>(nd.passive_child)].reset();
      break;
    }
    case RefStepper::ROOT: {
      const CountTable& t = *s.tables[static_cast<size_t>(x.node)];
      double total = 0.0;
      for (vertex_t i = 0; i < g.n; ++i) total += t.at(i, 0);
      s.total = total;
      break;
    }
  }
  const double dt = now_s() - t0;
  if (x.node >= 0) {
    s.node_sec[static_cast<size_t>(x.node)] += dt;
    if (x.kind == RefStepper::SPMM) s.node_spmm[static_cast<size_t>(x.node)] += dt;
    if (x.kind == RefStepper::EMA) s.node_ema[static_cast<size_t>(x.node)] += dt;
  } else {
    s.color_sec += dt;
  }
}

// Runs step i's units; *seconds = its wall time.  Returns the units run or -1.
int ref_step_run(void* sp, int i, double* seconds) {
  try {
    RefStepper& s = *static_cast<RefStepper*>(sp);
    if (i < 0 || static_cast<size_t>(i) + 1 >= s.cuts.size()) return -1;
    const double t0 = now_s();
    const size_t end = s.cuts[static_cast<size_t>(i) + 1];
    int ran = 0;
    for (; s.next < end; ++s.next, ++ran) ref_step_unit(s, s.units[s.next]);
    if (seconds) *seconds = now_s() - t0;
    return ran;
  } catch (const std::exception&) {
    return -1;
  }
}

// After the last step: the rooted total, and per node id {seconds, spmm, ema}
// (node_stats[3 * num_nodes]); out[0] = coloring seconds, out[1] = units.
int ref_step_finish(void* sp, double* total, double* node_stats, int* num_nodes, double* out) {
  try {
    RefStepper& s = *static_cast<RefStepper*>(sp);
    if (s.next != s.units.size()) return -1;
    *total = s.total;
    *num_nodes = static_cast<int>(s.plan.nodes.size());
    if (node_stats)
      for (size_t i = 0; i < s.plan.nodes.size(); ++i) {
        node_stats[3 * i] = s.node_sec[i];
        node_stats[3 * i + 1] = s.node_spmm[i];
        node_stats[3 * i + 2] = s.node_ema[i];
      }
    if (out) {
      out[0] = s.color_sec;
      out[1] = static_cast<double>(s.units.size());
    }
    return 0;
  } catch (const std::exception&) {
    return -1;
  }
}

void ref_step_free(void* sp) { delete static_cast<RefStepper*>(sp); }

}  // extern "C"
