/*
 * tcg_treecount.hpp -- the reference-side C++ binding of libtcg.so.
 *
 * Header-only adapter a maintainer of the reference (treecount, header-only
 * C++20) adds next to engines.hpp so that the B200 engine is a drop-in for
 * the vectorized path:
 *
 *   treecount::b200::run_iteration(g, plan, coloring, indexer, cfg)
 *       == treecount::run_iteration(EngineKind::vectorized, g, plan, coloring,
 *                                   indexer, cfg)                (engines.hpp:302-336)
 *   treecount::b200::estimate(g, t, iterations, seed, cfg)
 *       == treecount::estimate(g, t, EngineKind::vectorized, iterations, seed,
 *                              cfg)                             (estimator.hpp:49-93)
 *
 * Same inputs, same result structs (IterationResult with per_node NodeStats
 * and the optional full_table column; EstimateResult), and the reference's
 * own exception types: status codes from the C ABI are rethrown as
 * treecount::parse_error (graph.hpp:18-21), std::invalid_argument,
 * treecount::memory_budget_error (engines.hpp:37-44, with required_bytes),
 * std::logic_error and std::runtime_error (CUDA / non-finite).
 *
 * Needs the reference headers on the include path (-I .../proj/include) and
 * links with -L paper_1903_04395_b200 -ltcg.  Compiled by
 * tools/cpp_dropin/Makefile and tests/test_cpp_dropin.py.
 */
#pragma once

#include <cstdint>
#include <cstdio>
#include <stdexcept>
#include <string>
#include <vector>

#include "tcg.h"
#include "treecount/engines.hpp"
#include "treecount/estimator.hpp"

namespace treecount {
namespace b200 {

// status -> the reference's exception class
inline void check(int st) {
  if (st == TCG_OK) return;
  const std::string msg = tcg_last_error() ? tcg_last_error() : "";
  switch (st) {
    case TCG_EPARSE: throw parse_error(msg);
    case TCG_EINVAL: throw std::invalid_argument(msg);
    case TCG_ERESOURCE: {
      long long need = 0, budget = 0;  // "count tables need N bytes, over the budget of B"
      if (std::sscanf(msg.c_str(), "count tables need %lld bytes, over the budget of %lld", &need, &budget) == 2)
        throw memory_budget_error(need, budget);
      throw std::runtime_error(msg);  // device out of memory (no budget set)
    }
    case TCG_ELOGIC: throw std::logic_error(msg);
    default: throw std::runtime_error(msg);  // TCG_ECUDA, TCG_ENONFINITE
  }
}

// The template a plan was partitioned from: one cut edge per internal node
// (templates.hpp:143-160 PlanNode::cut_edge), the plan's root.
inline TemplateTree template_of(const PartitionPlan& plan) {
  TemplateTree t;
  t.k = plan.k;
  t.root = plan.root;
  for (const PlanNode& nd : plan.nodes)
    if (!nd.is_leaf()) t.edges.push_back(nd.cut_edge);
  return t;
}

// One device context holding a graph and a template (tcg_create +
// tcg_set_graph + tcg_set_template); colorings reuse it.
class Context {
 public:
  Context(const Graph& g, const TemplateTree& t, const EngineConfig& cfg = {}, int device = 0) {
    tcg_config c{};
    c.device = device;
    c.memory_budget = cfg.memory_budget;
    check(tcg_create(&c, &ctx_));
    try {
      check(tcg_set_graph(ctx_, g.n, g.csc_col_ptr.data(), g.csc_rows.data()));
      std::vector<int32_t> e;
      for (auto [u, v] : t.edges) {
        e.push_back(u);
        e.push_back(v);
      }
      check(tcg_set_template(ctx_, t.k, e.empty() ? nullptr : e.data(), t.root));
    } catch (...) {
      tcg_destroy(ctx_);
      throw;
    }
  }
  ~Context() { tcg_destroy(ctx_); }
  Context(const Context&) = delete;
  Context& operator=(const Context&) = delete;
  tcg_ctx* get() const { return ctx_; }

 private:
  tcg_ctx* ctx_ = nullptr;
};

// run_iteration(EngineKind::vectorized, ...) on the device: the caller's
// coloring, rooted total, per-node stats, optional full_table column 0.
inline IterationResult run_iteration(Context& ctx, const Graph& g, const PartitionPlan& plan,
                                     const Coloring& coloring, const ColorIndexer& indexer,
                                     const EngineConfig& cfg = {}) {
  if (static_cast<std::size_t>(coloring.color.size()) != static_cast<std::size_t>(g.n))
    throw std::invalid_argument("coloring size does not match graph");
  if (indexer.k() != plan.k) throw std::invalid_argument("indexer and plan disagree on k");
  IterationResult r;
  r.engine = EngineKind::vectorized;
  std::vector<double> pv(cfg.keep_full_table ? static_cast<std::size_t>(g.n) : 0);
  std::vector<tcg_node_stats> st(plan.nodes.size());
  check(tcg_run_coloring(ctx.get(), coloring.seed, coloring.color.data(), &r.rooted_total,
                         cfg.keep_full_table ? pv.data() : nullptr, st.data()));
  r.per_node.resize(plan.nodes.size());
  for (std::size_t i = 0; i < st.size(); ++i) {
    r.per_node[i].seconds = st[i].seconds;
    r.per_node[i].neighbor_passes = st[i].neighbor_passes;
    r.per_node[i].traversals = st[i].traversals;
    r.per_node[i].flops = st[i].flops;
  }
  if (cfg.keep_full_table) {
    r.full_table = CountTable(g.n, 1, Layout::column_major);
    for (vertex_t i = 0; i < g.n; ++i) r.full_table->at(i, 0) = pv[static_cast<std::size_t>(i)];
  }
  return r;
}

// Single-shot form with the reference's signature (builds the context).
inline IterationResult run_iteration(const Graph& g, const PartitionPlan& plan, const Coloring& coloring,
                                     const ColorIndexer& indexer, const EngineConfig& cfg = {},
                                     int device = 0) {
  Context ctx(g, template_of(plan), cfg, device);
  return run_iteration(ctx, g, plan, coloring, indexer, cfg);
}

// estimate(g, t, vectorized, iterations, seed, cfg): colorings seed + i on
// the device, the reference's estimator arithmetic (estimator.hpp:80-91).
inline EstimateResult estimate(const Graph& g, const TemplateTree& t, int iterations, std::uint64_t seed,
                               const EngineConfig& cfg = {}, int device = 0) {
  if (iterations < 1) throw std::invalid_argument("iterations must be >= 1");
  Context ctx(g, t, cfg, device);
  EstimateResult r;
  r.iterations = iterations;
  r.rooted_totals.resize(static_cast<std::size_t>(iterations));
  check(tcg_estimate(ctx.get(), seed, iterations, r.rooted_totals.data(), &r.estimate, &r.stderr_of_mean,
                     nullptr));
  tcg_plan p{};
  std::uint64_t aut = 1;
  check(tcg_get_plan(ctx.get(), &p, &aut));
  r.aut = aut;
  r.colorful_probability = colorful_probability(t.k);
  return r;
}

}  // namespace b200
}  // namespace treecount
