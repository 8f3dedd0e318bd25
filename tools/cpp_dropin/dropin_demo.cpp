// dropin_demo.cpp -- the reference-side C++ binding (include/tcg_treecount.hpp)
// compiled against the UNMODIFIED reference headers and libtcg.so.
//
// host part (no GPU needed): the C-ABI status codes come back as the
//   reference's own exception types (parse_error / invalid_argument).
// device part (when a B200 is visible): treecount::b200::run_iteration and
//   ::estimate against treecount::run_iteration / ::estimate
//   (EngineKind::vectorized) on the same graph, plan and colorings:
//   per-vertex full_table and totals within 1e-4 relative, memory_budget_error
//   with required_bytes on a tiny budget.
// Prints "host-ok", then "gpu-ok" or "no-device"; exit 0 on success.
#include <cmath>
#include <cstdio>
#include <exception>

#include "tcg_treecount.hpp"
#include "treecount/synthgen.hpp"

using namespace treecount;

static int fail(const char* what) {
  std::printf("FAIL: %s\n", what);
  return 1;
}

int main() {
  // ---- host part: error contract
  {
    const int32_t bad_edges[] = {0, 1, 0, 1};  // k=3 with a repeated edge: not a tree
    tcg_plan p{};
    bool ok = false;
    try {
      b200::check(tcg_partition(3, bad_edges, 0, &p));
    } catch (const parse_error&) {
      ok = true;
    }
    if (!ok) return fail("bad template did not raise treecount::parse_error");
    ok = false;
    const int32_t cs[] = {3, 1};  // not strictly increasing
    try {
      if (tcg_color_index_of(5, cs, 2) < 0) b200::check(TCG_EINVAL);
    } catch (const parse_error&) {
      return fail("an invalid_argument came back as parse_error");
    } catch (const std::invalid_argument&) {
      ok = true;
    }
    if (!ok) return fail("bad color set did not raise std::invalid_argument");
    // the adapter rebuilds the template from a reference PartitionPlan
    TemplateTree t = make_template({{0, 1}, {1, 2}, {0, 3}, {3, 4}}, 0);
    PartitionPlan plan = partition(t);
    TemplateTree t2 = b200::template_of(plan);
    if (partition(t2).dp_order != plan.dp_order) return fail("template_of does not reproduce the plan");
    std::printf("host-ok\n");
  }
  // ---- device part
  tcg_ctx* probe = nullptr;
  tcg_config c{};
  if (tcg_create(&c, &probe) != TCG_OK) {
    std::printf("no-device\n");
    return 0;
  }
  tcg_destroy(probe);
  RmatSpec spec;
  spec.scale = 12;
  spec.edges = 24ll << 12;
  spec.a = .45; spec.b = .15; spec.c = .15; spec.d = .25;
  spec.seed = 3;
  Graph g = generate_rmat(spec);
  TemplateTree t = make_template({{0, 1}, {1, 2}, {2, 3}, {0, 4}, {4, 5}, {4, 6}, {6, 7}, {0, 8}, {8, 9}, {9, 10}, {9, 11}}, 0);
  PartitionPlan plan = partition(t);
  ColorIndexer idx(t.k);
  EngineConfig cfg;
  cfg.keep_full_table = true;
  cfg.workers = 4;
  auto rel = [](double a, double b) { return std::fabs(a - b) / std::fmax(std::fabs(b), 1e-300); };
  for (std::uint64_t seed = 1; seed <= 3; ++seed) {
    Coloring col = random_coloring(g, t.k, seed);
    IterationResult want = treecount::run_iteration(EngineKind::vectorized, g, plan, col, idx, cfg);
    IterationResult got = b200::run_iteration(g, plan, col, idx, cfg);
    if (rel(got.rooted_total, want.rooted_total) > 1e-4) return fail("rooted_total differs");
    for (vertex_t v = 0; v < g.n; ++v) {
      const double a = got.full_table->at(v, 0), b = want.full_table->at(v, 0);
      if ((a == 0) != (b == 0) || rel(a, b) > 1e-4) return fail("full_table differs");
    }
    if (got.neighbor_passes() != want.neighbor_passes()) return fail("neighbor_passes differ");
  }
  EstimateResult er = treecount::estimate(g, t, EngineKind::vectorized, 4, 11, cfg);
  EstimateResult eg = b200::estimate(g, t, 4, 11, cfg);
  for (int i = 0; i < 4; ++i)
    if (rel(eg.rooted_totals[i], er.rooted_totals[i]) > 1e-4) return fail("estimate totals differ");
  if (rel(eg.estimate, er.estimate) > 1e-4 || eg.aut != er.aut) return fail("estimate differs");
  bool budget = false;
  try {
    EngineConfig tiny;
    tiny.memory_budget = 1024;
    b200::run_iteration(g, plan, random_coloring(g, t.k, 1), idx, tiny);
  } catch (const memory_budget_error& e) {
    budget = e.required_bytes > 1024;
  }
  if (!budget) return fail("tiny budget did not raise memory_budget_error");
  std::printf("gpu-ok n=%d estimate=%.6e\n", g.n, eg.estimate);
  return 0;
}
