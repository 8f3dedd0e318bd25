"""GPU parity tests: the sm_100a path (through the C ABI) against the pinned
CPU oracle and the reference's golden vectors.

Tolerances (north star): colorings bit-exact; count tables / per-vertex /
totals within 1e-4 relative.  Where every value is an integer below 2^24
(cfg1, the reference's KAT graphs) fp32 tables are exact, so those cases are
checked for exact equality.
"""
import os

import numpy as np
import pytest

import oracle as O
import paper_1903_04395_b200 as T
from conftest import CFG_TEMPLATES, GOLDEN, parents_to_edges

pytestmark = pytest.mark.gpu
REL = 1e-4


def ctx_for(g, t, keep=False, budget=0):
    c = T.Context(0, budget, keep)
    c.set_graph(g)
    c.set_template(t)
    return c


def rel_err(a, b):
    a, b = np.asarray(a, np.float64), np.asarray(b, np.float64)
    return float(np.max(np.abs(a - b) / np.maximum(np.abs(b), 1e-300), initial=0.0))


def assert_close(got, want, rel=REL):
    got, want = np.asarray(got, np.float64), np.asarray(want, np.float64)
    assert got.shape == want.shape
    assert np.array_equal(got == 0, want == 0), "zero pattern differs"
    assert rel_err(got, want) <= rel, rel_err(got, want)


# ------------------------------------------------------------------ colorings
@pytest.mark.parametrize("n", [1, 5, 155, 156, 311, 312, 313, 624, 1000, 100003])
@pytest.mark.parametrize("k", [1, 2, 5, 7, 12, 17, 20])
def test_coloring_bit_exact(n, k):
    g = T.from_edges([(0, 0)], n)
    c = T.random_coloring(g, k, 1 + n % 7)
    assert np.array_equal(c.color, O.random_coloring(n, k, 1 + n % 7))


def test_coloring_golden(kats):
    g = T.from_edges([(0, 0)], 24)
    for key, want in kats["coloring24"].items():
        k, seed = map(int, key.split("_"))
        assert T.random_coloring(g, k, seed).color.tolist() == want, key
    g = T.from_edges([(0, 0)], 100003)
    for k, d in kats["coloring100003_seed7"].items():
        c = T.random_coloring(g, int(k), 7).color.astype(np.int64)
        assert int(c.sum()) == d["sum"] and c[:16].tolist() == d["head"]


@pytest.mark.parametrize("limit_div", [3, 2, 1.05])
def test_coloring_rejection_path(limit_div):
    """Forced rejections (test hook on Rng::below's threshold) vs the oracle."""
    n, k = 50000, 7
    limit = int((2 ** 64 - 1) / limit_div)
    g = T.from_edges([(0, 0)], n)
    c = ctx_for(g, T.TemplateTree(k, [(i, i + 1) for i in range(k - 1)], 0))
    c.set_rejection_limit(limit)
    got = c.coloring(5)
    assert np.array_equal(got, O.random_coloring(n, k, 5, limit))


def test_coloring_distribution():
    # test_count_table.cpp:28-44: each color within 3 sigma of n/k
    n, k = 100000, 5
    c = T.random_coloring(T.from_edges([(0, 0)], n), k, 2024).color
    freq = np.bincount(c, minlength=k)
    sigma = np.sqrt(n * (1 / k) * (1 - 1 / k))
    assert np.all(np.abs(freq - n / k) <= 3 * sigma)


# ----------------------------------------------------------------------- SpMM
def spmm_ctx(g):
    c = T.Context(0)
    c.set_graph(g)
    return c


def dense_ref(g, x):
    y = np.zeros_like(x, dtype=np.float64)
    for v in range(g.n):
        y[v] = x[g.neighbors(v)].astype(np.float64).sum(axis=0)
    return y


def test_spmm_spec_examples():
    # test_la_kernels.cpp:24-43
    g = T.from_edges([(0, 1)])
    assert spmm_ctx(g).spmm(np.array([1, 2], np.float32)).ravel().tolist() == [2, 1]
    g = T.from_edges([(0, 1), (1, 2), (2, 0)])
    assert spmm_ctx(g).spmm(np.array([1, 2, 3], np.float32)).ravel().tolist() == [5, 4, 3]
    assert spmm_ctx(g).spmm(np.zeros(3, np.float32)).ravel().tolist() == [0, 0, 0]


def test_spmm_all_ones_is_degree():
    g = T.generate_rmat(T.RmatSpec(12, 8 << 12, .57, .19, .19, .05, 4))
    y = spmm_ctx(g).spmm(np.ones((g.n, 3), np.float32))
    assert np.array_equal(y[:, 0], np.diff(g.csc_col_ptr).astype(np.float32))


@pytest.mark.parametrize("width", [1, 3, 16, 17, 40])
def test_spmm_dense_reference_integer_valued(width):
    rng = np.random.default_rng(width)
    for trial in range(4):
        n = int(rng.integers(2, 400))
        e = rng.integers(0, n, size=(int(rng.integers(1, 6 * n)), 2))
        g = T.from_edges(e, n)
        x = rng.integers(0, 17, size=(n, width)).astype(np.float32)
        assert np.array_equal(spmm_ctx(g).spmm(x), dense_ref(g, x).astype(np.float32))


def test_spmm_hub_rows_split_segments():
    """Rows longer than one segment (kSegMax=1024) take the fp64 partial path."""
    hub_deg = 5000
    e = [(0, v) for v in range(1, hub_deg + 1)] + [(1, v) for v in range(2, 2100)]
    g = T.from_edges(e)
    rng = np.random.default_rng(0)
    x = rng.integers(0, 1000, size=(g.n, 20)).astype(np.float32)
    y = spmm_ctx(g).spmm(x)
    assert np.array_equal(y, dense_ref(g, x).astype(np.float32))


# ------------------------------------------------ production rooted SpMM (tcg_spmm_rooted)
def rooted_table(rng, n, k, s, colors, hi=1000):
    """Random integer-valued passive table, rooted: M[u, S] = 0 unless c(u) in S."""
    ix = T.ColorIndexer(k)
    has = np.array([[c in ix.set_of(S, s) for c in range(k)] for S in range(ix.num_sets(s))])  # [S, c]
    x = rng.integers(0, hi, size=(n, ix.num_sets(s))).astype(np.float32)
    x[~has[:, colors].T] = 0
    return x, has


def dense_rooted_ref(g, x, has, colors):
    y = dense_ref(g, x)
    y[has[:, colors].T] = 0  # only the columns missing c(v) are computed
    return y


@pytest.mark.parametrize("pair", [False, True])
def test_spmm_rooted_spec_examples(pair):
    # test_la_kernels.cpp:24-43 through the production kernel: with k = 2 (3 for
    # the pair layout), s = 1 and colors c, the consumed column of row v is
    # {c(u)} for its neighbours u, so y carries the spmv KATs
    k = 3 if pair else 2
    g = T.from_edges([(0, 1)])
    c = spmm_ctx(g)
    x = np.zeros((2, k), np.float32)
    x[0, 0], x[1, 1] = 1, 2
    y = c.spmm_rooted(k, 1, np.array([0, 1], np.uint8), x, pair)
    assert y[0, 1] == 2 and y[1, 0] == 1
    g = T.from_edges([(0, 1), (1, 2), (2, 0)])
    x = np.zeros((3, k), np.float32)
    for v, val in enumerate([1, 2, 3]):
        x[v, v % k] = val
    y = spmm_ctx(g).spmm_rooted(k, 1, np.array([v % k for v in range(3)], np.uint8), x, pair)
    if not pair:  # k = 2: vertices 0 and 2 share color 0
        assert y[0, 1] == 2 and y[1, 0] == 1 + 3 and y[2, 1] == 2
    else:
        assert y[0, 1] == 2 and y[0, 2] == 3 and y[1, 0] == 1 and y[1, 2] == 3 and y[2, 0] == 1 and y[2, 1] == 2


@pytest.mark.parametrize("pair", [False, True])
@pytest.mark.parametrize("k,s", [(5, 2), (7, 3), (12, 4), (12, 5), (15, 3)])
def test_spmm_rooted_dense_reference_integer_valued(k, s, pair):
    """The default SpMM kernel (spmm_rooted) is EXACT on integer-valued tables
    (fp32 8-neighbour trees below 2^24, fp64 run sums): random graphs whose
    rows include hubs above one segment (1,024) and above one bucketing chunk
    (4,096 neighbours: bucket_long), against the dense reference."""
    rng = np.random.default_rng(k * 100 + s + pair)
    for trial in range(3):
        n = int(rng.integers(200, 9000))
        e = [tuple(x) for x in rng.integers(0, n, size=(int(rng.integers(2, 12)) * n, 2))]
        hubs = rng.choice(n, size=3, replace=False)
        for h, d in zip(hubs, (n - 1, 5000, 1500)):
            e += [(int(h), int(u)) for u in rng.choice(n, size=min(d, n - 1), replace=False) if u != h]
        g = T.from_edges(e, n)
        colors = rng.integers(0, k, size=n).astype(np.uint8)
        x, has = rooted_table(rng, n, k, s, colors, hi=1000)
        y = spmm_ctx(g).spmm_rooted(k, s, colors, x, pair)
        assert np.array_equal(y, dense_rooted_ref(g, x, has, colors).astype(np.float32)), (trial, n)


def test_spmm_rooted_isolated_and_empty():
    g = T.from_edges([(0, 1)], 40)  # 38 isolated vertices (compacted away internally)
    k, s = 4, 2
    colors = (np.arange(40) % k).astype(np.uint8)
    x, has = rooted_table(np.random.default_rng(1), 40, k, s, colors)
    y = spmm_ctx(g).spmm_rooted(k, s, colors, x)
    assert np.array_equal(y, dense_rooted_ref(g, x, has, colors).astype(np.float32))
    assert np.all(y[2:] == 0)


# ---------------------------------------------------------------- engine KATs
def test_engine_kat_k3_edge():
    # test_engines.cpp:28-41
    g = T.from_edges([(0, 1), (1, 2), (2, 0)])
    t = T.make_template([(0, 1)], 0)
    r = T.run_iteration(T.EngineKind.b200, g, T.partition(t), T.Coloring(np.array([0, 1, 0], np.uint8)),
                        T.ColorIndexer(2), T.EngineConfig(keep_full_table=True))
    assert r.rooted_total == 4.0
    assert r.full_table.ravel().tolist() == [1.0, 2.0, 1.0]


def test_engine_kat_single_vertex():
    g = T.generate_erdos_renyi(37, 0.1, 2)
    t = T.single_vertex_template()
    r = T.run_iteration(T.EngineKind.b200, g, t, T.random_coloring(g, 1, 5))
    assert r.rooted_total == 37.0
    e = T.estimate(g, t, T.EngineKind.b200, 3, 1)
    assert e.estimate == 37.0


def test_engine_kat_k3_path_rainbow():
    g = T.from_edges([(0, 1), (1, 2), (2, 0)])
    t = T.make_template([(0, 1), (1, 2)])
    r = T.run_iteration(T.EngineKind.b200, g, t, T.Coloring(np.array([0, 1, 2], np.uint8)))
    assert r.rooted_total == 6.0


def test_pass_counts_follow_table2():
    # test_engines.cpp:158-186: neighbor passes = sum over internal nodes of C(k, |T_p|)
    g = T.generate_erdos_renyi(40, 0.1, 3)
    k = 5
    t = T.make_template([(v - 1, v) for v in range(1, k)])
    plan = T.partition(t)
    ix = T.ColorIndexer(k)
    r = T.run_iteration(T.EngineKind.b200, g, plan, T.random_coloring(g, k, 19))
    want = sum(ix.num_sets(plan.node(nd.passive_child).size) for nd in plan.nodes if not nd.is_leaf())
    assert r.neighbor_passes() == want
    assert r.traversals() == want * g.n


# ------------------------------------------------------------- oracle parity
def test_cfg1_bit_exact(cfg1_golden):
    gold = cfg1_golden
    g = T.Graph.from_csr(16384, gold["row_ptr"], gold["col"])
    t = T.template_from_parents(CFG_TEMPLATES["cfg1"], 0)
    c = ctx_for(g, t)
    total, pv, _ = c.run_coloring(1, per_vertex=True)
    assert total == 41315622.0
    assert np.array_equal(pv, gold["per_vertex_seed1"])
    totals, est, se, pve = c.estimate(1, 10, per_vertex=True)
    assert totals.tolist() == gold["totals_seeds1_10"].tolist()
    assert est == float(gold["estimate"]) and se == float(gold["stderr"])
    # per-vertex estimate = mean of per-vertex root counts / (aut * k!/k^k)
    acc = np.zeros(16384)
    for s in range(1, 11):
        acc += c.run_coloring(s, per_vertex=True)[1]
    assert_close(pve, acc / 10 / (2 * T.colorful_probability(5)), 1e-12)


def test_small_instances_exact(kats):
    """Reference-generated instances (random graphs/trees/roots/colorings)."""
    for inst in kats["small_instances"]:
        g = T.from_edges(inst["edges"], inst["n"])
        t = T.template_from_parents(inst["parents"], inst["root"])
        c = ctx_for(g, t)
        total, pv, _ = c.run_coloring(inst["seed"], per_vertex=True)
        assert total == inst["total"]
        assert pv.tolist() == inst["per_vertex"]


def _random_case(rng, n, k, deg):
    e = rng.integers(0, n, size=(int(deg * n / 2), 2))
    g = T.from_edges(e, n)
    parents = [-1] + [int(rng.integers(0, v)) for v in range(1, k)]
    return g, parents


@pytest.mark.parametrize("seed", range(6))
def test_node_tables_match_oracle(seed):
    """Every internal node table and every SpMM output P' vs the oracle."""
    rng = np.random.default_rng(100 + seed)
    n, k = int(rng.integers(50, 3000)), int(rng.integers(3, 11))
    g, parents = _random_case(rng, n, k, float(rng.integers(2, 40)))
    root = int(rng.integers(0, k))
    t = T.template_from_parents(parents, root)
    c = ctx_for(g, t, keep=True)
    total, pv, _ = c.run_coloring(seed, per_vertex=True)
    plan = O.partition(k, parents_to_edges(parents), root)
    colors = O.random_coloring(n, k, seed)
    ototal, opv, tabs = O.run_iteration(n, g.csc_col_ptr, g.csc_rows, plan, colors, want_tables=True)
    assert np.array_equal(c.coloring(seed), colors)
    for nid, want in tabs.items():
        got = c.node_table(nid, 0)
        assert_close(got, want)
    # SpMM outputs of internal passive children
    for nd in T.partition(t).nodes:
        if nd.is_leaf():
            continue
        p = nd.passive_child
        if not T.partition(t).node(p).is_leaf():
            want = np.stack([tabs[p][g.neighbors(v)].sum(axis=0) for v in range(n)])
            # P'[v, T] is computed where T misses c(v) (the consumed columns)
            sp = T.partition(t).node(p).size
            ix = T.ColorIndexer(k)
            has = np.array([[c in ix.set_of(S, sp) for c in range(k)] for S in range(ix.num_sets(sp))])
            want[has[:, colors].T] = 0.0
            assert_close(c.node_table(p, 1), want)
    assert_close(pv, opv)
    assert rel_err([total], [ototal]) <= 1e-12 or rel_err([total], [ototal]) <= REL


@pytest.mark.parametrize("k", [13, 16])
def test_large_k_unstaged_ema(k):
    """k >= 13 produces eMA nodes whose tiles do not fit in shared memory
    (the global-operand variant) -- still parity with the oracle."""
    rng = np.random.default_rng(k)
    g, parents = _random_case(rng, 120, k, 12)
    t = T.template_from_parents(parents, 0)
    c = ctx_for(g, t)
    total, pv, _ = c.run_coloring(3, per_vertex=True)
    plan = O.partition(k, parents_to_edges(parents), 0)
    ototal, opv, _ = O.run_iteration(g.n, g.csc_col_ptr, g.csc_rows, plan, O.random_coloring(g.n, k, 3))
    assert_close(pv, opv)
    assert rel_err([total], [ototal]) <= REL


@pytest.mark.parametrize("name", ["cfg4", "cfg5"])
def test_k15_k17_templates_small_graph(name):
    """The cfg4/cfg5 templates (k=15/17): wide nodes take the vertex-per-CTA
    eMA kernels (blocked, active-leaf, root) -- parity with the oracle."""
    g = T.generate_rmat(T.RmatSpec(9, 48 << 9, .45, .15, .15, .25, 7))
    parents = CFG_TEMPLATES[name]
    k = len(parents)
    c = ctx_for(g, T.template_from_parents(parents, 0))
    total, pv, _ = c.run_coloring(2, per_vertex=True)
    plan = O.partition(k, parents_to_edges(parents), 0)
    ototal, opv, _ = O.run_iteration(g.n, g.csc_col_ptr, g.csc_rows, plan, O.random_coloring(g.n, k, 2))
    assert ototal > 0
    assert_close(pv, opv)
    assert rel_err([total], [ototal]) <= REL


def test_given_coloring_matches_seeded(cfg1_golden):
    gold = cfg1_golden
    g = T.Graph.from_csr(16384, gold["row_ptr"], gold["col"])
    t = T.template_from_parents(CFG_TEMPLATES["cfg1"], 0)
    c = ctx_for(g, t)
    colors = O.random_coloring(16384, 5, 4)
    a = c.run_coloring(0, colors=colors)[0]
    b = c.run_coloring(4)[0]
    assert a == b == float(gold["totals_seeds1_10"][3])


def test_prefetched_next_coloring_is_the_seeded_coloring():
    """run_coloring(seed) generates the coloring of seed + 1 on a side stream (graphs of >= 65,536
    vertices): consecutive seeds, a repeated seed, a jump, a template with another k in between and
    a caller-given coloring must all give what a context that never prefetches gives."""
    g = T.generate_rmat(T.RmatSpec(17, 4 << 17, .57, .19, .19, .05, 3))
    t5 = T.template_from_parents([-1, 0, 1, 1, 3], 0)
    t3 = T.template_from_parents([-1, 0, 0], 0)

    def fresh(t, seed):  # (first call of a new context: nothing prefetched)
        return ctx_for(g, t).run_coloring(seed)[0]

    c = ctx_for(g, t5)
    want = {s: fresh(t5, s) for s in (7, 8, 9, 20)}
    assert [c.run_coloring(s)[0] for s in (7, 8, 9, 9, 20, 8)] == [want[s] for s in (7, 8, 9, 9, 20, 8)]
    colors = O.random_coloring(g.n, 5, 9)
    assert c.run_coloring(0, colors=colors)[0] == want[9]
    assert np.array_equal(c.coloring(9), colors)
    c.run_coloring(30)                       # leaves seed 31 of k = 5 prefetched
    c.set_template(t3)
    assert c.run_coloring(31)[0] == fresh(t3, 31)
    c.set_template(t5)
    assert c.run_coloring(32)[0] == fresh(t5, 32)


def test_set_graph_buffer_reuse():
    """One context, a sequence of host-CSR graphs that grow, shrink and grow
    again (device graph buffers, the device-built schedules, the arena and the
    estimate buffers are reused when they fit): every result equals the oracle."""
    parents = [-1, 0, 1, 2, 0, 4, 4, 6, 0, 8]
    k = len(parents)
    plan = O.partition(k, parents_to_edges(parents), 0)
    t = T.template_from_parents(parents, 0)
    c = T.Context(0)
    c.set_template(t)
    rng = np.random.default_rng(11)
    for i, (scale, ef) in enumerate([(9, 16), (12, 48), (8, 8), (12, 24), (11, 64)]):
        g = T.generate_rmat(T.RmatSpec(scale, ef << scale, .45, .15, .15, .25, 1 + i))
        rp = np.ascontiguousarray(g.csc_col_ptr, np.int64)
        cl = np.ascontiguousarray(g.csc_rows, np.int32)
        c.set_graph_csr(g.n, rp, cl)
        seed = int(rng.integers(1, 1 << 30))
        totals, est, se, pv = c.estimate(seed, 2, per_vertex=True)
        want = []
        opv = np.zeros(g.n)
        for j in range(2):
            colors = O.random_coloring(g.n, k, seed + j)
            tot, vv, _ = O.run_iteration(g.n, g.csc_col_ptr, g.csc_rows, plan, colors)
            want.append(tot)
            opv += vv
        assert rel_err(totals, want) <= REL, (i, totals, want)
        scale_f = est / np.mean(totals) if np.mean(totals) else 1.0
        assert_close(pv, opv / 2 * scale_f)


# ------------------------------------------------------------ full-size cases
def _load(name):
    p = os.path.join(GOLDEN, f"{name}.npz")
    if not os.path.exists(p):
        pytest.skip(f"{name} golden fixture not generated")
    return dict(np.load(p))


CFG_GRAPH = {"cfg2": (20, 16 << 20, .57, .19, .19, .05, 1), "cfg3": (20, 100 << 20, .45, .15, .15, .25, 1)}


@pytest.mark.parametrize("name", ["cfg2", "cfg3"])
def test_full_size_against_reference(name):
    gold = _load(name)
    g = T.generate_rmat(T.RmatSpec(*CFG_GRAPH[name]))
    assert g.n == int(gold["n"]) and g.nnz() == int(gold["nnz"])
    assert int(g.csc_col_ptr.sum() % (1 << 61)) == int(gold["row_ptr_checksum"])
    t = T.template_from_parents(CFG_TEMPLATES[name], 0)
    c = ctx_for(g, t)
    idx = gold["sample_idx"]
    for i, s in enumerate(gold["seeds"]):
        total, pv, _ = c.run_coloring(int(s), per_vertex=True)
        assert rel_err([total], [gold["totals"][i]]) <= REL
        assert_close(pv[idx], gold[f"pv_seed{int(s)}"])
        if i == 0:
            assert rel_err([pv.sum()], [gold[f"pv_sum_seed{int(s)}"]]) <= REL
            assert int((pv == 0).sum()) == int(gold[f"zero_rows_seed{int(s)}"])


def test_relabeling_invariance():
    """Size-independent property: permuting vertex ids (and the coloring with
    them) permutes the per-vertex counts and leaves the total unchanged."""
    g = T.generate_rmat(T.RmatSpec(16, 16 << 16, .57, .19, .19, .05, 2))
    t = T.template_from_parents(CFG_TEMPLATES["cfg2"], 0)
    colors = O.random_coloring(g.n, 7, 9)
    tot, pv, _ = ctx_for(g, t).run_coloring(0, colors=colors, per_vertex=True)
    perm = np.random.default_rng(1).permutation(g.n).astype(np.int32)
    src = np.repeat(np.arange(g.n, dtype=np.int32), np.diff(g.csc_col_ptr))
    e = np.stack([perm[src], perm[g.csc_rows]], 1)
    g2 = T.from_edges(e, g.n)
    colors2 = np.empty_like(colors)
    colors2[perm] = colors
    tot2, pv2, _ = ctx_for(g2, t).run_coloring(0, colors=colors2, per_vertex=True)
    assert rel_err([tot2], [tot]) <= 1e-9
    assert_close(pv2[perm], pv, 1e-6)


def test_root_independence_of_totals():
    """Totals do not depend on the template root (SURVEY finding 9)."""
    g = T.generate_rmat(T.RmatSpec(14, 16 << 14, .57, .19, .19, .05, 3))
    parents = CFG_TEMPLATES["cfg3"]
    totals = [ctx_for(g, T.template_from_parents(parents, r)).run_coloring(5)[0] for r in (0, 3, 7, -1)]
    for x in totals[1:]:
        assert rel_err([x], [totals[0]]) <= 1e-6


def test_estimate_is_mean_of_colorings():
    g = T.generate_rmat(T.RmatSpec(13, 8 << 13, .45, .15, .15, .25, 4))
    t = T.template_from_parents(CFG_TEMPLATES["cfg2"], 0)
    c = ctx_for(g, t)
    totals, est, se, _ = c.estimate(11, 5)
    single = [c.run_coloring(11 + i)[0] for i in range(5)]
    assert totals.tolist() == single
    o = O.estimate(g.n, g.csc_col_ptr, g.csc_rows, 7, parents_to_edges(CFG_TEMPLATES["cfg2"]), 0, 5, 11)
    assert rel_err(totals, o["rooted_totals"]) <= REL
    assert rel_err([est], [o["estimate"]]) <= REL


# ------------------------------------------------------------------- errors
def test_memory_budget_refusal():
    g = T.generate_erdos_renyi(100, 0.05, 5)
    t = T.make_template([(v - 1, v) for v in range(1, 6)])
    c = ctx_for(g, t, budget=1024)
    with pytest.raises(T.MemoryBudgetError) as ei:
        c.run_coloring(1)
    assert ei.value.required_bytes > 1024
    assert c.required_device_bytes() > 0


def test_bad_coloring_refused():
    g = T.from_edges([(0, 1), (1, 2)])
    c = ctx_for(g, T.make_template([(0, 1)], 0))
    with pytest.raises(T.InvalidArgument):
        c.run_coloring(0, colors=np.array([0, 1, 5], np.uint8))
    with pytest.raises(T.InvalidArgument):
        c.run_coloring(0, colors=np.array([0, 1], np.uint8))


def test_iterations_must_be_positive():
    g = T.from_edges([(0, 1)])
    with pytest.raises(T.InvalidArgument) as ei:
        T.estimate(g, T.make_template([(0, 1)], 0), T.EngineKind.b200, 0, 1)
    assert not isinstance(ei.value, T.ParseError)


def test_isolated_and_empty_rows():
    g = T.from_edges([(0, 1)], 50)  # 48 isolated vertices
    t = T.make_template([(0, 1), (1, 2)], 0)
    c = ctx_for(g, t)
    total, pv, _ = c.run_coloring(2, per_vertex=True)
    assert total == 0.0 and np.all(pv == 0)


def test_set_graph_csr_validated_on_device():
    """tcg_set_graph uploads the caller's CSR and checks the reference's Graph
    invariants on the device: ids in range, no self-loops, rows strictly
    ascending (graph.hpp:65-95 produces exactly such rows)."""
    c = T.Context(0)
    c.set_template(T.make_template([(0, 1), (1, 2)], 0))
    rp = np.array([0, 1, 3, 4], np.int64)
    c.set_graph_csr(3, rp, np.array([1, 0, 2, 1], np.int32))  # the path 0-1-2
    total, _, _ = c.run_coloring(1)
    assert total >= 0
    for bad in ([1, 0, 3, 1],      # id out of range
                [1, 1, 2, 1],      # self-loop in row 1
                [1, 2, 0, 1]):     # row 1 not ascending
        with pytest.raises(T.ParseError):
            c.set_graph_csr(3, rp, np.array(bad, np.int32))
    with pytest.raises(T.ParseError):
        c.set_graph_csr(3, np.array([0, 2, 1, 4], np.int64), np.array([1, 0, 2, 1], np.int32))
    # the context is usable again after a rejected graph
    c.set_graph_csr(3, rp, np.array([1, 0, 2, 1], np.int32))
    assert c.run_coloring(1)[0] == total


def test_host_csr_and_graph_handle_agree():
    """The e2e entry (host CSR buffers, device validation, O(n) host schedules)
    and the Graph-handle entry give identical results."""
    g = T.generate_rmat(T.RmatSpec(13, 24 << 13, .45, .15, .15, .25, 4))
    t = T.template_from_parents(CFG_TEMPLATES["cfg3"], 0)
    a = ctx_for(g, t)
    b = T.Context(0)
    b.set_template(t)
    b.set_graph_csr(g.n, np.ascontiguousarray(g.csc_col_ptr), np.ascontiguousarray(g.csc_rows))
    ta, pa, _ = a.run_coloring(3, per_vertex=True)
    tb, pb, _ = b.run_coloring(3, per_vertex=True)
    assert ta == tb and np.array_equal(pa, pb)


# ------------------------------------------------- device CSR build (from_edges)
@pytest.mark.parametrize("trial", range(4))
def test_device_from_edges_equals_reference_csr(trial):
    """tcg_set_graph_edges builds graph.hpp:65-95's CSR on the device (radix
    sort + dedup): identical to the host from_edges on raw edge lists with
    self-loops, duplicates and both directions; results are bit-identical."""
    rng = np.random.default_rng(trial)
    n = int(rng.integers(2, 30000))
    m = int(rng.integers(1, 12 * n))
    e = rng.integers(0, n, size=(m, 2)).astype(np.int32)
    e[: m // 10, 1] = e[: m // 10, 0]            # self-loops
    e = np.concatenate([e, e[: m // 5, ::-1], e[: m // 7]])  # reversed + exact duplicates
    n_hint = -1 if trial % 2 == 0 else n + 5
    want = T.from_edges(e, n_hint)
    c = T.Context(0)
    c.set_graph_edges(e, n_hint)
    rp, col = c.graph_csr()
    assert np.array_equal(rp, want.csc_col_ptr) and np.array_equal(col, want.csc_rows)
    t = T.template_from_parents(CFG_TEMPLATES["cfg2"], 0)
    c.set_template(t)
    a = ctx_for(want, t)
    ta, pa, _ = a.run_coloring(7, per_vertex=True)
    tb, pb, _ = c.run_coloring(7, per_vertex=True)
    assert ta == tb and np.array_equal(pa, pb)


def test_device_from_edges_errors_and_empty():
    c = T.Context(0)
    with pytest.raises(T.ParseError):
        c.set_graph_edges(np.array([[0, 7]], np.int32), 5)
    with pytest.raises(T.ParseError):
        c.set_graph_edges(np.array([[-1, 2]], np.int32))
    c.set_graph_edges(np.zeros((0, 2), np.int32), 4)  # 4 isolated vertices
    rp, col = c.graph_csr()
    assert rp.tolist() == [0, 0, 0, 0, 0] and col.size == 0
    c.set_graph_edges(np.array([[3, 3], [1, 0], [0, 1]], np.int32))
    rp, col = c.graph_csr()
    assert rp.tolist() == [0, 1, 2, 2, 2] and col.tolist() == [1, 0]


def test_device_from_edges_rmat_scale():
    """An R-MAT edge stream of 2^22 edges (hub rows, heavy duplication)."""
    g = T.generate_rmat(T.RmatSpec(16, 64 << 16, .57, .19, .19, .05, 5))
    src = np.repeat(np.arange(g.n, dtype=np.int32), np.diff(g.csc_col_ptr))
    e = np.stack([src, g.csc_rows], 1)
    e = np.concatenate([e, e[::3]])               # duplicates
    c = T.Context(0)
    c.set_graph_edges(np.random.default_rng(0).permutation(e), g.n)
    rp, col = c.graph_csr()
    assert np.array_equal(rp, g.csc_col_ptr) and np.array_equal(col, g.csc_rows)


# ------------------------------------------------------ multi-device context
def test_multi_device_context_spreads_colorings():
    """tcg_create_multi: one context over several devices (here device 0 twice:
    two independent engines, no collective) -- estimate() spreads colorings
    seed+i over them; totals equal the single-device context's bit for bit."""
    g = T.generate_rmat(T.RmatSpec(14, 16 << 14, .45, .15, .15, .25, 2))
    t = T.template_from_parents(CFG_TEMPLATES["cfg3"], 0)
    one = ctx_for(g, t)
    multi = T.Context(devices=[0, 0])
    multi.set_graph(g)
    multi.set_template(t)
    for iters in (1, 2, 5):
        a = one.estimate(3, iters, per_vertex=True)
        b = multi.estimate(3, iters, per_vertex=True)
        assert a[0].tolist() == b[0].tolist()
        assert rel_err([b[1]], [a[1]]) <= 1e-12 and rel_err([b[2]], [a[2]]) <= 1e-12 or iters == 1
        assert_close(b[3], a[3], 1e-12)
    tm, totals = multi.time(7, 4)
    assert totals.tolist() == one.estimate(7, 4)[0].tolist()
