"""Pin the CPU oracle (oracle/tc_oracle.c) before trusting it.

Checks the C restatement against (a) the golden vectors generated from the
UNMODIFIED reference (tests/golden/, via tests/golden/make_golden.py), (b) the
published KATs quoted in SURVEY.md 8(c), and (c) the compiled reference itself
when oracle/_ref/libtcref.so is present (this container; skipped elsewhere).
"""
import numpy as np
import pytest

import oracle as O
from conftest import CFG_TEMPLATES, parents_to_edges

needs_ref = pytest.mark.skipif(not O.ref_available(), reason="oracle/_ref not built")


def test_mt19937_64_standard_kat():
    # [rand.predef]: default-seeded mt19937_64, 10000th output
    assert O.mt_first(5489, 10000)[-1] == 9981545732273789042


def test_rng_seed1_first_outputs(kats):
    assert O.mt_first(1, 3) == kats["rng1_first3"]


@pytest.mark.parametrize("k,expect", [
    (5, "3 2 0 1 4 4 3 0 3 4 1 3 2 2 0 3 4 0 3 0 3 2 3 2"),
    (7, "2 2 4 5 2 0 6 4 2 0 5 1 2 3 0 6 0 3 5 3 1 4 6 2"),
    (12, "8 6 6 6 0 9 8 9 8 4 8 11 5 11 8 9 1 6 11 8 11 7 8 3"),
    (15, "8 12 0 6 9 9 8 0 8 4 11 8 2 2 5 3 4 0 8 5 8 7 8 12"),
    (17, "9 15 2 15 6 0 14 0 13 4 9 3 16 14 16 4 14 0 0 9 15 9 0 12"),
])
def test_random_coloring_survey_kats(k, expect):
    assert " ".join(map(str, O.random_coloring(24, k, 1))) == expect


def test_random_coloring_golden(kats):
    for key, want in kats["coloring24"].items():
        k, seed = map(int, key.split("_"))
        assert O.random_coloring(24, k, seed).tolist() == want, key
    for k, d in kats["coloring100003_seed7"].items():
        c = O.random_coloring(100003, int(k), 7).astype(np.int64)
        assert int(c.sum()) == d["sum"]
        assert int((c * (np.arange(c.size) % 9973)).sum()) == d["wsum"]


def test_rejection_path_consumes_extra_draws():
    # limit_override forces rejections; result must follow the redraw rule
    n, k, seed = 2000, 7, 3
    limit = (2 ** 64 - 1) // 3
    c = O.random_coloring(n, k, seed, limit)
    words = O.mt_first(seed, 8 * n)
    acc = [w % k for w in words if w < limit][:n]
    assert c.tolist() == acc


def test_combinadic_kats():
    assert O.index_of([0, 1]) == 0 and O.index_of([0, 2]) == 1 and O.index_of([1, 2]) == 2
    assert O.index_of([1]) == 1
    assert O.set_of(3, 2, 2) == [1, 2]
    for k in range(1, 9):
        for h in range(1, k + 1):
            seen = {O.index_of(O.set_of(k, i, h)) for i in range(O.binom(k, h))}
            assert seen == set(range(O.binom(k, h)))


def test_split_table_golden(kats):
    for key, want in kats["splits"].items():
        k, ps, as_ = map(int, key.split("_"))
        st = O.split_table(k, ps, as_)
        for f in ("active_index", "passive_index", "grouped_parent", "grouped_active"):
            assert st[f].tolist() == want[f], (key, f)


def test_split_table_spec_example():
    # test_color_index.cpp:69-84
    st = O.split_table(3, 2, 1)
    assert st["active_index"][:2].tolist() == [0, 1]
    assert st["passive_index"][:2].tolist() == [1, 0]
    assert st["grouped_parent"][:2].tolist() == [0, 1]


def test_plans_and_aut_golden(kats):
    for name, parents in CFG_TEMPLATES.items():
        k = len(parents)
        e = parents_to_edges(parents)
        assert O.automorphisms(k, e) == kats["plans"][f"{name}_root0"]["aut"]
        for root in (0, -1):
            want = kats["plans"][f"{name}_root{root}"]
            p = O.partition(k, e, root)
            assert p.root == want["root"] and p.num_nodes == want["num_nodes"]
            assert list(p.size)[:p.num_nodes] == want["size"]
            assert list(p.active_child)[:p.num_nodes] == want["active"]
            assert list(p.passive_child)[:p.num_nodes] == want["passive"]
            assert list(p.dp_order)[:p.num_nodes] == want["dp_order"]
            assert O.estimate_bytes(p, 1000) == want["estimate_bytes_n1000"]


def test_survey_aut_values():
    # aut = 2 / 8 / 2 / 1 / 2 for cfg1..5
    got = [O.automorphisms(len(p), parents_to_edges(p)) for p in CFG_TEMPLATES.values()]
    assert got == [2, 8, 2, 1, 2]


def test_cfg1_golden(cfg1_golden):
    g = cfg1_golden
    n = 16384
    plan = O.partition(5, parents_to_edges(CFG_TEMPLATES["cfg1"]), 0)
    colors = O.random_coloring(n, 5, 1)
    total, pv, _ = O.run_iteration(n, g["row_ptr"], g["col"], plan, colors)
    assert total == 41315622.0 == float(g["total_seed1"])
    assert np.array_equal(pv, g["per_vertex_seed1"])
    assert pv[:8].tolist() == [2565, 2487, 3192, 3462, 1666, 1240, 1833, 2551]
    r = O.estimate(n, g["row_ptr"], g["col"], 5, parents_to_edges(CFG_TEMPLATES["cfg1"]), 0, 10, 1)
    assert r["rooted_totals"].tolist() == g["totals_seeds1_10"].tolist()
    assert r["estimate"] == float(g["estimate"]) and r["aut"] == 2


def test_small_instances_bit_exact(kats):
    for inst in kats["small_instances"]:
        n, rp, col = O.csr_from_edges(inst["edges"], inst["n"])
        k = inst["k"]
        plan = O.partition(k, parents_to_edges(inst["parents"]), inst["root"])
        colors = O.random_coloring(n, k, inst["seed"])
        total, pv, _ = O.run_iteration(n, rp, col, plan, colors)
        assert total == inst["total"]
        assert pv.tolist() == inst["per_vertex"]


def test_engine_kats():
    # test_engines.cpp:28-41: K3, edge template, coloring [0,1,0]
    n, rp, col = O.csr_from_edges([(0, 1), (1, 2), (2, 0)])
    plan = O.partition(2, [(0, 1)], 0)
    total, pv, _ = O.run_iteration(n, rp, col, plan, np.array([0, 1, 0], np.uint8))
    assert total == 4.0 and pv.tolist() == [1.0, 2.0, 1.0]
    # test_engines.cpp:56-67: K3, 3-path, rainbow -> 6
    plan = O.partition(3, [(0, 1), (1, 2)], -1)
    total, _, _ = O.run_iteration(n, rp, col, plan, np.array([0, 1, 2], np.uint8))
    assert total == 6.0


@needs_ref
def test_oracle_matches_reference_csr_and_rmat():
    rng = np.random.default_rng(3)
    for trial in range(10):
        n = int(rng.integers(1, 300))
        e = rng.integers(0, n, size=(int(rng.integers(0, 3 * n + 1)), 2)).astype(np.int32)
        a = O.csr_from_edges(e, n)
        b = O.RefGraph.from_edges(e, n).csr()
        assert a[0] == b[0] and np.array_equal(a[1], b[1]) and np.array_equal(a[2], b[2])
    a = O.generate_rmat(12, 16 << 12, .45, .15, .15, .25, 9)
    b = O.RefGraph.rmat(12, 16 << 12, .45, .15, .15, .25, 9).csr()
    assert np.array_equal(a[1], b[1]) and np.array_equal(a[2], b[2])


@needs_ref
def test_oracle_matches_reference_random_trees():
    import ctypes as C
    R = O.ref()
    rng = np.random.default_rng(11)
    for trial in range(40):
        k = int(rng.integers(2, 12))
        parents = [-1] + [int(rng.integers(0, v)) for v in range(1, k)]
        e = np.array(parents_to_edges(parents), np.int32).reshape(-1)
        root = int(rng.integers(-1, k))
        sz = np.zeros(2 * k - 1, np.intc); rt = np.zeros_like(sz); ac = np.zeros_like(sz)
        pa = np.zeros_like(sz); dp = np.zeros_like(sz); fr = C.c_int()
        R.ref_plan(k, e, root, sz, rt, ac, pa, dp, C.byref(fr))
        p = O.partition(k, parents_to_edges(parents), root)
        assert list(p.size)[:2 * k - 1] == sz.tolist()
        assert list(p.dp_order)[:2 * k - 1] == dp.tolist()
        assert list(p.active_child)[:2 * k - 1] == ac.tolist()
        assert O.automorphisms(k, parents_to_edges(parents)) == R.ref_automorphisms(k, e)


@needs_ref
@pytest.mark.parametrize("steps", [1, 3, 7, 40])
def test_reference_stepper_is_run_iteration(steps):
    """bench.py --impl reference times ONE full coloring in K slices (ref_driver.cpp
    RefStepper); the replay must be bit-identical to random_coloring + run_iteration
    (engines.hpp:106-132) and execute every unit."""
    g = O.RefGraph.rmat(11, 24 << 11, .45, .15, .15, .25, 3)
    parents = CFG_TEMPLATES["cfg3"]
    e = np.array(parents_to_edges(parents), np.int32).reshape(-1)
    want, _, node_sec = O.ref_run_iteration_stats(g, len(parents), e, 0, 5, 4)
    st = O.RefStepper(g, len(parents), e, 0, 5, 4, steps)
    for i in range(steps):
        st.run(i)
    got, node_stats, extra = st.finish()
    assert got == want
    assert node_stats.shape == (len(node_sec), 3)
    # every internal node ran its SpMM batches and eMA pairs
    assert np.all((node_stats[:, 1] > 0) == (node_stats[:, 2] > 0))
    assert int(extra[1]) > steps


@needs_ref
def test_reference_stepper_refuses_unfinished():
    g = O.RefGraph.rmat(9, 8 << 9, .57, .19, .19, .05, 1)
    e = np.array(parents_to_edges(CFG_TEMPLATES["cfg1"]), np.int32).reshape(-1)
    st = O.RefStepper(g, 5, e, 0, 1, 2, 4)
    st.run(0)
    with pytest.raises(RuntimeError):
        st.finish()
