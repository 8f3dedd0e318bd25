"""CPU tests of the product's host side (no GPU): the C ABI library loads and
exports every declared symbol, and the C++ host subsystems (CSR build, R-MAT
input generator, template validation/partition, |Aut|, combinadic split
tables, estimate_bytes) agree with the pinned oracle bit for bit."""
import ctypes as C

import numpy as np
import pytest

import oracle as O
import paper_1903_04395_b200 as T
from paper_1903_04395_b200 import _native as N
from conftest import CFG_TEMPLATES, parents_to_edges


def test_library_exports_every_header_symbol():
    syms = N.header_symbols()
    assert len(syms) >= 30
    missing = [s for s in syms if not hasattr(N.lib, s)]
    assert not missing, missing


def test_version_string_names_sm100a():
    assert b"sm_100a" in N.lib.tcg_version()


def _csr_eq(g, ref):
    n, rp, col = ref
    return g.n == n and np.array_equal(g.csc_col_ptr, rp) and np.array_equal(g.csc_rows, col)


def test_from_edges_matches_oracle_random():
    rng = np.random.default_rng(1)
    for trial in range(30):
        n = int(rng.integers(1, 500))
        m = int(rng.integers(0, 4 * n))
        e = rng.integers(0, n, size=(m, 2)).astype(np.int32)
        hint = n if trial % 2 else -1
        if m == 0 and hint < 0:
            continue
        assert _csr_eq(T.from_edges(e, hint), O.csr_from_edges(e, hint)), trial


def test_from_edges_spec_examples():
    # test_graph.cpp:48-64: K3, single edge, path; self-loops and duplicates dropped
    g = T.from_edges([(0, 1), (1, 2), (2, 0)])
    assert g.csc_col_ptr.tolist() == [0, 2, 4, 6] and g.csc_rows.tolist() == [1, 2, 0, 2, 0, 1]
    g = T.from_edges([(0, 1), (1, 0), (1, 1), (0, 1)])
    assert g.m == 1 and g.csc_rows.tolist() == [1, 0]
    g = T.from_edges([(0, 1)], 5)
    assert g.n == 5 and g.degree(4) == 0


def test_from_edges_rejects_out_of_range():
    with pytest.raises(T.ParseError):
        T.from_edges([(0, 7)], 5)
    with pytest.raises(T.ParseError):
        T.from_edges([(-1, 2)])


def test_graph_from_csr_validates():
    g = T.Graph.from_csr(3, [0, 2, 4, 6], [1, 2, 0, 2, 0, 1])
    assert g.m == 3
    with pytest.raises(T.ParseError):
        T.Graph.from_csr(2, [0, 1, 1], [1])          # not symmetric
    with pytest.raises(T.ParseError):
        T.Graph.from_csr(2, [0, 1, 2], [0, 1])       # self loops
    with pytest.raises(T.ParseError):
        T.Graph.from_csr(3, [0, 2, 3, 4], [2, 1, 0, 0])  # unsorted row


@pytest.mark.parametrize("scale,ef,probs,seed", [
    (10, 16, (.57, .19, .19, .05), 1), (12, 8, (.45, .15, .15, .25), 3), (7, 100, (.25, .25, .25, .25), 9)])
def test_rmat_matches_oracle(scale, ef, probs, seed):
    g = T.generate_rmat(T.RmatSpec(scale, ef << scale, *probs, seed))
    assert _csr_eq(g, O.generate_rmat(scale, ef << scale, *probs, seed))


def test_rmat_spec_validation():
    # synthgen.hpp:40-46 throws std::invalid_argument (not parse_error)
    for spec in (T.RmatSpec(0, 10, .25, .25, .25, .25, 1), T.RmatSpec(5, 10, .5, .25, .25, .25, 1)):
        with pytest.raises(T.InvalidArgument) as ei:
            T.generate_rmat(spec)
        assert not isinstance(ei.value, T.ParseError)


def test_template_validation():
    with pytest.raises(T.ParseError):
        T.make_template([(0, 1), (1, 2), (2, 0)])    # cycle: 3 edges for 3 vertices
    with pytest.raises(T.ParseError):
        T.make_template([(0, 1), (2, 3), (3, 4)])    # wrong edge count / disconnected
    with pytest.raises(T.ParseError):
        T.make_template([(0, 0)])
    with pytest.raises(T.ParseError):
        T.make_template([(0, 1)], 5)
    # default root = max degree, smallest id (templates.hpp:67-74)
    assert T.make_template([(0, 1), (1, 2), (1, 3)]).root == 1
    assert T.template_from_parents(CFG_TEMPLATES["cfg2"], -1).root == 1  # SURVEY finding 9


def test_partition_matches_oracle_and_golden(kats):
    for name, parents in CFG_TEMPLATES.items():
        for root in (0, -1):
            want = kats["plans"][f"{name}_root{root}"]
            t = T.template_from_parents(parents, root)
            p = T.partition(t)
            assert p.root == want["root"]
            assert [nd.size for nd in p.nodes] == want["size"]
            assert [nd.active_child for nd in p.nodes] == want["active"]
            assert [nd.passive_child for nd in p.nodes] == want["passive"]
            assert p.dp_order == want["dp_order"]
            assert T.automorphism_count(t) == want["aut"]
            assert T.estimate_bytes(p, 1000) == want["estimate_bytes_n1000"]


def test_partition_and_aut_random_trees():
    rng = np.random.default_rng(5)
    for trial in range(200):
        k = int(rng.integers(1, 21))
        parents = [-1] + [int(rng.integers(0, v)) for v in range(1, k)]
        e = parents_to_edges(parents)
        if k == 1:
            continue
        root = int(rng.integers(-1, k))
        op = O.partition(k, e, root)
        t = T.make_template(e, root)
        p = T.partition(t)
        assert p.dp_order == list(op.dp_order)[:op.num_nodes]
        assert [nd.size for nd in p.nodes] == list(op.size)[:op.num_nodes]
        assert [nd.root for nd in p.nodes] == list(op.node_root)[:op.num_nodes]
        assert T.automorphism_count(t) == O.automorphisms(k, e)


def test_aut_brute_force_small():
    from itertools import permutations
    rng = np.random.default_rng(8)
    for trial in range(30):
        k = int(rng.integers(2, 8))
        parents = [-1] + [int(rng.integers(0, v)) for v in range(1, k)]
        e = parents_to_edges(parents)
        es = {frozenset(x) for x in e}
        brute = sum(all(frozenset((p[u], p[v])) in es for u, v in e) for p in permutations(range(k)))
        assert T.automorphism_count(T.make_template(e, 0)) == brute


def test_split_tables_match_oracle():
    for k in range(2, 13):
        ix = T.ColorIndexer(k)
        for ps in range(2, k + 1):
            for as_ in range(1, ps):
                if ix.num_sets(ps) * ix.binom(ps, as_) > 200000:
                    continue
                st = T.build_split_table(ps, as_, ix)
                o = O.split_table(k, ps, as_)
                assert np.array_equal(st.active_index, o["active_index"])
                assert np.array_equal(st.passive_index, o["passive_index"])
                assert np.array_equal(st.grouped_parent, o["grouped_parent"])
                assert np.array_equal(st.grouped_active, o["grouped_active"])


def test_split_table_rejects_empty_child():
    ix = T.ColorIndexer(3)
    with pytest.raises(T.InvalidArgument):
        T.build_split_table(2, 2, ix)
    with pytest.raises(T.InvalidArgument):
        T.build_split_table(2, 0, ix)


def test_color_indexer():
    ix = T.ColorIndexer(3)
    assert ix.index_of([0, 1]) == 0 and ix.index_of([0, 2]) == 1 and ix.index_of([1, 2]) == 2
    assert ix.set_of(2, 2) == [1, 2]
    with pytest.raises(T.InvalidArgument):
        ix.index_of([1, 1])
    with pytest.raises(T.InvalidArgument):
        ix.set_of(3, 2)
    with pytest.raises(T.InvalidArgument):
        T.ColorIndexer(21)
    assert T.ColorIndexer(20).binom(20, 10) == 184756
    for k in range(1, 11):
        ix = T.ColorIndexer(k)
        for h in range(1, k + 1):
            for i in range(ix.num_sets(h)):
                assert ix.index_of(ix.set_of(i, h)) == i


def test_colorful_probability():
    import math
    for k in range(1, 21):
        assert T.colorful_probability(k) == O.colorful_probability(k)
        assert abs(T.colorful_probability(k) - math.factorial(k) / k ** k) < 1e-12


def test_engine_requires_gpu_or_fails_loudly():
    """Without a usable B200 the device engine refuses with a CUDA/EINVAL
    status -- there is no CPU fallback."""
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    with pytest.raises((T.CudaError, T.InvalidArgument)):
        T.Context(0)


def test_non_b200_engine_kinds_refused():
    g = T.from_edges([(0, 1)])
    with pytest.raises(T.InvalidArgument):
        T.estimate(g, T.make_template([(0, 1)], 0), T.EngineKind.vectorized, 1, 1)


def _rooted_layout(k, s):
    info = np.zeros(4, np.int32)
    N.check(N.lib.tcg_rooted_layout(k, s, info.ctypes.data, None, None))
    zw, groups, full, store = (int(x) for x in info)
    perm = np.zeros(full, np.int32)
    slot_col = np.zeros(k * groups * zw, np.int32)
    N.check(N.lib.tcg_rooted_layout(k, s, info.ctypes.data, perm.ctypes.data, slot_col.ctypes.data))
    return zw, groups, store, perm, slot_col.reshape(k, groups, zw)


@pytest.mark.parametrize("k,s", [(5, 2), (7, 3), (12, 2), (12, 3), (12, 4), (12, 8), (15, 5), (17, 4), (17, 7)])
def test_rooted_layout_partition(k, s):
    """Rooted-color compression layout (csrc/host.cpp build_rooted_layout):
    every color set lands in exactly one group, every group holds at most zw
    sets of each color, each color's slots of a group list exactly the group's
    sets containing it, and P' storage columns are a group-major 8-aligned
    bijection of the combinadic columns."""
    from math import comb
    zw, groups, store, perm, slot_col = _rooted_layout(k, s)
    full = comb(k, s)
    lb = -(-comb(k - 1, s - 1) // zw)
    assert lb <= groups <= lb + lb // 16 + 2
    assert len(set(perm.tolist())) == full and perm.min() >= 0 and perm.max() < store
    ci = T.ColorIndexer(k)
    members = {}
    for c in range(k):
        seen = set()
        for g in range(groups):
            cols = [int(x) for x in slot_col[c, g] if x >= 0]
            assert len(cols) <= zw
            for x in cols:
                assert c in ci.set_of(x, s)
                assert x not in seen
                seen.add(x)
                members.setdefault(x, set()).add(g)
        # every set containing c has exactly one slot of color c
        assert seen == {x for x in range(full) if c in ci.set_of(x, s)}
    # each set belongs to one group for all its colors
    assert all(len(gs) == 1 for gs in members.values()) and len(members) == full
    # storage columns: group-major, groups 8-aligned
    grp = {x: next(iter(members[x])) for x in range(full)}
    order = sorted(range(full), key=lambda x: perm[x])
    assert [grp[x] for x in order] == sorted(grp[x] for x in order)
    assert store % 8 == 0


@pytest.mark.parametrize("k,s,a,V", [(16, 11, 7, 2), (16, 7, 3, 8), (14, 10, 7, 4), (16, 11, 7, 1),
                                     (12, 8, 4, 8), (9, 5, 2, 4), (19, 9, 4, 2)])
def test_rtv_task_layout(k, s, a, V):
    """Work layout of the vertex-per-CTA blocked eMA (csrc/engine.cu build_rtv_tasks; the (k, s, a)
    here are the rooted problems of cfg5 nodes 1 / 2 and cfg4 node 1, and smaller ones): the library
    checks that every (group, block) of the split enumeration sits exactly once where the kernel
    reads it; here also the counts (groups = the (S2, s1) classes over the k - 6 high colours,
    block steps padded per task) and that the bank-aware order is no worse than 1.5x
    conflict-free."""
    from math import comb
    info = np.zeros(6, np.int64)
    N.check(N.lib.tcg_rtv_task_layout(k, s, a, V, info.ctypes.data))
    tasks, groups, steps, runs, wave, ideal = (int(x) for x in info)
    gpt = 32 // V
    assert groups == sum(comb(k - 6, t) for t in range(k - 5) if 0 <= s - t <= 6)
    assert -(-groups // gpt) <= tasks <= -(-groups // gpt) + 7     # (one partial task per shape at most)
    assert steps >= 1 and runs >= 1
    assert ideal <= wave <= 1.5 * ideal


def test_rtv_task_layout_rejects_bad_arguments():
    info = np.zeros(6, np.int64)
    for bad in ((16, 11, 7, 3), (5, 3, 1, 2), (16, 1, 1, 2), (16, 11, 11, 2), (21, 11, 7, 2)):
        with pytest.raises(T.InvalidArgument):
            N.check(N.lib.tcg_rtv_task_layout(*bad, info.ctypes.data))
