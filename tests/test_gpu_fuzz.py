"""Randomized end-to-end parity of every public path on small inputs: graphs
with isolated vertices, empty and dense rows, k = 1..10 random trees and roots;
run_coloring (per-vertex + total) against the oracle, estimate() (batched on
the device for small graphs) equal to the single colorings bit for bit, the
device CSR build (tcg_set_graph_edges) equal to the host CSR, and the
multi-device context equal to one device."""
import numpy as np
import pytest

import oracle as O
import paper_1903_04395_b200 as T
from conftest import parents_to_edges

pytestmark = pytest.mark.gpu


def _close(got, want, rel=1e-4):
    got, want = np.asarray(got, np.float64), np.asarray(want, np.float64)
    assert np.array_equal(got == 0, want == 0), "zero pattern differs"
    err = float(np.max(np.abs(got - want) / np.maximum(np.abs(want), 1e-300), initial=0.0))
    assert err <= rel, err


@pytest.mark.parametrize("case", range(24))
def test_random_end_to_end(case):
    rng = np.random.default_rng(5000 + case)
    n = int(rng.integers(1, 2500))
    kind = case % 4
    if kind == 0:    # sparse with many isolated vertices
        m = int(rng.integers(0, n))
        e = rng.integers(0, n, size=(m, 2))
    elif kind == 1:  # dense-ish
        e = rng.integers(0, n, size=(int(rng.integers(1, 20)) * n, 2))
    elif kind == 2:  # a hub plus noise
        e = np.concatenate([np.stack([np.zeros(n, np.int64), np.arange(n)], 1),
                            rng.integers(0, n, size=(2 * n, 2))])
    else:            # R-MAT-like skew via squared uniforms
        m = 8 * n
        e = (np.stack([rng.random(m) ** 2, rng.random(m) ** 2], 1) * n).astype(np.int64)
    e = e.astype(np.int32)
    g = T.from_edges(e, n)
    k = int(rng.integers(1, 11))
    parents = [-1] + [int(rng.integers(0, v)) for v in range(1, k)]
    root = int(rng.integers(0, k))
    t = T.template_from_parents(parents, root)
    c = T.Context(0)
    c.set_graph(g)
    c.set_template(t)
    seed = int(rng.integers(1, 1 << 20))
    total, pv, _ = c.run_coloring(seed, per_vertex=True)
    plan = O.partition(k, parents_to_edges(parents), root)
    ototal, opv, _ = O.run_iteration(g.n, g.csc_col_ptr, g.csc_rows, plan, O.random_coloring(g.n, k, seed))
    _close(pv, opv)
    _close([total], [ototal])
    iters = int(rng.integers(1, 8))
    totals, est, se, pve = c.estimate(seed, iters, per_vertex=True)
    singles = [c.run_coloring(seed + i)[0] for i in range(iters)]
    assert list(totals) == singles
    # the device-built CSR and the multi-device context give the same numbers
    d = T.Context(devices=[0, 0])
    d.set_graph_edges(e, n)
    rp, col = d.graph_csr()
    assert np.array_equal(rp, g.csc_col_ptr) and np.array_equal(col, g.csc_rows)
    d.set_template(t)
    t2 = d.estimate(seed, iters, per_vertex=True)
    assert list(t2[0]) == singles
    _close(t2[3], pve, 1e-12)
