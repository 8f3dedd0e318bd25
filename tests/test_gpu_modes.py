"""GPU parity of the engine's alternative kernel paths, selected by the
environment variables the engine reads once per process (each case runs in a
child process):

* TCG_RT_VTX=2 -- every non-leaf node through the vertex-per-CTA rooted eMA
  (ema_rtv_blocked / ema_rtv_root), which by default only the wide k=15/17
  nodes take;
* TCG_ROOTED_EMA=0 -- full-table eMA (ema_node / ema_blocked / ema_vtx_*)
  behind the rooted SpMM;
* TCG_ROOTED=0 -- full-table panel SpMM and full-table eMA;
* TCG_PSTREAM=2 -- streamed active-leaf SpMM epilogues (P' never
  materialized) also in contexts that keep their tables, so every node table
  of a streamed node is checked; TCG_PSTREAM=0 -- always a full P';
* TCG_ROOTED_PARTS=1 with TCG_PART_KB=16 -- the rooted SpMM split into
  colour-class parts (P' accumulated across parts);
* TCG_PAIR=0 -- no pair layout (every rooted SpMM over the k-color slot
  layout); TCG_PAIR=2 -- the pair layout for every node whose copies fit;
* TCG_VIRT=0 -- every active-leaf table materialized (no virtual tables);
* TCG_RELABEL=0 -- no degree relabeling / isolated-vertex compaction (the
  caller's vertex ids are the internal rows);
* TCG_DEDUP=0 -- identical sub-templates recomputed (no aliasing);
* TCG_EMA_BLOCKED=0 -- no register-blocked eMA (every non-leaf node through
  the generic rooted node kernels);
* TCG_RTV_PLEAF=0 -- wide nodes over a leaf passive child through
  ema_rtv_blocked instead of the drop-table kernel;
* TCG_RT_WARP=0 -- narrow rooted nodes CTA-per-tile instead of warp-per-tile;
* TCG_ROOTED=0 with TCG_PART_KB=64 -- full-table SpMM in many vertex-range parts;
* TCG_RT_TMA=1 -- the blocked rooted eMA as the persistent kernel with
  TMA-engine (cp.async.bulk) staging of the next tile (ema_rt_blocked_tma;
  measured slower, so not the default);
* TCG_RT_PIPE=1 -- the blocked rooted eMA as the warp-specialized cp.async
  pipeline (ema_rt_blocked_pipe: producer warps, one group queue across
  tiles; opt-in);
* TCG_BATCH=0 -- no batched colorings (every coloring its own DP).

Each child compares per-vertex counts, totals and every internal node table
with the oracle (1e-4 relative, zero patterns exact).
"""
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

CHILD = r"""
import sys
import numpy as np
sys.path.insert(0, {root!r})
sys.path.insert(0, {tests!r})
import oracle as O
import paper_1903_04395_b200 as T
from conftest import CFG_TEMPLATES, parents_to_edges

def check(got, want):
    got, want = np.asarray(got, np.float64), np.asarray(want, np.float64)
    assert got.shape == want.shape
    assert np.array_equal(got == 0, want == 0), "zero pattern differs"
    err = float(np.max(np.abs(got - want) / np.maximum(np.abs(want), 1e-300), initial=0.0))
    assert err <= 1e-4, err

def run(g, parents, root, seed, tables):
    k = len(parents)
    t = T.template_from_parents(parents, root)
    c = T.Context(0, 0, tables)
    c.set_graph(g)
    c.set_template(t)
    total, pv, _ = c.run_coloring(seed, per_vertex=True)
    plan = O.partition(k, parents_to_edges(parents), root)
    ototal, opv, tabs = O.run_iteration(g.n, g.csc_col_ptr, g.csc_rows, plan, O.random_coloring(g.n, k, seed),
                                        want_tables=tables)
    check(pv, opv)
    check([total], [ototal])
    if tables:
        for nid, want in tabs.items():
            check(c.node_table(nid, 0), want)
    # estimate() (batched on the device for small graphs unless TCG_BATCH=0):
    # every coloring's total equals its own run_coloring, bit for bit
    totals, est, se, pve = c.estimate(seed, 3, per_vertex=True)
    singles = [c.run_coloring(seed + i)[0] for i in range(3)]
    assert list(totals) == singles, (list(totals), singles)

rng = np.random.default_rng(7)
for case in range(5):
    n, k = int(rng.integers(50, 2000)), int(rng.integers(7, 12))
    e = rng.integers(0, n, size=(int(rng.integers(2, 30) * n / 2), 2))
    g = T.from_edges(e, n)
    parents = [-1] + [int(rng.integers(0, v)) for v in range(1, k)]
    run(g, parents, int(rng.integers(0, k)), case + 1, True)
g = T.generate_rmat(T.RmatSpec(9, 48 << 9, .45, .15, .15, .25, 7))
for name in ("cfg3", "cfg4", "cfg5"):
    run(g, CFG_TEMPLATES[name], 0, 2, name == "cfg3")
print("OK")
"""


@pytest.mark.parametrize("env", [{"TCG_RT_VTX": "2"}, {"TCG_ROOTED_EMA": "0"}, {"TCG_ROOTED": "0"},
                                 {"TCG_PSTREAM": "2"}, {"TCG_PSTREAM": "0"}, {"TCG_ROOTED_PARTS": "1", "TCG_PART_KB": "16"},
                                 {"TCG_PAIR": "0"}, {"TCG_PAIR": "2"}, {"TCG_VIRT": "0"}, {"TCG_RELABEL": "0"},
                                 {"TCG_DEDUP": "0"}, {"TCG_EMA_BLOCKED": "0"}, {"TCG_RTV_PLEAF": "0"},
                                 {"TCG_RT_WARP": "0"}, {"TCG_ROOTED": "0", "TCG_PART_KB": "64"}, {"TCG_RT_TMA": "1"},
                                 {"TCG_BATCH": "0"}, {"TCG_RT_PIPE": "1"}],
                         ids=["rt_vtx_all", "full_table_ema", "full_table_spmm", "pstream_all", "pstream_off",
                              "rooted_parts", "pair_off", "pair_all", "virt_off", "relabel_off", "dedup_off",
                              "blocked_off", "pleaf_off", "rt_warp_off", "full_table_parts", "rt_tma_on",
                              "batch_off", "rt_pipe_on"])
def test_kernel_path_parity(env):
    code = CHILD.format(root=ROOT, tests=os.path.join(ROOT, "tests"))
    r = subprocess.run([sys.executable, "-c", code], env={**os.environ, **env}, capture_output=True, text=True,
                       timeout=900)
    assert r.returncode == 0 and r.stdout.strip().endswith("OK"), r.stdout[-2000:] + r.stderr[-4000:]
