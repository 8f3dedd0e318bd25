"""Generate tests/golden/ fixtures by running the UNMODIFIED reference.

Run here (where /root/reference exists):  python tests/golden/make_golden.py [--big]
Uses oracle/_ref/libtcref.so (ref_driver.cpp over /root/reference/proj/include,
built with the reference's own flags).  The fixtures travel with the repo; the
GPU box never reads /root/reference.

Outputs
  kats.json        colorings / MT / split / plan / aut / estimate_bytes KATs, small-instance totals
  cfg1.npz         cfg1 graph CSR + per-vertex root counts seed 1 + totals seeds 1..10
  cfg2.npz         cfg2 totals seeds 1..2 + per-vertex root counts (seed 1) on a fixed vertex sample  [--big]
  cfg3.npz         cfg3 total seed 1 + per-vertex sample                                             [--big]
  cfg3_full.npz    cfg3 seeds 1..3: totals + the WHOLE per-vertex root vector (float32)              [--r2]
  cfg4t.npz        cfg4 template (k=15) on R-MAT scale 18 ef32 (.57,.19,.19,.05), seeds 1..2, full
                   per-vertex (fp64): 261K-vertex graph with hub rows far above 1,024 neighbours    [--r2]
  cfg5t.npz        cfg5 template (k=17) on R-MAT scale 16 ef100 (.45,.15,.15,.25), seed 1, full
                   per-vertex (fp64)                                                                 [--r2]
cfg2 seeds 1..10 are not stored: tests/test_parity_scale.py runs oracle/_ref on the GPU box's host
(7-8 s per coloring) and compares the whole per-vertex vector.
"""
from __future__ import annotations

import argparse
import ctypes as C
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
import oracle as O  # noqa: E402

OUT = os.path.dirname(os.path.abspath(__file__))

CFG_TEMPLATES = {
    "cfg1": [-1, 0, 1, 1, 3],
    "cfg2": [-1, 0, 0, 1, 1, 2, 2],
    "cfg3": [-1, 0, 1, 2, 0, 4, 4, 6, 0, 8, 9, 9],
    "cfg4": [-1, 0, 1, 2, 3, 0, 5, 6, 0, 8, 8, 10, 10, 12, 13],
    "cfg5": [-1, 0, 1, 2, 3, 4, 0, 6, 7, 8, 0, 10, 11, 11, 0, 14, 15],
}
CFG_GRAPHS = {
    "cfg2": (20, 16 << 20, .57, .19, .19, .05, 1),
    "cfg3": (20, 100 << 20, .45, .15, .15, .25, 1),
    # scaled-down graphs of the cfg4 / cfg5 shape: the full ones need 432 / 276 GB of fp64 tables
    "cfg4t": (18, 32 << 18, .57, .19, .19, .05, 1),
    "cfg5t": (16, 100 << 16, .45, .15, .15, .25, 1),
}
R2_TEMPLATES = {"cfg3_full": "cfg3", "cfg4t": "cfg4", "cfg5t": "cfg5"}


def cfg1_edges(n=16384, seed=1):
    """Rng(1); 8n draws of (below(n), below(n)), keep u != v."""
    g = C.create_string_buffer(312 * 8 + 16)
    O.lib().orc_mt_seed(g, seed)
    nxt = O.lib().orc_mt_next

    def below(b):
        lim = (2 ** 64 - 1) // b * b
        while True:
            x = nxt(g)
            if x < lim:
                return x % b
    e = []
    for _ in range(8 * n):
        u, v = below(n), below(n)
        if u != v:
            e.append((u, v))
    return np.array(e, np.int32)


def eflat(parents):
    return np.array(O.parent_array_edges(parents), np.int32).reshape(-1)


def ref_run(g, k, edges, root, colors, workers=8):
    R = O.ref()
    n, _, _ = g.csr()
    total = C.c_double()
    pv = np.zeros(max(n, 1))
    rc = R.ref_run_iteration(g.h, k, edges, root, colors, workers, 16, C.byref(total),
                             pv.ctypes.data, None)
    assert rc == 0
    return total.value, pv[:n]


def ref_estimate(g, k, edges, root, iters, seed, workers=8):
    R = O.ref()
    totals = np.zeros(iters)
    est, se, aut, secs = C.c_double(), C.c_double(), C.c_uint64(), C.c_double()
    assert R.ref_estimate(g.h, k, edges, root, iters, seed, workers, totals, C.byref(est),
                          C.byref(se), C.byref(aut), C.byref(secs)) == 0
    return totals, est.value, se.value, aut.value


def kats():
    R = O.ref()
    out = {}
    mt = np.zeros(3, np.uint64)
    R.ref_mt_first(1, 3, mt)
    out["rng1_first3"] = [int(x) for x in mt]
    col = {}
    for k in (1, 2, 3, 5, 7, 12, 15, 17, 20):
        for seed in (1, 2, 12345):
            c = np.zeros(24, np.uint8)
            R.ref_random_coloring(24, k, seed, c)
            col[f"{k}_{seed}"] = [int(x) for x in c]
    out["coloring24"] = col
    # longer colorings: hashes of n=100003 (k=5,7,12,17)
    big = {}
    for k in (5, 7, 12, 17):
        c = np.zeros(100003, np.uint8)
        R.ref_random_coloring(100003, k, 7, c)
        big[str(k)] = {"sum": int(c.astype(np.int64).sum()),
                       "wsum": int((c.astype(np.int64) * (np.arange(c.size) % 9973)).sum()),
                       "head": [int(x) for x in c[:16]], "tail": [int(x) for x in c[-16:]]}
    out["coloring100003_seed7"] = big
    # plans, aut, estimate_bytes for the five BASELINE templates (root 0) + default root
    plans = {}
    for name, parents in CFG_TEMPLATES.items():
        k = len(parents)
        e = eflat(parents)
        for root in (0, -1):
            sz = np.zeros(2 * k - 1, np.intc); rt = np.zeros_like(sz); ac = np.zeros_like(sz)
            pa = np.zeros_like(sz); dp = np.zeros_like(sz); fr = C.c_int()
            nn = R.ref_plan(k, e, root, sz, rt, ac, pa, dp, C.byref(fr))
            plans[f"{name}_root{root}"] = dict(
                k=k, root=fr.value, num_nodes=nn, size=sz.tolist(), node_root=rt.tolist(),
                active=ac.tolist(), passive=pa.tolist(), dp_order=dp.tolist(),
                aut=int(R.ref_automorphisms(k, e)),
                estimate_bytes_n1000=int(R.ref_estimate_bytes(k, e, root, 1000)))
    out["plans"] = plans
    # split tables (full, small shapes)
    splits = {}
    for k, ps, as_ in ((3, 2, 1), (5, 3, 1), (5, 4, 2), (7, 4, 3), (12, 5, 1), (12, 9, 5), (6, 6, 3)):
        cs, pairs = O.binom(k, ps), O.binom(ps, as_)
        cp, partners = O.binom(k, ps - as_), O.binom(k - (ps - as_), as_)
        ai = np.zeros(cs * pairs, np.int32); pi = np.zeros_like(ai)
        gp = np.zeros(cp * partners, np.int32); ga = np.zeros_like(gp)
        assert R.ref_split_table(k, ps, as_, ai, pi, gp, ga) == 0
        splits[f"{k}_{ps}_{as_}"] = dict(active_index=ai.tolist(), passive_index=pi.tolist(),
                                        grouped_parent=gp.tolist(), grouped_active=ga.tolist())
    out["splits"] = splits
    # engine KATs (test_engines.cpp:28-67) and small random instances with per-vertex outputs
    small = []
    rng = np.random.default_rng(20261020)
    for trial in range(24):
        n = int(rng.integers(5, 200))
        m = int(rng.integers(1, 4 * n))
        edges = rng.integers(0, n, size=(m, 2)).astype(np.int32)
        k = int(rng.integers(2, 9))
        parents = [-1] + [int(rng.integers(0, v)) for v in range(1, k)]
        root = int(rng.integers(-1, k))
        g = O.RefGraph.from_edges(edges, n)
        nn, rp, cl = g.csr()
        colors = np.zeros(n, np.uint8)
        seed = 100 + trial
        R.ref_random_coloring(n, k, seed, colors)
        e = eflat(parents)
        total, pv = ref_run(g, k, e, root, colors)
        small.append(dict(n=n, edges=edges.tolist(), k=k, parents=parents, root=root, seed=seed,
                          total=total, per_vertex=pv.tolist()))
    out["small_instances"] = small
    return out


def cfg1():
    edges = cfg1_edges()
    g = O.RefGraph.from_edges(edges, 16384)
    n, rp, cl = g.csr()
    k, e = 5, eflat(CFG_TEMPLATES["cfg1"])
    colors = np.zeros(n, np.uint8)
    O.ref().ref_random_coloring(n, k, 1, colors)
    total, pv = ref_run(g, k, e, 0, colors)
    totals, est, se, aut = ref_estimate(g, k, e, 0, 10, 1)
    np.savez_compressed(os.path.join(OUT, "cfg1.npz"), row_ptr=rp, col=cl, per_vertex_seed1=pv,
                        total_seed1=total, totals_seeds1_10=totals, estimate=est, stderr=se, aut=aut)
    print("cfg1", total, est, se, aut)


def vertex_sample(n, rp, count=20000):
    deg = np.diff(rp)
    hubs = np.argsort(-deg, kind="stable")[:256]
    rs = np.random.default_rng(7).choice(n, size=min(count, n), replace=False)
    return np.unique(np.concatenate([hubs, rs, np.arange(min(64, n))])).astype(np.int64)


def big_cfg(name, seeds):
    t0 = time.time()
    g = O.RefGraph.rmat(*CFG_GRAPHS[name])
    n, rp, cl = g.csr()
    print(name, "graph", n, rp[-1], f"{time.time() - t0:.1f}s", flush=True)
    parents = CFG_TEMPLATES[name]
    k, e = len(parents), eflat(parents)
    totals, samples = [], {}
    idx = vertex_sample(n, rp)
    for s in seeds:
        colors = np.zeros(n, np.uint8)
        O.ref().ref_random_coloring(n, k, s, colors)
        t0 = time.time()
        total, pv = ref_run(g, k, e, 0, colors, workers=os.cpu_count())
        print(name, "seed", s, repr(total), f"{time.time() - t0:.1f}s", flush=True)
        totals.append(total)
        samples[f"pv_seed{s}"] = pv[idx]
        if s == seeds[0]:
            samples["pv_sum_seed%d" % s] = pv.sum()
            samples["pv_max_seed%d" % s] = pv.max()
            samples["zero_rows_seed%d" % s] = np.flatnonzero(pv == 0).size
    np.savez_compressed(os.path.join(OUT, f"{name}.npz"), seeds=np.array(seeds), totals=np.array(totals),
                        sample_idx=idx, nnz=rp[-1], n=n, row_ptr_checksum=int(rp.sum() % (1 << 61)),
                        col_checksum=int((cl.astype(np.int64) * (np.arange(cl.size) % 1000003)).sum() % (1 << 61)),
                        **samples)


def full_cfg(name, seeds, dtype):
    """Whole per-vertex root vectors of the reference for several seeds (round-2 fixtures)."""
    gname = "cfg3" if name == "cfg3_full" else name
    t0 = time.time()
    g = O.RefGraph.rmat(*CFG_GRAPHS[gname])
    n, rp, cl = g.csr()
    print(name, "graph", n, rp[-1], "maxdeg", int(np.diff(rp).max()), f"{time.time() - t0:.1f}s",
          flush=True)
    parents = CFG_TEMPLATES[R2_TEMPLATES[name]]
    k, e = len(parents), eflat(parents)
    out = {}
    totals, secs = [], []
    for s in seeds:
        colors = np.zeros(n, np.uint8)
        O.ref().ref_random_coloring(n, k, s, colors)
        t0 = time.time()
        total, pv = ref_run(g, k, e, 0, colors, workers=os.cpu_count())
        secs.append(time.time() - t0)
        print(name, "seed", s, repr(total), f"{secs[-1]:.1f}s", flush=True)
        totals.append(total)
        out[f"pv_seed{s}"] = pv.astype(dtype)
        out[f"pv_sum_seed{s}"] = pv.sum()
    np.savez_compressed(os.path.join(OUT, f"{name}.npz"), seeds=np.array(seeds),
                        totals=np.array(totals), ref_seconds=np.array(secs), n=n, nnz=rp[-1],
                        graph=np.array(CFG_GRAPHS[gname][:6]), graph_seed=CFG_GRAPHS[gname][6],
                        parents=np.array(parents), pv_dtype=np.dtype(dtype).name,
                        row_ptr_checksum=int(rp.sum() % (1 << 61)),
                        col_checksum=int((cl.astype(np.int64) * (np.arange(cl.size) % 1000003)).sum()
                                         % (1 << 61)), **out)


if __name__ == "__main__":
    ap = argparse.ArgumentParser()
    ap.add_argument("--big", action="store_true", help="also cfg2 (and cfg3 with --cfg3)")
    ap.add_argument("--cfg3", action="store_true")
    ap.add_argument("--r2", nargs="*", default=None,
                    help="round-2 full per-vertex fixtures: cfg4t cfg5t cfg3_full (default all)")
    a = ap.parse_args()
    if a.r2 is not None:
        for name in a.r2 or ["cfg4t", "cfg5t", "cfg3_full"]:
            if name == "cfg3_full":
                full_cfg(name, [1, 2, 3], np.float32)
            elif name == "cfg4t":
                full_cfg(name, [1, 2], np.float64)
            else:
                full_cfg(name, [1], np.float64)
        sys.exit(0)
    with open(os.path.join(OUT, "kats.json"), "w") as f:
        json.dump(kats(), f)
    cfg1()
    if a.big:
        big_cfg("cfg2", [1, 2])
    if a.cfg3:
        big_cfg("cfg3", [1])
