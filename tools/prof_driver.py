"""Short profiling driver: W warm-up colorings then C profiled colorings of a
bench config (used under ncu; see profiles/README.md)."""
import argparse
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
import paper_1903_04395_b200 as T  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="cfg3")
ap.add_argument("--warmup", type=int, default=1)
ap.add_argument("--colorings", type=int, default=1)
ap.add_argument("--stats", action="store_true", help="print per-node device times")
ap.add_argument("--scale", type=int, default=0, help="override the R-MAT scale (edge factor kept)")
a = ap.parse_args()
spec, parents, _, _ = bench.CONFIGS[a.config]
if a.scale:
    spec = (a.scale, (spec[1] >> spec[0]) << a.scale) + tuple(spec[2:])
g = T.generate_rmat(T.RmatSpec(*spec))
t = T.template_from_parents(parents, 0)
ctx = T.Context(0)
ctx.set_graph(g)
ctx.set_template(t)
if a.warmup:
    ctx.time(1, a.warmup)
tm, totals = ctx.time(100, a.colorings, per_kernel=False)
print(f"{a.config}: {tm.total_ms / a.colorings:.3f} ms/coloring, launches {tm.launches}")
if a.stats:
    plan, _ = ctx.plan()
    total, _, st = ctx.run_coloring(7, stats=True)
    for nd in plan.nodes:
        if nd.is_leaf():
            continue
        s = st[nd.id]
        print(f"node {nd.id:2d} size {nd.size:2d} a={plan.node(nd.active_child).size:2d} "
              f"p={plan.node(nd.passive_child).size:2d}: spmm {s.spmm_seconds * 1e3:8.3f} ms "
              f"ema {s.ema_seconds * 1e3:8.3f} ms  ema {s.ema_bytes / max(s.ema_seconds, 1e-12) / 1e9:7.1f} GB/s "
              f"{s.ema_flops / max(s.ema_seconds, 1e-12) / 1e12:6.2f} TFLOP/s")
