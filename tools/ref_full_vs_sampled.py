"""Validate the sampled CPU-baseline model against a FULL timed coloring.

Runs, on this host, the unmodified reference (oracle/_ref) on the bench graph
(built by the reference's own generate_rmat):
  * ref_time_sampled (the model bench.py's cpu_baseline reports),
  * random_coloring + run_iteration(EngineKind::vectorized) in one call, with
    the per-node NodeStats::seconds (engines.hpp:53-61, 106-132),
  * the K-slice replay bench.py --impl reference uses (RefStepper),
and prints one comparison record (JSON) plus the per-node split.

  python tools/ref_full_vs_sampled.py --config cfg3 [--out profiles/r02_ref_full_vs_sampled.txt]
"""
import argparse
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import oracle as O  # noqa: E402
from bench import CONFIGS  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="cfg3")
ap.add_argument("--out", default=None)
ap.add_argument("--steps", type=int, default=5)
a = ap.parse_args()
spec, parents, _, desc = CONFIGS[a.config]
k = len(parents)
e = np.array(O.parent_array_edges(parents), np.int32).reshape(-1)
cores = O.physical_cores()
t0 = time.perf_counter()
g = O.RefGraph.rmat(*spec)
n, rp, _ = g.csr()
gsec = time.perf_counter() - t0
out = np.zeros(8)
t0 = time.perf_counter()
assert O.ref().ref_time_sampled(g.h, k, e, 0, 1, cores, 1, 32, out) == 0
sample_wall = time.perf_counter() - t0
total, full_s, node_sec = O.ref_run_iteration_stats(g, k, e, 0, 1, cores)
st = O.RefStepper(g, k, e, 0, 1, cores, a.steps)
step_s = [st.run(i) for i in range(a.steps)]
t2, node_stats, extra = st.finish()
plan = O.partition(k, O.parent_array_edges(parents), 0)
rec = {
    "config": a.config, "workload": desc, "n": n, "nnz": int(rp[-1]), "cores": cores,
    "lscpu_physical_cores": cores, "os_cpu_count": os.cpu_count(), "graph_build_s": round(gsec, 1),
    "model_ms": out[0] * 1e3, "model_spmm_ms": out[1] * 1e3, "model_ema_ms": out[2] * 1e3,
    "model_sample_wall_s": round(sample_wall, 1),
    "full_run_iteration_ms": full_s * 1e3, "full_total": total,
    "stepped_ms": sum(step_s) * 1e3, "stepped_total": t2, "stepped_step_s": [round(x, 2) for x in step_s],
    "stepped_spmm_ms": float(node_stats[:, 1].sum() * 1e3), "stepped_ema_ms": float(node_stats[:, 2].sum() * 1e3),
    "model_over_full": out[0] / full_s, "stepped_over_full": sum(step_s) / full_s,
    "totals_identical": total == t2,
}
lines = [json.dumps(rec), "node  size  run_iteration NodeStats::seconds  stepped seconds (spmm, ema)"]
for i in range(len(node_sec)):
    lines.append(f"{i:4d}  {plan.size[i]:4d}  {node_sec[i]:10.3f}  {node_stats[i, 0]:10.3f} "
                 f"({node_stats[i, 1]:.3f}, {node_stats[i, 2]:.3f})")
txt = "\n".join(lines)
print(txt)
if a.out:
    with open(a.out, "w") as f:
        f.write(txt + "\n")
