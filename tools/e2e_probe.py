"""Time the e2e pieces of bench.py's e2e step (set_graph_csr from pinned host
buffers, estimate) to see where the host/driver time goes."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import bench  # noqa: E402
import paper_1903_04395_b200 as T  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "cfg3"
spec, parents, ncol, _ = bench.CONFIGS[cfg]
g = T.generate_rmat(T.RmatSpec(*spec))
rp_t = torch.empty(g.csc_col_ptr.shape[0], dtype=torch.int64, pin_memory=True)
cl_t = torch.empty(g.csc_rows.shape[0], dtype=torch.int32, pin_memory=True)
rp, cl = rp_t.numpy(), cl_t.numpy()
rp[:] = g.csc_col_ptr
cl[:] = g.csc_rows
t = T.template_from_parents(parents, 0)
ctx = T.Context(0)
ctx.set_template(t)
ctx.set_graph_csr(g.n, rp, cl)
ctx.estimate(1, 1)
for i in range(4):
    t0 = time.perf_counter()
    ctx.set_graph_csr(g.n, rp, cl)
    t1 = time.perf_counter()
    tot, est, se, pv = ctx.estimate(1 + i * ncol, ncol, per_vertex=True)
    t2 = time.perf_counter()
    print(f"{cfg} step {i}: set_graph_csr {1e3 * (t1 - t0):.1f} ms, estimate({ncol}) {1e3 * (t2 - t1):.1f} ms")
# device time of the same colorings (CUDA events) next to the host wall clock of estimate()
tm, _ = ctx.time(1, ncol, per_kernel=False)
t0 = time.perf_counter()
ctx.estimate(1, ncol, per_vertex=False)
t1 = time.perf_counter()
print(f"{cfg}: device time of {ncol} colorings {tm.total_ms:.1f} ms; estimate() without per-vertex {1e3 * (t1 - t0):.1f} ms")
