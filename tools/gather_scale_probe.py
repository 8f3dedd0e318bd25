"""L2-footprint probe for the SpMM: the same R-MAT shape (cfg3 edge factor and
probabilities, k=12 template) at several scales; prints the SpMM phase's
gathered-bytes rate per scale (a copy's footprint halves per scale step)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1903_04395_b200 as T  # noqa: E402

parents = [-1, 0, 1, 2, 0, 4, 4, 6, 0, 8, 9, 9]
for scale in [int(x) for x in (sys.argv[1:] or ["18", "19", "20"])]:
    g = T.generate_rmat(T.RmatSpec(scale, 100 << scale, .45, .15, .15, .25, 1))
    c = T.Context(0)
    c.set_graph(g)
    c.set_template(T.template_from_parents(parents, 0))
    c.time(1, 2)
    tm, _ = c.time(10, 3, per_kernel=True)
    print(f"scale {scale}: n {g.n} nnz {g.nnz()} ms/coloring {tm.total_ms / 3:.2f} spmm {tm.spmm_ms / 3:.2f} "
          f"gathered {tm.spmm_gathered_bytes / (tm.spmm_ms * 1e-3) / 1e12:.2f} TB/s "
          f"per-nnz {tm.total_ms / 3 / g.nnz() * 1e9:.3f} ns", flush=True)
