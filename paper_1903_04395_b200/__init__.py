"""treecount-b200: B200-native pruned color-coding DP (PGBSC, arXiv 1903.04395).

The product is libtcg.so (C ABI in include/tcg.h): C++ host code for the CSR,
template partition, combinadic split tables and estimator scaling, and
hand-written sm_100a kernels for the per-coloring DP (on-device MT19937-64
coloring, neighbour-histogram / panel SpMM, fused eMA, fp64 root).
`treecount` mirrors the reference C++ API (engines.hpp / estimator.hpp).
"""
from . import _native  # noqa: F401  (raises ImportError if libtcg.so is missing)
from .treecount import *  # noqa: F401,F403
from .treecount import (Context, EngineConfig, EngineKind, Graph, TemplateTree, estimate,
                        from_edges, generate_rmat, make_template, partition, run_iteration)

__all__ = ["Context", "EngineConfig", "EngineKind", "Graph", "TemplateTree", "estimate",
           "from_edges", "generate_rmat", "make_template", "partition", "run_iteration"]
