"""Python mirror of the reference `treecount` API for the hot path, backed by libtcg.so.

Same names, argument meaning and error behaviour as the reference headers
(/root/reference/proj/include/treecount/*.hpp), so code and tests written
against `treecount::estimate` / `run_iteration` read the same here.  The one
engine is `EngineKind.b200` -- the sm_100a SpMM + fused-eMA path; the
reference's CPU engines (`baseline`, `pruned`, `vectorized`) are not part of
this package (their results are the parity target, see oracle/).

Host pieces (CSR construction, plan, split tables, |Aut|) run in the native
library's C++ host code; every count table lives on the GPU.
"""
from __future__ import annotations

import ctypes as C
import enum
import time
import weakref
from dataclasses import dataclass, field
from typing import Optional

import numpy as np

from . import _native as N
from ._native import (CudaError, InvalidArgument, LogicError, MemoryBudgetError, NonFiniteError, ParseError,
                      TcgError, check, lib)

kMaxTemplateSize = N.TCG_MAX_K  # color_index.hpp:15


def _ptr(a: np.ndarray):
    return a.ctypes.data_as(C.c_void_p) if a is not None else None


# ------------------------------------------------------------------- graph
class Graph:
    """Undirected simple graph as symmetric CSR (graph.hpp:27-42).

    `csc_col_ptr` (int64, n+1) and `csc_rows` (int32, 2m) are the reference's
    kernel form; the matrix is symmetric so CSC == CSR."""

    def __init__(self, handle):
        self._h = C.c_void_p(handle)
        n, m, nnz, mx = C.c_int32(), C.c_int64(), C.c_int64(), C.c_int32()
        check(lib.tcg_graph_info(self._h, C.byref(n), C.byref(m), C.byref(nnz), C.byref(mx)))
        self.n, self.m, self.max_degree = n.value, m.value, mx.value
        rp = lib.tcg_graph_row_ptr(self._h)
        cl = lib.tcg_graph_col(self._h)
        self.csc_col_ptr = np.ctypeslib.as_array(rp, shape=(self.n + 1,))
        self.csc_rows = (np.ctypeslib.as_array(cl, shape=(nnz.value,)) if nnz.value
                         else np.zeros(0, np.int32))
        self._fin = weakref.finalize(self, lib.tcg_graph_destroy, self._h)

    def nnz(self) -> int:
        return 2 * self.m

    def degree(self, v: int) -> int:
        return int(self.csc_col_ptr[v + 1] - self.csc_col_ptr[v])

    def neighbors(self, v: int) -> np.ndarray:
        return self.csc_rows[self.csc_col_ptr[v]:self.csc_col_ptr[v + 1]]

    @classmethod
    def from_csr(cls, n: int, row_ptr, col) -> "Graph":
        rp = np.ascontiguousarray(row_ptr, dtype=np.int64)
        cl = np.ascontiguousarray(col, dtype=np.int32)
        h = C.c_void_p()
        check(lib.tcg_graph_from_csr(n, _ptr(rp), _ptr(cl) if cl.size else None, C.byref(h)))
        return cls(h.value)


def from_edges(edges, n_hint: int = -1) -> Graph:
    """graph.hpp:65-95: symmetrize by union, drop self-loops, dedup, sort."""
    e = np.ascontiguousarray(np.asarray(edges, dtype=np.int32).reshape(-1, 2))
    h = C.c_void_p()
    check(lib.tcg_graph_from_edges(_ptr(e) if e.size else None, e.shape[0], n_hint, C.byref(h)))
    return Graph(h.value)


@dataclass
class RmatSpec:  # synthgen.hpp:14-21
    scale: int = 10
    edges: int = 0
    a: float = 0.25
    b: float = 0.25
    c: float = 0.25
    d: float = 0.25
    seed: int = 0


def generate_rmat(spec: RmatSpec) -> Graph:
    """synthgen.hpp:40-74 (same MT19937-64 edge stream, then from_edges)."""
    h = C.c_void_p()
    check(lib.tcg_generate_rmat(spec.scale, spec.edges, spec.a, spec.b, spec.c, spec.d,
                                spec.seed, C.byref(h)))
    return Graph(h.value)


def generate_erdos_renyi(n: int, p: float, seed: int) -> Graph:
    h = C.c_void_p()
    check(lib.tcg_generate_erdos_renyi(n, p, seed, C.byref(h)))
    return Graph(h.value)


# ---------------------------------------------------------------- template
@dataclass
class TemplateTree:  # templates.hpp:19-33
    k: int
    edges: list
    root: int = 0

    def _edge_array(self) -> np.ndarray:
        a = np.asarray(self.edges, dtype=np.int32).reshape(-1)
        return np.ascontiguousarray(a) if a.size else np.zeros(2, np.int32)


def make_template(edges, root: int = -1) -> TemplateTree:
    """templates.hpp:80-90: validate; root = -1 picks max degree, smallest id."""
    edges = [(int(u), int(v)) for u, v in edges]
    k = max(max(u, v) for u, v in edges) + 1 if edges else 0
    if k == 0:
        raise ParseError("not a tree: empty template")
    if len(edges) != k - 1:  # templates.hpp:38-41
        raise ParseError(f"not a tree: {len(edges)} edges for {k} vertices")
    plan = N.TcgPlan()
    t = TemplateTree(k, edges, root)
    check(lib.tcg_partition(k, _ptr(t._edge_array()), root, C.byref(plan)))
    t.root = plan.root
    return t


def single_vertex_template() -> TemplateTree:
    return TemplateTree(1, [], 0)


def template_from_parents(parents, root: int = 0) -> TemplateTree:
    """BASELINE.json parent array -> edges (p[v], v), rooted at `root`."""
    if len(parents) == 1:  # k = 1 (templates.hpp single_vertex_template)
        return single_vertex_template()
    return make_template([(int(parents[v]), v) for v in range(1, len(parents))], root)


@dataclass
class PlanNode:  # templates.hpp:143-160
    id: int
    size: int
    root: int
    active_child: int
    passive_child: int
    parent: int

    def is_leaf(self) -> bool:
        return self.size == 1


@dataclass
class PartitionPlan:  # templates.hpp:162-170
    k: int
    root: int
    nodes: list
    dp_order: list

    def node(self, i: int) -> PlanNode:
        return self.nodes[i]

    def full_node(self) -> int:
        return self.dp_order[-1]


def _plan_from_c(p: N.TcgPlan) -> PartitionPlan:
    nodes = [PlanNode(i, p.size[i], p.node_root[i], p.active_child[i], p.passive_child[i],
                      p.parent[i]) for i in range(p.num_nodes)]
    return PartitionPlan(p.k, p.root, nodes, [p.dp_order[i] for i in range(p.num_nodes)])


def partition(t: TemplateTree) -> PartitionPlan:
    """templates.hpp:249-259."""
    p = N.TcgPlan()
    check(lib.tcg_partition(t.k, _ptr(t._edge_array()), t.root, C.byref(p)))
    return _plan_from_c(p)


def automorphism_count(t: TemplateTree) -> int:
    """templates.hpp:326-339."""
    out = C.c_uint64()
    check(lib.tcg_automorphisms(t.k, _ptr(t._edge_array()), C.byref(out)))
    return out.value


def estimate_bytes(plan: PartitionPlan, n: int, k: Optional[int] = None) -> int:
    """count_table.hpp:113-133 (the reference's fp64 liveness model)."""
    p = N.TcgPlan()
    p.k, p.root, p.num_nodes = plan.k, plan.root, len(plan.nodes)
    for i, nd in enumerate(plan.nodes):
        p.size[i], p.active_child[i], p.passive_child[i] = nd.size, nd.active_child, nd.passive_child
    for i, x in enumerate(plan.dp_order):
        p.dp_order[i] = x
    return int(lib.tcg_estimate_bytes(C.byref(p), n))


# ------------------------------------------------------------- color index
class ColorIndexer:
    """color_index.hpp:20-82 (combinadic index, Eq. 1)."""

    def __init__(self, k: int):
        if k < 1 or k > kMaxTemplateSize:
            raise InvalidArgument(f"color count k must be in [1, {kMaxTemplateSize}]")
        self._k = k

    def k(self) -> int:
        return self._k

    def binom(self, a: int, b: int) -> int:
        if b < 0 or b > a:
            return 0
        from math import comb
        return comb(a, b)

    def num_sets(self, h: int) -> int:
        return self.binom(self._k, h)

    def index_of(self, colors) -> int:
        c = np.ascontiguousarray(colors, dtype=np.int32)
        r = lib.tcg_color_index_of(self._k, _ptr(c), len(c))
        if r < 0:
            raise InvalidArgument((lib.tcg_last_error() or b"").decode())
        return int(r)

    def set_of(self, index: int, h: int) -> list:
        out = np.zeros(max(h, 1), np.int32)
        check(lib.tcg_color_set_of(self._k, index, h, _ptr(out)))
        return [int(x) for x in out[:h]]


@dataclass
class SplitTable:  # color_index.hpp:91-101
    parent_size: int
    active_size: int
    passive_size: int
    parent_cols: int
    active_cols: int
    passive_cols: int
    pairs_per_parent: int
    partners_per_passive: int
    active_index: np.ndarray
    passive_index: np.ndarray
    grouped_parent: np.ndarray
    grouped_active: np.ndarray


def build_split_table(parent_size: int, active_size: int, indexer: ColorIndexer) -> SplitTable:
    """color_index.hpp:103-180."""
    k = indexer.k()
    passive = parent_size - active_size
    if active_size < 1 or passive < 1:
        raise InvalidArgument("split requires nonempty active and passive children")
    if parent_size > k:
        raise InvalidArgument("sub-template larger than color count")
    cs, ca, cp = indexer.num_sets(parent_size), indexer.num_sets(active_size), indexer.num_sets(passive)
    pairs, partners = indexer.binom(parent_size, active_size), indexer.binom(k - passive, active_size)
    arrs = [np.zeros(cs * pairs, np.int32) for _ in range(4)]
    check(lib.tcg_split_table(k, parent_size, active_size, *[_ptr(a) for a in arrs]))
    return SplitTable(parent_size, active_size, passive, cs, ca, cp, pairs, partners, *arrs)


def build_plan_splits(plan: PartitionPlan, indexer: ColorIndexer) -> list:
    """color_index.hpp:190-197 (None for leaves)."""
    return [None if nd.is_leaf() else
            build_split_table(nd.size, plan.node(nd.active_child).size, indexer)
            for nd in plan.nodes]


def colorful_probability(k: int) -> float:
    """estimator.hpp:29-33: k!/k^k as a product of i/k."""
    return float(lib.tcg_colorful_probability(k))


# ------------------------------------------------------------------ engine
class EngineKind(enum.Enum):
    baseline = "baseline"      # reference CPU engines: not provided here
    pruned = "pruned"
    vectorized = "vectorized"
    b200 = "b200"              # this package: sm_100a SpMM + fused eMA


def engine_name(k: EngineKind) -> str:
    return k.value


def engine_from_name(s: str) -> EngineKind:
    try:
        return EngineKind(s)
    except ValueError:
        raise InvalidArgument(f"unknown engine '{s}'") from None


@dataclass
class EngineConfig:  # engines.hpp:46-51 (+ device)
    workers: int = 1                 # CPU detail of the reference; ignored
    batch: int = 16                  # Z of the reference (results are Z-independent); ignored
    memory_budget: int = 0           # bytes of device count tables; 0 = unlimited
    keep_full_table: bool = False
    device: int = 0
    keep_node_tables: bool = False   # inspection: keep every node table on device


@dataclass
class NodeStats:  # engines.hpp:53-61 (+ device phase split)
    seconds: float = 0.0
    neighbor_passes: int = 0
    traversals: int = 0
    flops: int = 0
    spmm_seconds: float = 0.0
    ema_seconds: float = 0.0
    spmm_bytes: int = 0
    ema_bytes: int = 0
    ema_flops: int = 0


@dataclass
class IterationResult:  # engines.hpp:63-84
    engine: EngineKind = EngineKind.b200
    rooted_total: float = 0.0
    per_node: list = field(default_factory=list)
    full_table: Optional[np.ndarray] = None   # n x 1 fp64 (keep_full_table)

    def neighbor_passes(self) -> int:
        return sum(s.neighbor_passes for s in self.per_node)

    def traversals(self) -> int:
        return sum(s.traversals for s in self.per_node)

    def flops(self) -> int:
        return sum(s.flops for s in self.per_node)


@dataclass
class Coloring:  # count_table.hpp:85-88
    color: np.ndarray
    seed: int = 0


class Context:
    """One device engine (tcg_ctx): graph + template resident on one GPU, or --
    with `devices=[...]` (tcg_create_multi) -- on several GPUs of this process,
    colorings of estimate()/time() spread over them."""

    def __init__(self, device: int = 0, memory_budget: int = 0, keep_tables: bool = False, devices=None):
        cfg = N.TcgConfig()
        cfg.device, cfg.memory_budget = device, memory_budget
        cfg.flags = N.TCG_KEEP_TABLES if keep_tables else 0
        h = C.c_void_p()
        if devices is not None:
            ids = (C.c_int * len(devices))(*devices)
            check(lib.tcg_create_multi(C.byref(cfg), ids, len(devices), C.byref(h)))
        else:
            check(lib.tcg_create(C.byref(cfg), C.byref(h)))
        self._h = h
        self._fin = weakref.finalize(self, lib.tcg_destroy, h)
        self.n = None
        self.k = None
        self.graph = None

    # -- vertex sharding; call before set_graph -------------
    def set_shard_torch(self, rank: int, world: int, group=None) -> None:
        """Device transport through torch.distributed (NCCL over NVLink/NVSwitch
        when the process group is NCCL): the engine hands device pointers, the
        panel is all-gathered with all_gather_into_tensor on zero-copy views."""
        import torch
        import torch.distributed as dist
        dev = torch.device("cuda", torch.cuda.current_device())

        class _Dev:  # __cuda_array_interface__ view of a raw device buffer
            def __init__(self, ptr, nbytes):
                self.__cuda_array_interface__ = {"shape": (nbytes,), "typestr": "|u1", "descr": [("", "|u1")],
                                                 "data": (ptr, False), "strides": None, "version": 2}

        def fn(user, send, nbytes, recv):
            try:
                src = torch.as_tensor(_Dev(send, nbytes), device=dev)
                dst = torch.as_tensor(_Dev(recv, nbytes * world), device=dev)
                dist.all_gather_into_tensor(dst, src, group=group)
                torch.cuda.current_stream().synchronize()
                return 0
            except Exception:  # noqa: BLE001 -- reported as a status code
                import traceback
                traceback.print_exc()
                return 1
        self._allgather_cb = N.ALLGATHER_FN(fn)  # keep alive
        check(lib.tcg_set_shard_device(self._h, rank, world, C.cast(self._allgather_cb, C.c_void_p), None))

    def set_shard_nccl(self, rank: int, world: int, exchange=None) -> None:
        """The library's own NCCL data plane (tcg_set_shard_nccl): rank 0 creates
        the NCCL unique id, `exchange(id_bytes_or_None) -> id_bytes` hands it to
        every rank (default: torch.distributed.broadcast_object_list over the
        default process group), and each rank's context builds its
        communicator; panel all-gathers then run asynchronously on the
        library's communication stream."""
        _nccl_env()
        ident = None
        if rank == 0:
            buf = (C.c_uint8 * N.TCG_NCCL_ID_BYTES)()
            check(lib.tcg_nccl_unique_id(buf))
            ident = bytes(buf)
        if world > 1:
            if exchange is None:
                import torch.distributed as dist
                box = [ident]
                dist.broadcast_object_list(box, src=0)
                ident = box[0]
            else:
                ident = exchange(ident)
        buf = (C.c_uint8 * N.TCG_NCCL_ID_BYTES).from_buffer_copy(ident)
        check(lib.tcg_set_shard_nccl(self._h, rank, world, buf))

    def set_shard_loopback(self, rank: int, hub: "LoopbackHub") -> None:
        """In-process rank of a LoopbackHub (tcg_set_shard_loopback)."""
        self._hub = hub  # keep the hub alive as long as this context
        check(lib.tcg_set_shard_loopback(self._h, rank, hub._h))

    def set_shard_host(self, rank: int, world: int, allgather) -> None:
        """Host transport: allgather(send: bytes-like np.uint8 array) -> np.uint8
        array of world*len(send) bytes in rank order (e.g. gloo)."""
        def fn(user, send, nbytes, recv):
            try:
                src = np.ctypeslib.as_array((C.c_uint8 * nbytes).from_address(send)).copy()
                out = np.asarray(allgather(src), dtype=np.uint8).reshape(-1)
                dst = np.ctypeslib.as_array((C.c_uint8 * out.size).from_address(recv))
                dst[:] = out
                return 0
            except Exception:  # noqa: BLE001 -- reported as a status code
                return 1
        self._allgather_cb = N.ALLGATHER_FN(fn)  # keep alive
        check(lib.tcg_set_shard_host(self._h, rank, world, C.cast(self._allgather_cb, C.c_void_p), None))

    def set_graph(self, g: Graph) -> None:
        check(lib.tcg_set_graph_handle(self._h, g._h))
        self.n, self.graph = g.n, g

    def set_graph_csr(self, n: int, row_ptr: np.ndarray, col: np.ndarray) -> None:
        """Host CSR buffers, copied host -> device (the e2e path)."""
        check(lib.tcg_set_graph(self._h, n, _ptr(row_ptr), _ptr(col) if col.size else None))
        self.n, self.graph = n, None

    def set_graph_edges(self, edges, n_hint: int = -1) -> None:
        """graph.hpp:65-95 from_edges on the device (tcg_set_graph_edges)."""
        e = np.ascontiguousarray(np.asarray(edges, dtype=np.int32).reshape(-1, 2))
        check(lib.tcg_set_graph_edges(self._h, _ptr(e) if e.size else None, e.shape[0], n_hint))
        self.graph = None
        self.n = int(self.graph_csr()[0].shape[0] - 1)

    def graph_csr(self):
        """(row_ptr, col) of the context's graph over the caller's vertex ids."""
        n, nnz = C.c_int32(), C.c_int64()
        check(lib.tcg_get_graph_csr(self._h, C.byref(n), C.byref(nnz), None, None))
        rp = np.zeros(n.value + 1, np.int64)
        col = np.zeros(max(nnz.value, 1), np.int32)
        check(lib.tcg_get_graph_csr(self._h, None, None, _ptr(rp), _ptr(col)))
        return rp, col[:nnz.value]

    def set_template(self, t: TemplateTree) -> None:
        check(lib.tcg_set_template(self._h, t.k, _ptr(t._edge_array()), t.root))
        self.k = t.k

    def plan(self) -> tuple:
        p, aut = N.TcgPlan(), C.c_uint64()
        check(lib.tcg_get_plan(self._h, C.byref(p), C.byref(aut)))
        return _plan_from_c(p), aut.value

    def required_device_bytes(self) -> int:
        b = C.c_int64()
        check(lib.tcg_required_device_bytes(self._h, C.byref(b)))
        return b.value

    def coloring(self, seed: int) -> np.ndarray:
        out = np.zeros(max(self.n, 1), np.uint8)
        check(lib.tcg_coloring(self._h, seed, _ptr(out)))
        return out[:self.n]

    def run_coloring(self, seed: int = 0, colors: Optional[np.ndarray] = None,
                     per_vertex: bool = False, stats: bool = False):
        total = C.c_double()
        pv = np.zeros(max(self.n, 1), np.float64) if per_vertex else None
        st = (N.TcgNodeStats * N.TCG_MAX_NODES)() if stats else None
        cl = np.ascontiguousarray(colors, dtype=np.uint8) if colors is not None else None
        if cl is not None and cl.shape[0] != self.n:
            raise InvalidArgument("coloring size does not match graph")
        check(lib.tcg_run_coloring(self._h, seed, _ptr(cl) if cl is not None and cl.size else None,
                                   C.byref(total), _ptr(pv), st))
        return total.value, (pv[:self.n] if pv is not None else None), st

    def estimate(self, seed: int, iterations: int, per_vertex: bool = False):
        totals = np.zeros(max(iterations, 1), np.float64)
        est, se = C.c_double(), C.c_double()
        pv = np.zeros(max(self.n, 1), np.float64) if per_vertex else None
        check(lib.tcg_estimate(self._h, seed, iterations, _ptr(totals), C.byref(est),
                               C.byref(se), _ptr(pv)))
        return totals[:iterations], est.value, se.value, (pv[:self.n] if pv is not None else None)

    def node_table(self, node_id: int, which: int = 0) -> np.ndarray:
        plan, _ = self.plan()
        size = plan.node(node_id).size
        cols = 1 if node_id == plan.full_node() else (
            self.k if size == 1 else ColorIndexer(self.k).num_sets(size))
        out = np.zeros((self.n, cols), np.float64)
        check(lib.tcg_node_table(self._h, node_id, which, _ptr(out)))
        return out

    def spmm(self, x: np.ndarray) -> np.ndarray:
        x = np.ascontiguousarray(x, dtype=np.float32)
        if x.ndim == 1:
            x = x[:, None]
        y = np.zeros_like(x)
        check(lib.tcg_spmm(self._h, _ptr(x), x.shape[1], _ptr(y)))
        return y

    def spmm_rooted(self, k: int, s: int, colors: np.ndarray, x: np.ndarray, pair: bool = False) -> np.ndarray:
        """Y = A M through the production rooted SpMM (tcg_spmm_rooted); only the
        columns missing c(v) are computed (the rest are 0)."""
        x = np.ascontiguousarray(x, dtype=np.float32)
        colors = np.ascontiguousarray(colors, dtype=np.uint8)
        y = np.zeros_like(x)
        check(lib.tcg_spmm_rooted(self._h, k, s, 1 if pair else 0, _ptr(colors), _ptr(x), _ptr(y)))
        return y

    def set_rejection_limit(self, limit: int) -> None:
        check(lib.tcg_set_rejection_limit(self._h, limit))

    def kernel_launches(self) -> int:
        return int(lib.tcg_kernel_launches(self._h))

    def time(self, seed: int, count: int, per_kernel: bool = False):
        """Device-timed batch of colorings (CUDA events on the engine stream)."""
        if count < 1:
            return N.TcgTiming(), np.zeros(0)
        tm = N.TcgTiming()
        totals = np.zeros(count, np.float64)
        check(lib.tcg_time_colorings(self._h, seed, count, int(per_kernel), _ptr(totals), C.byref(tm)))
        return tm, totals


class LoopbackHub:
    """`world` in-process ranks exchanging panels by device-to-device copies
    (tcg_loopback_create); drive each rank's context from its own thread."""

    def __init__(self, world: int):
        h = C.c_void_p()
        check(lib.tcg_loopback_create(world, C.byref(h)))
        self._h = h
        self.world = world
        self._fin = weakref.finalize(self, lib.tcg_loopback_destroy, h)


def _nccl_env() -> None:
    """Point the library at the NCCL this Python environment ships (PyTorch's
    nvidia-nccl wheel) unless TCG_NCCL_LIB is set; an NCCL already loaded in
    the process is preferred by the library itself."""
    import os
    if os.environ.get("TCG_NCCL_LIB"):
        return
    try:
        import nvidia.nccl
        for d in nvidia.nccl.__path__:
            p = os.path.join(d, "lib", "libnccl.so.2")
            if os.path.exists(p):
                os.environ["TCG_NCCL_LIB"] = p
                return
    except ImportError:
        pass


def shard_bounds(g: Graph, world: int) -> np.ndarray:
    """Row bounds of `world` vertex shards (balanced by degree + average degree)."""
    out = np.zeros(world + 1, np.int64)
    check(lib.tcg_shard_bounds(g.n, _ptr(np.ascontiguousarray(g.csc_col_ptr)), world, _ptr(out)))
    return out


# Contexts behind the reference-style free functions, keyed by (graph, template, cfg).
_ctx_cache: dict = {}


def _context(g: Graph, t: TemplateTree, cfg: EngineConfig) -> Context:
    key = (id(g), t.k, tuple(map(tuple, t.edges)), t.root, cfg.device, cfg.memory_budget,
           cfg.keep_node_tables)
    ent = _ctx_cache.get(key)
    if ent is not None and ent[0]() is g:
        return ent[1]
    ctx = Context(cfg.device, cfg.memory_budget, cfg.keep_node_tables)
    ctx.set_graph(g)
    ctx.set_template(t)
    if len(_ctx_cache) > 8:
        _ctx_cache.clear()
    _ctx_cache[key] = (weakref.ref(g), ctx)
    return ctx


def _require_b200(kind: EngineKind) -> None:
    if kind is not EngineKind.b200:
        raise InvalidArgument(f"engine '{kind.value}' is a reference CPU engine; this package "
                         "provides EngineKind.b200")


def random_coloring(g: Graph, k: int, seed: int, device: int = 0) -> Coloring:
    """count_table.hpp:90-99, generated on the GPU (bit-exact MT19937-64)."""
    if k < 1:
        raise InvalidArgument("k must be >= 1")
    ctx = _context(g, single_vertex_template() if k == 1 else
                   TemplateTree(k, [(i, i + 1) for i in range(k - 1)], 0), EngineConfig(device=device))
    return Coloring(ctx.coloring(seed), seed)


def _template_of_plan(plan: PartitionPlan) -> TemplateTree:
    # rebuild the template edges from the plan's cut edges (each internal node
    # cuts (root, passive child's root)) -- the plan determines the tree.
    edges = [(nd.root, plan.node(nd.passive_child).root) for nd in plan.nodes if not nd.is_leaf()]
    return TemplateTree(plan.k, edges, plan.root)


def run_iteration(kind: EngineKind, g: Graph, plan_or_template, coloring: Coloring,
                  indexer: Optional[ColorIndexer] = None,
                  cfg: Optional[EngineConfig] = None) -> IterationResult:
    """engines.hpp:302-307: one coloring through the b200 engine."""
    _require_b200(kind)
    cfg = cfg or EngineConfig()
    t = (plan_or_template if isinstance(plan_or_template, TemplateTree)
         else _template_of_plan(plan_or_template))
    if indexer is not None and indexer.k() != t.k:
        raise InvalidArgument("indexer and plan disagree on k")
    if len(coloring.color) != g.n:
        raise InvalidArgument("coloring size does not match graph")
    ctx = _context(g, t, cfg)
    total, pv, st = ctx.run_coloring(coloring.seed, coloring.color, per_vertex=cfg.keep_full_table,
                                     stats=True)
    plan, _ = ctx.plan()
    per_node = [NodeStats(s.seconds, s.neighbor_passes, s.traversals, s.flops, s.spmm_seconds,
                          s.ema_seconds, s.spmm_bytes, s.ema_bytes, s.ema_flops)
                for s in list(st)[:len(plan.nodes)]]
    return IterationResult(EngineKind.b200, total, per_node,
                           pv.reshape(-1, 1) if pv is not None else None)


@dataclass
class EstimateResult:  # estimator.hpp:12-27
    iterations: int = 0
    rooted_totals: list = field(default_factory=list)
    colorful_probability: float = 0.0
    aut: int = 1
    estimate: float = 0.0
    stderr_of_mean: float = 0.0
    neighbor_passes: int = 0
    traversals: int = 0
    flops: int = 0
    iteration_seconds: list = field(default_factory=list)
    per_node_seconds: list = field(default_factory=list)
    per_vertex_estimate: Optional[np.ndarray] = None

    def scale(self) -> float:
        return 1.0 / (self.aut * self.colorful_probability)


def estimate(g: Graph, t: TemplateTree, kind: EngineKind, iterations: int, seed: int,
             cfg: Optional[EngineConfig] = None, per_vertex: bool = False) -> EstimateResult:
    """estimator.hpp:49-93: colorings seed, seed+1, ...; scaled by 1/(aut * k!/k^k)."""
    _require_b200(kind)
    if iterations < 1:
        raise InvalidArgument("iterations must be >= 1")
    cfg = cfg or EngineConfig()
    ctx = _context(g, t, cfg)
    plan, aut = ctx.plan()
    t0 = time.perf_counter()
    totals, est, se, pv = ctx.estimate(seed, iterations, per_vertex)
    secs = time.perf_counter() - t0
    kk = ColorIndexer(t.k)
    passes = sum(kk.num_sets(plan.node(nd.passive_child).size) for nd in plan.nodes if not nd.is_leaf())
    return EstimateResult(iterations=iterations, rooted_totals=list(totals),
                          colorful_probability=colorful_probability(t.k), aut=aut, estimate=est,
                          stderr_of_mean=se, neighbor_passes=passes * iterations,
                          traversals=passes * iterations * g.n,
                          iteration_seconds=[secs / iterations] * iterations,
                          per_vertex_estimate=pv)
