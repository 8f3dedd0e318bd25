"""ctypes front for the CPU oracle -- TEST INFRASTRUCTURE ONLY.

`oracle` is the parity checker for the B200 path: a plain-C restatement of the
reference's pruned color-coding DP (tc_oracle.c) plus, where /root/reference
was present at build time, the UNMODIFIED reference compiled into
oracle/_ref/libtcref.so (ref_driver.cpp).  Only tests/, __graft_entry__.smoke()
and bench.py's cpu_baseline / --impl reference legs may import this package.
The product package (paper_1903_04395_b200) never does.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
_LIB = os.path.join(HERE, "libtc_oracle.so")
_REF = os.path.join(HERE, "_ref", "libtcref.so")

_i32p = np.ctypeslib.ndpointer(np.int32, flags="C")
_i64p = np.ctypeslib.ndpointer(np.int64, flags="C")
_u8p = np.ctypeslib.ndpointer(np.uint8, flags="C")
_f64p = np.ctypeslib.ndpointer(np.float64, flags="C")
_u64p = np.ctypeslib.ndpointer(np.uint64, flags="C")

MAXK = 20
MAXNODES = 2 * MAXK - 1


class OrcPlan(C.Structure):
    _fields_ = [("k", C.c_int), ("root", C.c_int), ("num_nodes", C.c_int),
                ("size", C.c_int * MAXNODES), ("node_root", C.c_int * MAXNODES),
                ("active_child", C.c_int * MAXNODES), ("passive_child", C.c_int * MAXNODES),
                ("parent", C.c_int * MAXNODES), ("dp_order", C.c_int * MAXNODES)]


def build(ref: bool = False) -> None:
    """Compile the restatement (and, if asked and /root/reference exists, the reference)."""
    targets = ["all"] + (["ref"] if ref and os.path.isdir("/root/reference/proj/include") else [])
    subprocess.run(["make", "-s", "-C", HERE] + targets, check=True)


_lib = None
_ref = None


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(
                os.path.join(HERE, "tc_oracle.c")):
            build()
        L = C.CDLL(_LIB)
        L.orc_random_coloring.argtypes = [C.c_int32, C.c_int, C.c_uint64, C.c_uint64, _u8p]
        L.orc_csr_from_edges.argtypes = [_i32p, C.c_int64, C.c_int32, C.POINTER(C.c_int32),
                                         C.POINTER(C.POINTER(C.c_int64)),
                                         C.POINTER(C.POINTER(C.c_int32)), C.POINTER(C.c_int64)]
        L.orc_generate_rmat.argtypes = [C.c_int, C.c_int64, C.c_double, C.c_double, C.c_double,
                                        C.c_double, C.c_uint64, C.POINTER(C.c_int32),
                                        C.POINTER(C.POINTER(C.c_int64)),
                                        C.POINTER(C.POINTER(C.c_int32)), C.POINTER(C.c_int64)]
        L.orc_free.argtypes = [C.c_void_p]
        L.orc_binom.restype = C.c_int64
        L.orc_binom.argtypes = [C.c_int, C.c_int]
        L.orc_index_of.restype = C.c_int64
        L.orc_index_of.argtypes = [np.ctypeslib.ndpointer(np.intc, flags="C"), C.c_int]
        L.orc_set_of.argtypes = [C.c_int, C.c_int64, C.c_int, np.ctypeslib.ndpointer(np.intc, flags="C")]
        L.orc_split_table.argtypes = [C.c_int, C.c_int, C.c_int, _i32p, _i32p, _i32p, _i32p]
        L.orc_partition.argtypes = [C.c_int, _i32p, C.c_int, C.POINTER(OrcPlan)]
        L.orc_automorphisms.restype = C.c_uint64
        L.orc_automorphisms.argtypes = [C.c_int, _i32p]
        L.orc_estimate_bytes.restype = C.c_int64
        L.orc_estimate_bytes.argtypes = [C.POINTER(OrcPlan), C.c_int64]
        L.orc_run_iteration.restype = C.c_double
        L.orc_run_iteration.argtypes = [C.c_int32, _i64p, _i32p, C.POINTER(OrcPlan), _u8p,
                                        C.c_void_p, C.POINTER(C.c_void_p)]
        L.orc_colorful_probability.restype = C.c_double
        L.orc_colorful_probability.argtypes = [C.c_int]
        L.orc_estimate.argtypes = [C.c_int32, _i64p, _i32p, C.c_int, _i32p, C.c_int, C.c_int,
                                   C.c_uint64, _f64p, C.POINTER(C.c_double),
                                   C.POINTER(C.c_double), C.POINTER(C.c_uint64)]
        L.orc_mt_seed.argtypes = [C.c_void_p, C.c_uint64]
        L.orc_mt_next.restype = C.c_uint64
        L.orc_mt_next.argtypes = [C.c_void_p]
        _lib = L
    return _lib


def _edges_arr(edges) -> np.ndarray:
    a = np.ascontiguousarray(np.asarray(edges, dtype=np.int32).reshape(-1))
    return a if a.size else np.zeros(2, np.int32)


def parent_array_edges(parents) -> list[tuple[int, int]]:
    """BASELINE.json parent array -> template edges (p[v], v) for v >= 1."""
    return [(int(parents[v]), v) for v in range(1, len(parents))]


# ----------------------------------------------------------------------- rng
def mt_first(seed: int, count: int) -> list[int]:
    buf = C.create_string_buffer(312 * 8 + 16)
    lib().orc_mt_seed(buf, seed)
    return [lib().orc_mt_next(buf) for _ in range(count)]


def random_coloring(n: int, k: int, seed: int, limit_override: int = 0) -> np.ndarray:
    out = np.empty(max(n, 1), np.uint8)
    lib().orc_random_coloring(n, k, seed, limit_override, out)
    return out[:n]


# --------------------------------------------------------------------- graph
def _take_csr(n, rp, cl, nnz):
    row_ptr = np.ctypeslib.as_array(rp, shape=(n.value + 1,)).copy()
    col = np.ctypeslib.as_array(cl, shape=(max(nnz.value, 1),))[:nnz.value].copy()
    lib().orc_free(C.cast(rp, C.c_void_p))
    lib().orc_free(C.cast(cl, C.c_void_p))
    return n.value, row_ptr, col


def csr_from_edges(edges, n_hint: int = -1):
    e = np.ascontiguousarray(np.asarray(edges, dtype=np.int32).reshape(-1, 2))
    n, nnz = C.c_int32(), C.c_int64()
    rp, cl = C.POINTER(C.c_int64)(), C.POINTER(C.c_int32)()
    flat = e.reshape(-1) if e.size else np.zeros(2, np.int32)
    if lib().orc_csr_from_edges(flat, e.shape[0], n_hint, C.byref(n), C.byref(rp), C.byref(cl),
                                C.byref(nnz)) != 0:
        raise ValueError("vertex id out of range")
    return _take_csr(n, rp, cl, nnz)


def generate_rmat(scale, edges, a, b, c, d, seed):
    n, nnz = C.c_int32(), C.c_int64()
    rp, cl = C.POINTER(C.c_int64)(), C.POINTER(C.c_int32)()
    if lib().orc_generate_rmat(scale, edges, a, b, c, d, seed, C.byref(n), C.byref(rp),
                               C.byref(cl), C.byref(nnz)) != 0:
        raise ValueError("bad rmat spec")
    return _take_csr(n, rp, cl, nnz)


# ------------------------------------------------------------ color indexing
def binom(a: int, b: int) -> int:
    return int(lib().orc_binom(a, b))


def index_of(colors) -> int:
    c = np.ascontiguousarray(colors, dtype=np.intc)
    return int(lib().orc_index_of(c, len(c)))


def set_of(k: int, index: int, h: int) -> list[int]:
    out = np.zeros(max(h, 1), np.intc)
    lib().orc_set_of(k, index, h, out)
    return [int(x) for x in out[:h]]


def split_table(k: int, parent: int, active: int) -> dict:
    passive = parent - active
    cs, cp = binom(k, parent), binom(k, passive)
    pairs, partners = binom(parent, active), binom(k - passive, active)
    ai = np.zeros(max(cs * pairs, 1), np.int32)
    pi = np.zeros_like(ai)
    gp = np.zeros(max(cp * partners, 1), np.int32)
    ga = np.zeros_like(gp)
    if lib().orc_split_table(k, parent, active, ai, pi, gp, ga) != 0:
        raise ValueError("bad split")
    return dict(parent_cols=cs, passive_cols=cp, active_cols=binom(k, active),
                pairs_per_parent=pairs, partners_per_passive=partners,
                active_index=ai, passive_index=pi, grouped_parent=gp, grouped_active=ga)


# ------------------------------------------------------------------ template
def partition(k: int, edges, root: int = -1) -> OrcPlan:
    plan = OrcPlan()
    if lib().orc_partition(k, _edges_arr(edges), root, C.byref(plan)) != 0:
        raise ValueError("not a tree")
    return plan


def plan_nodes(plan: OrcPlan) -> list[dict]:
    return [dict(id=i, size=plan.size[i], root=plan.node_root[i],
                 active=plan.active_child[i], passive=plan.passive_child[i])
            for i in range(plan.num_nodes)]


def automorphisms(k: int, edges) -> int:
    return int(lib().orc_automorphisms(k, _edges_arr(edges)))


def estimate_bytes(plan: OrcPlan, n: int) -> int:
    return int(lib().orc_estimate_bytes(C.byref(plan), n))


def colorful_probability(k: int) -> float:
    return float(lib().orc_colorful_probability(k))


# ------------------------------------------------------------------------ DP
def run_iteration(n, row_ptr, col, plan: OrcPlan, colors, want_tables: bool = False):
    """One coloring; returns (rooted_total, per_vertex, tables|None).

    tables[id] (internal nodes and the root) is the node's n x C(k,|T_s|)
    table, returned vertex-major (n, C) for convenience."""
    pv = np.zeros(max(n, 1), np.float64)
    slots = (C.c_void_p * MAXNODES)()
    col = np.ascontiguousarray(col, dtype=np.int32) if len(col) else np.zeros(1, np.int32)
    total = lib().orc_run_iteration(n, np.ascontiguousarray(row_ptr, dtype=np.int64), col,
                                    C.byref(plan), np.ascontiguousarray(colors, dtype=np.uint8)
                                    if n else np.zeros(1, np.uint8),
                                    pv.ctypes.data, slots if want_tables else None)
    tables = None
    if want_tables:
        tables = {}
        for i in range(plan.num_nodes):
            if slots[i]:
                c = binom(plan.k, plan.size[i])
                arr = np.ctypeslib.as_array(C.cast(slots[i], C.POINTER(C.c_double)), shape=(c, n))
                tables[i] = arr.T.copy()
                lib().orc_free(slots[i])
    return total, pv[:n], tables


def estimate(n, row_ptr, col, k, edges, root, iterations, seed):
    totals = np.zeros(iterations, np.float64)
    est, se, aut = C.c_double(), C.c_double(), C.c_uint64()
    lib().orc_estimate(n, np.ascontiguousarray(row_ptr, dtype=np.int64),
                       np.ascontiguousarray(col, dtype=np.int32) if len(col) else np.zeros(1, np.int32),
                       k, _edges_arr(edges), root, iterations, seed, totals, C.byref(est),
                       C.byref(se), C.byref(aut))
    return dict(rooted_totals=totals, estimate=est.value, stderr_of_mean=se.value, aut=aut.value)


# ------------------------------------------------- the compiled reference (_ref)
def ref_available() -> bool:
    return os.path.exists(_REF)


def ref():
    """The UNMODIFIED reference (oracle/_ref/libtcref.so), via ref_driver.cpp."""
    global _ref
    if _ref is None:
        if not os.path.exists(_REF):
            build(ref=True)
        if not os.path.exists(_REF):
            raise RuntimeError("oracle/_ref/libtcref.so not built (needs /root/reference)")
        R = C.CDLL(_REF)
        vp = C.c_void_p
        R.ref_random_coloring.argtypes = [C.c_int32, C.c_int, C.c_uint64, _u8p]
        R.ref_mt_first.argtypes = [C.c_uint64, C.c_int, _u64p]
        R.ref_graph_from_edges.restype = vp
        R.ref_graph_from_edges.argtypes = [_i32p, C.c_int64, C.c_int32]
        R.ref_generate_rmat.restype = vp
        R.ref_generate_rmat.argtypes = [C.c_int, C.c_int64, C.c_double, C.c_double, C.c_double,
                                        C.c_double, C.c_uint64]
        R.ref_generate_erdos_renyi.restype = vp
        R.ref_generate_erdos_renyi.argtypes = [C.c_int32, C.c_double, C.c_uint64]
        R.ref_graph_from_csr.restype = vp
        R.ref_graph_from_csr.argtypes = [C.c_int32, _i64p, _i32p]
        R.ref_graph_info.argtypes = [vp, C.POINTER(C.c_int32), C.POINTER(C.c_int64)]
        R.ref_graph_csr.argtypes = [vp, _i64p, _i32p]
        R.ref_graph_free.argtypes = [vp]
        ip = np.ctypeslib.ndpointer(np.intc, flags="C")
        R.ref_plan.argtypes = [C.c_int, _i32p, C.c_int, ip, ip, ip, ip, ip, C.POINTER(C.c_int)]
        R.ref_split_table.argtypes = [C.c_int, C.c_int, C.c_int, _i32p, _i32p, _i32p, _i32p]
        R.ref_automorphisms.restype = C.c_uint64
        R.ref_automorphisms.argtypes = [C.c_int, _i32p]
        R.ref_estimate_bytes.restype = C.c_int64
        R.ref_estimate_bytes.argtypes = [C.c_int, _i32p, C.c_int, C.c_int64]
        R.ref_run_iteration.argtypes = [vp, C.c_int, _i32p, C.c_int, _u8p, C.c_int, C.c_int,
                                        C.POINTER(C.c_double), C.c_void_p, C.POINTER(C.c_double)]
        R.ref_estimate.argtypes = [vp, C.c_int, _i32p, C.c_int, C.c_int, C.c_uint64, C.c_int,
                                   _f64p, C.POINTER(C.c_double), C.POINTER(C.c_double),
                                   C.POINTER(C.c_uint64), C.POINTER(C.c_double)]
        R.ref_time_sampled.argtypes = [vp, C.c_int, _i32p, C.c_int, C.c_uint64, C.c_int, C.c_int,
                                       C.c_int, _f64p]
        R.ref_run_iteration_stats.argtypes = [vp, C.c_int, _i32p, C.c_int, C.c_uint64, C.c_int, C.c_int,
                                              C.POINTER(C.c_double), C.POINTER(C.c_double), _f64p,
                                              C.POINTER(C.c_int)]
        R.ref_step_begin.restype = vp
        R.ref_step_begin.argtypes = [vp, C.c_int, _i32p, C.c_int, C.c_uint64, C.c_int, C.c_int, C.c_int]
        R.ref_step_run.argtypes = [vp, C.c_int, C.POINTER(C.c_double)]
        R.ref_step_finish.argtypes = [vp, C.POINTER(C.c_double), _f64p, C.POINTER(C.c_int), _f64p]
        R.ref_step_free.argtypes = [vp]
        _ref = R
    return _ref


def physical_cores() -> int:
    """Physical cores of this host (lscpu: sockets x cores per socket), else os.cpu_count()."""
    try:
        out = subprocess.run(["lscpu"], capture_output=True, text=True, timeout=10).stdout
        f = {}
        for line in out.splitlines():
            if ":" in line:
                a, b = line.split(":", 1)
                f[a.strip()] = b.strip()
        cores = int(f["Core(s) per socket"]) * int(f.get("Socket(s)", "1"))
        if cores > 0:
            return cores
    except Exception:  # noqa: BLE001
        pass
    return os.cpu_count() or 1


class RefStepper:
    """One coloring of the UNMODIFIED reference vectorized engine, replayed in
    `steps` slices of about equal estimated cost (ref_driver.cpp RefStepper):
    random_coloring, init_leaf_table, load_batch + spmm_csc per Z-batch and
    ema() per grouped split, in IterationRun::run's order (engines.hpp:106-132,
    224-268).  Bit-identical to run_iteration; every unit is executed."""

    def __init__(self, g: "RefGraph", k: int, edges, root: int, seed: int, workers: int, steps: int,
                 batch: int = 16):
        self.g = g  # keep the graph alive
        e = np.ascontiguousarray(np.asarray(edges, np.int32).reshape(-1))
        self.h = ref().ref_step_begin(g.h, k, e if e.size else np.zeros(2, np.int32), root, seed, workers,
                                      batch, steps)
        if not self.h:
            raise RuntimeError("reference stepper refused the input")
        self.steps = steps

    def run(self, i: int) -> float:
        sec = C.c_double()
        if ref().ref_step_run(self.h, i, C.byref(sec)) < 0:
            raise RuntimeError(f"reference step {i} failed")
        return sec.value

    def finish(self):
        total, nn = C.c_double(), C.c_int()
        ns = np.zeros(3 * MAXNODES)
        out = np.zeros(2)
        if ref().ref_step_finish(self.h, C.byref(total), ns, C.byref(nn), out) != 0:
            raise RuntimeError("reference stepper not finished")
        return total.value, ns[:3 * nn.value].reshape(nn.value, 3), out

    def __del__(self):
        if getattr(self, "h", None) and _ref is not None:
            _ref.ref_step_free(self.h)
            self.h = None


def ref_run_iteration_stats(g: "RefGraph", k: int, edges, root: int, seed: int, workers: int, batch: int = 16):
    """random_coloring + run_iteration(vectorized) in one call, timed, with NodeStats::seconds."""
    e = np.ascontiguousarray(np.asarray(edges, np.int32).reshape(-1))
    total, sec, nn = C.c_double(), C.c_double(), C.c_int()
    ns = np.zeros(MAXNODES)
    if ref().ref_run_iteration_stats(g.h, k, e if e.size else np.zeros(2, np.int32), root, seed, workers, batch,
                                     C.byref(total), C.byref(sec), ns, C.byref(nn)) != 0:
        raise RuntimeError("reference run_iteration failed")
    return total.value, sec.value, ns[:nn.value]


class RefGraph:
    """A reference treecount::Graph held by the compiled reference."""

    def __init__(self, handle):
        if not handle:
            raise ValueError("reference refused the graph")
        self.h = handle

    @classmethod
    def from_edges(cls, edges, n_hint=-1):
        e = np.ascontiguousarray(np.asarray(edges, dtype=np.int32).reshape(-1, 2))
        return cls(ref().ref_graph_from_edges(e.reshape(-1) if e.size else np.zeros(2, np.int32),
                                              e.shape[0], n_hint))

    @classmethod
    def from_csr(cls, n, row_ptr, col):
        col = np.ascontiguousarray(col, dtype=np.int32)
        return cls(ref().ref_graph_from_csr(n, np.ascontiguousarray(row_ptr, dtype=np.int64),
                                            col if col.size else np.zeros(1, np.int32)))

    @classmethod
    def rmat(cls, scale, edges, a, b, c, d, seed):
        return cls(ref().ref_generate_rmat(scale, edges, a, b, c, d, seed))

    def csr(self):
        n, nnz = C.c_int32(), C.c_int64()
        ref().ref_graph_info(self.h, C.byref(n), C.byref(nnz))
        rp = np.zeros(n.value + 1, np.int64)
        cl = np.zeros(max(nnz.value, 1), np.int32)
        ref().ref_graph_csr(self.h, rp, cl)
        return n.value, rp, cl[:nnz.value]

    def __del__(self):
        if getattr(self, "h", None) and _ref is not None:
            _ref.ref_graph_free(self.h)
            self.h = None
