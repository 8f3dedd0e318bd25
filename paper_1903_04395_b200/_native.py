"""ctypes binding of libtcg.so (the C ABI in include/tcg.h).

The native library is the product: there is no Python or CPU fallback for the
device path.  If libtcg.so is missing this module raises ImportError (build it
with `make -C paper_1903_04395_b200` or `python -c "import __graft_entry__ as g;
g.build()"`).
"""
from __future__ import annotations

import ctypes as C
import os
import re

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "libtcg.so")
HEADER = os.path.join(os.path.dirname(HERE), "include", "tcg.h")

if not os.path.exists(LIB_PATH):
    raise ImportError(f"{LIB_PATH} is missing: the CUDA extension has not been built "
                      "(run `make -C paper_1903_04395_b200`)")

lib = C.CDLL(LIB_PATH)

TCG_OK, TCG_EINVAL, TCG_ERESOURCE, TCG_ECUDA, TCG_ENONFINITE, TCG_ELOGIC, TCG_EPARSE = range(7)
TCG_MAX_K = 20
TCG_MAX_NODES = 2 * TCG_MAX_K - 1
TCG_KEEP_TABLES = 1
TCG_NCCL_ID_BYTES = 128


class TcgPlan(C.Structure):
    _fields_ = [("k", C.c_int), ("root", C.c_int), ("num_nodes", C.c_int),
                ("size", C.c_int * TCG_MAX_NODES), ("node_root", C.c_int * TCG_MAX_NODES),
                ("active_child", C.c_int * TCG_MAX_NODES),
                ("passive_child", C.c_int * TCG_MAX_NODES),
                ("parent", C.c_int * TCG_MAX_NODES), ("dp_order", C.c_int * TCG_MAX_NODES)]


class TcgConfig(C.Structure):
    _fields_ = [("device", C.c_int), ("memory_budget", C.c_int64), ("flags", C.c_int),
                ("reserved", C.c_int * 5)]


class TcgNodeStats(C.Structure):
    _fields_ = [("seconds", C.c_double), ("spmm_seconds", C.c_double),
                ("ema_seconds", C.c_double), ("neighbor_passes", C.c_uint64),
                ("traversals", C.c_uint64), ("flops", C.c_uint64), ("spmm_bytes", C.c_uint64),
                ("ema_bytes", C.c_uint64), ("ema_flops", C.c_uint64)]


class TcgTiming(C.Structure):
    _fields_ = [("total_ms", C.c_double), ("spmm_ms", C.c_double), ("ema_ms", C.c_double),
                ("spmm_launches", C.c_int64), ("ema_launches", C.c_int64), ("launches", C.c_int64),
                ("spmm_alg_bytes", C.c_double), ("hist_alg_bytes", C.c_double),
                ("ema_alg_bytes", C.c_double), ("ema_flops", C.c_double),
                ("spmm_gathered_bytes", C.c_double)]


vp, i32, i64, u64, dbl = C.c_void_p, C.c_int32, C.c_int64, C.c_uint64, C.c_double
P = C.POINTER

_SIGS = {
    "tcg_last_error": (C.c_char_p, []),
    "tcg_version": (C.c_char_p, []),
    "tcg_graph_from_edges": (C.c_int, [vp, i64, i32, P(vp)]),
    "tcg_graph_from_csr": (C.c_int, [i32, vp, vp, P(vp)]),
    "tcg_generate_rmat": (C.c_int, [C.c_int, i64, dbl, dbl, dbl, dbl, u64, P(vp)]),
    "tcg_generate_erdos_renyi": (C.c_int, [i32, dbl, u64, P(vp)]),
    "tcg_graph_info": (C.c_int, [vp, P(i32), P(i64), P(i64), P(i32)]),
    "tcg_graph_row_ptr": (P(i64), [vp]),
    "tcg_graph_col": (P(i32), [vp]),
    "tcg_graph_destroy": (None, [vp]),
    "tcg_partition": (C.c_int, [C.c_int, vp, C.c_int, P(TcgPlan)]),
    "tcg_automorphisms": (C.c_int, [C.c_int, vp, P(u64)]),
    "tcg_split_table": (C.c_int, [C.c_int, C.c_int, C.c_int, vp, vp, vp, vp]),
    "tcg_color_index_of": (i64, [C.c_int, vp, C.c_int]),
    "tcg_color_set_of": (C.c_int, [C.c_int, i64, C.c_int, vp]),
    "tcg_estimate_bytes": (i64, [P(TcgPlan), i64]),
    "tcg_colorful_probability": (dbl, [C.c_int]),
    "tcg_rooted_layout": (C.c_int, [C.c_int, C.c_int, vp, vp, vp]),
    "tcg_rtv_task_layout": (C.c_int, [C.c_int, C.c_int, C.c_int, C.c_int, vp]),
    "tcg_create": (C.c_int, [P(TcgConfig), P(vp)]),
    "tcg_destroy": (None, [vp]),
    "tcg_set_graph": (C.c_int, [vp, i32, vp, vp]),
    "tcg_set_graph_handle": (C.c_int, [vp, vp]),
    "tcg_set_template": (C.c_int, [vp, C.c_int, vp, C.c_int]),
    "tcg_required_device_bytes": (C.c_int, [vp, P(i64)]),
    "tcg_get_plan": (C.c_int, [vp, P(TcgPlan), P(u64)]),
    "tcg_coloring": (C.c_int, [vp, u64, vp]),
    "tcg_run_coloring": (C.c_int, [vp, u64, vp, P(dbl), vp, vp]),
    "tcg_estimate": (C.c_int, [vp, u64, C.c_int, vp, P(dbl), P(dbl), vp]),
    "tcg_node_table": (C.c_int, [vp, C.c_int, C.c_int, vp]),
    "tcg_spmm": (C.c_int, [vp, vp, C.c_int, vp]),
    "tcg_spmm_rooted": (C.c_int, [vp, C.c_int, C.c_int, C.c_int, vp, vp, vp]),
    "tcg_set_graph_edges": (C.c_int, [vp, vp, i64, i32]),
    "tcg_get_graph_csr": (C.c_int, [vp, P(i32), P(i64), vp, vp]),
    "tcg_set_rejection_limit": (C.c_int, [vp, u64]),
    "tcg_time_colorings": (C.c_int, [vp, u64, C.c_int, C.c_int, vp, P(TcgTiming)]),
    "tcg_kernel_launches": (i64, [vp]),
    "tcg_shard_bounds": (C.c_int, [i32, vp, C.c_int, vp]),
    "tcg_set_shard_device": (C.c_int, [vp, C.c_int, C.c_int, vp, vp]),
    "tcg_set_shard_host": (C.c_int, [vp, C.c_int, C.c_int, vp, vp]),
    "tcg_nccl_unique_id": (C.c_int, [vp]),
    "tcg_create_multi": (C.c_int, [vp, vp, C.c_int, P(vp)]),
    "tcg_loopback_create": (C.c_int, [C.c_int, P(vp)]),
    "tcg_loopback_destroy": (None, [vp]),
    "tcg_set_shard_loopback": (C.c_int, [vp, C.c_int, vp]),
    "tcg_device_count_of": (C.c_int, [vp]),
    "tcg_set_shard_nccl": (C.c_int, [vp, C.c_int, C.c_int, vp]),
}

# int (*)(void* user, const void* send, size_t bytes, void* recv)
ALLGATHER_FN = C.CFUNCTYPE(C.c_int, C.c_void_p, C.c_void_p, C.c_size_t, C.c_void_p)

for _name, (_res, _args) in _SIGS.items():
    _f = getattr(lib, _name)
    _f.restype = _res
    _f.argtypes = _args


def header_symbols() -> list[str]:
    """Every function declared in include/tcg.h."""
    text = open(HEADER).read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(tcg_[a-z_0-9]+)\s*\(", text)))


class TcgError(Exception):
    """Base for status codes other than TCG_OK."""


class InvalidArgument(TcgError, ValueError):
    """TCG_EINVAL: the reference's std::invalid_argument."""


class ParseError(InvalidArgument):
    """TCG_EPARSE: the reference's treecount::parse_error (graph / template input).
    (A subclass of InvalidArgument so callers catching either see both.)"""


class MemoryBudgetError(TcgError, RuntimeError):
    """TCG_ERESOURCE: memory_budget_error (engines.hpp:37-44) or device OOM."""

    def __init__(self, msg):
        super().__init__(msg)
        m = re.search(r"need (\d+) bytes", msg)
        self.required_bytes = int(m.group(1)) if m else None


class CudaError(TcgError, RuntimeError):
    """TCG_ECUDA."""


class NonFiniteError(TcgError, ArithmeticError):
    """TCG_ENONFINITE: rooted total overflowed fp64."""


class LogicError(TcgError, RuntimeError):
    """TCG_ELOGIC: std::logic_error."""


_ERR = {TCG_EINVAL: InvalidArgument, TCG_EPARSE: ParseError, TCG_ERESOURCE: MemoryBudgetError, TCG_ECUDA: CudaError,
        TCG_ENONFINITE: NonFiniteError, TCG_ELOGIC: LogicError}


def check(status: int) -> None:
    if status != TCG_OK:
        msg = (lib.tcg_last_error() or b"").decode()
        raise _ERR.get(status, TcgError)(msg or f"tcg status {status}")
