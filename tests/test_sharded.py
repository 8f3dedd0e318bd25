"""Vertex-sharded engine: row shards + all-gathered SpMM panels.

CPU: the shard partition (contiguous, covering, balanced).
GPU: world=1 through the NCCL transport, and world=2 as two processes on ONE
GPU through the host transport (gloo all-gather on the host -- no kernel waits
on another rank), both against the oracle and the unsharded engine.
"""
import os
import socket

import numpy as np
import pytest

import oracle as O
import paper_1903_04395_b200 as T
from conftest import CFG_TEMPLATES, parents_to_edges


def test_shard_bounds_contiguous_and_balanced():
    g = T.generate_rmat(T.RmatSpec(14, 16 << 14, .57, .19, .19, .05, 1))
    deg = np.diff(g.csc_col_ptr)
    avg = deg.mean()
    for world in (1, 2, 3, 4, 8):
        b = T.shard_bounds(g, world)
        assert b[0] == 0 and b[-1] == g.n and np.all(np.diff(b) >= 0)
        w = np.array([deg[b[r]:b[r + 1]].sum() + avg * (b[r + 1] - b[r]) for r in range(world)])
        # no shard exceeds its share by more than the heaviest single row
        assert w.max() <= w.sum() / world + deg.max() + avg + 1


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _get(q, procs, timeout=300):
    """Queue get that fails fast when a worker died instead of waiting."""
    import queue
    import time
    t0 = time.time()
    while time.time() - t0 < timeout:
        try:
            return q.get(timeout=2)
        except queue.Empty:
            if any(p.exitcode not in (None, 0) for p in procs):
                raise AssertionError(f"worker failed: {[p.exitcode for p in procs]}")
    raise AssertionError("timed out waiting for workers")


def _ref(g, parents, seed):
    k = len(parents)
    plan = O.partition(k, parents_to_edges(parents), 0)
    return O.run_iteration(g.n, g.csc_col_ptr, g.csc_rows, plan, O.random_coloring(g.n, k, seed))


def _nccl_world1_worker(port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    import torch
    import torch.distributed as dist
    torch.cuda.set_device(0)
    dist.init_process_group("nccl", rank=0, world_size=1)
    import paper_1903_04395_b200 as TT
    g = TT.generate_rmat(TT.RmatSpec(13, 16 << 13, .57, .19, .19, .05, 3))
    c = TT.Context(0)
    c.set_shard_torch(0, 1)
    c.set_graph(g)
    c.set_template(TT.template_from_parents(CFG_TEMPLATES["cfg2"], 0))
    total, pv, _ = c.run_coloring(5, per_vertex=True)
    totals, est, se, _ = c.estimate(5, 3)
    q.put((total, pv, list(totals)))
    dist.destroy_process_group()


@pytest.mark.gpu
def test_sharded_world1_torch_nccl():
    """The production transport (torch.distributed NCCL, device pointers) at world=1."""
    import torch.multiprocessing as mp
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    p = ctx.Process(target=_nccl_world1_worker, args=(_free_port(), q))
    p.start()
    total, pv, totals = _get(q, [p])
    p.join(timeout=120)
    assert p.exitcode == 0
    g = T.generate_rmat(T.RmatSpec(13, 16 << 13, .57, .19, .19, .05, 3))
    ot, opv, _ = _ref(g, CFG_TEMPLATES["cfg2"], 5)
    assert abs(total - ot) <= 1e-4 * ot
    assert np.max(np.abs(pv - opv) / np.maximum(opv, 1)) <= 1e-4
    assert totals[0] == total


@pytest.mark.gpu
def test_sharded_world1_host():
    g = T.generate_rmat(T.RmatSpec(13, 16 << 13, .57, .19, .19, .05, 3))
    parents = CFG_TEMPLATES["cfg2"]
    c = T.Context(0)
    c.set_shard_host(0, 1, lambda a: a)
    c.set_graph(g)
    c.set_template(T.template_from_parents(parents, 0))
    total, pv, _ = c.run_coloring(5, per_vertex=True)
    ot, opv, _ = _ref(g, parents, 5)
    assert abs(total - ot) <= 1e-4 * ot
    assert np.max(np.abs(pv - opv) / np.maximum(opv, 1)) <= 1e-4
    totals, est, se, _ = c.estimate(5, 3)
    assert totals[0] == total


@pytest.mark.gpu
def test_shard_after_template_replans():
    """set_template before set_shard_*: the template is re-planned for the
    sharded context (no pair layout), so a pair-eligible k=12 template runs."""
    g = T.generate_rmat(T.RmatSpec(11, 48 << 11, .45, .15, .15, .25, 3))
    parents = CFG_TEMPLATES["cfg3"]
    c = T.Context(0)
    c.set_template(T.template_from_parents(parents, 0))
    c.set_shard_host(0, 1, lambda a: a)
    c.set_graph(g)
    total, pv, _ = c.run_coloring(2, per_vertex=True)
    ot, opv, _ = _ref(g, parents, 2)
    assert abs(total - ot) <= 1e-4 * ot
    assert np.max(np.abs(pv - opv) / np.maximum(opv, 1)) <= 1e-4


def _worker(rank, world, port, name, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    import torch
    import torch.distributed as dist
    dist.init_process_group("gloo", rank=rank, world_size=world)

    def allgather(arr):
        t = torch.from_numpy(arr)
        outs = [torch.empty_like(t) for _ in range(world)]
        dist.all_gather(outs, t)
        return torch.cat(outs).numpy()

    import paper_1903_04395_b200 as TT
    g = TT.generate_rmat(TT.RmatSpec(12, 24 << 12, .45, .15, .15, .25, 5))
    c = TT.Context(0)
    c.set_shard_host(rank, world, allgather)
    c.set_graph(g)
    c.set_template(TT.template_from_parents(CFG_TEMPLATES[name], 0))
    total, pv, _ = c.run_coloring(9, per_vertex=True)
    totals, est, se, pve = c.estimate(9, 2, per_vertex=True)
    q.put((rank, total, pv, list(totals), est, pve))
    dist.destroy_process_group()


@pytest.mark.gpu
@pytest.mark.parametrize("name", ["cfg2", "cfg3"])
def test_sharded_two_ranks_host_transport(name):
    import torch.multiprocessing as mp
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, name, q)) for r in range(2)]
    for p in procs:
        p.start()
    out = sorted((_get(q, procs) for _ in procs), key=lambda x: x[0])
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    g = T.generate_rmat(T.RmatSpec(12, 24 << 12, .45, .15, .15, .25, 5))
    parents = CFG_TEMPLATES[name]
    ot, opv, _ = _ref(g, parents, 9)
    for rank, total, pv, totals, est, pve in out:
        assert abs(total - ot) <= 1e-4 * ot
        assert np.max(np.abs(pv - opv) / np.maximum(opv, 1)) <= 1e-4
        assert totals[0] == total
    # both ranks report identical (rank-ordered) results
    assert out[0][1] == out[1][1] and out[0][3] == out[1][3]
    assert np.array_equal(out[0][5], out[1][5])
    # and the sharded result equals the unsharded engine's within fp rounding
    c = T.Context(0)
    c.set_graph(g)
    c.set_template(T.template_from_parents(parents, 0))
    t1, _, _ = c.run_coloring(9)
    assert abs(t1 - out[0][1]) <= 1e-6 * t1


def _nccl_owned_worker(q):
    import paper_1903_04395_b200 as TT
    out = []
    g = TT.generate_rmat(TT.RmatSpec(12, 32 << 12, .45, .15, .15, .25, 6))
    for name in ("cfg2", "cfg3"):
        c = TT.Context(0)
        c.set_shard_nccl(0, 1)  # the library's own communicator (world 1: no exchange)
        c.set_graph(g)
        c.set_template(TT.template_from_parents(CFG_TEMPLATES[name], 0))
        total, pv, _ = c.run_coloring(4, per_vertex=True)
        totals, _, _, _ = c.estimate(4, 2)
        out.append((name, total, pv, list(totals)))
    q.put(out)


@pytest.mark.gpu
def test_sharded_world1_library_nccl():
    """tcg_set_shard_nccl: the library-owned NCCL communicator (dlopen'd NCCL,
    async all-gathers on the comm stream, group g+1 prefetched while group g's
    SpMM runs) -- k=12 has 6+ compressed groups per SpMM, so the double buffer
    and its events are exercised -- against the oracle."""
    import torch.multiprocessing as mp
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    p = ctx.Process(target=_nccl_owned_worker, args=(q,))
    p.start()
    out = _get(q, [p])
    p.join(timeout=120)
    assert p.exitcode == 0
    g = T.generate_rmat(T.RmatSpec(12, 32 << 12, .45, .15, .15, .25, 6))
    for name, total, pv, totals in out:
        ot, opv, _ = _ref(g, CFG_TEMPLATES[name], 4)
        assert abs(total - ot) <= 1e-4 * ot, name
        assert np.max(np.abs(pv - opv) / np.maximum(opv, 1)) <= 1e-4, name
        assert totals[0] == total


def test_nccl_unique_id_on_host():
    """The library resolves NCCL at run time (dlopen) and produces the 128-byte
    bootstrap id rank 0 hands to the other ranks (tcg_nccl_unique_id) -- host
    only, no GPU needed; two ids differ (fresh bootstrap each call)."""
    import ctypes as C
    from paper_1903_04395_b200 import _native as N
    from paper_1903_04395_b200 import treecount as TC
    TC._nccl_env()
    a, b = (C.c_uint8 * N.TCG_NCCL_ID_BYTES)(), (C.c_uint8 * N.TCG_NCCL_ID_BYTES)()
    assert N.lib.tcg_nccl_unique_id(a) == 0, N.lib.tcg_last_error()
    assert N.lib.tcg_nccl_unique_id(b) == 0
    assert any(bytes(a)) and bytes(a) != bytes(b)
    assert N.lib.tcg_nccl_unique_id(None) == N.TCG_EINVAL


@pytest.mark.gpu
@pytest.mark.parametrize("world", [2, 3])
@pytest.mark.parametrize("name", ["cfg2", "cfg3"])
def test_sharded_loopback_world_n(world, name):
    """world in-process ranks on ONE GPU through the loopback transport, which
    has the NCCL transport's async contract: the rooted SpMM's panels are
    all-gathered on the communication stream, group g+1 while group g's
    gathers run (double buffer, events only).  Every rank's context runs in
    its own thread; results match the oracle and are identical across ranks."""
    import threading
    g = T.generate_rmat(T.RmatSpec(12, 24 << 12, .45, .15, .15, .25, 5))
    parents = CFG_TEMPLATES[name]
    hub = T.LoopbackHub(world)
    ctxs = []
    for r in range(world):
        c = T.Context(0)
        c.set_shard_loopback(r, hub)
        c.set_graph(g)
        c.set_template(T.template_from_parents(parents, 0))
        ctxs.append(c)
    out, err = [None] * world, []

    def rank_main(r):
        try:
            total, pv, _ = ctxs[r].run_coloring(9, per_vertex=True)
            totals, est, se, pve = ctxs[r].estimate(9, 2, per_vertex=True)
            out[r] = (total, pv, list(totals), pve)
        except Exception as ex:  # noqa: BLE001
            err.append(ex)
    th = [threading.Thread(target=rank_main, args=(r,)) for r in range(world)]
    for t in th:
        t.start()
    for t in th:
        t.join(timeout=600)
    assert not err, err
    ot, opv, _ = _ref(g, parents, 9)
    for total, pv, totals, pve in out:
        assert abs(total - ot) <= 1e-4 * ot
        assert np.max(np.abs(pv - opv) / np.maximum(opv, 1)) <= 1e-4
        assert totals[0] == total
    assert all(o[0] == out[0][0] and o[2] == out[0][2] for o in out)
    assert all(np.array_equal(o[3], out[0][3]) for o in out)
