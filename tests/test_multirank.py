"""world_size-2 gloo tests of bench.py's multi-rank plumbing (CPU).

The N>1 path is replicas: every rank runs its own colorings (seed offset by
rank), timing is reduced with MAX over ranks, value = max time / (N*K)."""
import os
import socket

import pytest
import torch.multiprocessing as mp


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank),
                      WORLD_SIZE=str(world), LOCAL_RANK=str(rank))
    import bench
    r, w, local, dist = bench.dist_init()
    assert (r, w) == (rank, world) and dist.get_backend() == "gloo"
    mx = bench.allreduce_max(dist, float(10 + rank * 5), local)
    bench.barrier(dist, local)
    seeds = bench.rank_seeds(rank, warmup=3, steps=5)
    q.put((rank, mx, seeds))
    dist.destroy_process_group()


def test_two_rank_replicas_gloo():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    out = sorted(q.get(timeout=120) for _ in procs)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert [o[1] for o in out] == [15.0, 15.0]          # max over ranks
    s0, s1 = out[0][2], out[1][2]
    assert not set(s0) & set(s1)                          # disjoint colorings per rank
    assert len(s0) == len(s1) == 8


def test_single_rank_defaults():
    import bench
    os.environ.pop("WORLD_SIZE", None)
    r, w, local, dist = bench.dist_init()
    assert (r, w, dist) == (0, 1, None)
    assert bench.allreduce_max(None, 3.5, 0) == 3.5
    assert bench.rank_seeds(0, 3, 2) == [1, 2, 3, 4, 5]
