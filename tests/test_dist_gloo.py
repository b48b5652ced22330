"""Multi-process (world_size 2, gloo, CPU) checks of bench.py's distributed host
logic: max-over-ranks timing and per-rank replica inputs."""
from __future__ import annotations

import os
import socket

import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp


def _free_port() -> int:
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    import sys
    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    import bench
    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank, world_size=world)
    try:
        ms = 10.0 + 5.0 * rank                       # rank 1 is the slow one
        got = bench.max_over_ranks(ms, world)
        seeds = bench.replica_seeds(rank)
        obj = [None] * world
        dist.all_gather_object(obj, seeds)
        q.put((rank, got, obj))
    finally:
        dist.destroy_process_group()


@pytest.mark.timeout(120)
def test_max_over_ranks_and_replica_seeds():
    world = 2
    port = _free_port()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=100) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    for rank, got, seeds in res:
        assert got == 15.0                           # max over ranks, on every rank
        assert len(set(seeds)) == world              # independent replicas per rank


def test_single_rank_passthrough():
    import bench
    assert bench.max_over_ranks(3.5, 1) == 3.5


def test_grid_layout_roundtrip():
    """2-D block-cyclic host layout: default grids, local shapes,
    scatter/gather round trip, and that every tile lands on rank (I % P, J % Q)."""
    import paper_1907_01063_b200 as sc
    assert [sc.dist_grid(g) for g in (1, 2, 4, 8, 6, 3)] == [(1, 1), (1, 2), (2, 2), (2, 4), (2, 3), (1, 3)]
    B = sc.DIST_BLOCK
    for n, P, Q in [(1792, 2, 2), (2304, 2, 4), (768, 4, 1), (1280, 3, 2)]:
        T = n // B
        A = torch.arange(n * n, dtype=torch.float64).reshape(n, n)
        locs = [sc.dist_scatter2(A, P, Q, r // Q, r % Q) for r in range(P * Q)]
        assert sum(l.numel() for l in locs) == n * n
        for r, l in enumerate(locs):
            p, q = divmod(r, Q)
            assert tuple(l.shape) == sc.dist_local_shape(n, P, Q, p, q)
            for li, I in enumerate(range(p, T, P)):
                for lj, J in enumerate(range(q, T, Q)):
                    assert l[li * B, lj * B] == A[I * B, J * B]
        assert torch.equal(sc.dist_gather2(locs, n, P, Q), A)
