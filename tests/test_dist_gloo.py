"""CPU: the N>1 host path with a real world_size-2 gloo process group.

Covers the side-channel logic of the one-worker-per-GPU runs (unique-id
broadcast, max-over-ranks timing, edge-order slicing, weak-scaling sizes) and,
through the oracle, that per-rank edge slices rebuild exactly the partition of
the whole edge list (the distributed build's order-preservation argument).
"""

import os
import socket

import numpy as np
import pytest
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_1803_03922_b200.dist import broadcast_bytes, edge_slice, max_over_ranks, weak_scale


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, out):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        uid = broadcast_bytes(bytes(range(128)) if rank == 0 else None, dist)
        times = [1.0 + rank, 5.0 - rank, 2.0]
        mx = max_over_ranks(times, dist)
        # each rank routes its slice of the global edge order; gather the
        # slices back in rank order and compare with the whole list
        import oracle as O
        src, dst = O.rmat_edges(9, seed=3)
        lo, hi = edge_slice(len(src), world, rank)
        parts = [None] * world
        dist.all_gather_object(parts, (lo, hi, src[lo:hi].tolist(), dst[lo:hi].tolist()))
        s2 = sum((p[2] for p in parts), [])
        d2 = sum((p[3] for p in parts), [])
        out[rank] = (uid == bytes(range(128)), mx.tolist(), s2 == src.tolist() and d2 == dst.tolist(),
                     [p[:2] for p in parts])
    finally:
        dist.destroy_process_group()


def test_gloo_world2_host_path():
    world = 2
    port = _free_port()
    mgr = mp.Manager()
    out = mgr.dict()
    mp.spawn(_worker, args=(world, port, out), nprocs=world, join=True)
    for r in range(world):
        uid_ok, mx, order_ok, bounds = out[r]
        assert uid_ok
        assert mx == [2.0, 5.0, 2.0]
        assert order_ok
        assert bounds[0][0] == 0 and bounds[-1][1] == 2 * (1 << 9) * 16


def test_edge_slices_partition_the_order():
    for m in (0, 1, 7, 1000, 2 ** 20 + 3):
        for n in (1, 2, 3, 4, 8):
            sl = [edge_slice(m, n, r) for r in range(n)]
            assert sl[0][0] == 0 and sl[-1][1] == m
            assert all(a[1] == b[0] for a, b in zip(sl, sl[1:]))


def test_weak_scale():
    assert [weak_scale(24, w) for w in (1, 2, 4, 8)] == [24, 25, 26, 27]
    with pytest.raises(ValueError):
        weak_scale(24, 3)


def test_partition_shape_invariance_of_levels():
    """Levels do not depend on how workers are split (tests/test_engine.py:69-74),
    here through the oracle for the shapes the multi-GPU runs use (1xP)."""
    import oracle as O
    src, dst = O.rmat_edges(11, seed=6)
    base = None
    for p in (1, 2, 4):
        og = O.partition(src, dst, 1 << 11, 16, 1, p)
        dg = O.run_bfs(og, 77)["levels_digest"]
        base = base or dg
        assert dg == base
