"""Host-side plumbing for one-worker-per-GPU runs (torchrun + NCCL).

torch.distributed (any backend; gloo is enough) is only the side channel
that carries the 128-byte NCCL unique id and the per-step timing maxima;
every data-path collective is NCCL inside libdbfs (csrc/dist.cu).
"""

from __future__ import annotations

import os

import numpy as np


def env_world():
    """(world, rank, local_rank) from the torchrun environment."""
    return (int(os.environ.get("WORLD_SIZE", "1")), int(os.environ.get("RANK", "0")),
            int(os.environ.get("LOCAL_RANK", "0")))


def edge_slice(m: int, nranks: int, rank: int) -> tuple[int, int]:
    """Contiguous slice [lo, hi) of the global edge order owned by `rank`
    (csrc/build.cu uses the same split for generated edges): concatenating
    the slices in rank order restores the reference's edge order, which keeps
    every CSR row in the reference's neighbour order."""
    per = -(-m // nranks) if nranks else m
    lo = min(m, per * rank)
    return lo, min(m, lo + per)


def broadcast_bytes(payload: bytes | None, tdist, src: int = 0) -> bytes:
    """Broadcast a small byte string (the NCCL unique id) over torch.distributed."""
    box = [payload if tdist.get_rank() == src else None]
    tdist.broadcast_object_list(box, src=src)
    return box[0]


def max_over_ranks(values, tdist) -> np.ndarray:
    """Element-wise max over ranks (per-step times: a step lasts as long as its slowest rank)."""
    import torch
    t = torch.tensor(np.asarray(values, dtype=np.float64))
    tdist.all_reduce(t, op=tdist.ReduceOp.MAX)
    return t.numpy()


def weak_scale(base_scale: int, world: int) -> int:
    """Weak scaling keeps 2^base_scale vertices per GPU: scale = base + log2(world)."""
    if world & (world - 1):
        raise ValueError("weak scaling needs a power-of-two GPU count")
    return base_scale + world.bit_length() - 1


def init_nccl_context(ctx, tdist):
    """Give a libdbfs Context an NCCL communicator spanning the torch.distributed world."""
    from . import _lib
    rank, world = tdist.get_rank(), tdist.get_world_size()
    uid = broadcast_bytes(_lib.nccl_unique_id() if rank == 0 else None, tdist)
    ctx.init_dist(uid, world, rank)
    return ctx
