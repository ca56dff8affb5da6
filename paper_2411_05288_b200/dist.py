"""Multi-GPU plumbing: one process per GPU (torchrun), vocabulary rows
sharded contiguously over the ranks (VM.cpp:65-80), and the NCCL group of
the C ABI bootstrapped through torch.distributed.

torch.distributed is plumbing only (rendezvous, the unique-id broadcast and
the timing max): every data-path exchange — the [2 x T] stats all-gather of
C1, the dX all-reduce, the loss all-reduce, the input-layer all-reduce — is
an NCCL call inside libvpipe_b200.so on the context's stream.
"""
from __future__ import annotations

import os
from typing import Tuple

import torch
import torch.distributed as dist


def env() -> Tuple[int, int, int]:
    """(rank, world_size, local_rank) from the torchrun environment."""
    return (int(os.environ.get("RANK", "0")), int(os.environ.get("WORLD_SIZE", "1")),
            int(os.environ.get("LOCAL_RANK", "0")))


def shard_rows(V: int, world: int, rank: int) -> Tuple[int, int]:
    """Rows [row_begin, row_end) of shard `rank` (shard_weights, VM.cpp:65-80)."""
    if world < 1:
        raise ValueError("shard_weights: p must be >= 1")
    if V % world != 0:
        raise ValueError("shard_weights: V not divisible by p")
    rows = V // world
    return rank * rows, (rank + 1) * rows


def broadcast_bytes(payload: bytes | None, src: int = 0) -> bytes:
    """Broadcast a small byte string from `src` over the default process group."""
    obj = [payload]
    dist.broadcast_object_list(obj, src=src)
    return obj[0]


def init_comm(ctx) -> None:
    """Create the context's NCCL group: rank 0 makes the unique id, every rank joins."""
    rank, world = dist.get_rank(), dist.get_world_size()
    uid = broadcast_bytes(ctx.unique_id() if rank == 0 else None)
    ctx.comm_init(world, rank, uid)


def max_over_ranks(x: float, device=None) -> float:
    """Max of a host scalar over all ranks (step time is the slowest rank's)."""
    if not dist.is_initialized() or dist.get_world_size() == 1:
        return x
    t = torch.tensor([x], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())
