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


def init_comm(ctx, loopback: bool = False) -> None:
    """Create the context's collective group: rank 0 makes the id, every rank
    joins.  NCCL by default; loopback=True joins the library's loopback
    backend instead (ranks may share a GPU: dry runs of N ranks on fewer GPUs)."""
    rank, world = dist.get_rank(), dist.get_world_size()
    mk = ctx.loopback_id if loopback else ctx.unique_id
    uid = broadcast_bytes(mk() if rank == 0 else None)
    ctx.comm_init(world, rank, uid)


def max_over_ranks(x: float, device=None) -> float:
    """Max of a host scalar over all ranks (step time is the slowest rank's)."""
    if not dist.is_initialized() or dist.get_world_size() == 1:
        return x
    t = torch.tensor([x], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


# ---------------------------------------------------------------------------
# One process driving a whole group (C++-style single-process multi-rank):
# contexts on distinct GPUs get NCCL, contexts sharing a GPU the loopback
# backend (vp_comm_init_all).  Each rank is then driven from its own host
# thread, on its own stream (ctypes releases the GIL during library calls).
# ---------------------------------------------------------------------------
def local_group(p: int, devices=None):
    """p contexts (rank k on devices[k], default: all on the current GPU),
    each on a fresh stream, joined into one group."""
    from . import vocab_math as vm
    devices = list(devices) if devices is not None else [torch.cuda.current_device()] * p
    if len(devices) != p:
        raise ValueError("local_group: one device per rank")
    ctxs = []
    for d in devices:
        with torch.cuda.device(d):
            s = torch.cuda.Stream(d)
            with torch.cuda.stream(s):
                ctxs.append(vm.Context(d))
    vm.init_group(ctxs)
    return ctxs


def run_ranks(ctxs, fn):
    """Runs fn(rank, ctx) for every rank concurrently (one thread per rank, on
    the rank's device and stream); returns the results in rank order and
    re-raises the first rank's exception."""
    import threading
    out = [None] * len(ctxs)
    err = [None] * len(ctxs)

    def body(k):
        c = ctxs[k]
        try:
            with torch.cuda.device(c.device), torch.cuda.stream(c.stream):
                out[k] = fn(k, c)
        except BaseException as e:  # noqa: BLE001 - reported to the caller
            err[k] = e

    th = [threading.Thread(target=body, args=(k,)) for k in range(len(ctxs))]
    for t in th:
        t.start()
    for t in th:
        t.join()
    for e in err:
        if e is not None:
            raise e
    return out
