"""Batch-mode data parallelism for tensorized conv layers.

`b` appears only in the layer input X and the output of every layer expression
(reference layers.cpp:159-176, 180-318), so each sample's output depends only on
its own X slice and the (replicated) factors.  One process per GPU:
  * X and dY are split contiguously along `b` (shard_batch),
  * factors are replicated (same SplitMix64 seeds on every rank),
  * forward and backward run locally through libce,
  * the only collective is a SUM all-reduce of the factor gradients
    (allreduce_factor_grads), NCCL over NVLink on B200, gloo in the CPU tests.
Input (X) gradients stay sharded.  The compute function is pluggable so the
same host logic is exercised by the gloo tests with the FP64 oracle on CPU.
"""
from __future__ import annotations

from typing import Callable, List, Optional, Sequence, Tuple

import torch
import torch.distributed as dist


def shard_range(batch: int, rank: int, world: int) -> Tuple[int, int]:
    """Contiguous [lo, hi) slice of the batch owned by `rank` (earlier ranks take the remainder)."""
    base, rem = divmod(batch, world)
    lo = rank * base + min(rank, rem)
    return lo, lo + base + (1 if rank < rem else 0)


def shard_batch(x: torch.Tensor, rank: int, world: int, axis: int = 0) -> torch.Tensor:
    lo, hi = shard_range(x.shape[axis], rank, world)
    return x.narrow(axis, lo, hi - lo).contiguous()


def allreduce_factor_grads(grads: Sequence[Optional[torch.Tensor]], group=None,
                           skip: Sequence[int] = (0,)) -> List[Optional[torch.Tensor]]:
    """SUM all-reduce of every gradient except those in `skip` (the batch-sharded X).

    Factor gradients of one layer are flattened into a single buffer so the layer
    costs one collective (bucketed like DDP), then scattered back in place."""
    out, work = allreduce_factor_grads_async(grads, group, skip)
    if work is not None:
        work.wait()
    return out


def allreduce_factor_grads_async(grads: Sequence[Optional[torch.Tensor]], group=None,
                                 skip: Sequence[int] = (0,)):
    """As allreduce_factor_grads, but returns (views, work) without ordering the caller's
    stream after the collective: the next layer's backward overlaps it, and
    `work.wait()` (stream-side, no host sync) orders whatever reads the reduced
    gradients.  work is None when there is nothing to reduce."""
    if not dist.is_available() or not dist.is_initialized() or dist.get_world_size(group) == 1:
        return list(grads), None
    idx = [i for i, g in enumerate(grads) if g is not None and i not in skip]
    if not idx:
        return list(grads), None
    flat = torch.cat([grads[i].reshape(-1) for i in idx])
    work = dist.all_reduce(flat, op=dist.ReduceOp.SUM, group=group, async_op=True)
    out = list(grads)
    pos = 0
    for i in idx:
        n = grads[i].numel()
        out[i] = flat[pos:pos + n].view_as(grads[i])
        pos += n
    return out, work


def init_ce_comm(ctx, group=None) -> None:
    """Join `ctx` (a device.Context, one per GPU) to a libce NCCL communicator over the
    ranks of the torch.distributed group: rank 0 creates the unique id, a broadcast
    (any backend) hands it out, then ce_ctx_init_comm."""
    from .device import nccl_unique_id
    rank, world = dist.get_rank(group), dist.get_world_size(group)
    obj = [nccl_unique_id() if rank == 0 else None]
    dist.broadcast_object_list(obj, src=0, group=group)
    ctx.init_comm(world, rank, obj[0])


def allreduce_factor_grads_ce(ctx, grads: Sequence[Optional[torch.Tensor]],
                              skip: Sequence[int] = (0,)) -> List[Optional[torch.Tensor]]:
    """Factor-gradient SUM through libce's communicator (ce_allreduce_grads): one NCCL
    group per layer on the context's comm stream, in place, overlapping whatever is
    queued next on the context stream; call ctx.comm_wait() before reading the grads."""
    ctx.allreduce_grads([g for i, g in enumerate(grads) if g is not None and i not in skip])
    return list(grads)


def data_parallel_step(inputs: Sequence[torch.Tensor], dout: torch.Tensor, rank: int, world: int,
                       fwd_bwd: Callable[[List[torch.Tensor], torch.Tensor], Tuple[torch.Tensor, List[torch.Tensor]]],
                       group=None):
    """Shard X and dY along b, run `fwd_bwd` on the local shard, all-reduce factor grads.

    Returns (local output shard, [local dX shard, reduced factor grads...])."""
    xs = [shard_batch(inputs[0], rank, world)] + list(inputs[1:])
    dy = shard_batch(dout, rank, world)
    out, grads = fwd_bwd(xs, dy)
    return out, allreduce_factor_grads(grads, group)
