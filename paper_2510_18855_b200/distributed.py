"""Token-sharded data parallelism for the IcePop objective.

Rank r owns the contiguous global token range [start_r, end_r) of the packed batch;
sequences may straddle ranks. ``cu_seqlens``, ``group_offsets`` and the advantages are
replicated, so every rank computes the exact per-token weight
w_t = 1/(n_groups * G_g * |y_i|) (objective.py:215) of its own tokens with no exchange.
The only collectives are the ones the objective really needs:

* ``allreduce_stats`` -- the fp64 partial sums (J, popped / token counts, entropy and
  log-prob sums, KL) summed across ranks, and the device error word OR-ed;
* ``allreduce_grad``  -- dW summed across ranks, in buckets on a side stream so it can
  overlap later work (dHidden stays rank-local).

All of it is plain ``torch.distributed`` (NCCL on the GPU box, gloo in the CPU tests).
"""

from __future__ import annotations

import torch
import torch.distributed as dist

from . import _lib
from .loss import PackedBatch


def shard_range(n_tokens: int, world: int, rank: int, align: int = 1) -> tuple[int, int]:
    """Contiguous [start, end) of rank `rank`; sizes differ by at most `align` tokens."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError("invalid rank/world")
    units = (n_tokens + align - 1) // align
    base, extra = divmod(units, world)
    start_u = rank * base + min(rank, extra)
    end_u = start_u + base + (1 if rank < extra else 0)
    return min(n_tokens, start_u * align), min(n_tokens, end_u * align)


def shard_batch(hidden: torch.Tensor, batch: PackedBatch, rank: int, world: int, align: int = 1):
    """This rank's rows of hidden and per-token tensors; replicated metadata unchanged."""
    n = hidden.shape[0]
    if batch.token_offset != 0:
        raise ValueError("shard_batch expects the full (unsharded) batch")
    s, e = shard_range(n, world, rank, align)
    local = PackedBatch(
        tokens=batch.tokens[s:e],
        lp_train_old=batch.lp_train_old[s:e],
        lp_infer_old=batch.lp_infer_old[s:e],
        cu_seqlens=batch.cu_seqlens,
        group_offsets=batch.group_offsets,
        advantages=batch.advantages,
        rewards=batch.rewards,
        token_offset=s,
    )
    return hidden[s:e], local


def allreduce_stats(stats: torch.Tensor, group=None) -> torch.Tensor:
    """Sum the fp64 statistics across ranks; OR the error bits (include/icepop.h).

    The error word cannot be summed (two ranks with bit 1 would read as bit 2), so it is
    expanded into one 0/1 slot per bit and reduced with MAX. Works in place on `stats`.
    """
    if not dist.is_available() or not dist.is_initialized() or dist.get_world_size(group) == 1:
        return stats
    dev = stats.device
    nbits = 4
    err = stats[_lib.STAT_ERRORS].to(torch.int64)
    bits = ((err >> torch.arange(nbits, device=dev)) & 1).to(torch.float64)
    body = stats[: _lib.STAT_ERRORS].clone()
    dist.all_reduce(body, op=dist.ReduceOp.SUM, group=group)
    dist.all_reduce(bits, op=dist.ReduceOp.MAX, group=group)
    word = (bits.to(torch.int64) << torch.arange(nbits, device=dev)).sum().to(torch.float64)
    stats[: _lib.STAT_ERRORS] = body
    stats[_lib.STAT_ERRORS] = word
    return stats


def allreduce_grad(grad: torch.Tensor, group=None, bucket_bytes: int = 256 << 20, stream=None):
    """Sum dW across ranks in flat buckets; returns the work handles (async) or None.

    With `stream` given the buckets are issued on that stream after it waits for the
    current one, so the reduction overlaps whatever the caller launches next; call
    ``wait_grad(handles)`` before reading `grad`.
    """
    if not dist.is_available() or not dist.is_initialized() or dist.get_world_size(group) == 1:
        return None
    flat = grad.view(-1)
    per = max(1, bucket_bytes // flat.element_size())
    handles = []
    ctx = torch.cuda.stream(stream) if (stream is not None and grad.is_cuda) else None
    if ctx is not None:
        stream.wait_stream(torch.cuda.current_stream(grad.device))
        ctx.__enter__()
    try:
        for s in range(0, flat.numel(), per):
            handles.append(dist.all_reduce(flat[s:s + per], op=dist.ReduceOp.SUM, group=group, async_op=True))
    finally:
        if ctx is not None:
            ctx.__exit__(None, None, None)
    return handles


def wait_grad(handles) -> None:
    for h in handles or ():
        h.wait()
