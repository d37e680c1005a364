"""The step after the loss: the reference's ascent update on the device.

``sgd_update_`` restates objective.py:301-326 (``sgd_update`` / ``momentum_update``) as one
CUDA kernel over an fp32 master copy (with an optional bf16 copy the lm_head GEMMs read),
keeping the reference's contract: lr <= 0 -> ValueError, beta outside [0, 1) -> ValueError,
non-finite weights -> NumericError (objective.py:309-310).

``sharded_sgd_step`` is the ZeRO-style data-parallel form: reduce-scatter dW (half the
traffic of an all-reduce), update this rank's shard of the master weights and velocity,
all-gather the bf16 weights.
"""

from __future__ import annotations

import torch
import torch.distributed as dist

from . import _lib
from .loss import _on_device


@_on_device
def sgd_update_(weight: torch.Tensor, grad: torch.Tensor, lr: float, velocity: torch.Tensor | None = None,
                beta: float = 0.9, weight_bf16: torch.Tensor | None = None, check: bool = True) -> torch.Tensor:
    """In place: v = beta v + g (if velocity) else v = g; weight += lr v (gradient ASCENT)."""
    from .loss import _lib_for, _stream

    lib = _lib_for(weight)
    for name, t in (("weight", weight), ("grad", grad), ("velocity", velocity)):
        if t is not None and (t.dtype != torch.float32 or not t.is_contiguous()):
            raise ValueError(f"{name} must be a contiguous float32 tensor")
    if grad.shape != weight.shape or (velocity is not None and velocity.shape != weight.shape):
        raise ValueError("gradient shape does not match parameters")
    if weight_bf16 is not None and (weight_bf16.dtype != torch.bfloat16 or weight_bf16.numel() != weight.numel()
                                    or not weight_bf16.is_contiguous()):
        raise ValueError("weight_bf16 must be a contiguous bf16 tensor with the weight's size")
    stats = torch.zeros(_lib.NSTATS, dtype=torch.float64, device=weight.device) if check else None
    _lib.check(lib.icepop_sgd_update_f32(weight.data_ptr(), grad.data_ptr(), _lib.ptr(velocity),
                                         _lib.ptr(weight_bf16), weight.numel(), float(lr), float(beta),
                                         _lib.ptr(stats), _stream(weight.device)))
    if check:
        _lib.check(lib.icepop_finish(stats.data_ptr(), _stream(weight.device)))
    return weight


def shard_bounds(numel: int, world: int, rank: int) -> tuple[int, int, int]:
    """(start, end, padded shard size) of rank's contiguous shard of a flat parameter."""
    per = -(-numel // world)
    return min(numel, rank * per), min(numel, (rank + 1) * per), per


def sharded_sgd_step(grad_full: torch.Tensor, master_shard: torch.Tensor, weight_bf16_full: torch.Tensor, lr: float,
                     velocity_shard: torch.Tensor | None = None, beta: float = 0.9, group=None, update_fn=None):
    """ZeRO-1 step: reduce-scatter dW, ascend this rank's shard, all-gather bf16 weights.

    grad_full: this rank's partial dW (any shape, fp32); master_shard / velocity_shard: this
    rank's padded shard (fp32, size shard_bounds(...)[2]); weight_bf16_full: the replicated
    bf16 weights, overwritten with the gathered update. `update_fn(master, grad, velocity,
    out_bf16)` defaults to the CUDA kernel (tests substitute a reference on CPU).
    """
    world = dist.get_world_size(group)
    rank = dist.get_rank(group)
    numel = grad_full.numel()
    _, _, per = shard_bounds(numel, world, rank)
    flat = grad_full.reshape(-1)
    if per * world != numel:
        flat = torch.nn.functional.pad(flat, (0, per * world - numel))
    gshard = torch.empty(per, dtype=flat.dtype, device=flat.device)
    dist.reduce_scatter_tensor(gshard, flat.contiguous(), op=dist.ReduceOp.SUM, group=group)
    out_bf16 = torch.empty(per, dtype=torch.bfloat16, device=flat.device)
    if update_fn is None:
        sgd_update_(master_shard, gshard, lr, velocity_shard, beta, out_bf16)
    else:
        update_fn(master_shard, gshard, velocity_shard, out_bf16)
    gathered = torch.empty(per * world, dtype=torch.bfloat16, device=flat.device)
    dist.all_gather_into_tensor(gathered, out_bf16, group=group)
    weight_bf16_full.view(-1).copy_(gathered[:numel])
    return weight_bf16_full
