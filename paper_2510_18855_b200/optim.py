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


class ShardedAscent:
    """ZeRO-1 ascent step fed by the fused dW reduce-scatter (objective.py:301-326).

    dW rows (V for a [V,d] weight, d for [d,V]) are owned in contiguous shards of ``shard_rows``
    rows, the layout of ``icepop_bwd_bf16_rs``: K5's epilogue stores every dW row into its owner's
    slot over NVLink, so no reduce-scatter runs after the backward. ``step()`` then, per owned
    shard: folds the slots in rank order (the summed dW rows), runs the fp32 ascent update with
    momentum on the master shard and writes its bf16 copy (one kernel, ``sgd_update_``), and
    all-gathers the bf16 shards into the replicated weight the GEMMs read (in place).

    ``emulate=True`` runs ``world`` ranks' shards in this process with the slot buffers in local
    memory (tests on one GPU: ranks take turns, no kernel waits on another); otherwise the group's
    ranks exchange slot handles (``distributed.PeerSlots``) and gather over the group.
    """

    def __init__(self, weight: torch.Tensor, lr: float, beta: float | None = None, group=None,
                 world: int | None = None, emulate: bool = False, _ops=None, _update_fn=None):
        if weight.dtype != torch.bfloat16 or weight.dim() != 2 or not weight.is_contiguous():
            raise ValueError("weight must be a contiguous 2-D bf16 tensor (the replicated GEMM copy)")
        if not lr > 0:
            raise ValueError("learning rate must be positive")
        if beta is not None and not 0.0 <= beta < 1.0:
            raise ValueError("momentum beta must be in [0, 1)")
        self.weight, self.lr, self.beta, self.group, self.emulate = weight, float(lr), beta, group, emulate
        self._update_fn = _update_fn  # tests on CPU: a torch stand-in for the CUDA update
        self.rows, self.row_len = weight.shape
        if emulate:
            self.world, self.rank = int(world or 1), 0
            owned = range(self.world)
        else:
            self.world = dist.get_world_size(group) if dist.is_initialized() else 1
            self.rank = dist.get_rank(group) if dist.is_initialized() else 0
            owned = [self.rank]
        per = -(-self.rows // self.world)
        while (per * self.row_len) % 4:
            per += 1
        self.shard_rows = per
        self.shard_elems = per * self.row_len
        dev = weight.device
        flat = weight.reshape(-1)
        self.master, self.velocity, self.grad, self.out_bf16 = {}, {}, {}, {}
        for r in owned:
            m = torch.zeros(self.shard_elems, dtype=torch.float32, device=dev)
            n = self._valid(r)
            if n:
                m[:n] = flat[r * self.shard_elems:r * self.shard_elems + n].float()
            self.master[r] = m
            self.velocity[r] = torch.zeros_like(m) if beta is not None else None
            self.grad[r] = torch.empty_like(m)
            self.out_bf16[r] = torch.empty(self.shard_elems, dtype=torch.bfloat16, device=dev)
        if emulate:
            self._slots = {o: torch.zeros(self.world * self.shard_elems, dtype=torch.float32, device=dev)
                           for o in owned}
            self._peer = None
        else:
            from .distributed import PeerSlots

            self._slots = None
            self._peer = PeerSlots(self.shard_rows, self.row_len, group, _ops=_ops)

    def _valid(self, r: int) -> int:
        return max(0, min(self.shard_elems, self.rows * self.row_len - r * self.shard_elems))

    def shard_of(self, t: torch.Tensor, r: int) -> torch.Tensor:
        """Rank r's rows of a weight-shaped tensor, flat (its valid part)."""
        n = self._valid(r)
        return t.reshape(-1)[r * self.shard_elems:r * self.shard_elems + n]

    def velocity_shard(self, r: int | None = None) -> torch.Tensor:
        r = self.rank if r is None else r
        return self.velocity[r][:self._valid(r)]

    def rs_target(self, rank: int | None = None) -> _lib.RsTarget:
        """The icepop_rs_target rank `rank` passes to icepop_bwd_bf16_rs (loss.icepop_bwd_reduce_scatter)."""
        if self._peer is not None:
            return self._peer.target()
        t = _lib.RsTarget(world=self.world, rank=self.rank if rank is None else rank, shard_rows=self.shard_rows)
        for o in range(self.world):
            t.slots[o] = self._slots[o].data_ptr()
        return t

    def _update_shard(self, r: int) -> None:
        n = self._valid(r)
        if n and self._update_fn is not None:
            v = self.velocity[r][:n] if self.velocity[r] is not None else None
            self._update_fn(self.master[r][:n], self.grad[r][:n], v, self.out_bf16[r][:n])
        elif n:
            sgd_update_(self.master[r][:n], self.grad[r][:n], self.lr,
                        self.velocity[r][:n] if self.velocity[r] is not None else None,
                        self.beta if self.beta is not None else 0.0, self.out_bf16[r][:n])

    def step(self) -> torch.Tensor:
        """Fold -> update -> gather; returns the (updated in place) bf16 weight."""
        from .loss import _stream

        from .distributed import stream_barrier

        lib = _lib.load()
        flat = self.weight.reshape(-1)
        if self._peer is not None and self.world > 1:
            stream_barrier(self.group)  # every rank's K5 has stored its rows into the owners' slots
        for r in self.master:
            if self._peer is not None:
                self._peer.fold(self.grad[r])
            else:
                _lib.check(lib.icepop_rs_fold(self._slots[r].data_ptr(), self.world, self.shard_elems,
                                              self.grad[r].data_ptr(), _stream(self.weight.device)))
            self._update_shard(r)
        if self.emulate or self.world == 1:
            for r in self.master:
                n = self._valid(r)
                flat[r * self.shard_elems:r * self.shard_elems + n].copy_(self.out_bf16[r][:n])
            return self.weight
        gathered = torch.empty(self.world * self.shard_elems, dtype=torch.bfloat16, device=self.weight.device)
        if dist.get_backend(self.group) == "gloo":  # CPU collectives (tests)
            parts = [torch.empty(self.shard_elems, dtype=torch.bfloat16) for _ in range(self.world)]
            dist.all_gather(parts, self.out_bf16[self.rank].cpu(), group=self.group)
            gathered.copy_(torch.cat(parts))
        else:
            dist.all_gather_into_tensor(gathered, self.out_bf16[self.rank], group=self.group)
        flat.copy_(gathered[:flat.numel()])
        return self.weight

    def close(self) -> None:
        if self._peer is not None:
            self._peer.close()
            self._peer = None
