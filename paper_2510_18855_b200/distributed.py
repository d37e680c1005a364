"""Token-sharded data parallelism for the IcePop objective.

Rank r owns the contiguous global token range [start_r, end_r) of the packed batch;
sequences may straddle ranks. ``cu_seqlens``, ``group_offsets`` and the advantages are
replicated, so every rank computes the exact per-token weight
w_t = 1/(n_groups * G_g * |y_i|) (objective.py:215) of its own tokens with no exchange.
The only collectives are the ones the objective really needs:

* ``allreduce_stats`` -- the fp64 partial sums (J, popped / token counts, entropy and
  log-prob sums, KL) summed across ranks, and the device error word OR-ed;
* ``allreduce_grad``  -- dW summed across ranks, in buckets on a side stream so it can
  overlap later work (dHidden stays rank-local);
* ``PeerSlots``       -- the fused alternative: K5's epilogue stores every dW row straight
  into its owner rank's slot over NVLink (CUDA IPC peer memory), so the reduce-scatter
  overlaps the GEMM tile by tile; the owner then folds the slots in rank order.

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
        calib=batch.calib[s:e] if batch.calib is not None else None,
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


def stream_barrier(group=None, device=None) -> None:
    """Cross-rank barrier ordered on the current stream (a 1-element NCCL all-reduce): work
    queued after it starts only when every rank has finished the work queued before it."""
    if not dist.is_available() or not dist.is_initialized() or dist.get_world_size(group) == 1:
        return
    if device is None:
        device = "cpu" if dist.get_backend(group) == "gloo" else torch.cuda.current_device()
    if str(device) == "cpu" and torch.cuda.is_available() and torch.cuda.is_initialized():
        # a CPU collective does not wait for the CUDA stream: drain it first, so the barrier
        # still means "this rank's queued device work (e.g. the fold reading the slots) is done"
        torch.cuda.current_stream().synchronize()
    t = torch.zeros(1, device=device)
    dist.all_reduce(t, group=group)


class PeerSlots:
    """Peer-mapped slot buffers for the fused dW reduce-scatter (include/icepop.h).

    Collective constructor: every rank allocates world x shard_rows x row_len fp32 (its slot
    buffer), exports a CUDA IPC handle, all-gathers the handles and imports the peers'
    buffers. ``target()`` is the icepop_rs_target for icepop_bwd_bf16_rs; ``fold(out)`` sums
    this rank's slots in rank order into `out` (its dW shard) after ``stream_barrier``.
    """

    def __init__(self, shard_rows: int, row_len: int, group=None, _ops=None):
        self.group = group
        self.world = dist.get_world_size(group) if dist.is_initialized() else 1
        self.rank = dist.get_rank(group) if dist.is_initialized() else 0
        if self.world > 8:
            raise ValueError("the fused reduce-scatter supports up to 8 ranks (one NVSwitch node)")
        self.shard_rows, self.row_len = int(shard_rows), int(row_len)
        self.shard_elems = self.shard_rows * self.row_len
        if self.shard_elems % 4:
            raise ValueError("shard_rows * row_len must be a multiple of 4")
        ops = _ops or _LibPeerOps()
        self._ops = ops
        self.local = ops.alloc(self.world * self.shard_elems * 4)
        handle = ops.export(self.local)
        handles = [None] * self.world
        if self.world > 1:
            dist.all_gather_object(handles, handle, group=group)
        else:
            handles = [handle]
        self.slots = []
        self._imported = []
        for o, h in enumerate(handles):
            if o == self.rank:
                self.slots.append(self.local)
            else:
                p = ops.import_(h)
                self._imported.append(p)
                self.slots.append(p)

    def target(self) -> _lib.RsTarget:
        t = _lib.RsTarget(world=self.world, rank=self.rank, shard_rows=self.shard_rows)
        for o, p in enumerate(self.slots):
            t.slots[o] = p
        return t

    def fold(self, out: torch.Tensor, release: bool = True) -> torch.Tensor:
        """out (fp32, shard_elems) = sum of this rank's slots over ranks 0..world-1.

        With ``release`` (default) a second ``stream_barrier`` follows the fold: a peer's next
        K5 (which stores into these slots) cannot start before every rank has folded, so the
        slots are never overwritten while still being read (write-after-read across steps)."""
        if out.dtype != torch.float32 or out.numel() != self.shard_elems or not out.is_contiguous():
            raise ValueError("out must be a contiguous fp32 tensor of shard_rows * row_len elements")
        self._ops.fold(self.local, self.world, self.shard_elems, out)
        if release and self.world > 1:
            stream_barrier(self.group)
        return out

    def close(self) -> None:
        for p in self._imported:
            self._ops.close(p)
        self._imported = []
        if self.local:
            self._ops.free(self.local)
            self.local = None


class _LibPeerOps:
    """libicepop's peer-memory entry points (CUDA IPC)."""

    def __init__(self):
        import ctypes

        self._ct = ctypes
        self.lib = _lib.load()

    def alloc(self, nbytes):
        p = self._ct.c_void_p()
        _lib.check(self.lib.icepop_peer_alloc(nbytes, self._ct.byref(p)))
        return p.value

    def export(self, ptr):
        h = (self._ct.c_ubyte * 64)()
        _lib.check(self.lib.icepop_peer_export(ptr, h))
        return bytes(h)

    def import_(self, handle):
        buf = (self._ct.c_ubyte * 64).from_buffer_copy(handle)
        p = self._ct.c_void_p()
        _lib.check(self.lib.icepop_peer_import(buf, self._ct.byref(p)))
        return p.value

    def fold(self, local, world, shard_elems, out):
        _lib.check(self.lib.icepop_rs_fold(local, world, shard_elems, out.data_ptr(),
                                           torch.cuda.current_stream(out.device).cuda_stream))

    def close(self, ptr):
        _lib.check(self.lib.icepop_peer_close(ptr))

    def free(self, ptr):
        _lib.check(self.lib.icepop_peer_free(ptr))
