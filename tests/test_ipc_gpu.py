"""The real CUDA IPC path of the fused dW reduce-scatter, across processes.

`world` processes share the one GPU of the box (the pool has one). Each is a token-shard
rank: it maps its peers' slot buffers with ``PeerSlots`` (icepop_peer_alloc / export /
import, CUDA IPC handles exchanged over gloo), runs its shard's backward with K5 storing
dW rows into the owners' slots, and folds its own slots. No kernel waits on another
process: the ranks are ordered by host barriers after ``torch.cuda.synchronize()``.
On an NVSwitch box the same stores cross NVLink; here they land in the same HBM, which is
what lets one GPU check the handle exchange, the cross-process stores and the fold.
"""

from __future__ import annotations

import os
import socket

import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu


def _free_port() -> int:
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _ipc_rank(rank, world, port, q):
    import torch.distributed as dist

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import paper_2510_18855_b200.loss as L
        from paper_2510_18855_b200.distributed import PeerSlots, shard_range
        from test_dense_gpu import _batch, _case, _rel

        dev = torch.device("cuda", 0)
        torch.cuda.set_device(dev)
        c = _case(n_seqs=6, seed=53, lens=[310, 150, 270, 95, 400, 333])
        H, W = c["H"].to(dev), c["W"].to(dev)
        V, d = W.shape
        cfg = L.IcePopConfig()
        f_full = L.icepop_fwd(H, W, _batch(c, dev), cfg, store_probs=True)
        _, gw_ref = L.icepop_bwd(H, W, _batch(c, dev), f_full, cfg, need_hidden=False)

        shard_rows = -(-V // world)
        peer = PeerSlots(shard_rows, d)
        s, e = shard_range(len(c["tokens"]), world, rank)
        b = _batch(c, dev, slice(s, e))
        f = L.icepop_fwd(H[s:e], W, b, cfg, store_probs=True)
        L.icepop_bwd_reduce_scatter(H[s:e], W, b, f, peer.target(), cfg, need_hidden=False)
        torch.cuda.synchronize()
        dist.barrier()  # every rank's stores into every owner's slots are complete
        out = torch.empty(shard_rows * d, dtype=torch.float32, device=dev)
        peer.fold(out, release=False)
        torch.cuda.synchronize()
        dist.barrier()  # nobody unmaps or frees a slot buffer before every fold is done
        lo, hi = rank * shard_rows, min((rank + 1) * shard_rows, V)
        mine = out.view(shard_rows, d)[: hi - lo].cpu().numpy()
        ok_finite = bool(np.isfinite(mine).all())
        rel = _rel(mine, gw_ref[lo:hi].cpu().numpy())
        peer.close()
        q.put((rank, (ok_finite, rel, hi - lo)))
    except Exception as ex:  # noqa: BLE001
        q.put((rank, ex))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_fused_reduce_scatter_over_cuda_ipc(cuda_device, world):
    import torch.multiprocessing as mp

    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_ipc_rank, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    try:
        out = dict(q.get(timeout=240) for _ in procs)
    finally:
        for p in procs:
            p.join(timeout=60)
            if p.is_alive():
                p.kill()
    for r in range(world):
        v = out[r]
        if isinstance(v, Exception):
            raise v
        ok_finite, rel, rows = v
        assert rows > 0 and ok_finite, (r, v)
        assert rel < 1e-5, (r, rel)


def _composed_rank(rank, world, port, q):
    """One rank of the composed ZeRO step over real CUDA IPC: K5 stores dW rows into the owners'
    slots, ShardedAscent folds this rank's slots, runs the momentum update on its fp32 shard and
    all-gathers the bf16 shards (over gloo here)."""
    import torch.distributed as dist

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import paper_2510_18855_b200.loss as L
        from paper_2510_18855_b200.distributed import shard_range
        from paper_2510_18855_b200.optim import ShardedAscent
        from test_dense_gpu import _batch, _case

        dev = torch.device("cuda", 0)
        torch.cuda.set_device(dev)
        c = _case(n_seqs=6, seed=54, lens=[310, 150, 270, 95, 400, 333])
        H, W = c["H"].to(dev), c["W"].to(dev)
        cfg = L.IcePopConfig()
        lr, beta = 0.5, 0.9
        f_full = L.icepop_fwd(H, W, _batch(c, dev), cfg, store_probs=True)
        _, gw = L.icepop_bwd(H, W, _batch(c, dev), f_full, cfg, need_hidden=False)
        want = (W.float() + lr * gw).to(torch.bfloat16)  # first momentum step from v = 0: w + lr g

        weight = W.clone()
        opt = ShardedAscent(weight, lr, beta=beta)
        s, e = shard_range(len(c["tokens"]), world, rank)
        b = _batch(c, dev, slice(s, e))
        f = L.icepop_fwd(H[s:e], W, b, cfg, store_probs=True)
        L.icepop_bwd_reduce_scatter(H[s:e], W, b, f, opt.rs_target(), cfg, need_hidden=False)
        opt.step()
        torch.cuda.synchronize()
        diff = float((weight.float() - want.float()).abs().max())
        scale = float(want.float().abs().max())
        dist.barrier()  # nobody unmaps a slot buffer before every rank is done
        opt.close()
        q.put((rank, (diff, scale)))
    except Exception as ex:  # noqa: BLE001
        q.put((rank, ex))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_composed_zero_step_over_cuda_ipc(cuda_device, world):
    import torch.multiprocessing as mp

    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_composed_rank, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    try:
        out = dict(q.get(timeout=240) for _ in procs)
    finally:
        for p in procs:
            p.join(timeout=60)
            if p.is_alive():
                p.kill()
    for r in range(world):
        v = out[r]
        if isinstance(v, Exception):
            raise v
        diff, scale = v
        assert diff <= 2 ** -7 * scale, (r, diff, scale)  # one bf16 step: fp32 fma vs torch's rounding
