"""Multi-rank host logic on CPU (gloo, world_size 2): token sharding, the fp64 statistics
all-reduce with OR-ed error bits, bucketed dW all-reduce, and that per-rank partial sums
of the oracle over token shards (sequences cut mid-way) reproduce the full-batch objective."""

from __future__ import annotations

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from conftest import golden_hidden, load_golden, oracle_kwargs


def _free_port() -> int:
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, fn, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        q.put((rank, fn(rank, world)))
    except Exception as e:  # noqa: BLE001
        q.put((rank, e))
    finally:
        dist.destroy_process_group()


def run_ranks(fn, world=2):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, fn, q)) for r in range(world)]
    for p in procs:
        p.start()
    out = dict(q.get(timeout=120) for _ in procs)
    for p in procs:
        p.join(timeout=60)
    for r, v in out.items():
        if isinstance(v, Exception):
            raise v
    return [out[r] for r in range(world)]


@pytest.mark.parametrize("n,world,align", [(10, 2, 1), (10, 3, 1), (1000, 8, 128), (5, 8, 1), (0, 2, 1)])
def test_shard_range_partitions(n, world, align):
    from paper_2510_18855_b200.distributed import shard_range

    ranges = [shard_range(n, world, r, align) for r in range(world)]
    assert ranges[0][0] == 0 and ranges[-1][1] == n
    for (a0, a1), (b0, b1) in zip(ranges, ranges[1:]):
        assert a1 == b0 and a0 <= a1
    sizes = [b - a for a, b in ranges]
    assert max(sizes) - min(sizes) <= align


def _stats_fn(rank, world):
    from paper_2510_18855_b200.distributed import allreduce_stats

    s = torch.tensor([1.5 * (rank + 1), 1.0, 10.0, 2.0, 0.5, -3.0, 0.0, float(1 << rank)], dtype=torch.float64)
    allreduce_stats(s)
    return s.tolist()


def test_allreduce_stats_sums_and_ors_error_bits():
    out = run_ranks(_stats_fn)
    for s in out:
        assert s[:7] == [4.5, 2.0, 20.0, 4.0, 1.0, -6.0, 0.0]
        assert s[7] == 3.0  # bit0 | bit1, not 1 + 2 misread


def _same_bits_fn(rank, world):
    from paper_2510_18855_b200.distributed import allreduce_stats

    s = torch.zeros(8, dtype=torch.float64)
    s[7] = 1.0
    allreduce_stats(s)
    return s[7].item()


def test_allreduce_stats_same_bit_on_two_ranks_stays_that_bit():
    assert run_ranks(_same_bits_fn) == [1.0, 1.0]


def _grad_fn(rank, world):
    from paper_2510_18855_b200.distributed import allreduce_grad, wait_grad

    g = torch.arange(1000, dtype=torch.float32).reshape(10, 100) * (rank + 1)
    wait_grad(allreduce_grad(g, bucket_bytes=256))  # 64-element buckets
    return g.numpy()


def test_allreduce_grad_buckets():
    out = run_ranks(_grad_fn)
    ref = np.arange(1000, dtype=np.float32).reshape(10, 100) * 3
    for g in out:
        assert np.array_equal(g, ref)


def _per_token_oracle(d):
    """Per-token pieces of J and the diagnostics for the full batch (oracle)."""
    from oracle.icepop_oracle import icepop_dense, per_token_weights

    o = icepop_dense(golden_hidden(d), d["weight"], d["tokens"], d["lp_train_old"], d["lp_infer_old"],
                     d["cu_seqlens"], d["group_offsets"], d["advantages"], **oracle_kwargs(d))
    w = per_token_weights(d["cu_seqlens"], d["group_offsets"])
    return o, w


def _shard_objective_fn(rank, world):
    from paper_2510_18855_b200.distributed import allreduce_stats, shard_range

    d = load_golden("medium_icepop")
    o, w = _per_token_oracle(d)
    s, e = shard_range(len(d["tokens"]), world, rank)
    kept = o["kept"][s:e]
    ent = o["entropy"][s:e]
    stats = torch.tensor([float((w[s:e] * o["surrogate"][s:e]).sum()), float((~kept).sum()), float(e - s),
                          float(ent.sum()), float(ent[~kept].sum()), float(o["lp_cur"][s:e].sum()), 0.0, 0.0],
                         dtype=torch.float64)
    allreduce_stats(stats)
    return stats.tolist(), o["objective"], o["n_clipped"], o["token_count"]


@pytest.mark.parametrize("world", [2, 3])
def test_token_shards_reproduce_full_batch_objective(world):
    """Ranks cut sequences mid-way; the per-token weights still come out exact."""
    d = load_golden("medium_icepop")
    cu = d["cu_seqlens"]
    from paper_2510_18855_b200.distributed import shard_range

    cuts = [shard_range(len(d["tokens"]), world, r)[0] for r in range(1, world)]
    assert any(c not in set(cu.tolist()) for c in cuts), "fixture should cut a sequence"
    out = run_ranks(_shard_objective_fn, world=world)
    stats, J, n_clipped, n_tok = out[0]
    assert stats[0] == pytest.approx(J, rel=1e-12, abs=1e-15)
    assert stats[1] == n_clipped and stats[2] == n_tok


def _sharded_fn(rank, world):
    from paper_2510_18855_b200.optim import shard_bounds, sharded_sgd_step

    torch.manual_seed(0)
    w_full = torch.randn(7, 13)
    grads = [torch.randn(7, 13) for _ in range(world)]
    s, e, per = shard_bounds(w_full.numel(), world, rank)
    master = torch.zeros(per)
    master[: e - s] = w_full.view(-1)[s:e]
    vel = torch.zeros(per)

    def ref_update(m, gsh, v, out):  # objective.py:314-326 in torch (test stand-in for the CUDA kernel)
        v.mul_(0.5).add_(gsh)
        m.add_(0.1 * v)
        out.copy_(m.to(torch.bfloat16))

    wb = torch.empty(7, 13, dtype=torch.bfloat16)
    sharded_sgd_step(grads[rank], master, wb, 0.1, vel, 0.5, update_fn=ref_update)
    return wb.float().numpy(), (w_full + 0.1 * sum(grads)).to(torch.bfloat16).float().numpy()


@pytest.mark.parametrize("world", [2, 3])
def test_sharded_sgd_step_reduce_scatter_all_gather(world):
    out = run_ranks(_sharded_fn, world=world)
    for wb, ref in out:
        np.testing.assert_allclose(wb, ref, rtol=1e-2, atol=1e-2)
    assert all(np.array_equal(out[0][0], o[0]) for o in out)


class _FakePeerOps:
    """Host stand-in for the CUDA IPC entry points: 'pointers' are ids, handles are bytes."""

    def __init__(self, rank):
        self.rank = rank

    def alloc(self, nbytes):
        return 1000 + self.rank

    def export(self, ptr):
        return f"handle-{ptr}".encode()

    def import_(self, handle):
        return 5000 + int(handle.decode().split("-")[1])

    def close(self, ptr):
        pass

    def free(self, ptr):
        pass


def _peer_slots_fn(rank, world):
    from paper_2510_18855_b200.distributed import PeerSlots

    ps = PeerSlots(shard_rows=5, row_len=8, _ops=_FakePeerOps(rank))
    t = ps.target()
    return [t.slots[o] for o in range(world)], t.world, t.rank, t.shard_rows


@pytest.mark.parametrize("world", [2, 3])
def test_peer_slots_exchange_handles(world):
    """Every rank maps every owner's slot buffer: its own locally, the others via import."""
    out = run_ranks(_peer_slots_fn, world=world)
    for r, (slots, w, rk, sr) in enumerate(out):
        assert (w, rk, sr) == (world, r, 5)
        assert slots[r] == 1000 + r
        assert [s for o, s in enumerate(slots) if o != r] == [5000 + 1000 + o for o in range(world) if o != r]


class _RecordingPeerOps(_FakePeerOps):
    """Fake ops whose fold logs this rank's event; the log is shared through a file."""

    def __init__(self, rank, log):
        super().__init__(rank)
        self.log = log

    def fold(self, local, world, shard_elems, out):
        import time

        time.sleep(0.3 * (world - 1 - self.rank))  # lower ranks fold late
        with open(self.log, "a") as f:
            f.write(f"fold {self.rank}\n")


def _fold_release_fn(rank, world):
    from paper_2510_18855_b200.distributed import PeerSlots

    log = os.environ["ICEPOP_TEST_FOLD_LOG"]
    ps = PeerSlots(shard_rows=5, row_len=8, _ops=_RecordingPeerOps(rank, log))
    ps.fold(torch.empty(40, dtype=torch.float32))
    # after fold returns, the next step's K5 may store into peers' slots: every rank must
    # already have folded
    with open(log, "a") as f:
        f.write(f"next {rank}\n")
    return True


@pytest.mark.parametrize("world", [2, 3])
def test_peer_slots_fold_releases_slots_only_after_every_rank_folded(world, tmp_path, monkeypatch):
    """Write-after-read across steps: no rank leaves fold() (and so no rank's next K5 writes
    into a peer slot) before every owner has finished reading its slots."""
    log = tmp_path / "fold.log"
    monkeypatch.setenv("ICEPOP_TEST_FOLD_LOG", str(log))
    run_ranks(_fold_release_fn, world=world)
    lines = log.read_text().split()
    events = [(lines[i], int(lines[i + 1])) for i in range(0, len(lines), 2)]
    last_fold = max(i for i, (e, _) in enumerate(events) if e == "fold")
    first_next = min(i for i, (e, _) in enumerate(events) if e == "next")
    assert last_fold < first_next, events


class _FoldingPeerOps(_FakePeerOps):
    """Fake ops whose fold writes the owner's summed dW shard (what the CUDA fold of the slots
    K5 filled would produce): the sum over ranks of each rank's seeded partial dW."""

    def __init__(self, rank, world, shape):
        super().__init__(rank)
        self.world, self.shape = world, shape

    def fold(self, local, world, shard_elems, out):
        full = sum(_partial_dw(r, self.shape) for r in range(world)).reshape(-1)
        lo = self.rank * shard_elems
        part = full[lo:lo + shard_elems]
        out.zero_()
        out[:part.numel()] = part


def _partial_dw(rank, shape):
    return torch.randn(shape, generator=torch.Generator().manual_seed(100 + rank))


def _composed_fn(rank, world):
    from paper_2510_18855_b200.optim import ShardedAscent

    shape = (37, 16)  # 37 dW rows: the last shard is ragged
    w0 = torch.randn(shape, generator=torch.Generator().manual_seed(7))
    weight = w0.to(torch.bfloat16)
    lr, beta = 0.25, 0.5

    def ref_update(m, g, v, out):  # objective.py:314-326 in torch (stand-in for the CUDA kernel)
        v.mul_(beta).add_(g)
        m.add_(lr * v)
        out.copy_(m.to(torch.bfloat16))

    opt = ShardedAscent(weight, lr, beta=beta, _ops=_FoldingPeerOps(rank, world, shape), _update_fn=ref_update)
    assert opt.world == world and opt.rank == rank
    opt.step()
    opt.step()  # velocity carries over: v2 = beta v1 + g
    return weight.float().numpy(), w0.numpy()


@pytest.mark.parametrize("world", [2, 3])
def test_sharded_ascent_composed_step_gloo(world):
    """ShardedAscent.step over gloo: each rank folds its shard of the summed dW (the fused
    reduce-scatter's slots), runs the momentum update on its fp32 master shard, and the bf16
    shards are all-gathered into every rank's replicated weight; two steps equal two unsharded
    momentum steps on the summed dW."""
    out = run_ranks(_composed_fn, world=world)
    shape = (37, 16)
    g = sum(_partial_dw(r, shape) for r in range(world))
    w = torch.from_numpy(out[0][1]).to(torch.bfloat16).float()  # the master starts from the bf16 weight
    v = torch.zeros(shape)
    for _ in range(2):
        v = 0.5 * v + g
        w = w + 0.25 * v
    want = w.to(torch.bfloat16).float().numpy()
    for wb, _ in out:
        np.testing.assert_array_equal(wb, want)
