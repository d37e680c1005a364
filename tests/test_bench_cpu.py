"""Host-side logic of bench.py (no GPU): the synthetic batch, the zero-advantage option, the
CPU-sample sizing and the reference arm's line on a tiny configuration."""

from __future__ import annotations

import sys
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))

import bench  # noqa: E402

TINY = dict(name="tiny", seqs=4, seq_len=32, hidden=64, vocab=256, group=2, seed=7, sigma_inf=0.233)


def test_batch_is_seeded_and_rank_sharded():
    a = bench.make_batch_host(TINY, 0, 2)
    b = bench.make_batch_host(TINY, 0, 2)
    c = bench.make_batch_host(TINY, 1, 2)
    assert np.array_equal(a["rewards"], b["rewards"]) and np.array_equal(a["cu"], b["cu"])
    assert a["n_local"] == c["n_local"] == TINY["seqs"] * TINY["seq_len"]
    assert c["token_offset"] == a["n_local"]  # rank 1 owns the second contiguous range
    assert a["cu"][-1] == 2 * a["n_local"] and len(a["go"]) == 2 * TINY["seqs"] // TINY["group"] + 1


def test_zero_advantage_groups():
    cfg = dict(TINY, seqs=16)
    m = bench.make_batch_host(cfg, 0, 1, zero_adv_frac=0.5)
    go, r = m["go"], m["rewards"]
    same = [len(set(r[go[g]:go[g + 1]])) == 1 for g in range(len(go) - 1)]
    assert sum(same) >= (len(go) - 1) // 2


def test_cpu_sample_sizing_reaches_target():
    rng = np.random.default_rng(0)
    W64 = rng.standard_normal((TINY["vocab"], TINY["hidden"])) * 0.1
    n = bench.sample_tokens(TINY, W64, target_s=0.05)
    assert n >= 128 and n % 2 == 0
    dt, got = bench.time_oracle(TINY, n, W64)
    assert got == n and dt > 0


def test_reference_arm_line(capsys, monkeypatch):
    import json

    monkeypatch.setitem(bench.CONFIGS, "tiny", TINY)

    class A:
        config, steps, warmup, cpu_tokens = "tiny", 2, 1, 64

    monkeypatch.setattr(bench, "time_reference_own", lambda cfg: None)
    bench.run_reference(A)
    line = json.loads(capsys.readouterr().out.strip().splitlines()[-1])
    assert line["impl"] == "reference" and line["value"] > 0 and line["unit"] == "tokens/s"
    assert line["e2e"]["h2d_bytes_per_step"] == 0 and line["cpu_baseline"]["kind"] == "port"
