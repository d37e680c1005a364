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


def _run_bench(*args, env_extra=None, timeout=240):
    import os
    import subprocess

    env = {k: v for k, v in os.environ.items() if k not in ("WORLD_SIZE", "RANK", "LOCAL_RANK")}
    env.update(env_extra or {})
    return subprocess.run([sys.executable, str(ROOT / "bench.py"), *args], capture_output=True, text=True,
                          timeout=timeout, env=env, cwd=str(ROOT))


def test_gpus_2_self_launches_two_gloo_ranks():
    """`bench.py --gpus 2` without torchrun starts two ranks itself (gloo dry run on CPU): both
    take their token shard, the stats all-reduce sums them, rank 0 alone prints."""
    import json

    r = _run_bench("--gpus", "2", "--dry-run", "--config", "c1")
    assert r.returncode == 0, r.stderr[-2000:]
    lines = [json.loads(x) for x in r.stdout.splitlines() if x.startswith("{")]
    assert len(lines) == 1, r.stdout
    line = lines[0]
    assert line["n_gpus"] == 2 and line["dry_run"] is True
    assert [x["rank"] for x in line["ranks"]] == [0, 1]
    assert line["ranks"][1]["token_offset"] == line["ranks"][0]["tokens"] == 4096
    assert line["global_tokens"] == 2 * 4096


def test_gpus_1_dry_run_is_one_rank():
    import json

    r = _run_bench("--gpus", "1", "--dry-run", "--config", "c1")
    assert r.returncode == 0, r.stderr[-2000:]
    line = json.loads([x for x in r.stdout.splitlines() if x.startswith("{")][-1])
    assert line["n_gpus"] == 1 and len(line["ranks"]) == 1


def test_gpus_n_refuses_without_gpus():
    """More ranks than visible GPUs: a clear refusal, never a silent 1-GPU run."""
    r = _run_bench("--gpus", "2", "--steps", "1", "--warmup", "3", env_extra={"CUDA_VISIBLE_DEVICES": ""})
    assert r.returncode == 2 and "refusing" in r.stderr


def test_world_size_mismatch_refuses():
    r = _run_bench("--gpus", "4", "--dry-run", env_extra={"WORLD_SIZE": "2", "RANK": "0"})
    assert r.returncode == 2 and "WORLD_SIZE=2" in r.stderr
