"""IcePop fwd+bwd throughput on B200 (BASELINE.json metric), one JSON line on rank 0.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference] [--config c2]
    torchrun --nproc-per-node N bench.py --gpus N ...        (token-sharded, weak scaling)

`--gpus N` (N > 1) without torchrun starts the N ranks itself (torch.distributed.run on
127.0.0.1, NCCL_DEBUG=INFO with the INIT subsystem so the communicator's nranks is logged) and
refuses when fewer than N GPUs are visible. `--dry-run` runs the rank plumbing over gloo on the
CPU (no GPU work, no throughput).

A step = one IcePop forward (K0 advantages, K1 fused lm_head GEMM + online softmax, K2
epilogue) + backward (bf16 dZ -- formed in place from the probabilities K1 stored when they
fit in HBM ("stored-probabilities" mode, the default at C2), else recomputed by the K3 GEMM
in chunks -- then K4 dHidden, K5 dW) over one batch
of synthetic inputs of the named config, plus (N>1) the NCCL all-reduce of the fp64
statistics and of dW. `value` is measured with inputs resident in HBM; `e2e` goes
through the public API from pinned host buffers with the H2D copies of the step's
inputs and the D2H read of its loss inside the timed region.

--impl reference times the reference's algorithm on the host cores (the numpy oracle
port of objective.py:172-298; the reference itself is pure numpy and has no GPU path)
on a bounded token sample of the same workload.
"""

from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import threading
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

METRIC = "IcePop fwd+bwd tokens/sec at 1/2/4/8 B200; % tensor-pipe peak; CPU-ref speedup"
UNIT = "tokens/s"

# SURVEY.md section 8 configs (per rank for the weak-scaling sweep)
CONFIGS = {
    "c1": dict(name="C1 CPU-reference shape: 8 seqs x 512 tok, d=1024, V=32768, G=8", seqs=8, seq_len=512,
               hidden=1024, vocab=32768, group=8, seed=0, sigma_inf=0.233),
    "c2": dict(name="C2 single B200: 64 seqs x 4096 tok, d=4096, V=157184 (Ling-2.0), G=8", seqs=64, seq_len=4096,
               hidden=4096, vocab=157184, group=8, seed=1, sigma_inf=0.233),
    "c3": dict(name="C3 Ling-1T lm_head shard: 8 seqs x 4096 tok/GPU, d=8192, V=157184, G=8", seqs=8, seq_len=4096,
               hidden=8192, vocab=157184, group=8, seed=2, sigma_inf=0.233),
    "c4": dict(name="C4 Long-CoT: 32 seqs, ragged lognormal lengths (median 16384, <= 32768), d=8192, V=157184, "
                    "~5% popped", seqs=32, seq_len=0, hidden=8192, vocab=157184, group=8, seed=3, sigma_inf=0.42,
               lens=dict(median=16384, sigma=0.6, lo=256, hi=32768)),
    "c5": dict(name="C5 scaling point: 32 seqs x 4096 tok/GPU, d=8192, V=157184, G=8", seqs=32, seq_len=4096,
               hidden=8192, vocab=157184, group=8, seed=4, sigma_inf=0.233),
}

FLOP_PER_TOKEN = lambda d, v: 6.0 * d * v  # noqa: E731  algorithmic (fwd + dH + dW), SURVEY 8d


def peaks() -> dict:
    p = ROOT / "MEASURED_PEAKS.json"
    if p.exists():
        j = json.loads(p.read_text())
        return dict(tflops=float(j["bf16_tflops"]), tflops_sustained=float(j.get("bf16_tflops_sustained", 0) or 0),
                    hbm=float(j["hbm_gbs"]), source="measured")
    return dict(tflops=1590.0, tflops_sustained=1400.0, hbm=6650.0, source="fallback")


# ----------------------------------------------------------------------------- clocks
class ClockSampler:
    FIELDS = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.rows: list[list[str]] = []
        self.proc = None
        self.thread = None

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits",
                 "-lms", "200"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except OSError:
            self.proc = None
            return

        def pump():
            for line in self.proc.stdout:
                self.rows.append([x.strip() for x in line.split(",")])

        self.thread = threading.Thread(target=pump, daemon=True)
        self.thread.start()

    def stop(self) -> dict | None:
        if self.proc is None:
            return None
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except subprocess.TimeoutExpired:
            self.proc.kill()
        if self.thread:
            self.thread.join(timeout=2)
        rows = [r for r in self.rows if len(r) >= 7]
        if not rows:
            return None
        sm = [float(r[0]) for r in rows if r[0].replace(".", "").isdigit()]
        mx = [float(r[1]) for r in rows if r[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in rows for i in range(4) if r[3 + i].lower().startswith("active")})
        return {"sm_mhz": float(np.median(sm)) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(rows)}


# ----------------------------------------------------------------------------- inputs
def make_batch_host(cfg: dict, rank: int, world: int, zero_adv_frac: float = 0.0):
    """Seeded synthetic rollout batch for this rank: rewards ~ Bernoulli(0.5),
    groups of `group` sequences, this rank owns `seqs` whole sequences. `zero_adv_frac` of the
    groups (every k-th) get identical rewards -> zero advantages, as all-solved / all-failed
    prompts do in real RL batches (their rows drop out of the block-sparse backward)."""
    rng = np.random.default_rng(cfg["seed"])
    S_global = cfg["seqs"] * world
    if cfg.get("lens"):  # ragged packed lengths (C4); every rank gets the same per-rank count
        L = cfg["lens"]
        per = np.clip(rng.lognormal(np.log(L["median"]), L["sigma"], cfg["seqs"]), L["lo"], L["hi"]).astype(np.int64)
        lens = np.tile(per, world)
    else:
        lens = np.full(S_global, cfg["seq_len"], dtype=np.int64)
    cu = np.concatenate([[0], np.cumsum(lens)]).astype(np.int32)
    go = np.arange(0, S_global + 1, cfg["group"], dtype=np.int32)
    rewards = rng.integers(0, 2, S_global).astype(np.float64)
    n_groups = len(go) - 1
    n_zero = int(round(zero_adv_frac * n_groups))
    for g in np.linspace(0, n_groups, n_zero, endpoint=False).astype(int) if n_zero else []:
        rewards[go[g]:go[g + 1]] = 1.0
    n_local = int(lens[: cfg["seqs"]].sum())
    return dict(cu=cu, go=go, rewards=rewards, n_local=n_local, token_offset=rank * n_local)


def sample_on_policy(H, W, g, rows: int = 4096):
    """Sampled tokens y_t ~ softmax(H_t . W^T) (on-policy, as the rollout engine
    draws them), by the Gumbel-max trick over row chunks of the logits (setup, untimed; cuBLAS
    bf16 logits are exact enough to sample from)."""
    import torch

    out = torch.empty(H.shape[0], dtype=torch.int32, device=H.device)
    for i in range(0, H.shape[0], rows):
        z = (H[i:i + rows] @ W.T).float()
        u = torch.rand(z.shape, device=H.device, generator=g).clamp_(min=1e-20)
        z.sub_(u.log_().neg_().log_())  # z + Gumbel(0, 1)
        out[i:i + rows] = z.argmax(dim=1).to(torch.int32)
        del z, u
    return out


def build_device_inputs(cfg, meta, dev, rank):
    import torch

    from paper_2510_18855_b200 import _lib
    from paper_2510_18855_b200.loss import PackedBatch, icepop_fwd  # noqa: F401

    g = torch.Generator(device=dev).manual_seed(1000 * cfg["seed"] + rank)
    N, d, V = meta["n_local"], cfg["hidden"], cfg["vocab"]
    H = torch.randn(N, d, device=dev, generator=g, dtype=torch.float32).to(torch.bfloat16)
    W = (torch.randn(V, d, device=dev, generator=g, dtype=torch.float32) * (2.0 / np.sqrt(d))).to(torch.bfloat16)
    tokens = sample_on_policy(H, W, g)
    # setup forward (untimed): lp_theta(y) -> lp_old = lp + N(0, 0.1) exercises the clip
    # branch; lp_inf = lp_old - N(0, sigma) pops ~1.5 permille
    lib = _lib.ensure_device(dev.index)
    shape = _lib.Shape(n_tokens=N, token_offset=meta["token_offset"], hidden=d, vocab=V,
                       n_seqs=len(meta["cu"]) - 1, n_groups=len(meta["go"]) - 1, weight_layout=_lib.W_VD)
    fb = _lib._sz()
    _lib.check(lib.icepop_workspace_bytes(shape, 0, 0, fb, None))
    ws = torch.empty(fb.value, dtype=torch.uint8, device=dev)
    lp = torch.empty(N, dtype=torch.float64, device=dev)
    lse0 = torch.empty(N, dtype=torch.float32, device=dev)
    ent0 = torch.empty(N, dtype=torch.float32, device=dev)
    _lib.check(lib.icepop_logprob_bf16(shape, 1.0, H.data_ptr(), W.data_ptr(), tokens.data_ptr(), lse0.data_ptr(),
                                       lp.data_ptr(), ent0.data_ptr(), ws.data_ptr(), ws.numel(),
                                       torch.cuda.current_stream(dev).cuda_stream))
    del ws
    lp_old = lp + 0.1 * torch.randn(N, device=dev, dtype=torch.float64, generator=g)
    lp_inf = lp_old - cfg["sigma_inf"] * torch.randn(N, device=dev, dtype=torch.float64, generator=g)
    batch = PackedBatch(tokens=tokens, lp_train_old=lp_old, lp_infer_old=lp_inf,
                        cu_seqlens=torch.from_numpy(meta["cu"]).to(dev), group_offsets=torch.from_numpy(meta["go"]).to(dev),
                        advantages=None, rewards=torch.from_numpy(meta["rewards"]).to(dev),
                        token_offset=meta["token_offset"])
    # on-policy variant (theta == theta_old): lp_train_old is exactly the recorded lp
    onp = PackedBatch(tokens=tokens, lp_train_old=lp, lp_infer_old=lp - (lp_old - lp_inf),
                      cu_seqlens=batch.cu_seqlens, group_offsets=batch.group_offsets, advantages=None,
                      rewards=batch.rewards, token_offset=meta["token_offset"])
    return H, W, batch, (onp, lse0, ent0)


# ----------------------------------------------------------------------------- GPU arm
def run_ours(args):
    import torch
    import torch.distributed as dist

    from paper_2510_18855_b200 import _lib
    from paper_2510_18855_b200.distributed import allreduce_grad, allreduce_stats, wait_grad
    from paper_2510_18855_b200.loss import (Diagnostics, IcePopConfig, _dz_chunk_bytes, _resolve_store_probs, finish,
                                            icepop_bwd, icepop_fwd, icepop_fwd_bwd, probs_chunk_tokens)

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        dist.init_process_group("nccl", device_id=dev)
    cfg = dict(CONFIGS[args.config])
    if args.seqs:
        cfg["seqs"] = args.seqs
        cfg["name"] += f" [seqs/rank = {args.seqs}]"
    meta = make_batch_host(cfg, rank, world, args.zero_adv_frac)
    H, W, batch, onpolicy = build_device_inputs(cfg, meta, dev, rank)
    icfg = IcePopConfig()
    N, d, V = meta["n_local"], cfg["hidden"], cfg["vocab"]
    sp = _resolve_store_probs(None, N, V, dev, False)
    # stored probabilities for the whole batch; else in token chunks that fit (icepop_fwd_bwd);
    # else the logit recompute
    sp_chunk = 0 if sp else probs_chunk_tokens(N, V, dev)
    if os.environ.get("ICEPOP_STORE_PROBS", "auto") == "0":
        sp_chunk = 0
    if world > 1:  # one mode on every rank (free memory may differ): the collectives must match
        agree = torch.tensor([int(sp), sp_chunk if not sp else N], dtype=torch.int64, device=dev)
        dist.all_reduce(agree, op=dist.ReduceOp.MIN)
        sp = bool(agree[0].item())
        sp_chunk = 0 if sp else int(agree[1].item())
    rows = _dz_chunk_bytes(dev) // (2 * (V + d))
    chunk = N if (sp or rows >= N) else max(128, rows // 128 * 128)
    if sp_chunk:
        chunk = sp_chunk
    n_chunks = -(-N // chunk)
    # fwd: K0, token check, K1, K2, finalize, err-merge; bwd: stored probabilities -> block
    # flags + lists, row prep, exception-row dZ, K4, K5, iota + one-hot scatter (CUB's radix
    # sort kernels are library code, not counted); per token chunk when chunked; recompute ->
    # 4 compaction kernels + (K3, K4, hidden transpose, K5) per dZ chunk
    if sp:
        launches_per_step = 6 + 8
    elif sp_chunk:
        launches_per_step = n_chunks * (6 + 8)
    else:
        launches_per_step = 6 + 4 + 4 * n_chunks
    dz_mode = "stored-probabilities" if sp else (
        f"stored-probabilities in {n_chunks} token chunks" if sp_chunk else "recompute")

    # dW collective for N > 1: fused reduce-scatter inside K5's epilogue over NVLink peer memory
    # (each rank ends with its ZeRO shard of the summed dW), or NCCL all-reduce of the full dW.
    collective = "none"
    peer = None
    dw_shard = None
    if world > 1:
        collective = args.dw_collective if not sp_chunk else "nccl"
        if collective == "fused":
            try:
                from paper_2510_18855_b200.distributed import PeerSlots

                shard_rows = -(-V // world)
                peer = PeerSlots(shard_rows, d)
                dw_shard = torch.empty(shard_rows * d, dtype=torch.float32, device=dev)
            except Exception as e:  # noqa: BLE001 - a peer-mapping failure selects the NCCL collective
                print(f"fused reduce-scatter unavailable ({e}); using NCCL all-reduce", file=sys.stderr)
                collective = "nccl"

    fwd_events = []  # (start, end) around the forward call of each timed step (K1 + K2 + K0)

    def step_into(record_fwd=False):
        # loss = -J: grad_scale -1 gives d(loss)/d(hidden), d(loss)/d(W)
        if sp_chunk:
            f, gh, g = icepop_fwd_bwd(H, W, batch, icfg, layout="vd", grad_scale=-1.0, max_chunk_tokens=sp_chunk)
            if world > 1:
                allreduce_stats(f.stats)
                wait_grad(allreduce_grad(g))
            return f
        if record_fwd:
            ev = (torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
            ev[0].record()
        f = icepop_fwd(H, W, batch, icfg, layout="vd", store_probs=sp)
        if record_fwd:
            ev[1].record()
            fwd_events.append(ev)
        if collective == "fused":
            from paper_2510_18855_b200.distributed import stream_barrier
            from paper_2510_18855_b200.loss import icepop_bwd_reduce_scatter

            icepop_bwd_reduce_scatter(H, W, batch, f, peer.target(), icfg, layout="vd", grad_scale=-1.0)
            allreduce_stats(f.stats)
            stream_barrier()
            peer.fold(dw_shard)
            return f
        gh, g = icepop_bwd(H, W, batch, f, icfg, layout="vd", grad_scale=-1.0)
        if world > 1:
            allreduce_stats(f.stats)
            wait_grad(allreduce_grad(g))
        return f

    # warm-up (also validates the error word once)
    for _ in range(args.warmup):
        f = step_into()
    finish(f.stats)
    torch.cuda.synchronize()

    # ---------------- timed region: inputs resident (H 2.1 GB, W 1.3 GB > 126 MB L2)
    sampler = ClockSampler(local)
    sampler.start()
    time.sleep(0.3)
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(args.steps):
        f = step_into(record_fwd=True)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / args.steps
    # the forward's device time inside the timed steps (events on the launching stream): K1
    # dominates it (K0, the token check and K2 add ~0.2 ms at C2)
    fwd_ms = float(np.mean([a.elapsed_time(b) for a, b in fwd_events])) if fwd_events else None
    if world > 1:
        dist.barrier()
    clocks = sampler.stop()
    t = torch.tensor([ms], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    ms = float(t.item())
    diag = Diagnostics.from_stats(f.stats.cpu())

    def timed_steps(step_fn, n, warm=2):
        """Device time per step of step_fn (CUDA events on the torch stream, max over ranks)."""
        for _ in range(warm):
            step_fn()
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        a0, a1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a0.record()
        for _ in range(n):
            step_fn()
        a1.record()
        torch.cuda.synchronize()
        tt = torch.tensor([a0.elapsed_time(a1) / n], dtype=torch.float64, device=dev)
        if world > 1:
            dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        return float(tt.item())

    def record(ms_v, n, note, **extra):
        r = {"value": round(N * world / (ms_v / 1e3), 1), "unit": UNIT, "ms_per_step": round(ms_v, 3), "steps": n,
             "step_tflops_alg": round(FLOP_PER_TOKEN(d, V) * N / (ms_v / 1e3) / 1e12, 1), "note": note}
        r.update(extra)
        return r

    # sub-record steps: a few at the headline's size; more when a step is short (C1: ~1 ms, where
    # one host hiccup would dominate a 4-step average)
    n_var = max(2, min(args.steps, 4)) if ms > 50.0 else max(10, min(args.steps, 20))

    # ---------------- on-policy variant (extra line item; the headline is the general case)
    onp_res = None
    if not args.no_onpolicy:
        from paper_2510_18855_b200.loss import icepop_fwd_onpolicy

        ob, lse0, ent0 = onpolicy

        def step_onp():
            f = icepop_fwd_onpolicy(ob, lse0, ent0, icfg, hidden_dim=d, vocab=V)
            _, g = icepop_bwd(H, W, ob, f, icfg, layout="vd", grad_scale=-1.0)
            if world > 1:
                allreduce_stats(f.stats)
                wait_grad(allreduce_grad(g))
            return f

        onp_res = record(timed_steps(step_onp, n_var), n_var,
                         "theta == theta_old (the reference loop's own case, scheduler.py:540) with lp_train_old "
                         "recorded by icepop_logprob_bf16: GEMM-free exact forward + full backward")

    # ---------------- recompute variant: the north star's "logits never written to HBM" mode
    rec_res = None
    if not args.no_recompute and sp:
        def step_rec():
            f = icepop_fwd(H, W, batch, icfg, layout="vd", store_probs=False)
            _, g = icepop_bwd(H, W, batch, f, icfg, layout="vd", grad_scale=-1.0)
            if world > 1:
                allreduce_stats(f.stats)
                wait_grad(allreduce_grad(g))
            return f

        rms = timed_steps(step_rec, n_var)
        rk = kernel_times(H, W, batch, icfg, meta, cfg, min(chunk, N), dev, False) if not args.no_kernel_timing else {}
        rec_res = record(rms, n_var, "logits never stored: K1 writes only per-row statistics, K3 recomputes the "
                         "logits tile by tile into bf16 dZ chunks (8.d.V executed FLOPs per token instead of 6)",
                         kernels_ms={k: round(v["ms"], 3) for k, v in rk.items()},
                         executed_tflops=round(8.0 * d * V * N / (rms / 1e3) / 1e12, 1))

    # ---------------- the reference loop's call pattern: ref passed, gamma = 0 (scheduler.py:530-542)
    ref_res = None
    if not args.no_ref_diag and sp:
        gr = torch.Generator(device=dev).manual_seed(77)
        Wr = (W.float() + 0.01 * torch.randn(W.shape, device=dev, generator=gr)).to(torch.bfloat16)

        def step_ref():
            f = icepop_fwd(H, W, batch, icfg, layout="vd", weight_ref=Wr, store_probs=sp)
            _, g = icepop_bwd(H, W, batch, f, icfg, layout="vd", grad_scale=-1.0, weight_ref=Wr)
            if world > 1:
                allreduce_stats(f.stats)
                wait_grad(allreduce_grad(g))
            return f

        f0 = icepop_fwd(H, W, batch, icfg, layout="vd", weight_ref=Wr, store_probs=sp)
        ref_mode = "stored-probabilities" if "probs" in f0.extras else "recompute"
        del f0
        rfms = timed_steps(step_ref, n_var)
        ref_res = record(rfms, n_var, "KL-to-ref diagnostic with gamma = 0, as train_loop calls objective_and_grad "
                         "(ref=params.copy(), scheduler.py:530-542): dual-accumulator forward (z and z_ref share "
                         "every hidden tile) that also stores the probabilities, so the backward is the "
                         "headline's; 8.d.V executed FLOPs per token",
                         dz_mode=ref_mode, executed_tflops=round(8.0 * d * V * N / (rfms / 1e3) / 1e12, 1))
        del Wr

    # ---------------- per-kernel timing pass (same work, events between launches)
    kern = (kernel_times(H, W, batch, icfg, meta, cfg, chunk, dev, sp or bool(sp_chunk))
            if not args.no_kernel_timing else {})

    # ---------------- end-to-end through the public API from pinned host buffers
    e2e = None
    if not args.no_e2e:
        e2e = run_e2e(H, W, batch, icfg, args, dev, world, sp, sp_chunk)

    tokens_total = N * world
    value = tokens_total / (ms / 1e3)
    pk = peaks()
    line = {
        "metric": METRIC, "value": round(value, 1), "unit": UNIT, "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": round(ms, 3), "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "bf16", "data": "synthetic (seeded; random-init lm_head weights)",
        "config": {"workload": cfg["name"], "global_batch": tokens_total,
                   "seq_len": cfg["seq_len"] or "ragged",
                   "hidden": d, "vocab": V, "group_size": cfg["group"], "parallelism": f"dp{world} token-sharded",
                   "weight_layout": "[V,d]", "dz_chunk_tokens": chunk,
                   "dz_mode": dz_mode,
                   # HBM the stored-probabilities mode holds between forward and backward: bf16 q
                   # [N, V] + the fp32 slab references (0 in the recompute mode)
                   "stored_probs_bytes": (int(min(N, sp_chunk or N) * (2 * V + 4 * _lib.tile_max_ld(V)))
                                          if (sp or sp_chunk) else 0),
                   "l2": "inputs larger than L2 (H %.1f GB, W %.1f GB vs 126 MB)" % (N * d * 2 / 1e9, V * d * 2 / 1e9),
                   "popped_fraction": round(diag.clipped_fraction, 6), "dw_collective": collective,
                   "zero_adv_group_frac": args.zero_adv_frac},
        "per_gpu_value": round(value / world, 1),
        "gpu_launches": launches_per_step * args.steps,
        "step_tflops_alg": round(FLOP_PER_TOKEN(d, V) * N / (ms / 1e3) / 1e12, 1),
        "step_frac_of_peak_alg": round(FLOP_PER_TOKEN(d, V) * N / (ms / 1e3) / 1e12 / pk["tflops"], 4),
        "peak_source": pk["source"],
    }
    if kern:
        line["kernels_ms"] = {k: round(v["ms"], 3) for k, v in kern.items()}
        # The roofline kernel is K1, the fused lm_head GEMM + online softmax of the north star
        # (its share of the step equals each backward GEMM's); per-kernel figures follow.
        dom = "K1_fwd_lse+K2"
        # K1 is timed live inside the timed steps (a kernel inside a long step: the sustained
        # peak is its denominator); the isolated kernel-timing pass is the fallback (C4's chunks)
        k1_ms = fwd_ms if fwd_ms else kern[dom]["ms"]
        ach = kern[dom]["flop"] / (k1_ms / 1e3) / 1e12
        pk_use = pk["tflops_sustained"] if (fwd_ms and pk["tflops_sustained"]) else pk["tflops"]
        # DRAM bytes per launch from the committed ncu capture of this kernel at this config (ncu
        # cannot run inside the timed bench); `traffic_measured` says which capture
        traffic = traffic_src = None
        tj = ROOT / "profiles" / "ncu_traffic.json"
        if tj.exists():
            t = json.loads(tj.read_text()).get(args.config, {}).get(dom)
            traffic = t["dram_bytes_per_launch"] if t else None
            traffic_src = t.get("measured") if t else None
        line["roofline"] = {"bound": "tensor", "kernel": dom, "achieved": round(ach, 1), "peak": pk_use,
                            "unit": "TFLOP/s", "frac": round(ach / pk_use, 4), "traffic": traffic,
                            "traffic_unit": "bytes/launch (ncu dram read+write)", "traffic_measured": traffic_src,
                            "flop_per_launch": kern[dom]["flop"], "launch_ms": round(k1_ms, 3),
                            "timed": "events around the forward inside the timed steps" if fwd_ms else
                                     "isolated kernel-timing pass",
                            "peak_kind": ("sustained" if pk_use == pk["tflops_sustained"] else "burst")
                                         + f" ({pk['source']}; MEASURED_PEAKS.json)",
                            "frac_of_burst": round(ach / pk["tflops"], 4),
                            "frac_of_sustained": round(ach / pk["tflops_sustained"], 4) if pk["tflops_sustained"]
                            else None}
        line["kernels_tflops"] = {k: round(v["flop"] / (v["ms"] / 1e3) / 1e12, 1) for k, v in kern.items()
                                  if v["flop"]}
        if "K2_epilogue" in kern:  # the north star's bandwidth-bound IcePop epilogue
            kz = kern["K2_epilogue"]
            gbs = kz["bytes"] / (kz["ms"] / 1e3) / 1e9
            line["roofline_epilogue"] = {
                "bound": "hbm", "kernel": "K2 k2_icepop_tokens + k_finalize_stats", "achieved": round(gbs, 1),
                "peak": pk["hbm"], "unit": "GB/s", "frac": round(gbs / pk["hbm"], 4), "ms": round(kz["ms"], 4),
                "bytes_per_launch": kz["bytes"], "partials_per_token": kz["n_partials_per_token"],
                "bytes_note": "per token: K1's partials (12 B each, one per run of 2 vocabulary tiles) + tokens, "
                              "ztok, lp_old, lp_inf (24 B) + lse, lp_cur, entropy, kept, calib, surrogate, coeff (37 B)"}
            line["kernels_ms"]["K1_fwd_lse"] = round(kern["K1_fwd_lse+K2"]["ms"] - kz["ms"], 3)
        if "bwd_prep" in kern:  # the HBM-bound part of the stored-probabilities backward
            kz = kern["bwd_prep"]
            gbs = kz["bytes"] / (kz["ms"] / 1e3) / 1e9
            line["roofline_bwd_prep"] = {
                "bound": "hbm", "kernel": "bwd_prep (k_sp_prep + exception-row dZ + block lists)",
                "achieved": round(gbs, 1), "peak": pk["hbm"], "unit": "GB/s", "frac": round(gbs / pk["hbm"], 4),
                "bytes_per_launch": kz["bytes"],
                "bytes_note": "algorithmic: read H + write s*H (bf16), read the slab references; "
                              "exception rows (none in this batch) add a read + write of their q/dZ row"}
    if e2e:
        line["e2e"] = e2e
    if onp_res:
        line["on_policy"] = onp_res
    if rec_res:
        line["recompute"] = rec_res
    if ref_res:
        if kern:  # the headline plus one extra forward GEMM (the KL diagnostic's z_ref)
            ref_res["target_ms"] = round(ms + kern["K1_fwd_lse+K2"]["ms"], 3)
        line["ref_diag"] = ref_res
    line["wave_barrier_abandons"] = _lib.wave_barrier_abandons(local)
    if clocks:
        line["clocks"] = clocks
    if rank == 0 and not args.no_dropin:
        line["dropin_c1"] = run_dropin_c1(dev)
    if rank == 0 and world == 1 and not args.no_cpu:
        line["cpu_baseline"] = cpu_baseline(cfg, H, W, batch, meta, args.cpu_tokens)
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()
    if rank == 0:
        print(json.dumps(line), flush=True)


def _k1_parts(n: int, v: int, d: int, sms: int = 148) -> int:
    """K1 partials per token (icepop_abi.cu k1_parts with the automatic run length)."""
    m_t, n_t, units = -(-n // 256), -(-v // 256), sms // 2
    r = 2
    while r > 1 and m_t * -(-n_t // r) < 16 * units:
        r //= 2
    return -(-n_t // r)


def kernel_times(H, W, batch, icfg, meta, cfg, chunk, dev, sp=False):
    """Average device time of K1(+K2), the dZ producer (K3 recompute GEMM, or the in-place
    pass over the stored probabilities), K4, K5 launched one by one on the torch stream. With
    stored probabilities in token chunks (chunk < N) they are timed on the first chunk."""
    import torch

    from paper_2510_18855_b200 import _lib
    from paper_2510_18855_b200.loss import PackedBatch, icepop_fwd

    lib = _lib.ensure_device(dev.index)
    st = torch.cuda.current_stream(dev)
    N, d, V = meta["n_local"], cfg["hidden"], cfg["vocab"]
    if sp and chunk < N:
        H = H[:chunk]
        batch = PackedBatch(batch.tokens[:chunk], batch.lp_train_old[:chunk], batch.lp_infer_old[:chunk],
                            batch.cu_seqlens, batch.group_offsets, batch.advantages, batch.rewards,
                            token_offset=batch.token_offset)
        N = chunk
    res = {}

    def timed(name, fn, flop, reps=2, nbytes=None, spin=8_000_000):
        fn()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        # a device spin ahead of the start event lets the host enqueue every rep first, so a
        # short kernel (K2: ~0.2 ms, less than one Python call's host time) is timed without the
        # host's call overhead between reps
        torch.cuda._sleep(spin)
        a.record(st)
        for _ in range(reps):
            fn()
        b.record(st)
        torch.cuda.synchronize()
        res[name] = {"ms": a.elapsed_time(b) / reps, "flop": flop, "count": 1}
        if nbytes is not None:
            res[name]["bytes"] = nbytes

    holder = {}

    def fwd():
        holder.clear()
        holder["f"] = icepop_fwd(H, W, batch, icfg, layout="vd", store_probs=sp, keep_workspace=True)

    timed("K1_fwd_lse+K2", fwd, 2.0 * N * d * V)
    f = holder["f"]
    # K2 alone (the IcePop epilogue over K1's run partials, re-run from the forward's workspace):
    # its HBM bytes per token are the partials (one per run of 2 vocabulary tiles, 12 B each) plus
    # the per-token inputs (tokens, ztok, lp_old, lp_inf: 24 B) and outputs (lse, lp_cur,
    # entropy, kept, calib, surrogate, coeff: 37 B)
    from paper_2510_18855_b200.loss import icepop_epilogue

    n_parts = _k1_parts(N, V, d)
    timed("K2_epilogue", lambda: icepop_epilogue(batch, f, icfg), 0.0, reps=10, spin=60_000_000,
          nbytes=N * (12 * n_parts + 24 + 37))
    res["K2_epilogue"]["n_partials_per_token"] = n_parts
    s = st.cuda_stream
    if sp:
        # the stored-probabilities backward with null gradients and its workspace runs only its
        # preparation (block lists, row scales and s*H, dZ of exception rows); K4/K5 follow as
        # plain GEMMs on the stored probabilities (their row-scale / one-hot epilogue work is
        # negligible). Repeated calls over the same buffers take the same time.
        from paper_2510_18855_b200.loss import _sp_workspace

        nc = N
        dz = f.extras["probs"]
        tm = f.extras["tile_max"]
        shape = _lib.Shape(n_tokens=N, token_offset=0, hidden=d, vocab=V, n_seqs=batch.n_seqs,
                           n_groups=batch.n_groups, weight_layout=_lib.W_VD)
        saved = _lib.Saved(tokens=batch.tokens.data_ptr(), lse=f.lse.data_ptr(), coeff=f.coeff.data_ptr(),
                           probs=dz.data_ptr(), tile_max=tm.data_ptr(), lp_cur=f.lp_cur.data_ptr())
        wsp = _sp_workspace(N, d, V, batch.n_seqs, dev)
        nbytes = 4 * N * d + 4 * N * tm.shape[1] + N
        if wsp is not None:
            timed("bwd_prep", lambda: _lib.check(lib.icepop_bwd_bf16(shape, icfg.to_c(), H.data_ptr(), W.data_ptr(),
                                                                     None, saved, -1.0, None, 0, None, 0,
                                                                     wsp.data_ptr(), wsp.numel(), s)),
                  0.0, nbytes=nbytes)
            del wsp
    else:
        nc = min(chunk, N)
        dz = torch.empty((nc, V), dtype=torch.bfloat16, device=dev)
        shape = _lib.Shape(n_tokens=nc, token_offset=0, hidden=d, vocab=V, n_seqs=batch.n_seqs,
                           n_groups=batch.n_groups, weight_layout=_lib.W_VD)
        saved = _lib.Saved(tokens=batch.tokens.data_ptr(), lse=f.lse.data_ptr(), coeff=f.coeff.data_ptr())
        timed("K3_dz", lambda: _lib.check(lib.icepop_dz_bf16(shape, 1.0, H.data_ptr(), W.data_ptr(), None, saved,
                                                             -1.0, dz.data_ptr(), V, s)),
              2.0 * nc * d * V)
    gh = torch.empty((nc, d), dtype=torch.bfloat16, device=dev)
    gw = torch.zeros((V, d), dtype=torch.float32, device=dev)
    timed("K4_dhidden", lambda: _lib.check(lib.icepop_gemm_bf16(dz.data_ptr(), W.data_ptr(), gh.data_ptr(), nc, d, V,
                                                                0, 1, 0, 0, s)), 2.0 * nc * d * V)
    # as in the step: a single (or first) chunk overwrites dW; recompute-mode later chunks accumulate.
    # The row-scaled stored-probabilities backward feeds K5 the scaled hidden transposed (K-major,
    # written by its prep kernel); the recompute mode reads H as it is (MN-major)
    k5_acc = 0 if (sp or nc >= N) else 1
    hk = H[:nc].t().contiguous() if sp else H
    timed("K5_dweight", lambda: _lib.check(lib.icepop_gemm_bf16(dz.data_ptr(), hk.data_ptr(), gw.data_ptr(), V, d, nc,
                                                                1, 0 if sp else 1, 1, k5_acc, s)), 2.0 * nc * d * V)
    del dz, gh, gw, hk
    holder.clear()
    return res


def run_e2e(H, W, batch, icfg, args, dev, world, sp=False, sp_chunk=0):
    """Public API from pinned host inputs: every step's inputs are copied H2D and its loss
    read back D2H inside the timed region. The copy of step k+1 runs on a side stream while
    step k computes (double-buffered device inputs, as a data-loader prefetch would)."""
    import torch
    import torch.distributed as dist

    from paper_2510_18855_b200.distributed import allreduce_grad, allreduce_stats, wait_grad
    from paper_2510_18855_b200.loss import PackedBatch, icepop_bwd, icepop_fwd, icepop_fwd_bwd

    host = {k: v.cpu().pin_memory() for k, v in dict(H=H, tokens=batch.tokens, lp_old=batch.lp_train_old,
                                                     lp_inf=batch.lp_infer_old, cu=batch.cu_seqlens,
                                                     go=batch.group_offsets, rewards=batch.rewards).items()}
    bufs = [{k: torch.empty_like(v, device=dev) for k, v in host.items()} for _ in range(2)]
    h2d = sum(v.numel() * v.element_size() for v in host.values())
    out_host = torch.empty(8, dtype=torch.float64).pin_memory()
    # the first step's copy cannot overlap anything: time 16 to 32 steps so that this start-up
    # exposure (~40 ms at C2) stays small (every step's copy is still inside the timed region)
    steps = max(16, min(args.steps, 32))
    main = torch.cuda.current_stream(dev)
    copy_stream = torch.cuda.Stream(dev)
    copied = [torch.cuda.Event(), torch.cuda.Event()]
    consumed = [torch.cuda.Event(), torch.cuda.Event()]
    for e in consumed:
        e.record(main)

    def issue_copy(k):
        i = k % 2
        with torch.cuda.stream(copy_stream):
            copy_stream.wait_event(consumed[i])
            for name in host:
                bufs[i][name].copy_(host[name], non_blocking=True)
            copied[i].record(copy_stream)

    last = {}

    def compute(k):
        i = k % 2
        main.wait_event(copied[i])
        d = bufs[i]
        b = PackedBatch(d["tokens"], d["lp_old"], d["lp_inf"], d["cu"], d["go"], None, d["rewards"], batch.token_offset)
        if sp_chunk:
            f, _, g = icepop_fwd_bwd(d["H"], W, b, icfg, layout="vd", grad_scale=-1.0, max_chunk_tokens=sp_chunk)
            last["chunks"] = f.extras.get("chunks", 1)
        else:
            f = icepop_fwd(d["H"], W, b, icfg, layout="vd", store_probs=sp)
            _, g = icepop_bwd(d["H"], W, b, f, icfg, layout="vd", grad_scale=-1.0)
        if world > 1:
            allreduce_stats(f.stats)
            wait_grad(allreduce_grad(g))
        consumed[i].record(main)
        out_host.copy_(f.stats, non_blocking=True)

    issue_copy(0)  # warm-up step (untimed)
    compute(0)
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(main)
    copy_stream.wait_event(a)  # no copy of the timed steps starts before the timed region
    issue_copy(0)
    for k in range(steps):
        if k + 1 < steps:
            issue_copy(k + 1)
        compute(k)
    b.record(main)
    torch.cuda.synchronize()
    ms = a.elapsed_time(b) / steps
    t = torch.tensor([ms], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    ms = float(t.item())
    out = {"value": round(H.shape[0] * world / (ms / 1e3), 1), "unit": UNIT, "h2d_bytes_per_step": int(h2d),
           "d2h_bytes_per_step": 64, "ms_per_step": round(ms, 3), "steps": steps,
           "note": "pinned host inputs; step k+1's H2D overlaps step k on a copy stream"}
    if "chunks" in last:
        out["token_chunks"] = last["chunks"]
    return out


# ----------------------------------------------------------------------------- reference-facing API
def run_dropin_c1(dev, reps: int = 12) -> dict:
    """BASELINE configs[0] (8 x 512 tokens, 1,024 features, V = 32,768, one GRPO group of 8)
    through the drop-in ``objective_and_grad`` -- the call the reference's own loop makes
    (scheduler.py:540-542) -- with its Python records and host fp64 weights in, the fp64
    gradient and per-token diagnostics out, and the lp_cur write-back into every TokenRecord:
    wall clock per call (median), bf16 tensor-core path, with a fresh gradient array and with a
    reused ``grad_out``."""
    import copy
    from dataclasses import dataclass

    import torch

    from paper_2510_18855_b200 import objective as O

    @dataclass
    class Task:
        prompt_id: int

    @dataclass
    class Rollout:
        tokens: list

    @dataclass
    class Params:
        weights: np.ndarray
        version_id: int = 0

        @property
        def n_features(self):
            return self.weights.shape[0]

    rng = np.random.default_rng(0)
    S, T, nf, V = 8, 512, 1024, 32768
    w = rng.normal(0.0, 0.8, (nf, V))
    task = Task(prompt_id=17)
    rollouts = []
    for _ in range(S):
        lp = rng.normal(-10.4, 0.3, T)
        inf = lp - rng.normal(0, 0.233, T)
        rollouts.append(Rollout([O.TokenRecord(int(y), float(b), float(a), float(a), 0)
                                 for y, a, b in zip(rng.integers(0, V, T), lp, inf)]))
    rewards = [float(x) for x in rng.integers(0, 2, S)]
    groups = [O.PromptGroup(task=task, rollouts=rollouts, rewards=rewards,
                            advantages=list(O.group_advantages(rewards)) if len(set(rewards)) > 1 else [0.0] * S)]
    theta = Params(w)
    cfg, bounds = O.ObjectiveConfig(), O.MaskingBounds()
    buf = np.empty_like(w)
    out = {}
    with torch.cuda.device(dev):
        for name, kw in (("fresh_grad", {}), ("grad_out", {"grad_out": buf})):
            r = None
            for _ in range(3):  # steady state: the caller holds the previous result (two gradient buffers)
                r = O.objective_and_grad(copy.deepcopy(groups), theta, theta, None, cfg, bounds, precision="bf16", **kw)
            ts = []
            for _ in range(reps):
                gs = copy.deepcopy(groups)
                t0 = time.perf_counter()
                r = O.objective_and_grad(gs, theta, theta, None, cfg, bounds, precision="bf16", **kw)
                ts.append(time.perf_counter() - t0)
            ms = 1e3 * float(np.median(ts))
            out[name] = {"ms_per_call": round(ms, 2), "value": round(S * T / (ms / 1e3), 1)}
    return {"unit": UNIT, "config": "C1: 8 x 512 tokens, n_features 1,024, V 32,768, 1 GRPO group of 8 (synthetic)",
            "h2d_bytes_per_call": int(nf * V * 2 + S * T * (4 + 8 + 8 + 8 * 4)),
            "d2h_bytes_per_call": int(nf * V * 8 + S * T * 8 * 4),
            "token_count": r.token_count, "calls": reps, **out,
            "note": "wall clock of objective_and_grad(precision='bf16'): record packing, H2D of the bf16 "
                    "weights (cast on the host into pinned memory), multi-hot H on the device, the fused "
                    "fwd+bwd kernels, D2H of the fp64 gradient and the per-token diagnostics, write-back"}


# ----------------------------------------------------------------------------- CPU baseline
def cpu_sample(cfg, n_tokens, seed=0):
    """A bounded host sample of the same workload: 1 group of 2 sequences."""
    rng = np.random.default_rng(seed)
    d, V = cfg["hidden"], cfg["vocab"]
    T = max(1, n_tokens // 2)
    H = rng.standard_normal((2 * T, d), dtype=np.float32).astype(np.float64)
    tokens = rng.integers(0, V, 2 * T).astype(np.int32)
    lp_old = rng.normal(-12.0, 0.3, 2 * T)
    lp_inf = lp_old - rng.normal(0, cfg["sigma_inf"], 2 * T)
    return H, tokens, lp_old, lp_inf, np.array([0, T, 2 * T], dtype=np.int32), np.array([0, 2], dtype=np.int32), \
        np.array([1.0, -1.0])


def time_oracle(cfg, n_tokens, W64, seed=0):
    from oracle.icepop_oracle import icepop_dense

    H, tok, lpo, lpi, cu, go, adv = cpu_sample(cfg, n_tokens, seed)
    t0 = time.perf_counter()
    icepop_dense(H, W64, tok, lpo, lpi, cu, go, adv, layout="vd")
    return time.perf_counter() - t0, len(tok)


def blas_threads() -> int:
    try:
        from threadpoolctl import threadpool_info

        n = [i.get("num_threads", 0) for i in threadpool_info() if i.get("user_api") == "blas"]
        return max(n) if n else 1
    except Exception:  # noqa: BLE001
        return os.cpu_count() or 1


def sample_tokens(cfg, W64, target_s: float) -> int:
    """Tokens per CPU sample so one sample takes about target_s. A call costs a + b*n: a fixed
    part (the fp64 V x d gradient buffer the reference also allocates per call) plus a
    per-token part. Fit both from two timed sizes so the sample is large enough that the
    measured throughput approaches the per-token rate (a small sample would understate the
    CPU and overstate the GPU's speed-up)."""
    n1, n2 = 32, 256
    time_oracle(cfg, 16, W64, seed=997)  # warm-up: first-touch of the fp64 buffers, BLAS threads
    t1, _ = time_oracle(cfg, n1, W64, seed=998)
    t2, _ = time_oracle(cfg, n2, W64, seed=999)
    # slope floor 1 ms/token (measured 5-7 ms on the pool's hosts): a noisy fit cannot blow the
    # sample up past ~target_s / 1 ms tokens
    b = max((t2 - t1) / (n2 - n1), 1e-3)
    a = max(t1 - b * n1, 0.0)
    n = int(max(n2, min(8192, (target_s - a) / b)))
    return n + n % 2


def cpu_baseline(cfg, H, W, batch, meta, n_tokens):
    W64 = W.float().cpu().numpy().astype(np.float64)
    n_tokens = n_tokens or sample_tokens(cfg, W64, 20.0)  # ~10-30 s of CPU work
    dt, n = time_oracle(cfg, n_tokens, W64)
    return {"value": round(n / dt, 3), "unit": UNIT, "cores": blas_threads(), "kind": "port",
            "sample": f"{n} tokens (1 group x 2 seqs) at d={cfg['hidden']}, V={cfg['vocab']}, fp64 numpy oracle "
                      f"(objective.py:172-298 restated densely, oracle/icepop_oracle.py), {dt:.1f} s"}


def time_reference_own(cfg, target_s: float = 10.0, seed: int = 0):
    """The unmodified reference's own objective_and_grad (the baseline/_ref install, imported
    as a package, none of our code on the path) on one group of 2 synthetic rollouts at the
    config's vocabulary with n_features = d. Its policy is a 4-hot gather (policy.py:279-289),
    so a token costs O(V) regardless of d, plus np.add.at into the full [d, V] gradient
    (objective.py:265-266). Sized like the oracle sample (fixed + per-token fit). None if the
    reference is not installed."""
    ref_dir = ROOT / "baseline" / "_ref"
    if not (ref_dir / "mismatchlab").exists():
        return None
    if str(ref_dir) not in sys.path:
        sys.path.insert(0, str(ref_dir))
    import mismatchlab as ml
    from mismatchlab.tasks import TaskKind

    rng = np.random.default_rng(seed)
    d, V = cfg["hidden"], cfg["vocab"]
    theta = ml.PolicyParams(weights=rng.standard_normal((d, V), dtype=np.float32).astype(np.float64) * 0.02)
    ocfg = ml.ObjectiveConfig(group_size=2)

    def call(n_tok):
        task = ml.TaskSpec(TaskKind.PARITY_MATCH, 100, 0, 4)
        rollouts = []
        for r in range(2):
            recs = []
            for _ in range(max(1, n_tok // 2)):
                lp_old = float(-np.log(V) + rng.normal(0, 0.3))
                recs.append(ml.TokenRecord(token=int(rng.integers(0, V)), logp_infer_old=lp_old - float(rng.normal(0, 0.2)),
                                           logp_train_old=lp_old, logp_train_cur=lp_old, gen_version=0))
            rollouts.append(ml.Rollout(task=task, stream=np.random.default_rng(r), uid=r, group_uid=0, tokens=recs,
                                       terminal=True))
        group = ml.PromptGroup(task=task, rollouts=rollouts, rewards=[1.0, 0.0], advantages=[1.0, -1.0])
        t0 = time.perf_counter()
        ml.objective_and_grad([group], theta, theta, None, ocfg, ml.MaskingBounds())
        return time.perf_counter() - t0, 2 * max(1, n_tok // 2)

    t1, n1 = call(8)
    t2, n2 = call(64)
    b = max((t2 - t1) / (n2 - n1), 1e-6)
    a = max(t1 - b * n1, 0.0)
    n = int(max(64, min(4096, (target_s - a) / b)))
    dt, n = call(n)
    return {"value": round(n / dt, 3), "unit": UNIT, "cores": 1, "kind": "reference",
            "sample": f"{n} tokens (1 group x 2 synthetic rollouts), n_features = d = {d}, V = {V}, "
                      f"unmodified mismatchlab.objective_and_grad (baseline/_ref), {dt:.1f} s",
            "note": "the reference's own 4-hot-gather numpy path (single-threaded); the line's value is "
                    "the dense fp64 restatement on all cores (faster, so the conservative baseline)"}


def run_reference(args):
    """--impl reference: the reference's algorithm on host cores (rank 0 only)."""
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    if rank != 0:
        return
    cfg = CONFIGS[args.config]
    try:  # torchrun sets OMP_NUM_THREADS=1; rank 0 alone runs here, so give BLAS every host core
        from threadpoolctl import threadpool_limits

        threadpool_limits(os.cpu_count())
    except Exception:  # noqa: BLE001
        pass
    rng = np.random.default_rng(123)
    W64 = (rng.standard_normal((cfg["vocab"], cfg["hidden"]), dtype=np.float32) * (2.0 / np.sqrt(cfg["hidden"]))
           ).astype(np.float64)
    # Each timed step is one call on a token sample sized so the whole run takes ~2.5 minutes
    # (8-30 s per step): the larger the sample, the better the call's fixed part (the fp64 V x d
    # gradient buffer the reference allocates per call, ~3 s at C2) is amortised, as it would be
    # over a full batch. Warm-up steps only warm BLAS threads and the buffers: small samples.
    target_s = min(30.0, max(8.0, 150.0 / max(args.steps, 1)))
    n_tok = args.cpu_tokens or sample_tokens(cfg, W64, target_s)
    for i in range(args.warmup):
        time_oracle(cfg, min(n_tok, 64), W64, seed=i)
    tot_t, tot_n = 0.0, 0
    for i in range(args.steps):
        dt, n = time_oracle(cfg, n_tok, W64, seed=100 + i)
        tot_t += dt
        tot_n += n
    value = tot_n / tot_t
    line = {
        "metric": METRIC, "value": round(value, 3), "unit": UNIT, "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": round(1e3 * tot_t / args.steps, 3), "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic (seeded)", "impl": "reference",
        "config": {"workload": CONFIGS[args.config]["name"], "hidden": cfg["hidden"], "vocab": cfg["vocab"],
                   "parallelism": "host cores (numpy/OpenBLAS)"},
        "cpu_baseline": {"value": round(value, 3), "unit": UNIT, "cores": blas_threads(), "kind": "port",
                         "sample": f"{n_tok} tokens per step (1 group x 2 seqs), fp64 numpy restatement "
                                   "of objective.py:172-298 (oracle/icepop_oracle.py)"},
        "e2e": {"value": round(value, 3), "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    try:  # the reference's own objective_and_grad, reported beside the port
        own = time_reference_own(cfg)
        if own:
            line["reference_own"] = own
    except Exception as e:  # noqa: BLE001 - informational only
        line["reference_own"] = {"unavailable": f"{type(e).__name__}: {e}"[:200]}
    print(json.dumps(line), flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--config", choices=sorted(CONFIGS), default="c2")
    ap.add_argument("--cpu-tokens", type=int, default=0, help="CPU sample size (0 = size it to a few seconds)")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--no-kernel-timing", action="store_true")
    ap.add_argument("--no-onpolicy", action="store_true")
    ap.add_argument("--no-recompute", action="store_true", help="skip the recompute-mode sub-record")
    ap.add_argument("--no-dropin", action="store_true", help="skip the reference-API (objective_and_grad) record")
    ap.add_argument("--no-ref-diag", action="store_true", help="skip the ref-passed (gamma = 0) sub-record")
    ap.add_argument("--seqs", type=int, default=0,
                    help="override the config's sequences per rank (e.g. the C5 sweep: 16/32/64/128/256)")
    ap.add_argument("--zero-adv-frac", type=float, default=0.0,
                    help="fraction of prompt groups with identical rewards (zero advantages)")
    ap.add_argument("--dw-collective", choices=["fused", "nccl"], default="fused",
                    help="N>1: dW reduce-scatter fused into K5 over NVLink, or NCCL all-reduce")
    ap.add_argument("--dry-run", action="store_true",
                    help="CPU only: launch the ranks over gloo and run the host-side plumbing (shards, "
                         "stats all-reduce, max-over-ranks timing) without any GPU work")
    args = ap.parse_args()
    if args.gpus < 1:
        ap.error("--gpus must be >= 1")
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        sys.exit(self_launch(args))  # one process per GPU, as the driver's torchrun does
    world = int(os.environ.get("WORLD_SIZE", "1"))
    if world != args.gpus:
        print(f"bench.py: --gpus {args.gpus} but WORLD_SIZE={world}; refusing to time a different "
              "number of ranks than requested", file=sys.stderr)
        sys.exit(2)
    if args.warmup < 3 and args.impl == "ours":
        print("warning: the timing rules ask for >= 3 warm-up steps", file=sys.stderr)
    if args.impl == "reference":
        run_reference(args)
    elif args.dry_run:
        run_dry(args)
    else:
        run_ours(args)


def self_launch(args) -> int:
    """`bench.py --gpus N` without torchrun: start N ranks (one process per GPU) with
    torch.distributed.run on 127.0.0.1 and return its exit code. Refuses, never silently runs
    fewer ranks, when fewer than N GPUs are visible (the reference arm needs no GPU; the gloo
    dry run none either)."""
    n = args.gpus
    if args.impl == "ours" and not args.dry_run:
        import torch

        have = torch.cuda.device_count()
        if have < n:
            print(f"bench.py: --gpus {n} needs {n} visible GPUs, found {have}; refusing", file=sys.stderr)
            return 2
    env = dict(os.environ)
    env.setdefault("NCCL_DEBUG", "INFO")  # the driver checks nranks=N in NCCL's init lines
    env.setdefault("NCCL_DEBUG_SUBSYS", "INIT")
    env.setdefault("OMP_NUM_THREADS", "4")
    import socket

    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={n}",
           "--master-addr=127.0.0.1", f"--master-port={port}", str(Path(__file__).resolve())] + sys.argv[1:]
    return subprocess.call(cmd, env=env)


def run_dry(args):
    """--dry-run: every rank joins a gloo group, takes its token shard of the config's batch,
    all-reduces a stats vector (the fp64 statistics exchange) and the max of its host-timed
    no-op step (the bench's max-over-ranks rule); rank 0 prints the line. No GPU work, no
    throughput claim: it proves the launcher and the rank plumbing."""
    import torch
    import torch.distributed as dist

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    if world > 1:
        dist.init_process_group("gloo")
    cfg = dict(CONFIGS[args.config])
    meta = make_batch_host(cfg, rank, world, args.zero_adv_frac)
    stats = torch.zeros(8, dtype=torch.float64)
    stats[2] = meta["n_local"]
    t0 = time.perf_counter()
    if world > 1:
        dist.all_reduce(stats)
    ms = torch.tensor([1e3 * (time.perf_counter() - t0)], dtype=torch.float64)
    ranks = torch.tensor([rank, meta["token_offset"], meta["n_local"]], dtype=torch.int64)
    gathered = [torch.zeros_like(ranks) for _ in range(world)]
    if world > 1:
        dist.all_reduce(ms, op=dist.ReduceOp.MAX)
        dist.all_gather(gathered, ranks)
    else:
        gathered = [ranks]
    if rank == 0:
        print(json.dumps({"metric": METRIC, "dry_run": True, "value": None, "unit": UNIT, "n_gpus": world,
                          "ranks": [{"rank": int(g[0]), "token_offset": int(g[1]), "tokens": int(g[2])}
                                    for g in gathered],
                          "global_tokens": int(stats[2].item()), "ms_allreduce_max": round(float(ms.item()), 3),
                          "config": {"workload": cfg["name"], "parallelism": f"dp{world} token-sharded",
                                     "backend": "gloo"}}), flush=True)
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
