"""Generate the golden vectors that pin the oracle and the CUDA path.

Runs ONLY in the build container, where the unmodified reference is importable from
/root/reference/pkg/src (it does not exist on the GPU box; the .npz files produced
here travel instead). Every output is computed by the reference's own
``objective_and_grad`` (objective.py:172-298) / ``group_advantages``
(objective.py:153-159) on batches built through the reference's real rollout path
(scheduler.run_iteration), exactly as its test_objective.py:42-53 ``make_batch`` does.

Weights are rounded to bf16-representable fp64 values before the reference sees them,
so one fixture checks both the fp64 validation path (tight tolerance) and the bf16
tensor-core path (H = multihot(feats) is exact in bf16).

    PYTHONDONTWRITEBYTECODE=1 PYTHONPATH=/root/reference/pkg/src python tests/golden/make_golden.py
"""

from __future__ import annotations

import math
import sys
from pathlib import Path

import numpy as np
import torch

REF_SRC = Path("/root/reference/pkg/src")
OUT = Path(__file__).resolve().parent

sys.path.insert(0, str(REF_SRC))
from mismatchlab import (  # noqa: E402
    Algo,
    BudgetConfig,
    Context,
    MaskingBounds,
    ObjectiveConfig,
    PolicyParams,
    PromptGroup,
    Rollout,
    SyntheticPromptSource,
    TaskSpec,
    TokenRecord,
    Vocabulary,
    group_advantages,
    infer_engine,
    init_params,
    log_prob,
    make_state,
    objective_and_grad,
    run_iteration,
    train_engine,
)
from mismatchlab.objective import _rollout_feats  # noqa: E402
from mismatchlab.tasks import TaskKind  # noqa: E402


def bf16_exact(w: np.ndarray) -> np.ndarray:
    return torch.from_numpy(w).to(torch.bfloat16).to(torch.float64).numpy()


def rollout_batch(seed, scale, vocab_size, max_len, n_features, budget, prompts, group_size, init_scale=0.7):
    vocab = Vocabulary(size=vocab_size)
    engine = infer_engine(scale, 7)
    params = init_params(vocab, n_features=n_features, init_scale=init_scale, seed=seed)
    source = SyntheticPromptSource(vocab, max_len=max_len)
    state = make_state(seed, vocab, engine, source)
    cfg = BudgetConfig(token_budget=budget, infer_capacity=max(8, prompts * group_size), prompts_per_iteration=prompts)
    _, groups = run_iteration(state, params, cfg, ObjectiveConfig(group_size=group_size))
    assert groups
    # Binary task rewards are often constant within a group (all advantages 0, J = 0);
    # re-draw continuous rewards so every group carries signal, with the reference's own
    # group_advantages producing the advantages.
    rng = np.random.default_rng(seed + 1000)
    for g in groups:
        g.rewards = [float(x) for x in rng.normal(0.5, 0.5, len(g.rollouts))]
        g.advantages = [float(a) for a in group_advantages(g.rewards)]
    return params, groups


def manual_group(theta, specs, advantages):
    """test_objective.py:56-77: single-token rollouts with crafted (token, calib, ratio)."""
    task = TaskSpec(TaskKind.PARITY_MATCH, 100, 0, 4)
    rollouts = []
    for token, calib, ratio in specs:
        ctx = Context(task.prompt_id, ())
        lp_cur = log_prob(theta, ctx, token, train_engine())
        lp_old = lp_cur - math.log(ratio)
        rec = TokenRecord(token=token, logp_infer_old=lp_old - math.log(calib), logp_train_old=lp_old,
                          logp_train_cur=lp_cur, gen_version=theta.version_id)
        rollouts.append(Rollout(task=task, stream=np.random.default_rng(0), uid=0, group_uid=0, tokens=[rec],
                                terminal=True))
    return PromptGroup(task=task, rollouts=rollouts, rewards=[0.0] * len(specs), advantages=advantages)


def pack(groups, n_features):
    feats, tokens, lp_old, lp_inf, cu, go, adv, rew, pid = [], [], [], [], [0], [0], [], [], []
    for g in groups:
        for rollout, a, r in zip(g.rollouts, g.advantages, g.rewards):
            f = _rollout_feats(g.task, rollout.tokens, n_features)
            feats.append(f)
            tokens += [rec.token for rec in rollout.tokens]
            lp_old += [rec.logp_train_old for rec in rollout.tokens]
            lp_inf += [rec.logp_infer_old for rec in rollout.tokens]
            cu.append(cu[-1] + len(rollout.tokens))
            adv.append(a)
            rew.append(r)
            pid.append(g.task.prompt_id)
        go.append(go[-1] + len(g.rollouts))
    return dict(
        feats=np.concatenate(feats).astype(np.int64),
        tokens=np.asarray(tokens, dtype=np.int32),
        lp_train_old=np.asarray(lp_old),
        lp_infer_old=np.asarray(lp_inf),
        cu_seqlens=np.asarray(cu, dtype=np.int32),
        group_offsets=np.asarray(go, dtype=np.int32),
        advantages=np.asarray(adv),
        rewards=np.asarray(rew),
        prompt_ids=np.asarray(pid, dtype=np.int64),
    )


def run_case(name, groups, theta, theta_old, ref, algo, kl_coeff, temperature, bounds=MaskingBounds(0.5, 5.0),
             clip_eps=0.2, tis_cap=2.0):
    g_size = max(2, len(groups[0].rollouts))
    cfg = ObjectiveConfig(algo=algo, kl_coeff=kl_coeff, group_size=g_size, clip_eps=clip_eps, tis_cap=tis_cap)
    out = objective_and_grad(groups, theta, theta_old, ref, cfg, bounds, temperature)
    lp_written = np.asarray([rec.logp_train_cur for g in groups for r in g.rollouts for rec in r.tokens])
    data = pack(groups, theta.n_features)
    data.update(
        weight=theta.weights,
        weight_ref=(ref.weights if ref is not None else np.zeros((0, 0))),
        has_ref=np.asarray(ref is not None),
        alpha=np.asarray(bounds.alpha),
        beta=np.asarray(bounds.beta),
        clip_eps=np.asarray(clip_eps),
        tis_cap=np.asarray(tis_cap),
        temperature=np.asarray(temperature),
        kl_coeff=np.asarray(kl_coeff),
        algo=np.asarray(algo.value),
        out_objective=np.asarray(out.objective_value),
        out_kept=out.per_token_mask_kept,
        out_clipped_fraction=np.asarray(out.clipped_fraction),
        out_grad=out.grad,
        out_kl_to_ref=np.asarray(out.kl_to_ref),
        out_token_count=np.asarray(out.token_count),
        out_mean_logp=np.asarray(out.mean_logp),
        out_entropy_all=np.asarray(out.entropy_all),
        out_entropy_clipped=np.asarray(out.entropy_clipped),
        out_surrogate=out.per_token_surrogate,
        out_calibration=out.per_token_calibration,
        out_entropy=out.per_token_entropy,
        out_lp_cur=lp_written,
    )
    np.savez_compressed(OUT / f"{name}.npz", **data)
    print(f"{name}: tokens={out.token_count} popped={int((~out.per_token_mask_kept).sum())} "
          f"J={out.objective_value:.6g} |grad|={out.grad_norm:.4g}")


def perturbed(params, sigma, seed):
    rng = np.random.default_rng(seed)
    return PolicyParams(bf16_exact(params.weights + rng.normal(0, sigma, params.weights.shape)), params.version_id)


def main() -> None:
    # 1. test_objective.py-style small batch (FD-test shapes, vocab rounded up to 8)
    params, groups = rollout_batch(seed=11, scale=0.12, vocab_size=8, max_len=4, n_features=16, budget=30,
                                   prompts=3, group_size=2)
    params = PolicyParams(bf16_exact(params.weights), params.version_id)
    theta = perturbed(params, 0.05, 1)
    ref = PolicyParams(bf16_exact(init_params(Vocabulary(size=8), n_features=16, init_scale=0.5, seed=99).weights))
    for algo in Algo:
        run_case(f"small_{algo.value}", groups, theta, params, None, algo, 0.0, 1.0)
    run_case("small_icepop_kl", groups, theta, params, ref, Algo.ICEPOP, 0.4, 1.0)
    run_case("small_icepop_refdiag", groups, theta, params, ref, Algo.ICEPOP, 0.0, 1.0)

    # 2. medium batch with real mismatch: popped tokens and clipped ratios
    params, groups = rollout_batch(seed=5, scale=0.03, vocab_size=64, max_len=24, n_features=64, budget=600,
                                   prompts=6, group_size=4, init_scale=0.9)
    params = PolicyParams(bf16_exact(params.weights), params.version_id)
    theta = perturbed(params, 0.25, 2)
    run_case("medium_icepop", groups, theta, params, None, Algo.ICEPOP, 0.0, 1.0)
    run_case("medium_tis", groups, theta, params, None, Algo.TIS, 0.0, 1.0)
    run_case("medium_icepop_narrow", groups, theta, params, None, Algo.ICEPOP, 0.0, 1.0,
             bounds=MaskingBounds(0.8, 1.25))

    # 3. temperature != 1
    params, groups = rollout_batch(seed=7, scale=0.06, vocab_size=16, max_len=12, n_features=32, budget=200,
                                   prompts=4, group_size=3)
    params = PolicyParams(bf16_exact(params.weights), params.version_id)
    theta = perturbed(params, 0.1, 3)
    run_case("temp_icepop", groups, theta, params, None, Algo.ICEPOP, 0.0, 0.7)

    # 4. crafted clip / mask cases (test_objective.py:238-270)
    theta = PolicyParams(bf16_exact(init_params(Vocabulary(size=8), n_features=16, init_scale=0.4, seed=10).weights))
    g = manual_group(theta, [(1, 1.0, 1.35), (2, 1.0, 0.7), (3, 0.2, 1.0), (4, 9.0, 1.0), (5, 1.2, 1.1),
                             (6, 0.5, 1.0), (7, 5.0, 0.9)],
                     advantages=[1.0, -1.0, 0.5, -0.5, 1.0, 0.25, -0.75])
    run_case("manual_clip", [g], theta, theta, None, Algo.ICEPOP, 0.0, 1.0)

    # 5. group advantages (objective.py:153-159), bit-exact targets
    rng = np.random.default_rng(0)
    sets = [[1.0, 1.0, 1.0, 1.0], [1.0, 0.0], [1e-7, 0.0], list(rng.integers(0, 2, 8).astype(float)),
            list(rng.normal(0, 1, 8)), list(rng.normal(3, 2, 16)), list(rng.random(200)), list(rng.random(3))]
    rewards = np.concatenate([np.asarray(s, dtype=np.float64) for s in sets])
    offsets = np.cumsum([0] + [len(s) for s in sets]).astype(np.int32)
    adv = np.concatenate([group_advantages(s) for s in sets])
    np.savez_compressed(OUT / "advantages.npz", rewards=rewards, group_offsets=offsets, advantages=adv)
    print(f"advantages: {len(sets)} groups")


C1_SEQS, C1_LEN, C1_D, C1_V = 8, 512, 1024, 32768
C1_W_SEED, C1_W_SCALE, C1_PROJ_SEED = 2510, 0.8, 7


def c1_weights() -> np.ndarray:
    """BASELINE configs[0]'s weights, regenerated identically by tests/test_parity_gpu.py
    (numpy PCG64 is platform-independent), so the 268 MB matrix never enters the repo."""
    w = np.random.default_rng(C1_W_SEED).normal(0.0, C1_W_SCALE, (C1_D, C1_V))
    return bf16_exact(w)


def c1_case() -> None:
    """BASELINE configs[0] at full size, through the reference's own objective_and_grad: one
    GRPO group of 8 rollouts x 512 tokens, n_features (hidden) 1,024, vocab 32,768, default
    alpha/beta, IcePop. lp_train_old = lp_cur + N(0, 0.1) (from a first reference pass, which
    writes logp_train_cur back into the records) and lp_infer_old = lp_train_old - N(0, 0.233),
    as in SURVEY.md 8d. The gradient is stored as its Frobenius norm and a fixed random
    projection (grad @ R, R ~ N(0, 1) [V, 4]) instead of 268 MB of fp64."""
    rng = np.random.default_rng(123)
    theta = PolicyParams(c1_weights(), 0)
    task = TaskSpec(TaskKind.PARITY_MATCH, 4242, 0, C1_LEN)
    rollouts = []
    for i in range(C1_SEQS):
        toks = rng.integers(0, C1_V, C1_LEN)
        recs = [TokenRecord(token=int(t), logp_infer_old=0.0, logp_train_old=0.0, logp_train_cur=0.0, gen_version=0)
                for t in toks]
        rollouts.append(Rollout(task=task, stream=np.random.default_rng(i), uid=i, group_uid=0, tokens=recs,
                                terminal=True))
    rewards = [float(x) for x in rng.normal(0.5, 0.5, C1_SEQS)]
    group = PromptGroup(task=task, rollouts=rollouts, rewards=rewards,
                        advantages=[float(a) for a in group_advantages(rewards)])
    cfg = ObjectiveConfig(algo=Algo.ICEPOP, group_size=C1_SEQS)
    bounds = MaskingBounds(0.5, 5.0)
    objective_and_grad([group], theta, theta, None, cfg, bounds, 1.0)  # writes logp_train_cur
    for r in rollouts:
        for rec in r.tokens:
            rec.logp_train_old = rec.logp_train_cur + float(rng.normal(0.0, 0.1))
            rec.logp_infer_old = rec.logp_train_old - float(rng.normal(0.0, 0.233))
    out = objective_and_grad([group], theta, theta, None, cfg, bounds, 1.0)
    lp_written = np.asarray([rec.logp_train_cur for r in rollouts for rec in r.tokens])
    data = pack([group], C1_D)
    proj = np.random.default_rng(C1_PROJ_SEED).standard_normal((C1_V, 4))
    data.update(
        out_kept=out.per_token_mask_kept,
        out_lp_cur=lp_written,
        out_surrogate=out.per_token_surrogate,
        out_calibration=out.per_token_calibration,
        out_entropy=out.per_token_entropy,
        out_objective=np.asarray(out.objective_value),
        out_clipped_fraction=np.asarray(out.clipped_fraction),
        out_token_count=np.asarray(out.token_count),
        out_mean_logp=np.asarray(out.mean_logp),
        out_entropy_all=np.asarray(out.entropy_all),
        out_grad_norm=np.asarray(np.linalg.norm(out.grad)),
        out_grad_proj=out.grad @ proj,
    )
    np.savez_compressed(OUT / "c1_config0.npz", **data)
    print(f"c1_config0: tokens={out.token_count} popped={int((~out.per_token_mask_kept).sum())} "
          f"J={out.objective_value:.6g} |grad|={out.grad_norm:.4g}")


C2S_SEQS, C2S_LEN, C2S_D, C2S_V = 8, 4096, 4096, 157184
C2S_W_SEED, C2S_W_SCALE = 2511, 0.5


def c2s_weights() -> np.ndarray:
    """Weights of the C2-width slice (n_features = d = 4,096, V = 157,184), regenerated by the
    GPU test from the same seed."""
    w = np.random.default_rng(C2S_W_SEED).normal(0.0, C2S_W_SCALE, (C2S_D, C2S_V))
    return bf16_exact(w)


def c2_slice_case(name: str = "c2_slice", d: int = C2S_D, seq_len: int = C2S_LEN, w_seed: int = C2S_W_SEED,
                  w_scale: float = C2S_W_SCALE, kl_coeff: float = 0.0, ref_seed: int | None = None,
                  algo: Algo = Algo.ICEPOP, temperature: float = 1.0) -> None:
    """One GRPO group (8 rollouts x 4,096 tokens = 32,768 tokens) at BASELINE configs[1]'s full
    width (hidden 4,096, vocab 157,184) through the reference's own objective_and_grad (one
    pass, ~10 min on one core: a 4-hot gather and np.add.at over T x V per rollout). lp_train_old
    comes from the same 4-hot logits (policy.py:279-289, computed here with numpy) plus N(0, 0.1),
    lp_infer_old = lp_train_old - N(0, 0.233). Stored like c1_config0 (gradient norm and
    projection)."""
    rng = np.random.default_rng(321)
    theta = PolicyParams(bf16_exact(np.random.default_rng(w_seed).normal(0.0, w_scale, (d, C2S_V))), 0)
    task = TaskSpec(TaskKind.PARITY_MATCH, 5151, 0, seq_len)
    toks_all = rng.integers(0, C2S_V, (C2S_SEQS, seq_len))
    rollouts = []
    for i in range(C2S_SEQS):
        recs = [TokenRecord(token=int(t), logp_infer_old=0.0, logp_train_old=0.0, logp_train_cur=0.0, gen_version=0)
                for t in toks_all[i]]
        rollouts.append(Rollout(task=task, stream=np.random.default_rng(i), uid=i, group_uid=0, tokens=recs,
                                terminal=True))
        feats = _rollout_feats(task, recs, d)
        z = (theta.weights[feats[:, 0]] + theta.weights[feats[:, 1]] + theta.weights[feats[:, 2]] +
             theta.weights[feats[:, 3]]) / temperature
        m = z.max(axis=1)
        lse = m + np.log(np.exp(z - m[:, None]).sum(axis=1))
        lp = z[np.arange(seq_len), toks_all[i]] - lse
        del z
        for rec, l in zip(recs, lp):
            rec.logp_train_old = float(l) + float(rng.normal(0.0, 0.1))
            rec.logp_infer_old = rec.logp_train_old - float(rng.normal(0.0, 0.233))
    rewards = [float(x) for x in rng.normal(0.5, 0.5, C2S_SEQS)]
    group = PromptGroup(task=task, rollouts=rollouts, rewards=rewards,
                        advantages=[float(a) for a in group_advantages(rewards)])
    ref = None
    if ref_seed is not None:  # KL-to-ref term (objective.py:254-263) against a perturbed reference policy
        ref = PolicyParams(bf16_exact(theta.weights + np.random.default_rng(ref_seed).normal(0.0, 0.1, theta.weights.shape)))
    cfg = ObjectiveConfig(algo=algo, group_size=C2S_SEQS, kl_coeff=kl_coeff)
    out = objective_and_grad([group], theta, theta, ref, cfg, MaskingBounds(0.5, 5.0), temperature)
    lp_written = np.asarray([rec.logp_train_cur for r in rollouts for rec in r.tokens])
    data = pack([group], d)
    proj = np.random.default_rng(C1_PROJ_SEED).standard_normal((C2S_V, 4))
    data.update(
        out_kept=out.per_token_mask_kept,
        out_lp_cur=lp_written,
        out_surrogate=out.per_token_surrogate,
        out_calibration=out.per_token_calibration,
        out_entropy=out.per_token_entropy,
        out_objective=np.asarray(out.objective_value),
        out_clipped_fraction=np.asarray(out.clipped_fraction),
        out_token_count=np.asarray(out.token_count),
        out_grad_norm=np.asarray(np.linalg.norm(out.grad)),
        out_grad_proj=out.grad @ proj,
        out_kl_to_ref=np.asarray(out.kl_to_ref),
        kl_coeff=np.asarray(kl_coeff),
        algo=np.asarray(algo.value),
        temperature=np.asarray(temperature),
        ref_seed=np.asarray(-1 if ref_seed is None else ref_seed),
    )
    np.savez_compressed(OUT / f"{name}.npz", **data)
    print(f"{name}: tokens={out.token_count} popped={int((~out.per_token_mask_kept).sum())} "
          f"J={out.objective_value:.6g} |grad|={out.grad_norm:.4g}")


if __name__ == "__main__":
    main()
    c1_case()
    c2_slice_case()
    # BASELINE configs[2]/[4] width (hidden 8,192), a shorter group (8 x 2,048 tokens)
    c2_slice_case("c3_slice", d=8192, seq_len=2048, w_seed=2512, w_scale=0.5)
    # the KL-to-ref term (gamma = 0.4) at configs[1]'s width: the dual-accumulator GEMMs
    c2_slice_case("c2_slice_kl", seq_len=2048, kl_coeff=0.4, ref_seed=77)
    # TIS at temperature 0.7, configs[1]'s width
    c2_slice_case("c2_slice_tis", seq_len=2048, algo=Algo.TIS, temperature=0.7)
