"""The drop-in objective_and_grad on the GPU, held to the reference's own test semantics
(test_objective.py:133-281, test_discrepancy.py:166-178) and to its golden outputs.

Inputs are plain duck-typed objects (task.prompt_id, rollout.tokens, TokenRecord, params
with .weights/.version_id/.n_features), so no reference code is needed on the GPU box.
"""

from __future__ import annotations

import math
from dataclasses import dataclass, field

import numpy as np
import pytest

from conftest import golden_cases, load_golden

pytestmark = pytest.mark.gpu


@dataclass
class Task:
    prompt_id: int


@dataclass
class Rollout:
    tokens: list = field(default_factory=list)


@dataclass
class Params:
    weights: np.ndarray
    version_id: int = 0

    @property
    def n_features(self):
        return self.weights.shape[0]

    def copy(self):
        return Params(self.weights.copy(), self.version_id)


def _obj():
    from paper_2510_18855_b200 import objective

    return objective


def groups_from_golden(d):
    O = _obj()
    cu, go = d["cu_seqlens"], d["group_offsets"]
    groups = []
    for g in range(len(go) - 1):
        rollouts, rewards, advs = [], [], []
        for i in range(go[g], go[g + 1]):
            recs = [O.TokenRecord(int(d["tokens"][t]), float(d["lp_infer_old"][t]), float(d["lp_train_old"][t]),
                                  float(d["lp_train_old"][t]), 0) for t in range(cu[i], cu[i + 1])]
            rollouts.append(Rollout(recs))
            rewards.append(float(d["rewards"][i]))
            advs.append(float(d["advantages"][i]))
        groups.append(O.PromptGroup(task=Task(int(d["prompt_ids"][go[g]])), rollouts=rollouts, rewards=rewards,
                                    advantages=advs))
    return groups


def cfg_of(d, **over):
    O = _obj()
    kw = dict(algo=O.Algo(d["algo"]), clip_eps=d["clip_eps"], kl_coeff=d["kl_coeff"], group_size=2,
              tis_cap=d["tis_cap"])
    kw.update(over)
    return O.ObjectiveConfig(**kw), O.MaskingBounds(d["alpha"], d["beta"])


def log_prob(theta: Params, prompt_id: int, token: int, temperature=1.0):
    """policy.log_prob for an empty history, restated (policy.py:388-394)."""
    from paper_2510_18855_b200.features import feature_rows

    rows = feature_rows(prompt_id, -1, -1, theta.n_features)
    z = sum(theta.weights[r] for r in rows) / temperature
    m = z.max()
    return float(z[token] - m - math.log(np.exp(z - m).sum()))


def manual_group(theta, specs, advantages, prompt_id=100):
    """test_objective.py:56-77."""
    O = _obj()
    rollouts = []
    for token, calib, ratio in specs:
        lp_cur = log_prob(theta, prompt_id, token)
        lp_old = lp_cur - math.log(ratio)
        rollouts.append(Rollout([O.TokenRecord(token, lp_old - math.log(calib), lp_old, lp_cur, theta.version_id)]))
    return O.PromptGroup(task=Task(prompt_id), rollouts=rollouts, rewards=[0.0] * len(specs), advantages=advantages)


def rand_params(n_features, vocab, scale, seed):
    return Params(np.random.default_rng(seed).normal(0, scale, (n_features, vocab)))


# ------------------------------------------------------------------ golden parity
@pytest.mark.parametrize("name", golden_cases())
def test_dropin_fp64_matches_reference_golden(name):
    O = _obj()
    d = load_golden(name)
    groups = groups_from_golden(d)
    theta = Params(d["weight"], 1)
    ref = Params(d["weight_ref"], 0) if d["has_ref"] else None
    cfg, bounds = cfg_of(d)
    out = O.objective_and_grad(groups, theta, Params(d["weight"], 0), ref, cfg, bounds, d["temperature"])
    assert out.objective_value == pytest.approx(d["out_objective"], rel=1e-10, abs=1e-14)
    assert np.array_equal(out.per_token_mask_kept, d["out_kept"])
    assert out.clipped_fraction == d["out_clipped_fraction"] and out.token_count == d["out_token_count"]
    np.testing.assert_allclose(out.grad, d["out_grad"], rtol=1e-9, atol=1e-13)
    np.testing.assert_allclose(out.per_token_surrogate, d["out_surrogate"], rtol=1e-10, atol=1e-13)
    np.testing.assert_allclose(out.per_token_entropy, d["out_entropy"], rtol=1e-12, atol=1e-13)
    assert out.kl_to_ref == pytest.approx(d["out_kl_to_ref"], rel=1e-10, abs=1e-14)
    # lp_cur written back into every TokenRecord (objective.py:224-225)
    written = [rec.logp_train_cur for g in groups for r in g.rollouts for rec in r.tokens]
    np.testing.assert_allclose(written, d["out_lp_cur"], rtol=1e-12, atol=1e-13)


@pytest.mark.parametrize("name", ["small_icepop", "medium_icepop", "medium_tis", "temp_icepop", "small_icepop_kl",
                                  "small_icepop_refdiag"])
def test_dropin_bf16_matches_reference_golden(name):
    O = _obj()
    d = load_golden(name)
    cfg, bounds = cfg_of(d)
    ref = Params(d["weight_ref"], 0) if d["has_ref"] else None
    out = O.objective_and_grad(groups_from_golden(d), Params(d["weight"], 1), Params(d["weight"], 0), ref, cfg,
                               bounds, d["temperature"], precision="bf16")
    assert np.array_equal(out.per_token_mask_kept, d["out_kept"])
    assert out.objective_value == pytest.approx(d["out_objective"], rel=2e-3, abs=1e-5)
    assert out.kl_to_ref == pytest.approx(d["out_kl_to_ref"], rel=1e-2, abs=1e-4)
    assert np.linalg.norm(out.grad - d["out_grad"]) / np.linalg.norm(d["out_grad"]) < 1e-2


@pytest.mark.parametrize("precision", ["bf16", "fp64"])
def test_dropin_grad_out_receives_the_same_gradient(precision):
    """grad_out (keyword extension): the gradient lands in the caller's array, bit-identical to
    the freshly allocated one, and LossBreakdown.grad is that array; a bad buffer is refused."""
    O = _obj()
    d = load_golden("medium_icepop")
    cfg, bounds = cfg_of(d)
    args = (Params(d["weight"], 1), Params(d["weight"], 0), None, cfg, bounds, d["temperature"])
    fresh = O.objective_and_grad(groups_from_golden(d), *args, precision=precision)
    buf = np.full(d["weight"].shape, np.nan)
    out = O.objective_and_grad(groups_from_golden(d), *args, precision=precision, grad_out=buf)
    assert out.grad is buf
    assert np.array_equal(buf, fresh.grad)
    assert out.objective_value == fresh.objective_value
    for bad in (np.zeros(d["weight"].shape, np.float32), np.zeros((2, 3)), np.asfortranarray(buf)):
        with pytest.raises(ValueError):
            O.objective_and_grad(groups_from_golden(d), *args, precision=precision, grad_out=bad)


# ------------------------------------------------------------------ reference semantics
def test_degenerate_case_all_algorithms_bit_identical():
    """test_objective.py:133-146: calib == 1 and theta == theta_old -> algos agree bitwise."""
    O = _obj()
    d = load_golden("small_icepop")
    d["lp_infer_old"] = d["lp_train_old"].copy()
    theta = Params(d["weight"], 0)
    res = {}
    for algo in O.Algo:
        cfg, bounds = cfg_of(d, algo=algo)
        res[algo] = O.objective_and_grad(groups_from_golden(d), theta, theta, theta.copy(), cfg, bounds)
    base = res[O.Algo.ICEPOP]
    assert base.clipped_fraction == 0.0
    for algo in (O.Algo.GRPO, O.Algo.TIS):
        assert res[algo].objective_value == base.objective_value
        assert np.array_equal(res[algo].grad, base.grad)


def test_zero_advantages_give_zero_objective_and_gradient():
    """test_objective.py:149-155."""
    O = _obj()
    d = load_golden("medium_icepop")
    groups = groups_from_golden(d)
    for g in groups:
        g.advantages = [0.0] * len(g.advantages)
    cfg, bounds = cfg_of(d)
    out = O.objective_and_grad(groups, Params(d["weight"]), Params(d["weight"]), None, cfg, bounds)
    assert out.objective_value == 0.0
    assert np.all(out.grad == 0.0)


def finite_difference_grad(groups, theta, theta_old, ref, cfg, bounds, h=1e-6):
    O = _obj()
    fd = np.zeros_like(theta.weights)
    for i in range(theta.weights.shape[0]):
        for j in range(theta.weights.shape[1]):
            wp, wm = theta.weights.copy(), theta.weights.copy()
            wp[i, j] += h
            wm[i, j] -= h
            up = O.objective_and_grad(groups, Params(wp, theta.version_id), theta_old, ref, cfg, bounds)
            dn = O.objective_and_grad(groups, Params(wm, theta.version_id), theta_old, ref, cfg, bounds)
            fd[i, j] = (up.objective_value - dn.objective_value) / (2 * h)
    return fd


@pytest.mark.parametrize("algo,kl_coeff", [("icepop", 0.0), ("grpo", 0.0), ("tis", 0.0), ("icepop", 0.4)])
def test_gradient_matches_finite_differences(algo, kl_coeff):
    """test_objective.py:172-182 (fp64 validation path)."""
    O = _obj()
    d = load_golden("small_icepop")
    groups = groups_from_golden(d)
    theta_old = Params(d["weight"][:10, :8].copy(), 0)
    # shrink to the FD test's shapes: 10 features, vocab 8 (tokens < 8 already)
    for g in groups:
        g.task = Task(g.task.prompt_id)
    theta = Params(theta_old.weights + np.random.default_rng(1).normal(0, 0.05, theta_old.weights.shape), 0)
    ref = rand_params(10, 8, 0.5, 99)
    cfg, bounds = cfg_of(d, algo=O.Algo(algo), kl_coeff=kl_coeff)
    out = O.objective_and_grad(groups, theta, theta_old, ref, cfg, bounds)
    fd = finite_difference_grad(groups, theta, theta_old, ref, cfg, bounds)
    rel = np.abs(out.grad - fd) / np.maximum(1.0, np.abs(out.grad))
    assert rel.max() < 1e-5


def test_masked_tokens_contribute_exactly_zero_gradient():
    """test_objective.py:185-226."""
    from paper_2510_18855_b200.features import feature_rows

    O = _obj()
    theta = rand_params(64, 8, 0.5, 8)
    cfg = O.ObjectiveConfig(group_size=2)
    bounds = O.MaskingBounds(0.5, 5.0)
    rows_a = set(feature_rows(100, -1, -1, 64))
    rows_b = set(feature_rows(205, -1, -1, 64))
    private_b = rows_b - rows_a
    assert private_b

    def build(th):
        rollouts = []
        for pid, token, calib in ((100, 1, 1.0), (205, 2, 0.2)):
            lp = log_prob(th, pid, token)
            rollouts.append(Rollout([O.TokenRecord(token, lp - math.log(calib), lp, lp, th.version_id)]))
        # the pair uses prompt 100 for the group, but each rollout's features follow its own task in the
        # reference test; here rollouts share the group's task, so give each its own single-rollout group
        return [O.PromptGroup(task=Task(100), rollouts=[rollouts[0]], rewards=[1.0], advantages=[1.0]),
                O.PromptGroup(task=Task(205), rollouts=[rollouts[1]], rewards=[0.0], advantages=[-1.0])]

    base_groups = build(theta)
    base = O.objective_and_grad(base_groups, theta, theta, None, cfg, bounds)
    assert list(base.per_token_mask_kept) == [True, False]
    assert base.clipped_fraction == 0.5
    perturbed = theta.weights.copy()
    for row in private_b:
        perturbed[row, :] += 0.37
    out_p = O.objective_and_grad(base_groups, Params(perturbed, theta.version_id), theta, None, cfg, bounds)
    assert abs(out_p.objective_value - base.objective_value) < 1e-12
    for row in private_b:
        assert np.all(base.grad[row, :] == 0.0)
        assert np.all(out_p.grad[row, :] == 0.0)


def test_wide_bounds_reduce_masked_variant_to_unmasked():
    """test_objective.py:229-235."""
    O = _obj()
    d = load_golden("medium_icepop")
    wide = O.MaskingBounds(alpha=1e-12, beta=1e12)
    theta = Params(d["weight"])
    ice = O.objective_and_grad(groups_from_golden(d), theta, theta, None, O.ObjectiveConfig(group_size=2), wide)
    grpo = O.objective_and_grad(groups_from_golden(d), theta, theta, None,
                                O.ObjectiveConfig(algo=O.Algo.GRPO, group_size=2), wide)
    assert ice.objective_value == grpo.objective_value
    assert np.array_equal(ice.grad, grpo.grad)


def test_clip_branch_zeroes_gradient_on_both_sides():
    """test_objective.py:238-247."""
    O = _obj()
    theta = rand_params(16, 8, 0.4, 10)
    group = manual_group(theta, [(1, 1.0, 1.35), (2, 1.0, 0.7)], advantages=[1.0, -1.0])
    out = O.objective_and_grad([group], theta, theta, None, O.ObjectiveConfig(group_size=2, clip_eps=0.2),
                               O.MaskingBounds(0.5, 5.0))
    assert np.all(out.grad == 0.0)
    assert out.per_token_surrogate == pytest.approx([1.2 * 1.0, 0.8 * -1.0])


def test_truncated_variant_agrees_with_masked_inside_common_region():
    """test_objective.py:250-261."""
    O = _obj()
    theta = rand_params(16, 8, 0.4, 12)
    specs = [(1, 0.3, 1.0), (2, 0.7, 1.1), (3, 1.9, 0.95), (4, 2.6, 1.0), (5, 6.0, 1.0)]
    advs = [1.0, -0.5, 0.5, 1.0, -1.0]
    b = O.MaskingBounds(0.5, 5.0)
    ice = O.objective_and_grad([manual_group(theta, specs, advs)], theta, theta, None,
                               O.ObjectiveConfig(algo=O.Algo.ICEPOP, group_size=2), b)
    tis = O.objective_and_grad([manual_group(theta, specs, advs)], theta, theta, None,
                               O.ObjectiveConfig(algo=O.Algo.TIS, group_size=2, tis_cap=2.0), b)
    calib = ice.per_token_calibration
    common = (calib >= 0.5) & (calib <= 2.0)
    assert common.sum() == 2
    assert np.array_equal(ice.per_token_surrogate[common], tis.per_token_surrogate[common])


def test_clipped_fraction_counts_masked_tokens():
    """test_objective.py:264-270."""
    O = _obj()
    theta = rand_params(16, 8, 0.4, 13)
    group = manual_group(theta, [(1, 0.2, 1.0), (2, 1.0, 1.0), (3, 9.0, 1.0), (4, 1.2, 1.0)],
                         advantages=[1.0, -1.0, 0.5, -0.5])
    out = O.objective_and_grad([group], theta, theta, None, O.ObjectiveConfig(group_size=2), O.MaskingBounds())
    assert out.clipped_fraction == pytest.approx(2 / 4)
    assert out.token_count == 4
    assert math.isfinite(out.entropy_clipped)


def test_empty_group_empty_rollout_and_versions_fail():
    """test_objective.py:273-281 plus the version guards of objective.py:190-213."""
    O = _obj()
    theta = rand_params(16, 8, 0.4, 1)
    cfg, b = O.ObjectiveConfig(group_size=2), O.MaskingBounds()
    with pytest.raises(ValueError):
        O.objective_and_grad([], theta, theta, None, cfg, b)
    group = manual_group(theta, [(1, 1.0, 1.0)], advantages=[0.0])
    group.rollouts[0].tokens = []
    with pytest.raises(ValueError):
        O.objective_and_grad([group], theta, theta, None, cfg, b)
    with pytest.raises(ValueError):
        O.objective_and_grad([manual_group(theta, [(1, 1.0, 1.0)], [1.0])], Params(theta.weights, 0),
                             Params(theta.weights, 1), None, cfg, b)
    g = manual_group(theta, [(1, 1.0, 1.0)], [1.0])
    g.rollouts[0].tokens[0].gen_version = 5
    with pytest.raises(ValueError):
        O.objective_and_grad([g], theta, theta, None, cfg, b)


def test_numeric_error_on_calibration_overflow():
    O = _obj()
    from paper_2510_18855_b200.errors import NumericError

    theta = rand_params(16, 8, 0.4, 3)
    g = manual_group(theta, [(1, 1.0, 1.0), (2, 1.0, 1.0)], [1.0, -1.0])
    g.rollouts[0].tokens[0].logp_infer_old = -800.0  # exp(lp_old + 800) overflows
    with pytest.raises(NumericError):
        O.objective_and_grad([g], theta, theta, None, O.ObjectiveConfig(group_size=2), O.MaskingBounds())


def test_mask_set_monotonicity():
    """test_discrepancy.py:166-178: narrow-bound popped set contains the wide-bound one."""
    O = _obj()
    d = load_golden("medium_icepop")
    theta = Params(d["weight"])
    outs = [O.objective_and_grad(groups_from_golden(d), theta, theta, None, O.ObjectiveConfig(group_size=2),
                                 O.MaskingBounds(a, b)) for a, b in ((0.8, 1.25), (0.5, 5.0))]
    narrow_popped, wide_popped = ~outs[0].per_token_mask_kept, ~outs[1].per_token_mask_kept
    assert np.all(narrow_popped[wide_popped])
    assert narrow_popped.sum() > wide_popped.sum()


def test_group_advantages_on_device():
    """test_objective.py:105-130 through the K0 kernel."""
    O = _obj()
    assert np.all(O.group_advantages([1.0, 1.0, 1.0, 1.0]) == 0.0)
    assert O.group_advantages([1.0, 0.0]) == pytest.approx([1.0, -1.0], abs=1e-15)
    assert O.group_advantages([1e-7, 0.0]) == pytest.approx([5e-8 / 1e-6, -5e-8 / 1e-6])
    with pytest.raises(ValueError):
        O.group_advantages([1.0])
    rng = np.random.default_rng(5)
    rewards = [1.0, 0.0, 1.0, 0.0, 0.0, 1.0, 1.0, 1.0]
    base = O.group_advantages(rewards)
    for _ in range(5):
        perm = rng.permutation(len(rewards))
        assert np.array_equal(O.group_advantages([rewards[i] for i in perm]), base[perm])


@pytest.mark.parametrize("precision", ["fp64", "bf16"])
def test_error_order_and_progressive_write_back(precision):
    """The reference raises in loop order (objective.py:204-242): a NumericError in group 1
    comes before a ValueError in group 2, and lp_cur has been written back for every rollout up
    to the failing one (a calibration overflow fails after that rollout's write-back)."""
    O = _obj()
    from paper_2510_18855_b200.errors import NumericError

    theta = rand_params(16, 8, 0.4, 5)
    cfg, b = O.ObjectiveConfig(group_size=2), O.MaskingBounds()
    g0 = manual_group(theta, [(1, 1.0, 1.0), (2, 1.0, 1.0)], [1.0, -1.0])
    g1 = manual_group(theta, [(3, 1.0, 1.0), (4, 1.0, 1.0)], [1.0, -1.0])
    g2 = manual_group(theta, [(5, 1.0, 1.0), (6, 1.0, 1.0)], [1.0, -1.0])
    g1.rollouts[1].tokens[0].logp_infer_old = -800.0  # calibration overflow in group 1, rollout 1
    g2.rollouts[1].tokens = []                         # and a ValueError later, in group 2
    recs = [r.tokens[0] for g in (g0, g1, g2) for r in g.rollouts if r.tokens]
    for r in recs:
        r.logp_train_cur = 123.0
    with pytest.raises(NumericError, match="calibration"):
        O.objective_and_grad([g0, g1, g2], theta, theta, None, cfg, b, precision=precision)
    # rollouts 0..3 (through the failing one) were written back, group 2's were not reached
    assert all(r.logp_train_cur != 123.0 for r in recs[:4]) and recs[4].logp_train_cur == 123.0
    g1.rollouts[1].tokens[0].logp_infer_old = g1.rollouts[1].tokens[0].logp_train_old
    with pytest.raises(ValueError, match="empty rollout"):
        O.objective_and_grad([g0, g1, g2], theta, theta, None, cfg, b, precision=precision)
    assert recs[4].logp_train_cur != 123.0  # group 2's first rollout was computed before the error


def test_grad_out_untouched_on_error_and_must_not_alias_parameters():
    O = _obj()
    from paper_2510_18855_b200.errors import NumericError

    theta = rand_params(16, 8, 0.4, 6)
    cfg, b = O.ObjectiveConfig(group_size=2), O.MaskingBounds()
    g = manual_group(theta, [(1, 1.0, 1.0), (2, 1.0, 1.0)], [1.0, -1.0])
    g.rollouts[0].tokens[0].logp_infer_old = -800.0
    buf = np.full_like(theta.weights, 7.0)
    with pytest.raises(NumericError):
        O.objective_and_grad([g], theta, theta, None, cfg, b, grad_out=buf)
    assert (buf == 7.0).all()
    with pytest.raises(ValueError, match="share memory"):
        O.objective_and_grad([g], theta, theta, None, cfg, b, grad_out=theta.weights)


@pytest.mark.parametrize("precision", ["bf16", "fp64"])
def test_fresh_gradients_never_alias_while_held(precision):
    """Fresh gradients come back in pooled page-locked buffers: a buffer is reused only once the
    array returned in it (and every view of it) is gone, so gradients the caller holds never
    change under later calls."""
    import gc

    O = _obj()
    cfg, b = O.ObjectiveConfig(group_size=2), O.MaskingBounds()
    held, copies = [], []
    for seed in range(4):
        theta = rand_params(24, 16, 0.5, 40 + seed)  # the same shape every call: the same pool
        g = manual_group(theta, [(1, 1.0, 1.0), (2, 1.0, 1.0)], [1.0, -1.0])
        out = O.objective_and_grad([g], theta, theta, None, cfg, b, precision=precision)
        held.append(out.grad[2:])  # a view keeps the buffer taken
        copies.append(out.grad.copy())
        del out
    for i in range(len(held)):
        for j in range(i):
            assert not np.shares_memory(held[i], held[j])
        assert np.array_equal(held[i], copies[i][2:])
    # released buffers are handed out again (and hold the new call's gradient)
    del held
    gc.collect()
    theta = rand_params(24, 16, 0.5, 50)
    g = manual_group(theta, [(1, 1.0, 1.0), (2, 1.0, 1.0)], [1.0, -1.0])
    out = O.objective_and_grad([g], theta, theta, None, cfg, b, precision=precision)
    pooled = [slot[0].numpy() for slot in O._GRAD_POOL[theta.weights.shape]]
    assert any(np.shares_memory(out.grad, p) for p in pooled)
    ref = O.objective_and_grad([manual_group(theta, [(1, 1.0, 1.0), (2, 1.0, 1.0)], [1.0, -1.0])], theta, theta,
                               None, cfg, b, precision=precision, grad_out=np.empty_like(theta.weights))
    assert np.array_equal(out.grad, ref.grad)


def test_mask_uses_numpys_calibration_bits():
    """per_token_calibration is numpy's exp(lp_old - lp_inf) itself, and the mask follows it even
    for a ratio sitting exactly on a bound (objective.py:227-232)."""
    O = _obj()
    theta = rand_params(16, 8, 0.4, 7)
    g = manual_group(theta, [(1, 0.5, 1.0), (2, 5.0, 1.0), (3, 1.0, 1.0)], [1.0, -1.0, 0.5])
    out = O.objective_and_grad([g], theta, theta, None, O.ObjectiveConfig(group_size=2), O.MaskingBounds())
    lp_old = np.array([r.tokens[0].logp_train_old for r in g.rollouts])
    lp_inf = np.array([r.tokens[0].logp_infer_old for r in g.rollouts])
    c = np.exp(lp_old - lp_inf)
    assert np.array_equal(out.per_token_calibration, c)
    assert np.array_equal(out.per_token_mask_kept, (c >= 0.5) & (c <= 5.0))


@pytest.mark.parametrize("vocab", [10, 37])
def test_bf16_pads_a_vocabulary_not_a_multiple_of_8(vocab):
    """The bf16 path pads V to a multiple of 8 with columns held at logit -1e4 (one always-on
    feature row): the results match the fp64 path within the bf16 tolerances and the gradient
    keeps the reference's shape."""
    import torch

    O = _obj()
    theta = rand_params(21, vocab, 0.5, 8)  # bf16-exact weights: both paths see the same policy
    theta.weights = torch.from_numpy(theta.weights).to(torch.bfloat16).double().numpy()
    g = manual_group(theta, [(1, 1.0, 1.1), (2, 0.9, 1.0), (3, 1.2, 0.95), (vocab - 1, 1.0, 1.0)],
                     [1.0, -1.0, 0.5, -0.5])
    cfg, b = O.ObjectiveConfig(group_size=2), O.MaskingBounds()
    a = O.objective_and_grad([g], theta, theta, None, cfg, b, precision="fp64")
    c = O.objective_and_grad([g], theta, theta, None, cfg, b, precision="bf16")
    assert c.grad.shape == theta.weights.shape
    assert np.array_equal(a.per_token_mask_kept, c.per_token_mask_kept)
    assert c.objective_value == pytest.approx(a.objective_value, rel=1e-3, abs=1e-6)
    assert np.linalg.norm(c.grad - a.grad) <= 1e-2 * np.linalg.norm(a.grad)
    np.testing.assert_allclose(c.per_token_entropy, a.per_token_entropy, atol=2e-3)
    # a smaller problem reusing the same padded staging shape right after a larger one
    small = Params(theta.weights[:17].copy())
    gs = manual_group(small, [(1, 1.0, 1.1), (2, 0.9, 1.0)], [1.0, -1.0])
    a2 = O.objective_and_grad([gs], small, small, None, cfg, b, precision="fp64")
    c2 = O.objective_and_grad([gs], small, small, None, cfg, b, precision="bf16")
    assert c2.objective_value == pytest.approx(a2.objective_value, rel=1e-3, abs=1e-6)
