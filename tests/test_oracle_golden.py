"""Pin the CPU oracle to the reference's own outputs (tests/golden, made by the
unmodified mismatchlab.objective_and_grad) -- runs on the CPU container."""

from __future__ import annotations

import math

import numpy as np
import pytest

from conftest import GOLDEN, golden_cases, golden_hidden, load_golden, oracle_kwargs
from oracle.icepop_oracle import group_advantages, icepop_dense, per_token_weights, token_terms


@pytest.mark.parametrize("name", golden_cases())
def test_oracle_matches_reference_golden(name):
    d = load_golden(name)
    o = icepop_dense(golden_hidden(d), d["weight"], d["tokens"], d["lp_train_old"], d["lp_infer_old"],
                     d["cu_seqlens"], d["group_offsets"], d["advantages"], **oracle_kwargs(d))
    assert np.array_equal(o["kept"], d["out_kept"])
    assert o["token_count"] == d["out_token_count"]
    assert o["clipped_fraction"] == d["out_clipped_fraction"]
    # calibration is input-only and computed with the same numpy expression: bit-exact
    assert np.array_equal(o["calib"], d["out_calibration"])
    np.testing.assert_allclose(o["lp_cur"], d["out_lp_cur"], rtol=1e-13, atol=1e-14)
    np.testing.assert_allclose(o["surrogate"], d["out_surrogate"], rtol=1e-12, atol=1e-15)
    np.testing.assert_allclose(o["entropy"], d["out_entropy"], rtol=1e-13, atol=1e-14)
    assert o["objective"] == pytest.approx(d["out_objective"], rel=1e-12, abs=1e-15)
    assert o["kl_to_ref"] == pytest.approx(d["out_kl_to_ref"], rel=1e-12, abs=1e-15)
    if math.isnan(d["out_entropy_clipped"]):
        assert math.isnan(o["entropy_clipped"])
    else:
        assert o["entropy_clipped"] == pytest.approx(d["out_entropy_clipped"], rel=1e-13)
    # dense H^T dZ vs the reference's 4x np.add.at scatter
    np.testing.assert_allclose(o["grad_weight"], d["out_grad"], rtol=1e-11, atol=1e-15)


@pytest.mark.parametrize("name", golden_cases())
def test_token_terms_match_reference_golden(name):
    """The vectorised per-token terms (used by the full-size GPU checks) on the reference's own
    lp_cur reproduce its mask, calibration and surrogate (KL cases: surrogate excludes kl)."""
    d = load_golden(name)
    kw = oracle_kwargs(d)
    t = token_terms(d["out_lp_cur"], d["lp_train_old"], d["lp_infer_old"], d["cu_seqlens"], d["group_offsets"],
                    d["advantages"], alpha=kw["alpha"], beta=kw["beta"], clip_eps=kw["clip_eps"],
                    tis_cap=kw["tis_cap"], temperature=kw["temperature"], algo=kw["algo"])
    assert np.array_equal(t["kept"], d["out_kept"])
    assert np.array_equal(t["calib"], d["out_calibration"])
    np.testing.assert_allclose(t["surrogate"], d["out_surrogate"], rtol=1e-12, atol=1e-15)


def test_oracle_layouts_agree():
    d = load_golden("medium_icepop")
    h = golden_hidden(d)
    args = (d["tokens"], d["lp_train_old"], d["lp_infer_old"], d["cu_seqlens"], d["group_offsets"], d["advantages"])
    a = icepop_dense(h, d["weight"], *args, layout="dv")
    b = icepop_dense(h, np.ascontiguousarray(d["weight"].T), *args, layout="vd")
    np.testing.assert_allclose(a["grad_weight"], b["grad_weight"].T, rtol=1e-13, atol=1e-16)
    np.testing.assert_allclose(a["grad_hidden"], b["grad_hidden"], rtol=1e-13, atol=1e-16)


def test_oracle_dhidden_matches_finite_differences():
    """dH has no reference analogue: check the oracle's dJ/dH by central differences."""
    d = load_golden("small_icepop")
    h = golden_hidden(d)
    args = (d["weight"], d["tokens"], d["lp_train_old"], d["lp_infer_old"], d["cu_seqlens"], d["group_offsets"],
            d["advantages"])
    kw = oracle_kwargs(d)
    o = icepop_dense(h, *args, **kw)
    rng = np.random.default_rng(0)
    eps = 1e-6
    for _ in range(12):
        t, f = int(rng.integers(h.shape[0])), int(rng.integers(h.shape[1]))
        hp, hm = h.copy(), h.copy()
        hp[t, f] += eps
        hm[t, f] -= eps
        fd = (icepop_dense(hp, *args, need_grads=False, **kw)["objective"]
              - icepop_dense(hm, *args, need_grads=False, **kw)["objective"]) / (2 * eps)
        assert abs(fd - o["grad_hidden"][t, f]) <= 1e-6 * max(1.0, abs(fd))


def test_group_advantages_golden():
    z = np.load(GOLDEN / "advantages.npz")
    off = z["group_offsets"]
    got = np.concatenate([group_advantages(z["rewards"][off[g]:off[g + 1]]) for g in range(len(off) - 1)])
    assert np.array_equal(got, z["advantages"])


def _np_pairwise(a):
    """The association order the CUDA K0 kernel implements (token_kernels.cuh)."""
    n = len(a)
    if n < 8:
        res = 0.0
        for x in a:
            res += x
        return res
    if n <= 128:
        r = list(a[:8])
        i = 8
        while i < n - (n % 8):
            for j in range(8):
                r[j] += a[i + j]
            i += 8
        res = ((r[0] + r[1]) + (r[2] + r[3])) + ((r[4] + r[5]) + (r[6] + r[7]))
        while i < n:
            res += a[i]
            i += 1
        return res
    n2 = n // 2
    n2 -= n2 % 8
    return _np_pairwise(a[:n2]) + _np_pairwise(a[n2:])


def test_k0_summation_order_is_numpys():
    """The CUDA advantages kernel restates numpy's pairwise sum; prove the order is bit-exact."""
    z = np.load(GOLDEN / "advantages.npz")
    off = z["group_offsets"]
    for g in range(len(off) - 1):
        r = [float(x) for x in z["rewards"][off[g]:off[g + 1]]]
        n = len(r)
        mean = _np_pairwise(r) / n
        var = _np_pairwise([(x - mean) * (x - mean) for x in r]) / n
        std = math.sqrt(var)
        adv = np.asarray([(x - mean) / max(std, 1e-6) for x in r])
        assert np.array_equal(adv, z["advantages"][off[g]:off[g + 1]]), f"group {g}"


def test_per_token_weights_counts_popped_tokens():
    """w_t = 1/(n_groups G |y_i|) keeps popped tokens in the denominator (objective.py:215)."""
    d = load_golden("medium_icepop")
    w = per_token_weights(d["cu_seqlens"], d["group_offsets"])
    n_groups = len(d["group_offsets"]) - 1
    assert w.sum() == pytest.approx(1.0, rel=1e-12)  # each group's rollouts average to 1/n_groups
    assert len(w) == d["out_token_count"] and n_groups >= 2


@pytest.mark.parametrize("bad", ["empty_group", "empty_rollout"])
def test_oracle_error_semantics(bad):
    d = load_golden("small_icepop")
    cu = d["cu_seqlens"].copy()
    go = d["group_offsets"].copy()
    if bad == "empty_group":
        go = np.concatenate([go[:1], go])
    else:
        cu = np.concatenate([cu[:1], cu])
        go = go + np.concatenate([[0], np.ones(len(go) - 1, dtype=go.dtype)])
    with pytest.raises(ValueError):
        icepop_dense(golden_hidden(d), d["weight"], d["tokens"], d["lp_train_old"], d["lp_infer_old"], cu, go,
                     np.concatenate([[0.0], d["advantages"]]))


def test_oracle_matches_reference_at_config0_full_size():
    """BASELINE configs[0] (8 x 512 tokens, hidden 1,024, vocab 32K, GRPO group 8) through the
    reference's own objective_and_grad vs the oracle: mask bit-exact, lp_cur / surrogate /
    entropy / objective to fp64 rounding, gradient through its norm and a fixed projection."""
    from conftest import C1_PROJ_SEED, load_c1
    from paper_2510_18855_b200.features import multihot

    d, w = load_c1()
    h = multihot(d["feats"], w.shape[0])
    o = icepop_dense(h, w, d["tokens"], d["lp_train_old"], d["lp_infer_old"], d["cu_seqlens"], d["group_offsets"],
                     d["advantages"], layout="dv")
    assert np.array_equal(o["kept"], d["out_kept"]) and o["token_count"] == int(d["out_token_count"]) == 4096
    assert np.array_equal(o["calib"], d["out_calibration"])
    np.testing.assert_allclose(o["lp_cur"], d["out_lp_cur"], rtol=1e-12, atol=1e-12)
    np.testing.assert_allclose(o["surrogate"], d["out_surrogate"], rtol=1e-10, atol=1e-15)
    np.testing.assert_allclose(o["entropy"], d["out_entropy"], rtol=1e-12)
    assert o["objective"] == pytest.approx(float(d["out_objective"]), rel=1e-10)
    proj = np.random.default_rng(C1_PROJ_SEED).standard_normal((w.shape[1], 4))
    np.testing.assert_allclose(o["grad_weight"] @ proj, d["out_grad_proj"], rtol=1e-9, atol=1e-12)
    assert np.linalg.norm(o["grad_weight"]) == pytest.approx(float(d["out_grad_norm"]), rel=1e-10)
