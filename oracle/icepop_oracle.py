"""CPU ORACLE -- TEST INFRASTRUCTURE ONLY.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s ``cpu_baseline`` /
``--impl reference`` legs may import this module, and only as the checker or the
timed CPU baseline. The product path (``paper_2510_18855_b200``) never imports it
and fails loudly without its CUDA library.

A numpy fp64 restatement of the reference's hot path, generalised from its 4-hot
feature gather to a dense hidden matrix H (the 4-hot case is H = multihot(feats),
SURVEY.md load-bearing fact 2):

* ``group_advantages``     follows objective.py:153-159
* ``log_softmax_rows``     follows policy.py:350-355
* ``token_terms``          the per-token part of objective.py:215-252 (weights, calibration
                           mask, ratio, clip, surrogate, gradient coefficient) vectorised over
                           a whole packed batch, for checks at full size where the logits come
                           from a chunked GPU fp32 reference instead of numpy
* ``icepop_dense``         follows objective.py:204-298 line by line, with
                           ``batched_train_logits`` (policy.py:279-289) replaced by H.W
                           and the ``np.add.at`` scatter (objective.py:265-266) by H^T.dZ;
                           dH = dZ.W^T is the one output with no reference analogue.

Parity pinning: tests/test_oracle_golden.py checks this restatement against golden
vectors produced by the UNMODIFIED reference (tests/golden/make_golden.py imports
mismatchlab and calls its own objective_and_grad), so the oracle is pinned, not
self-certified.
"""

from __future__ import annotations

import math

import numpy as np

ALGOS = ("icepop", "grpo", "tis")


def group_advantages(rewards) -> np.ndarray:
    """objective.py:153-159 -- z-score with a 1e-6 population-std floor."""
    r = np.asarray(rewards, dtype=np.float64)
    if r.size < 2:
        raise ValueError("advantage normalization needs a group of >= 2 rewards")
    std = float(r.std())
    return (r - r.mean()) / max(std, 1e-6)


def log_softmax_rows(logits: np.ndarray) -> tuple[np.ndarray, np.ndarray]:
    """policy.py:350-355 -- (log_probs, probs), exact log-sum-exp, no flooring."""
    shifted = logits - logits.max(axis=1, keepdims=True)
    e = np.exp(shifted)
    z = e.sum(axis=1, keepdims=True)
    return shifted - np.log(z), e / z


def _logits(h: np.ndarray, w: np.ndarray, layout: str, temperature: float) -> np.ndarray:
    """policy.py:279-289 with the 4-hot gather generalised to H.W."""
    if temperature <= 0:
        raise ValueError("temperature must be positive")
    logits = h @ w if layout == "dv" else h @ w.T
    if temperature != 1.0:
        logits = logits / temperature
    if not np.isfinite(logits).all():
        raise FloatingPointError("non-finite logits (corrupted parameters)")
    return logits


def icepop_dense(
    hidden: np.ndarray,
    weight: np.ndarray,
    tokens: np.ndarray,
    lp_train_old: np.ndarray,
    lp_infer_old: np.ndarray,
    cu_seqlens: np.ndarray,
    group_offsets: np.ndarray,
    advantages: np.ndarray,
    *,
    alpha: float = 0.5,
    beta: float = 5.0,
    clip_eps: float = 0.2,
    tis_cap: float = 2.0,
    temperature: float = 1.0,
    kl_coeff: float = 0.0,
    algo: str = "icepop",
    layout: str = "dv",
    weight_ref: np.ndarray | None = None,
    need_grads: bool = True,
) -> dict:
    """The IcePop objective, its exact gradients and diagnostics, in fp64.

    Returns a dict with per-token arrays (group-major order, objective.py:271-276):
    lse, lp_cur, entropy, kept, calib, surrogate, coeff, kl; scalars objective,
    clipped_fraction, token_count, mean_logp, entropy_all, entropy_clipped, kl_to_ref;
    and (need_grads) grad_weight (ascent dJ/dW in ``layout``) and grad_hidden (dJ/dH).
    """
    if algo not in ALGOS:
        raise ValueError(f"unknown algo {algo!r}")
    h_all = np.asarray(hidden, dtype=np.float64)
    w = np.asarray(weight, dtype=np.float64)
    w_ref = None if weight_ref is None else np.asarray(weight_ref, dtype=np.float64)
    n_groups = len(group_offsets) - 1
    if n_groups < 1:
        raise ValueError("objective needs at least one prompt group")
    n_total = int(cu_seqlens[-1])
    grad_w = np.zeros_like(w) if need_grads else None
    grad_h = np.zeros_like(h_all) if need_grads else None
    out = {k: np.zeros(n_total) for k in ("lse", "lp_cur", "entropy", "calib", "surrogate", "coeff", "kl")}
    out["kept"] = np.zeros(n_total, dtype=bool)
    total = 0.0
    for g in range(n_groups):
        s0, s1 = int(group_offsets[g]), int(group_offsets[g + 1])
        if s1 <= s0:
            raise ValueError("empty prompt group")
        G = s1 - s0
        group_value = 0.0
        for i in range(s0, s1):
            t0, t1 = int(cu_seqlens[i]), int(cu_seqlens[i + 1])
            n_tok = t1 - t0
            if n_tok <= 0:
                raise ValueError("empty rollout in prompt group")
            advantage = float(advantages[i])
            weight_t = 1.0 / (n_groups * G * n_tok)  # objective.py:215
            tok = np.asarray(tokens[t0:t1], dtype=np.int64)
            lp_old = np.asarray(lp_train_old[t0:t1], dtype=np.float64)
            lp_inf = np.asarray(lp_infer_old[t0:t1], dtype=np.float64)
            pos = np.arange(n_tok)
            h = h_all[t0:t1]
            logits = _logits(h, w, layout, temperature)
            log_probs, probs = log_softmax_rows(logits)
            lp_cur = log_probs[pos, tok]  # objective.py:223
            calib = np.exp(lp_old - lp_inf)  # objective.py:227
            if not np.isfinite(calib).all():
                raise FloatingPointError("calibration ratio overflow")
            if algo == "icepop":
                kept = (calib >= alpha) & (calib <= beta)
                factor = np.where(kept, calib, 0.0)
            elif algo == "grpo":
                kept = np.ones(n_tok, dtype=bool)
                factor = calib
            else:
                kept = np.ones(n_tok, dtype=bool)
                factor = np.minimum(calib, tis_cap)
            ratio = np.exp(lp_cur - lp_old)  # objective.py:240
            if not np.isfinite(ratio).all():
                raise FloatingPointError("importance ratio overflow")
            unclipped = ratio * advantage
            clipped = np.clip(ratio, 1.0 - clip_eps, 1.0 + clip_eps) * advantage
            active = unclipped <= clipped
            pg_values = factor * np.where(active, unclipped, clipped)
            coeffs = np.where(active, weight_t * factor * ratio * advantage / temperature, 0.0)
            kl_values = np.zeros(n_tok)
            grad_logits = None
            if need_grads:
                grad_logits = -coeffs[:, None] * probs
                grad_logits[pos, tok] += coeffs
            if w_ref is not None:
                ref_log_probs, _ = log_softmax_rows(_logits(h, w_ref, layout, temperature))
                diff = log_probs - ref_log_probs
                kl_values = (probs * diff).sum(axis=1)
                if kl_coeff > 0.0 and need_grads:
                    grad_logits -= (weight_t * kl_coeff / temperature) * (probs * (diff - kl_values[:, None]))
            if need_grads:
                # dW = H^T dZ  (the reference's np.add.at scatter, objective.py:265-266)
                if layout == "dv":
                    grad_w += h.T @ grad_logits
                    grad_h[t0:t1] = grad_logits @ w.T
                else:
                    grad_w += grad_logits.T @ h
                    grad_h[t0:t1] = grad_logits @ w
            token_values = pg_values - kl_coeff * kl_values
            group_value += float(token_values.sum()) / (G * n_tok)
            sl = slice(t0, t1)
            out["lse"][sl] = logits.max(axis=1) + np.log(np.exp(logits - logits.max(axis=1, keepdims=True)).sum(axis=1))
            out["lp_cur"][sl] = lp_cur
            out["entropy"][sl] = -(probs * log_probs).sum(axis=1)
            out["kept"][sl] = kept
            out["calib"][sl] = calib
            out["surrogate"][sl] = pg_values
            out["coeff"][sl] = coeffs
            out["kl"][sl] = kl_values
        total += group_value
    objective = total / n_groups
    if not math.isfinite(objective) or (need_grads and not np.isfinite(grad_w).all()):
        raise FloatingPointError("objective or gradient is not finite")
    kept_arr = out["kept"]
    n_clipped = int((~kept_arr).sum())
    out.update(
        objective=objective,
        clipped_fraction=n_clipped / kept_arr.size,
        token_count=int(kept_arr.size),
        mean_logp=float(out["lp_cur"].mean()),
        entropy_all=float(out["entropy"].mean()),
        entropy_clipped=float(out["entropy"][~kept_arr].mean()) if n_clipped else math.nan,
        kl_to_ref=float(out["kl"].mean()),
        n_clipped=n_clipped,
    )
    if need_grads:
        out["grad_weight"] = grad_w
        out["grad_hidden"] = grad_h
    return out


def token_terms(lp_cur, lp_train_old, lp_infer_old, cu_seqlens, group_offsets, advantages, *, alpha=0.5, beta=5.0,
                clip_eps=0.2, tis_cap=2.0, temperature=1.0, algo="icepop") -> dict:
    """Per-token IcePop terms given lp_cur, fp64, vectorised (objective.py:215-252; the same
    expressions as icepop_dense's inner loop): calib, kept, ratio, active, surrogate, coeff."""
    if algo not in ALGOS:
        raise ValueError(f"unknown algo {algo!r}")
    lp_cur = np.asarray(lp_cur, dtype=np.float64)
    lp_old = np.asarray(lp_train_old, dtype=np.float64)
    lp_inf = np.asarray(lp_infer_old, dtype=np.float64)
    cu = np.asarray(cu_seqlens, dtype=np.int64)
    seq_of = np.repeat(np.arange(len(cu) - 1), np.diff(cu))
    adv = np.asarray(advantages, dtype=np.float64)[seq_of]
    weight_t = per_token_weights(cu, np.asarray(group_offsets, dtype=np.int64))  # objective.py:215
    calib = np.exp(lp_old - lp_inf)  # objective.py:227
    if algo == "icepop":
        kept = (calib >= alpha) & (calib <= beta)
        factor = np.where(kept, calib, 0.0)
    elif algo == "grpo":
        kept = np.ones(lp_cur.size, dtype=bool)
        factor = calib
    else:
        kept = np.ones(lp_cur.size, dtype=bool)
        factor = np.minimum(calib, tis_cap)
    ratio = np.exp(lp_cur - lp_old)  # objective.py:240
    unclipped = ratio * adv
    clipped = np.clip(ratio, 1.0 - clip_eps, 1.0 + clip_eps) * adv
    active = unclipped <= clipped
    surrogate = factor * np.where(active, unclipped, clipped)
    coeff = np.where(active, weight_t * factor * ratio * adv / temperature, 0.0)  # objective.py:250
    return dict(calib=calib, kept=kept, ratio=ratio, active=active, surrogate=surrogate, coeff=coeff)


def per_token_weights(cu_seqlens: np.ndarray, group_offsets: np.ndarray) -> np.ndarray:
    """w_t = 1/(n_groups * G_g * |y_i|) for every token (objective.py:215)."""
    n_groups = len(group_offsets) - 1
    w = np.empty(int(cu_seqlens[-1]))
    for g in range(n_groups):
        G = int(group_offsets[g + 1] - group_offsets[g])
        for i in range(int(group_offsets[g]), int(group_offsets[g + 1])):
            t0, t1 = int(cu_seqlens[i]), int(cu_seqlens[i + 1])
            w[t0:t1] = 1.0 / (n_groups * G * (t1 - t0))
    return w
