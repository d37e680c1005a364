"""Drop-in replacement for mismatchlab's ``objective`` module (objective.py:1-326).

``objective_and_grad`` keeps the reference signature, validation order, exceptions,
``TokenRecord.logp_train_cur`` write-back and ``LossBreakdown`` fields, but runs on the
B200 through ``libicepop_b200.so``:

* ``precision="fp64"`` (default): the fp64 SIMT CUDA validation path -- the reference's
  exact-identity and finite-difference tests (test_objective.py) hold unchanged;
* ``precision="bf16"``: the tcgen05 tensor-core path (weights rounded to bf16, fp32
  accumulation; tolerances in tests/test_parity_gpu.py).

The reference's 4-hot feature contraction is packed as a dense multi-hot H
(features.py), so both precisions run the same dense kernels as a real lm_head.

When mismatchlab is importable its data classes are re-exported (so enum identity and
isinstance checks in the caller keep working); otherwise identical definitions are used.
:func:`install` rebinds the reference's three bindings of the name (objective.py,
scheduler.py:38 and __init__.py:33).
"""

from __future__ import annotations

import enum
import math
from dataclasses import dataclass, field
from typing import Any

import numpy as np

from .errors import NumericError

try:  # pragma: no cover - depends on the host environment
    from mismatchlab.objective import (  # type: ignore
        Algo,
        LossBreakdown,
        MaskingBounds,
        ObjectiveConfig,
        PromptGroup,
        TokenRecord,
    )

    _HAVE_REFERENCE = True
except Exception:  # noqa: BLE001
    _HAVE_REFERENCE = False

    class Algo(enum.Enum):  # objective.py:41-44
        ICEPOP = "icepop"
        GRPO = "grpo"
        TIS = "tis"

    @dataclass(frozen=True)
    class MaskingBounds:  # objective.py:47-56
        alpha: float = 0.5
        beta: float = 5.0

        def __post_init__(self) -> None:
            if not (0.0 < self.alpha <= 1.0 <= self.beta):
                raise ValueError(f"bounds must satisfy 0 < alpha <= 1 <= beta, got [{self.alpha}, {self.beta}]")

    @dataclass(frozen=True)
    class ObjectiveConfig:  # objective.py:66-82
        algo: Algo = Algo.ICEPOP
        clip_eps: float = 0.2
        kl_coeff: float = 0.0
        group_size: int = 8
        tis_cap: float = 2.0

        def __post_init__(self) -> None:
            if not 0.0 < self.clip_eps < 1.0:
                raise ValueError("clip_eps must be in (0, 1)")
            if self.kl_coeff < 0.0:
                raise ValueError("kl_coeff must be nonnegative")
            if self.group_size < 2:
                raise ValueError("group_size must be >= 2")
            if self.tis_cap <= 0.0:
                raise ValueError("tis_cap must be positive")

    @dataclass
    class TokenRecord:  # objective.py:85-103
        token: int
        logp_infer_old: float
        logp_train_old: float
        logp_train_cur: float
        gen_version: int

        def __post_init__(self) -> None:
            for name in ("logp_infer_old", "logp_train_old", "logp_train_cur"):
                if not math.isfinite(getattr(self, name)):
                    raise NumericError(f"TokenRecord.{name} is not finite")

    @dataclass
    class PromptGroup:  # objective.py:106-119
        task: Any
        rollouts: list
        rewards: list
        advantages: list

        def __post_init__(self) -> None:
            if not (len(self.rollouts) == len(self.rewards) == len(self.advantages)):
                raise ValueError("rollouts, rewards, and advantages must have equal length")
            if not all(math.isfinite(a) for a in self.advantages):
                raise NumericError("group advantages contain non-finite values")

    @dataclass
    class LossBreakdown:  # objective.py:122-139
        objective_value: float
        per_token_mask_kept: np.ndarray
        clipped_fraction: float
        grad: np.ndarray
        kl_to_ref: float
        token_count: int = 0
        mean_logp: float = 0.0
        entropy_all: float = 0.0
        entropy_clipped: float = math.nan
        per_token_surrogate: np.ndarray = field(default_factory=lambda: np.zeros(0))
        per_token_calibration: np.ndarray = field(default_factory=lambda: np.zeros(0))
        per_token_entropy: np.ndarray = field(default_factory=lambda: np.zeros(0))

        @property
        def grad_norm(self) -> float:
            return float(np.linalg.norm(self.grad))


_DEFAULT_PRECISION = "fp64"


def set_default_precision(precision: str) -> None:
    """Select the path used when objective_and_grad is called without ``precision``."""
    global _DEFAULT_PRECISION
    if precision not in ("fp64", "bf16"):
        raise ValueError("precision must be 'fp64' or 'bf16'")
    _DEFAULT_PRECISION = precision


def mask(k: float, bounds: MaskingBounds) -> float:
    """objective.py:59-63 -- k if alpha <= k <= beta (inclusive), else 0."""
    if not math.isfinite(k) or k <= 0.0:
        raise ValueError(f"mask argument must be a finite positive ratio, got {k}")
    return k if bounds.alpha <= k <= bounds.beta else 0.0


def group_advantages(rewards) -> np.ndarray:
    """objective.py:153-159 on the device (K0; bit-identical to numpy's mean/std)."""
    import torch

    from .loss import group_advantages as _k0

    r = np.asarray(rewards, dtype=np.float64)
    if r.size < 2:
        raise ValueError("advantage normalization needs a group of >= 2 rewards")
    dev = torch.device("cuda", torch.cuda.current_device())
    out = _k0(torch.from_numpy(r).to(dev), torch.tensor([0, r.size], dtype=torch.int32, device=dev))
    return out.cpu().numpy()


def empty_breakdown(params) -> LossBreakdown:
    """objective.py:142-150."""
    return LossBreakdown(objective_value=0.0, per_token_mask_kept=np.zeros(0, dtype=bool), clipped_fraction=0.0,
                         grad=np.zeros_like(params.weights), kl_to_ref=0.0)


def _algo_name(algo) -> str:
    return algo.value if hasattr(algo, "value") else str(algo)


@dataclass
class _Packed:
    tokens: np.ndarray
    lp_old: np.ndarray
    lp_inf: np.ndarray
    cu: np.ndarray
    go: np.ndarray
    adv: np.ndarray
    feats: np.ndarray
    records: list


def _pack(groups, theta, theta_old) -> _Packed:
    """Validate like objective.py:190-213 and flatten in group-major order (:271-276)."""
    from .features import rollout_feats

    if not groups:
        raise ValueError("objective needs at least one prompt group")
    if theta_old.version_id > theta.version_id:
        raise ValueError("theta_old must not be newer than theta")
    tokens, lp_old, lp_inf, cu, go, adv, feats, records = [], [], [], [0], [0], [], [], []
    for group in groups:
        if not group.rollouts:
            raise ValueError("empty prompt group")
        for rollout, advantage in zip(group.rollouts, group.advantages):
            toks = rollout.tokens
            if not toks:
                raise ValueError("empty rollout in prompt group")
            if any(rec.gen_version > theta_old.version_id for rec in toks):
                raise ValueError("token generated by a version newer than theta_old")
            ids = [rec.token for rec in toks]
            tokens += ids
            lp_old += [rec.logp_train_old for rec in toks]
            lp_inf += [rec.logp_infer_old for rec in toks]
            records += toks
            feats.append(rollout_feats(group.task.prompt_id, ids, theta.n_features))
            cu.append(cu[-1] + len(toks))
            adv.append(float(advantage))
        go.append(go[-1] + len(group.rollouts))
    return _Packed(np.asarray(tokens, dtype=np.int32), np.asarray(lp_old, dtype=np.float64),
                   np.asarray(lp_inf, dtype=np.float64), np.asarray(cu, dtype=np.int32),
                   np.asarray(go, dtype=np.int32), np.asarray(adv, dtype=np.float64), np.concatenate(feats), records)


def objective_and_grad(
    groups,
    theta,
    theta_old,
    ref,
    cfg,
    bounds,
    temperature: float = 1.0,
    *,
    precision: str | None = None,
    device=None,
    grad_out: np.ndarray | None = None,
) -> LossBreakdown:
    """Objective value and its exact analytic ascent gradient w.r.t. theta, on the GPU.

    Same contract as objective.py:172-298, including the write-back of the recomputed
    lp_cur into every TokenRecord (objective.py:224-225).

    ``grad_out`` (extension, keyword only): a C-contiguous float64 array shaped like
    theta.weights that receives the gradient and is returned as ``LossBreakdown.grad``.
    A trainer that reuses one buffer skips materialising a fresh 8*n_features*V-byte array per
    call, which dominates the call at small batches.
    """
    if grad_out is not None and (not isinstance(grad_out, np.ndarray) or grad_out.dtype != np.float64
                                 or grad_out.shape != tuple(theta.weights.shape)
                                 or not grad_out.flags.c_contiguous or not grad_out.flags.writeable):
        raise ValueError("grad_out must be a writeable C-contiguous float64 array shaped like theta.weights")
    import torch

    from .features import multihot_device
    from .loss import Diagnostics, IcePopConfig, PackedBatch, finish, icepop_bwd, icepop_fwd, icepop_fwd_bwd

    if temperature <= 0:
        raise ValueError("temperature must be positive")
    precision = precision or _DEFAULT_PRECISION
    p = _pack(groups, theta, theta_old)
    dev = torch.device(device) if device is not None else torch.device("cuda", torch.cuda.current_device())
    n_features, vocab = theta.weights.shape
    icfg = IcePopConfig(alpha=bounds.alpha, beta=bounds.beta, clip_eps=cfg.clip_eps, tis_cap=cfg.tis_cap,
                        temperature=float(temperature), kl_coeff=cfg.kl_coeff, algo=_algo_name(cfg.algo))
    batch = PackedBatch(
        tokens=torch.from_numpy(p.tokens).to(dev),
        lp_train_old=torch.from_numpy(p.lp_old).to(dev),
        lp_infer_old=torch.from_numpy(p.lp_inf).to(dev),
        cu_seqlens=torch.from_numpy(p.cu).to(dev),
        group_offsets=torch.from_numpy(p.go).to(dev),
        advantages=torch.from_numpy(p.adv).to(dev),
    )
    feats = torch.from_numpy(np.ascontiguousarray(p.feats, dtype=np.int64)).to(dev)
    if precision == "fp64":
        H = multihot_device(feats, n_features, torch.float64)
        W = torch.from_numpy(np.ascontiguousarray(theta.weights, dtype=np.float64)).to(dev)
        Wr = torch.from_numpy(np.ascontiguousarray(ref.weights, dtype=np.float64)).to(dev) if ref is not None else None
        fwd = icepop_fwd(H, W, batch, icfg, layout="dv", weight_ref=Wr)
        _, gw = icepop_bwd(H, W, batch, fwd, icfg, layout="dv", need_hidden=False, weight_ref=Wr)
    elif precision == "bf16":
        if vocab % 8:
            raise ValueError("the bf16 path needs a vocabulary size that is a multiple of 8")
        nf_pad = (n_features + 7) // 8 * 8  # zero feature rows are inert

        def pad_bf16(w):
            # round on the host (torch's threaded cast), copy a quarter of the fp64 bytes
            wb = torch.from_numpy(np.ascontiguousarray(w, dtype=np.float64)).to(torch.bfloat16)
            if nf_pad != n_features:
                wb = torch.cat([wb, wb.new_zeros((nf_pad - n_features, vocab))])
            return wb.to(dev)

        H = multihot_device(feats, nf_pad, torch.bfloat16)
        W = pad_bf16(theta.weights)
        Wr = pad_bf16(ref.weights) if ref is not None else None
        # value and gradient together: stored probabilities (in token chunks if needed)
        fwd, _, gw = icepop_fwd_bwd(H, W, batch, icfg, layout="dv", need_hidden=False, weight_ref=Wr)
        gw = gw[:n_features]
    else:
        raise ValueError("precision must be 'fp64' or 'bf16'")
    finish(fwd.stats)
    diag = Diagnostics.from_stats(fwd.stats.cpu())
    grad_finite = bool(torch.isfinite(gw).all())
    if grad_out is not None:
        torch.from_numpy(grad_out).copy_(gw.to(torch.float64))
        grad = grad_out
    else:
        grad = gw.to(torch.float64).cpu().numpy()
    lp_cur = fwd.lp_cur.cpu().numpy()
    for rec, value in zip(p.records, lp_cur):  # objective.py:224-225
        rec.logp_train_cur = float(value)
    if not math.isfinite(diag.objective_value) or not grad_finite:
        raise NumericError("objective or gradient is not finite")
    kept = fwd.kept.cpu().numpy().astype(bool)
    return LossBreakdown(
        objective_value=diag.objective_value,
        per_token_mask_kept=kept,
        clipped_fraction=diag.clipped_fraction,
        grad=grad,
        kl_to_ref=diag.kl_to_ref if ref is not None else 0.0,
        token_count=diag.token_count,
        mean_logp=diag.mean_logp,
        entropy_all=diag.entropy_all,
        entropy_clipped=diag.entropy_clipped,
        per_token_surrogate=fwd.surrogate.cpu().numpy(),
        per_token_calibration=fwd.calib.cpu().numpy(),
        per_token_entropy=fwd.entropy.to(torch.float64).cpu().numpy(),
    )


def _device_step(weights: np.ndarray, grad: np.ndarray, lr: float, velocity: np.ndarray | None = None,
                 beta: float = 0.0):
    """One fp64 ascent step on the GPU (icepop_sgd_update_f64, the reference's rounding bit for
    bit): returns (new weights, new velocity or None) as host arrays."""
    import torch

    from . import _lib
    from .loss import _stream

    dev = torch.device("cuda", torch.cuda.current_device())
    lib = _lib.ensure_device(dev.index)
    w = torch.from_numpy(np.ascontiguousarray(weights, dtype=np.float64)).to(dev)
    g = torch.from_numpy(np.ascontiguousarray(grad, dtype=np.float64)).to(dev)
    v = torch.from_numpy(np.ascontiguousarray(velocity, dtype=np.float64)).to(dev) if velocity is not None else None
    stats = torch.empty(_lib.NSTATS, dtype=torch.float64, device=dev)
    _lib.check(lib.icepop_sgd_update_f64(w.data_ptr(), w.data_ptr(), g.data_ptr(), _lib.ptr(v), _lib.ptr(v), w.numel(),
                                         float(lr), float(beta), stats.data_ptr(), _stream(dev)))
    err = int(stats[_lib.STAT_ERRORS].item())
    if err & 4:
        raise NumericError("parameter update produced non-finite weights")  # objective.py:309-310
    return w.cpu().numpy(), (v.cpu().numpy() if v is not None else None)


def sgd_update(theta, grad: np.ndarray, lr: float):
    """objective.py:301-311 on the device: gradient ascent w + lr g in fp64 with numpy's
    rounding (the same bits), version_id + 1, NumericError on non-finite weights."""
    if lr <= 0:
        raise ValueError("learning rate must be positive")
    if np.shape(grad) != theta.weights.shape:
        raise ValueError("gradient shape does not match parameters")
    weights, _ = _device_step(theta.weights, grad, lr)
    return type(theta)(weights=weights, version_id=theta.version_id + 1)


def momentum_update(theta, grad, velocity, lr: float, beta: float = 0.9):
    """objective.py:314-326 on the device: v' = beta v + g, then the ascent step with v'
    (one kernel); returns (new params, v')."""
    if not 0.0 <= beta < 1.0:
        raise ValueError("momentum beta must be in [0, 1)")
    if np.shape(velocity) != np.shape(grad):
        raise ValueError("velocity shape does not match the gradient")
    if lr <= 0:
        raise ValueError("learning rate must be positive")
    if np.shape(grad) != theta.weights.shape:
        raise ValueError("gradient shape does not match parameters")
    weights, new_velocity = _device_step(theta.weights, grad, lr, velocity, beta)
    return type(theta)(weights=weights, version_id=theta.version_id + 1), new_velocity


def delta_and_gap(params, probes, infer, temperature: float = 1.0, *, precision: str | None = None):
    """discrepancy.py:132-141 on the device: (mean over the probes of KL(p_infer || p_train),
    max |p_infer - p_train|).

    The inference engine's logits are the reference's own simulation of that engine
    (mismatchlab.policy.perturb_logits of the scaled train logits with noise_keys, policy.py:
    269-277, 341-347): the noise model is the engine's, not part of the path, and is not ported
    (SURVEY.md 8f-1), so this drop-in needs mismatchlab. The train logits (multi-hot H . W, the
    feature rows restated in features.py), the log-softmaxes, the KL and the gap run on the
    GPU (loss.delta_and_gap; fp64 by default like the objective, so the reference's exact and
    finite-difference tests hold)."""
    import torch
    from mismatchlab.policy import noise_keys, perturb_logits  # type: ignore  (the engine simulator)

    from .features import feature_rows, multihot_device
    from .loss import delta_and_gap as _device_delta_gap

    if not probes:
        raise ValueError("probe set must be non-empty")  # discrepancy.py:136-137
    if temperature <= 0:
        raise ValueError("temperature must be positive")
    precision = precision or _DEFAULT_PRECISION
    n_features, vocab = params.weights.shape
    feats = np.empty((len(probes), 4), dtype=np.int64)
    kf = np.empty(len(probes), dtype=np.uint64)
    kv = np.empty(len(probes), dtype=np.uint64)
    for i, ctx in enumerate(probes):
        prev, last = ctx.window()
        feats[i] = feature_rows(ctx.prompt_id, prev, last, n_features)
        kf[i], kv[i] = noise_keys(infer, params.version_id, ctx.prompt_id, prev, last)
    dev = torch.device("cuda", torch.cuda.current_device())
    fd = torch.from_numpy(feats).to(dev)
    W64 = torch.from_numpy(np.ascontiguousarray(params.weights, dtype=np.float64)).to(dev)
    H64 = multihot_device(fd, n_features, torch.float64)
    train = (H64 @ W64 / temperature).cpu().numpy()  # the simulator's input (the engine perturbs it)
    infer_logits = perturb_logits(train, kf, kv, infer.mismatch_scale)
    if precision == "fp64":
        d, g, _, _ = _device_delta_gap(H64, W64, torch.from_numpy(np.ascontiguousarray(infer_logits)).to(dev),
                                       layout="dv", temperature=temperature)
    elif precision == "bf16":
        nf_pad = (n_features + 7) // 8 * 8
        Wb = torch.zeros((nf_pad, vocab), dtype=torch.bfloat16, device=dev)
        Wb[:n_features] = W64.to(torch.bfloat16)
        d, g, _, _ = _device_delta_gap(multihot_device(fd, nf_pad, torch.bfloat16), Wb,
                                       torch.from_numpy(infer_logits.astype(np.float32)).to(dev), layout="dv",
                                       temperature=temperature)
    else:
        raise ValueError("precision must be 'fp64' or 'bf16'")
    out = torch.stack([d, g]).cpu().numpy()
    return float(out[0]), float(out[1])


def install(precision: str | None = None) -> None:
    """Rebind mismatchlab's objective_and_grad and the update step that follows
    it (sgd_update / momentum_update, scheduler.py:551-555) to this drop-in, in every module
    that binds the names (objective.py, scheduler.py:29-40, __init__.py:32-34)."""
    import mismatchlab  # type: ignore
    import mismatchlab.discrepancy  # type: ignore
    import mismatchlab.objective  # type: ignore
    import mismatchlab.scheduler  # type: ignore

    if precision is not None:
        set_default_precision(precision)
    for mod in (mismatchlab, mismatchlab.objective, mismatchlab.scheduler):
        mod.objective_and_grad = objective_and_grad
        mod.sgd_update = sgd_update
        mod.momentum_update = momentum_update
    # the discrepancy probe: measure() (discrepancy.py:144-161, called by train_loop) looks the
    # name up in its own module
    for mod in (mismatchlab, mismatchlab.discrepancy):
        mod.delta_and_gap = delta_and_gap


__all__ = [
    "Algo", "LossBreakdown", "MaskingBounds", "ObjectiveConfig", "PromptGroup", "TokenRecord", "empty_breakdown",
    "delta_and_gap", "group_advantages", "install", "mask", "momentum_update", "objective_and_grad",
    "set_default_precision", "sgd_update",
]
