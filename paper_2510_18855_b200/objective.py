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
import functools
import math
import operator
import weakref
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
_LAST_PATH = ""  # "full" or "onpolicy": the forward the last objective_and_grad call ran (tests)


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
    error: Exception | None = None  # the first validation error, raised after the prefix


_FIELDS = operator.attrgetter("token", "logp_train_old", "logp_infer_old", "gen_version")


def _pack(groups, theta, theta_old) -> _Packed:
    """Validate like objective.py:190-213 and flatten in group-major order (:271-276).

    The reference validates a group / rollout only when its loop reaches it, after computing
    (and writing back lp_cur for) every rollout before it, so a later ValueError can be preceded
    by a NumericError or by write-backs. Packing therefore stops at the first invalid group or
    rollout: the valid prefix is packed and that error is returned with it."""
    from .features import rollout_feats

    if not groups:
        raise ValueError("objective needs at least one prompt group")
    if theta_old.version_id > theta.version_id:
        raise ValueError("theta_old must not be newer than theta")
    rows, cu, go, adv, feats, records = [], [0], [0], [], [], []
    error = None
    for group in groups:
        if not group.rollouts:
            error = ValueError("empty prompt group")
            break
        for rollout, advantage in zip(group.rollouts, group.advantages):
            toks = rollout.tokens
            if not toks:
                error = ValueError("empty rollout in prompt group")
                break
            vals = list(map(_FIELDS, toks))
            if max(v[3] for v in vals) > theta_old.version_id:
                error = ValueError("token generated by a version newer than theta_old")
                break
            rows += vals
            records += toks
            feats.append(rollout_feats(group.task.prompt_id, [v[0] for v in vals], theta.n_features))
            cu.append(cu[-1] + len(toks))
            adv.append(float(advantage))
        if len(adv) > go[-1]:
            go.append(len(adv))
        if error is not None:
            break
    if not rows:
        return _Packed(*(np.zeros(0),) * 7, records=[], error=error)
    a = np.array(rows, dtype=np.float64)
    return _Packed(a[:, 0].astype(np.int32), np.ascontiguousarray(a[:, 1]), np.ascontiguousarray(a[:, 2]),
                   np.asarray(cu, dtype=np.int32), np.asarray(go, dtype=np.int32), np.asarray(adv, dtype=np.float64),
                   np.concatenate(feats), records, error)


# Host buffers reused across calls: pinned bf16 staging of the weights (the cast runs on the host's
# threads straight into pinned memory, then one fast DMA), and page-locked grad_out arrays.
_STAGING: dict = {}
_REGISTERED: dict = {}  # (address, nbytes) -> the array (kept alive while registered)


def _pinned_bf16(shape) -> "torch.Tensor":
    import torch

    t = _STAGING.get(shape)
    if t is None:
        _STAGING.clear()
        t = _STAGING[shape] = torch.zeros(shape, dtype=torch.bfloat16, pin_memory=True)
    return t


def _page_lock(arr: np.ndarray) -> None:
    """Register a reused grad_out buffer with CUDA once (cudaHostRegister) so the gradient's D2H
    runs at full DMA speed; at most two buffers stay registered (and referenced)."""
    import torch

    key = (arr.ctypes.data, arr.nbytes)
    if key in _REGISTERED:
        return
    cudart = torch.cuda.cudart()
    while len(_REGISTERED) >= 2:
        (addr, _), _old = _REGISTERED.popitem()
        cudart.cudaHostUnregister(addr)
    if int(cudart.cudaHostRegister(key[0], key[1], 0)) == 0:
        _REGISTERED[key] = arr


# Pinned host buffers that fresh gradients are returned in, per weights shape (the last two
# shapes): a buffer is handed out again once the array returned in it is gone (weak reference;
# views keep it alive). Returning pinned memory spares the D2H a staging copy, and reusing it
# spares a fresh 8 * n_features * V-byte page-locked allocation per call (~50-150 ms at C1).
_GRAD_POOL: dict = {}
_GRAD_POOL_MAX_BYTES = 2 << 30  # larger gradients are not pooled (2 x 2 shapes would pin > 8 GB)


def _fresh_grad(shape) -> tuple["torch.Tensor", np.ndarray]:
    import torch

    pool = _GRAD_POOL.pop(shape, [])
    _GRAD_POOL[shape] = pool  # most recently used last
    while len(_GRAD_POOL) > 2:
        _GRAD_POOL.pop(next(iter(_GRAD_POOL)))
    for slot in pool:
        if slot[1]() is None:
            arr = slot[0].numpy()
            slot[1] = weakref.ref(arr)
            return slot[0], arr
    t = torch.empty(shape, dtype=torch.float64, pin_memory=True)
    arr = t.numpy()
    if len(pool) < 2 and t.nbytes <= _GRAD_POOL_MAX_BYTES:  # bounded page-locked host memory
        pool.append([t, weakref.ref(arr)])
    return t, arr


def _write_back(records, lp_cur: list, n: int) -> None:
    """objective.py:224-225 for the first n packed tokens."""
    for rec, value in zip(records[:n], lp_cur[:n]):
        rec.logp_train_cur = value


# Vocabulary padding of the bf16 path: its TMA tensors need rows of a multiple of 16 bytes, so a
# vocabulary that is not a multiple of 8 is padded with columns whose logits are -1e4 (one extra
# always-on feature row carries that value into the padded columns only): they get probability
# exactly 0 in fp32, so no statistic, mask or gradient of a real column changes, and the padded
# rows / columns of the gradient are dropped.
_PAD_LOGIT = -1.0e4


def _bf16_shapes(n_features: int, vocab: int) -> tuple[int, int, bool]:
    """(feature rows, vocabulary columns, padded) of the bf16 operands."""
    pad = vocab % 8 != 0
    return (n_features + (1 if pad else 0) + 7) // 8 * 8, (vocab + 7) // 8 * 8, pad


def _bf16_hidden(feats, n_features: int, vocab: int):
    """Multi-hot H of the bf16 path (features.multihot_device), plus the padding feature."""
    import torch

    from .features import multihot_device

    nf_pad, _, pad = _bf16_shapes(n_features, vocab)
    H = multihot_device(feats, nf_pad, torch.bfloat16)
    if pad:
        H[:, n_features] = 1.0
    return H


def _bf16_weight_into(dst, w: np.ndarray, n_features: int, vocab: int):
    """Write weights [n_features, vocab] (fp64, host) into a bf16 buffer [nf_pad, v_pad] (a reused
    staging buffer: every element outside the weights is rewritten)."""
    import torch

    dst[:n_features, :vocab].copy_(torch.from_numpy(np.ascontiguousarray(w, dtype=np.float64)))
    dst[:n_features, vocab:] = 0.0
    dst[n_features:] = 0.0
    if vocab % 8:
        dst[n_features, vocab:] = _PAD_LOGIT
    return dst


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

    Same contract as objective.py:172-298: the same validation, the same exceptions in the
    same order (a rollout's NumericError -- non-finite logits, calibration or importance ratio
    -- before a later rollout's ValueError), and the write-back of the recomputed lp_cur into
    every TokenRecord the reference would have reached (objective.py:224-225). The calibration
    ratio is numpy's own exp(lp_old - lp_inf), handed to the kernels, so the mask is the
    reference's bit for bit.

    ``grad_out`` (extension, keyword only): a C-contiguous float64 array shaped like
    theta.weights that receives the gradient and is returned as ``LossBreakdown.grad``. It is
    page-locked once and kept referenced while registered (the last two such buffers), so a
    trainer that reuses it gets the gradient at DMA speed instead of materialising a fresh
    8 * n_features * V-byte array per call. It must not share memory with theta's or ref's
    weights, and it receives nothing when the call raises.
    """
    if grad_out is not None:
        if (not isinstance(grad_out, np.ndarray) or grad_out.dtype != np.float64
                or grad_out.shape != tuple(theta.weights.shape) or not grad_out.flags.c_contiguous
                or not grad_out.flags.writeable):
            raise ValueError("grad_out must be a writeable C-contiguous float64 array shaped like theta.weights")
        if np.shares_memory(grad_out, theta.weights) or (ref is not None and np.shares_memory(grad_out, ref.weights)):
            raise ValueError("grad_out must not share memory with the parameters")
    import torch

    from .features import multihot_device
    from .loss import Diagnostics, IcePopConfig, PackedBatch, icepop_fwd, icepop_fwd_bwd

    precision = precision or _DEFAULT_PRECISION
    if precision not in ("fp64", "bf16"):
        raise ValueError("precision must be 'fp64' or 'bf16'")
    n_features, vocab = theta.weights.shape
    p = _pack(groups, theta, theta_old)
    if not p.records:  # the first group / rollout is invalid
        raise p.error
    if temperature <= 0:  # batched_train_logits of the first rollout (policy.py:281-282)
        raise ValueError("temperature must be positive")
    if p.tokens.min() < 0 or p.tokens.max() >= vocab:
        raise ValueError("token id outside the vocabulary")
    dev = torch.device(device) if device is not None else torch.device("cuda", torch.cuda.current_device())
    icfg = IcePopConfig(alpha=bounds.alpha, beta=bounds.beta, clip_eps=cfg.clip_eps, tis_cap=cfg.tis_cap,
                        temperature=float(temperature), kl_coeff=cfg.kl_coeff, algo=_algo_name(cfg.algo))
    with np.errstate(over="ignore", invalid="ignore"):  # a non-finite ratio raises below, in the reference's order
        calib = np.exp(p.lp_old - p.lp_inf)  # objective.py:227, numpy's bits
        calib_c = np.where(np.isfinite(calib), calib, 0.0)
    batch = PackedBatch(
        tokens=torch.from_numpy(p.tokens).to(dev),
        lp_train_old=torch.from_numpy(p.lp_old).to(dev),
        lp_infer_old=torch.from_numpy(p.lp_inf).to(dev),
        cu_seqlens=torch.from_numpy(p.cu).to(dev),
        group_offsets=torch.from_numpy(p.go).to(dev),
        advantages=torch.from_numpy(p.adv).to(dev),
        calib=torch.from_numpy(calib_c).to(dev),
    )
    feats = torch.from_numpy(np.ascontiguousarray(p.feats, dtype=np.int64)).to(dev)
    need_grad = p.error is None  # a validation error later in the batch: the forward decides what raises
    gw = None
    # theta is theta_old with every lp_train_old recorded by record_train_logprobs under theta:
    # the exact on-policy forward (no forward GEMM; r == 1 bit for bit, as in the reference's loop)
    stash = _onpolicy_stash(p.records, theta, theta_old, temperature, precision) \
        if need_grad and ref is None and precision == "bf16" else None
    global _LAST_PATH
    _LAST_PATH = "onpolicy" if stash is not None else "full"
    with torch.cuda.device(dev):
        if stash is not None:
            from .loss import icepop_bwd, icepop_fwd_onpolicy

            nf, vp, _ = _bf16_shapes(n_features, vocab)
            H = _bf16_hidden(feats, n_features, vocab)
            W = _bf16_weight_into(torch.zeros((nf, vp), dtype=torch.bfloat16, device=dev), theta.weights,
                                  n_features, vocab)
            st = torch.from_numpy(stash).to(dev)
            fwd = icepop_fwd_onpolicy(batch, st[:, 0].to(torch.float32), st[:, 1].to(torch.float32), icfg,
                                      hidden_dim=nf, vocab=vp)
            _, gw = icepop_bwd(H, W, batch, fwd, icfg, layout="dv", need_hidden=False)
            gw = gw[:n_features, :vocab]
        elif precision == "fp64":
            H = multihot_device(feats, n_features, torch.float64)
            W = torch.from_numpy(np.ascontiguousarray(theta.weights, dtype=np.float64)).to(dev)
            Wr = torch.from_numpy(np.ascontiguousarray(ref.weights, dtype=np.float64)).to(dev) if ref is not None \
                else None
            fwd = icepop_fwd(H, W, batch, icfg, layout="dv", weight_ref=Wr)
            if need_grad:
                from .loss import icepop_bwd

                _, gw = icepop_bwd(H, W, batch, fwd, icfg, layout="dv", need_hidden=False, weight_ref=Wr)
        else:
            nf_pad, v_pad, _ = _bf16_shapes(n_features, vocab)  # zero feature rows are inert

            def upload(w):
                return _bf16_weight_into(_pinned_bf16((nf_pad, v_pad)), w, n_features, vocab).to(dev,
                                                                                                 non_blocking=True)

            H = _bf16_hidden(feats, n_features, vocab)
            W = upload(theta.weights)
            Wr = None
            if ref is not None:
                torch.cuda.current_stream(dev).synchronize()  # the staging buffer is reused
                Wr = upload(ref.weights)
            if need_grad:  # value and gradient together: stored probabilities (token chunks if needed)
                fwd, _, gw = icepop_fwd_bwd(H, W, batch, icfg, layout="dv", need_hidden=False, weight_ref=Wr)
                gw = gw[:n_features, :vocab]
            else:
                fwd = icepop_fwd(H, W, batch, icfg, layout="dv", weight_ref=Wr, store_probs=False)
        grad_finite = torch.isfinite(gw).all() if gw is not None else None
        host = torch.cat([fwd.lp_cur.to(torch.float64), fwd.entropy.to(torch.float64), fwd.surrogate,
                          fwd.kept.to(torch.float64), fwd.stats]).cpu().numpy()
    n = p.tokens.size
    lp_cur, entropy, surrogate, kept = host[:n], host[n:2 * n], host[2 * n:3 * n], host[3 * n:4 * n] != 0
    diag = Diagnostics.from_stats(host[4 * n:])
    lp_list = lp_cur.tolist()
    # the reference's per-rollout NumericErrors, in its order (policy.py:287-288, objective.py:
    # 228-229, 241-242): the first rollout with non-finite logits, calibration or ratio raises,
    # after writing back lp_cur for the rollouts before it (and for itself, unless its logits
    # are what failed)
    with np.errstate(over="ignore", invalid="ignore"):
        bad_logits = ~(np.isfinite(lp_cur) & np.isfinite(entropy))
        bad_calib = ~np.isfinite(calib)
        bad_ratio = ~np.isfinite(np.exp(lp_cur - p.lp_old))
    starts = p.cu[:-1]
    per_roll = np.stack([np.logical_or.reduceat(b, starts) for b in (bad_logits, bad_calib, bad_ratio)])
    failing = np.flatnonzero(per_roll.any(axis=0))
    if failing.size:
        r = int(failing[0])
        kind = int(np.argmax(per_roll[:, r]))
        _write_back(p.records, lp_list, int(p.cu[r + (0 if kind == 0 else 1)]))
        raise NumericError(("non-finite logits (corrupted parameters)", "calibration ratio overflow",
                            "importance ratio overflow")[kind])
    _write_back(p.records, lp_list, n)
    if p.error is not None:
        raise p.error
    if not math.isfinite(diag.objective_value) or not bool(grad_finite):
        raise NumericError("objective or gradient is not finite")
    with torch.cuda.device(dev):
        g64 = gw.to(torch.float64)
        if grad_out is not None:
            _page_lock(grad_out)
            torch.from_numpy(grad_out).copy_(g64)
            grad = grad_out
        else:
            out, grad = _fresh_grad(tuple(theta.weights.shape))
            out.copy_(g64)
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
        per_token_surrogate=surrogate,
        per_token_calibration=calib,
        per_token_entropy=entropy,
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


def _record_key(params, temperature: float, precision: str) -> tuple:
    return (id(params.weights), params.version_id, float(temperature), precision)


def record_train_logprobs(groups, params, temperature: float = 1.0, *, precision: str | None = None) -> int:
    """The training engine's old-logprob recording (scheduler.py:296-311) as ONE
    batched device forward -- the lm_head GEMM with the online log-softmax, no objective -- over
    every token generated by `params`' version (gen_version == params.version_id; tokens of
    older versions keep the values recorded when they were generated, as in the reference's
    partial rollouts). Writes TokenRecord.logp_train_old and logp_train_cur (the reference
    initialises both to the same value) and keeps the row's lse and entropy with the record, so
    objective_and_grad with theta is theta_old -- the reference loop's own call,
    scheduler.py:540-541 -- runs the exact on-policy forward (lp_cur == lp_train_old bit for bit,
    no forward GEMM: icepop_fwd_onpolicy). Returns the number of tokens recorded."""
    import torch

    from .features import multihot_device, rollout_feats
    from .loss import IcePopConfig, PackedBatch, icepop_fwd

    precision = precision or _DEFAULT_PRECISION
    n_features, vocab = params.weights.shape
    recs, feats = [], []
    for group in groups:
        for rollout in group.rollouts:
            toks = rollout.tokens
            if not toks:
                continue
            f = rollout_feats(group.task.prompt_id, [r.token for r in toks], n_features)
            keep = [i for i, r in enumerate(toks) if r.gen_version == params.version_id]
            recs += [toks[i] for i in keep]
            feats.append(f[keep])
    if not recs:
        return 0
    n = len(recs)
    dev = torch.device("cuda", torch.cuda.current_device())
    fd = torch.from_numpy(np.ascontiguousarray(np.concatenate(feats), dtype=np.int64)).to(dev)
    zeros = torch.zeros(n, dtype=torch.float64, device=dev)
    batch = PackedBatch(torch.tensor([r.token for r in recs], dtype=torch.int32, device=dev), zeros, zeros,
                        torch.tensor([0, n], dtype=torch.int32, device=dev),
                        torch.tensor([0, 1], dtype=torch.int32, device=dev),
                        torch.zeros(1, dtype=torch.float64, device=dev))
    cfg = IcePopConfig(temperature=float(temperature))
    if precision == "fp64":
        H = multihot_device(fd, n_features, torch.float64)
        W = torch.from_numpy(np.ascontiguousarray(params.weights, dtype=np.float64)).to(dev)
    elif precision == "bf16":
        nf_pad, v_pad, _ = _bf16_shapes(n_features, vocab)
        H = _bf16_hidden(fd, n_features, vocab)
        W = _bf16_weight_into(torch.zeros((nf_pad, v_pad), dtype=torch.bfloat16, device=dev), params.weights,
                              n_features, vocab)
    else:
        raise ValueError("precision must be 'fp64' or 'bf16'")
    f = icepop_fwd(H, W, batch, cfg, layout="dv", store_probs=False)
    lp = f.lp_cur.cpu().tolist()
    lse = f.lse.to(torch.float64).cpu().tolist()
    ent = f.entropy.to(torch.float64).cpu().tolist()
    key = _record_key(params, temperature, precision)
    for rec, a, b, c in zip(recs, lp, lse, ent):
        rec.logp_train_old = rec.logp_train_cur = a
        rec._icepop_record = (key, a, b, c)
    return n


def _onpolicy_stash(records, theta, theta_old, temperature: float, precision: str):
    """(lse, entropy) per record when every record was recorded by record_train_logprobs under
    theta (== theta_old) and still holds that logp_train_old; else None."""
    if theta is not theta_old and (theta.weights is not theta_old.weights or theta.version_id != theta_old.version_id):
        return None
    key = _record_key(theta, temperature, precision)
    out = []
    for rec in records:
        st = getattr(rec, "_icepop_record", None)
        if st is None or st[0] != key or st[1] != rec.logp_train_old:
            return None
        out.append((st[2], st[3]))
    return np.asarray(out, dtype=np.float64)


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
        nf_pad, v_pad, _ = _bf16_shapes(n_features, vocab)
        Wb = _bf16_weight_into(torch.zeros((nf_pad, v_pad), dtype=torch.bfloat16, device=dev), params.weights,
                               n_features, vocab)
        zi = np.full((len(probes), v_pad), -1e30, dtype=np.float32)  # padded columns: probability 0
        zi[:, :vocab] = infer_logits
        d, g, _, _ = _device_delta_gap(_bf16_hidden(fd, n_features, vocab), Wb, torch.from_numpy(zi).to(dev),
                                       layout="dv", temperature=temperature)
    else:
        raise ValueError("precision must be 'fp64' or 'bf16'")
    out = torch.stack([d, g]).cpu().numpy()
    return float(out[0]), float(out[1])


def _recording(step):
    """Wrap a scheduler iteration (run_iteration / run_iteration_baseline): after the reference
    generates and completes its groups, re-record the fresh tokens' logp_train_old in one batched
    device forward (record_train_logprobs), so the loop's objective_and_grad(groups, params,
    params, ...) takes the exact on-policy path."""

    @functools.wraps(step)
    def wrapper(state, params, cfg, group_cfg, *args, **kwargs):
        report, groups = step(state, params, cfg, group_cfg, *args, **kwargs)
        if groups:
            record_train_logprobs(groups, params, state.temperature)
        return report, groups

    wrapper.__wrapped_step__ = step
    return wrapper


def install(precision: str | None = None, *, record: bool = False) -> None:
    """Rebind mismatchlab's objective_and_grad, group_advantages, the update step
    that follows it (sgd_update / momentum_update, scheduler.py:551-555) and the discrepancy
    probe (delta_and_gap) to this drop-in, in every module that binds the names (objective.py,
    scheduler.py:29-40, discrepancy.py, __init__.py:15-34). ``record=True`` also re-records the
    fresh tokens' logp_train_old of every train_loop iteration on the device; a
    later objective_and_grad(groups, params, params, None, ...) on those groups runs the exact
    on-policy forward (bf16 precision; train_loop itself always passes a reference policy for
    the KL diagnostic, which needs the forward GEMM)."""
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
        mod.group_advantages = group_advantages  # K0 (objective.py:153-159, scheduler.py:353-354)
    # the discrepancy probe: measure() (discrepancy.py:144-161, called by train_loop) looks the
    # name up in its own module
    for mod in (mismatchlab, mismatchlab.discrepancy):
        mod.delta_and_gap = delta_and_gap
    if record:  # the old-logprob recording of train_loop's iterations on the device (8f-1)
        for name in ("run_iteration", "run_iteration_baseline"):
            step = getattr(mismatchlab.scheduler, name)
            if not hasattr(step, "__wrapped_step__"):
                setattr(mismatchlab.scheduler, name, _recording(step))


__all__ = [
    "Algo", "LossBreakdown", "MaskingBounds", "ObjectiveConfig", "PromptGroup", "TokenRecord", "empty_breakdown",
    "delta_and_gap", "group_advantages", "install", "mask", "momentum_update", "objective_and_grad",
    "record_train_logprobs", "set_default_precision", "sgd_update",
]
