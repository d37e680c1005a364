"""Tensor-level IcePop objective on B200: the torch face of ``libicepop_b200.so``.

Three layers, all on device, none with a CPU fallback:

* :func:`icepop_fwd` / :func:`icepop_bwd` -- functional forward (K1 fused lm_head GEMM +
  online log-softmax, K2 IcePop epilogue) and backward. The backward is either row-scaled
  GEMMs on the probabilities K1 stored when they fit in HBM (dH = s(Q.W) + cW[y],
  dW = Q^T(sH) + scatter), or bf16 dZ recomputed by the K3 GEMM in chunks, then K4 dHidden,
  K5 dW. Dispatched on dtype: bfloat16 -> tcgen05 path, float64 -> SIMT validation path.
* :func:`icepop_fwd_bwd` -- both in one call (objective_and_grad's shape), in token chunks
  when the whole batch's probabilities do not fit.
* :func:`icepop_loss` -- a ``torch.library`` custom op with autograd (loss = -J), for
  training code that wants ``loss.backward()``.
* :class:`PackedBatch` -- the packed per-token / per-sequence metadata the kernels read
  (the reference's ``PromptGroup``/``TokenRecord`` objects flattened in its own
  group-major order, objective.py:204-276).

Semantics follow objective.py:172-298; ``stats`` holds this
rank's partial sums (include/icepop.h ``enum icepop_stat``) -- sum them across ranks
(``paper_2510_18855_b200.distributed``) before deriving the global diagnostics.
"""

from __future__ import annotations

import functools
import math
import os
import time
from dataclasses import dataclass, field

import torch

from . import _lib

ALGOS = {"icepop": _lib.ALGO_ICEPOP, "grpo": _lib.ALGO_GRPO, "tis": _lib.ALGO_TIS}
LAYOUTS = {"dv": _lib.W_DV, "vd": _lib.W_VD}

# Largest bf16 dZ chunk the backward materialises (bytes); the rest of the batch is
# processed in further chunks with dW accumulated in place. Default: up to 96 GB, capped at
# 60% of the device memory free at call time (one chunk at C2: 82 GB; fewer chunks means
# fewer dW read-modify-writes and wave tails -- measured +0.3% at C2 vs 32 GB chunks).
DZ_CHUNK_BYTES = int(os.environ.get("ICEPOP_DZ_CHUNK_BYTES", str(96 * 10**9)))


# Stored-probabilities mode (include/icepop.h): K1 also writes bf16 q = 2^(z log2e - R)
# [N, V] so the backward needs no K3 logit recompute (6 instead of 8 N.d.V FLOPs per step).
# "auto" stores them when 2.N.V bytes fit in STORE_PROBS_FRACTION of the free device memory.
STORE_PROBS = os.environ.get("ICEPOP_STORE_PROBS", "auto")
STORE_PROBS_FRACTION = 0.6


def _resolve_store_probs(store_probs, n: int, v: int, device, kl_grad: bool) -> bool:
    """Whether the forward stores the probabilities. Never with the KL-to-ref gradient
    (gamma > 0: the recompute forms it); with a reference policy and gamma = 0 the KL term is a
    diagnostic of the forward only, so the probabilities are stored as usual."""
    if store_probs is None:
        store_probs = {"auto": None, "1": True, "0": False}.get(STORE_PROBS.lower(), None)
    if store_probs is False or kl_grad or v % 8 != 0 or n == 0:
        return False
    if store_probs is True:
        return True
    need = 2 * n * v + 4 * n * _lib.tile_max_ld(v)
    free = _free_bytes(device, need)
    return free is not None and need <= STORE_PROBS_FRACTION * free


_DRIVER_FREE: dict = {}  # device index -> (time, cudaMemGetInfo free bytes, torch reserved bytes then)


def _torch_counters(idx: int) -> tuple[int, int]:
    """(reserved, allocated) bytes of torch's caching allocator on device idx."""
    try:  # the flat counters directly: torch.cuda.memory_reserved() flattens every statistic
        st = torch._C._cuda_memoryStats(idx)
        return st["reserved_bytes"]["all"]["current"], st["allocated_bytes"]["all"]["current"]
    except Exception:  # noqa: BLE001
        return torch.cuda.memory_reserved(idx), torch.cuda.memory_allocated(idx)


def _free_bytes(device, need: int | None = None) -> int | None:
    """Device memory available to a new allocation: free in the driver plus what torch's
    caching allocator holds unused (e.g. the previous step's probabilities / dZ block).
    cudaMemGetInfo costs ~1 ms (7% of a drop-in call at C1): a reading under 2 s old is reused,
    less what torch reserved since, when `need` is at most a quarter of what it showed free."""
    try:
        idx = torch.device(device).index
        idx = torch.cuda.current_device() if idx is None else idx
        reserved, allocated = _torch_counters(idx)
        now = time.monotonic()
        hit = _DRIVER_FREE.get(idx)
        if need is None or hit is None or now - hit[0] > 2.0 or need > hit[1] // 4:
            hit = (now, torch.cuda.mem_get_info(idx)[0], reserved)
            _DRIVER_FREE[idx] = hit
        driver_free = hit[1] - max(0, reserved - hit[2])
        return driver_free + reserved - allocated
    except Exception:  # noqa: BLE001
        return None


def _take_probs(fwd: "IcePopForward", kl_grad: bool):
    """(probs, tile_max) of a stored-probabilities forward, or (None, None). The backward may
    overwrite rows of probs with dZ, so they are handed out once (a second backward recomputes)."""
    if kl_grad or fwd.extras.get("probs") is None:
        return None, None
    return fwd.extras.pop("probs"), fwd.extras.pop("tile_max")


def _bwd_workspace(n: int, d: int, v: int, n_seqs: int, device) -> torch.Tensor:
    """The recompute-mode backward workspace with the largest dZ chunk that allocates: the
    free-memory estimate counts torch's cached blocks, which fragmentation can make unusable
    for one large block, so an out-of-memory halves the chunk (down to 128 rows)."""
    cb = _dz_chunk_bytes(device, 2 * n * (v + d))
    while True:
        try:
            return torch.empty(bwd_workspace_bytes(n, d, v, n_seqs, cb), dtype=torch.uint8, device=device)
        except torch.OutOfMemoryError:
            if cb <= 128 * 2 * (v + d):
                raise
            cb = max(128 * 2 * (v + d), cb // 2)


SP_ROWSCALE = os.environ.get("ICEPOP_SP_ROWSCALE", "1") != "0"


def sp_workspace_bytes(n: int, d: int, v: int, n_seqs: int) -> int:
    """Bytes of the stored-probabilities (row-scaled) backward workspace for n tokens."""
    lib = _lib.load()
    shape = _lib.Shape(n_tokens=n, token_offset=0, hidden=d, vocab=v, n_seqs=max(n_seqs, 1), n_groups=1,
                       weight_layout=_lib.W_VD)
    b = _lib._sz()
    _lib.check(lib.icepop_workspace_bytes(shape, -1, 0, None, b))
    return max(b.value, 1)


def _sp_workspace(n: int, d: int, v: int, n_seqs: int, device) -> torch.Tensor | None:
    """Workspace of the stored-probabilities backward: block lists, row scales, s*H and the
    one-hot sort buffers (about 2*n*d bytes). None (no memory, or ICEPOP_SP_ROWSCALE=0): the
    backward then forms dZ in place over every row instead (same result up to rounding)."""
    if not SP_ROWSCALE:
        return None
    try:
        return torch.empty(sp_workspace_bytes(n, d, v, n_seqs), dtype=torch.uint8, device=device)
    except torch.OutOfMemoryError:
        return None


def _dz_chunk_bytes(device, need: int | None = None) -> int:
    """Bytes for the recompute backward's dZ chunk (+ transposed hidden rows): the cap, or 60%
    of the free device memory. `need` (the whole batch's bytes) lets a recent free-memory reading
    stand in when it is small against it (_free_bytes)."""
    free = _free_bytes(device, need)
    if free is None:
        return DZ_CHUNK_BYTES
    return max(1, min(DZ_CHUNK_BYTES, int(0.6 * free)))


@dataclass(frozen=True)
class IcePopConfig:
    """objective.py:47-82 (MaskingBounds + ObjectiveConfig) and the temperature."""

    alpha: float = 0.5
    beta: float = 5.0
    clip_eps: float = 0.2
    tis_cap: float = 2.0
    temperature: float = 1.0
    kl_coeff: float = 0.0
    algo: str = "icepop"

    def to_c(self) -> _lib.Config:
        if self.algo not in ALGOS:
            raise ValueError(f"unknown algorithm {self.algo!r}")
        return _lib.Config(
            alpha=self.alpha,
            beta=self.beta,
            clip_eps=self.clip_eps,
            tis_cap=self.tis_cap,
            temperature=self.temperature,
            kl_coeff=self.kl_coeff,
            algo=ALGOS[self.algo],
        )


@dataclass
class PackedBatch:
    """Packed rollout batch, device tensors.

    tokens / lp_train_old / lp_infer_old cover this rank's contiguous token range
    [token_offset, token_offset + n_local); cu_seqlens, group_offsets and advantages
    (or rewards) describe the GLOBAL batch and are replicated on every rank.
    """

    tokens: torch.Tensor  # int32 [n_local]
    lp_train_old: torch.Tensor  # float64 [n_local]
    lp_infer_old: torch.Tensor  # float64 [n_local]
    cu_seqlens: torch.Tensor  # int32 [S+1]
    group_offsets: torch.Tensor  # int32 [n_groups+1]
    advantages: torch.Tensor | None = None  # float64 [S]
    rewards: torch.Tensor | None = None  # float64 [S] (advantages computed by K0 if None)
    token_offset: int = 0
    calib: torch.Tensor | None = None  # float64 [n_local] caller-computed exp(lp_old - lp_inf), optional

    @property
    def n_seqs(self) -> int:
        return int(self.cu_seqlens.numel()) - 1

    @property
    def n_groups(self) -> int:
        return int(self.group_offsets.numel()) - 1

    def to_c(self) -> _lib.Batch:
        return _lib.Batch(
            tokens=_lib.ptr(self.tokens),
            lp_train_old=_lib.ptr(self.lp_train_old),
            lp_infer_old=_lib.ptr(self.lp_infer_old),
            cu_seqlens=_lib.ptr(self.cu_seqlens),
            group_offsets=_lib.ptr(self.group_offsets),
            advantages=_lib.ptr(self.advantages),
            rewards=_lib.ptr(self.rewards),
            calib=_lib.ptr(self.calib),
        )

    def validate(self) -> None:
        for name in ("tokens", "cu_seqlens", "group_offsets"):
            if getattr(self, name).dtype != torch.int32:
                raise ValueError(f"{name} must be int32")
        if self.calib is not None and (self.calib.dtype != torch.float64 or self.calib.numel() != self.tokens.numel()):
            raise ValueError("calib must be float64 with one entry per token")
        for name in ("lp_train_old", "lp_infer_old"):
            if getattr(self, name).dtype != torch.float64:
                raise ValueError(f"{name} must be float64 (the mask is computed bit-exactly in fp64)")
        if self.advantages is None and self.rewards is None:
            raise ValueError("either advantages or rewards must be given")
        if self.n_groups < 1:
            raise ValueError("objective needs at least one prompt group")


@dataclass
class IcePopForward:
    """Per-token outputs (this rank) and the fp64 partial statistics vector."""

    lse: torch.Tensor
    lp_cur: torch.Tensor
    entropy: torch.Tensor
    kept: torch.Tensor
    calib: torch.Tensor
    surrogate: torch.Tensor
    coeff: torch.Tensor
    stats: torch.Tensor  # float64 [8] on device
    kl: torch.Tensor | None = None
    lse_ref: torch.Tensor | None = None
    extras: dict = field(default_factory=dict)


def _shape(hidden: torch.Tensor, weight: torch.Tensor, layout: str, batch: PackedBatch) -> _lib.Shape:
    if layout not in LAYOUTS:
        raise ValueError(f"weight layout must be 'dv' ([d,V]) or 'vd' ([V,d]), got {layout!r}")
    if hidden.dim() != 2 or weight.dim() != 2:
        raise ValueError("hidden and weight must be 2-D")
    n, d = hidden.shape
    if layout == "dv":
        dw, v = weight.shape
    else:
        v, dw = weight.shape
    if dw != d:
        raise ValueError(f"hidden dim {d} does not match weight {tuple(weight.shape)} ({layout})")
    if batch.tokens.numel() != n or batch.lp_train_old.numel() != n or batch.lp_infer_old.numel() != n:
        raise ValueError("per-token tensors must have one entry per hidden row")
    return _lib.Shape(
        n_tokens=n,
        token_offset=batch.token_offset,
        hidden=d,
        vocab=v,
        n_seqs=batch.n_seqs,
        n_groups=batch.n_groups,
        weight_layout=LAYOUTS[layout],
    )


def _stream(device: torch.device) -> int:
    return torch.cuda.current_stream(device).cuda_stream


def _on_device(fn):
    """Run an entry point with its tensors' device current: the library launches on the current
    CUDA device, so a call on cuda:1 tensors while cuda:0 is current must switch first (the
    stream passed is always the tensors' device's current stream)."""

    @functools.wraps(fn)
    def wrapper(*args, **kwargs):
        t = args[0] if args else next(iter(kwargs.values()), None)
        if isinstance(t, PackedBatch):
            t = t.tokens
        if isinstance(t, torch.Tensor) and t.is_cuda:
            with torch.cuda.device(t.device):
                return fn(*args, **kwargs)
        return fn(*args, **kwargs)

    return wrapper


def _lib_for(t: torch.Tensor):
    if t.device.type != "cuda":
        raise RuntimeError("libicepop_b200 runs on CUDA tensors only (no CPU fallback)")
    return _lib.ensure_device(t.device.index if t.device.index is not None else torch.cuda.current_device())


@_on_device
def icepop_fwd(
    hidden: torch.Tensor,
    weight: torch.Tensor,
    batch: PackedBatch,
    cfg: IcePopConfig = IcePopConfig(),
    layout: str = "vd",
    weight_ref: torch.Tensor | None = None,
    store_probs: bool | None = None,
    probs_buffers: tuple[torch.Tensor, torch.Tensor] | None = None,
    keep_workspace: bool = False,
) -> IcePopForward:
    """Forward of the IcePop objective on this rank's tokens (objective.py:215-278).

    ``keep_workspace`` (bf16): keep K1's per-row partials in ``extras`` so that
    :func:`icepop_epilogue` can re-run the IcePop epilogue (other bounds, algorithm, clip
    epsilon or advantages) without another GEMM.

    ``store_probs`` (bf16 path): keep the bf16 probabilities for the backward (True / False /
    None = ``ICEPOP_STORE_PROBS``, default "auto": when they fit in device memory).
    ``probs_buffers``: caller-owned (probs [>=N, V] bf16, tile_max [>=N, tile_max_ld(V)] f32)
    to store them in (implies store_probs; icepop_fwd_bwd reuses one pair across token chunks).
    """
    lib = _lib_for(hidden)
    batch.validate()
    hidden = hidden.contiguous()
    weight = weight.contiguous()
    shape = _shape(hidden, weight, layout, batch)
    dev = hidden.device
    n = shape.n_tokens
    st = _stream(dev)
    stats = torch.empty(_lib.NSTATS, dtype=torch.float64, device=dev)
    kept = torch.empty(n, dtype=torch.uint8, device=dev)
    calib = torch.empty(n, dtype=torch.float64, device=dev)
    surrogate = torch.empty(n, dtype=torch.float64, device=dev)
    lp_cur = torch.empty(n, dtype=torch.float64, device=dev)
    c_cfg = cfg.to_c()
    c_batch = batch.to_c()
    if hidden.dtype == torch.bfloat16:
        if weight.dtype != torch.bfloat16:
            raise ValueError("bf16 hidden needs a bf16 weight")
        wr = None
        if weight_ref is not None:
            wr = weight_ref.contiguous()
            if wr.shape != weight.shape or wr.dtype != torch.bfloat16:
                raise ValueError("weight_ref must match weight's shape and dtype")
        lse = torch.empty(n, dtype=torch.float32, device=dev)
        entropy = torch.empty(n, dtype=torch.float32, device=dev)
        coeff = torch.empty(n, dtype=torch.float32, device=dev)
        kl = lse_ref = kl_w = None
        if wr is not None:
            kl = torch.empty(n, dtype=torch.float32, device=dev)
            lse_ref = torch.empty(n, dtype=torch.float32, device=dev)
            kl_w = torch.empty(n, dtype=torch.float32, device=dev)
        probs = tile_max = None
        kl_grad = wr is not None and cfg.kl_coeff > 0.0
        if probs_buffers is not None:
            pb, tb = probs_buffers
            tm_ld = _lib.tile_max_ld(shape.vocab)
            if (pb.dtype != torch.bfloat16 or pb.dim() != 2 or pb.shape[0] < n or pb.shape[1] != shape.vocab
                    or tb.dtype != torch.float32 or tb.dim() != 2 or tb.shape[0] < n or tb.shape[1] != tm_ld
                    or not pb.is_contiguous() or not tb.is_contiguous() or kl_grad):
                raise ValueError("probs_buffers must be contiguous (bf16 [>=N, V], f32 [>=N, tile_max_ld(V)]) "
                                 "and cannot be combined with the KL gradient (weight_ref with kl_coeff > 0)")
            probs, tile_max = pb[:n], tb[:n]
        elif _resolve_store_probs(store_probs, n, shape.vocab, dev, kl_grad):
            try:
                probs = torch.empty((n, shape.vocab), dtype=torch.bfloat16, device=dev)
                tile_max = torch.empty((n, _lib.tile_max_ld(shape.vocab)), dtype=torch.float32, device=dev)
            except torch.OutOfMemoryError:
                if store_probs is True:
                    raise
                probs = tile_max = None  # "auto": the recompute mode needs no [N, V] buffer
        fwd_b = _lib._sz()
        _lib.check(lib.icepop_workspace_bytes(shape, 0, 1 if wr is not None else 0, fwd_b, None))
        ws = torch.empty(max(fwd_b.value, 1), dtype=torch.uint8, device=dev)
        out = _lib.FwdOut(
            lse=lse.data_ptr(),
            lp_cur=lp_cur.data_ptr(),
            entropy=entropy.data_ptr(),
            kept=kept.data_ptr(),
            calib=calib.data_ptr(),
            surrogate=surrogate.data_ptr(),
            coeff=coeff.data_ptr(),
            stats=stats.data_ptr(),
            kl=_lib.ptr(kl),
            lse_ref=_lib.ptr(lse_ref),
            kl_w=_lib.ptr(kl_w),
            probs=_lib.ptr(probs),
            tile_max=_lib.ptr(tile_max),
        )
        _lib.check(lib.icepop_fwd_bf16(shape, c_cfg, hidden.data_ptr(), weight.data_ptr(), _lib.ptr(wr), c_batch,
                                       out, ws.data_ptr(), ws.numel(), st))
        f = IcePopForward(lse, lp_cur, entropy, kept, calib, surrogate, coeff, stats, kl=kl, lse_ref=lse_ref)
        f.extras["kl_w"] = kl_w
        if probs is not None:
            f.extras["probs"], f.extras["tile_max"] = probs, tile_max
        if keep_workspace:
            f.extras["fwd_workspace"] = (ws, shape, wr is not None)
            f.extras["temperature"] = cfg.temperature
        return f
    if hidden.dtype == torch.float64:
        if weight.dtype != torch.float64:
            raise ValueError("fp64 hidden needs an fp64 weight")
        wr = None
        if weight_ref is not None:
            wr = weight_ref.contiguous()
            if wr.shape != weight.shape or wr.dtype != torch.float64:
                raise ValueError("weight_ref must match weight's shape and dtype")
        lse = torch.empty(n, dtype=torch.float64, device=dev)
        entropy = torch.empty(n, dtype=torch.float64, device=dev)
        coeff = torch.empty(n, dtype=torch.float64, device=dev)
        kl = torch.zeros(n, dtype=torch.float64, device=dev)
        lse_ref = torch.zeros(n, dtype=torch.float64, device=dev)
        nb = _lib._sz()
        _lib.check(lib.icepop_workspace_bytes_f64(shape, 1 if wr is not None else 0, nb))
        ws = torch.empty(max(nb.value, 1), dtype=torch.uint8, device=dev)
        out = _lib.F64Out(
            lse=lse.data_ptr(),
            lp_cur=lp_cur.data_ptr(),
            entropy=entropy.data_ptr(),
            kl=kl.data_ptr(),
            lse_ref=lse_ref.data_ptr(),
            kept=kept.data_ptr(),
            calib=calib.data_ptr(),
            surrogate=surrogate.data_ptr(),
            coeff=coeff.data_ptr(),
            stats=stats.data_ptr(),
        )
        _lib.check(lib.icepop_fwd_f64(shape, c_cfg, hidden.data_ptr(), weight.data_ptr(), _lib.ptr(wr), c_batch,
                                      out, ws.data_ptr(), ws.numel(), st))
        return IcePopForward(lse, lp_cur, entropy, kept, calib, surrogate, coeff, stats, kl=kl, lse_ref=lse_ref)
    raise ValueError(f"unsupported dtype {hidden.dtype}: use bfloat16 (tensor cores) or float64 (validation)")


@_on_device
def icepop_epilogue(batch: PackedBatch, fwd: IcePopForward, cfg: IcePopConfig = IcePopConfig()) -> IcePopForward:
    """Re-run the IcePop epilogue (K2: log-softmax merge, mask, ratio, clip, surrogate,
    coefficients, statistics) over the K1 partials a ``keep_workspace=True`` forward kept, with
    another config / batch metadata (same tokens, weights and temperature). Returns new outputs;
    no GEMM runs. include/icepop.h icepop_fwd_epilogue_bf16."""
    if "fwd_workspace" not in fwd.extras:
        raise ValueError("the forward must be run with keep_workspace=True")
    ws, shape, with_ref = fwd.extras["fwd_workspace"]
    if cfg.temperature != fwd.extras.get("temperature", cfg.temperature):
        raise ValueError("the epilogue cannot change the temperature (the partials are of z / T)")
    lib = _lib_for(ws)
    batch.validate()
    n = int(shape.n_tokens)
    if batch.tokens.numel() != n:
        raise ValueError("batch does not match the forward's token count")
    dev = ws.device
    e = lambda dt: torch.empty(n, dtype=dt, device=dev)  # noqa: E731
    out = IcePopForward(e(torch.float32), e(torch.float64), e(torch.float32), e(torch.uint8), e(torch.float64),
                        e(torch.float64), e(torch.float32), torch.empty(_lib.NSTATS, dtype=torch.float64, device=dev))
    if with_ref:
        out.kl, out.lse_ref = e(torch.float32), e(torch.float32)
        out.extras["kl_w"] = e(torch.float32)
    sh = _lib.Shape(n_tokens=n, token_offset=batch.token_offset, hidden=shape.hidden, vocab=shape.vocab,
                    n_seqs=batch.n_seqs, n_groups=batch.n_groups, weight_layout=shape.weight_layout)
    c_out = _lib.FwdOut(lse=out.lse.data_ptr(), lp_cur=out.lp_cur.data_ptr(), entropy=out.entropy.data_ptr(),
                        kept=out.kept.data_ptr(), calib=out.calib.data_ptr(), surrogate=out.surrogate.data_ptr(),
                        coeff=out.coeff.data_ptr(), stats=out.stats.data_ptr(), kl=_lib.ptr(out.kl),
                        lse_ref=_lib.ptr(out.lse_ref), kl_w=_lib.ptr(out.extras.get("kl_w")))
    _lib.check(lib.icepop_fwd_epilogue_bf16(sh, cfg.to_c(), batch.to_c(), 1 if with_ref else 0, c_out, ws.data_ptr(),
                                            ws.numel(), _stream(dev)))
    return out


@_on_device
def icepop_logprob(hidden: torch.Tensor, weight: torch.Tensor, tokens: torch.Tensor, layout: str = "vd",
                   temperature: float = 1.0) -> tuple[torch.Tensor, torch.Tensor, torch.Tensor]:
    """log pi(y_t), lse_t and entropy_t with the K1 kernel (the train engine's lp recording,
    scheduler.py:296-311 / policy.py:411-442): returns (lp f64, lse f32, entropy f32)."""
    lib = _lib_for(hidden)
    if hidden.dtype != torch.bfloat16 or weight.dtype != torch.bfloat16:
        raise ValueError("icepop_logprob runs on bf16 hidden/weight")
    hidden, weight = hidden.contiguous(), weight.contiguous()
    n, d = hidden.shape
    v = weight.shape[1] if layout == "dv" else weight.shape[0]
    shape = _lib.Shape(n_tokens=n, token_offset=0, hidden=d, vocab=v, n_seqs=1, n_groups=1,
                       weight_layout=LAYOUTS[layout])
    dev = hidden.device
    fb = _lib._sz()
    _lib.check(lib.icepop_workspace_bytes(shape, 0, 0, fb, None))
    ws = torch.empty(max(fb.value, 1), dtype=torch.uint8, device=dev)
    lp = torch.empty(n, dtype=torch.float64, device=dev)
    lse = torch.empty(n, dtype=torch.float32, device=dev)
    ent = torch.empty(n, dtype=torch.float32, device=dev)
    _lib.check(lib.icepop_logprob_bf16(shape, float(temperature), hidden.data_ptr(), weight.data_ptr(),
                                       tokens.data_ptr(), lse.data_ptr(), lp.data_ptr(), ent.data_ptr(),
                                       ws.data_ptr(), ws.numel(), _stream(dev)))
    return lp, lse, ent


@_on_device
def icepop_fwd_onpolicy(batch: PackedBatch, lse_old: torch.Tensor, entropy_old: torch.Tensor | None,
                        cfg: IcePopConfig = IcePopConfig(), hidden_dim: int = 8, vocab: int = 8) -> IcePopForward:
    """Forward when theta == theta_old and batch.lp_train_old came from :func:`icepop_logprob`
    with the same weights: lp_cur == lp_train_old exactly, so no GEMM runs (6.d.V per token
    for the whole loss step instead of 8.d.V). Pair with icepop_bwd as usual."""
    lib = _lib_for(batch.tokens)
    batch.validate()
    n = batch.tokens.numel()
    dev = batch.tokens.device
    shape = _lib.Shape(n_tokens=n, token_offset=batch.token_offset, hidden=hidden_dim, vocab=vocab,
                       n_seqs=batch.n_seqs, n_groups=batch.n_groups, weight_layout=_lib.W_VD)
    f = IcePopForward(torch.empty(n, dtype=torch.float32, device=dev), torch.empty(n, dtype=torch.float64, device=dev),
                      torch.empty(n, dtype=torch.float32, device=dev), torch.empty(n, dtype=torch.uint8, device=dev),
                      torch.empty(n, dtype=torch.float64, device=dev), torch.empty(n, dtype=torch.float64, device=dev),
                      torch.empty(n, dtype=torch.float32, device=dev),
                      torch.empty(_lib.NSTATS, dtype=torch.float64, device=dev))
    fb = _lib._sz()  # (the workspace query wants the bf16 path's multiples of 8; the size only grows)
    ws_shape = _lib.Shape(n_tokens=n, token_offset=batch.token_offset, hidden=-(-hidden_dim // 8) * 8,
                          vocab=-(-vocab // 8) * 8, n_seqs=batch.n_seqs, n_groups=batch.n_groups,
                          weight_layout=_lib.W_VD)
    _lib.check(lib.icepop_workspace_bytes(ws_shape, 0, 0, fb, None))
    ws = torch.empty(max(fb.value, 1), dtype=torch.uint8, device=dev)
    out = _lib.FwdOut(lse=f.lse.data_ptr(), lp_cur=f.lp_cur.data_ptr(), entropy=f.entropy.data_ptr(),
                      kept=f.kept.data_ptr(), calib=f.calib.data_ptr(), surrogate=f.surrogate.data_ptr(),
                      coeff=f.coeff.data_ptr(), stats=f.stats.data_ptr())
    _lib.check(lib.icepop_fwd_onpolicy(shape, cfg.to_c(), batch.to_c(), lse_old.data_ptr(), _lib.ptr(entropy_old),
                                       out, ws.data_ptr(), ws.numel(), _stream(dev)))
    return f


@_on_device
def discrepancy(hidden: torch.Tensor, weight_p: torch.Tensor, weight_q: torch.Tensor, layout: str = "vd",
                temperature: float = 1.0) -> tuple[torch.Tensor, torch.Tensor]:
    """delta = mean_t KL(pi_p(.|t) || pi_q(.|t)) over the rows of `hidden` (the probe
    contexts), e.g. p = the inference engine's weights, q = the training weights
    (discrepancy.py:132-141). Returns (delta as a device fp64 scalar, per-row kl f32)."""
    lib = _lib_for(hidden)
    if hidden.dtype != torch.bfloat16 or weight_p.dtype != torch.bfloat16 or weight_q.dtype != torch.bfloat16:
        raise ValueError("discrepancy runs on bf16 hidden/weights")
    if weight_p.shape != weight_q.shape:
        raise ValueError("weight_p and weight_q must have the same shape")
    hidden, weight_p, weight_q = hidden.contiguous(), weight_p.contiguous(), weight_q.contiguous()
    n, d = hidden.shape
    v = weight_p.shape[1] if layout == "dv" else weight_p.shape[0]
    shape = _lib.Shape(n_tokens=n, token_offset=0, hidden=d, vocab=v, n_seqs=1, n_groups=1,
                       weight_layout=LAYOUTS[layout])
    dev = hidden.device
    fb = _lib._sz()
    _lib.check(lib.icepop_workspace_bytes(shape, 0, 1, fb, None))
    ws = torch.empty(max(fb.value, 1), dtype=torch.uint8, device=dev)
    kl = torch.empty(n, dtype=torch.float32, device=dev)
    mean = torch.empty((), dtype=torch.float64, device=dev)
    _lib.check(lib.icepop_kl_bf16(shape, float(temperature), hidden.data_ptr(), weight_p.data_ptr(),
                                  weight_q.data_ptr(), kl.data_ptr(), None, None, mean.data_ptr(), ws.data_ptr(),
                                  ws.numel(), _stream(dev)))
    return mean, kl


@_on_device
def delta_and_gap(hidden: torch.Tensor, weight: torch.Tensor, infer_logits: torch.Tensor, layout: str = "vd",
                  temperature: float = 1.0):
    """delta = mean_t KL(p_infer,t || p_train,t) and max_token_gap = max_{t,v} |p_infer - p_train|
    over the probe rows of `hidden` (discrepancy.py:132-141), given the inference engine's logits
    `infer_logits` [n, V] (already divided by the temperature, as the reference perturbs the
    scaled train logits). The train logits are H.W / temperature from the lm_head GEMM.

    bf16 hidden / weight with fp32 infer_logits (tensor cores), or all fp64 (SIMT, for the
    reference's exact tests). Returns (delta, max_gap) as device fp64 scalars and the per-row
    (kl, gap) fp64 vectors. include/icepop.h icepop_delta_gap_*."""
    lib = _lib_for(hidden)
    f64 = hidden.dtype == torch.float64
    if f64:
        if weight.dtype != torch.float64 or infer_logits.dtype != torch.float64:
            raise ValueError("the fp64 probe needs fp64 hidden, weight and infer_logits")
    elif hidden.dtype != torch.bfloat16 or weight.dtype != torch.bfloat16 or infer_logits.dtype != torch.float32:
        raise ValueError("the probe runs on bf16 hidden/weight with fp32 infer_logits (or all fp64)")
    hidden, weight, infer_logits = hidden.contiguous(), weight.contiguous(), infer_logits.contiguous()
    n, d = hidden.shape
    v = weight.shape[1] if layout == "dv" else weight.shape[0]
    if tuple(infer_logits.shape) != (n, v):
        raise ValueError(f"infer_logits must be [{n}, {v}]")
    shape = _lib.Shape(n_tokens=n, token_offset=0, hidden=d, vocab=v, n_seqs=1, n_groups=1,
                       weight_layout=LAYOUTS[layout])
    dev = hidden.device
    nb = _lib._sz()
    _lib.check(lib.icepop_delta_gap_workspace_bytes(shape, 1 if f64 else 0, nb))
    ws = torch.empty(max(nb.value, 1), dtype=torch.uint8, device=dev)
    kl = torch.empty(n, dtype=torch.float64, device=dev)
    gap = torch.empty(n, dtype=torch.float64, device=dev)
    out = torch.empty(2, dtype=torch.float64, device=dev)
    fn = lib.icepop_delta_gap_f64 if f64 else lib.icepop_delta_gap_bf16
    _lib.check(fn(shape, float(temperature), hidden.data_ptr(), weight.data_ptr(), infer_logits.data_ptr(),
                  kl.data_ptr(), gap.data_ptr(), out.data_ptr(), out.data_ptr() + 8, ws.data_ptr(), ws.numel(),
                  _stream(dev)))
    return out[0], out[1], kl, gap


def bwd_workspace_bytes(n_tokens: int, hidden: int, vocab: int, n_seqs: int, chunk_bytes: int | None = None) -> int:
    """Backward workspace for a dZ chunk of at most `chunk_bytes` (default DZ_CHUNK_BYTES)."""
    lib = _lib.load()
    shape = _lib.Shape(n_tokens=n_tokens, token_offset=0, hidden=hidden, vocab=vocab, n_seqs=max(n_seqs, 1),
                       n_groups=1, weight_layout=_lib.W_VD)
    cb = DZ_CHUNK_BYTES if chunk_bytes is None else chunk_bytes
    rows = cb // (2 * (vocab + hidden))  # a bf16 dZ row and the row of H transposed for K5
    chunk = n_tokens if rows >= n_tokens else max(128, rows // 128 * 128)
    bwd_b = _lib._sz()
    _lib.check(lib.icepop_workspace_bytes(shape, chunk, 0, None, bwd_b))
    return bwd_b.value


@_on_device
def icepop_bwd(
    hidden: torch.Tensor,
    weight: torch.Tensor,
    batch: PackedBatch,
    fwd: IcePopForward,
    cfg: IcePopConfig = IcePopConfig(),
    layout: str = "vd",
    grad_scale: float = 1.0,
    need_hidden: bool = True,
    need_weight: bool = True,
    grad_weight: torch.Tensor | None = None,
    weight_ref: torch.Tensor | None = None,
    grad_hidden_dtype: torch.dtype | None = None,
    workspace: torch.Tensor | None = None,
) -> tuple[torch.Tensor | None, torch.Tensor | None]:
    """Gradients of grad_scale * J: (d/dhidden, d/dweight), objective.py:250-266.

    ``grad_weight`` (f32 for bf16 inputs, f64 for fp64), if given, is accumulated into.
    ``workspace`` (bf16, stored-probabilities forward): a caller-owned uint8 buffer of at least
    sp_workspace_bytes(...) used instead of allocating one.
    """
    lib = _lib_for(hidden)
    hidden = hidden.contiguous()
    weight = weight.contiguous()
    shape = _shape(hidden, weight, layout, batch)
    dev = hidden.device
    st = _stream(dev)
    n, d, v = shape.n_tokens, shape.hidden, shape.vocab
    c_cfg = cfg.to_c()
    wshape = tuple(weight.shape)
    if hidden.dtype == torch.bfloat16:
        gh_dtype = grad_hidden_dtype or torch.bfloat16
        if gh_dtype not in (torch.bfloat16, torch.float32):
            raise ValueError("grad_hidden_dtype must be bfloat16 or float32")
        gh = torch.empty((n, d), dtype=gh_dtype, device=dev) if need_hidden else None
        accumulate = grad_weight is not None
        gw = grad_weight if accumulate else (torch.empty(wshape, dtype=torch.float32, device=dev) if need_weight else None)
        if gw is not None and (gw.dtype != torch.float32 or tuple(gw.shape) != wshape or not gw.is_contiguous()):
            raise ValueError("grad_weight must be a contiguous float32 tensor shaped like weight")
        wr = weight_ref.contiguous() if weight_ref is not None else None
        probs, tile_max = _take_probs(fwd, wr is not None and cfg.kl_coeff > 0.0)
        if probs is None:
            ws = _bwd_workspace(n, d, v, shape.n_seqs, dev)
        elif workspace is not None and SP_ROWSCALE and workspace.numel() >= sp_workspace_bytes(n, d, v, shape.n_seqs):
            ws = workspace
        else:
            ws = _sp_workspace(n, d, v, shape.n_seqs, dev)
        saved = _lib.Saved(tokens=batch.tokens.data_ptr(), lse=fwd.lse.data_ptr(), coeff=fwd.coeff.data_ptr(),
                           lse_ref=_lib.ptr(fwd.lse_ref), kl=_lib.ptr(fwd.kl), kl_w=_lib.ptr(fwd.extras.get("kl_w")),
                           probs=_lib.ptr(probs), tile_max=_lib.ptr(tile_max), lp_cur=_lib.ptr(fwd.lp_cur))
        _lib.check(lib.icepop_bwd_bf16(shape, c_cfg, hidden.data_ptr(), weight.data_ptr(), _lib.ptr(wr), saved,
                                       float(grad_scale), _lib.ptr(gh), 1 if gh_dtype == torch.float32 else 0,
                                       _lib.ptr(gw), 1 if accumulate else 0, _lib.ptr(ws),
                                       0 if ws is None else ws.numel(), st))
        return gh, gw
    if hidden.dtype == torch.float64:
        gh = torch.empty((n, d), dtype=torch.float64, device=dev) if need_hidden else None
        accumulate = grad_weight is not None
        gw = grad_weight if accumulate else (torch.empty(wshape, dtype=torch.float64, device=dev) if need_weight else None)
        wr = weight_ref.contiguous() if weight_ref is not None else None
        nb = _lib._sz()
        kl_grad = wr is not None and cfg.kl_coeff > 0.0
        _lib.check(lib.icepop_workspace_bytes_f64(shape, 1 if kl_grad else 0, nb))
        ws = torch.empty(max(nb.value, 1), dtype=torch.uint8, device=dev)
        f = _lib.F64Out(
            lse=fwd.lse.data_ptr(),
            lp_cur=fwd.lp_cur.data_ptr(),
            entropy=fwd.entropy.data_ptr(),
            kl=_lib.ptr(fwd.kl),
            lse_ref=_lib.ptr(fwd.lse_ref),
            kept=None,
            calib=None,
            surrogate=None,
            coeff=fwd.coeff.data_ptr(),
            stats=fwd.stats.data_ptr(),
        )
        _lib.check(lib.icepop_bwd_f64(shape, c_cfg, hidden.data_ptr(), weight.data_ptr(), _lib.ptr(wr),
                                      batch.to_c(), f, float(grad_scale), _lib.ptr(gh), _lib.ptr(gw),
                                      1 if accumulate else 0, ws.data_ptr(), ws.numel(), st))
        return gh, gw
    raise ValueError(f"unsupported dtype {hidden.dtype}")


@_on_device
def icepop_bwd_reduce_scatter(
    hidden: torch.Tensor,
    weight: torch.Tensor,
    batch: PackedBatch,
    fwd: IcePopForward,
    rs_target,
    cfg: IcePopConfig = IcePopConfig(),
    layout: str = "vd",
    grad_scale: float = 1.0,
    need_hidden: bool = True,
    weight_ref: torch.Tensor | None = None,
    grad_hidden_dtype: torch.dtype | None = None,
) -> torch.Tensor | None:
    """Backward whose dW leaves this rank inside K5's epilogue: every row goes to its owner's
    peer slot (``distributed.PeerSlots.target()``). Returns dHidden; dW is obtained by each
    owner with ``PeerSlots.fold`` after ``distributed.stream_barrier``."""
    lib = _lib_for(hidden)
    if hidden.dtype != torch.bfloat16:
        raise ValueError("the fused reduce-scatter runs on the bf16 path")
    hidden, weight = hidden.contiguous(), weight.contiguous()
    shape = _shape(hidden, weight, layout, batch)
    dev = hidden.device
    n, d, v = shape.n_tokens, shape.hidden, shape.vocab
    gh_dtype = grad_hidden_dtype or torch.bfloat16
    gh = torch.empty((n, d), dtype=gh_dtype, device=dev) if need_hidden else None
    wr = weight_ref.contiguous() if weight_ref is not None else None
    probs, tile_max = _take_probs(fwd, wr is not None and cfg.kl_coeff > 0.0)
    scratch = None
    if probs is None:
        ws = _bwd_workspace(n, d, v, shape.n_seqs, dev)
        single_chunk = ws.numel() >= bwd_workspace_bytes(n, d, v, shape.n_seqs, 2 * n * (v + d))
        scratch = None if single_chunk else torch.empty(tuple(weight.shape), dtype=torch.float32, device=dev)
    else:  # stored probabilities: one chunk; the one-hot part of dW goes straight to the slots
        ws = _sp_workspace(n, d, v, shape.n_seqs, dev)
    saved = _lib.Saved(tokens=batch.tokens.data_ptr(), lse=fwd.lse.data_ptr(), coeff=fwd.coeff.data_ptr(),
                       lse_ref=_lib.ptr(fwd.lse_ref), kl=_lib.ptr(fwd.kl), kl_w=_lib.ptr(fwd.extras.get("kl_w")),
                       probs=_lib.ptr(probs), tile_max=_lib.ptr(tile_max), lp_cur=_lib.ptr(fwd.lp_cur))
    _lib.check(lib.icepop_bwd_bf16_rs(shape, cfg.to_c(), hidden.data_ptr(), weight.data_ptr(), _lib.ptr(wr), saved,
                                      float(grad_scale), _lib.ptr(gh), 1 if gh_dtype == torch.float32 else 0,
                                      rs_target, _lib.ptr(scratch), _lib.ptr(ws), 0 if ws is None else ws.numel(),
                                      _stream(dev)))
    return gh


_PROBS_CHUNK_OK: dict = {}  # (device index, vocab) -> a token-chunk size whose buffers allocated


def probs_chunk_tokens(n: int, vocab: int, device) -> int:
    """Largest token count (multiple of 4096, or n) whose stored probabilities fit in
    STORE_PROBS_FRACTION of the device memory available now; 0 if not even 4096 do."""
    per = 2 * vocab + 4 * _lib.tile_max_ld(vocab)
    free = _free_bytes(device, per * n)
    if free is None:
        return 0
    rows = int(STORE_PROBS_FRACTION * free) // per
    if rows >= n:
        return n
    return rows // 4096 * 4096


@_on_device
def icepop_fwd_bwd(
    hidden: torch.Tensor,
    weight: torch.Tensor,
    batch: PackedBatch,
    cfg: IcePopConfig = IcePopConfig(),
    layout: str = "vd",
    grad_scale: float = 1.0,
    need_hidden: bool = True,
    grad_weight: torch.Tensor | None = None,
    weight_ref: torch.Tensor | None = None,
    grad_hidden_dtype: torch.dtype | None = None,
    max_chunk_tokens: int | None = None,
) -> tuple[IcePopForward, torch.Tensor | None, torch.Tensor]:
    """Forward and gradient in one call, as objective_and_grad returns them (objective.py:172-298).

    On the bf16 path the backward forms dZ from stored probabilities. When the whole batch's
    probabilities (2*N*V bytes) do not fit in device memory, the batch runs in token chunks
    that do fit. Each chunk is a token range with its global offset, exactly like a token
    shard (distributed.py): the statistics are summed (error bits OR-ed) and dW is accumulated.
    So the backward still executes 6.d.V instead of 8.d.V FLOPs per token. It falls back to
    icepop_fwd + icepop_bwd (logit recompute) for the KL gradient, fp64 inputs, or when not
    even 4096 tokens' probabilities fit. Returns (forward outputs, dHidden or None, dW f32).
    """
    n = hidden.shape[0]
    v = weight.shape[1] if layout == "dv" else weight.shape[0]
    kl_grad = weight_ref is not None and cfg.kl_coeff > 0.0
    usable = hidden.dtype == torch.bfloat16 and not kl_grad and v % 8 == 0 and n > 0 and hidden.is_cuda
    chunk = 0
    if usable:
        chunk = probs_chunk_tokens(n, v, hidden.device)
        if max_chunk_tokens:
            chunk = min(chunk, max_chunk_tokens)
    if chunk <= 0:
        f = icepop_fwd(hidden, weight, batch, cfg, layout, weight_ref=weight_ref)
        gh, gw = icepop_bwd(hidden, weight, batch, f, cfg, layout, grad_scale, need_hidden, True, grad_weight,
                            weight_ref, grad_hidden_dtype)
        return f, gh, gw
    if chunk >= n:
        f = icepop_fwd(hidden, weight, batch, cfg, layout, weight_ref=weight_ref, store_probs=True)
        gh, gw = icepop_bwd(hidden, weight, batch, f, cfg, layout, grad_scale, need_hidden, True, grad_weight,
                            weight_ref, grad_hidden_dtype=grad_hidden_dtype)
        return f, gh, gw
    dev = hidden.device
    gw = grad_weight if grad_weight is not None else torch.zeros(tuple(weight.shape), dtype=torch.float32, device=dev)
    gh = torch.empty((n, hidden.shape[1]), dtype=grad_hidden_dtype or torch.bfloat16, device=dev) if need_hidden \
        else None
    # One probabilities buffer (and backward workspace) for all chunks: re-allocating tens of GB
    # per chunk lets smaller allocations fragment torch's cache between chunks. If the estimate
    # was too optimistic for one block, the chunk halves (down to 4096 tokens), and the size that
    # allocated is remembered for this device and vocabulary, so a training loop does not pay a
    # failed allocation (and torch's cache flush behind it) on every step.
    n_seqs = batch.n_seqs
    key = (dev.index, v)
    chunk = min(chunk, _PROBS_CHUNK_OK.get(key, chunk))
    while True:
        try:
            bufs = (torch.empty((chunk, v), dtype=torch.bfloat16, device=dev),
                    torch.empty((chunk, _lib.tile_max_ld(v)), dtype=torch.float32, device=dev))
            break
        except torch.OutOfMemoryError:
            if chunk <= 4096:
                raise
            chunk = max(4096, chunk // 2 // 4096 * 4096)
            _PROBS_CHUNK_OK[key] = chunk
    ws = _sp_workspace(chunk, hidden.shape[1], v, n_seqs, dev)
    parts = []
    stats = torch.zeros(_lib.NSTATS, dtype=torch.float64, device=dev)
    for s0 in range(0, n, chunk):
        e0 = min(n, s0 + chunk)
        sub = PackedBatch(batch.tokens[s0:e0], batch.lp_train_old[s0:e0], batch.lp_infer_old[s0:e0],
                          batch.cu_seqlens, batch.group_offsets, batch.advantages, batch.rewards,
                          token_offset=batch.token_offset + s0,
                          calib=batch.calib[s0:e0] if batch.calib is not None else None)
        f = icepop_fwd(hidden[s0:e0], weight, sub, cfg, layout, weight_ref=weight_ref, probs_buffers=bufs)
        ghc, _ = icepop_bwd(hidden[s0:e0], weight, sub, f, cfg, layout, grad_scale, need_hidden, True, gw,
                            weight_ref, grad_hidden_dtype=grad_hidden_dtype, workspace=ws)
        if gh is not None:
            gh[s0:e0] = ghc
        stats[: _lib.STAT_ERRORS] += f.stats[: _lib.STAT_ERRORS]
        stats[_lib.STAT_ERRORS] = (stats[_lib.STAT_ERRORS].long() | f.stats[_lib.STAT_ERRORS].long()).double()
        parts.append(f)
    cat = lambda name: torch.cat([getattr(p, name) for p in parts])  # noqa: E731
    out = IcePopForward(cat("lse"), cat("lp_cur"), cat("entropy"), cat("kept"), cat("calib"), cat("surrogate"),
                        cat("coeff"), stats, kl=cat("kl") if weight_ref is not None else None,
                        lse_ref=cat("lse_ref") if weight_ref is not None else None)
    out.extras["chunks"] = len(parts)
    return out, gh, gw


@_on_device
def finish(stats: torch.Tensor) -> None:
    """One host sync; raise NumericError/ValueError from the device error word."""
    lib = _lib.load()
    _lib.check(lib.icepop_finish(stats.data_ptr(), _stream(stats.device)))


@dataclass
class Diagnostics:
    """Global diagnostics derived from the all-reduced stats (objective.py:282-298)."""

    objective_value: float
    clipped_fraction: float
    token_count: int
    mean_logp: float
    entropy_all: float
    entropy_clipped: float
    kl_to_ref: float

    @classmethod
    def from_stats(cls, stats) -> "Diagnostics":
        s = [float(x) for x in (stats.tolist() if hasattr(stats, "tolist") else stats)]
        n = s[_lib.STAT_TOKENS]
        popped = s[_lib.STAT_N_POPPED]
        return cls(
            objective_value=s[_lib.STAT_OBJECTIVE],
            clipped_fraction=popped / n if n else 0.0,
            token_count=int(round(n)),
            mean_logp=s[_lib.STAT_SUM_LOGP] / n if n else math.nan,
            entropy_all=s[_lib.STAT_SUM_ENTROPY] / n if n else math.nan,
            entropy_clipped=s[_lib.STAT_SUM_ENTROPY_POPPED] / popped if popped else math.nan,
            kl_to_ref=s[_lib.STAT_SUM_KL] / n if n else math.nan,
        )


# --------------------------------------------------------------------------- custom ops
# Two torch.library ops: the forward (pure) and the backward, which declares that it overwrites
# the stored probabilities (its dZ is formed in place in them), so functionalization and
# torch.compile see the mutation. The probabilities travel to the backward as a ctx attribute,
# not a saved tensor: they are consumed (and freed) by the first backward; a second one
# (retain_graph) recomputes the logits.
def _cfg_of(alpha, beta, clip_eps, tis_cap, temperature, kl_coeff, algo) -> IcePopConfig:
    return IcePopConfig(alpha, beta, clip_eps, tis_cap, temperature, kl_coeff, {v: k for k, v in ALGOS.items()}[algo])


@torch.library.custom_op("icepop_b200::icepop_loss", mutates_args=())
def _icepop_loss_op(
    hidden: torch.Tensor,
    weight: torch.Tensor,
    weight_ref: torch.Tensor | None,
    tokens: torch.Tensor,
    lp_train_old: torch.Tensor,
    lp_infer_old: torch.Tensor,
    cu_seqlens: torch.Tensor,
    group_offsets: torch.Tensor,
    advantages: torch.Tensor,
    alpha: float,
    beta: float,
    clip_eps: float,
    tis_cap: float,
    temperature: float,
    kl_coeff: float,
    algo: int,
    layout: int,
    token_offset: int,
    store_probs: bool,
) -> tuple[torch.Tensor, torch.Tensor, torch.Tensor, torch.Tensor, torch.Tensor, torch.Tensor, torch.Tensor,
           torch.Tensor, torch.Tensor, torch.Tensor, torch.Tensor, torch.Tensor]:
    cfg = _cfg_of(alpha, beta, clip_eps, tis_cap, temperature, kl_coeff, algo)
    batch = PackedBatch(tokens, lp_train_old, lp_infer_old, cu_seqlens, group_offsets, advantages,
                        token_offset=token_offset)
    sp = store_probs and hidden.dtype == torch.bfloat16
    f = icepop_fwd(hidden, weight, batch, cfg, "dv" if layout == _lib.W_DV else "vd", weight_ref=weight_ref,
                   store_probs=sp)
    loss = -f.stats[_lib.STAT_OBJECTIVE]
    empty = lambda dt: hidden.new_empty((0,), dtype=dt)  # noqa: E731  outputs must be fresh tensors
    probs = f.extras.get("probs")
    tile_max = f.extras.get("tile_max")
    if probs is None:
        probs, tile_max = empty(torch.bfloat16), empty(torch.float32)
    kl = f.kl if weight_ref is not None else empty(f.lse.dtype)
    lse_ref = f.lse_ref if weight_ref is not None else empty(f.lse.dtype)
    kl_w = f.extras.get("kl_w")
    if kl_w is None:
        kl_w = empty(torch.float32)
    return (loss, f.stats, f.lse, f.lp_cur, f.entropy, f.kept, f.coeff.to(torch.float64), kl, lse_ref, kl_w, probs,
            tile_max)


@_icepop_loss_op.register_fake
def _(hidden, weight, weight_ref, tokens, lp_train_old, lp_infer_old, cu_seqlens, group_offsets, advantages, alpha,
      beta, clip_eps, tis_cap, temperature, kl_coeff, algo, layout, token_offset, store_probs):
    n = hidden.shape[0]
    dev = hidden.device
    f64 = dict(dtype=torch.float64, device=dev)
    # lse / entropy / kl are f32 on the bf16 path and f64 on the validation path
    fx = dict(dtype=torch.float64 if hidden.dtype == torch.float64 else torch.float32, device=dev)
    v = weight.shape[1] if layout == _lib.W_DV else weight.shape[0]
    sp = store_probs and hidden.dtype == torch.bfloat16 and not (weight_ref is not None and kl_coeff > 0)
    ref = weight_ref is not None
    kl_w_n = n if ref and hidden.dtype == torch.bfloat16 else 0
    return (hidden.new_empty((), dtype=torch.float64), torch.empty(_lib.NSTATS, **f64), torch.empty(n, **fx),
            torch.empty(n, **f64), torch.empty(n, **fx), torch.empty(n, dtype=torch.uint8, device=dev),
            torch.empty(n, **f64), torch.empty(n if ref else 0, **fx), torch.empty(n if ref else 0, **fx),
            torch.empty(kl_w_n, dtype=torch.float32, device=dev),
            torch.empty((n, v) if sp else (0,), dtype=torch.bfloat16, device=dev),
            torch.empty((n, _lib.tile_max_ld(v)) if sp else (0,), dtype=torch.float32, device=dev))


@torch.library.custom_op("icepop_b200::icepop_loss_backward", mutates_args=("probs",))
def _icepop_loss_backward_op(
    grad_loss: torch.Tensor,
    hidden: torch.Tensor,
    weight: torch.Tensor,
    weight_ref: torch.Tensor | None,
    tokens: torch.Tensor,
    lp_train_old: torch.Tensor,
    lp_infer_old: torch.Tensor,
    cu_seqlens: torch.Tensor,
    group_offsets: torch.Tensor,
    advantages: torch.Tensor,
    lse: torch.Tensor,
    lp_cur: torch.Tensor,
    coeff: torch.Tensor,
    kl: torch.Tensor,
    lse_ref: torch.Tensor,
    kl_w: torch.Tensor,
    probs: torch.Tensor,
    tile_max: torch.Tensor,
    alpha: float,
    beta: float,
    clip_eps: float,
    tis_cap: float,
    temperature: float,
    kl_coeff: float,
    algo: int,
    layout: int,
    token_offset: int,
    need_hidden: bool,
    need_weight: bool,
) -> tuple[torch.Tensor, torch.Tensor]:
    """d(loss)/d(hidden), d(loss)/d(weight) for loss = -J (grad_loss scales them on the device,
    no host sync). Overwrites `probs` (when non-empty) with dZ rows."""
    cfg = _cfg_of(alpha, beta, clip_eps, tis_cap, temperature, kl_coeff, algo)
    batch = PackedBatch(tokens, lp_train_old, lp_infer_old, cu_seqlens, group_offsets, advantages,
                        token_offset=token_offset)
    scale = -grad_loss.to(torch.float64)
    ref = weight_ref is not None
    if hidden.dtype == torch.bfloat16:
        fwd = IcePopForward(lse, lp_cur, None, None, None, None, (coeff * scale).to(torch.float32), None,
                            kl=kl if ref else None, lse_ref=lse_ref if ref else None)
        if ref:  # the KL gradient's coefficient carries the same scale
            fwd.extras["kl_w"] = (kl_w.to(torch.float64) * scale).to(torch.float32)
        if probs.numel():
            fwd.extras["probs"], fwd.extras["tile_max"] = probs, tile_max
    else:
        fwd = IcePopForward(lse, torch.empty_like(lse, dtype=torch.float64), torch.empty_like(lse, dtype=torch.float64),
                            None, None, None, coeff * scale, torch.zeros(_lib.NSTATS, dtype=torch.float64,
                                                                         device=lse.device),
                            kl=kl if ref else None, lse_ref=lse_ref if ref else None)
    lay = "dv" if layout == _lib.W_DV else "vd"
    # the fp64 path takes the KL gradient's scale through grad_scale (its kl_w is formed inside)
    gscale = 1.0 if hidden.dtype == torch.bfloat16 or not ref or kl_coeff == 0.0 else None
    if gscale is None:  # fp64 with the KL gradient: one host read of grad_loss (validation path)
        gscale = float(-grad_loss.item())
        fwd.coeff = coeff
    gh, gw = icepop_bwd(hidden, weight, batch, fwd, cfg, lay, gscale, need_hidden, need_weight, weight_ref=weight_ref)
    gh = gh.to(hidden.dtype) if gh is not None else hidden.new_empty((0,))
    gw = gw.to(weight.dtype) if gw is not None else weight.new_empty((0,))
    return gh, gw


@_icepop_loss_backward_op.register_fake
def _(grad_loss, hidden, weight, weight_ref, tokens, lp_train_old, lp_infer_old, cu_seqlens, group_offsets,
      advantages, lse, lp_cur, coeff, kl, lse_ref, kl_w, probs, tile_max, alpha, beta, clip_eps, tis_cap,
      temperature, kl_coeff, algo, layout, token_offset, need_hidden, need_weight):
    return (torch.empty_like(hidden) if need_hidden else hidden.new_empty((0,)),
            torch.empty_like(weight) if need_weight else weight.new_empty((0,)))


def _setup_context(ctx, inputs, output):
    (hidden, weight, weight_ref, tokens, lp_old, lp_inf, cu, go, adv, alpha, beta, clip_eps, tis_cap, temperature,
     kl_coeff, algo, layout, token_offset, store_probs) = inputs
    loss, stats, lse, lp_cur, entropy, kept, coeff, kl, lse_ref, kl_w, probs, tile_max = output
    ctx.save_for_backward(hidden, weight, weight_ref, tokens, lp_old, lp_inf, cu, go, adv, lse, lp_cur, coeff, kl,
                          lse_ref, kl_w)
    ctx.cfg = (alpha, beta, clip_eps, tis_cap, temperature, kl_coeff, algo, layout, token_offset)
    # consumed by the first backward (its rows become dZ); not a saved tensor, so the declared
    # in-place write does not trip autograd's version check, and the memory is released after
    ctx.probs = (probs, tile_max) if probs.numel() else None


def _backward(ctx, grad_loss, *unused):
    hidden, weight, weight_ref, tokens, lp_old, lp_inf, cu, go, adv, lse, lp_cur, coeff, kl, lse_ref, kl_w = \
        ctx.saved_tensors
    probs, tile_max = ctx.probs if ctx.probs is not None else (hidden.new_empty((0,), dtype=torch.bfloat16),
                                                                hidden.new_empty((0,), dtype=torch.float32))
    ctx.probs = None  # a second backward (retain_graph) recomputes
    gh, gw = _icepop_loss_backward_op(grad_loss, hidden, weight, weight_ref, tokens, lp_old, lp_inf, cu, go, adv, lse,
                                      lp_cur, coeff, kl, lse_ref, kl_w, probs, tile_max, *ctx.cfg,
                                      ctx.needs_input_grad[0], ctx.needs_input_grad[1])
    return (gh if ctx.needs_input_grad[0] else None, gw if ctx.needs_input_grad[1] else None) + (None,) * 17


_icepop_loss_op.register_autograd(_backward, setup_context=_setup_context)


def icepop_loss(
    hidden: torch.Tensor,
    weight: torch.Tensor,
    batch: PackedBatch,
    cfg: IcePopConfig = IcePopConfig(),
    layout: str = "vd",
    store_probs: bool | None = None,
    weight_ref: torch.Tensor | None = None,
):
    """Differentiable IcePop loss (= -J on this rank's tokens) and per-token aux.

    Returns ``(loss, aux)`` with aux = dict(stats, lse, lp_cur, entropy, kept, coeff[, kl]).
    ``batch.advantages`` must be given (compute them with K0 via :func:`group_advantages` when
    starting from rewards). ``store_probs``: as in :func:`icepop_fwd` (the probabilities live
    until the first backward consumes them). ``weight_ref`` with ``cfg.kl_coeff`` adds the
    KL-to-ref term (objective.py:254-263; a frozen reference: it receives no gradient).
    """
    if batch.advantages is None:
        raise ValueError("icepop_loss needs batch.advantages (see group_advantages)")
    if layout not in LAYOUTS:
        raise ValueError(f"weight layout must be 'dv' or 'vd', got {layout!r}")
    v = weight.shape[1] if layout == "dv" else weight.shape[0]
    kl_grad = weight_ref is not None and cfg.kl_coeff > 0.0
    sp = hidden.is_cuda and hidden.dtype == torch.bfloat16 and _resolve_store_probs(
        store_probs, hidden.shape[0], v, hidden.device, kl_grad)
    wr = weight_ref.detach() if weight_ref is not None else None
    (loss, stats, lse, lp_cur, entropy, kept, coeff, kl, _lse_ref, _kl_w, _probs, _tile_max) = _icepop_loss_op(
        hidden, weight, wr, batch.tokens, batch.lp_train_old, batch.lp_infer_old, batch.cu_seqlens,
        batch.group_offsets, batch.advantages, cfg.alpha, cfg.beta, cfg.clip_eps, cfg.tis_cap, cfg.temperature,
        cfg.kl_coeff if weight_ref is not None else 0.0, ALGOS[cfg.algo], LAYOUTS[layout], batch.token_offset,
        bool(sp))
    aux = dict(stats=stats, lse=lse, lp_cur=lp_cur, entropy=entropy, kept=kept, coeff=coeff)
    if weight_ref is not None:
        aux["kl"] = kl
    return loss, aux


@_on_device
def group_advantages(rewards: torch.Tensor, group_offsets: torch.Tensor) -> torch.Tensor:
    """K0 on device: per-group z-scored rewards (objective.py:153-159), bit-identical to numpy."""
    lib = _lib_for(rewards)
    if rewards.dtype != torch.float64 or group_offsets.dtype != torch.int32:
        raise ValueError("rewards must be float64 and group_offsets int32")
    if group_offsets.device.type == "cpu":  # host offsets: validate, then move
        if bool((torch.diff(group_offsets) < 2).any()):
            raise ValueError("advantage normalization needs a group of >= 2 rewards")
        group_offsets = group_offsets.to(rewards.device)
    out = torch.empty_like(rewards)
    _lib.check(lib.icepop_group_advantages(rewards.data_ptr(), group_offsets.data_ptr(), group_offsets.numel() - 1,
                                           rewards.numel(), out.data_ptr(), _stream(rewards.device)))
    return out
