"""Dense (Ling-style) inputs on the bf16 tcgen05 path vs the fp64 oracle on the same
bf16-rounded inputs: ragged packed sequences, tails that are not tile multiples, both
weight layouts, both CTA configurations, token shards, error semantics and autograd.

Tolerances: kept mask / popped count bit-exact; lp_cur, entropy abs <= 2e-3 (+1e-3 rel);
objective rel <= 1e-3; dW, dH relative Frobenius error <= 1e-2.
"""

from __future__ import annotations

import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu


def _case(n_seqs=6, d=320, V=1000, seed=0, lens=None, group=3, sigma=0.3, layout="vd"):
    rng = np.random.default_rng(seed)
    lens = lens or list(rng.integers(40, 400, n_seqs))
    N = int(sum(lens))
    H = torch.from_numpy(rng.normal(0, 1, (N, d))).to(torch.bfloat16)
    shape_w = (V, d) if layout == "vd" else (d, V)
    W = torch.from_numpy(rng.normal(0, 2 / np.sqrt(d), shape_w)).to(torch.bfloat16)
    tokens = rng.integers(0, V, N).astype(np.int32)
    # lp_old near the model's own log-prob so ratios straddle the clip band
    Hd, Wd = H.double().numpy(), W.double().numpy()
    z = Hd @ (Wd.T if layout == "vd" else Wd)
    lse = z.max(1) + np.log(np.exp(z - z.max(1, keepdims=True)).sum(1))
    lp_old = z[np.arange(N), tokens] - lse + rng.normal(0, 0.15, N)
    lp_inf = lp_old - rng.normal(0, sigma, N)
    cu = np.concatenate([[0], np.cumsum(lens)]).astype(np.int32)
    go = np.arange(0, n_seqs + 1, group).astype(np.int32)
    if go[-1] != n_seqs:
        go = np.append(go, n_seqs).astype(np.int32)
    adv = rng.normal(0, 1, n_seqs)
    return dict(H=H, W=W, tokens=tokens, lp_old=lp_old, lp_inf=lp_inf, cu=cu, go=go, adv=adv, layout=layout)


def _batch(c, dev, sl=None):
    from paper_2510_18855_b200.loss import PackedBatch

    sl = sl or slice(0, len(c["tokens"]))
    return PackedBatch(torch.from_numpy(c["tokens"][sl]).to(dev), torch.from_numpy(c["lp_old"][sl]).to(dev),
                       torch.from_numpy(c["lp_inf"][sl]).to(dev), torch.from_numpy(c["cu"]).to(dev),
                       torch.from_numpy(c["go"]).to(dev), torch.from_numpy(c["adv"]).to(dev),
                       token_offset=sl.start or 0)


def _oracle(c, **kw):
    from oracle.icepop_oracle import icepop_dense

    return icepop_dense(c["H"].double().numpy(), c["W"].double().numpy(), c["tokens"], c["lp_old"], c["lp_inf"],
                        c["cu"], c["go"], c["adv"], layout=c["layout"], **kw)


def _rel(a, b):
    return float(np.linalg.norm(np.asarray(a, np.float64) - b) / max(np.linalg.norm(b), 1e-30))


@pytest.fixture(params=[1, 2], ids=["cta1", "cta2"])
def cta_group(request):
    from paper_2510_18855_b200 import _lib

    lib = _lib.ensure_device(0)
    _lib.check(lib.icepop_set_cta_group(request.param))
    yield request.param
    _lib.check(lib.icepop_set_cta_group(2))


@pytest.mark.parametrize("store_probs", [True, False], ids=["probs", "recompute"])
@pytest.mark.parametrize("layout", ["vd", "dv"])
@pytest.mark.parametrize("algo", ["icepop", "grpo", "tis"])
def test_dense_bf16_vs_oracle(cuda_device, cta_group, layout, algo, store_probs):
    from paper_2510_18855_b200.loss import Diagnostics, IcePopConfig, finish, icepop_bwd, icepop_fwd

    c = _case(seed=3, layout=layout)
    cfg = IcePopConfig(algo=algo)
    b = _batch(c, cuda_device)
    f = icepop_fwd(c["H"].to(cuda_device), c["W"].to(cuda_device), b, cfg, layout=layout, store_probs=store_probs)
    assert ("probs" in f.extras) == store_probs
    gh, gw = icepop_bwd(c["H"].to(cuda_device), c["W"].to(cuda_device), b, f, cfg, layout=layout,
                        grad_hidden_dtype=torch.float32)
    finish(f.stats)
    o = _oracle(c, algo=algo)
    diag = Diagnostics.from_stats(f.stats.cpu())
    assert np.array_equal(f.kept.cpu().numpy().astype(bool), o["kept"])
    assert diag.clipped_fraction == o["clipped_fraction"]
    if algo == "icepop":
        assert 0 < o["n_clipped"] < len(c["tokens"])  # the case really pops tokens
    np.testing.assert_allclose(f.lp_cur.cpu().numpy(), o["lp_cur"], atol=2e-3, rtol=1e-3)
    np.testing.assert_allclose(f.lse.cpu().numpy(), o["lse"], atol=2e-3, rtol=1e-4)
    np.testing.assert_allclose(f.entropy.cpu().numpy(), o["entropy"], atol=2e-3, rtol=1e-3)
    assert diag.objective_value == pytest.approx(o["objective"], rel=1e-3, abs=1e-6)
    assert _rel(gw.cpu().numpy(), o["grad_weight"]) < 1e-2
    assert _rel(gh.cpu().numpy(), o["grad_hidden"]) < 1e-2


def test_shards_sum_to_full_batch(cuda_device):
    """Token ranges cutting sequences mid-way (token_offset) reproduce the full batch."""
    from paper_2510_18855_b200.loss import IcePopConfig, icepop_bwd, icepop_fwd

    c = _case(n_seqs=5, seed=7)
    H, W = c["H"].to(cuda_device), c["W"].to(cuda_device)
    cfg = IcePopConfig()
    full = icepop_fwd(H, W, _batch(c, cuda_device), cfg)
    _, gw_full = icepop_bwd(H, W, _batch(c, cuda_device), full, cfg, need_hidden=False)
    N = len(c["tokens"])
    cuts = [0, int(c["cu"][1]) + 17, N // 2 + 3, N]
    stats = torch.zeros(8, dtype=torch.float64, device=cuda_device)
    gw = torch.zeros_like(gw_full)
    kept = []
    for s, e in zip(cuts, cuts[1:]):
        b = _batch(c, cuda_device, slice(s, e))
        f = icepop_fwd(H[s:e], W, b, cfg)
        icepop_bwd(H[s:e], W, b, f, cfg, need_hidden=False, grad_weight=gw)
        stats[:7] += f.stats[:7]
        kept.append(f.kept)
        assert torch.equal(f.calib, full.calib[s:e])
        assert torch.equal(f.coeff, full.coeff[s:e])
    assert torch.equal(torch.cat(kept), full.kept)
    torch.testing.assert_close(stats[:7], full.stats[:7], rtol=1e-9, atol=1e-12)
    assert _rel(gw.cpu().numpy(), gw_full.cpu().numpy()) < 1e-5


def test_backward_chunking_matches_single_chunk(cuda_device, monkeypatch):
    """A small dZ workspace forces several token chunks with dW accumulated in place."""
    import paper_2510_18855_b200.loss as L

    c = _case(n_seqs=4, seed=11, lens=[300, 260, 130, 500])
    H, W = c["H"].to(cuda_device), c["W"].to(cuda_device)
    f = L.icepop_fwd(H, W, _batch(c, cuda_device), L.IcePopConfig(), store_probs=False)  # chunks: recompute mode
    gh1, gw1 = L.icepop_bwd(H, W, _batch(c, cuda_device), f, L.IcePopConfig())
    monkeypatch.setattr(L, "DZ_CHUNK_BYTES", 256 * (1000 + H.shape[1]) * 2)  # 256-row chunks (dZ + H^T rows)
    gh2, gw2 = L.icepop_bwd(H, W, _batch(c, cuda_device), f, L.IcePopConfig())
    assert torch.equal(gh1, gh2)
    assert _rel(gw2.cpu().numpy(), gw1.cpu().numpy()) < 1e-5  # fp32 partial sums per chunk


def test_temperature(cuda_device):
    from paper_2510_18855_b200.loss import Diagnostics, IcePopConfig, icepop_bwd, icepop_fwd

    c = _case(seed=5)
    cfg = IcePopConfig(temperature=0.6)
    H, W = c["H"].to(cuda_device), c["W"].to(cuda_device)
    f = icepop_fwd(H, W, _batch(c, cuda_device), cfg)
    gh, gw = icepop_bwd(H, W, _batch(c, cuda_device), f, cfg, grad_hidden_dtype=torch.float32)
    o = _oracle(c, temperature=0.6)
    np.testing.assert_allclose(f.lp_cur.cpu().numpy(), o["lp_cur"], atol=3e-3, rtol=1e-3)
    assert Diagnostics.from_stats(f.stats.cpu()).objective_value == pytest.approx(o["objective"], rel=2e-3)
    assert _rel(gw.cpu().numpy(), o["grad_weight"]) < 1e-2
    assert _rel(gh.cpu().numpy(), o["grad_hidden"]) < 1e-2


def test_numeric_error_on_calibration_overflow(cuda_device):
    from paper_2510_18855_b200.errors import NumericError
    from paper_2510_18855_b200.loss import IcePopConfig, finish, icepop_fwd

    c = _case(seed=2)
    c["lp_old"] = c["lp_old"].copy()
    c["lp_old"][5] = 800.0  # exp(800 - lp_inf) overflows (objective.py:228-229)
    f = icepop_fwd(c["H"].to(cuda_device), c["W"].to(cuda_device), _batch(c, cuda_device), IcePopConfig())
    with pytest.raises(NumericError, match="calibration ratio overflow"):
        finish(f.stats)


def test_token_out_of_vocab_is_value_error(cuda_device):
    from paper_2510_18855_b200.loss import IcePopConfig, finish, icepop_fwd

    c = _case(seed=2)
    c["tokens"] = c["tokens"].copy()
    c["tokens"][3] = 1000  # == V
    f = icepop_fwd(c["H"].to(cuda_device), c["W"].to(cuda_device), _batch(c, cuda_device), IcePopConfig())
    with pytest.raises(ValueError, match="vocabulary"):
        finish(f.stats)


def test_config_validation_matches_reference():
    from paper_2510_18855_b200 import _lib
    from paper_2510_18855_b200.loss import IcePopConfig, icepop_fwd

    c = _case(seed=1)
    dev = torch.device("cuda", 0)
    for bad in (IcePopConfig(alpha=1.5), IcePopConfig(beta=0.9), IcePopConfig(clip_eps=1.0),
                IcePopConfig(tis_cap=0.0), IcePopConfig(temperature=0.0)):
        with pytest.raises(ValueError):
            icepop_fwd(c["H"].to(dev), c["W"].to(dev), _batch(c, dev), bad)
    assert _lib.load().icepop_abi_version() == _lib.ABI_VERSION


def test_custom_op_autograd_matches_functional(cuda_device):
    """loss = -J through torch.library custom op; grads equal -dJ/dW, -dJ/dH."""
    from paper_2510_18855_b200.loss import IcePopConfig, icepop_bwd, icepop_fwd, icepop_loss

    c = _case(seed=9)
    H = c["H"].to(cuda_device).requires_grad_(True)
    W = c["W"].to(cuda_device).requires_grad_(True)
    b = _batch(c, cuda_device)
    loss, aux = icepop_loss(H, W, b, IcePopConfig(), layout="vd")
    (2.0 * loss).backward()
    f = icepop_fwd(H.detach(), W.detach(), b, IcePopConfig())
    gh, gw = icepop_bwd(H.detach(), W.detach(), b, f, IcePopConfig(), grad_scale=-2.0,
                        grad_hidden_dtype=torch.float32)
    assert loss.item() == pytest.approx(-f.stats[0].item(), rel=1e-12)
    assert _rel(H.grad.float().cpu().numpy(), gh.cpu().numpy()) < 1e-2
    assert _rel(W.grad.float().cpu().numpy(), gw.cpu().numpy()) < 1e-2
    assert torch.equal(aux["kept"], f.kept)


def test_logprob_entry_matches_forward(cuda_device):
    """icepop_logprob_bf16 (recording lp_train_old, scheduler.py:296-311) == forward lp."""
    from paper_2510_18855_b200 import _lib
    from paper_2510_18855_b200.loss import IcePopConfig, icepop_fwd

    c = _case(seed=4)
    H, W = c["H"].to(cuda_device), c["W"].to(cuda_device)
    f = icepop_fwd(H, W, _batch(c, cuda_device), IcePopConfig())
    lib = _lib.ensure_device(0)
    N = H.shape[0]
    shape = _lib.Shape(n_tokens=N, token_offset=0, hidden=H.shape[1], vocab=W.shape[0], n_seqs=1, n_groups=1,
                       weight_layout=_lib.W_VD)
    fb = _lib._sz()
    _lib.check(lib.icepop_workspace_bytes(shape, 0, 0, fb, None))
    ws = torch.empty(fb.value, dtype=torch.uint8, device=cuda_device)
    lp = torch.empty(N, dtype=torch.float64, device=cuda_device)
    lse = torch.empty(N, dtype=torch.float32, device=cuda_device)
    ent = torch.empty(N, dtype=torch.float32, device=cuda_device)
    tok = torch.from_numpy(c["tokens"]).to(cuda_device)
    _lib.check(lib.icepop_logprob_bf16(shape, 1.0, H.data_ptr(), W.data_ptr(), tok.data_ptr(), lse.data_ptr(),
                                       lp.data_ptr(), ent.data_ptr(), ws.data_ptr(), ws.numel(),
                                       torch.cuda.current_stream().cuda_stream))
    torch.cuda.synchronize()
    assert torch.equal(lp, f.lp_cur) and torch.equal(lse, f.lse) and torch.equal(ent, f.entropy)


def test_long_cot_ragged_high_mask_rate(cuda_device):
    """C4-shaped (scaled): ragged lognormal lengths, ~5% popped tokens."""
    from paper_2510_18855_b200.loss import Diagnostics, IcePopConfig, finish, icepop_bwd, icepop_fwd

    rng = np.random.default_rng(42)
    lens = list(np.clip(rng.lognormal(np.log(600), 0.6, 8), 64, 2048).astype(int))
    c = _case(n_seqs=8, d=256, V=2048, seed=21, lens=lens, group=4, sigma=0.42)
    H, W = c["H"].to(cuda_device), c["W"].to(cuda_device)
    f = icepop_fwd(H, W, _batch(c, cuda_device), IcePopConfig())
    _, gw = icepop_bwd(H, W, _batch(c, cuda_device), f, IcePopConfig(), need_hidden=False)
    finish(f.stats)
    o = _oracle(c)
    d = Diagnostics.from_stats(f.stats.cpu())
    assert np.array_equal(f.kept.cpu().numpy().astype(bool), o["kept"])
    assert 0.02 < d.clipped_fraction < 0.10
    assert d.objective_value == pytest.approx(o["objective"], rel=1e-3)
    assert _rel(gw.cpu().numpy(), o["grad_weight"]) < 1e-2


@pytest.mark.parametrize("layout", ["vd", "dv"])
def test_skip_inactive_rows_matches_full_backward(cuda_device, cta_group, layout):
    """Zero-coefficient rows (zero-advantage sequences, popped and clip-inactive tokens) are
    compacted away in the backward; dHidden must be identical and dW equal up to fp32 order."""
    from paper_2510_18855_b200 import _lib
    from paper_2510_18855_b200.loss import IcePopConfig, icepop_bwd, icepop_fwd

    c = _case(n_seqs=8, seed=13, group=2, layout=layout, lens=[300, 170, 260, 90, 410, 333, 129, 257])
    c["adv"] = c["adv"].copy()
    c["adv"][[0, 1, 4, 5]] = 0.0  # two zero-variance groups
    H, W = c["H"].to(cuda_device), c["W"].to(cuda_device)
    cfg = IcePopConfig()
    b = _batch(c, cuda_device)
    f = icepop_fwd(H, W, b, cfg, layout=layout, store_probs=False)  # row skipping is a recompute-mode feature
    n_zero = int((f.coeff == 0).sum())
    assert n_zero > len(c["tokens"]) // 3
    lib = _lib.ensure_device(0)
    res = {}
    try:
        for skip in (0, 1):
            _lib.check(lib.icepop_set_skip_inactive(skip))
            res[skip] = icepop_bwd(H, W, b, f, cfg, layout=layout, grad_hidden_dtype=torch.float32)
    finally:
        _lib.check(lib.icepop_set_skip_inactive(1))
    (gh0, gw0), (gh1, gw1) = res[0], res[1]
    assert torch.equal(gh0, gh1)
    assert torch.all(gh1[f.coeff == 0] == 0)
    assert _rel(gw1.cpu().numpy(), gw0.cpu().numpy()) < 1e-5
    o = _oracle(c)
    assert _rel(gw1.cpu().numpy(), o["grad_weight"]) < 1e-2
    assert _rel(gh1.cpu().numpy(), o["grad_hidden"]) < 1e-2


def test_skip_inactive_all_rows_inactive(cuda_device):
    """Every coefficient zero: gradients are exactly zero (the GEMMs see an empty extent)."""
    from paper_2510_18855_b200.loss import IcePopConfig, icepop_bwd, icepop_fwd

    c = _case(n_seqs=4, seed=17, group=2)
    c["adv"] = np.zeros_like(c["adv"])
    H, W = c["H"].to(cuda_device), c["W"].to(cuda_device)
    f = icepop_fwd(H, W, _batch(c, cuda_device), IcePopConfig())
    gh, gw = icepop_bwd(H, W, _batch(c, cuda_device), f, IcePopConfig())
    assert torch.count_nonzero(gh) == 0 and torch.count_nonzero(gw) == 0


@pytest.mark.parametrize("kl_coeff,store_probs", [(0.0, False), (0.0, True), (0.4, None)],
                         ids=["gamma0-recompute", "gamma0-probs", "gamma0.4"])
@pytest.mark.parametrize("layout", ["vd", "dv"])
def test_kl_to_ref_bf16_vs_oracle(cuda_device, cta_group, layout, kl_coeff, store_probs):
    """KL-to-ref on tensor cores (objective.py:254-263): dual-accumulator GEMMs; the KL
    diagnostic always, its gradient when gamma > 0. With gamma = 0 (train_loop's own call,
    scheduler.py:530-542) the dual forward also stores the probabilities and the backward is
    the stored mode's."""
    from paper_2510_18855_b200.loss import Diagnostics, IcePopConfig, finish, icepop_bwd, icepop_fwd

    c = _case(seed=31, layout=layout, V=1000)
    rng = np.random.default_rng(7)
    Wr = torch.from_numpy(c["W"].double().numpy() + rng.normal(0, 0.05, tuple(c["W"].shape))).to(torch.bfloat16)
    cfg = IcePopConfig(kl_coeff=kl_coeff)
    H, W, Wrd = c["H"].to(cuda_device), c["W"].to(cuda_device), Wr.to(cuda_device)
    b = _batch(c, cuda_device)
    f = icepop_fwd(H, W, b, cfg, layout=layout, weight_ref=Wrd, store_probs=store_probs)
    assert ("probs" in f.extras) == bool(store_probs)
    gh, gw = icepop_bwd(H, W, b, f, cfg, layout=layout, weight_ref=Wrd, grad_hidden_dtype=torch.float32)
    finish(f.stats)
    from oracle.icepop_oracle import icepop_dense

    o = icepop_dense(c["H"].double().numpy(), c["W"].double().numpy(), c["tokens"], c["lp_old"], c["lp_inf"],
                     c["cu"], c["go"], c["adv"], layout=layout, kl_coeff=kl_coeff, weight_ref=Wr.double().numpy())
    d = Diagnostics.from_stats(f.stats.cpu())
    assert np.array_equal(f.kept.cpu().numpy().astype(bool), o["kept"])
    np.testing.assert_allclose(f.kl.cpu().numpy(), o["kl"], atol=2e-3, rtol=2e-2)
    assert d.kl_to_ref == pytest.approx(o["kl_to_ref"], rel=1e-2, abs=1e-4)
    assert d.objective_value == pytest.approx(o["objective"], rel=2e-3, abs=1e-5)
    assert _rel(gw.cpu().numpy(), o["grad_weight"]) < 1e-2
    assert _rel(gh.cpu().numpy(), o["grad_hidden"]) < 1e-2


@pytest.mark.parametrize("layout", ["vd", "dv"])
def test_kl_forward_statistics_identical_with_stored_probs(cuda_device, cta_group, layout):
    """The dual forward's statistics (lse, lp_cur, entropy, kl, mask, coefficients, stats) are
    the same bits whether or not it also stores the probabilities; the stored q and slab
    references match the plain forward's (same q = 2^(u - R) rule)."""
    from paper_2510_18855_b200.loss import IcePopConfig, icepop_fwd

    c = _case(seed=32, layout=layout, V=1000)
    rng = np.random.default_rng(8)
    Wr = torch.from_numpy(c["W"].double().numpy() + rng.normal(0, 0.05, tuple(c["W"].shape))).to(torch.bfloat16)
    H, W, Wrd = c["H"].to(cuda_device), c["W"].to(cuda_device), Wr.to(cuda_device)
    a = icepop_fwd(H, W, _batch(c, cuda_device), IcePopConfig(), layout=layout, weight_ref=Wrd, store_probs=True)
    b = icepop_fwd(H, W, _batch(c, cuda_device), IcePopConfig(), layout=layout, weight_ref=Wrd, store_probs=False)
    p = icepop_fwd(H, W, _batch(c, cuda_device), IcePopConfig(), layout=layout, store_probs=True)
    for name in ("lse", "lp_cur", "entropy", "kept", "calib", "surrogate", "coeff", "stats", "kl", "lse_ref"):
        assert torch.equal(getattr(a, name), getattr(b, name)), name
    nslab = -(-1000 // 64)
    assert torch.equal(a.extras["tile_max"][:, :nslab], p.extras["tile_max"][:, :nslab])
    qa, qp = a.extras["probs"].float(), p.extras["probs"].float()
    assert torch.allclose(qa, qp, rtol=2.0 ** -7, atol=1e-30)  # at most one bf16 step apart (exp2 rounding)


def test_on_policy_forward_equals_full_forward(cuda_device):
    """theta == theta_old with lp_train_old recorded by icepop_logprob: the GEMM-free
    forward is bit-identical to the full forward (r == 1 exactly), and so is the backward."""
    from paper_2510_18855_b200.loss import (IcePopConfig, PackedBatch, icepop_bwd, icepop_fwd, icepop_fwd_onpolicy,
                                            icepop_logprob)

    c = _case(seed=23)
    H, W = c["H"].to(cuda_device), c["W"].to(cuda_device)
    tok = torch.from_numpy(c["tokens"]).to(cuda_device)
    lp, lse, ent = icepop_logprob(H, W, tok)
    b = _batch(c, cuda_device)
    b = PackedBatch(b.tokens, lp, lp - torch.from_numpy(np.random.default_rng(0).normal(0, 0.3, len(c["tokens"]))).to(
        cuda_device), b.cu_seqlens, b.group_offsets, b.advantages)
    cfg = IcePopConfig()
    full = icepop_fwd(H, W, b, cfg, store_probs=False)  # both backwards recompute -> bit-identical
    onp = icepop_fwd_onpolicy(b, lse, ent, cfg, hidden_dim=H.shape[1], vocab=W.shape[0])
    for name in ("lse", "lp_cur", "entropy", "kept", "calib", "surrogate", "coeff", "stats"):
        assert torch.equal(getattr(full, name), getattr(onp, name)), name
    gh1, gw1 = icepop_bwd(H, W, b, full, cfg)
    gh2, gw2 = icepop_bwd(H, W, b, onp, cfg)
    assert torch.equal(gh1, gh2) and torch.equal(gw1, gw2)


@pytest.mark.parametrize("layout", ["vd", "dv"])
def test_discrepancy_probe_kl(cuda_device, cta_group, layout):
    """delta = mean KL(pi_p || pi_q) over probe rows (discrepancy.py:132-141) vs fp64 numpy."""
    from paper_2510_18855_b200.loss import discrepancy

    rng = np.random.default_rng(5)
    n, d, V = 300, 256, 1000
    H = torch.from_numpy(rng.normal(0, 1, (n, d))).to(torch.bfloat16)
    shp = (V, d) if layout == "vd" else (d, V)
    Wq = torch.from_numpy(rng.normal(0, 2 / np.sqrt(d), shp)).to(torch.bfloat16)
    Wp = torch.from_numpy(Wq.double().numpy() + rng.normal(0, 0.1, shp)).to(torch.bfloat16)
    mean, kl = discrepancy(H.to(cuda_device), Wp.to(cuda_device), Wq.to(cuda_device), layout=layout, temperature=0.9)

    def logp(W):
        z = H.double().numpy() @ (W.double().numpy().T if layout == "vd" else W.double().numpy()) / 0.9
        z = z - z.max(1, keepdims=True)
        return z - np.log(np.exp(z).sum(1, keepdims=True))

    lp, lq = logp(Wp), logp(Wq)
    ref = (np.exp(lp) * (lp - lq)).sum(1)
    np.testing.assert_allclose(kl.cpu().numpy(), ref, atol=2e-3, rtol=2e-2)
    assert mean.item() == pytest.approx(ref.mean(), rel=1e-2)


def test_sgd_update_on_device(cuda_device):
    """objective.py:301-326: ascent, momentum, version semantics left to the caller; errors."""
    from paper_2510_18855_b200.errors import NumericError
    from paper_2510_18855_b200.optim import sgd_update_

    g = torch.Generator(device="cpu").manual_seed(0)
    w0 = torch.randn(1000, 37, generator=g)
    gr = torch.randn(1000, 37, generator=g)
    w = w0.clone().to(cuda_device)
    v = torch.zeros_like(w)
    wb = torch.empty_like(w, dtype=torch.bfloat16)
    sgd_update_(w, gr.to(cuda_device), 0.1, v, 0.5, wb)
    sgd_update_(w, gr.to(cuda_device), 0.1, v, 0.5, wb)
    ref = w0 + 0.1 * gr + 0.1 * 1.5 * gr
    torch.testing.assert_close(w.cpu(), ref, rtol=1e-6, atol=1e-6)
    torch.testing.assert_close(v.cpu(), 1.5 * gr, rtol=1e-6, atol=1e-6)
    assert torch.equal(wb, w.to(torch.bfloat16))
    w2 = w0.clone().to(cuda_device)
    sgd_update_(w2, gr.to(cuda_device), 0.25)
    torch.testing.assert_close(w2.cpu(), w0 + 0.25 * gr, rtol=1e-6, atol=1e-6)
    with pytest.raises(ValueError):
        sgd_update_(w2, gr.to(cuda_device), 0.0)
    with pytest.raises(ValueError):
        sgd_update_(w2, gr.to(cuda_device), 0.1, torch.zeros_like(w2), 1.0)
    with pytest.raises(NumericError):
        sgd_update_(w2, torch.full_like(w2, 3e38), 10.0)


@pytest.mark.parametrize("store_probs", [True, False], ids=["probs", "recompute"])
def test_cuda_graph_capture_replays_fwd_bwd(cuda_device, store_probs):
    """fwd + bwd are sync-free (device-side extents, counters, error word), so one CUDA graph
    captures the whole step; replays match eager execution bit for bit."""
    from paper_2510_18855_b200.loss import IcePopConfig, icepop_bwd, icepop_fwd

    c = _case(seed=41)
    H, W = c["H"].to(cuda_device), c["W"].to(cuda_device)
    b = _batch(c, cuda_device)
    cfg = IcePopConfig()
    f0 = icepop_fwd(H, W, b, cfg, store_probs=store_probs)
    gh0, gw0 = icepop_bwd(H, W, b, f0, cfg)
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s):  # warm-up on the capture stream (allocator, lazy init)
        f = icepop_fwd(H, W, b, cfg, store_probs=store_probs)
        icepop_bwd(H, W, b, f, cfg)
    torch.cuda.current_stream().wait_stream(s)
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        fg = icepop_fwd(H, W, b, cfg, store_probs=store_probs)
        ghg, gwg = icepop_bwd(H, W, b, fg, cfg)
    for _ in range(2):
        g.replay()
        torch.cuda.synchronize()
        assert torch.equal(fg.stats, f0.stats) and torch.equal(fg.kept, f0.kept)
        assert torch.equal(ghg, gh0) and torch.equal(gwg, gw0)


@pytest.mark.parametrize("layout", ["vd", "dv"])
@pytest.mark.parametrize("world,chunked", [(1, False), (3, False), (3, True), (4, True)])
def test_fused_reduce_scatter_emulated_ranks(cuda_device, monkeypatch, layout, world, chunked):
    """K5 epilogue stores each dW row into its owner's slot (the NVLink path), emulated with
    `world` token-shard ranks run one after another on one GPU against slot buffers in device
    memory (no kernel waits on another); the owners' ordered folds reassemble dW exactly as
    the single-rank backward computes it."""
    import paper_2510_18855_b200.loss as L
    from paper_2510_18855_b200 import _lib
    from paper_2510_18855_b200.distributed import shard_range

    c = _case(n_seqs=6, seed=47, layout=layout, lens=[300, 170, 260, 90, 410, 333])
    c["adv"] = c["adv"].copy()
    c["adv"][[2, 3]] = 0.0  # exercise row skipping inside the ranks
    H, W = c["H"].to(cuda_device), c["W"].to(cuda_device)
    cfg = L.IcePopConfig()
    full_b = _batch(c, cuda_device)
    sp = not chunked  # dZ chunks exist only in recompute mode
    f = L.icepop_fwd(H, W, full_b, cfg, layout=layout, store_probs=sp)
    _, gw_ref = L.icepop_bwd(H, W, full_b, f, cfg, layout=layout, need_hidden=False)
    rows, row_len = W.shape  # dW has the weight's layout: rows = V (vd) or d (dv)
    V = W.shape[0] if layout == "vd" else W.shape[1]
    shard_rows = -(-rows // world)
    while (shard_rows * row_len) % 4:  # the fold works on float4
        shard_rows += 1
    slot_bufs = [torch.full((world * shard_rows * row_len,), float("nan"), device=cuda_device) for _ in range(world)]
    if chunked:
        monkeypatch.setattr(L, "DZ_CHUNK_BYTES", 256 * (V + H.shape[1]) * 2)  # 256-row dZ chunks -> local scratch
    N = len(c["tokens"])
    for r in range(world):
        s, e = shard_range(N, world, r)
        b = _batch(c, cuda_device, slice(s, e))
        fr = L.icepop_fwd(H[s:e], W, b, cfg, layout=layout, store_probs=sp)
        t = _lib.RsTarget(world=world, rank=r, shard_rows=shard_rows)
        for o in range(world):
            t.slots[o] = slot_bufs[o].data_ptr()
        L.icepop_bwd_reduce_scatter(H[s:e], W, b, fr, t, cfg, layout=layout, need_hidden=False)
    lib = _lib.ensure_device(0)
    shards = []
    for o in range(world):
        out = torch.empty(shard_rows * row_len, device=cuda_device)
        _lib.check(lib.icepop_rs_fold(slot_bufs[o].data_ptr(), world, shard_rows * row_len, out.data_ptr(),
                                      torch.cuda.current_stream().cuda_stream))
        shards.append(out.view(shard_rows, row_len))
    gw = torch.cat(shards)[:rows]
    torch.cuda.synchronize()
    assert torch.isfinite(gw).all()
    assert _rel(gw.cpu().numpy(), gw_ref.cpu().numpy()) < 1e-5


@pytest.mark.parametrize("run", [1, 3, 16])
@pytest.mark.parametrize("layout", ["vd", "dv"])
def test_k1_runs_merge_statistics(cuda_device, cta_group, layout, run):
    """K1 runs (icepop_set_k1_run): a CTA pair merges the softmax statistics of `run`
    consecutive vocabulary tiles in registers and writes one partial per run. The forward's
    per-token outputs agree with single-tile partials to fp32 rounding and with the oracle;
    the stored probabilities are the same bits."""
    from paper_2510_18855_b200 import _lib
    from paper_2510_18855_b200.loss import IcePopConfig, icepop_fwd

    lib = _lib.ensure_device(0)
    c = _case(seed=33, layout=layout, V=4096 + 40, d=256, n_seqs=6, lens=[700, 650, 300, 900, 128, 500])
    H, W = c["H"].to(cuda_device), c["W"].to(cuda_device)
    try:
        _lib.check(lib.icepop_set_k1_run(1))
        a = icepop_fwd(H, W, _batch(c, cuda_device), IcePopConfig(), layout=layout, store_probs=True)
        _lib.check(lib.icepop_set_k1_run(run))
        b = icepop_fwd(H, W, _batch(c, cuda_device), IcePopConfig(), layout=layout, store_probs=True)
    finally:
        _lib.check(lib.icepop_set_k1_run(0))
    assert torch.equal(a.extras["probs"], b.extras["probs"]) and torch.equal(a.extras["tile_max"], b.extras["tile_max"])
    assert torch.equal(a.kept, b.kept)
    torch.testing.assert_close(a.lse, b.lse, rtol=2e-6, atol=2e-6)
    torch.testing.assert_close(a.entropy, b.entropy, rtol=1e-5, atol=1e-5)
    torch.testing.assert_close(a.lp_cur, b.lp_cur, rtol=0, atol=3e-5)
    o = _oracle(c)
    np.testing.assert_allclose(b.lp_cur.cpu().numpy(), o["lp_cur"], atol=2e-3, rtol=1e-3)
    np.testing.assert_allclose(b.entropy.cpu().numpy(), o["entropy"], atol=2e-3, rtol=1e-3)


@pytest.mark.parametrize("with_ref", [False, True])
def test_epilogue_rerun_equals_full_forward(cuda_device, with_ref):
    """icepop_epilogue re-runs K2 over the K1 partials of a keep_workspace forward with another
    config: the same bits as a full forward with that config (no GEMM)."""
    from paper_2510_18855_b200.loss import IcePopConfig, icepop_epilogue, icepop_fwd

    c = _case(seed=34, V=1000)
    H, W = c["H"].to(cuda_device), c["W"].to(cuda_device)
    Wr = (W.float() + 0.05 * torch.randn_like(W.float())).to(torch.bfloat16) if with_ref else None
    f = icepop_fwd(H, W, _batch(c, cuda_device), IcePopConfig(), weight_ref=Wr, store_probs=False,
                   keep_workspace=True)
    for cfg in (IcePopConfig(alpha=0.8, beta=1.25), IcePopConfig(algo="tis", tis_cap=1.5, clip_eps=0.1)):
        e = icepop_epilogue(_batch(c, cuda_device), f, cfg)
        g = icepop_fwd(H, W, _batch(c, cuda_device), cfg, weight_ref=Wr, store_probs=False)
        for name in ("lse", "lp_cur", "entropy", "kept", "calib", "surrogate", "coeff", "stats"):
            assert torch.equal(getattr(e, name), getattr(g, name)), name
        if with_ref:
            assert torch.equal(e.kl, g.kl)


@pytest.mark.parametrize("kl_coeff", [0.0, 0.3])
def test_custom_op_kl_to_ref_autograd(cuda_device, kl_coeff):
    """icepop_loss with weight_ref: the KL diagnostic (gamma = 0) and its gradient (gamma > 0)
    through the custom ops equal the functional path's -2 dJ (objective.py:254-263)."""
    from paper_2510_18855_b200.loss import IcePopConfig, icepop_bwd, icepop_fwd, icepop_loss

    c = _case(seed=35, V=1000)
    rng = np.random.default_rng(9)
    Wr = torch.from_numpy(c["W"].double().numpy() + rng.normal(0, 0.05, tuple(c["W"].shape))).to(torch.bfloat16)
    Wr = Wr.to(cuda_device)
    cfg = IcePopConfig(kl_coeff=kl_coeff)
    H = c["H"].to(cuda_device).requires_grad_(True)
    W = c["W"].to(cuda_device).requires_grad_(True)
    b = _batch(c, cuda_device)
    loss, aux = icepop_loss(H, W, b, cfg, weight_ref=Wr)
    (2.0 * loss).backward()
    f = icepop_fwd(H.detach(), W.detach(), b, cfg, weight_ref=Wr)
    gh, gw = icepop_bwd(H.detach(), W.detach(), b, f, cfg, grad_scale=-2.0, weight_ref=Wr,
                        grad_hidden_dtype=torch.float32)
    assert loss.item() == pytest.approx(-f.stats[0].item(), rel=1e-12)
    assert torch.equal(aux["kl"], f.kl)
    assert _rel(H.grad.float().cpu().numpy(), gh.cpu().numpy()) < 1e-2
    assert _rel(W.grad.float().cpu().numpy(), gw.cpu().numpy()) < 1e-2


@pytest.mark.parametrize("store_probs", [True, False])
def test_custom_ops_pass_opcheck(cuda_device, store_probs):
    """torch.library.opcheck: the ops' schemas (the backward's declared write to the stored
    probabilities), fake-tensor shapes and autograd registration are consistent."""
    from paper_2510_18855_b200 import _lib
    from paper_2510_18855_b200.loss import _icepop_loss_backward_op, _icepop_loss_op

    c = _case(seed=36, V=512, d=128, n_seqs=3, lens=[100, 60, 90])
    H, W = c["H"].to(cuda_device), c["W"].to(cuda_device)
    b = _batch(c, cuda_device)
    args = (H, W, None, b.tokens, b.lp_train_old, b.lp_infer_old, b.cu_seqlens, b.group_offsets, b.advantages,
            0.5, 5.0, 0.2, 2.0, 1.0, 0.0, 0, _lib.W_VD, 0, store_probs)
    torch.library.opcheck(_icepop_loss_op, args, test_utils=("test_schema", "test_faketensor"))
    out = _icepop_loss_op(*args)
    (_, _, lse, lp_cur, _, _, coeff, kl, lse_ref, kl_w, probs, tile_max) = out
    bargs = (torch.ones((), dtype=torch.float64, device=cuda_device), H, W, None, b.tokens, b.lp_train_old,
             b.lp_infer_old, b.cu_seqlens, b.group_offsets, b.advantages, lse, lp_cur, coeff, kl, lse_ref, kl_w,
             probs, tile_max, 0.5, 5.0, 0.2, 2.0, 1.0, 0.0, 0, _lib.W_VD, 0, True, True)
    torch.library.opcheck(_icepop_loss_backward_op, bargs, test_utils=("test_schema", "test_faketensor"))


@pytest.mark.parametrize("mode", ["probs", "recompute", "ref"])
def test_out_of_range_tokens_raise_without_faulting(cuda_device, mode):
    """A token id outside [0, V) (here -1 and V) is reported as the reference's ValueError by the
    forward's error word; the kernels that index by token (K1's gather, K2's lookup of the
    token's partial, the lp recording) clamp and never read or write out of bounds."""
    from paper_2510_18855_b200.loss import IcePopConfig, finish, icepop_fwd, icepop_logprob

    c = _case(seed=41, V=1000, n_seqs=4, lens=[100, 90, 80, 70])
    c["tokens"][5] = -1
    c["tokens"][200] = 1000
    H, W = c["H"].to(cuda_device), c["W"].to(cuda_device)
    Wr = W if mode == "ref" else None
    f = icepop_fwd(H, W, _batch(c, cuda_device), IcePopConfig(), weight_ref=Wr, store_probs=(mode == "probs"))
    with pytest.raises(ValueError, match="outside the vocabulary"):
        finish(f.stats)
    lp, lse, _ = icepop_logprob(H, W, torch.from_numpy(c["tokens"]).to(cuda_device))
    torch.cuda.synchronize()  # a fault would surface here
    ok = np.ones(len(c["tokens"]), bool)
    ok[[5, 200]] = False
    assert torch.isfinite(lse).all() and np.isfinite(lp.cpu().numpy()[ok]).all()
