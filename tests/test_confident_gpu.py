"""Confident tokens: peaked logits with tokens sampled on-policy, so most sampled tokens have
p_y > 0.9 -- the regime real RL batches live in (SURVEY.md 8d asks for on-policy tokens).

The sampled token's entry of dZ is c (1 - p_y) (objective.py:251-252). The stored-probabilities
backward takes it from p_y = exp(lp_cur) in fp64 as a one-hot term with q_y zeroed; forming it
as c - c q_y 2^(-lse2) from the bf16 q_y would cancel and lose 2^-9 p_y / (1 - p_y) of it.
Checked per ROW of dHidden and per vocabulary entry of dW (a Frobenius norm over the whole
matrix hides a few bad rows), against the fp64 oracle on the same bf16 inputs, in both backward
modes, both weight layouts, with and without exception rows (slab maxima past +-60 in log2
units, whose dZ is formed in place).

Tolerances: the stored-probabilities mode's median and 95th-percentile per-row dH error on
rows with p_y > 0.9, and its median and worst per-entry dW error, are at most twice the
recompute mode's (+1e-4); absolute median per-row dH error <= 5e-3 on ordinary logits.
"""

from __future__ import annotations

import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu


def _peaked_case(seed, N, d, V, layout, sigma_logit, n_seqs=8, group=4):
    rng = np.random.default_rng(seed)
    H = torch.from_numpy(rng.normal(0, 1, (N, d))).to(torch.bfloat16)
    shape_w = (V, d) if layout == "vd" else (d, V)
    W = torch.from_numpy(rng.normal(0, sigma_logit / np.sqrt(d), shape_w)).to(torch.bfloat16)
    Hd, Wd = H.double().numpy(), W.double().numpy()
    z = Hd @ (Wd.T if layout == "vd" else Wd)
    z -= z.max(1, keepdims=True)
    p = np.exp(z)
    p /= p.sum(1, keepdims=True)
    # on-policy: y_t ~ softmax(z_t) (inverse CDF on fp64 probabilities)
    u = rng.random(N)
    tokens = np.minimum((p.cumsum(1) < u[:, None]).sum(1), V - 1).astype(np.int32)
    py = p[np.arange(N), tokens]
    lp = np.log(py)
    lp_old = lp + rng.normal(0, 0.05, N)
    lp_inf = lp_old - rng.normal(0, 0.2, N)
    lens = np.full(n_seqs, N // n_seqs)
    lens[-1] += N - lens.sum()
    cu = np.concatenate([[0], np.cumsum(lens)]).astype(np.int32)
    go = np.arange(0, n_seqs + 1, group).astype(np.int32)
    adv = rng.normal(0, 1, n_seqs)
    return dict(H=H, W=W, tokens=tokens, lp_old=lp_old, lp_inf=lp_inf, cu=cu, go=go, adv=adv, layout=layout,
                py=py)


def _run(c, dev, store_probs):
    from paper_2510_18855_b200.loss import IcePopConfig, PackedBatch, finish, icepop_bwd, icepop_fwd

    b = PackedBatch(torch.from_numpy(c["tokens"]).to(dev), torch.from_numpy(c["lp_old"]).to(dev),
                    torch.from_numpy(c["lp_inf"]).to(dev), torch.from_numpy(c["cu"]).to(dev),
                    torch.from_numpy(c["go"]).to(dev), torch.from_numpy(c["adv"]).to(dev))
    H, W = c["H"].to(dev), c["W"].to(dev)
    f = icepop_fwd(H, W, b, IcePopConfig(), layout=c["layout"], store_probs=store_probs)
    assert ("probs" in f.extras) == store_probs
    gh, gw = icepop_bwd(H, W, b, f, IcePopConfig(), layout=c["layout"], grad_hidden_dtype=torch.float32)
    finish(f.stats)
    return f, gh.double().cpu().numpy(), gw.double().cpu().numpy()


def _row_err(a, b):
    return np.linalg.norm(a - b, axis=1) / np.maximum(np.linalg.norm(b, axis=1), 1e-300)


def _vocab_rows(g, layout):
    return g if layout == "vd" else g.T  # one row per vocabulary entry


def _compare(c, dev):
    from oracle.icepop_oracle import icepop_dense

    o = icepop_dense(c["H"].double().numpy(), c["W"].double().numpy(), c["tokens"], c["lp_old"], c["lp_inf"],
                     c["cu"], c["go"], c["adv"], layout=c["layout"])
    conf = (c["py"] > 0.9) & (o["coeff"] != 0)
    assert conf.sum() >= 20, "the case must hold confident active tokens"
    gref = _vocab_rows(o["grad_weight"], c["layout"])
    nrm = np.linalg.norm(gref, axis=1)
    live = nrm > 1e-3 * nrm.max()
    res = {}
    for mode in (True, False):
        f, gh, gw = _run(c, dev, mode)
        assert np.array_equal(f.kept.cpu().numpy().astype(bool), o["kept"])
        eh = _row_err(gh, o["grad_hidden"])[conf]
        ew = _row_err(_vocab_rows(gw, c["layout"]), gref)[live]
        res[mode] = dict(h_med=float(np.median(eh)), h_p95=float(np.quantile(eh, 0.95)),
                         w_med=float(np.median(ew)), w_max=float(ew.max()))
    print(f"V={c['W'].numel() // c['H'].shape[1]} {c['layout']}: {int(conf.sum())} confident rows; "
          f"stored {res[True]}, recompute {res[False]}")
    return res


def _assert_stored_close(res):
    sp, rc = res[True], res[False]
    for k in ("h_med", "h_p95", "w_med", "w_max"):
        assert sp[k] <= 2.0 * rc[k] + 1e-4, (k, sp, rc)


@pytest.mark.parametrize("layout", ["vd", "dv"])
def test_confident_tokens_v1000(cuda_device, layout):
    """V = 1,000 (ragged last tile and slab), d = 256, logit std 8: median p_y ~ 0.6, a quarter
    of the tokens above 0.9."""
    c = _peaked_case(seed=71, N=1536, d=256, V=1000, layout=layout, sigma_logit=8.0)
    res = _compare(c, cuda_device)
    _assert_stored_close(res)
    assert res[True]["h_med"] <= 5e-3, res


@pytest.mark.parametrize("layout", ["vd", "dv"])
def test_confident_tokens_full_width_slice(cuda_device, layout):
    """The full Ling-2.0 vocabulary V = 157,184 (C2's width) at d = 256, logit std 10."""
    c = _peaked_case(seed=72, N=512, d=256, V=157184, layout=layout, sigma_logit=10.0)
    res = _compare(c, cuda_device)
    _assert_stored_close(res)
    assert res[True]["h_med"] <= 5e-3, res


def test_confident_tokens_exception_rows(cuda_device):
    """Logit std 16 puts slab maxima past 60 (log2 units) on most rows: their dZ is formed in
    place (k_dz_probs) with the same exact sampled-token entry."""
    c = _peaked_case(seed=73, N=1024, d=256, V=1000, layout="vd", sigma_logit=16.0)
    res = _compare(c, cuda_device)
    _assert_stored_close(res)


def test_stored_backward_requires_lp_cur(cuda_device):
    """The ABI rejects a stored-probabilities backward without saved->lp_cur."""
    from paper_2510_18855_b200 import _lib
    from paper_2510_18855_b200.loss import IcePopConfig, PackedBatch, icepop_fwd

    c = _peaked_case(seed=74, N=256, d=64, V=256, layout="vd", sigma_logit=4.0, n_seqs=4, group=2)
    dev = cuda_device
    b = PackedBatch(torch.from_numpy(c["tokens"]).to(dev), torch.from_numpy(c["lp_old"]).to(dev),
                    torch.from_numpy(c["lp_inf"]).to(dev), torch.from_numpy(c["cu"]).to(dev),
                    torch.from_numpy(c["go"]).to(dev), torch.from_numpy(c["adv"]).to(dev))
    H, W = c["H"].to(dev), c["W"].to(dev)
    f = icepop_fwd(H, W, b, IcePopConfig(), layout="vd", store_probs=True)
    lib = _lib.ensure_device(0)
    shape = _lib.Shape(n_tokens=256, token_offset=0, hidden=64, vocab=256, n_seqs=4, n_groups=2,
                       weight_layout=_lib.W_VD)
    saved = _lib.Saved(tokens=b.tokens.data_ptr(), lse=f.lse.data_ptr(), coeff=f.coeff.data_ptr(),
                       probs=f.extras["probs"].data_ptr(), tile_max=f.extras["tile_max"].data_ptr())
    gw = torch.empty((256, 64), dtype=torch.float32, device=dev)
    rc = lib.icepop_bwd_bf16(shape, IcePopConfig().to_c(), H.data_ptr(), W.data_ptr(), None, saved, 1.0, None, 0,
                             gw.data_ptr(), 0, None, 0, torch.cuda.current_stream().cuda_stream)
    assert rc == _lib.EINVAL and "lp_cur" in _lib.last_error()


def _one_minus_py(c):
    """fp64 1 - p_y = sum_{v != y} p_v of the bf16 inputs (no cancellation)."""
    Hd, Wd = c["H"].double().numpy(), c["W"].double().numpy()
    z = Hd @ (Wd.T if c["layout"] == "vd" else Wd)
    z -= z.max(1, keepdims=True)
    e = np.exp(z)
    rows = np.arange(len(z))
    ey = e[rows, c["tokens"]].copy()
    e[rows, c["tokens"]] = 0.0
    other = e.sum(1)
    return other / (other + ey)


@pytest.mark.parametrize("run", [1, 2, 16])
@pytest.mark.parametrize("case", ["v1000_std16", "full_width_std14"])
def test_confident_lp_keeps_one_minus_py(cuda_device, case, run):
    """lp_cur of a confident token keeps 1 - p_y = -expm1(lp_cur) to fp32 RELATIVE precision:
    K1's slab sums leave the sampled token out and K2 takes lp = log1p(-S_{v != y} / S) (with
    z_y - lse, lse's absolute rounding ~1e-6 would swamp 1 - p_y ~ 1e-6). Checked for the
    forward (K2) and the lp recording (icepop_logprob), at K1 run lengths 1 / 2 / 16 (the
    token's partial is flagged and merged at every level: slab, run, column half, K2), and for
    the KL-to-ref forward (the reference loop's call, gamma = 0; dual-accumulator epilogue), against
    fp64 on the same bf16 inputs, down to 1 - p_y ~ 4e-13. Bound: median relative error of
    1 - p_y <= 2e-5 and 99th percentile <= 2e-4 on rows with p_y > 0.9 (fp32 logits from a bf16
    GEMM; measured 3.4e-6 / 1.9e-5, profiles/r02_confident_lp.log)."""
    from paper_2510_18855_b200 import _lib
    from paper_2510_18855_b200.loss import IcePopConfig, PackedBatch, icepop_fwd, icepop_logprob

    if case == "v1000_std16":
        c = _peaked_case(seed=75, N=1024, d=256, V=1000, layout="vd", sigma_logit=16.0)
    else:
        c = _peaked_case(seed=76, N=512, d=256, V=157184, layout="dv", sigma_logit=14.0)
    q = _one_minus_py(c)
    conf = c["py"] > 0.9
    assert conf.sum() >= 50 and (q[conf] < 1e-4).sum() >= 5, "needs confident rows, some with 1 - p_y < 1e-4"
    dev = cuda_device
    b = PackedBatch(torch.from_numpy(c["tokens"]).to(dev), torch.from_numpy(c["lp_old"]).to(dev),
                    torch.from_numpy(c["lp_inf"]).to(dev), torch.from_numpy(c["cu"]).to(dev),
                    torch.from_numpy(c["go"]).to(dev), torch.from_numpy(c["adv"]).to(dev))
    H, W = c["H"].to(dev), c["W"].to(dev)
    lib = _lib.ensure_device(0)
    try:
        _lib.check(lib.icepop_set_k1_run(run))
        f = icepop_fwd(H, W, b, IcePopConfig(), layout=c["layout"], store_probs=False)
        lp_rec, _, _ = icepop_logprob(H, W, b.tokens, layout=c["layout"])
    finally:
        _lib.check(lib.icepop_set_k1_run(0))
    # the reference loop's own call (ref passed, gamma = 0): the dual-accumulator epilogue
    W_ref = (W.float() * 1.01).to(torch.bfloat16)
    fr = icepop_fwd(H, W, b, IcePopConfig(), layout=c["layout"], weight_ref=W_ref, store_probs=False)
    for name, lp in (("forward", f.lp_cur), ("recording", lp_rec), ("forward with ref", fr.lp_cur)):
        g = -np.expm1(lp.cpu().numpy())
        rel = np.abs(g - q)[conf] / q[conf]
        med, p99 = float(np.median(rel)), float(np.quantile(rel, 0.99))
        print(f"{case} run={run} {name}: {int(conf.sum())} confident rows, min 1-p_y {q[conf].min():.2e}, "
              f"rel err of 1-p_y median {med:.2e} p99 {p99:.2e}")
        assert med <= 2e-5 and p99 <= 2e-4, (name, med, p99)


def test_confident_tokens_with_kl_gradient(cuda_device):
    """The KL-to-ref gradient (gamma > 0: the recompute backward K3r, objective.py:254-263) on
    peaked on-policy logits: the sampled token's IcePop entry comes from lp_cur (dz_entry), so
    the per-row dH error on confident rows has a bf16-level median (<= 5e-3) against fp64. Its
    tail is set by the KL term itself: -(w gamma / T) p_y (log p_y - log p_ref,y - kl) is a
    difference of nearly equal log-probabilities, and with fp32 logits from the GEMM (absolute
    error ~1e-5) the rows whose difference is ~1e-4 keep only a few % of it (measured p95 7.5%,
    the dW Frobenius error 1.6e-3); an fp64 GEMM would be needed to do better."""
    from oracle.icepop_oracle import icepop_dense
    from paper_2510_18855_b200.loss import IcePopConfig, PackedBatch, finish, icepop_bwd, icepop_fwd

    c = _peaked_case(seed=77, N=1024, d=256, V=1000, layout="vd", sigma_logit=12.0)
    rng = np.random.default_rng(78)
    W_ref = (c["W"].float() + torch.from_numpy(rng.normal(0, 0.02, tuple(c["W"].shape))).float()).to(torch.bfloat16)
    dev = cuda_device
    b = PackedBatch(torch.from_numpy(c["tokens"]).to(dev), torch.from_numpy(c["lp_old"]).to(dev),
                    torch.from_numpy(c["lp_inf"]).to(dev), torch.from_numpy(c["cu"]).to(dev),
                    torch.from_numpy(c["go"]).to(dev), torch.from_numpy(c["adv"]).to(dev))
    H, W, Wr = c["H"].to(dev), c["W"].to(dev), W_ref.to(dev)
    cfg = IcePopConfig(kl_coeff=0.4)
    f = icepop_fwd(H, W, b, cfg, layout="vd", weight_ref=Wr)
    gh, gw = icepop_bwd(H, W, b, f, cfg, layout="vd", weight_ref=Wr, grad_hidden_dtype=torch.float32)
    finish(f.stats)
    o = icepop_dense(c["H"].double().numpy(), c["W"].double().numpy(), c["tokens"], c["lp_old"], c["lp_inf"],
                     c["cu"], c["go"], c["adv"], layout="vd", kl_coeff=0.4, weight_ref=W_ref.double().numpy())
    conf = (c["py"] > 0.9) & (o["coeff"] != 0)
    assert conf.sum() >= 20
    eh = _row_err(gh.double().cpu().numpy(), o["grad_hidden"])[conf]
    gref = o["grad_weight"]
    ew = np.linalg.norm(gw.double().cpu().numpy() - gref) / np.linalg.norm(gref)
    print(f"KL gradient, {int(conf.sum())} confident rows: dH median {np.median(eh):.2e} p95 "
          f"{np.quantile(eh, 0.95):.2e}; dW rel {ew:.2e}")
    assert np.median(eh) <= 5e-3 and ew <= 1e-2
