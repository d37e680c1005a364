"""Stored-probabilities mode (include/icepop.h `icepop_fwd_out.probs`): K1 also writes
q = exp(z - slab max) (64-column slabs) as bf16 and the backward forms dZ from it in place instead of
recomputing the logits with the K3 GEMM.

Checked here: the forward statistics are the same bits in both modes; q and the slab maxima
against an fp32 torch reference of the same logits (q within bf16 rounding, 2^-8 relative);
gradients against the recompute mode and the fp64 oracle (relative Frobenius <= 1e-2, the
bf16 path's tolerance); consumption semantics (a second backward recomputes); ABI errors;
and that the clipped TMA stores never write outside [N, V].
"""

from __future__ import annotations

import numpy as np
import pytest
import torch

from test_dense_gpu import _batch, _case, _oracle, _rel

pytestmark = pytest.mark.gpu

FWD_FIELDS = ("lse", "lp_cur", "entropy", "kept", "calib", "surrogate", "coeff", "stats")


@pytest.fixture(params=[1, 2], ids=["cta1", "cta2"])
def cta_group(request):
    from paper_2510_18855_b200 import _lib

    lib = _lib.ensure_device(0)
    _lib.check(lib.icepop_set_cta_group(request.param))
    yield request.param
    _lib.check(lib.icepop_set_cta_group(2))


def _logits(c, dev, temperature=1.0):
    H = c["H"].to(dev).float()
    W = c["W"].to(dev).float()
    return (H @ (W.T if c["layout"] == "vd" else W)) / temperature


@pytest.mark.parametrize("layout", ["vd", "dv"])
def test_forward_statistics_identical_in_both_modes(cuda_device, cta_group, layout):
    from paper_2510_18855_b200.loss import IcePopConfig, icepop_fwd

    c = _case(seed=51, layout=layout, V=1000)
    H, W = c["H"].to(cuda_device), c["W"].to(cuda_device)
    a = icepop_fwd(H, W, _batch(c, cuda_device), IcePopConfig(), layout=layout, store_probs=True)
    b = icepop_fwd(H, W, _batch(c, cuda_device), IcePopConfig(), layout=layout, store_probs=False)
    assert "probs" in a.extras and "probs" not in b.extras
    for name in FWD_FIELDS:
        assert torch.equal(getattr(a, name), getattr(b, name)), name


@pytest.mark.parametrize("temperature", [1.0, 0.7])
@pytest.mark.parametrize("layout", ["vd", "dv"])
def test_stored_probabilities_match_fp32_softmax(cuda_device, cta_group, layout, temperature):
    """q * 2^(R - lse log2 e) is the softmax (R: the per-slab reference in tile_max); V = 1000
    leaves a ragged last tile and a ragged last 64-column slab, N is not a multiple of 128."""
    from paper_2510_18855_b200 import _lib
    from paper_2510_18855_b200.loss import IcePopConfig, icepop_fwd

    c = _case(seed=52, layout=layout, V=1000)
    f = icepop_fwd(c["H"].to(cuda_device), c["W"].to(cuda_device), _batch(c, cuda_device),
                   IcePopConfig(temperature=temperature), layout=layout, store_probs=True)
    probs, tmax = f.extras["probs"].float(), f.extras["tile_max"]
    N, V = probs.shape
    S = _lib.PROBS_SLAB
    n_slabs = -(-V // S)
    assert N % 128 != 0 and tmax.shape == (N, _lib.tile_max_ld(V)) and tmax.shape[1] >= n_slabs
    tmax = tmax[:, :n_slabs]
    z = _logits(c, cuda_device, temperature)
    u = z * (1.0 / np.log(2.0))
    pad = n_slabs * S - V
    slab_max = torch.nn.functional.pad(u, (0, pad), value=-1e30).view(N, -1, S).amax(-1)
    # slab reference R: 0 while |slab max| <= 60 (log2 units), else the slab maximum
    assert torch.all(tmax == 0) and float(slab_max.abs().max()) < 60
    # q = 2^(u - R) = 2^u here, within bf16 rounding
    torch.testing.assert_close(probs, torch.exp2(u), rtol=8e-3, atol=0)
    scale = torch.exp2(tmax - (f.lse * (1.0 / np.log(2.0)))[:, None])
    p = probs * scale.repeat_interleave(S, dim=1)[:, :V]
    ref = torch.softmax(z, dim=1)
    torch.testing.assert_close(p, ref, rtol=8e-3, atol=1e-6)


@pytest.mark.parametrize("layout", ["vd", "dv"])
@pytest.mark.parametrize("algo", ["icepop", "tis"])
def test_backward_from_probs_matches_recompute_and_oracle(cuda_device, cta_group, layout, algo):
    from paper_2510_18855_b200.loss import IcePopConfig, icepop_bwd, icepop_fwd

    c = _case(seed=53, layout=layout, V=1000)
    c["adv"] = c["adv"].copy()
    c["adv"][[0, 1, 2]] = 0.0  # a zero-advantage group: its rows' dZ must come out exactly 0
    H, W = c["H"].to(cuda_device), c["W"].to(cuda_device)
    cfg = IcePopConfig(algo=algo)
    res = {}
    for sp in (True, False):
        f = icepop_fwd(H, W, _batch(c, cuda_device), cfg, layout=layout, store_probs=sp)
        res[sp] = icepop_bwd(H, W, _batch(c, cuda_device), f, cfg, layout=layout, grad_hidden_dtype=torch.float32)
        assert "probs" not in f.extras  # consumed
    (gh_p, gw_p), (gh_r, gw_r) = res[True], res[False]
    zero = (f.coeff == 0)
    assert int(zero.sum()) > 0 and torch.all(gh_p[zero] == 0)
    assert _rel(gw_p.cpu().numpy(), gw_r.cpu().numpy()) < 5e-3
    assert _rel(gh_p.cpu().numpy(), gh_r.cpu().numpy()) < 5e-3
    o = _oracle(c, algo=algo)
    assert _rel(gw_p.cpu().numpy(), o["grad_weight"]) < 1e-2
    assert _rel(gh_p.cpu().numpy(), o["grad_hidden"]) < 1e-2


def test_second_backward_recomputes(cuda_device):
    """The first backward overwrites the probabilities with dZ; a second one on the same
    forward falls back to the logit recompute and equals a recompute-mode backward exactly."""
    from paper_2510_18855_b200.loss import IcePopConfig, icepop_bwd, icepop_fwd

    c = _case(seed=54)
    H, W = c["H"].to(cuda_device), c["W"].to(cuda_device)
    cfg = IcePopConfig()
    f = icepop_fwd(H, W, _batch(c, cuda_device), cfg, store_probs=True)
    icepop_bwd(H, W, _batch(c, cuda_device), f, cfg)
    gh2, gw2 = icepop_bwd(H, W, _batch(c, cuda_device), f, cfg)
    fr = icepop_fwd(H, W, _batch(c, cuda_device), cfg, store_probs=False)
    gh3, gw3 = icepop_bwd(H, W, _batch(c, cuda_device), fr, cfg)
    assert torch.equal(gh2, gh3) and torch.equal(gw2, gw3)


def test_autograd_retain_graph_second_backward(cuda_device):
    """icepop_loss with stored probabilities: backward twice (retain_graph) gives the same
    gradients within tolerance (the second pass recomputes)."""
    from paper_2510_18855_b200.loss import IcePopConfig, icepop_loss

    c = _case(seed=55)
    H = c["H"].to(cuda_device).requires_grad_(True)
    W = c["W"].to(cuda_device).requires_grad_(True)
    loss, _ = icepop_loss(H, W, _batch(c, cuda_device), IcePopConfig(), store_probs=True)
    loss.backward(retain_graph=True)
    g1 = (H.grad.float().clone(), W.grad.float().clone())
    H.grad = W.grad = None
    loss.backward()
    assert _rel(H.grad.float().cpu().numpy(), g1[0].cpu().numpy()) < 1e-2
    assert _rel(W.grad.float().cpu().numpy(), g1[1].cpu().numpy()) < 1e-2


def test_probs_with_weight_ref_only_without_kl_gradient(cuda_device):
    """weight_ref with gamma > 0 (the KL gradient): the forward keeps the recompute mode even
    when asked; with gamma = 0 (a forward-only diagnostic) it stores the probabilities."""
    from paper_2510_18855_b200.loss import IcePopConfig, icepop_fwd

    c = _case(seed=56, V=1000)
    H, W = c["H"].to(cuda_device), c["W"].to(cuda_device)
    f = icepop_fwd(H, W, _batch(c, cuda_device), IcePopConfig(kl_coeff=0.3), weight_ref=W.clone(), store_probs=True)
    assert "probs" not in f.extras
    f = icepop_fwd(H, W, _batch(c, cuda_device), IcePopConfig(), weight_ref=W.clone(), store_probs=True)
    assert "probs" in f.extras


def _c_fwd(c, dev, probs, tile_max, weight_ref=None, kl_coeff=0.0):
    from paper_2510_18855_b200 import _lib
    from paper_2510_18855_b200.loss import IcePopConfig, _shape

    H, W = c["H"].to(dev), c["W"].to(dev)
    b = _batch(c, dev)
    shape = _shape(H, W, c["layout"], b)
    n = shape.n_tokens
    outs = {k: torch.empty(n, dtype=t, device=dev) for k, t in
            (("lse", torch.float32), ("lp_cur", torch.float64), ("entropy", torch.float32), ("kept", torch.uint8),
             ("calib", torch.float64), ("surrogate", torch.float64), ("coeff", torch.float32))}
    stats = torch.empty(_lib.NSTATS, dtype=torch.float64, device=dev)
    kl = [torch.empty(n, dtype=torch.float32, device=dev) for _ in range(3)] if weight_ref is not None else [None] * 3
    fb = _lib._sz()
    lib = _lib.ensure_device(0)
    _lib.check(lib.icepop_workspace_bytes(shape, 0, 1 if weight_ref is not None else 0, fb, None))
    ws = torch.empty(fb.value, dtype=torch.uint8, device=dev)
    out = _lib.FwdOut(stats=stats.data_ptr(), kl=_lib.ptr(kl[0]), lse_ref=_lib.ptr(kl[1]), kl_w=_lib.ptr(kl[2]),
                      probs=_lib.ptr(probs), tile_max=_lib.ptr(tile_max),
                      **{k: v.data_ptr() for k, v in outs.items()})
    rc = lib.icepop_fwd_bf16(shape, IcePopConfig(kl_coeff=kl_coeff).to_c(), H.data_ptr(), W.data_ptr(), _lib.ptr(weight_ref),
                             b.to_c(), out, ws.data_ptr(), ws.numel(), torch.cuda.current_stream().cuda_stream)
    return rc, shape, b, outs


def test_abi_rejects_invalid_probs_arguments(cuda_device):
    from paper_2510_18855_b200 import _lib
    from paper_2510_18855_b200.loss import IcePopConfig

    lib = _lib.ensure_device(0)
    c = _case(seed=57, V=1000)
    N = len(c["tokens"])
    probs = torch.empty((N, 1000), dtype=torch.bfloat16, device=cuda_device)
    tm = torch.empty((N, _lib.tile_max_ld(1000)), dtype=torch.float32, device=cuda_device)
    rc, *_ = _c_fwd(c, cuda_device, probs, None)
    assert rc == _lib.EINVAL  # tile_max missing
    rc, *_ = _c_fwd(c, cuda_device, probs, tm, weight_ref=c["W"].to(cuda_device), kl_coeff=0.3)
    assert rc == _lib.EINVAL  # no stored probabilities with the KL gradient (gamma > 0)
    flat = torch.empty(N * 1000 + 8, dtype=torch.bfloat16, device=cuda_device)
    rc, *_ = _c_fwd(c, cuda_device, flat[1:1 + N * 1000], tm)
    assert rc == _lib.EINVAL  # probs not 16-byte aligned
    # backward: saved probs with gamma > 0 is rejected
    rc, shape, b, outs = _c_fwd(c, cuda_device, probs, tm)
    assert rc == _lib.OK
    saved = _lib.Saved(tokens=b.tokens.data_ptr(), lse=outs["lse"].data_ptr(), coeff=outs["coeff"].data_ptr(),
                       lse_ref=outs["lse"].data_ptr(), kl=outs["lse"].data_ptr(), kl_w=outs["lse"].data_ptr(),
                       probs=probs.data_ptr(), tile_max=tm.data_ptr())
    H, W = c["H"].to(cuda_device), c["W"].to(cuda_device)
    rc = lib.icepop_bwd_bf16(shape, IcePopConfig(kl_coeff=0.3).to_c(), H.data_ptr(), W.data_ptr(), W.data_ptr(),
                             saved, 1.0, None, 0, None, 0, None, 0, torch.cuda.current_stream().cuda_stream)
    assert rc == _lib.EINVAL


@pytest.mark.parametrize("with_ref", [False, True], ids=["K1", "K1-dual"])
def test_clipped_probability_stores_stay_in_bounds(cuda_device, cta_group, with_ref):
    """The TMA stores of q are clipped to [N, V]: guard bands around the buffer stay intact
    (N = 1,111 rows is not a multiple of 32 or 128; V = 1,000 ends mid 64-column slab), for K1
    and for the dual-accumulator forward (weight_ref with gamma = 0) that also stores them."""
    from paper_2510_18855_b200 import _lib

    c = _case(seed=58, V=1000, lens=[500, 411, 200], n_seqs=3)
    N, V, G = len(c["tokens"]), 1000, 4096
    buf = torch.full((N * V + 2 * G,), 12345.0, dtype=torch.bfloat16, device=cuda_device)
    # 16-byte aligned start G elements in (G * 2 bytes)
    probs = buf[G:G + N * V].view(N, V)
    L = _lib.tile_max_ld(V)
    tm_buf = torch.full((N * L + 2 * 64,), 777.0, dtype=torch.float32, device=cuda_device)
    tm = tm_buf[64:64 + N * L].view(N, L)
    rc, *_ = _c_fwd(c, cuda_device, probs, tm, weight_ref=c["W"].to(cuda_device) if with_ref else None)
    assert rc == _lib.OK
    torch.cuda.synchronize()
    assert torch.all(buf[:G] == 12345.0) and torch.all(buf[G + N * V:] == 12345.0)
    assert torch.all(tm_buf[:64] == 777.0) and torch.all(tm_buf[64 + N * L:] == 777.0)
    assert torch.isfinite(probs.float()).all() and float(probs.float().min()) >= 0.0


@pytest.mark.parametrize("layout", ["vd", "dv"])
def test_long_k_backward_wide_tiles(cuda_device, layout):
    """V >= 16384 (K4 long-K) and N >= 16384 tokens (K5 long-K): the backward GEMMs run on
    256 x 512 tiles; dW and dH equal the 256 x 256 tiles' bit for bit and the recompute-mode
    backward within the bf16 tolerance."""
    from paper_2510_18855_b200 import _lib
    from paper_2510_18855_b200.loss import IcePopConfig, icepop_bwd, icepop_fwd

    lib = _lib.ensure_device(0)
    c = _case(n_seqs=6, d=256, V=16512, seed=61, layout=layout, lens=[3000, 2900, 2800, 2700, 2600, 2640])
    assert len(c["tokens"]) >= 16384
    H, W = c["H"].to(cuda_device), c["W"].to(cuda_device)
    cfg = IcePopConfig()
    res = {}
    try:
        _lib.check(lib.icepop_set_skip_inactive(0))  # keep dZ rows in token order for the reference below
        for wide in (1, 0):
            _lib.check(lib.icepop_set_wide_tiles(2 * wide))  # 2: 512-wide tiles forced
            f = icepop_fwd(H, W, _batch(c, cuda_device), cfg, layout=layout, store_probs=True)
            gh, gw = icepop_bwd(H, W, _batch(c, cuda_device), f, cfg, layout=layout, grad_hidden_dtype=torch.float32)
            res[wide] = (gh, gw)
        fr = icepop_fwd(H, W, _batch(c, cuda_device), cfg, layout=layout, store_probs=False)
        ghr, gwr = icepop_bwd(H, W, _batch(c, cuda_device), fr, cfg, layout=layout, grad_hidden_dtype=torch.float32)
    finally:
        _lib.check(lib.icepop_set_wide_tiles(1))
        _lib.check(lib.icepop_set_skip_inactive(1))
    (gh1, gw1), (gh0, gw0) = res[1], res[0]
    assert torch.equal(gh1, gh0) and torch.equal(gw1, gw0)
    assert _rel(gw1.cpu().numpy(), gwr.cpu().numpy()) < 5e-3
    assert _rel(gh1.cpu().numpy(), ghr.cpu().numpy()) < 5e-3


@pytest.mark.parametrize("layout", ["vd", "dv"])
def test_stored_probs_block_sparse_backward(cuda_device, cta_group, layout):
    """Stored-probabilities backward with block-sparse K4/K5 (two zero-advantage groups +
    scattered popped/clip-inactive tokens): 64-token blocks / 256-token tiles without an
    active row are skipped. They hold only zero dZ rows, so dH and dW equal the dense pass bit
    for bit; both vs the oracle."""
    from paper_2510_18855_b200 import _lib
    from paper_2510_18855_b200.loss import IcePopConfig, icepop_bwd, icepop_fwd

    c = _case(n_seqs=8, seed=71, group=2, layout=layout, V=1000, lens=[300, 170, 260, 90, 410, 333, 129, 257])
    c["adv"] = c["adv"].copy()
    c["adv"][[0, 1, 4, 5]] = 0.0
    H, W = c["H"].to(cuda_device), c["W"].to(cuda_device)
    cfg = IcePopConfig()
    lib = _lib.ensure_device(0)
    res = {}
    try:
        for skip in (0, 1):
            _lib.check(lib.icepop_set_skip_inactive(skip))
            f = icepop_fwd(H, W, _batch(c, cuda_device), cfg, layout=layout, store_probs=True)
            res[skip] = icepop_bwd(H, W, _batch(c, cuda_device), f, cfg, layout=layout,
                                   grad_hidden_dtype=torch.float32)
    finally:
        _lib.check(lib.icepop_set_skip_inactive(1))
    (gh0, gw0), (gh1, gw1) = res[0], res[1]
    assert int((f.coeff == 0).sum()) > len(c["tokens"]) // 3
    assert torch.equal(gh0, gh1)
    assert torch.all(gh1[f.coeff == 0] == 0)
    assert torch.equal(gw1, gw0)
    o = _oracle(c)
    assert _rel(gw1.cpu().numpy(), o["grad_weight"]) < 1e-2
    assert _rel(gh1.cpu().numpy(), o["grad_hidden"]) < 1e-2


def test_stored_probs_compaction_accumulates_into_grad_weight(cuda_device):
    """grad_weight given (accumulate) with compacted rows: adds onto the existing values."""
    from paper_2510_18855_b200.loss import IcePopConfig, icepop_bwd, icepop_fwd

    c = _case(n_seqs=4, seed=72, group=2, V=1000)
    c["adv"] = c["adv"].copy()
    c["adv"][[0, 1]] = 0.0
    H, W = c["H"].to(cuda_device), c["W"].to(cuda_device)
    cfg = IcePopConfig()
    f = icepop_fwd(H, W, _batch(c, cuda_device), cfg, store_probs=True)
    _, gw = icepop_bwd(H, W, _batch(c, cuda_device), f, cfg, need_hidden=False)
    base = torch.full_like(gw, 0.25)
    f2 = icepop_fwd(H, W, _batch(c, cuda_device), cfg, store_probs=True)
    icepop_bwd(H, W, _batch(c, cuda_device), f2, cfg, need_hidden=False, grad_weight=base)
    torch.testing.assert_close(base, gw + 0.25, rtol=0, atol=1e-6)


@pytest.mark.parametrize("layout", ["vd", "dv"])
def test_fwd_bwd_token_chunks_match_whole_batch(cuda_device, layout):
    """icepop_fwd_bwd in token chunks (stored probabilities per chunk, sequences cut mid-way):
    same kept mask, per-token outputs and dH bits as the whole batch; stats and dW within fp
    summation order (error bits OR-ed)."""
    from paper_2510_18855_b200.loss import IcePopConfig, icepop_fwd_bwd

    c = _case(n_seqs=6, seed=81, layout=layout, V=1000, lens=[3000, 2100, 1700, 900, 4000, 2500])
    c["adv"] = c["adv"].copy()
    c["adv"][[0, 1, 2]] = 0.0
    H, W = c["H"].to(cuda_device), c["W"].to(cuda_device)
    cfg = IcePopConfig()
    f1, gh1, gw1 = icepop_fwd_bwd(H, W, _batch(c, cuda_device), cfg, layout, grad_scale=-1.0,
                                  grad_hidden_dtype=torch.float32)
    f2, gh2, gw2 = icepop_fwd_bwd(H, W, _batch(c, cuda_device), cfg, layout, grad_scale=-1.0,
                                  grad_hidden_dtype=torch.float32, max_chunk_tokens=4096)
    assert f2.extras["chunks"] == -(-len(c["tokens"]) // 4096) > 1
    for name in ("lse", "lp_cur", "entropy", "kept", "calib", "surrogate", "coeff"):
        assert torch.equal(getattr(f1, name), getattr(f2, name)), name
    assert torch.equal(gh1, gh2)
    torch.testing.assert_close(f2.stats[:7], f1.stats[:7], rtol=1e-9, atol=1e-12)
    assert f2.stats[7].item() == f1.stats[7].item()
    # dW: per-chunk fp32 partial sums regroup the token sum (measured rel ~1.1e-5)
    assert _rel(gw2.cpu().numpy(), gw1.cpu().numpy()) < 5e-5
    o = _oracle(c)
    assert _rel(-gw2.cpu().numpy(), o["grad_weight"]) < 1e-2


def test_caller_owned_probs_buffers_and_workspace(cuda_device):
    """icepop_fwd(probs_buffers=...) with buffers longer than N and icepop_bwd(workspace=...)
    (how icepop_fwd_bwd reuses one allocation across token chunks) give the same bits as
    the self-allocating calls; malformed buffers are rejected before any launch."""
    from paper_2510_18855_b200 import _lib
    from paper_2510_18855_b200.loss import IcePopConfig, icepop_bwd, icepop_fwd, sp_workspace_bytes

    c = _case(n_seqs=6, seed=93, V=1000)
    H, W = c["H"].to(cuda_device), c["W"].to(cuda_device)
    n, d, V = H.shape[0], H.shape[1], W.shape[0]
    cfg = IcePopConfig()
    f1 = icepop_fwd(H, W, _batch(c, cuda_device), cfg, store_probs=True)
    gh1, gw1 = icepop_bwd(H, W, _batch(c, cuda_device), f1, cfg)
    bufs = (torch.full((n + 100, V), 7.0, dtype=torch.bfloat16, device=cuda_device),
            torch.empty((n + 100, _lib.tile_max_ld(V)), dtype=torch.float32, device=cuda_device))
    ws = torch.empty(sp_workspace_bytes(n, d, V, len(c["cu"]) - 1) + 512, dtype=torch.uint8, device=cuda_device)
    f2 = icepop_fwd(H, W, _batch(c, cuda_device), cfg, probs_buffers=bufs)
    gh2, gw2 = icepop_bwd(H, W, _batch(c, cuda_device), f2, cfg, workspace=ws)
    assert torch.equal(f1.stats, f2.stats) and torch.equal(f1.kept, f2.kept)
    assert torch.equal(gh1, gh2) and torch.equal(gw1, gw2)
    assert torch.all(bufs[0][n:] == 7.0)  # rows past N untouched
    with pytest.raises(ValueError):
        icepop_fwd(H, W, _batch(c, cuda_device), cfg, probs_buffers=(bufs[0][:, :-8], bufs[1]))
    with pytest.raises(ValueError):
        icepop_fwd(H, W, _batch(c, cuda_device), cfg, probs_buffers=(bufs[0][: n - 1], bufs[1]))


@pytest.mark.parametrize("n_tok,d,V,layout", [
    (1, 64, 64, "vd"), (7, 8, 72, "dv"), (63, 24, 136, "vd"), (65, 32, 1000, "dv"), (129, 256, 520, "vd"),
    (300, 40, 2056, "dv"),
])
def test_odd_shapes_all_modes(cuda_device, n_tok, d, V, layout):
    """Edge shapes through the stored-probabilities (block-sparse) and recompute backwards:
    N below one tile / not a multiple of 64, V a multiple of 8 only, tiny d; both vs the oracle."""
    from paper_2510_18855_b200.loss import IcePopConfig, icepop_bwd, icepop_fwd

    lens = [max(1, n_tok // 2), n_tok - max(1, n_tok // 2)] if n_tok > 1 else [1]
    lens = [x for x in lens if x > 0]
    c = _case(n_seqs=len(lens), d=d, V=V, seed=90 + n_tok, layout=layout, lens=lens, group=len(lens))
    H, W = c["H"].to(cuda_device), c["W"].to(cuda_device)
    cfg = IcePopConfig(algo="tis")  # no popped tokens: a 1-token batch still has a gradient
    res = {}
    for sp in (True, False):
        f = icepop_fwd(H, W, _batch(c, cuda_device), cfg, layout=layout, store_probs=sp)
        res[sp] = (f, *icepop_bwd(H, W, _batch(c, cuda_device), f, cfg, layout=layout,
                                  grad_hidden_dtype=torch.float32))
    o = _oracle(c, algo="tis")
    for sp, (f, gh, gw) in res.items():
        assert np.array_equal(f.kept.cpu().numpy().astype(bool), o["kept"])
        np.testing.assert_allclose(f.lp_cur.cpu().numpy(), o["lp_cur"], atol=2e-3, rtol=1e-3)
        if np.linalg.norm(o["grad_weight"]) > 0:
            assert _rel(gw.cpu().numpy(), o["grad_weight"]) < 1e-2, sp
            assert _rel(gh.cpu().numpy(), o["grad_hidden"]) < 1e-2, sp



@pytest.mark.parametrize("kind", ["large", "shifted"])
@pytest.mark.parametrize("layout", ["vd", "dv"])
def test_exception_rows_out_of_reference_range(cuda_device, layout, kind):
    """Rows whose logits leave the +-60 (log2) range of the stored-probabilities reference:
    "large" = logits of std ~40 (slab maxima beyond +60), "shifted" = every logit of half the
    rows moved by -100 through a constant feature (maxima below -60). Those rows take the dZ
    pass in place, the others the row-scaled GEMMs; both vs the recompute mode and the oracle."""
    from paper_2510_18855_b200.loss import IcePopConfig, icepop_bwd, icepop_fwd

    c = _case(n_seqs=4, d=64, V=1000, seed=95, layout=layout, lens=[120, 90, 150, 70], group=2)
    Hn, Wn = c["H"].double().numpy().copy(), c["W"].double().numpy().copy()
    if kind == "large":
        Wn *= 20.0
    else:
        Hn[:, 0] = 0.0
        Hn[: len(Hn) // 2, 0] = 1.0
        if layout == "vd":
            Wn[:, 0] = -100.0
        else:
            Wn[0, :] = -100.0
    c["H"], c["W"] = torch.from_numpy(Hn).to(torch.bfloat16), torch.from_numpy(Wn).to(torch.bfloat16)
    # lp_old near the new model's own log-probs so the ratios stay in range
    from oracle.icepop_oracle import icepop_dense

    o0 = icepop_dense(c["H"].double().numpy(), c["W"].double().numpy(), c["tokens"], c["lp_old"], c["lp_old"],
                      c["cu"], c["go"], c["adv"], layout=layout)
    rng = np.random.default_rng(3)
    c["lp_old"] = o0["lp_cur"] + rng.normal(0, 0.1, len(c["tokens"]))
    c["lp_inf"] = c["lp_old"] - rng.normal(0, 0.2, len(c["tokens"]))
    H, W = c["H"].to(cuda_device), c["W"].to(cuda_device)
    cfg = IcePopConfig()
    f = icepop_fwd(H, W, _batch(c, cuda_device), cfg, layout=layout, store_probs=True)
    assert bool((f.extras["tile_max"] != 0).any())  # some slabs carry their own reference
    gh, gw = icepop_bwd(H, W, _batch(c, cuda_device), f, cfg, layout=layout, grad_hidden_dtype=torch.float32)
    fr = icepop_fwd(H, W, _batch(c, cuda_device), cfg, layout=layout, store_probs=False)
    ghr, gwr = icepop_bwd(H, W, _batch(c, cuda_device), fr, cfg, layout=layout, grad_hidden_dtype=torch.float32)
    assert torch.isfinite(gw).all() and torch.isfinite(gh).all()
    # "shifted": dH along the constant feature is -100 * sum_v dZ[t, v], exactly 0 -- pure
    # cancellation noise in any bf16 mode (the recompute mode's included), so compare the rest
    cols = slice(1, None) if kind == "shifted" else slice(None)
    assert _rel(gw.cpu().numpy(), gwr.cpu().numpy()) < 5e-3
    assert _rel(gh[:, cols].cpu().numpy(), ghr[:, cols].cpu().numpy()) < 5e-3
    o = _oracle(c)
    assert np.array_equal(f.kept.cpu().numpy().astype(bool), o["kept"])
    assert _rel(gw.cpu().numpy(), o["grad_weight"]) < 1e-2
    assert _rel(gh[:, cols].cpu().numpy(), o["grad_hidden"][:, cols]) < 1e-2


@pytest.mark.parametrize("pattern", ["all_same", "last_column", "few_ids"])
@pytest.mark.parametrize("layout", ["vd", "dv"])
def test_onehot_scatter_token_patterns(cuda_device, layout, pattern):
    """The row-scaled backward's one-hot scatter (dW[y] += c H[t], tokens radix-sorted by id)
    and K4's W[y] gather under skewed token streams: one id for every token (a single run of
    N), ids in the last (ragged) vocab slab, a handful of ids. Same gradients as the
    recompute mode; repeated runs bit-identical."""
    from paper_2510_18855_b200.loss import IcePopConfig, icepop_bwd, icepop_fwd

    V = 1000
    c = _case(n_seqs=4, d=96, V=V, seed=97, layout=layout, lens=[400, 300, 350, 250], group=2)
    N = len(c["tokens"])
    rng = np.random.default_rng(5)
    if pattern == "all_same":
        c["tokens"] = np.full(N, 17, dtype=np.int32)
    elif pattern == "last_column":
        c["tokens"] = rng.integers(V - 40, V, N).astype(np.int32)
    else:
        c["tokens"] = rng.choice(np.array([0, 5, 999, 500], dtype=np.int32), N)
    H, W = c["H"].to(cuda_device), c["W"].to(cuda_device)
    cfg = IcePopConfig(algo="tis")
    out = []
    for sp in (True, True, False):
        f = icepop_fwd(H, W, _batch(c, cuda_device), cfg, layout=layout, store_probs=sp)
        out.append(icepop_bwd(H, W, _batch(c, cuda_device), f, cfg, layout=layout, grad_hidden_dtype=torch.float32))
    (gh1, gw1), (gh2, gw2), (ghr, gwr) = out
    assert torch.equal(gh1, gh2) and torch.equal(gw1, gw2)
    assert _rel(gw1.cpu().numpy(), gwr.cpu().numpy()) < 5e-3
    assert _rel(gh1.cpu().numpy(), ghr.cpu().numpy()) < 5e-3


@pytest.mark.parametrize("V,layout", [(1000, "vd"), (520, "dv"), (2048, "vd")])
def test_k1_wide_tile_matches_default(cuda_device, V, layout):
    """K1 on 256x512 tiles (icepop_set_k1_wide(1): one accumulator released in halves, columns
    of a tile interleaved across the CTA pair) against the default 256x256 tiles: the same
    logits per element, so the stored probabilities and slab references are the same bits and
    the kept mask is identical; the statistics differ only by the partial grouping. V = 520
    leaves a wide tile whose second half lies past V (slab references beyond tile_max_ld)."""
    from paper_2510_18855_b200 import _lib
    from paper_2510_18855_b200.loss import IcePopConfig, icepop_bwd, icepop_fwd

    c = _case(seed=97, layout=layout, V=V)
    H, W = c["H"].to(cuda_device), c["W"].to(cuda_device)
    cfg = IcePopConfig()
    lib = _lib.ensure_device(0)
    res = {}
    try:
        for wide in (0, 1):
            _lib.check(lib.icepop_set_k1_wide(wide))
            f = icepop_fwd(H, W, _batch(c, cuda_device), cfg, layout=layout, store_probs=True)
            probs, tmax = f.extras["probs"].clone(), f.extras["tile_max"].clone()
            gh, gw = icepop_bwd(H, W, _batch(c, cuda_device), f, cfg, layout=layout, grad_hidden_dtype=torch.float32)
            res[wide] = (f, probs, tmax, gh, gw)
    finally:
        _lib.check(lib.icepop_set_k1_wide(0))
    (f0, p0, t0, gh0, gw0), (f1, p1, t1, gh1, gw1) = res[0], res[1]
    n_slabs = -(-V // _lib.PROBS_SLAB)
    assert torch.equal(p0, p1)
    assert torch.equal(t0[:, :n_slabs], t1[:, :n_slabs])
    assert torch.equal(f0.kept, f1.kept)
    torch.testing.assert_close(f1.lse, f0.lse, rtol=1e-6, atol=1e-6)
    torch.testing.assert_close(f1.lp_cur, f0.lp_cur, rtol=0, atol=1e-5)
    assert _rel(gw1.cpu().numpy(), gw0.cpu().numpy()) < 1e-4
    assert _rel(gh1.cpu().numpy(), gh0.cpu().numpy()) < 1e-4
    o = _oracle(c)
    assert _rel(gw1.cpu().numpy(), o["grad_weight"]) < 1e-2


def test_fwd_bwd_chunk_allocation_fallback(cuda_device, monkeypatch):
    """icepop_fwd_bwd's probabilities buffer: if the chunk the memory estimate picked does not
    allocate, the chunk halves, the result equals that chunking, and the size that allocated
    is remembered (later calls do not pay the failed allocation again)."""
    import paper_2510_18855_b200.loss as L
    from paper_2510_18855_b200.loss import IcePopConfig, icepop_fwd_bwd

    c = _case(n_seqs=6, seed=88, V=1000, lens=[3000, 2100, 1700, 900, 4000, 2500])
    H, W = c["H"].to(cuda_device), c["W"].to(cuda_device)
    cfg = IcePopConfig()
    ref, gh_ref, gw_ref = icepop_fwd_bwd(H, W, _batch(c, cuda_device), cfg, grad_hidden_dtype=torch.float32,
                                         max_chunk_tokens=4096)
    real_empty = torch.empty
    calls = []

    def fake_empty(*shape, **kw):
        size = tuple(shape[0]) if len(shape) == 1 and isinstance(shape[0], tuple) else tuple(shape)
        if kw.get("dtype") == torch.bfloat16 and len(size) == 2 and size[1] == 1000:
            calls.append(size[0])
            if size[0] > 4096:
                raise torch.OutOfMemoryError("simulated")
        return real_empty(*shape, **kw)

    key = (cuda_device.index if cuda_device.index is not None else 0, 1000)
    L._PROBS_CHUNK_OK.pop(key, None)
    monkeypatch.setattr(L.torch, "empty", fake_empty)
    try:
        f, gh, gw = icepop_fwd_bwd(H, W, _batch(c, cuda_device), cfg, grad_hidden_dtype=torch.float32,
                                   max_chunk_tokens=8192)
        assert calls[:2] == [8192, 4096] and L._PROBS_CHUNK_OK[key] == 4096
        calls.clear()
        icepop_fwd_bwd(H, W, _batch(c, cuda_device), cfg, grad_hidden_dtype=torch.float32, max_chunk_tokens=8192)
        assert calls[0] == 4096  # remembered: no failed attempt
    finally:
        monkeypatch.undo()
        L._PROBS_CHUNK_OK.pop(key, None)
    assert f.extras["chunks"] == ref.extras["chunks"]
    for name in ("lse", "lp_cur", "kept", "coeff"):
        assert torch.equal(getattr(f, name), getattr(ref, name)), name
    assert torch.equal(gh, gh_ref) and torch.equal(gw, gw_ref)
