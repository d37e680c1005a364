"""CUDA path vs the reference's own outputs (golden vectors) and vs the oracle.

Tolerances (stated here):
  * kept mask, popped count, token count: bit-exact (input-only, fp64 on device);
  * fp64 validation path: per-token values and the gradient within 1e-10 relative
    (summation order differs from numpy's);
  * bf16 tensor-core path (H multi-hot exact in bf16, W bf16-exact, fp32 accumulate):
    lp_cur / entropy abs <= 2e-3 (+ 1e-3 relative), objective relative <= 1e-3 (abs 1e-5),
    dW / dH relative Frobenius error <= 1e-2 (bf16 dZ dominates), tokens whose clip
    branch sits within 1e-3 of 1 +- eps excluded from the exact-branch comparisons.
"""

from __future__ import annotations

import math

import numpy as np
import pytest
import torch

from conftest import golden_cases, golden_hidden, load_golden, oracle_kwargs

pytestmark = pytest.mark.gpu


def _batch(d, dev, token_slice=None, use_rewards=False):
    from paper_2510_18855_b200.loss import PackedBatch

    sl = token_slice or slice(0, len(d["tokens"]))
    return PackedBatch(
        tokens=torch.from_numpy(d["tokens"][sl].astype(np.int32)).to(dev),
        lp_train_old=torch.from_numpy(d["lp_train_old"][sl]).to(dev),
        lp_infer_old=torch.from_numpy(d["lp_infer_old"][sl]).to(dev),
        cu_seqlens=torch.from_numpy(d["cu_seqlens"].astype(np.int32)).to(dev),
        group_offsets=torch.from_numpy(d["group_offsets"].astype(np.int32)).to(dev),
        advantages=None if use_rewards else torch.from_numpy(d["advantages"]).to(dev),
        rewards=torch.from_numpy(d["rewards"]).to(dev) if use_rewards else None,
        token_offset=sl.start or 0,
    )


def _cfg(d):
    from paper_2510_18855_b200.loss import IcePopConfig

    return IcePopConfig(alpha=d["alpha"], beta=d["beta"], clip_eps=d["clip_eps"], tis_cap=d["tis_cap"],
                        temperature=d["temperature"], kl_coeff=d["kl_coeff"], algo=d["algo"])


def _rel(a, b):
    a = np.asarray(a, dtype=np.float64)
    b = np.asarray(b, dtype=np.float64)
    den = max(np.linalg.norm(b), 1e-30)
    return float(np.linalg.norm(a - b) / den)


@pytest.mark.parametrize("name", golden_cases())
def test_fp64_path_matches_reference_golden(cuda_device, name):
    from paper_2510_18855_b200.loss import Diagnostics, finish, icepop_bwd, icepop_fwd

    d = load_golden(name)
    H = torch.from_numpy(golden_hidden(d)).to(cuda_device)
    W = torch.from_numpy(d["weight"]).to(cuda_device)
    Wr = torch.from_numpy(d["weight_ref"]).to(cuda_device) if d["has_ref"] else None
    batch = _batch(d, cuda_device)
    cfg = _cfg(d)
    f = icepop_fwd(H, W, batch, cfg, layout="dv", weight_ref=Wr)
    _, gw = icepop_bwd(H, W, batch, f, cfg, layout="dv", weight_ref=Wr, need_hidden=False)
    finish(f.stats)
    diag = Diagnostics.from_stats(f.stats.cpu())
    assert np.array_equal(f.kept.cpu().numpy().astype(bool), d["out_kept"])
    assert diag.token_count == d["out_token_count"]
    assert diag.clipped_fraction == d["out_clipped_fraction"]
    np.testing.assert_allclose(f.calib.cpu().numpy(), d["out_calibration"], rtol=4.5e-16, atol=0)
    np.testing.assert_allclose(f.lp_cur.cpu().numpy(), d["out_lp_cur"], rtol=1e-12, atol=1e-13)
    np.testing.assert_allclose(f.surrogate.cpu().numpy(), d["out_surrogate"], rtol=1e-10, atol=1e-13)
    np.testing.assert_allclose(f.entropy.cpu().numpy(), d["out_entropy"], rtol=1e-12, atol=1e-13)
    assert diag.objective_value == pytest.approx(d["out_objective"], rel=1e-10, abs=1e-14)
    assert diag.mean_logp == pytest.approx(d["out_mean_logp"], rel=1e-12)
    assert diag.entropy_all == pytest.approx(d["out_entropy_all"], rel=1e-12)
    if math.isnan(d["out_entropy_clipped"]):
        assert math.isnan(diag.entropy_clipped)
    else:
        assert diag.entropy_clipped == pytest.approx(d["out_entropy_clipped"], rel=1e-12)
    assert diag.kl_to_ref == pytest.approx(d["out_kl_to_ref"], rel=1e-10, abs=1e-14)
    g = gw.cpu().numpy()
    np.testing.assert_allclose(g, d["out_grad"], rtol=1e-9, atol=1e-13)


@pytest.fixture(params=[1, 2], ids=["cta1", "cta2"])
def cta_group(request):
    from paper_2510_18855_b200 import _lib

    lib = _lib.ensure_device(0)
    _lib.check(lib.icepop_set_cta_group(request.param))
    yield request.param
    _lib.check(lib.icepop_set_cta_group(2))


@pytest.mark.parametrize("store_probs", [None, False], ids=["auto", "recompute"])
@pytest.mark.parametrize("name", [n for n in golden_cases() if "kl" not in n and "refdiag" not in n])
def test_bf16_path_matches_reference_golden(cuda_device, cta_group, name, store_probs):
    from paper_2510_18855_b200.loss import Diagnostics, finish, icepop_bwd, icepop_fwd

    d = load_golden(name)
    H = torch.from_numpy(golden_hidden(d)).to(torch.bfloat16).to(cuda_device)
    W = torch.from_numpy(d["weight"]).to(torch.bfloat16).to(cuda_device)
    assert torch.equal(W.double().cpu(), torch.from_numpy(d["weight"])), "fixture weights must be bf16-exact"
    batch = _batch(d, cuda_device)
    cfg = _cfg(d)
    f = icepop_fwd(H, W, batch, cfg, layout="dv", store_probs=store_probs)  # auto: probs when vocab % 8 == 0
    gh, gw = icepop_bwd(H, W, batch, f, cfg, layout="dv", grad_hidden_dtype=torch.float32)
    finish(f.stats)
    diag = Diagnostics.from_stats(f.stats.cpu())
    # input-only quantities: bit-exact
    assert np.array_equal(f.kept.cpu().numpy().astype(bool), d["out_kept"])
    assert diag.token_count == d["out_token_count"]
    assert diag.clipped_fraction == d["out_clipped_fraction"]
    # CUDA's fp64 exp and numpy's may differ by one ulp (the mask is still bit-exact
    # unless a calibration ratio sits within an ulp of alpha or beta)
    np.testing.assert_allclose(f.calib.cpu().numpy(), d["out_calibration"], rtol=4.5e-16, atol=0)
    # GEMM-dependent quantities: tolerance
    np.testing.assert_allclose(f.lp_cur.cpu().numpy(), d["out_lp_cur"], atol=2e-3, rtol=1e-3)
    np.testing.assert_allclose(f.entropy.cpu().numpy(), d["out_entropy"], atol=2e-3, rtol=1e-3)
    assert diag.objective_value == pytest.approx(d["out_objective"], rel=1e-3, abs=1e-5)
    assert _rel(gw.cpu().numpy(), d["out_grad"]) < 1e-2
    # dH has no reference analogue: check against the oracle restatement
    from oracle.icepop_oracle import icepop_dense

    o = icepop_dense(golden_hidden(d), d["weight"], d["tokens"], d["lp_train_old"], d["lp_infer_old"],
                     d["cu_seqlens"], d["group_offsets"], d["advantages"], **oracle_kwargs(d))
    assert _rel(gh.cpu().numpy(), o["grad_hidden"]) < 1e-2


def test_group_advantages_bit_exact(cuda_device):
    from paper_2510_18855_b200.loss import group_advantages

    z = np.load(__import__("conftest").GOLDEN / "advantages.npz")
    out = group_advantages(torch.from_numpy(z["rewards"]).to(cuda_device),
                           torch.from_numpy(z["group_offsets"]).to(cuda_device))
    np.testing.assert_array_equal(out.cpu().numpy(), z["advantages"])


@pytest.mark.parametrize("dtype", [torch.float64, torch.bfloat16])
def test_rewards_path_uses_k0(cuda_device, dtype):
    """Passing rewards instead of advantages runs K0 on device with identical results."""
    from paper_2510_18855_b200.loss import icepop_fwd

    d = load_golden("medium_icepop")
    H = torch.from_numpy(golden_hidden(d)).to(dtype).to(cuda_device)
    W = torch.from_numpy(d["weight"]).to(dtype).to(cuda_device)
    a = icepop_fwd(H, W, _batch(d, cuda_device), _cfg(d), layout="dv")
    b = icepop_fwd(H, W, _batch(d, cuda_device, use_rewards=True), _cfg(d), layout="dv")
    assert torch.equal(a.surrogate, b.surrogate)
    assert torch.equal(a.stats, b.stats)


@pytest.mark.parametrize("path", ["fp64", "bf16_probs", "bf16_recompute"])
def test_config0_full_size_matches_reference(cuda_device, path):
    """BASELINE configs[0] at full size (8 x 512 tokens, hidden 1,024, vocab 32,768, GRPO
    group 8, default alpha/beta) against the reference's own objective_and_grad
    (tests/golden/c1_config0.npz): mask, token and popped counts bit-exact on every path;
    fp64 path to fp64 rounding; bf16 path within the stated tolerances; dW through its norm
    and a fixed random projection (the fixture stores grad @ R, not 268 MB)."""
    from conftest import C1_PROJ_SEED, load_c1
    from paper_2510_18855_b200.features import multihot
    from paper_2510_18855_b200.loss import Diagnostics, IcePopConfig, finish, icepop_bwd, icepop_fwd

    d, w = load_c1()
    h = multihot(d["feats"], w.shape[0])
    dt = torch.float64 if path == "fp64" else torch.bfloat16
    H = torch.from_numpy(h).to(dt).to(cuda_device)
    W = torch.from_numpy(w).to(dt).to(cuda_device)
    batch = _batch(d, cuda_device)
    cfg = IcePopConfig()
    kw = {} if path == "fp64" else dict(store_probs=(path == "bf16_probs"))
    f = icepop_fwd(H, W, batch, cfg, layout="dv", **kw)
    _, gw = icepop_bwd(H, W, batch, f, cfg, layout="dv", need_hidden=False)
    finish(f.stats)
    diag = Diagnostics.from_stats(f.stats.cpu())
    assert np.array_equal(f.kept.cpu().numpy().astype(bool), d["out_kept"])
    assert diag.token_count == int(d["out_token_count"]) == 4096
    assert diag.clipped_fraction == float(d["out_clipped_fraction"]) > 0
    np.testing.assert_allclose(f.calib.cpu().numpy(), d["out_calibration"], rtol=4.5e-16, atol=0)
    proj = np.random.default_rng(C1_PROJ_SEED).standard_normal((w.shape[1], 4))
    g = gw.double().cpu().numpy()
    if path == "fp64":
        np.testing.assert_allclose(f.lp_cur.cpu().numpy(), d["out_lp_cur"], rtol=1e-12, atol=1e-12)
        np.testing.assert_allclose(f.entropy.cpu().numpy(), d["out_entropy"], rtol=1e-12)
        assert diag.objective_value == pytest.approx(float(d["out_objective"]), rel=1e-10)
        np.testing.assert_allclose(g @ proj, d["out_grad_proj"], rtol=1e-9, atol=1e-12)
        assert np.linalg.norm(g) == pytest.approx(float(d["out_grad_norm"]), rel=1e-10)
    else:
        np.testing.assert_allclose(f.lp_cur.cpu().numpy(), d["out_lp_cur"], atol=2e-3, rtol=1e-3)
        np.testing.assert_allclose(f.entropy.cpu().numpy(), d["out_entropy"], atol=2e-3, rtol=1e-3)
        assert diag.objective_value == pytest.approx(float(d["out_objective"]), rel=1e-3, abs=1e-5)
        assert _rel(g @ proj, d["out_grad_proj"]) < 1e-2
        assert np.linalg.norm(g) == pytest.approx(float(d["out_grad_norm"]), rel=1e-2)


@pytest.mark.parametrize("store_probs", [True, False], ids=["probs", "recompute"])
@pytest.mark.parametrize("name", ["c2_slice", "c3_slice", "c2_slice_tis"])
def test_full_width_slice_matches_reference(cuda_device, name, store_probs):
    """One GRPO group at BASELINE's full lm_head width against the reference's own
    objective_and_grad (H = the reference's 4-hot features, exact in bf16): c2_slice = 8 x 4,096
    tokens at hidden 4,096 (configs[1]), c3_slice = 8 x 2,048 tokens at hidden 8,192
    (configs[2]-[4]), c2_slice_tis = TIS at temperature 0.7, 8 x 2,048 tokens at hidden 4,096;
    vocab 157,184. Mask and counts bit-exact; lp_cur / entropy / objective /
    dW (norm and a fixed projection) within the bf16 path's tolerances."""
    from conftest import C1_PROJ_SEED, GOLDEN, load_slice
    from paper_2510_18855_b200.features import multihot
    from paper_2510_18855_b200.loss import Diagnostics, IcePopConfig, finish, icepop_bwd, icepop_fwd

    if not (GOLDEN / f"{name}.npz").exists():
        pytest.skip(f"{name}.npz not generated")
    d, w = load_slice(name)
    H = torch.from_numpy(multihot(d["feats"], w.shape[0])).to(torch.bfloat16).to(cuda_device)
    W = w.to(cuda_device)
    batch = _batch(d, cuda_device)
    cfg = IcePopConfig(algo=str(d["algo"]) if "algo" in d else "icepop",
                       temperature=float(d["temperature"]) if "temperature" in d else 1.0)
    f = icepop_fwd(H, W, batch, cfg, layout="dv", store_probs=store_probs)
    _, gw = icepop_bwd(H, W, batch, f, cfg, layout="dv", need_hidden=False)
    finish(f.stats)
    diag = Diagnostics.from_stats(f.stats.cpu())
    assert np.array_equal(f.kept.cpu().numpy().astype(bool), d["out_kept"])
    assert diag.token_count == int(d["out_token_count"]) == len(d["tokens"])
    assert diag.clipped_fraction == float(d["out_clipped_fraction"])
    np.testing.assert_allclose(f.calib.cpu().numpy(), d["out_calibration"], rtol=4.5e-16, atol=0)
    np.testing.assert_allclose(f.lp_cur.cpu().numpy(), d["out_lp_cur"], atol=2e-3, rtol=1e-3)
    np.testing.assert_allclose(f.entropy.cpu().numpy(), d["out_entropy"], atol=2e-3, rtol=1e-3)
    assert diag.objective_value == pytest.approx(float(d["out_objective"]), rel=1e-3, abs=1e-5)
    proj = torch.from_numpy(np.random.default_rng(C1_PROJ_SEED).standard_normal((w.shape[1], 4))).to(cuda_device)
    gp = (gw.double() @ proj).cpu().numpy()
    assert _rel(gp, d["out_grad_proj"]) < 1e-2
    assert float(torch.linalg.vector_norm(gw.double())) == pytest.approx(float(d["out_grad_norm"]), rel=1e-2)


def test_full_width_kl_slice_matches_reference(cuda_device):
    """The KL-to-ref term (gamma = 0.4, objective.py:254-263) at configs[1]'s width (8 x 2,048
    tokens, hidden 4,096, vocab 157,184; reference policy = W + N(0, 0.1)) against the
    reference's own objective_and_grad (tests/golden/c2_slice_kl.npz): the dual-accumulator
    K1r/K3r GEMMs. Mask and counts bit-exact; kl_to_ref, objective, lp_cur and dW (norm and
    projection) within the bf16 path's tolerances."""
    from conftest import C1_PROJ_SEED, GOLDEN, load_slice, slice_weight_ref
    from paper_2510_18855_b200.features import multihot
    from paper_2510_18855_b200.loss import Diagnostics, IcePopConfig, finish, icepop_bwd, icepop_fwd

    if not (GOLDEN / "c2_slice_kl.npz").exists():
        pytest.skip("c2_slice_kl.npz not generated")
    d, w = load_slice("c2_slice_kl")
    wr = slice_weight_ref("c2_slice_kl")
    H = torch.from_numpy(multihot(d["feats"], w.shape[0])).to(torch.bfloat16).to(cuda_device)
    W, Wr = w.to(cuda_device), wr.to(cuda_device)
    batch = _batch(d, cuda_device)
    cfg = IcePopConfig(kl_coeff=float(d["kl_coeff"]))
    f = icepop_fwd(H, W, batch, cfg, layout="dv", weight_ref=Wr)
    _, gw = icepop_bwd(H, W, batch, f, cfg, layout="dv", weight_ref=Wr, need_hidden=False)
    finish(f.stats)
    diag = Diagnostics.from_stats(f.stats.cpu())
    assert np.array_equal(f.kept.cpu().numpy().astype(bool), d["out_kept"])
    assert diag.token_count == int(d["out_token_count"]) == len(d["tokens"])
    assert diag.clipped_fraction == float(d["out_clipped_fraction"])
    np.testing.assert_allclose(f.lp_cur.cpu().numpy(), d["out_lp_cur"], atol=2e-3, rtol=1e-3)
    assert diag.kl_to_ref == pytest.approx(float(d["out_kl_to_ref"]), rel=1e-2, abs=1e-5)
    assert diag.objective_value == pytest.approx(float(d["out_objective"]), rel=1e-3, abs=1e-5)
    proj = torch.from_numpy(np.random.default_rng(C1_PROJ_SEED).standard_normal((w.shape[1], 4))).to(cuda_device)
    assert _rel((gw.double() @ proj).cpu().numpy(), d["out_grad_proj"]) < 1e-2
    assert float(torch.linalg.vector_norm(gw.double())) == pytest.approx(float(d["out_grad_norm"]), rel=1e-2)
