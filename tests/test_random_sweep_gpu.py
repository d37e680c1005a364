"""Seeded random sweep over shapes and options on the bf16 path vs the fp64 oracle: N (1 to
3,000, ragged sequences), d and V (multiples of 8 only), both weight layouts, the three
algorithms, temperature, both backward modes and both CTA configurations. Tolerances as in
test_dense_gpu.py: kept mask exact, lp_cur abs <= 2e-3 (+1e-3 rel), dW/dH rel <= 1e-2."""

from __future__ import annotations

import os

import numpy as np
import pytest
import torch

from test_dense_gpu import _batch, _oracle, _rel

pytestmark = pytest.mark.gpu


def _random_case(seed):
    rng = np.random.default_rng(1000 + seed)
    n_seqs = int(rng.integers(1, 7)) * 2
    lens = [int(x) for x in rng.integers(1, 500, n_seqs)]
    d = int(rng.integers(1, 40)) * 8
    V = int(rng.integers(1, 400)) * 8
    layout = ["vd", "dv"][int(rng.integers(0, 2))]
    N = sum(lens)
    H = torch.from_numpy(rng.normal(0, 1, (N, d))).to(torch.bfloat16)
    shape_w = (V, d) if layout == "vd" else (d, V)
    W = torch.from_numpy(rng.normal(0, 2 / np.sqrt(d), shape_w)).to(torch.bfloat16)
    T = float(rng.choice([1.0, 0.7, 1.3]))
    tokens = rng.integers(0, V, N).astype(np.int32)
    Hd, Wd = H.double().numpy(), W.double().numpy()
    z = Hd @ (Wd.T if layout == "vd" else Wd) / T
    lse = z.max(1) + np.log(np.exp(z - z.max(1, keepdims=True)).sum(1))
    lp_old = z[np.arange(N), tokens] - lse + rng.normal(0, 0.15, N)
    lp_inf = lp_old - rng.normal(0, 0.3, N)
    cu = np.concatenate([[0], np.cumsum(lens)]).astype(np.int32)
    go = np.arange(0, n_seqs + 1, 2).astype(np.int32)
    adv = rng.normal(0, 1, n_seqs)
    algo = ["icepop", "grpo", "tis"][int(rng.integers(0, 3))]
    return dict(H=H, W=W, tokens=tokens, lp_old=lp_old, lp_inf=lp_inf, cu=cu, go=go, adv=adv, layout=layout), T, algo, \
        bool(rng.integers(0, 2)), int(rng.integers(1, 3))


# ICEPOP_SWEEP_SEEDS widens the sweep for one-off stress runs (the suite runs 64)
@pytest.mark.parametrize("seed", range(int(os.environ.get("ICEPOP_SWEEP_SEEDS", "64"))))
def test_random_config_vs_oracle(cuda_device, seed):
    from paper_2510_18855_b200 import _lib
    from paper_2510_18855_b200.loss import IcePopConfig, icepop_bwd, icepop_fwd

    c, T, algo, sp, cg = _random_case(seed)
    lib = _lib.ensure_device(0)
    _lib.check(lib.icepop_set_cta_group(cg))
    try:
        cfg = IcePopConfig(algo=algo, temperature=T)
        H, W = c["H"].to(cuda_device), c["W"].to(cuda_device)
        f = icepop_fwd(H, W, _batch(c, cuda_device), cfg, layout=c["layout"], store_probs=sp)
        gh, gw = icepop_bwd(H, W, _batch(c, cuda_device), f, cfg, layout=c["layout"],
                            grad_hidden_dtype=torch.float32)
    finally:
        _lib.check(lib.icepop_set_cta_group(2))
    o = _oracle(c, algo=algo, temperature=T)
    assert np.array_equal(f.kept.cpu().numpy().astype(bool), o["kept"])
    np.testing.assert_allclose(f.lp_cur.cpu().numpy(), o["lp_cur"], atol=2e-3, rtol=1e-3)
    if np.linalg.norm(o["grad_weight"]) > 1e-12:
        assert _rel(gw.cpu().numpy(), o["grad_weight"]) < 1e-2
        assert _rel(gh.cpu().numpy(), o["grad_hidden"]) < 1e-2
