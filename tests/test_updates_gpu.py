"""The step after the loss on the GPU.

* The drop-in's sgd_update / momentum_update run the reference's fp64 ascent step in one CUDA
  kernel (icepop_sgd_update_f64) and give the reference's bits (tests/golden/updates.npz, made
  by the unmodified reference: make_golden_next.py), version_id + 1, and its exceptions.
* install() rebinds the update names wherever the reference binds them (scheduler.py:29-40,
  __init__.py:32-34), so train_loop's update (scheduler.py:551-555) runs on the device.
* The tensor-level composed ZeRO step: the fused K5 reduce-scatter's shard (PeerSlots.fold) ->
  the sharded fp32 device update -> the bf16 all-gather, emulated for 3 ranks on one GPU (the
  slot buffers in local memory, no kernel waiting on another), equals the unsharded update.
"""

from __future__ import annotations

from dataclasses import dataclass
from pathlib import Path

import numpy as np
import pytest
import torch

from conftest import GOLDEN

pytestmark = pytest.mark.gpu
ROOT = Path(__file__).resolve().parents[1]


@dataclass
class Params:
    weights: np.ndarray
    version_id: int = 0


def _golden():
    with np.load(GOLDEN / "updates.npz") as z:
        return {k: z[k] for k in z.files}


def test_sgd_update_matches_reference_bits(cuda_device):
    from paper_2510_18855_b200.objective import sgd_update

    d = _golden()
    theta = Params(d["w"].copy(), int(d["version"]))
    s1 = sgd_update(theta, d["g"], float(d["lr1"]))
    assert s1.version_id == int(d["s1_version"]) and isinstance(s1, Params)
    assert np.array_equal(s1.weights, d["s1"])
    s2 = sgd_update(s1, d["g"] * 0.5, float(d["lr2"]))
    assert s2.version_id == int(d["s2_version"]) and np.array_equal(s2.weights, d["s2"])
    assert np.array_equal(theta.weights, d["w"])  # pure: the input parameters are untouched


def test_momentum_update_matches_reference_bits(cuda_device):
    from paper_2510_18855_b200.objective import momentum_update

    d = _golden()
    theta = Params(d["w"].copy(), int(d["version"]))
    p1, v1 = momentum_update(theta, d["g"], d["v"], float(d["lr_m"]), float(d["beta1"]))
    assert np.array_equal(p1.weights, d["p1"]) and np.array_equal(v1, d["v1"])
    assert p1.version_id == int(d["p1_version"])
    p2, v2 = momentum_update(p1, d["g"], v1, float(d["lr_m"]), float(d["beta2"]))
    assert np.array_equal(p2.weights, d["p2"]) and np.array_equal(v2, d["v2"])


def test_update_errors_match_reference(cuda_device):
    from paper_2510_18855_b200.errors import NumericError
    from paper_2510_18855_b200.objective import momentum_update, sgd_update

    theta = Params(np.zeros((4, 8)))
    with pytest.raises(ValueError, match="learning rate"):
        sgd_update(theta, np.zeros((4, 8)), 0.0)
    with pytest.raises(ValueError, match="shape"):
        sgd_update(theta, np.zeros((4, 7)), 0.1)
    with pytest.raises(ValueError, match="beta"):
        momentum_update(theta, np.zeros((4, 8)), np.zeros((4, 8)), 0.1, beta=1.0)
    big = Params(np.full((4, 8), 1e308))
    with pytest.raises(NumericError, match="non-finite"):  # objective.py:309-310
        sgd_update(big, np.full((4, 8), 1e308), 10.0)


def test_install_rebinds_the_update(cuda_device, mismatchlab_ref):
    """install() puts the device update where train_loop looks it up (scheduler.py:551-555)."""
    import mismatchlab.objective
    import mismatchlab.scheduler

    from paper_2510_18855_b200 import objective

    ml = mismatchlab_ref
    objective.install()
    for m in (ml, mismatchlab.objective, mismatchlab.scheduler):
        assert m.sgd_update is objective.sgd_update and m.momentum_update is objective.momentum_update
    d = _golden()
    p = ml.PolicyParams(weights=d["w"].copy(), version_id=int(d["version"]))
    out = mismatchlab.scheduler.sgd_update(p, d["g"], float(d["lr1"]))
    assert isinstance(out, ml.PolicyParams) and np.array_equal(out.weights, d["s1"])


@pytest.mark.parametrize("world", [1, 3])
@pytest.mark.parametrize("layout", ["vd", "dv"])
def test_composed_zero_step_emulated_ranks(cuda_device, layout, world):
    """K5's fused reduce-scatter -> fold -> sharded device update (momentum) -> bf16 all-gather,
    for `world` emulated ranks run one after another on this GPU, equals one unsharded step on
    the summed dW."""
    from paper_2510_18855_b200 import _lib
    from paper_2510_18855_b200.distributed import shard_batch
    from paper_2510_18855_b200.loss import IcePopConfig, icepop_bwd, icepop_bwd_reduce_scatter, icepop_fwd
    from paper_2510_18855_b200.optim import ShardedAscent
    from test_dense_gpu import _batch, _case

    c = _case(seed=41, layout=layout, V=1000, d=256)
    H, W = c["H"].to(cuda_device), c["W"].to(cuda_device)
    full = _batch(c, cuda_device)
    cfg = IcePopConfig()
    rows = W.shape[0]  # dW rows: V ([V,d]) or d ([d,V])
    row_len = W.shape[1]
    lr, beta = 0.3, 0.9
    # reference: the unsharded dW and one fp32 momentum step on it
    f = icepop_fwd(H, W, full, cfg, layout=layout)
    _, gw = icepop_bwd(H, W, full, f, cfg, layout=layout, need_hidden=False)
    master = W.float().clone()
    vel0 = torch.randn(W.shape, device=cuda_device, generator=torch.Generator(device=cuda_device).manual_seed(3))
    vel = vel0.clone()
    want_v = beta * vel + gw
    want_w = (master + lr * want_v).to(torch.bfloat16)
    # emulated ranks: every rank's K5 stores its dW rows into the owners' slots (local memory)
    opt = ShardedAscent(W, lr=lr, beta=beta, world=world, emulate=True)
    for r in range(world):
        opt.velocity_shard(r).copy_(opt.shard_of(vel0, r))
    for r in range(world):
        h, b = shard_batch(H, full, r, world)
        fr = icepop_fwd(h, W, b, cfg, layout=layout)
        icepop_bwd_reduce_scatter(h, W, b, fr, opt.rs_target(r), cfg, layout=layout, need_hidden=False)
    w_new = opt.step()  # fold per owner, sharded update, gather into the bf16 weights
    assert w_new.data_ptr() == W.data_ptr()
    assert torch.equal(w_new, want_w) or float((w_new.float() - want_w.float()).abs().max()) <= 2 ** -7 * float(
        want_w.float().abs().max())
    assert _lib.ABI_VERSION == 4
