"""The discrepancy probe: delta = mean KL(p_infer || p_train) over the probe
set and max_token_gap = max |p_infer - p_train| (discrepancy.py:132-141), on the GPU.

Pinned against tests/golden/discrepancy.npz, made by the unmodified reference
(make_golden_next.py): the probe set of make_probes, the feature rows of each probe, the
inference engine's logits (the reference's own perturbation of the scaled train logits) and
its delta and gap, for a heavily and a mildly mismatched engine and two temperatures.
Tolerances: fp64 path 1e-12 relative (the GEMM sums the 4-hot rows in another order);
bf16 path (weights bf16-exact, infer logits rounded to fp32) 1e-5 relative on delta, 1e-5 on the gap.
"""

from __future__ import annotations

from pathlib import Path

import numpy as np
import pytest
import torch

from conftest import GOLDEN

pytestmark = pytest.mark.gpu
ROOT = Path(__file__).resolve().parents[1]
CASES = ("big", "big_t08", "small")


def _golden():
    with np.load(GOLDEN / "discrepancy.npz") as z:
        return {k: z[k] for k in z.files}


@pytest.mark.parametrize("case", CASES)
@pytest.mark.parametrize("precision", ["fp64", "bf16"])
def test_delta_and_gap_vs_reference(cuda_device, case, precision):
    from paper_2510_18855_b200.features import multihot_device
    from paper_2510_18855_b200.loss import delta_and_gap

    d = _golden()
    w = d["weights"]
    feats = torch.from_numpy(d["feats"].astype(np.int64)).to(cuda_device)
    T = float(d[f"temperature_{case}"])
    if precision == "fp64":
        H = multihot_device(feats, w.shape[0], torch.float64)
        W = torch.from_numpy(w).to(cuda_device)
        zi = torch.from_numpy(d[f"infer_{case}"]).to(cuda_device)
        tol_d, tol_g = 1e-12, 1e-12
    else:
        H = multihot_device(feats, w.shape[0], torch.bfloat16)
        W = torch.from_numpy(w).to(torch.bfloat16).to(cuda_device)
        zi = torch.from_numpy(d[f"infer_{case}"].astype(np.float32)).to(cuda_device)
        tol_d, tol_g = 1e-5, 1e-5
    delta, gap, kl, rowgap = delta_and_gap(H, W, zi, layout="dv", temperature=T)
    assert float(delta) == pytest.approx(float(d[f"delta_{case}"]), rel=tol_d, abs=1e-12)
    assert float(gap) == pytest.approx(float(d[f"gap_{case}"]), rel=tol_g, abs=tol_g)
    assert float(kl.mean()) == pytest.approx(float(delta), rel=1e-12)
    assert float(rowgap.max()) == float(gap)
    assert bool((kl >= -1e-12).all())  # KL is nonnegative (test_discrepancy.py:51-59)


def test_identical_engines_give_exactly_zero(cuda_device):
    """Infer logits equal to the train logits: delta and gap exactly 0 (test_discrepancy.py:35-41)."""
    from paper_2510_18855_b200.features import multihot_device
    from paper_2510_18855_b200.loss import delta_and_gap

    d = _golden()
    H = multihot_device(torch.from_numpy(d["feats"].astype(np.int64)).to(cuda_device), d["weights"].shape[0],
                        torch.float64)
    W = torch.from_numpy(d["weights"]).to(cuda_device)
    zi = (H @ W).contiguous()
    delta, gap, _, _ = delta_and_gap(H, W, zi, layout="dv")
    assert float(delta) == 0.0 and float(gap) == 0.0


def test_empty_probe_set_is_value_error(cuda_device):
    from paper_2510_18855_b200.loss import delta_and_gap

    H = torch.zeros((0, 8), dtype=torch.float64, device=cuda_device)
    W = torch.zeros((8, 16), dtype=torch.float64, device=cuda_device)
    with pytest.raises(ValueError, match="probe set"):
        delta_and_gap(H, W, torch.zeros((0, 16), dtype=torch.float64, device=cuda_device), layout="dv")


def test_dropin_delta_and_gap_and_install(cuda_device, mismatchlab_ref):
    """The drop-in delta_and_gap(params, probes, infer, temperature) against the reference
    itself (its probes, engine and noise model from the baseline/_ref install), and install()
    rebinding measure()'s lookup (discrepancy.py:144-161)."""
    import mismatchlab.discrepancy as D

    from paper_2510_18855_b200 import objective

    ml = mismatchlab_ref
    d = _golden()
    probes = ml.make_probes(96, ml.Vocabulary(size=64), seed=11)
    params = ml.PolicyParams(weights=d["weights"], version_id=int(d["version"]))
    for case in CASES:
        eng = ml.infer_engine(float(d[f"scale_{case}"]), 5)
        got = objective.delta_and_gap(params, probes, eng, float(d[f"temperature_{case}"]))
        assert got[0] == pytest.approx(float(d[f"delta_{case}"]), rel=1e-12)
        assert got[1] == pytest.approx(float(d[f"gap_{case}"]), rel=1e-12, abs=1e-15)
    objective.install()
    assert D.delta_and_gap is objective.delta_and_gap and ml.delta_and_gap is objective.delta_and_gap
    s = D.measure(params, probes, ml.infer_engine(0.02, 5), 1.0, step=3)
    assert s.step == 3 and s.delta == pytest.approx(float(d["delta_small"]), rel=1e-12)
