"""Shared fixtures. `-m gpu` tests need a B200 and the built libicepop_b200.so;
everything else runs on the CPU build container."""

from __future__ import annotations

import functools
import sys
from pathlib import Path

import numpy as np
import pytest

ROOT = Path(__file__).resolve().parents[1]
GOLDEN = ROOT / "tests" / "golden"
if str(ROOT) not in sys.path:
    sys.path.insert(0, str(ROOT))


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (sm_100a) and libicepop_b200.so")


def golden_cases() -> list[str]:
    """The small/medium reference cases (c1_config0, BASELINE configs[0] at full size, has its
    own schema and tests)."""
    return sorted(p.stem for p in GOLDEN.glob("*.npz")
                  if p.stem not in ("advantages", "c1_config0", "updates", "discrepancy", "lp_record")
                  and "slice" not in p.stem)


def load_c1() -> tuple[dict, np.ndarray]:
    """BASELINE configs[0] fixture (tests/golden/make_golden.py c1_case) and its regenerated
    bf16-exact weights [n_features = 1024, V = 32768] (fp64)."""
    import torch

    with np.load(GOLDEN / "c1_config0.npz") as z:
        d = {k: z[k] for k in z.files}
    w = np.random.default_rng(2510).normal(0.0, 0.8, (1024, 32768))
    w = torch.from_numpy(w).to(torch.bfloat16).to(torch.float64).numpy()
    return d, w


C1_PROJ_SEED = 7


# full-width slice fixtures (make_golden.py c2_slice_case): name -> (weight seed, hidden d)
SLICES = {"c2_slice": (2511, 4096), "c3_slice": (2512, 8192), "c2_slice_kl": (2511, 4096),
          "c2_slice_tis": (2511, 4096)}


def slice_weight_ref(name: str):
    """The reference policy of a KL slice fixture: bf16(W + N(0, 0.1)) with the fixture's
    ref_seed, W the bf16-exact weights (make_golden.py c2_slice_case)."""
    import torch

    seed, d_hidden = SLICES[name]
    with np.load(GOLDEN / f"{name}.npz") as z:
        ref_seed = int(z["ref_seed"])
    w = np.random.default_rng(seed).normal(0.0, 0.5, (d_hidden, 157184))
    w = torch.from_numpy(w).to(torch.bfloat16).to(torch.float64).numpy()
    w += np.random.default_rng(ref_seed).normal(0.0, 0.1, w.shape)
    return torch.from_numpy(w).to(torch.bfloat16)


@functools.lru_cache(maxsize=2)
def load_slice(name: str):
    """A full-width slice fixture (one GRPO group of 8 rollouts at V = 157,184) and its
    regenerated weights as a bf16 torch tensor [d, V] (exact: the reference saw the same
    bf16-rounded values in fp64)."""
    import torch

    seed, d_hidden = SLICES[name]
    with np.load(GOLDEN / f"{name}.npz") as z:
        d = {k: z[k] for k in z.files}
    w = np.random.default_rng(seed).normal(0.0, 0.5, (d_hidden, 157184))
    return d, torch.from_numpy(w).to(torch.bfloat16)


def load_golden(name: str) -> dict:
    with np.load(GOLDEN / f"{name}.npz") as z:
        d = {k: z[k] for k in z.files}
    for k in ("alpha", "beta", "clip_eps", "tis_cap", "temperature", "kl_coeff", "out_objective",
              "out_clipped_fraction", "out_kl_to_ref", "out_mean_logp", "out_entropy_all", "out_entropy_clipped"):
        d[k] = float(d[k])
    d["algo"] = str(d["algo"])
    d["has_ref"] = bool(d["has_ref"])
    d["out_token_count"] = int(d["out_token_count"])
    return d


def golden_hidden(d: dict) -> np.ndarray:
    """H = multihot(feats): the reference's 4-hot contraction as a dense matrix."""
    from paper_2510_18855_b200.features import multihot

    return multihot(d["feats"], d["weight"].shape[0])


def oracle_kwargs(d: dict) -> dict:
    return dict(alpha=d["alpha"], beta=d["beta"], clip_eps=d["clip_eps"], tis_cap=d["tis_cap"],
                temperature=d["temperature"], kl_coeff=d["kl_coeff"], algo=d["algo"], layout="dv",
                weight_ref=d["weight_ref"] if d["has_ref"] else None)


@pytest.fixture(scope="session")
def cuda_device():
    import torch

    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    return torch.device("cuda", 0)


REF_INSTALL = ROOT / "baseline" / "_ref"
_BOUND = ("objective_and_grad", "sgd_update", "momentum_update", "delta_and_gap", "group_advantages")


@pytest.fixture
def mismatchlab_ref():
    """The unmodified reference (the baseline/_ref install, which travels to the GPU box), with
    every name the drop-in's install() rebinds restored afterwards."""
    if not (REF_INSTALL / "mismatchlab").exists():
        pytest.skip("the reference install (baseline/_ref) is not present")
    if str(REF_INSTALL) not in sys.path:
        sys.path.insert(0, str(REF_INSTALL))
    import mismatchlab
    import mismatchlab.discrepancy
    import mismatchlab.objective
    import mismatchlab.scheduler

    from paper_2510_18855_b200 import objective as dropin

    precision = dropin._DEFAULT_PRECISION  # install(precision=...) changes it for the process
    mods = (mismatchlab, mismatchlab.objective, mismatchlab.scheduler, mismatchlab.discrepancy)
    saved = {(m, n): getattr(m, n) for m in mods for n in _BOUND + ("run_iteration", "run_iteration_baseline")
             if hasattr(m, n)}
    try:
        yield mismatchlab
    finally:
        for (m, n), f in saved.items():
            setattr(m, n, f)
        dropin.set_default_precision(precision)
