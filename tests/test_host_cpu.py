"""Host-side logic on CPU: the C-ABI library loads and exports every declared symbol,
the ctypes structs match the C layout, and the feature-hash restatement matches the
reference's feature rows recorded in the golden vectors."""

from __future__ import annotations

import re
import subprocess
from pathlib import Path

import numpy as np
import pytest

from conftest import ROOT, golden_cases, load_golden

HEADER = ROOT / "include" / "icepop.h"


def _declared_functions() -> list[str]:
    text = HEADER.read_text()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(icepop_[a-z0-9_]+)\s*\(", text)))


def test_library_exports_every_declared_symbol():
    from paper_2510_18855_b200 import _lib

    lib = _lib.load()
    declared = _declared_functions()
    assert len(declared) >= 12
    for name in declared:
        assert hasattr(lib, name), f"missing export {name}"
        assert name in _lib.SIGNATURES, f"no ctypes signature for {name}"
    assert set(_lib.SIGNATURES) == set(declared)
    out = subprocess.run(["nm", "-D", "--defined-only", str(_lib.LIB_PATH)], capture_output=True, text=True,
                         check=True).stdout
    for name in declared:
        assert re.search(rf"\bT {name}$", out, re.M), f"{name} not a defined text symbol"
    assert lib.icepop_abi_version() == _lib.ABI_VERSION == 4


def test_library_has_sm100a_tensor_core_code():
    """The shipped .so carries tcgen05 MMA / TMA / TMEM loads, not legacy HMMA."""
    from paper_2510_18855_b200 import _lib

    sass = subprocess.run(["cuobjdump", "-sass", str(_lib.LIB_PATH)], capture_output=True, text=True).stdout
    if not sass:
        pytest.skip("cuobjdump unavailable")
    assert "UTCHMMA" in sass and "UTMALDG" in sass and "LDTM" in sass
    assert "sm_100a" in subprocess.run(["cuobjdump", "-lelf", str(_lib.LIB_PATH)], capture_output=True,
                                       text=True).stdout


def test_ctypes_struct_layout_matches_c(tmp_path: Path):
    from paper_2510_18855_b200 import _lib

    src = tmp_path / "layout.c"
    src.write_text(
        '#include <stdio.h>\n#include <stddef.h>\n#include "icepop.h"\n'
        "int main(void){printf(\"%zu %zu %zu %zu %zu %zu %zu %zu %zu %zu\\n\", sizeof(icepop_config), sizeof(icepop_shape),"
        " sizeof(icepop_batch), sizeof(icepop_fwd_out), sizeof(icepop_f64_out), offsetof(icepop_shape, n_seqs),"
        " offsetof(icepop_config, algo), sizeof(icepop_saved), offsetof(icepop_saved, tile_max), offsetof(icepop_saved, lp_cur));return 0;}\n")
    exe = tmp_path / "layout"
    subprocess.run(["gcc", "-I", str(ROOT / "include"), str(src), "-o", str(exe)], check=True)
    got = [int(x) for x in subprocess.run([str(exe)], capture_output=True, text=True, check=True).stdout.split()]
    import ctypes

    want = [ctypes.sizeof(_lib.Config), ctypes.sizeof(_lib.Shape), ctypes.sizeof(_lib.Batch),
            ctypes.sizeof(_lib.FwdOut), ctypes.sizeof(_lib.F64Out), _lib.Shape.n_seqs.offset,
            _lib.Config.algo.offset, ctypes.sizeof(_lib.Saved), _lib.Saved.tile_max.offset, _lib.Saved.lp_cur.offset]
    assert got == want


def test_no_cpu_fallback_on_cpu_tensors():
    import torch

    from paper_2510_18855_b200.loss import PackedBatch, icepop_fwd

    b = PackedBatch(torch.zeros(2, dtype=torch.int32), torch.zeros(2, dtype=torch.float64),
                    torch.zeros(2, dtype=torch.float64), torch.tensor([0, 1, 2], dtype=torch.int32),
                    torch.tensor([0, 2], dtype=torch.int32), torch.zeros(2, dtype=torch.float64))
    with pytest.raises(RuntimeError, match="no CPU fallback"):
        icepop_fwd(torch.zeros(2, 8, dtype=torch.bfloat16), torch.zeros(8, 8, dtype=torch.bfloat16), b)


@pytest.mark.parametrize("name", golden_cases())
def test_feature_hash_matches_reference_rows(name):
    from paper_2510_18855_b200.features import rollout_feats

    d = load_golden(name)
    cu = d["cu_seqlens"]
    nf = d["weight"].shape[0]
    for i in range(len(cu) - 1):
        got = rollout_feats(int(d["prompt_ids"][i]), d["tokens"][cu[i]:cu[i + 1]], nf)
        assert np.array_equal(got, d["feats"][cu[i]:cu[i + 1]])


def test_vectorised_feature_hash_equals_the_scalar_walk():
    """rollout_feats (numpy uint64, all positions at once) equals the reference's per-position
    walk of feature_rows (objective.py:162-169, policy.py:229-260) bit for bit, including
    negative / 63-bit prompt ids, large token ids and 1- and 2-token rollouts."""
    from paper_2510_18855_b200.features import feature_rows, rollout_feats

    rng = np.random.default_rng(5)
    for _ in range(200):
        T = int(rng.integers(1, 40))
        nf = int(rng.integers(1, 5000))
        pid = int(rng.integers(-2 ** 62, 2 ** 62))
        toks = [int(x) for x in rng.integers(0, 2 ** 31 - 1, T)]
        ref, prev, last = [], -1, -1
        for t in toks:
            ref.append(feature_rows(pid, prev, last, nf))
            prev, last = last, t
        assert np.array_equal(rollout_feats(pid, toks, nf), np.array(ref, dtype=np.int64).reshape(-1, 4))


def test_multihot_counts_duplicates():
    from paper_2510_18855_b200.features import multihot

    h = multihot(np.array([[1, 1, 3, 0], [2, 2, 2, 2]]), 4)
    assert h.tolist() == [[1, 2, 0, 1], [0, 0, 4, 0]]


def _records(O, toks, version=0):
    return [O.TokenRecord(int(t), -1.0, -1.1, -1.1, version) for t in toks]


def test_pack_stops_at_the_first_invalid_rollout():
    """The drop-in validates like objective.py:204-213, in the reference's loop order: the valid
    prefix is packed and the first invalid group / rollout comes back as the error to raise after
    the prefix has been computed (a NumericError in the prefix comes first)."""
    from dataclasses import dataclass

    from paper_2510_18855_b200 import objective as O

    @dataclass
    class Task:
        prompt_id: int

    @dataclass
    class Rollout:
        tokens: list

    @dataclass
    class Params:
        weights: np.ndarray
        version_id: int = 1

        @property
        def n_features(self):
            return self.weights.shape[0]

    theta = Params(np.zeros((16, 8)))
    g1 = O.PromptGroup(Task(3), [Rollout(_records(O, [1, 2, 3])), Rollout(_records(O, [4]))], [1.0, 0.0], [1.0, -1.0])
    g2 = O.PromptGroup(Task(4), [Rollout(_records(O, [5, 6])), Rollout([])], [1.0, 0.0], [1.0, -1.0])
    p = O._pack([g1, g2], theta, theta)
    assert isinstance(p.error, ValueError) and "empty rollout" in str(p.error)
    assert p.tokens.tolist() == [1, 2, 3, 4, 5, 6] and p.cu.tolist() == [0, 3, 4, 6] and p.go.tolist() == [0, 2, 3]
    assert len(p.records) == 6 and p.feats.shape == (6, 4)
    g3 = O.PromptGroup(Task(5), [Rollout(_records(O, [7], version=2))], [1.0], [0.0])
    p = O._pack([g1, g3], theta, theta)
    assert "newer than theta_old" in str(p.error) and p.cu.tolist() == [0, 3, 4] and p.go.tolist() == [0, 2]
    p = O._pack([O.PromptGroup(Task(6), [], [], []), g1], theta, theta)
    assert "empty prompt group" in str(p.error) and not p.records
    p = O._pack([g1], theta, theta)
    assert p.error is None and p.lp_old.tolist() == [-1.1] * 4 and p.lp_inf.tolist() == [-1.0] * 4
    with pytest.raises(ValueError, match="at least one prompt group"):
        O._pack([], theta, theta)
    with pytest.raises(ValueError, match="newer than theta"):
        O._pack([g1], Params(theta.weights, 0), theta)
