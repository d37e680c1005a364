"""The reference's OWN test modules, unchanged, against the drop-in.

__graft_entry__.build() copies pkg/tests/test_objective.py, test_discrepancy.py and
test_scheduler.py from the reference into baseline/_ref_tests/ (git-ignored; it travels to the
GPU box with the baseline/_ref install) next to a generated conftest.py that calls
``paper_2510_18855_b200.objective.install()`` before the modules import mismatchlab's names. So
their objective_and_grad, group_advantages, sgd_update / momentum_update, delta_and_gap and
train_loop (which calls all of them) run on the GPU through this library, and every assertion
is the reference's own: finite differences < 1e-5, exact-zero gradients, bit-identical
degeneracies, mask and clip algebra, bit-identical replays of train_loop.
"""

from __future__ import annotations

import os
import re
import subprocess
import sys
from pathlib import Path

import pytest

pytestmark = pytest.mark.gpu
ROOT = Path(__file__).resolve().parents[1]
SUITE = ROOT / "baseline" / "_ref_tests"


# On the bf16 tensor-core path the tests that resolve the weights below bf16's resolution cannot
# hold: the finite differences use h = 1e-6, and an exactly-zero delta at
# mismatch scale 0 (also what makes the theorem fit "vacuous") needs the inference logits in the
# train logits' own rounding, while the drop-in's train logits come from bf16 weights. They are
# deselected; everything else runs.
BF16_DESELECT = ("not finite_differences and not zero_scale_gives_exactly_zero_delta "
                 "and not zero_scale_is_vacuous")


@pytest.mark.parametrize("precision", ["fp64", "bf16"])
@pytest.mark.parametrize("module", ["test_objective.py", "test_discrepancy.py", "test_scheduler.py"])
def test_reference_suite_passes_unchanged(cuda_device, module, precision):
    if not (SUITE / module).exists() or not (ROOT / "baseline" / "_ref" / "mismatchlab").exists():
        pytest.skip("the reference's tests / install are not present (run __graft_entry__.build() where "
                    "/root/reference exists)")
    env = dict(os.environ, ICEPOP_DROPIN_PRECISION=precision, PYTHONDONTWRITEBYTECODE="1")
    sel = ["-k", BF16_DESELECT] if precision == "bf16" else []
    r = subprocess.run([sys.executable, "-m", "pytest", str(SUITE / module), "-q", "-p", "no:cacheprovider",
                        "--rootdir", str(SUITE), *sel], capture_output=True, text=True, cwd=str(SUITE), env=env,
                       timeout=1200)
    tail = r.stdout[-3000:] + r.stderr[-2000:]
    assert r.returncode == 0, tail
    m = re.search(r"(\d+) passed", r.stdout)
    assert m and int(m.group(1)) > 0, tail
    print(f"{module} [{precision}]: {m.group(0)} under install()")
