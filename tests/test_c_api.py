"""The C ABI used from C alone (examples/c_api_example.c): it compiles and links against
include/icepop.h + libicepop_b200.so on CPU; on a B200 it runs one fwd+bwd step and its
statistics and dW equal, bit for bit, the same step through the Python layer."""

from __future__ import annotations

import shutil
import subprocess
from pathlib import Path

import numpy as np
import pytest

ROOT = Path(__file__).resolve().parents[1]
CUDA = Path("/usr/local/cuda")


def _build(tmp_path: Path) -> Path:
    if shutil.which("gcc") is None or not (CUDA / "include" / "cuda_runtime.h").exists():
        pytest.skip("gcc or CUDA headers unavailable")
    from paper_2510_18855_b200 import _lib

    exe = tmp_path / "c_api_example"
    lib_dir = _lib.LIB_PATH.parent
    subprocess.run(["gcc", "-O2", "-std=c11", "-Wall", "-Werror", "-I", str(ROOT / "include"),
                    "-I", str(CUDA / "include"), str(ROOT / "examples" / "c_api_example.c"), "-L", str(lib_dir),
                    "-licepop_b200", "-L", str(CUDA / "lib64"), "-lcudart", "-lm", f"-Wl,-rpath,{lib_dir}",
                    "-o", str(exe)], check=True)
    return exe


def test_c_example_compiles_and_links(tmp_path):
    exe = _build(tmp_path)
    assert exe.exists()


@pytest.mark.gpu
def test_c_example_matches_python_layer(tmp_path, cuda_device):
    import torch

    import paper_2510_18855_b200.loss as L
    from paper_2510_18855_b200.loss import IcePopConfig, PackedBatch, icepop_bwd, icepop_fwd

    if not L.SP_ROWSCALE:
        pytest.skip("ICEPOP_SP_ROWSCALE=0 takes another backward path than the C example")
    exe = _build(tmp_path)
    dump = tmp_path / "dump.bin"
    r = subprocess.run([str(exe), str(dump)], capture_output=True, text=True, timeout=120)
    assert r.returncode == 0, r.stderr
    assert "objective=" in r.stdout
    N, d, V, S = 1000, 256, 2048, 4
    raw = dump.read_bytes()
    off = 0

    def take(dtype, n):
        nonlocal off
        a = np.frombuffer(raw, dtype=dtype, count=n, offset=off)
        off += a.nbytes
        return a

    H = torch.from_numpy(take(np.int16, N * d).copy()).view(torch.bfloat16).view(N, d).to(cuda_device)
    W = torch.from_numpy(take(np.int16, V * d).copy()).view(torch.bfloat16).view(V, d).to(cuda_device)
    tokens = torch.from_numpy(take(np.int32, N).copy()).to(cuda_device)
    lp_old = torch.from_numpy(take(np.float64, N).copy()).to(cuda_device)
    lp_inf = torch.from_numpy(take(np.float64, N).copy()).to(cuda_device)
    c_stats = take(np.float64, 8)
    c_gw = take(np.float32, V * d).reshape(V, d)
    assert off == len(raw)
    b = PackedBatch(tokens, lp_old, lp_inf, torch.arange(0, N + 1, N // S, dtype=torch.int32, device=cuda_device),
                    torch.tensor([0, 2, 4], dtype=torch.int32, device=cuda_device), None,
                    torch.tensor([1.0, 0.0, 0.0, 1.0], dtype=torch.float64, device=cuda_device))
    f = icepop_fwd(H, W, b, IcePopConfig(), store_probs=True)
    _, gw = icepop_bwd(H, W, b, f, IcePopConfig(), grad_scale=-1.0)
    assert np.array_equal(f.stats.cpu().numpy(), c_stats)
    assert np.array_equal(gw.cpu().numpy(), c_gw)
    assert c_stats[2] == N and np.abs(c_gw).sum() > 0
