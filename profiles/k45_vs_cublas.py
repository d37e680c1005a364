"""The backward's long-K GEMMs at their C2 shapes (per 32,768-token slice) against cuBLAS,
each sustained for a few seconds under the power cap:
  K4  dH = P . W        [N x V] . [V x d]   (K = V = 157,184)
  K5  dW = P^T . H      [V x N] . [N x d]   (K = N tokens)
This library: icepop_gemm_bf16 (the same long-K kernels K4/K5 run: 256 x 512 CTA-pair tiles in
static waves), fp32 output; cuBLAS: torch.matmul, bf16 output (its fp32-output path is slower).

    python profiles/k45_vs_cublas.py [--tokens 32768] [--seconds 4]
"""

from __future__ import annotations

import argparse
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))

from k1_vs_cublas import sustained  # noqa: E402

from paper_2510_18855_b200 import _lib  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--tokens", type=int, default=32768)
    ap.add_argument("--hidden", type=int, default=4096)
    ap.add_argument("--vocab", type=int, default=157184)
    ap.add_argument("--seconds", type=float, default=4.0)
    ap.add_argument("--ncu", choices=["k4", "k5"], default=None, help="launch one GEMM twice (for ncu -s 1 -c 1)")
    a = ap.parse_args()
    dev = torch.device("cuda", 0)
    N, d, V = a.tokens, a.hidden, a.vocab
    g = torch.Generator(device=dev).manual_seed(0)
    P = (torch.rand(N, V, device=dev, generator=g) * 1e-4).to(torch.bfloat16)
    W = (torch.randn(V, d, device=dev, generator=g) * (2.0 / d ** 0.5)).to(torch.bfloat16)
    H = torch.randn(N, d, device=dev, generator=g).to(torch.bfloat16)
    dH16 = torch.empty(N, d, device=dev, dtype=torch.bfloat16)
    dW16 = torch.empty(V, d, device=dev, dtype=torch.bfloat16)
    dH = torch.empty(N, d, device=dev, dtype=torch.float32)
    dW = torch.empty(V, d, device=dev, dtype=torch.float32)
    flop = 2.0 * N * d * V
    lib = _lib.ensure_device(0)
    st = torch.cuda.current_stream().cuda_stream
    if a.ncu:
        for _ in range(2):
            if a.ncu == "k4":
                _lib.check(lib.icepop_gemm_bf16(P.data_ptr(), W.data_ptr(), dH.data_ptr(), N, d, V, 0, 1, 1, 0, st))
            else:
                _lib.check(lib.icepop_gemm_bf16(P.data_ptr(), H.data_ptr(), dW.data_ptr(), V, d, N, 1, 1, 1, 0, st))
        torch.cuda.synchronize()
        return
    for _ in range(2):
        sustained("cuBLAS  K4 shape P W -> bf16", lambda: torch.matmul(P, W, out=dH16), flop, a.seconds)
        sustained("icepop  K4 shape P W -> f32", lambda: _lib.check(lib.icepop_gemm_bf16(
            P.data_ptr(), W.data_ptr(), dH.data_ptr(), N, d, V, 0, 1, 1, 0, st)), flop, a.seconds)
        sustained("cuBLAS  K5 shape P^T H -> bf16", lambda: torch.matmul(P.T, H, out=dW16), flop, a.seconds)
        sustained("icepop  K5 shape P^T H -> f32", lambda: _lib.check(lib.icepop_gemm_bf16(
            P.data_ptr(), H.data_ptr(), dW.data_ptr(), V, d, N, 1, 1, 1, 0, st)), flop, a.seconds)
    torch.cuda.synchronize()
    ref = torch.matmul(P[:256].float(), W.float())
    err = ((dH[:256] - ref).norm() / ref.norm()).item()
    print(f"check: K4-shape rel err vs fp32 matmul {err:.2e}")


if __name__ == "__main__":
    main()
