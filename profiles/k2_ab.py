"""Time the K2 epilogue alone (icepop_epilogue over a kept K1 workspace) at C2, device time only.

    ICEPOP_B200_LIB=path/to/lib.so python profiles/k2_ab.py [--tokens 262144]

A ~5 ms device spin ahead of the start event lets the host enqueue every rep first.
"""

from __future__ import annotations

import argparse
import os
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))

from paper_2510_18855_b200.loss import IcePopConfig, PackedBatch, icepop_epilogue, icepop_fwd  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--tokens", type=int, default=262144)
    ap.add_argument("--hidden", type=int, default=4096)
    ap.add_argument("--vocab", type=int, default=157184)
    ap.add_argument("--reps", type=int, default=20)
    a = ap.parse_args()
    dev = torch.device("cuda", 0)
    N, d, V = a.tokens, a.hidden, a.vocab
    g = torch.Generator(device=dev).manual_seed(0)
    H = torch.randn(N, d, device=dev, generator=g).to(torch.bfloat16)
    W = (torch.randn(V, d, device=dev, generator=g) * (2.0 / d ** 0.5)).to(torch.bfloat16)
    tokens = torch.randint(0, V, (N,), device=dev, generator=g, dtype=torch.int32)
    T = 4096 if N % 4096 == 0 else N
    S = N // T
    batch = PackedBatch(tokens, torch.full((N,), -12.0, dtype=torch.float64, device=dev),
                        torch.full((N,), -12.0, dtype=torch.float64, device=dev),
                        torch.arange(0, N + 1, T, dtype=torch.int32, device=dev),
                        torch.tensor([0, S], dtype=torch.int32, device=dev),
                        torch.linspace(-1, 1, S, dtype=torch.float64, device=dev))
    cfg = IcePopConfig()
    f = icepop_fwd(H, W, batch, cfg, layout="vd", store_probs=False, keep_workspace=True)
    for _ in range(3):
        icepop_epilogue(batch, f, cfg)
    torch.cuda.synchronize()
    res = []
    for _ in range(3):
        a0, a1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda._sleep(8_000_000)
        a0.record()
        for _ in range(a.reps):
            icepop_epilogue(batch, f, cfg)
        a1.record()
        torch.cuda.synchronize()
        res.append(a0.elapsed_time(a1) / a.reps)
    print(f"{os.environ.get('ICEPOP_B200_LIB', 'in-tree')}: K2 epilogue {min(res):.4f} ms (runs {res})")


if __name__ == "__main__":
    main()
