"""Operand major-ness A/B of the long-K GEMMs at K4 / K5 shapes (32,768-token slice), sustained:
every combination of K-major / MN-major A and B (transposed copies of the operands), reporting
TFLOP/s, SM clock and TFLOP/s per GHz (the power cap moves the clock, so per-clock rate compares
the kernels' efficiency).

    python profiles/major_ab.py [--tokens 32768] [--seconds 3]
"""

from __future__ import annotations

import argparse
import sys
import time
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))

from paper_2510_18855_b200 import _lib  # noqa: E402


def clock():
    import pynvml

    pynvml.nvmlInit()
    h = pynvml.nvmlDeviceGetHandleByIndex(0)
    return pynvml.nvmlDeviceGetClockInfo(h, pynvml.NVML_CLOCK_SM)


def sustained(fn, flop, seconds):
    fn()
    torch.cuda.synchronize()
    t0 = time.time()
    while time.time() - t0 < seconds / 2:
        fn()
        torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    reps = 6
    mhz = []
    a.record()
    for _ in range(reps):
        fn()
        mhz.append(clock())
    b.record()
    torch.cuda.synchronize()
    ms = a.elapsed_time(b) / reps
    return ms, flop / ms / 1e9, sorted(mhz)[len(mhz) // 2]


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--tokens", type=int, default=32768)
    ap.add_argument("--hidden", type=int, default=4096)
    ap.add_argument("--vocab", type=int, default=157184)
    ap.add_argument("--seconds", type=float, default=3.0)
    a = ap.parse_args()
    dev = torch.device("cuda", 0)
    N, d, V = a.tokens, a.hidden, a.vocab
    g = torch.Generator(device=dev).manual_seed(0)
    P = (torch.rand(N, V, device=dev, generator=g) * 1e-4).to(torch.bfloat16)
    PT = P.t().contiguous()
    W = (torch.randn(V, d, device=dev, generator=g) * (2.0 / d ** 0.5)).to(torch.bfloat16)
    WT = W.t().contiguous()
    H = torch.randn(N, d, device=dev, generator=g).to(torch.bfloat16)
    HT = H.t().contiguous()
    lib = _lib.ensure_device(0)
    st = torch.cuda.current_stream().cuda_stream
    flop = 2.0 * N * d * V
    dH = torch.empty(N, d, device=dev, dtype=torch.float32)
    dW = torch.empty(V, d, device=dev, dtype=torch.float32)
    cases = [
        # name, A, B, C, M, Ncols, K, a_mn, b_mn
        ("K4 A=P(K-major)  B=W(MN-major)", P, W, dH, N, d, V, 0, 1),
        ("K4 A=P(K-major)  B=W^T(K-major)", P, WT, dH, N, d, V, 0, 0),
        ("K4 A=P^T(MN-major) B=W(MN-major)", PT, W, dH, N, d, V, 1, 1),
        ("K4 A=P^T(MN-major) B=W^T(K-major)", PT, WT, dH, N, d, V, 1, 0),
        ("K5 A=P(MN-major) B=H(MN-major)", P, H, dW, V, d, N, 1, 1),
        ("K5 A=P(MN-major) B=H^T(K-major)", P, HT, dW, V, d, N, 1, 0),
        ("K5 A=P^T(K-major) B=H(MN-major)", PT, H, dW, V, d, N, 0, 1),
        ("K5 A=P^T(K-major) B=H^T(K-major)", PT, HT, dW, V, d, N, 0, 0),
    ]
    for rnd in range(2):
        for name, A, B, C, M, Nc, K, am, bm in cases:
            ms, tf, mhz = sustained(lambda: _lib.check(lib.icepop_gemm_bf16(A.data_ptr(), B.data_ptr(), C.data_ptr(), M, Nc,
                                                                            K, am, bm, 1, 0, st)), flop, a.seconds)
            print(f"round {rnd} {name:36s} {ms:8.3f} ms {tf:8.1f} TFLOP/s  {mhz} MHz  {tf / mhz * 1000:7.1f} TFLOP/s/GHz",
                  flush=True)


if __name__ == "__main__":
    main()
