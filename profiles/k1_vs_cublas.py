"""K1's shape as a plain GEMM: cuBLAS (torch.matmul, bf16 out) vs this library's plain GEMM
(icepop_gemm_bf16, bf16 out) vs K1 itself (fused softmax statistics + stored probabilities),
each run back to back for a few seconds (sustained, under the power cap), with the SM clock.

    python profiles/k1_vs_cublas.py [--tokens 32768] [--seconds 4]
"""

from __future__ import annotations

import argparse
import sys
import time
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))

from paper_2510_18855_b200 import _lib  # noqa: E402
from paper_2510_18855_b200.loss import IcePopConfig, PackedBatch, icepop_fwd  # noqa: E402


def clock_mhz():
    try:
        import pynvml

        pynvml.nvmlInit()
        h = pynvml.nvmlDeviceGetHandleByIndex(0)
        return pynvml.nvmlDeviceGetClockInfo(h, pynvml.NVML_CLOCK_SM), pynvml.nvmlDeviceGetPowerUsage(h) / 1000
    except Exception:  # noqa: BLE001
        return -1, -1


def sustained(name, fn, flop, seconds):
    fn()
    torch.cuda.synchronize()
    t0 = time.time()
    n = 0
    while time.time() - t0 < seconds / 2:  # reach the power-capped steady state first
        fn()
        n += 1
        torch.cuda.synchronize()
    reps = max(2, n)
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for i in range(reps):
        fn()
        if i == reps // 2:
            mhz, w = clock_mhz()
    b.record()
    torch.cuda.synchronize()
    ms = a.elapsed_time(b) / reps
    print(f"{name:34s} {ms:8.3f} ms {flop / ms / 1e9:8.1f} TFLOP/s  sm {mhz} MHz  {w:.0f} W", flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--tokens", type=int, default=32768)
    ap.add_argument("--hidden", type=int, default=4096)
    ap.add_argument("--vocab", type=int, default=157184)
    ap.add_argument("--seconds", type=float, default=4.0)
    a = ap.parse_args()
    dev = torch.device("cuda", 0)
    N, d, V = a.tokens, a.hidden, a.vocab
    g = torch.Generator(device=dev).manual_seed(0)
    H = torch.randn(N, d, device=dev, generator=g).to(torch.bfloat16)
    W = (torch.randn(V, d, device=dev, generator=g) * (2.0 / d ** 0.5)).to(torch.bfloat16)
    C = torch.empty(N, V, device=dev, dtype=torch.bfloat16)
    flop = 2.0 * N * d * V
    lib = _lib.ensure_device(0)
    st = torch.cuda.current_stream().cuda_stream
    tokens = torch.randint(0, V, (N,), device=dev, generator=g, dtype=torch.int32)
    T = 4096 if N % 4096 == 0 else N
    S = N // T
    batch = PackedBatch(tokens, torch.full((N,), -12.0, dtype=torch.float64, device=dev),
                        torch.full((N,), -12.0, dtype=torch.float64, device=dev),
                        torch.arange(0, N + 1, T, dtype=torch.int32, device=dev),
                        torch.tensor([0, S], dtype=torch.int32, device=dev),
                        torch.linspace(-1, 1, S, dtype=torch.float64, device=dev))
    for _ in range(2):
        sustained("cuBLAS  H W^T -> bf16", lambda: torch.matmul(H, W.T, out=C), flop, a.seconds)
        sustained("icepop  plain GEMM -> bf16", lambda: _lib.check(lib.icepop_gemm_bf16(
            H.data_ptr(), W.data_ptr(), C.data_ptr(), N, V, d, 0, 0, 0, 0, st)), flop, a.seconds)
        sustained("icepop  K1 + K2 (stored probs)", lambda: icepop_fwd(H, W, batch, IcePopConfig(), layout="vd",
                                                                      store_probs=True), flop, a.seconds)
        sustained("icepop  K1 + K2 (statistics only)", lambda: icepop_fwd(H, W, batch, IcePopConfig(), layout="vd",
                                                                         store_probs=False), flop, a.seconds)


if __name__ == "__main__":
    main()
