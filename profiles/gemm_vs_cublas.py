"""Plain bf16 GEMM: libicepop tcgen05 kernel (cta_group 1 and 2) vs torch.matmul (cuBLAS).

    python profiles/gemm_vs_cublas.py [--size 8192] [--reps 10]
"""
import argparse
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2510_18855_b200 import _lib  # noqa: E402


def bench(fn, reps):
    for _ in range(2):
        fn()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(reps):
        fn()
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) / reps


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--size", type=int, default=8192)
    ap.add_argument("--reps", type=int, default=10)
    ap.add_argument("--only", default="")
    a = ap.parse_args()
    n = a.size
    A = torch.randn(n, n, device="cuda").to(torch.bfloat16)
    B = torch.randn(n, n, device="cuda").to(torch.bfloat16)
    C = torch.empty(n, n, device="cuda", dtype=torch.bfloat16)
    lib = _lib.ensure_device(0)
    st = torch.cuda.current_stream().cuda_stream
    flop = 2.0 * n ** 3
    if not a.only or a.only == "cublas":
        ms = bench(lambda: torch.matmul(A, B.T, out=C), a.reps)
        print(f"cublas      {ms:8.3f} ms {flop / ms / 1e9:8.1f} TFLOP/s", flush=True)
    for cg in (1, 2):
        if a.only and a.only != f"cta{cg}":
            continue
        _lib.check(lib.icepop_set_cta_group(cg))
        ms = bench(lambda: _lib.check(lib.icepop_gemm_bf16(A.data_ptr(), B.data_ptr(), C.data_ptr(), n, n, n, 0, 0, 0,
                                                           0, st)), a.reps)
        print(f"icepop cta{cg} {ms:8.3f} ms {flop / ms / 1e9:8.1f} TFLOP/s", flush=True)


if __name__ == "__main__":
    main()
