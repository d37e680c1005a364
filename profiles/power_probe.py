"""Sustained clock / power / throughput of each GEMM kind under the 1 kW cap.

Runs every kernel back to back for ~`--seconds` while sampling nvidia-smi, so kernels can
be compared by energy per FLOP on the same box (cuBLAS as the yardstick).

    python profiles/power_probe.py [--seconds 4] [--tokens 65536]
"""
import argparse
import subprocess
import sys
import threading
import time
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2510_18855_b200 import _lib  # noqa: E402
from paper_2510_18855_b200.loss import IcePopConfig, PackedBatch, icepop_fwd  # noqa: E402


def sample(stop, rows):
    p = subprocess.Popen(["nvidia-smi", "-i", "0", "--query-gpu=clocks.sm,power.draw", "--format=csv,noheader,nounits",
                          "-lms", "100"], stdout=subprocess.PIPE, text=True)
    while not stop.is_set():
        line = p.stdout.readline()
        if line:
            rows.append([float(x) for x in line.split(",")])
    p.terminate()


def run(name, fn, flop, seconds):
    fn()
    torch.cuda.synchronize()
    rows, stop = [], threading.Event()
    th = threading.Thread(target=sample, args=(stop, rows), daemon=True)
    th.start()
    time.sleep(0.2)
    t0 = time.time()
    n = 0
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    while time.time() - t0 < seconds:
        fn()
        n += 1
        if n % 4 == 0:
            torch.cuda.synchronize()
    b.record()
    torch.cuda.synchronize()
    stop.set()
    th.join(timeout=3)
    ms = a.elapsed_time(b) / n
    r = np.asarray(rows[len(rows) // 4:]) if rows else np.zeros((1, 2))
    print(f"{name:28s} {flop / ms / 1e9:8.1f} TFLOP/s  sm {np.median(r[:, 0]):6.0f} MHz  "
          f"power {np.median(r[:, 1]):6.0f} W  TFLOP/J {flop / ms / 1e9 / max(np.median(r[:, 1]), 1):.3f}", flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--seconds", type=float, default=4.0)
    ap.add_argument("--tokens", type=int, default=65536)
    ap.add_argument("--fused-only", action="store_true")
    ap.add_argument("--cgs", default="1,2")
    ap.add_argument("--majors", action="store_true", help="also K4's shape with an MN-major A operand")
    ap.add_argument("--only", default="", help="comma list of kernel names to run (K1,K1p,K3,K4,K5)")
    a = ap.parse_args()
    cgs = [int(x) for x in a.cgs.split(",")]
    dev = torch.device("cuda", 0)
    lib = _lib.ensure_device(0)
    st = torch.cuda.current_stream().cuda_stream
    n = 8192
    A = torch.randn(n, n, device=dev).to(torch.bfloat16)
    B = torch.randn(n, n, device=dev).to(torch.bfloat16)
    C = torch.empty(n, n, device=dev, dtype=torch.bfloat16)
    if not a.fused_only:
        run("cublas 8192^3", lambda: torch.matmul(A, B.T, out=C), 2.0 * n ** 3, a.seconds)
    for cg in ([] if a.fused_only else cgs):
        _lib.check(lib.icepop_set_cta_group(cg))
        run(f"icepop gemm 8192^3 cta{cg}", lambda: _lib.check(lib.icepop_gemm_bf16(
            A.data_ptr(), B.data_ptr(), C.data_ptr(), n, n, n, 0, 0, 0, 0, st)), 2.0 * n ** 3, a.seconds)
    del A, B, C
    N, d, V = a.tokens, 4096, 157184
    g = torch.Generator(device=dev).manual_seed(0)
    H = torch.randn(N, d, device=dev, generator=g).to(torch.bfloat16)
    W = (torch.randn(V, d, device=dev, generator=g) * (2.0 / d ** 0.5)).to(torch.bfloat16)
    tokens = torch.randint(0, V, (N,), device=dev, generator=g, dtype=torch.int32)
    S = N // 4096
    batch = PackedBatch(tokens, torch.full((N,), -12.0, dtype=torch.float64, device=dev),
                        torch.full((N,), -12.0, dtype=torch.float64, device=dev),
                        torch.arange(0, N + 1, 4096, dtype=torch.int32, device=dev),
                        torch.tensor([0, S], dtype=torch.int32, device=dev),
                        torch.linspace(-1, 1, S, dtype=torch.float64, device=dev))
    dz = torch.empty((N, V), dtype=torch.bfloat16, device=dev)
    gh = torch.empty((N, d), dtype=torch.bfloat16, device=dev)
    gw = torch.zeros((V, d), dtype=torch.float32, device=dev)
    shape = _lib.Shape(n_tokens=N, token_offset=0, hidden=d, vocab=V, n_seqs=S, n_groups=1, weight_layout=_lib.W_VD)
    flop = 2.0 * N * d * V
    only = set(x for x in a.only.split(",") if x)

    def want(k):
        return not only or k in only

    for cg in cgs:
        _lib.check(lib.icepop_set_cta_group(cg))
        f = icepop_fwd(H, W, batch, IcePopConfig(), layout="vd", store_probs=False)
        if want("K1"):
            run(f"K1 fwd cta{cg}", lambda: icepop_fwd(H, W, batch, IcePopConfig(), layout="vd", store_probs=False),
                flop, a.seconds)
        if want("K1p"):
            del dz  # the stored probabilities take its place
            run(f"K1 fwd+probs cta{cg}", lambda: icepop_fwd(H, W, batch, IcePopConfig(), layout="vd",
                                                            store_probs=True), flop, a.seconds)
            dz = torch.empty((N, V), dtype=torch.bfloat16, device=dev)
        if want("K3"):
            run(f"K3 dz cta{cg}", lambda: _lib.check(lib.icepop_dz_bf16(
                shape, 1.0, H.data_ptr(), W.data_ptr(), None, _lib.Saved(tokens=tokens.data_ptr(),
                lse=f.lse.data_ptr(), coeff=f.coeff.data_ptr()), -1.0, dz.data_ptr(), V, st)), flop, a.seconds)
        if want("K4"):
            run(f"K4 dhidden cta{cg}", lambda: _lib.check(lib.icepop_gemm_bf16(
                dz.data_ptr(), W.data_ptr(), gh.data_ptr(), N, d, V, 0, 1, 0, 0, st)), flop, a.seconds)
        if want("K5"):
            run(f"K5 dweight cta{cg}", lambda: _lib.check(lib.icepop_gemm_bf16(
                dz.data_ptr(), H.data_ptr(), gw.data_ptr(), V, d, N, 1, 1, 0, 0, st)), flop, a.seconds)
        if a.majors:  # same GEMM as K4 with A stored [K, M] (dZ^T): the cost of an MN-major A
            dzt = dz.t().contiguous()
            run(f"K4 shape, A MN-major cta{cg}", lambda: _lib.check(lib.icepop_gemm_bf16(
                dzt.data_ptr(), W.data_ptr(), gh.data_ptr(), N, d, V, 1, 1, 0, 0, st)), flop, a.seconds)
            del dzt


if __name__ == "__main__":
    main()
