"""Launch each IcePop kernel of a step once at a C2-shaped problem, for ncu.

    python profiles/profile_kernels.py [--tokens 16384] [--mode probs|recompute]
    ncu --set full -k regex:"umma_gemm|k_dz_probs" -s 4 -c 4 -o prof python profiles/profile_kernels.py

All four are launched once as warm-up (skipped by `-s 4`), then once each for profiling.
Order: K1 (fwd LSE; with --mode probs it also stores the bf16 probabilities), the dZ
producer (recompute: the K3 GEMM; probs: the in-place k_dz_probs pass), K4 (dHidden),
K5 (dWeight).
"""

from __future__ import annotations

import argparse
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))

from paper_2510_18855_b200 import _lib  # noqa: E402
from paper_2510_18855_b200.loss import IcePopConfig, PackedBatch, icepop_fwd  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--tokens", type=int, default=16384)
    ap.add_argument("--hidden", type=int, default=4096)
    ap.add_argument("--vocab", type=int, default=157184)
    ap.add_argument("--mode", choices=["probs", "recompute"], default="probs")
    a = ap.parse_args()
    sp = a.mode == "probs"
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
    lib = _lib.ensure_device(0)
    st = torch.cuda.current_stream().cuda_stream
    dz = None if sp else torch.empty((N, V), dtype=torch.bfloat16, device=dev)
    gh = torch.empty((N, d), dtype=torch.bfloat16, device=dev)
    gw = torch.zeros((V, d), dtype=torch.float32, device=dev)
    shape = _lib.Shape(n_tokens=N, token_offset=0, hidden=d, vocab=V, n_seqs=S, n_groups=1, weight_layout=_lib.W_VD)
    holder = {}

    def k1():
        holder.clear()  # the previous forward's probabilities are released first
        holder["f"] = icepop_fwd(H, W, batch, IcePopConfig(), layout="vd", store_probs=sp)
        if sp:
            holder["dz"] = holder["f"].extras["probs"]

    def k3():
        f = holder["f"]
        saved = _lib.Saved(tokens=tokens.data_ptr(), lse=f.lse.data_ptr(), coeff=f.coeff.data_ptr())
        if sp:  # the stored-probabilities backward with null gradients = the dZ pass alone
            saved.probs, saved.tile_max = f.extras["probs"].data_ptr(), f.extras["tile_max"].data_ptr()
            saved.lp_cur = f.lp_cur.data_ptr()
            _lib.check(lib.icepop_bwd_bf16(shape, IcePopConfig().to_c(), H.data_ptr(), W.data_ptr(), None, saved,
                                           -1.0, None, 0, None, 0, None, 0, st))
        else:
            _lib.check(lib.icepop_dz_bf16(shape, 1.0, H.data_ptr(), W.data_ptr(), None, saved, -1.0, dz.data_ptr(),
                                          V, st))

    def zbuf():
        return holder["dz"] if sp else dz

    def k4():
        _lib.check(lib.icepop_gemm_bf16(zbuf().data_ptr(), W.data_ptr(), gh.data_ptr(), N, d, V, 0, 1, 0, 0, st))

    # K5 as in the step: the stored-probabilities backward reads the hidden rows transposed
    # (K-major, written by its prep kernel); the recompute mode transposes each dZ chunk's rows
    HT = H.t().contiguous()

    def k5():
        _lib.check(lib.icepop_gemm_bf16(zbuf().data_ptr(), HT.data_ptr(), gw.data_ptr(), V, d, N, 1, 0, 1, 1, st))

    kernels = (("K1", k1), ("dZ" if sp else "K3", k3), ("K4", k4), ("K5", k5))
    for _, fn in kernels:  # warm-ups first, so `ncu -s 4 -c 4` sees K1, K3, K4, K5 in order
        fn()
    torch.cuda.synchronize()
    for name, fn in kernels:
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        fn()
        e1.record()
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1)
        if name == "dZ":
            print(f"{name}: {ms:.3f} ms  {4.0 * N * V / ms / 1e6:.1f} GB/s (read + write bf16)", flush=True)
        else:
            print(f"{name}: {ms:.3f} ms  {2.0 * N * d * V / ms / 1e9:.1f} TFLOP/s", flush=True)


if __name__ == "__main__":
    main()
