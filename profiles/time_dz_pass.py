"""Time the stored-probabilities dZ pass at C2 shape: alone (no workspace) vs with the
block-list kernels of the block-sparse K4/K5 (workspace given), for a chosen fraction of
zero-coefficient rows.

    python profiles/time_dz_pass.py [--tokens 262144] [--inactive 0.016]
"""
import argparse
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2510_18855_b200 import _lib  # noqa: E402
from paper_2510_18855_b200.loss import IcePopConfig  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--tokens", type=int, default=262144)
    ap.add_argument("--hidden", type=int, default=4096)
    ap.add_argument("--vocab", type=int, default=157184)
    ap.add_argument("--inactive", type=float, default=0.016)
    ap.add_argument("--reps", type=int, default=5)
    a = ap.parse_args()
    dev = torch.device("cuda", 0)
    N, d, V = a.tokens, a.hidden, a.vocab
    lib = _lib.ensure_device(0)
    g = torch.Generator(device=dev).manual_seed(0)
    probs = torch.empty((N, V), dtype=torch.bfloat16, device=dev)
    for i in range(0, N, 4096):  # in row chunks: an fp32 [N, V] temporary would not fit
        probs[i:i + 4096] = torch.rand((min(4096, N - i), V), device=dev, generator=g)
    tm = torch.zeros((N, _lib.tile_max_ld(V)), device=dev)
    lse = torch.full((N,), 12.0, device=dev)
    coeff = torch.randn(N, device=dev, generator=g) * 1e-4
    coeff[torch.rand(N, device=dev, generator=g) < a.inactive] = 0.0
    tokens = torch.randint(0, V, (N,), device=dev, generator=g, dtype=torch.int32)
    lp_cur = torch.full((N,), -3.0, dtype=torch.float64, device=dev)
    H = torch.zeros((N, d), dtype=torch.bfloat16, device=dev)
    W = torch.zeros((V, d), dtype=torch.bfloat16, device=dev)
    shape = _lib.Shape(n_tokens=N, token_offset=0, hidden=d, vocab=V, n_seqs=1, n_groups=1, weight_layout=_lib.W_VD)
    b = _lib._sz()
    _lib.check(lib.icepop_workspace_bytes(shape, -1, 0, None, b))
    ws = torch.empty(b.value, dtype=torch.uint8, device=dev)
    saved = _lib.Saved(tokens=tokens.data_ptr(), lse=lse.data_ptr(), coeff=coeff.data_ptr(), probs=probs.data_ptr(),
                       tile_max=tm.data_ptr(), lp_cur=lp_cur.data_ptr())
    st = torch.cuda.current_stream().cuda_stream
    active = int((coeff != 0).sum())
    for name, w in (("dZ pass", None), ("dZ pass + block lists", ws)):
        def run():
            _lib.check(lib.icepop_bwd_bf16(shape, IcePopConfig().to_c(), H.data_ptr(), W.data_ptr(), None, saved,
                                           -1.0, None, 0, None, 0, _lib.ptr(w), 0 if w is None else w.numel(), st))
        run()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(a.reps):
            run()
        e1.record()
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / a.reps
        nbytes = 4 * active * V + 2 * (N - active) * V
        print(f"{name:22s} {ms:8.3f} ms  {nbytes / ms / 1e6:8.1f} GB/s algorithmic  (active {active}/{N})", flush=True)


if __name__ == "__main__":
    main()
