"""A/B of K1's run length (icepop_set_k1_run) at C2 on one box: the forward (K1 + K2) with
stored probabilities, interleaved repetitions per setting, median ms and TFLOP/s."""
import statistics
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2510_18855_b200 import _lib  # noqa: E402
from paper_2510_18855_b200.loss import IcePopConfig, PackedBatch, icepop_fwd  # noqa: E402

N, d, V = int(sys.argv[1]) if len(sys.argv) > 1 else 262144, 4096, 157184
runs = [int(x) for x in sys.argv[2].split(",")] if len(sys.argv) > 2 else [1, 4, 16]
dev = torch.device("cuda", 0)
lib = _lib.ensure_device(0)
g = torch.Generator(device=dev).manual_seed(0)
H = torch.randn(N, d, device=dev, generator=g).to(torch.bfloat16)
W = (torch.randn(V, d, device=dev, generator=g) * (2.0 / d ** 0.5)).to(torch.bfloat16)
tokens = torch.randint(0, V, (N,), device=dev, generator=g, dtype=torch.int32)
S = N // 4096
b = PackedBatch(tokens, torch.full((N,), -12.0, dtype=torch.float64, device=dev),
                torch.full((N,), -12.0, dtype=torch.float64, device=dev),
                torch.arange(0, N + 1, 4096, dtype=torch.int32, device=dev),
                torch.tensor([0, S], dtype=torch.int32, device=dev), torch.linspace(-1, 1, S, dtype=torch.float64,
                                                                                   device=dev))
probs = torch.empty((N, V), dtype=torch.bfloat16, device=dev)
tm = torch.empty((N, _lib.tile_max_ld(V)), dtype=torch.float32, device=dev)
res = {r: [] for r in runs}
for rep in range(4):
    for r in runs:
        _lib.check(lib.icepop_set_k1_run(r))
        icepop_fwd(H, W, b, IcePopConfig(), layout="vd", probs_buffers=(probs, tm))
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        icepop_fwd(H, W, b, IcePopConfig(), layout="vd", probs_buffers=(probs, tm))
        e1.record()
        torch.cuda.synchronize()
        res[r].append(e0.elapsed_time(e1))
for r in runs:
    ms = statistics.median(res[r])
    print(f"run {r:2d}: {ms:.2f} ms  {2.0 * N * d * V / ms / 1e9:.1f} TFLOP/s  all {[round(x, 1) for x in res[r]]}",
          flush=True)
_lib.check(lib.icepop_set_k1_run(0))
