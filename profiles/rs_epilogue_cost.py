"""Cost of the fused dW reduce-scatter epilogue (icepop_bwd_bf16_rs) on one B200.

Rank 0 of an emulated N-rank job runs its C3 shard (32,768 tokens, d = 8,192, V = 157,184)
with K5's epilogue routing every dW row to its owner's slot. The N slot buffers live in this
GPU's memory, so the stores go to local HBM instead of NVLink peers: this measures the
epilogue's routing cost, not the link. Compared with the plain backward (dW stored locally),
interleaved, CUDA events on the launching stream; plus the owner's ordered fold.

    python profiles/rs_epilogue_cost.py [--world 8] [--reps 4]
"""
import argparse
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import bench  # noqa: E402
from paper_2510_18855_b200 import _lib  # noqa: E402
from paper_2510_18855_b200.loss import IcePopConfig, icepop_bwd, icepop_bwd_reduce_scatter, icepop_fwd  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--world", type=int, default=8)
    ap.add_argument("--reps", type=int, default=4)
    ap.add_argument("--config", default="c3", choices=sorted(bench.CONFIGS))
    a = ap.parse_args()
    dev = torch.device("cuda", 0)
    cfg = bench.CONFIGS[a.config]
    meta = bench.make_batch_host(cfg, 0, 1)
    H, W, batch, _ = bench.build_device_inputs(cfg, meta, dev, 0)
    icfg = IcePopConfig()
    V, d = W.shape
    world = a.world
    shard_rows = -(-V // world)
    shard_elems = shard_rows * d
    slots = [torch.empty(world * shard_elems, dtype=torch.float32, device=dev) for _ in range(world)]
    target = _lib.RsTarget(world=world, rank=0, shard_rows=shard_rows)
    for o in range(world):
        target.slots[o] = slots[o].data_ptr()
    out = torch.empty(shard_elems, dtype=torch.float32, device=dev)
    lib = _lib.ensure_device(0)
    st = torch.cuda.current_stream()

    def plain():
        f = icepop_fwd(H, W, batch, icfg, layout="vd", store_probs=True)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        icepop_bwd(H, W, batch, f, icfg, layout="vd", grad_scale=-1.0)
        e1.record()
        return e0, e1

    def fused():
        f = icepop_fwd(H, W, batch, icfg, layout="vd", store_probs=True)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        icepop_bwd_reduce_scatter(H, W, batch, f, target, icfg, layout="vd", grad_scale=-1.0)
        e1.record()
        return e0, e1

    def fold():
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        _lib.check(lib.icepop_rs_fold(slots[0].data_ptr(), world, shard_elems, out.data_ptr(), st.cuda_stream))
        e1.record()
        return e0, e1

    for fn in (plain, fused, fold):
        fn()
    torch.cuda.synchronize()
    res = {"plain": [], "fused": [], "fold": []}
    for _ in range(a.reps):
        for name, fn in (("plain", plain), ("fused", fused), ("fold", fold)):
            e0, e1 = fn()
            torch.cuda.synchronize()
            res[name].append(e0.elapsed_time(e1))
    med = {k: sorted(v)[len(v) // 2] for k, v in res.items()}
    n = H.shape[0]
    dw_bytes = V * d * 4
    print(f"{a.config} rank shard: {n} tokens, d={d}, V={V}, emulated world {world}")
    print(f"backward, dW stored locally : {med['plain']:.2f} ms  (all: {[round(x, 2) for x in res['plain']]})")
    print(f"backward, fused reduce-scatter: {med['fused']:.2f} ms  (all: {[round(x, 2) for x in res['fused']]})"
          f"  -> {100 * (med['fused'] / med['plain'] - 1):+.2f}%")
    print(f"owner fold of {world} slots ({shard_elems * 4 * world / 1e9:.2f} GB read): {med['fold']:.3f} ms")
    peer = dw_bytes * (world - 1) / world
    print(f"NVLink bytes this rank sends per step: {peer / 1e9:.2f} GB; over the backward that is "
          f"{peer / (med['fused'] / 1e3) / 1e9:.0f} GB/s against ~900 GB/s per direction (NVLink 5)")


if __name__ == "__main__":
    main()
