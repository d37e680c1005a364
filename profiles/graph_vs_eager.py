"""Is the bench step host-bound anywhere? Time the C2 stored-probabilities step eagerly and
as a CUDA-graph replay (the step is sync-free and capturable), interleaved on one box.

    python profiles/graph_vs_eager.py [--rounds 3] [--steps 4] [--config c2]
"""
import argparse
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import bench  # noqa: E402
from paper_2510_18855_b200.loss import IcePopConfig, icepop_bwd, icepop_fwd  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--rounds", type=int, default=3)
    ap.add_argument("--steps", type=int, default=4)
    ap.add_argument("--config", default="c2", choices=sorted(bench.CONFIGS))
    a = ap.parse_args()
    dev = torch.device("cuda", 0)
    cfg = bench.CONFIGS[a.config]
    meta = bench.make_batch_host(cfg, 0, 1)
    H, W, batch, _ = bench.build_device_inputs(cfg, meta, dev, 0)
    icfg = IcePopConfig()
    out = {}

    def step():
        f = icepop_fwd(H, W, batch, icfg, layout="vd", store_probs=True)
        _, g = icepop_bwd(H, W, batch, f, icfg, layout="vd", grad_scale=-1.0)
        out["f"], out["g"] = f, g

    for _ in range(2):
        step()
    torch.cuda.synchronize()
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s):
        step()
    torch.cuda.current_stream().wait_stream(s)
    torch.cuda.synchronize()
    graph = torch.cuda.CUDAGraph()
    with torch.cuda.graph(graph):
        step()
    torch.cuda.synchronize()

    def timed(fn):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(a.steps):
            fn()
        e1.record()
        torch.cuda.synchronize()
        return e0.elapsed_time(e1) / a.steps

    for r in range(a.rounds):
        te = timed(step)
        tg = timed(graph.replay)
        print(f"round {r}: eager {te:.2f} ms/step  graph {tg:.2f} ms/step  ({(te - tg) / te * 100:+.2f}%)", flush=True)


if __name__ == "__main__":
    main()
