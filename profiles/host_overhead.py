"""Where does the C1 e2e step (pinned host inputs) lose time against the device-resident step?

Times at one config, on one box:
  * the device-resident step (CUDA events),
  * the host issue time of one step (wall clock of the Python calls, GPU queue not full),
  * bench.run_e2e as shipped,
and prints a cProfile of the host side of 50 resident steps (top functions by own time).

    python profiles/host_overhead.py [--config c1] [--steps 50]
"""
import argparse
import cProfile
import io
import pstats
import sys
import time
from pathlib import Path
from types import SimpleNamespace

import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import bench  # noqa: E402
from paper_2510_18855_b200.loss import IcePopConfig, icepop_bwd, icepop_fwd  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="c1", choices=sorted(bench.CONFIGS))
    ap.add_argument("--steps", type=int, default=50)
    a = ap.parse_args()
    dev = torch.device("cuda", 0)
    cfg = bench.CONFIGS[a.config]
    meta = bench.make_batch_host(cfg, 0, 1)
    H, W, batch, _ = bench.build_device_inputs(cfg, meta, dev, 0)
    icfg = IcePopConfig()

    def step():
        f = icepop_fwd(H, W, batch, icfg, layout="vd", store_probs=True)
        _, g = icepop_bwd(H, W, batch, f, icfg, layout="vd", grad_scale=-1.0)
        return f, g

    for _ in range(5):
        step()
    torch.cuda.synchronize()

    # device-resident step time
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(a.steps):
        step()
    e1.record()
    torch.cuda.synchronize()
    dev_ms = e0.elapsed_time(e1) / a.steps

    # host issue time per step (synchronise after every step so the queue never fills)
    host = []
    for _ in range(a.steps):
        t0 = time.perf_counter()
        step()
        host.append((time.perf_counter() - t0) * 1e3)
        torch.cuda.synchronize()
    host.sort()
    print(f"{a.config}: device-resident step {dev_ms:.3f} ms; host issue per step median {host[len(host) // 2]:.3f} ms "
          f"(min {host[0]:.3f}, max {host[-1]:.3f})")

    pr = cProfile.Profile()
    pr.enable()
    for _ in range(a.steps):
        step()
    pr.disable()
    torch.cuda.synchronize()
    s = io.StringIO()
    pstats.Stats(pr, stream=s).sort_stats("tottime").print_stats(25)
    print(s.getvalue())

    args = SimpleNamespace(steps=16, no_e2e=False)
    e2e = bench.run_e2e(H, W, batch, icfg, args, dev, 1, sp=True)
    print("bench.run_e2e:", e2e)


if __name__ == "__main__":
    main()
