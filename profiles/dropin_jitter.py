"""Per-call wall clock of the drop-in objective_and_grad at C1 (bench.py's dropin_c1 setup), 20
calls each: fresh gradient array, with / without a gc.collect() before each call, and with
grad_out; prints every call so outliers are visible.

    python profiles/dropin_jitter.py
"""
import copy
import gc
import sys
import time
from dataclasses import dataclass
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2510_18855_b200 import objective as O  # noqa: E402


@dataclass
class Task:
    prompt_id: int


@dataclass
class Rollout:
    tokens: list


@dataclass
class Params:
    weights: np.ndarray
    version_id: int = 0

    @property
    def n_features(self):
        return self.weights.shape[0]


def main():
    rng = np.random.default_rng(0)
    S, T, nf, V = 8, 512, 1024, 32768
    w = rng.normal(0.0, 0.8, (nf, V))
    task = Task(prompt_id=17)
    rollouts = []
    for _ in range(S):
        lp = rng.normal(-10.4, 0.3, T)
        inf = lp - rng.normal(0, 0.233, T)
        rollouts.append(Rollout([O.TokenRecord(int(y), float(b), float(a), float(a), 0)
                                 for y, a, b in zip(rng.integers(0, V, T), lp, inf)]))
    rewards = [float(x) for x in rng.integers(0, 2, S)]
    groups = [O.PromptGroup(task=task, rollouts=rollouts, rewards=rewards,
                            advantages=list(O.group_advantages(rewards)))]
    theta = Params(w)
    cfg, bounds = O.ObjectiveConfig(), O.MaskingBounds()
    buf = np.empty_like(w)
    for name, kw, collect in (("fresh", {}, False), ("fresh+gc.collect", {}, True), ("grad_out", {"grad_out": buf}, False)):
        for _ in range(2):
            O.objective_and_grad(copy.deepcopy(groups), theta, theta, None, cfg, bounds, precision="bf16", **kw)
        ts = []
        r = None
        for _ in range(20):
            gs = copy.deepcopy(groups)
            if collect:
                gc.collect()
            t0 = time.perf_counter()
            r = O.objective_and_grad(gs, theta, theta, None, cfg, bounds, precision="bf16", **kw)
            ts.append(1e3 * (time.perf_counter() - t0))
        print(f"{name:18s} median {np.median(ts):7.2f} ms  calls " + " ".join(f"{t:.1f}" for t in ts), flush=True)
        del r


if __name__ == "__main__":
    main()
