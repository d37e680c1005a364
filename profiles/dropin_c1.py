"""Switch the import: BASELINE configs[0] through the reference-facing API on both sides.

The same C1 batch (tests/golden/c1_config0.npz: 8 x 512 tokens, 1,024 features, V = 32,768,
one GRPO group of 8) as the reference's own Python objects (mismatchlab PromptGroup /
TokenRecord / PolicyParams from the baseline/_ref install), passed to
  * the unmodified reference ``mismatchlab.objective_and_grad`` (numpy, host), and
  * the drop-in ``paper_2510_18855_b200.objective.objective_and_grad`` (bf16 tensor-core path
    and fp64 validation path), wall clock per call: packing of the Python records, the
    multi-hot H, H2D of inputs and weights, both kernels, D2H of the 268 MB fp64 gradient and
    the per-token diagnostics, and the write-back into every TokenRecord.
Outputs are compared (mask bit-exact; objective and gradient norm relative).

    python profiles/dropin_c1.py [--reps 10]
"""
import argparse
import copy
import sys
import time
from pathlib import Path

import numpy as np
import torch

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT / "baseline" / "_ref"))
sys.path.insert(0, str(ROOT / "tests"))
sys.path.insert(0, str(ROOT))
import mismatchlab as ml  # noqa: E402
from conftest import load_c1  # noqa: E402
from mismatchlab.tasks import TaskKind  # noqa: E402

from paper_2510_18855_b200 import objective as dropin  # noqa: E402


def make_groups(d):
    cu, go = d["cu_seqlens"], d["group_offsets"]
    groups = []
    for g in range(len(go) - 1):
        task = ml.TaskSpec(TaskKind.PARITY_MATCH, int(d["prompt_ids"][go[g]]), 0, 4)
        rollouts = []
        for i in range(go[g], go[g + 1]):
            recs = [ml.TokenRecord(token=int(d["tokens"][t]), logp_infer_old=float(d["lp_infer_old"][t]),
                                   logp_train_old=float(d["lp_train_old"][t]),
                                   logp_train_cur=float(d["lp_train_old"][t]), gen_version=0)
                    for t in range(cu[i], cu[i + 1])]
            rollouts.append(ml.Rollout(task=task, stream=np.random.default_rng(i), uid=int(i), group_uid=g,
                                       tokens=recs, terminal=True))
        groups.append(ml.PromptGroup(task=task, rollouts=rollouts,
                                     rewards=[float(r) for r in d["rewards"][go[g]:go[g + 1]]],
                                     advantages=[float(a) for a in d["advantages"][go[g]:go[g + 1]]]))
    return groups


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--reps", type=int, default=10)
    ap.add_argument("--profile", action="store_true", help="cProfile one bf16 call (top 20 by own time)")
    a = ap.parse_args()
    d, w = load_c1()
    n_tok = int(d["cu_seqlens"][-1])
    theta = ml.PolicyParams(weights=w)
    cfg, bounds = ml.ObjectiveConfig(), ml.MaskingBounds()
    assert dropin.Algo is ml.Algo  # the drop-in re-exports the reference's types

    groups = make_groups(d)
    t0 = time.perf_counter()
    ref = ml.objective_and_grad(groups, theta, theta, None, cfg, bounds)
    t_ref = time.perf_counter() - t0
    print(f"C1 ({n_tok} tokens, {w.shape[0]} features, V {w.shape[1]}): reference objective_and_grad "
          f"{t_ref:.2f} s = {n_tok / t_ref:.1f} tokens/s (single-threaded numpy)")

    for precision in ("bf16", "fp64"):
        gs = copy.deepcopy(groups)
        out = dropin.objective_and_grad(gs, theta, theta, None, cfg, bounds, precision=precision)  # warm-up
        torch.cuda.synchronize()
        ts = []
        for _ in range(a.reps):
            gs = copy.deepcopy(groups)
            t0 = time.perf_counter()
            out = dropin.objective_and_grad(gs, theta, theta, None, cfg, bounds, precision=precision)
            ts.append(time.perf_counter() - t0)
        ts.sort()
        t = ts[len(ts) // 2]
        if a.profile:
            import cProfile
            import pstats

            gs = copy.deepcopy(groups)
            pr = cProfile.Profile()
            pr.enable()
            dropin.objective_and_grad(gs, theta, theta, None, cfg, bounds, precision=precision)
            pr.disable()
            pstats.Stats(pr).sort_stats("tottime").print_stats(20)
        kept_eq = np.array_equal(np.asarray(out.per_token_mask_kept), np.asarray(ref.per_token_mask_kept))
        j_rel = abs(out.objective_value - ref.objective_value) / max(abs(ref.objective_value), 1e-30)
        g_rel = float(np.linalg.norm(out.grad - ref.grad) / max(np.linalg.norm(ref.grad), 1e-30))
        buf = np.empty_like(w)
        tb = []
        for _ in range(a.reps):
            gs = copy.deepcopy(groups)
            t0 = time.perf_counter()
            dropin.objective_and_grad(gs, theta, theta, None, cfg, bounds, precision=precision, grad_out=buf)
            tb.append(time.perf_counter() - t0)
        tb.sort()
        print(f"drop-in {precision} with a reused grad_out: {tb[len(tb) // 2] * 1e3:.1f} ms per call "
              f"({t_ref / tb[len(tb) // 2]:.0f}x the reference); same grad bits as the fresh array: "
              f"{np.array_equal(buf, out.grad)}")
        print(f"drop-in {precision}: {t * 1e3:.1f} ms per call (median of {a.reps}; min {ts[0] * 1e3:.1f}) = "
              f"{n_tok / t:.0f} tokens/s, {t_ref / t:.0f}x the reference; mask bit-exact {kept_eq}, "
              f"J rel {j_rel:.2e}, grad rel {g_rel:.2e}, token_count {out.token_count}, "
              f"clipped_fraction {out.clipped_fraction} (ref {ref.clipped_fraction})")


if __name__ == "__main__":
    main()
