"""Small run of every libicepop entry point, for compute-sanitizer (one tool per call).

    python profiles/sanitize_case.py && compute-sanitizer --tool memcheck python profiles/sanitize_case.py
"""
import sys
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2510_18855_b200 import _lib  # noqa: E402
from paper_2510_18855_b200.loss import (IcePopConfig, PackedBatch, discrepancy, finish, icepop_bwd,  # noqa: E402
                                        icepop_fwd, icepop_fwd_onpolicy, icepop_logprob)
from paper_2510_18855_b200.optim import sgd_update_  # noqa: E402


def main():
    dev = torch.device("cuda", 0)
    rng = np.random.default_rng(0)
    lens = [130, 77, 300, 45]
    N, d, V = sum(lens), 192, 520
    H = torch.from_numpy(rng.normal(0, 1, (N, d))).to(torch.bfloat16).to(dev)
    W = torch.from_numpy(rng.normal(0, 0.15, (V, d))).to(torch.bfloat16).to(dev)
    Wr = (W.float() + 0.01).to(torch.bfloat16)
    tok = torch.from_numpy(rng.integers(0, V, N).astype(np.int32)).to(dev)
    lp, lse, ent = icepop_logprob(H, W, tok)
    lp_old = lp + torch.from_numpy(rng.normal(0, 0.1, N)).to(dev)
    lp_inf = lp_old - torch.from_numpy(rng.normal(0, 0.4, N)).to(dev)
    cu = torch.tensor(np.concatenate([[0], np.cumsum(lens)]).astype(np.int32), device=dev)
    go = torch.tensor([0, 2, 4], dtype=torch.int32, device=dev)
    adv = torch.tensor([1.0, 0.0, -0.5, 0.0], dtype=torch.float64, device=dev)
    b = PackedBatch(tok, lp_old, lp_inf, cu, go, adv)
    lib = _lib.ensure_device(0)
    for cg in (1, 2):
        _lib.check(lib.icepop_set_cta_group(cg))
        for kl in (0.0, 0.3):
            cfg = IcePopConfig(kl_coeff=kl)
            f = icepop_fwd(H, W, b, cfg, weight_ref=Wr if kl else None)
            icepop_bwd(H, W, b, f, cfg, weight_ref=Wr if kl else None, grad_hidden_dtype=torch.float32)
            finish(f.stats)
        ob = PackedBatch(tok, lp, lp - 0.1, cu, go, adv)
        f = icepop_fwd_onpolicy(ob, lse, ent, IcePopConfig(), hidden_dim=d, vocab=V)
        icepop_bwd(H, W, ob, f, IcePopConfig())
        discrepancy(H, Wr, W)
    Hd, Wd = H.double(), W.double().t().contiguous()
    f = icepop_fwd(Hd, Wd, b, IcePopConfig(kl_coeff=0.2), layout="dv", weight_ref=Wd + 0.01)
    icepop_bwd(Hd, Wd, b, f, IcePopConfig(kl_coeff=0.2), layout="dv", weight_ref=Wd + 0.01)
    w32 = W.float().contiguous()
    sgd_update_(w32, torch.ones_like(w32), 0.1, torch.zeros_like(w32), 0.5, torch.empty_like(W))
    torch.cuda.synchronize()
    print("sanitize case ok")


if __name__ == "__main__":
    main()
