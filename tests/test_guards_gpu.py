"""Out-of-bounds write detection (compute-sanitizer is closed on this pool): every buffer
the kernels write -- workspace, dHidden, dW, per-token outputs -- is a view into a larger
allocation whose guard bands hold a sentinel; after fwd + bwd on shapes whose tails do not
align with any tile (N, d, V not multiples of 128/256) the guards must be intact."""

from __future__ import annotations

import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu

GUARD = 1 << 16  # bytes on each side
SENT = 0xA5


def guarded(nbytes: int, dev):
    buf = torch.full((nbytes + 2 * GUARD,), SENT, dtype=torch.uint8, device=dev)
    return buf, buf[GUARD:GUARD + nbytes]


def intact(buf) -> bool:
    return bool((buf[:GUARD] == SENT).all()) and bool((buf[-GUARD:] == SENT).all())


def typed(view, dtype, shape):
    return view.view(dtype).view(shape)


@pytest.mark.parametrize("cg", [1, 2])
@pytest.mark.parametrize("layout", ["vd", "dv"])
@pytest.mark.parametrize("ref", [False, True])
def test_no_out_of_bounds_writes(cuda_device, cg, layout, ref):
    from paper_2510_18855_b200 import _lib
    from paper_2510_18855_b200.loss import IcePopConfig, PackedBatch, bwd_workspace_bytes

    lib = _lib.ensure_device(0)
    _lib.check(lib.icepop_set_cta_group(cg))
    try:
        rng = np.random.default_rng(1)
        lens = [131, 90, 112]
        N, d, V = sum(lens), 200, 1000
        st = torch.cuda.current_stream().cuda_stream
        H = torch.from_numpy(rng.normal(0, 1, (N, d))).to(torch.bfloat16).to(cuda_device)
        wshape = (V, d) if layout == "vd" else (d, V)
        W = torch.from_numpy(rng.normal(0, 0.1, wshape)).to(torch.bfloat16).to(cuda_device)
        Wr = (W.float() * 1.01).to(torch.bfloat16) if ref else None
        tok = torch.from_numpy(rng.integers(0, V, N).astype(np.int32)).to(cuda_device)
        lp_old = torch.from_numpy(rng.normal(-7, 0.3, N)).to(cuda_device)
        lp_inf = lp_old - torch.from_numpy(rng.normal(0, 0.5, N)).to(cuda_device)
        cu = torch.tensor(np.concatenate([[0], np.cumsum(lens)]).astype(np.int32), device=cuda_device)
        go = torch.tensor([0, 3], dtype=torch.int32, device=cuda_device)
        adv = torch.tensor([1.0, -0.5, 0.0], dtype=torch.float64, device=cuda_device)
        b = PackedBatch(tok, lp_old, lp_inf, cu, go, adv)
        cfg = IcePopConfig(kl_coeff=0.3 if ref else 0.0)
        shape = _lib.Shape(n_tokens=N, token_offset=0, hidden=d, vocab=V, n_seqs=3, n_groups=1,
                           weight_layout=_lib.W_VD if layout == "vd" else _lib.W_DV)
        fb = _lib._sz()
        _lib.check(lib.icepop_workspace_bytes(shape, 0, 1 if ref else 0, fb, None))
        bufs = {}

        def out(name, n, dtype):
            raw, view = guarded(n * torch.empty((), dtype=dtype).element_size(), cuda_device)
            bufs[name] = raw
            return typed(view, dtype, (n,))

        ws_raw, ws = guarded(fb.value, cuda_device)
        bufs["fwd_ws"] = ws_raw
        lse, ent, coeff = out("lse", N, torch.float32), out("ent", N, torch.float32), out("coeff", N, torch.float32)
        lp, calib, sur = out("lp", N, torch.float64), out("calib", N, torch.float64), out("sur", N, torch.float64)
        kept, stats = out("kept", N, torch.uint8), out("stats", 8, torch.float64)
        kl, lser, klw = out("kl", N, torch.float32), out("lser", N, torch.float32), out("klw", N, torch.float32)
        fo = _lib.FwdOut(lse=lse.data_ptr(), lp_cur=lp.data_ptr(), entropy=ent.data_ptr(), kept=kept.data_ptr(),
                         calib=calib.data_ptr(), surrogate=sur.data_ptr(), coeff=coeff.data_ptr(),
                         stats=stats.data_ptr(), kl=kl.data_ptr(), lse_ref=lser.data_ptr(), kl_w=klw.data_ptr())
        _lib.check(lib.icepop_fwd_bf16(shape, cfg.to_c(), H.data_ptr(), W.data_ptr(), _lib.ptr(Wr), b.to_c(), fo,
                                       ws.data_ptr(), ws.numel(), st))
        bw = bwd_workspace_bytes(N, d, V, 3, chunk_bytes=128 * (V + d) * 2)  # 128-row chunks: several tails
        bws_raw, bws = guarded(bw, cuda_device)
        bufs["bwd_ws"] = bws_raw
        gh_raw, ghv = guarded(N * d * 4, cuda_device)
        gw_raw, gwv = guarded(V * d * 4, cuda_device)
        bufs["gh"], bufs["gw"] = gh_raw, gw_raw
        sv = _lib.Saved(tokens=tok.data_ptr(), lse=lse.data_ptr(), coeff=coeff.data_ptr(), lse_ref=lser.data_ptr(),
                        kl=kl.data_ptr(), kl_w=klw.data_ptr())
        _lib.check(lib.icepop_bwd_bf16(shape, cfg.to_c(), H.data_ptr(), W.data_ptr(), _lib.ptr(Wr), sv, -1.0,
                                       ghv.data_ptr(), 1, gwv.data_ptr(), 0, bws.data_ptr(), bws.numel(), st))
        _lib.check(lib.icepop_finish(stats.data_ptr(), st))
        torch.cuda.synchronize()
        bad = [k for k, v in bufs.items() if not intact(v)]
        assert not bad, f"guard bands overwritten: {bad}"
        assert torch.isfinite(typed(gwv, torch.float32, (V * d,))).all()
    finally:
        _lib.check(lib.icepop_set_cta_group(2))
