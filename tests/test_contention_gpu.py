"""The long-K GEMMs (K4 dHidden, K5 dW) run static waves with a grid barrier between k-chunks,
which keeps the operand slices a wave shares in L2. Their grid is sized for an idle GPU. Here a
kernel on a side stream holds 40 SMs until a flag is set AFTER the GEMM on the main stream --
the shape of an NCCL kernel waiting on its peers. Part of the GEMM's grid cannot start until
the resident part has finished, so a barrier that waited for every unit would deadlock. The
barrier instead gives up after ICEPOP_WAVE_TIMEOUT_US and the GEMM completes with the same
result (checked against torch), the holder is released by the flag (not by its own safety
timeout), and the library's abandon counter records the event.
"""

from __future__ import annotations

import ctypes
import time
from pathlib import Path

import pytest
import torch

pytestmark = pytest.mark.gpu

HELPERS = Path(__file__).resolve().parent / "native" / "libicepop_testhelpers.so"


def _helpers():
    if not HELPERS.exists():
        pytest.fail(f"{HELPERS} missing: run `make` (it is built with the library)")
    h = ctypes.CDLL(str(HELPERS))
    h.th_hold_sms.argtypes = [ctypes.c_int, ctypes.c_int, ctypes.c_void_p, ctypes.c_longlong, ctypes.c_void_p,
                              ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p]
    h.th_set_flag.argtypes = [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p]
    return h


@pytest.mark.parametrize("a_mn,b_mn", [(False, True), (True, True)], ids=["K4-majors", "K5-majors"])
def test_long_k_gemm_completes_while_sms_are_held(cuda_device, a_mn, b_mn):
    from paper_2510_18855_b200 import _lib

    lib = _lib.ensure_device(0)
    h = _helpers()
    M, N, K = 4096, 4096, 32768  # 512 k-blocks: a long-K GEMM of 128 wide pair tiles (two waves: barriers)
    g = torch.Generator(device=cuda_device).manual_seed(5)
    A = torch.randn((K, M) if a_mn else (M, K), device=cuda_device, generator=g).to(torch.bfloat16)
    B = torch.randn((K, N) if b_mn else (N, K), device=cuda_device, generator=g).to(torch.bfloat16)
    C = torch.empty((M, N), dtype=torch.float32, device=cuda_device)
    flag = torch.zeros(1, dtype=torch.int32, device=cuda_device)
    status = torch.zeros(1, dtype=torch.int32, device=cuda_device)
    started = torch.zeros(1, dtype=torch.int32, device=cuda_device)
    # load the helper kernels first: a kernel's first launch (CUDA lazy loading) waits for the
    # kernels already running, here the holder (the library preloads its own kernels)
    assert h.th_set_flag(status.data_ptr(), None, torch.cuda.current_stream().cuda_stream) == 0
    assert h.th_hold_sms(1, 1024, status.data_ptr(), 0, started.data_ptr(), started.data_ptr(), None,
                         torch.cuda.current_stream().cuda_stream) == 0
    torch.cuda.synchronize()
    status.zero_()
    started.zero_()
    torch.cuda.synchronize()
    before = _lib.wave_barrier_abandons(0)
    # non-default streams on both sides: the legacy default stream would serialise the flag
    # kernel behind the holder by itself (implicit synchronisation), deadlocking any GEMM
    side = torch.cuda.Stream(cuda_device)
    main = torch.cuda.Stream(cuda_device)
    assert h.th_hold_sms(40, 200 * 1024, flag.data_ptr(), 10_000_000_000, status.data_ptr(), started.data_ptr(),
                         None, side.cuda_stream) == 0
    time.sleep(0.05)  # the holder blocks are resident before the GEMM launches
    _lib.check(lib.icepop_gemm_bf16(A.data_ptr(), B.data_ptr(), C.data_ptr(), M, N, K, int(a_mn), int(b_mn), 1, 0,
                                    main.cuda_stream))
    assert h.th_set_flag(flag.data_ptr(), None, main.cuda_stream) == 0
    torch.cuda.synchronize()
    assert int(started.item()) == 40
    assert int(status.item()) == 0, "the holder timed out: the GEMM did not finish while SMs were held"
    assert _lib.wave_barrier_abandons(0) > before
    ref = (A.float().T if a_mn else A.float()) @ (B.float() if b_mn else B.float().T)
    err = float((C - ref).norm() / ref.norm())
    assert err < 1e-4, err  # fp32 accumulation over K = 32,768 in both
