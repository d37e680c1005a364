"""Probe: a long-K GEMM (wave barriers) while a side-stream kernel holds 40 SMs until a flag that
is set after the GEMM (tests/test_contention_gpu.py's scenario), with kernel-side timestamps."""
import ctypes, sys, time
import torch
sys.path.insert(0, '.')
from paper_2510_18855_b200 import _lib
lib = _lib.ensure_device(0)
h = ctypes.CDLL('tests/native/libicepop_testhelpers.so')
h.th_hold_sms.argtypes = [ctypes.c_int, ctypes.c_int, ctypes.c_void_p, ctypes.c_longlong, ctypes.c_void_p,
                          ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p]
h.th_set_flag.argtypes = [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p]
dev = torch.device('cuda', 0)
M, N, K = 4096, 4096, 32768
A = torch.randn((M, K), device=dev).to(torch.bfloat16)
B = torch.randn((K, N), device=dev).to(torch.bfloat16)
C = torch.empty((M, N), dtype=torch.float32, device=dev)
for main_kind in ('default', 'side'):
    main = torch.cuda.current_stream() if main_kind == 'default' else torch.cuda.Stream()
    def gemm():
        _lib.check(lib.icepop_gemm_bf16(A.data_ptr(), B.data_ptr(), C.data_ptr(), M, N, K, 0, 1, 1, 0, main.cuda_stream))
    gemm(); torch.cuda.synchronize()
    flag = torch.zeros(1, dtype=torch.int32, device=dev)
    status = torch.zeros(1, dtype=torch.int32, device=dev)
    started = torch.zeros(1, dtype=torch.int32, device=dev)
    times = torch.tensor([2**62, 0, 0], dtype=torch.int64, device=dev)
    torch.cuda.synchronize()
    side = torch.cuda.Stream()
    t0 = time.time()
    assert h.th_hold_sms(40, 200*1024, flag.data_ptr(), 3_000_000_000, status.data_ptr(), started.data_ptr(),
                         times.data_ptr(), side.cuda_stream) == 0
    time.sleep(0.05)
    a0 = _lib.wave_barrier_abandons(0)
    gemm()
    rc = h.th_set_flag(flag.data_ptr(), times.data_ptr(), main.cuda_stream)
    torch.cuda.synchronize()
    t = times.tolist()
    print(main_kind, 'rc', rc, 'wall', round(time.time() - t0, 3), 'status', status.item(), 'started', started.item(),
          'abandons', _lib.wave_barrier_abandons(0) - a0, 'hold->set ms', (t[2] - t[0]) / 1e6,
          'hold->end ms', (t[1] - t[0]) / 1e6, flush=True)
