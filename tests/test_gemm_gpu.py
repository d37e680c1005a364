"""tcgen05 GEMM core (K4/K5 building block) vs torch fp32 matmul, all operand majors."""

from __future__ import annotations

import pytest
import torch

pytestmark = pytest.mark.gpu


@pytest.fixture(params=[1, 2], ids=["cta1", "cta2"])
def cta_group(request):
    from paper_2510_18855_b200 import _lib

    lib = _lib.ensure_device(0)
    _lib.check(lib.icepop_set_cta_group(request.param))
    yield request.param
    _lib.check(lib.icepop_set_cta_group(2))


def _gemm(A, B, M, N, K, a_mn, b_mn, c_f32=True, accumulate=False, C=None):
    from paper_2510_18855_b200 import _lib

    lib = _lib.ensure_device(0)
    A_st = A.t().contiguous() if a_mn else A.contiguous()
    B_st = B.t().contiguous() if b_mn else B.contiguous()
    if C is None:
        C = torch.zeros(M, N, dtype=torch.float32 if c_f32 else torch.bfloat16, device=A.device)
    _lib.check(lib.icepop_gemm_bf16(A_st.data_ptr(), B_st.data_ptr(), C.data_ptr(), M, N, K, int(a_mn), int(b_mn),
                                    int(c_f32), int(accumulate), torch.cuda.current_stream().cuda_stream))
    torch.cuda.synchronize()
    return C


@pytest.mark.parametrize("a_mn,b_mn", [(0, 0), (0, 1), (1, 0), (1, 1)])
@pytest.mark.parametrize("M,N,K", [(128, 256, 64), (296, 520, 200), (1024, 2048, 512), (136, 264, 1000),
                                   (520, 136, 72)])
def test_gemm_majors(cuda_device, cta_group, a_mn, b_mn, M, N, K):
    g = torch.Generator(device="cpu").manual_seed(M * 7 + N + K)
    A = torch.randn(M, K, generator=g).to(torch.bfloat16).to(cuda_device)
    B = torch.randn(N, K, generator=g).to(torch.bfloat16).to(cuda_device)
    C = _gemm(A, B, M, N, K, a_mn, b_mn)
    ref = A.double() @ B.double().T
    err = (C.double() - ref).abs().max().item()
    assert err <= 1e-3 * (K ** 0.5), f"max abs err {err}"


def test_gemm_bf16_out_and_accumulate(cuda_device, cta_group):
    M, N, K = 256, 512, 320
    A = torch.randn(M, K, device=cuda_device).to(torch.bfloat16)
    B = torch.randn(N, K, device=cuda_device).to(torch.bfloat16)
    ref = A.double() @ B.double().T
    Cb = _gemm(A, B, M, N, K, 0, 0, c_f32=False)
    assert (Cb.double() - ref).abs().max().item() < 0.02 * ref.abs().max().item()
    C0 = torch.ones(M, N, device=cuda_device)
    C1 = _gemm(A, B, M, N, K, 1, 1, accumulate=True, C=C0)
    assert torch.allclose(C1.double(), ref + 1.0, atol=1e-2, rtol=1e-4)


@pytest.fixture
def wide_tiles():
    from paper_2510_18855_b200 import _lib

    lib = _lib.ensure_device(0)

    def set_(on):  # on: 512-wide tiles forced (2), not only where they fill the GPU (1)
        _lib.check(lib.icepop_set_wide_tiles(2 if on else 0))

    yield set_
    _lib.check(lib.icepop_set_wide_tiles(1))


@pytest.mark.parametrize("a_mn,b_mn", [(0, 0), (0, 1), (1, 0), (1, 1)])
@pytest.mark.parametrize("M,N,K", [(600, 1304, 16448), (256, 512, 16384), (136, 2104, 20000), (4096, 4096, 16448)])
def test_gemm_long_k_wide_tiles(cuda_device, wide_tiles, a_mn, b_mn, M, N, K):
    """K >= 16384 is the long-K path: static waves with the k-chunk barrier when the tiles take
    more than one wave (the 4096 x 4096 case), the dynamic schedule otherwise; on CTA pairs the
    256 x 512 tiles (two N = 256 MMAs into one accumulator, pair-interleaved B rows). Same
    per-element k order as the 256 x 256 tiles, so the two agree bit for bit; both vs fp64."""
    g = torch.Generator(device="cpu").manual_seed(M + N + K)
    A = torch.randn(M, K, generator=g).to(torch.bfloat16).to(cuda_device)
    B = torch.randn(N, K, generator=g).to(torch.bfloat16).to(cuda_device)
    wide_tiles(True)
    Cw = _gemm(A, B, M, N, K, a_mn, b_mn)
    Cw_acc = _gemm(A, B, M, N, K, a_mn, b_mn, accumulate=True, C=torch.full((M, N), 0.5, device=cuda_device))
    Cw_bf = _gemm(A, B, M, N, K, a_mn, b_mn, c_f32=False)
    wide_tiles(False)
    Cn = _gemm(A, B, M, N, K, a_mn, b_mn)
    ref = A.double() @ B.double().T
    assert (Cw.double() - ref).abs().max().item() <= 1e-3 * (K ** 0.5)
    assert torch.equal(Cw, Cn)
    assert torch.equal(Cw_acc, Cw + 0.5)
    assert torch.equal(Cw_bf, Cw.to(torch.bfloat16))


def test_small_long_k_output_takes_narrow_tiles_with_same_bits(cuda_device, wide_tiles):
    """A long-K GEMM whose output is too small to fill the GPU with 256x512 tiles (C1's dH:
    4,096 x 1,024 at K = 32,768) runs on 256x256 tiles by default; all three settings give the
    same bits (fp32 accumulation order along K is the same for both tile widths)."""
    from paper_2510_18855_b200 import _lib

    lib = _lib.ensure_device(0)
    M, N, K = 4096, 1024, 32768
    g = torch.Generator(device=cuda_device).manual_seed(5)
    A = torch.randn(M, K, device=cuda_device, generator=g).to(torch.bfloat16)
    B = torch.randn(K, N, device=cuda_device, generator=g).to(torch.bfloat16)
    st = torch.cuda.current_stream().cuda_stream
    outs = []
    for mode in (1, 2, 0):
        _lib.check(lib.icepop_set_wide_tiles(mode))
        C = torch.empty(M, N, device=cuda_device, dtype=torch.float32)
        _lib.check(lib.icepop_gemm_bf16(A.data_ptr(), B.data_ptr(), C.data_ptr(), M, N, K, 0, 1, 1, 0, st))
        outs.append(C)
    torch.cuda.synchronize()
    assert torch.equal(outs[0], outs[1]) and torch.equal(outs[0], outs[2])
    ref = A.float() @ B.float()
    assert float((outs[0] - ref).norm() / ref.norm()) < 1e-4  # fp32 summation order over K = 32,768
