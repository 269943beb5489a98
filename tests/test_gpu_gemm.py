"""K4 on the B200: tcgen05 tile GEMM vs a float64 reference.

Tolerance (BASELINE north star): bf16 inputs, fp32 accumulation, max relative
error <= 1e-2 against the fp64 product of the same (bf16-rounded) inputs,
measured as max|C - C64| / max|C64|.
"""

import pytest

from paper_2507_17087_b200.gemm import tile_gemm

pytestmark = pytest.mark.gpu

TOL = 1e-2


def _ref(A, Bt):
    return A.double() @ Bt.double().T


def _rel(C, R):
    return float((C.double() - R).abs().max() / R.abs().max().clamp_min(1e-30))


@pytest.mark.parametrize("M,N,K", [(128, 256, 64), (256, 512, 128), (128, 256, 4096),
                                   (1000, 700, 320), (4096, 4096, 4096), (300, 1000, 8),
                                   (1024, 2048, 1024), (2048, 256, 16384)])
def test_gemm_matches_fp64(cuda, M, N, K):
    torch = cuda
    g = torch.Generator(device="cuda").manual_seed(M * 7 + N * 3 + K)
    A = (torch.rand(M, K, device="cuda", generator=g) * 2 - 1).to(torch.bfloat16)
    Bt = (torch.rand(N, K, device="cuda", generator=g) * 2 - 1).to(torch.bfloat16)
    C = tile_gemm(A, Bt)
    torch.cuda.synchronize()
    R = _ref(A, Bt)
    assert _rel(C, R) <= TOL
    # fp32 accumulation of exact bf16 products: far tighter than the contract
    assert _rel(C, R) < 1e-3


@pytest.mark.parametrize("M,N,K", [(512, 768, 256), (2048, 1280, 512), (1100, 900, 192)])
def test_gemm_accumulate_and_bf16_out(cuda, M, N, K):
    torch = cuda
    A = torch.randn(M, K, device="cuda").to(torch.bfloat16)
    Bt = torch.randn(N, K, device="cuda").to(torch.bfloat16)
    C0 = torch.randn(M, N, device="cuda")
    C = C0.clone()
    tile_gemm(A, Bt, C, accumulate=True)
    R = C0.double() + _ref(A, Bt)
    assert _rel(C, R) < 1e-4
    Cb = tile_gemm(A, Bt, out_dtype=torch.bfloat16)
    assert Cb.dtype == torch.bfloat16
    assert _rel(Cb, _ref(A, Bt)) < TOL


def test_gemm_strided_views(cuda):
    torch = cuda
    big = torch.randn(600, 1024, device="cuda").to(torch.bfloat16)
    A = big[:, :512]           # lda = 1024
    Bt = big[100:356, 512:]    # ldb = 1024
    C = tile_gemm(A, Bt)
    assert _rel(C, _ref(A, Bt)) < 1e-4


@pytest.mark.parametrize("M,N,K", [(512, 512, 512), (1000, 700, 320), (128, 256, 32), (2048, 1024, 4096),
                                   (512, 384, 1000)])
def test_tf32_gemm(cuda, M, N, K):
    from paper_2507_17087_b200.gemm import tile_gemm_tf32

    torch = cuda
    g = torch.Generator(device="cuda").manual_seed(M + N + K)
    A = torch.rand(M, K, device="cuda", generator=g) * 2 - 1
    Bt = torch.rand(N, K, device="cuda", generator=g) * 2 - 1
    C = tile_gemm_tf32(A, Bt)
    R = A.double() @ Bt.double().T
    assert _rel(C, R) <= TOL  # tf32 operands: ~1e-3 relative
    C2 = tile_gemm_tf32(A, Bt, C.clone(), accumulate=True)
    assert _rel(C2, 2 * R) <= TOL
