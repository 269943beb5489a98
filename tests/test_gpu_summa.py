"""Mapped SUMMA executor on one GPU: the Mapple tile mapping drives the
layout, the result matches float64 within the north-star tolerance."""

import pytest

from paper_2507_17087_b200.executors.summa import MappedGemm, synth

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("M,N,K", [(1024, 1024, 1024), (2048, 1024, 512), (1000, 1300, 640)])
def test_single_gpu_summa_matches_fp64(cuda, M, N, K):
    torch = cuda
    ex = MappedGemm(M, N, K, seed=7)
    C = ex.step()
    torch.cuda.synchronize()
    A = synth((0, M), (0, K), K, 7, "cuda").double()
    Bt = synth((0, N), (0, K), K, 8, "cuda").double()
    R = A @ Bt.T
    err = float((C.double() - R).abs().max() / R.abs().max())
    assert err <= 1e-2 and err < 1e-3
    assert ex.layout.grid == (1, 1) and ex.recv_bytes == 0
    ex.close()
