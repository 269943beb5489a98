"""Tile GEMM on the tcgen05 tensor cores (K4) -- the per-processor product of
the mapped matmul workloads (no reference code).

`tile_gemm(A, Bt, C)` computes C (+)= A @ Bt.T with A [M, K] and Bt [N, K]
bf16 row-major (both K-contiguous), fp32 accumulation in TMEM, C fp32 or bf16.
"""

from __future__ import annotations

from . import native


def tile_gemm(A, Bt, C=None, *, accumulate: bool = False, out_dtype=None, stream=None):
    torch = native.require_cuda()
    if A.dtype != torch.bfloat16 or Bt.dtype != torch.bfloat16:
        raise ValueError("A and Bt must be bf16")
    if A.dim() != 2 or Bt.dim() != 2 or A.shape[1] != Bt.shape[1]:
        raise ValueError(f"shape mismatch: A {tuple(A.shape)}, Bt {tuple(Bt.shape)}")
    if A.stride(1) != 1 or Bt.stride(1) != 1:
        raise ValueError("A and Bt must be row-major (K contiguous)")
    M, K = A.shape
    N = Bt.shape[0]
    if C is None:
        C = torch.zeros if accumulate else torch.empty
        C = C((M, N), dtype=out_dtype or torch.float32, device=A.device)
    if C.shape != (M, N) or C.stride(1) != 1 or C.dtype not in (torch.float32, torch.bfloat16):
        raise ValueError("C must be a row-major fp32/bf16 [M, N] tensor")
    with torch.cuda.device(A.device):
        native.check(native.lib().pm_gemm_bf16(
            A.data_ptr(), A.stride(0), Bt.data_ptr(), Bt.stride(0), C.data_ptr(), C.stride(0),
            M, N, K, int(C.dtype == torch.bfloat16), int(accumulate),
            native.stream_ptr(stream)), "pm_gemm_bf16")
    return C


def tile_gemm_tf32(A, Bt, C=None, *, accumulate: bool = False, stream=None):
    """C (+)= A @ Bt.T on fp32 operands via the TF32 tensor cores (fp32 accumulate)."""
    torch = native.require_cuda()
    if A.dtype != torch.float32 or Bt.dtype != torch.float32:
        raise ValueError("A and Bt must be fp32")
    if A.dim() != 2 or Bt.dim() != 2 or A.shape[1] != Bt.shape[1]:
        raise ValueError(f"shape mismatch: A {tuple(A.shape)}, Bt {tuple(Bt.shape)}")
    if A.stride(1) != 1 or Bt.stride(1) != 1:
        raise ValueError("A and Bt must be row-major (K contiguous)")
    M, K = A.shape
    N = Bt.shape[0]
    if C is None:
        C = (torch.zeros if accumulate else torch.empty)((M, N), dtype=torch.float32,
                                                         device=A.device)
    if C.shape != (M, N) or C.stride(1) != 1 or C.dtype != torch.float32:
        raise ValueError("C must be a row-major fp32 [M, N] tensor")
    with torch.cuda.device(A.device):
        native.check(native.lib().pm_gemm_tf32(
            A.data_ptr(), A.stride(0), Bt.data_ptr(), Bt.stride(0), C.data_ptr(), C.stride(0),
            M, N, K, int(accumulate), native.stream_ptr(stream)), "pm_gemm_tf32")
    return C
