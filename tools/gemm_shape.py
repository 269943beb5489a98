"""Run pm_gemm (and torch.matmul) on one M x N x K shape, for ncu experiments."""
import sys
sys.path.insert(0, ".")
import torch
from paper_2507_17087_b200.gemm import tile_gemm
M, N, K = (int(x) for x in sys.argv[1:4])
A = torch.randn(M, K, device="cuda").to(torch.bfloat16)
Bt = torch.randn(N, K, device="cuda").to(torch.bfloat16)
C = torch.empty(M, N, device="cuda", dtype=torch.bfloat16)
for _ in range(3):
    tile_gemm(A, Bt, C)
    torch.matmul(A, Bt.T, out=C)
torch.cuda.synchronize()
print("ok")
