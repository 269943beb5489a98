"""Run one pm_gemm and one torch.matmul of the same shape (for side-by-side ncu)."""
import sys
sys.path.insert(0, ".")
import torch
from paper_2507_17087_b200.gemm import tile_gemm
n = int(sys.argv[1]) if len(sys.argv) > 1 else 16384
A = torch.randn(n, n, device="cuda").to(torch.bfloat16)
Bt = torch.randn(n, n, device="cuda").to(torch.bfloat16)
Cb = torch.empty(n, n, device="cuda", dtype=torch.bfloat16)
for _ in range(2):
    tile_gemm(A, Bt, Cb)
    torch.matmul(A, Bt.T, out=Cb)
torch.cuda.synchronize()
tile_gemm(A, Bt, Cb)
torch.matmul(A, Bt.T, out=Cb)
torch.cuda.synchronize()
print("ok")
