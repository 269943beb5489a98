"""Quick K4 timing probe (CUDA events) vs torch.matmul on the same box."""
import sys, time
sys.path.insert(0, ".")
import torch
from paper_2507_17087_b200.gemm import tile_gemm

def bench(fn, iters=10):
    for _ in range(3): fn()
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(iters): fn()
    e.record(); torch.cuda.synchronize()
    return s.elapsed_time(e) / iters

for n in [int(x) for x in (sys.argv[1:] or ["4096", "8192", "16384"])]:
    A = torch.randn(n, n, device="cuda").to(torch.bfloat16)
    Bt = torch.randn(n, n, device="cuda").to(torch.bfloat16)
    C = torch.empty(n, n, device="cuda")
    ms = bench(lambda: tile_gemm(A, Bt, C))
    ms_t = bench(lambda: torch.matmul(A, Bt.T))
    fl = 2 * n ** 3
    print(f"N={n}: pm_gemm {ms:.3f} ms {fl/ms/1e9:.1f} TF/s | torch {ms_t:.3f} ms {fl/ms_t/1e9:.1f} TF/s", flush=True)
