"""K2 (stable partition) timing on 1.07e9 ids / 8 bins, for ncu launch lists."""
import sys
sys.path.insert(0, ".")
import torch
from paper_2507_17087_b200.ownership import partition
n = int(sys.argv[1]) if len(sys.argv) > 1 else 1 << 30
nb = int(sys.argv[2]) if len(sys.argv) > 2 else 8
g = torch.Generator(device="cuda").manual_seed(0)
# block-structured ids like a mapped stencil launch (long runs of one owner)
ids = (torch.arange(n, device="cuda", dtype=torch.int64) * nb // n).to(torch.int32)
for _ in range(3):
    partition(ids, nb, check=False)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(5):
    partition(ids, nb, check=False)
e1.record(); torch.cuda.synchronize()
print("ms", e0.elapsed_time(e1) / 5)
