"""HBM write ceiling vs the K2 scatter: fill_ / zero_ of 4.29 GB (1.07e9 int32) and the K2
partition of 1.07e9 block-structured ids (tools/k2_probe.py), CUDA events, 5 reps each."""
import sys
sys.path.insert(0, ".")
import torch  # noqa: E402
from paper_2507_17087_b200.ownership import partition  # noqa: E402

n = 1 << 30
x = torch.empty(n, dtype=torch.int32, device="cuda")
ids = (torch.arange(n, device="cuda", dtype=torch.int64) * 8 // n).to(torch.int32)


def t(fn, reps=5):
    for _ in range(2):
        fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps


for name, fn in (("fill_", lambda: x.fill_(7)), ("zero_", lambda: x.zero_()),
                 ("copy (r+w)", lambda: x.copy_(ids)),
                 ("k2 partition", lambda: partition(ids, 8, check=False))):
    ms = t(fn)
    print(f"{name:14s} {ms:.4f} ms  {4 * n / ms / 1e6:.0f} GB/s (4 B/elem)")
