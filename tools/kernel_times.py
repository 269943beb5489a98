"""Warm per-kernel device times (torch.profiler / CUPTI, no replay) of K1, K2, fused K1+K2 and
K3 on the 32768^2 launch: which pass of each call holds the time."""
import sys
sys.path.insert(0, ".")
import torch  # noqa: E402
from torch.profiler import ProfilerActivity, profile  # noqa: E402

from paper_2507_17087_b200.dsl import compile_mapper, parse  # noqa: E402
from paper_2507_17087_b200.ownership import partition  # noqa: E402
from paper_2507_17087_b200.spaces import MachineShape  # noqa: E402
from paper_2507_17087_b200.transfer import halo_lists  # noqa: E402

src = ("m = Machine(GPU)\ndef blk(Tuple p, Tuple s):\n"
       "    q = m.merge(0, 1).decompose(0, s)\n    return q[*(p * q.size / s)]\n"
       "IndexTaskMap t blk\n")
L = 32768
fn = compile_mapper(parse(src), "t", MachineShape("GPU", 1, 8))
ids = fn.map_ispace((L, L))
partition(ids, 8)
fn.map_partition((L, L))
cap = halo_lists(ids, (L, L), (1, 1), 8).total
for _ in range(2):
    halo_lists(ids, (L, L), (1, 1), 8, capacity=cap)
torch.cuda.synchronize()
with profile(activities=[ProfilerActivity.CUDA]) as prof:
    for _ in range(5):
        fn.map_ispace((L, L), out=ids, check=False)
        partition(ids, 8, check=False)
        fn.map_partition((L, L), check=False)
        halo_lists(ids, (L, L), (1, 1), 8, capacity=cap)
    torch.cuda.synchronize()
print(prof.key_averages().table(sort_by="cuda_time_total", row_limit=25, max_name_column_width=70))
