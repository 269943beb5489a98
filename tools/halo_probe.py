"""K3 timing on the 32768^2 stencil launch (decompose block mapper, 8 processors)."""
import sys
sys.path.insert(0, ".")
import torch
from paper_2507_17087_b200.dsl import compile_mapper, parse
from paper_2507_17087_b200.spaces import MachineShape
from paper_2507_17087_b200.transfer import halo_lists

L = int(sys.argv[1]) if len(sys.argv) > 1 else 32768
src = ("m = Machine(GPU)\ndef blk(Tuple p, Tuple s):\n"
       "    q = m.merge(0, 1).decompose(0, s)\n    return q[*(p * q.size / s)]\n"
       "IndexTaskMap t blk\n")
fn = compile_mapper(parse(src), "t", MachineShape("GPU", 1, 8))
owner = fn.map_ispace((L, L))
r = halo_lists(owner, (L, L), (1, 1), 8)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(3):
    r = halo_lists(owner, (L, L), (1, 1), 8)
e1.record()
torch.cuda.synchronize()
print({"k3_ms": round(e0.elapsed_time(e1) / 3, 3)})
