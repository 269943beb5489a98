"""K3 timing on the 32768^2 stencil launch (decompose block mapper, 8 processors):
the whole halo_lists call and its count pass alone (counts_only)."""
import sys
sys.path.insert(0, ".")
import torch
from paper_2507_17087_b200.dsl import compile_mapper, parse
from paper_2507_17087_b200.spaces import MachineShape
from paper_2507_17087_b200.transfer import halo_lists

L = int(sys.argv[1]) if len(sys.argv) > 1 else 32768
P = int(sys.argv[2]) if len(sys.argv) > 2 else 8
src = ("m = Machine(GPU)\ndef blk(Tuple p, Tuple s):\n"
       "    q = m.merge(0, 1).decompose(0, s)\n    return q[*(p * q.size / s)]\n"
       "IndexTaskMap t blk\n")
fn = compile_mapper(parse(src), "t", MachineShape("GPU", 1, P))
owner = fn.map_ispace((L, L))
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
out = {"L": L, "P": P}
cap = halo_lists(owner, (L, L), (1, 1), P).total
for name, kw in (("k3_ms", {}), ("k3_cap_ms", {"capacity": cap}),
                 ("count_ms", {"counts_only": True})):
    r = halo_lists(owner, (L, L), (1, 1), P, **kw)
    torch.cuda.synchronize()
    e0.record()
    for _ in range(10):
        r = halo_lists(owner, (L, L), (1, 1), P, **kw)
    e1.record()
    torch.cuda.synchronize()
    out[name] = round(e0.elapsed_time(e1) / 10, 4)
out["entries"] = r.total
out["count_gbs"] = round(4 * L * L / (out["count_ms"] * 1e-3) / 1e9, 1)
out["k3_gbs"] = round((4 * L * L + 9 * r.total) / (out["k3_ms"] * 1e-3) / 1e9, 1)
out["k3_cap_gbs"] = round((4 * L * L + 9 * r.total) / (out["k3_cap_ms"] * 1e-3) / 1e9, 1)
print(out)
