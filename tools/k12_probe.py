"""K1 / K2 / fused K1+K2 timings on the 32768^2 stencil launch (ncu target too)."""
import sys
sys.path.insert(0, ".")
import torch
from paper_2507_17087_b200.dsl import compile_mapper, parse
from paper_2507_17087_b200.ownership import partition
from paper_2507_17087_b200.spaces import MachineShape

SRC = """
m = Machine(GPU)
def blk(Tuple p, Tuple s):
    q = m.merge(0, 1).decompose(0, s)
    return q[*(p * q.size / s)]
def cyc(Tuple p, Tuple s):
    q = m.merge(0, 1)
    return q[(p[0] * 7 + p[1] * 13) % q.size[0]]
IndexTaskMap blk blk
IndexTaskMap cyc cyc
"""
L = 32768
reps = int(sys.argv[1]) if len(sys.argv) > 1 else 10
for task in ("blk", "cyc"):
    fn = compile_mapper(parse(SRC), task, MachineShape("GPU", 1, 8))
    ids = fn.map_ispace((L, L))
    partition(ids, 8)
    fn.map_partition((L, L))
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    res = {}
    for name, f in (("k1", lambda: fn.map_ispace((L, L), out=ids, check=False)),
                    ("k2", lambda: partition(ids, 8, check=False)),
                    ("k12", lambda: fn.map_partition((L, L), check=False))):
        e0.record()
        for _ in range(reps):
            f()
        e1.record()
        torch.cuda.synchronize()
        res[name] = round(e0.elapsed_time(e1) / reps, 3)
    print(task, res, flush=True)
