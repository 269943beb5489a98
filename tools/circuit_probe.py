"""One GPU circuit iteration timing (ncu target): 96 pieces x 20000 wires, 1000 steps."""
import sys
sys.path.insert(0, ".")
import torch
from paper_2507_17087_b200.executors.circuit import CircuitSpec, MappedCircuit

steps = int(sys.argv[1]) if len(sys.argv) > 1 else 1000
ex = MappedCircuit(CircuitSpec(96, 5000, 20000, steps=steps, seed=7))
ex.step()
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(3):
    ex.step()
e1.record()
torch.cuda.synchronize()
ms = e0.elapsed_time(e1) / 3
w = ex.work()
print({"ms_per_iteration": round(ms, 3), "fp32_ops_per_s": w["fp32_ops"] / (ms * 1e-3)})
