"""Dump one circuit step's state (tools/circuit_exact.py OUT.npz), to compare the packed
FP32-pair wire kernel with the scalar one bit for bit (PM_CIRCUIT_SCALAR=1)."""
import sys
sys.path.insert(0, ".")
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2507_17087_b200.executors.circuit import CircuitSpec, MappedCircuit  # noqa: E402

ex = MappedCircuit(CircuitSpec(8, 500, 2000, steps=50, seed=3))
for _ in range(3):
    ex.step()
torch.cuda.synchronize()
arrs = {k: getattr(ex, k).detach().cpu().numpy() for k in ("current", "wire_volt", "volt")
        if hasattr(ex, k)}
np.savez(sys.argv[1], **arrs)
print({k: a.shape for k, a in arrs.items()})
