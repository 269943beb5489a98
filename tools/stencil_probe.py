"""Single-GPU stencil sweep rate (cells/s, fraction of HBM) for tile-height experiments."""
import sys, json
sys.path.insert(0, ".")
import torch
from paper_2507_17087_b200.executors.stencil import MappedStencil
L = int(sys.argv[1]) if len(sys.argv) > 1 else 32768
ex = MappedStencil(L, L, halo_check=False)
ex.run(10); torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record(); ex.run(40); e1.record(); torch.cuda.synchronize()
ms = e0.elapsed_time(e1) / 40
print(json.dumps({"ms_per_sweep": ms, "cells_per_s": L * L / ms * 1e3, "gbs": 8 * L * L / ms / 1e6}))
