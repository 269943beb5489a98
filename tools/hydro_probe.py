"""Per-phase timing of the PENNANT-style step on one GPU (ncu target too)."""
import ctypes
import sys
sys.path.insert(0, ".")
import torch
from paper_2507_17087_b200 import native
from paper_2507_17087_b200.executors.hydro import HydroSpec, MappedHydro

zx, zy = (int(sys.argv[1]), int(sys.argv[2])) if len(sys.argv) > 2 else (16384, 4096)
ex = MappedHydro(HydroSpec(zx, zy))
lib = native.lib()
cs = native.stream_ptr(torch.cuda.current_stream())
for _ in range(3):
    ex.step()
torch.cuda.synchronize()
e = [torch.cuda.Event(enable_timing=True) for _ in range(3)]
t = [0.0, 0.0]
reps = 10
for _ in range(reps):
    e[0].record()
    lib.pm_hydro_step(ctypes.byref(ex.view), 0, cs)
    e[1].record()
    lib.pm_hydro_step(ctypes.byref(ex.view), 1, cs)
    e[2].record()
    torch.cuda.synchronize()
    t[0] += e[0].elapsed_time(e[1]) / reps
    t[1] += e[1].elapsed_time(e[2]) / reps
print({"zones_ms": round(t[0], 4), "points_ms": round(t[1], 4), "zones": zx * zy})
