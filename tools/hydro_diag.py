"""Hydro 8-rank diagnosis: run-to-run spread and distance to a single-GPU run of the
same mesh (PM_TEST_BACKEND=gloo for oversubscribed ranks)."""
import json
import os
import sys

sys.path.insert(0, ".")
import numpy as np
import torch
import torch.distributed as dist
from paper_2507_17087_b200.executors.hydro import HydroSpec, MappedHydro

rank, world = int(os.environ.get("RANK", 0)), int(os.environ.get("WORLD_SIZE", 1))
backend = os.environ.get("PM_TEST_BACKEND", "nccl")
torch.cuda.set_device(int(os.environ.get("LOCAL_RANK", rank)) % torch.cuda.device_count())
dist.init_process_group(backend)
Lx, Ly, steps = 48, 40, int(sys.argv[1]) if len(sys.argv) > 1 else 20


def run(w, r):
    ex = MappedHydro(HydroSpec(Lx, Ly), mapping="decompose", rank=r, world=w,
                     group=None if w > 1 else None)
    for _ in range(steps):
        ex.step()
    torch.cuda.synchronize()
    n = ex.point_ids.numel()
    out = {int(p): (float(u), float(v)) for p, u, v in
           zip(ex.point_ids.tolist(), ex.ux[:n].tolist(), ex.uy[:n].tolist())}
    return out


a = run(world, rank)
dist.barrier()
b = run(world, rank)
dist.barrier()
# single-GPU reference of the same mesh in this process (world 1: no peers)
os.environ["WORLD_SIZE"] = "1"
ref = MappedHydro(HydroSpec(Lx, Ly), mapping="decompose", rank=0, world=1)
for _ in range(steps):
    ref.step()
torch.cuda.synchronize()
R = {int(p): (float(u), float(v)) for p, u, v in
     zip(ref.point_ids.tolist(), ref.ux.tolist(), ref.uy.tolist())}
umax = max(abs(x) for uv in R.values() for x in uv) or 1.0
runrun = max(abs(a[p][i] - b[p][i]) for p in a for i in (0, 1)) / umax
vs1 = max(abs(a[p][i] - R[p][i]) for p in a for i in (0, 1)) / umax
worst = max(a, key=lambda p: abs(a[p][0] - R[p][0]) + abs(a[p][1] - R[p][1]))
res = [None] * world
dist.all_gather_object(res, {"rank": rank, "run_to_run": runrun, "vs_world1": vs1,
                             "worst_point": worst, "worst": [a[worst], R[worst]],
                             "npts": len(a)})
if rank == 0:
    print(json.dumps({"steps": steps, "results": res}))
dist.barrier()
dist.destroy_process_group()
