"""Multi-GPU stencil sweep time per mapping (torchrun, one rank per GPU): per-rank and
max-over-ranks ms/sweep; PM_STENCIL_TR selects the tile height."""
import json
import os
import sys

sys.path.insert(0, ".")
import torch
import torch.distributed as dist
from paper_2507_17087_b200.executors.stencil import MappedStencil

rank, world = int(os.environ.get("RANK", 0)), int(os.environ.get("WORLD_SIZE", 1))
torch.cuda.set_device(int(os.environ.get("LOCAL_RANK", rank)))
if world > 1:
    dist.init_process_group("nccl", device_id=torch.device("cuda", torch.cuda.current_device()))
rows, cols = int(sys.argv[1]), int(sys.argv[2])
out = {"rows": rows, "cols": cols, "tr": os.environ.get("PM_STENCIL_TR", "16")}
for mapping in ("decompose", "heuristic"):
    ex = MappedStencil(rows, cols, mapping=mapping, rank=rank, world=world, halo_check=False)
    ex.run(10)
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    ex.run(40)
    e1.record()
    torch.cuda.synchronize()
    ms = torch.tensor([e0.elapsed_time(e1) / 40], device="cuda")
    allms = [torch.zeros_like(ms) for _ in range(world)]
    if world > 1:
        dist.all_gather(allms, ms)
    else:
        allms = [ms]
    out[mapping] = {"grid": list(ex.grid), "rect": [ex.mr, ex.mc],
                    "ms": [round(float(x), 4) for x in allms]}
    if world > 1:
        dist.barrier()
    ex.close()
    del ex
    torch.cuda.empty_cache()
if rank == 0:
    print(json.dumps(out))
if world > 1:
    dist.destroy_process_group()
