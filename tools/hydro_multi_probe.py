"""Where the multi-GPU hydro step's time goes (torchrun, one rank per GPU): the full step
(barrier, zones, barrier, points), the two kernels alone with the barriers left out (timing
only -- the result is not valid then), and the barrier kernel alone; max over ranks."""
import ctypes
import json
import os
import sys

sys.path.insert(0, ".")
import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402

from paper_2507_17087_b200 import native  # noqa: E402
from paper_2507_17087_b200.executors.hydro import HydroSpec, MappedHydro  # noqa: E402


def timed(fn, reps, world):
    torch.cuda.synchronize()
    dist.barrier()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        fn()
    e1.record()
    torch.cuda.synchronize()
    t = torch.tensor([e0.elapsed_time(e1) / reps], device="cuda")
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return round(float(t), 4)


def main():
    rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
    torch.cuda.set_device(int(os.environ.get("LOCAL_RANK", rank)))
    dist.init_process_group("nccl", device_id=torch.device("cuda", torch.cuda.current_device()))
    lib = native.lib()
    out = {"world": world}
    for mapping in ("decompose", "heuristic"):
        ex = MappedHydro(HydroSpec(16384, 4096), mapping=mapping, rank=rank, world=world)
        cs = native.stream_ptr(torch.cuda.current_stream())
        for _ in range(3):
            ex.step()
        r = {"step": timed(ex.step, 20, world)}
        r["zones_only"] = timed(lambda: lib.pm_hydro_step(ctypes.byref(ex.view), 0, cs), 20, world)
        r["points_only"] = timed(lambda: lib.pm_hydro_step(ctypes.byref(ex.view), 1, cs), 20, world)
        r["barrier_only"] = timed(lambda: ex._barrier(), 50, world)
        r["zones"] = int(ex.view.n_zones)
        r["points"] = int(ex.view.n_points)
        zs = [None] * world
        dist.all_gather_object(zs, (r["zones"], r["points"]))
        r["zones_points_per_rank"] = zs
        out[mapping] = r
        dist.barrier()
        ex.close()
        del ex
        torch.cuda.empty_cache()
    if rank == 0:
        print(json.dumps(out))
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
