"""Johnson / COSMA 3-D multiplies under both mappings (torchrun, one rank per GPU):
ms per step, max over ranks.  For A/B of GEMM knobs on the K-split (reduce-adding) grids."""
import json
import os
import sys

sys.path.insert(0, ".")
import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402

from paper_2507_17087_b200.executors.grid3d import MappedGemm3D  # noqa: E402


def main():
    rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
    torch.cuda.set_device(int(os.environ.get("LOCAL_RANK", rank)))
    dist.init_process_group("nccl", device_id=torch.device("cuda", torch.cuda.current_device()))
    out = {"world": world, "env": {k: v for k, v in os.environ.items() if k.startswith("PM_")}}
    shapes = {"johnson": (32768, 32768, 32768), "cosma": (65536, 16384, 16384)}
    only = os.environ.get("PROBE_SHAPES")
    if only:
        shapes = {k: v for k, v in shapes.items() if k in only.split(",")}
    maps = os.environ.get("PROBE_MAPPINGS", "decompose,heuristic").split(",")
    for name, (M, N, K) in shapes.items():
        for mapping in maps:
            ex = MappedGemm3D(M, N, K, mapping=mapping, rank=rank, world=world, seed=99)
            for _ in range(3):
                ex.step()
            ex.result()
            torch.cuda.synchronize()
            dist.barrier()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            for _ in range(5):
                ex.step()
            ex.result()
            e1.record()
            torch.cuda.synchronize()
            t = torch.tensor([e0.elapsed_time(e1) / 5], device="cuda")
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            ms = float(t)
            out[f"{name}_{mapping}"] = {"grid": list(ex.grid), "ms": round(ms, 3),
                                        "tflops": round(2.0 * M * N * K / ms / 1e9, 1)}
            ex.close()
            del ex
            torch.cuda.empty_cache()
            dist.barrier()
    if rank == 0:
        print(json.dumps(out))
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
