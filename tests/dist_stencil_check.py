"""Multi-GPU check of the mapped stencil with the fused NVLink halo exchange
against the float64 oracle (run under torchrun, one rank per GPU)."""

import json
import os
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))

import numpy as np  # noqa: E402
import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402

from oracle.numerics import jacobi5  # noqa: E402
from paper_2507_17087_b200.executors.stencil import MappedStencil, init_grid  # noqa: E402


def main():
    rank, world = int(os.environ.get("RANK", 0)), int(os.environ.get("WORLD_SIZE", 1))
    # PM_TEST_BACKEND=gloo: host collectives over gloo, so more ranks than GPUs can
    # share the box (rank r on GPU r % n; peers on the same GPU through CUDA IPC) --
    # exercises the 8-GPU paths on a 4-GPU box; the executors' data path has no NCCL
    backend = os.environ.get("PM_TEST_BACKEND", "nccl")
    local = int(os.environ.get("LOCAL_RANK", rank)) % torch.cuda.device_count()
    torch.cuda.set_device(local)
    if world > 1:
        dist.init_process_group(backend, **({"device_id": torch.device("cuda", local)}
                                            if backend == "nccl" else {}))
    out = []
    for rows, cols, sweeps in [(64, 96, 7), (300, 2100, 5), (1024, 4096, 12)]:
        for mapping in ("decompose", "heuristic"):
            ex = MappedStencil(rows, cols, mapping=mapping, rank=rank, world=world, seed=3)
            ex.run(sweeps)
            ex.run(sweeps)  # a second batch continues the flag protocol
            torch.cuda.synchronize()
            got = ex.current().double().cpu().numpy()
            g0 = init_grid((0, rows), (0, cols), cols, 3, "cuda").double().cpu().numpy()
            want = jacobi5(g0, 2 * sweeps)
            r0, r1, c0, c1 = ex.rects[rank]
            err = float(np.abs(got - want[r0:r1, c0:c1]).max())
            out.append({"shape": [rows, cols], "mapping": mapping, "grid": list(ex.grid),
                        "rank": rank, "err": err, "halo_cells": ex.halo_cells,
                        "model_halo": ex.model_halo})
            if world > 1:
                dist.barrier()
            ex.close()
    allr = [out]
    if world > 1:
        allr = [None] * world
        dist.all_gather_object(allr, out)
    if rank == 0:
        flat = [r for rs in allr for r in rs]
        ok = all(r["err"] < 1e-5 and r["halo_cells"] == r["model_halo"] for r in flat)
        print(json.dumps({"ok": ok, "world": world, "results": flat}))
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
