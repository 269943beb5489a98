"""Multi-GPU check of the 3-D executor (Johnson / COSMA grids) with the fused
GEMM + reduce-scatter over NVLink.  Run under torchrun, one rank per GPU.

    torchrun --nproc-per-node N --master-addr 127.0.0.1 tests/dist_grid3d_check.py
"""

import json
import os
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))

import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402

from paper_2507_17087_b200.executors.grid3d import MappedGemm3D  # noqa: E402
from paper_2507_17087_b200.executors.summa import synth  # noqa: E402


def main():
    rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
    # PM_TEST_BACKEND=gloo: host collectives over gloo, so more ranks than GPUs can
    # share the box (rank r on GPU r % n; peers on the same GPU through CUDA IPC) --
    # exercises the 8-GPU paths on a 4-GPU box; the executors' data path has no NCCL
    backend = os.environ.get("PM_TEST_BACKEND", "nccl")
    local = int(os.environ.get("LOCAL_RANK", rank)) % torch.cuda.device_count()
    torch.cuda.set_device(local)
    dist.init_process_group(backend, **({"device_id": torch.device("cuda", local)}
                                            if backend == "nccl" else {}))
    out = []
    shapes = [(2048, 1024, 2048), (4096, 1024, 1024), (1024, 1536, 3072)]
    for M, N, K in shapes:
        for mapping in ("decompose", "heuristic"):
            ex = MappedGemm3D(M, N, K, mapping=mapping, rank=rank, world=world, seed=5)
            for _ in range(3):  # exercise the double-buffered C and the barriers
                ex.step()
            C = ex.result()
            torch.cuda.synchronize()
            r0 = ex.rows[0] + ex.my_rows[0]
            r1 = ex.rows[0] + ex.my_rows[1]
            A = synth((r0, r1), (0, K), K, 5, "cuda").double()
            Bt = synth(ex.cols, (0, K), K, 6, "cuda").double()
            R = A @ Bt.T
            err = float((C.double() - R).abs().max() / R.abs().max()) if R.numel() else 0.0
            out.append({"shape": [M, N, K], "mapping": mapping, "grid": list(ex.grid),
                        "rank": rank, "err": err, "comm": ex.comm})
            dist.barrier()
            ex.close()
    allr = [None] * world
    dist.all_gather_object(allr, out)
    if rank == 0:
        flat = [r for rs in allr for r in rs]
        print(json.dumps({"ok": all(r["err"] < 1e-3 for r in flat), "world": world,
                          "results": flat}))
    dist.barrier()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
