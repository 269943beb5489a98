"""Feasibility / regression check: the GEMM's TMA reduce-add epilogue writing
into a PEER GPU's buffer over NVLink (CUDA IPC mapping).  Both ranks add their
partial product into rank 0's C and into their own C; rank 0 checks the sum.

    torchrun --nproc-per-node 2 --master-addr 127.0.0.1 tests/dist_peer_gemm_check.py
"""

import json
import os
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))

import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402

from paper_2507_17087_b200 import native  # noqa: E402
from paper_2507_17087_b200.executors.summa import synth  # noqa: E402
from paper_2507_17087_b200.peer import PeerBuffers  # noqa: E402


def main():
    rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
    torch.cuda.set_device(rank)
    dist.init_process_group("nccl", device_id=torch.device("cuda", rank))
    M, N, K = 2048, 1024, 512
    A = synth((rank * M, (rank + 1) * M), (0, K), K, 3, "cuda")
    Bt = synth((0, N), (0, K), K, 4, "cuda")
    C = torch.zeros(M, N, device="cuda")
    peers = PeerBuffers({"C": C}, rank, world)
    torch.cuda.synchronize()
    dist.barrier()
    lib = native.lib()
    for dst in range(world):  # add my partial into every rank's C
        native.check(lib.pm_gemm_bf16(A.data_ptr(), K, Bt.data_ptr(), K, peers.ptrs["C"][dst], N,
                                      M, N, K, 0, 1, native.stream_ptr()), "pm_gemm_bf16")
    torch.cuda.synchronize()
    dist.barrier()
    want = sum(synth((r * M, (r + 1) * M), (0, K), K, 3, "cuda").double() for r in range(world))
    want = want @ Bt.double().T
    err = float((C.double() - want).abs().max() / want.abs().max())
    errs = [None] * world
    dist.all_gather_object(errs, err)
    if rank == 0:
        print(json.dumps({"ok": max(errs) < 1e-4, "errs": errs}))
    dist.barrier()
    peers.close()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
