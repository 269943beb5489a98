"""Multi-rank check of the peer-memory barriers (csrc/barrier.cu) used by the
Cannon / 2.5D / 3-D executors: `PeerBarrier.copy_then_wait` (SM copies + the
barrier in one launch) with cross-rank pushes, checked for data and ordering,
and the plain `PeerBarrier()` ordering a peer store against the next round.

Round t: every rank pushes its round-t pattern into the right neighbour's
inbox (a peer pointer) with copy_then_wait; once that returns on the stream,
the inbox must already hold the left neighbour's round-t pattern (the
barrier orders every rank's copies before anyone continues).  A device-side
mismatch counter is read once at the end.  Run under torchrun (NCCL, one rank
per GPU) or with PM_TEST_BACKEND=gloo (ranks sharing GPUs).
"""

import json
import os
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))

import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402

from paper_2507_17087_b200.peer import PeerBarrier, PeerBuffers  # noqa: E402


def main():
    rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
    backend = os.environ.get("PM_TEST_BACKEND", "nccl")
    local = int(os.environ.get("LOCAL_RANK", rank)) % torch.cuda.device_count()
    torch.cuda.set_device(local)
    dist.init_process_group(backend, **({"device_id": torch.device("cuda", local)}
                                        if backend == "nccl" else {}))
    dev = torch.device("cuda", local)
    words = 1 << 16  # 256 KiB per copy: spread over many CTAs of the copy kernel
    rounds = 12
    inbox = torch.zeros(2, words, dtype=torch.int32, device=dev)
    out = torch.zeros(rounds, words, dtype=torch.int32, device=dev)
    for t in range(rounds):
        out[t] = (rank * 1000003 + t * 7919 + torch.arange(words, device=dev)) % (1 << 30)
    peers = PeerBuffers({"inbox": inbox}, rank, world)
    bar = PeerBarrier(rank, world)
    bad = torch.zeros(1, dtype=torch.int64, device=dev)
    right, left = (rank + 1) % world, (rank - 1) % world
    cs = torch.cuda.current_stream()
    expect = [(left * 1000003 + t * 7919 + torch.arange(words, device=dev)) % (1 << 30)
              for t in range(rounds)]
    torch.cuda.synchronize()
    dist.barrier()
    for t in range(rounds):
        slot = t % 2
        dst = peers.ptrs["inbox"][right] + slot * words * 4
        bar.copy_then_wait([(dst, out[t].data_ptr(), words * 4)], cs)
        bad += (inbox[slot] != expect[t]).sum()
        # the slot is overwritten two rounds later: everyone has checked it by then
        bar(cs)
    # mixed: a copy list of several pieces, including a local one
    pieces = [(peers.ptrs["inbox"][right], out[0].data_ptr(), 4096 * 4),
              (peers.ptrs["inbox"][right] + 4096 * 4, out[1].data_ptr() + 4096 * 4, 8192 * 4),
              (inbox[1].data_ptr(), out[2].data_ptr(), 1024 * 4)]
    bar.copy_then_wait(pieces, cs)
    bad += (inbox[0, :4096] != expect[0][:4096]).sum()
    bad += (inbox[0, 4096:12288] != expect[1][4096:12288]).sum()
    bad += (inbox[1, :1024] != out[2][:1024]).sum()
    bar(cs)
    torch.cuda.synchronize()
    res = {"rank": rank, "mismatches": int(bad.item())}
    allr = [None] * world
    dist.all_gather_object(allr, res)
    if rank == 0:
        print(json.dumps({"ok": all(r["mismatches"] == 0 for r in allr), "world": world,
                          "results": allr}))
    dist.barrier()
    bar.close()
    peers.close()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
