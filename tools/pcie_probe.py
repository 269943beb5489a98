"""Host <-> GPU copy bandwidth with every rank copying at once (torchrun, one rank per GPU):
the ceiling of bench.py's e2e leg.  Per rank: H2D alone, D2H alone, both concurrently, for a
contiguous 1 GiB pinned buffer and for the strided column slice the SUMMA e2e copies."""
import json
import os
import sys

sys.path.insert(0, ".")
import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402


def timed(fn, reps=3):
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
    return float(t)


def main():
    rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
    torch.cuda.set_device(int(os.environ.get("LOCAL_RANK", rank)))
    dist.init_process_group("nccl", device_id=torch.device("cuda", torch.cuda.current_device()))
    n = 1 << 30
    h = torch.empty(n, dtype=torch.uint8).pin_memory()
    h2 = torch.empty(n, dtype=torch.uint8).pin_memory()
    d = torch.empty(n, dtype=torch.uint8, device="cuda")
    d2 = torch.empty(n, dtype=torch.uint8, device="cuda")
    s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
    out = {"world": world}

    def both():
        cur = torch.cuda.current_stream()
        s1.wait_stream(cur)
        s2.wait_stream(cur)
        with torch.cuda.stream(s1):
            d.copy_(h, non_blocking=True)
        with torch.cuda.stream(s2):
            h2.copy_(d2, non_blocking=True)
        cur.wait_stream(s1)
        cur.wait_stream(s2)

    out["h2d_ms"] = timed(lambda: d.copy_(h, non_blocking=True))
    out["d2h_ms"] = timed(lambda: h2.copy_(d2, non_blocking=True))
    out["both_ms"] = timed(both)
    gb = n / 1e9
    out["h2d_gbs_per_gpu"] = gb / out["h2d_ms"] * 1e3
    out["d2h_gbs_per_gpu"] = gb / out["d2h_ms"] * 1e3
    out["both_gbs_per_gpu"] = 2 * gb / out["both_ms"] * 1e3
    out["total_both_gbs"] = out["both_gbs_per_gpu"] * world
    # strided: 16 KB rows out of 64 KB host rows (a 1/4 column slice of a bf16 32768-wide
    # matrix), 1 GiB moved
    rows = n // (16 << 10)
    hs = torch.empty(rows, 64 << 10, dtype=torch.uint8).pin_memory()
    ds = torch.empty(rows, 16 << 10, dtype=torch.uint8, device="cuda")
    out["h2d_strided_ms"] = timed(lambda: ds.copy_(hs[:, :16 << 10], non_blocking=True))
    out["h2d_strided_gbs_per_gpu"] = gb / out["h2d_strided_ms"] * 1e3
    allr = [None] * world
    dist.all_gather_object(allr, out)
    if rank == 0:
        print(json.dumps(allr[0]))
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
