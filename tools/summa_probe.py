"""Per-rank anatomy of the mapped SUMMA step (torchrun, one rank per GPU): the step time
of every rank, and from an instrumented pass each GEMM launch's start / end on the compute
stream relative to the step start (idle = waiting for pulls or launch gaps)."""
import json
import os
import sys

sys.path.insert(0, ".")
import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402

from paper_2507_17087_b200.executors.summa import MappedGemm  # noqa: E402
from paper_2507_17087_b200.gemm import tile_gemm  # noqa: E402


def main():
    rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
    torch.cuda.set_device(int(os.environ.get("LOCAL_RANK", rank)))
    dist.init_process_group("nccl", device_id=torch.device("cuda", torch.cuda.current_device()))
    S = int(os.environ.get("PROBE_SIZE", "32768"))
    lanes = int(os.environ.get("PROBE_LANES", "4"))
    ex = MappedGemm(S, S, S, mapping="decompose", rank=rank, world=world, seed=1,
                    copy_streams=lanes)
    cs = torch.cuda.current_stream()
    for _ in range(3):
        ex.step()
    torch.cuda.synchronize()
    dist.barrier()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(cs)
    for _ in range(10):
        ex.step()
    e1.record(cs)
    torch.cuda.synchronize()
    step_ms = e0.elapsed_time(e1) / 10
    # instrumented pass (op by op, events around every launch)
    dist.barrier()
    t0 = torch.cuda.Event(enable_timing=True)
    for s in ex.copy_streams:
        s.wait_event(ex.done)
    t0.record(cs)
    pull_marks = []
    for name, q, row0, rows, k0, k1, si, ev in ex.pulls:
        st = ex.copy_streams[si]
        st.wait_event(t0)
        ex._copy(name, q, row0, rows, k0, k1, st)
        ev.record(st)
        pe = torch.cuda.Event(enable_timing=True)
        pe.record(st)
        pull_marks.append((pe, (name, q, rows, k1 - k0, si)))
    marks = []
    for r0, r1, k0, k1, acc, evs, c0, c1 in ex.gemms:
        for ev in evs:
            cs.wait_event(ev)
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(cs)
        tile_gemm(ex.A[r0:r1, k0:k1], ex.Bt[c0:c1, k0:k1], ex.C[r0:r1, c0:c1], accumulate=acc,
                  stream=cs)
        b.record(cs)
        marks.append((a, b, (r1 - r0, c1 - c0, k1 - k0)))
    ex.done.record(cs)
    torch.cuda.synchronize()
    launches = [{"start": round(t0.elapsed_time(a), 3), "ms": round(a.elapsed_time(b), 3),
                 "mnk": mnk, "tflops": round(2 * mnk[0] * mnk[1] * mnk[2] / a.elapsed_time(b) / 1e9)}
                for a, b, mnk in marks]
    pulls = [{"done": round(t0.elapsed_time(e), 3), "what": w, "mb": w[2] * w[3] * 2 / 1e6}
             for e, w in pull_marks]
    res = {"rank": rank, "step_ms": round(step_ms, 3), "launches": launches, "pulls": pulls}
    allr = [None] * world
    dist.all_gather_object(allr, res)
    if rank == 0:
        print(json.dumps(allr))
    ex.close()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
