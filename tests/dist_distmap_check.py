"""Multi-GPU check of the sharded launch mapping (distmap.map_launch_sharded;
torchrun, one rank per GPU): K1 + K2 per chunk, NCCL count all-gather and
ownership all-to-all-v.  Small launches vs the oracle's shard-tree leaves;
the 32768^2 stencil launch vs a one-GPU K1 + K2 of the whole launch; errors
raised identically on every rank (lowest failing point wins)."""

import json
import os
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))

import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402

from oracle import mapple_oracle as O  # noqa: E402
from paper_2507_17087_b200 import distmap  # noqa: E402
from paper_2507_17087_b200.dsl import compile_mapper, parse  # noqa: E402
from paper_2507_17087_b200.ownership import partition  # noqa: E402
from paper_2507_17087_b200.spaces import MachineShape  # noqa: E402

MAPPERS = """
m = Machine(GPU)
def blk(Tuple p, Tuple s):
    q = m.merge(0, 1).decompose(0, s)
    return q[*(p * q.size / s)]
def cyc(Tuple p, Tuple s):
    q = m.merge(0, 1)
    return q[(p[0] * 7 + p[1] * 3) % q.size[0]]
def bad(Tuple p, Tuple s):
    q = m.merge(0, 1)
    a = (p[0] == 5) ? 99 : 0
    b = 4 / (13 - p[0])
    return q[a + b * 0]
IndexTaskMap blk blk
IndexTaskMap cyc cyc
IndexTaskMap bad bad
"""


def main():
    rank, world = int(os.environ.get("RANK", 0)), int(os.environ.get("WORLD_SIZE", 1))
    local = int(os.environ.get("LOCAL_RANK", rank))
    torch.cuda.set_device(local)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    prog = parse(MAPPERS)
    res = []
    for task, machine, ispace in [("blk", (2, 4), (40, 52)), ("cyc", (1, 6), (33, 17)),
                                  ("blk", (1, 8), (7, 9))]:
        fn = compile_mapper(prog, task, MachineShape("GPU", *machine))
        ids = O.map_launch(prog, task, ("GPU", *machine), ispace)
        pts = O.row_major(ispace)
        leaves = O.shard_leaves(task, pts, [divmod(x, machine[1]) for x in ids])
        P = machine[0] * machine[1]
        for fused in (True, False):
            for exchange in (True, False):
                sh = distmap.map_launch_sharded(fn, ispace, rank=rank, world=world,
                                                fused=fused, exchange=exchange)
                mine = {p: sh.lists[p].tolist() for p in sh.procs}
                allr = [mine]
                if world > 1:
                    allr = [None] * world
                    dist.all_gather_object(allr, mine)
                if exchange:
                    got = {p: v for d in allr for p, v in d.items()}
                else:  # chunk-major concatenation == the global list
                    got = {p: [x for d in allr for x in d[p]] for p in range(P)}
                ok = sorted(got) == list(range(P))
                for _, (tgt, lpts) in leaves.items():
                    p = tgt[0] * machine[1] + tgt[1]
                    ok &= [pts[i] for i in got.get(p, [])] == list(lpts)
                ok &= all(len(got[p]) == 0 for p in got if p not in
                          {t[0] * machine[1] + t[1] for t, _ in leaves.values()})
                res.append({"case": f"{task} {machine} {ispace} fused={fused} "
                            f"exchange={exchange}", "ok": bool(ok)})
    # the 32768^2 stencil launch (configs[4]) on 8 processors vs one-GPU K1 + K2
    L = 32768
    fn = compile_mapper(prog, "blk", MachineShape("GPU", 1, 8))
    sh = distmap.map_launch_sharded(fn, (L, L), rank=rank, world=world)
    full = partition(fn.map_ispace((L, L)), 8)
    ok = True
    for p in sh.procs:
        ref = full.points_of(p)
        ok &= bool(sh.lists[p].numel() == ref.numel() and torch.equal(sh.lists[p].long(), ref.long()))
    ok &= sh.totals == full.counts.tolist()
    del full
    res.append({"case": "stencil 32768^2 blk (1,8)", "ok": bool(ok), "rank": rank})
    # timing: K1 + K2 + all-gather + all-to-all, strong scaling of the 1.07e9-point launch
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(3):
        distmap.map_launch_sharded(fn, (L, L), rank=rank, world=world)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / 3
    e0.record()
    for _ in range(3):
        distmap.map_launch_sharded(fn, (L, L), rank=rank, world=world, exchange=False)
    e1.record()
    torch.cuda.synchronize()
    ms_local = e0.elapsed_time(e1) / 3
    lo, hi = distmap.chunk(L * L, world, rank)
    e0.record()
    for _ in range(3):
        ids = fn.map_ispace((L, L), lo, hi - lo, check=False)
    e1.record()
    torch.cuda.synchronize()
    k1_ms = e0.elapsed_time(e1) / 3
    e0.record()
    for _ in range(3):
        partition(ids, 8, check=False)
    e1.record()
    torch.cuda.synchronize()
    k2_ms = e0.elapsed_time(e1) / 3
    # errors: the lowest failing point (row 5: index out of range) wins on every rank,
    # although the other ranks' chunks only hit the division by zero at row 13
    fn = compile_mapper(prog, "bad", MachineShape("GPU", 1, 4))
    try:
        distmap.map_launch_sharded(fn, (16, 4), rank=rank, world=world)
        err = None
    except Exception as e:  # noqa: BLE001
        err = f"{type(e).__name__}: {e}"
    want = None
    try:
        O.map_launch(prog, "bad", ("GPU", 1, 4), (16, 4))
    except Exception as e:  # noqa: BLE001
        want = f"{type(e).__name__}: {e}"
    # messages of failure sites are point-independent ("index out of range"), the
    # reference's carry the offending value; classes and the failing site must agree
    ok = (err is not None and want is not None and err.split(":")[0] == want.split(":")[0]
          and ("out of range" in err) == ("out of range" in want))
    res.append({"case": "error", "ok": ok, "got": err, "want": want})
    allres = [res]
    if world > 1:
        allres = [None] * world
        dist.all_gather_object(allres, res)
        t = torch.tensor([ms, ms_local], device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms, ms_local = t.tolist()
    if rank == 0:
        flat = [r for rs in allres for r in rs]
        print(json.dumps({"ok": all(r["ok"] for r in flat), "world": world,
                          "ms_sharded_32768sq": ms, "points_per_s": L * L / (ms * 1e-3),
                          "ms_no_exchange": ms_local,
                          "rank0_k1_ms": k1_ms, "rank0_k2_ms": k2_ms,
                          "results": flat}))
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
