"""Multi-GPU check of the mapped Cannon / 2.5D executor (torchrun, one rank per GPU):
C vs float64, block moves vs the schedule's count, the tile owners vs the oracle's
evaluation of the same Mapple mapper."""

import json
import os
import sys
from math import isqrt
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))

import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402

from oracle import mapple_oracle as O  # noqa: E402
from paper_2507_17087_b200.dsl import parse  # noqa: E402
from paper_2507_17087_b200.executors.cannon import HIER_MAPPERS, MappedCannon, cannon_moves  # noqa: E402
from paper_2507_17087_b200.executors.summa import synth  # noqa: E402


def main():
    import faulthandler

    faulthandler.dump_traceback_later(int(os.environ.get("PM_HANG_DUMP_S", "240")), exit=False)
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
    configs = []
    for c in (1, 2, 4, 8):
        if world % c == 0 and isqrt(world // c) ** 2 * c == world and isqrt(world // c) % c == 0:
            configs.append(c)
    for c in configs:
        for dtype, N, graph in (("fp32", 1024, False), ("fp32", 1024, True), ("bf16", 2048, False),
                                ("bf16", 2048, True)):
            if dtype == "fp32" and c > 1:
                continue
            print(f"[rank {rank}] c={c} {dtype} N={N} graph={graph}", file=sys.stderr, flush=True)
            ex = MappedCannon(N, layers=c, rank=rank, world=world, dtype=dtype, seed=21,
                              graph=graph)
            for _ in range(5):  # eager warm-up per buffer, then graph capture + replays
                ex.step()
            C = ex.result()
            torch.cuda.synchronize()
            i, j, l = ex.coord
            nb = ex.nb
            r0, r1 = ex.my_rows
            tdt = torch.float32 if dtype == "fp32" else torch.bfloat16
            A = synth((i * nb + r0, i * nb + r1), (0, N), N, 21, "cuda", dtype=tdt).double()
            Bt = synth((j * nb, (j + 1) * nb), (0, N), N, 22, "cuda", dtype=tdt).double()
            R = A @ Bt.T
            err = float((C.double() - R).abs().max() / R.abs().max())
            moves = [None] * world
            if world > 1:
                dist.all_gather_object(moves, ex.moved_blocks)
            else:
                moves = [ex.moved_blocks]
            q = ex.q
            task = "cannon" if c == 1 else "solomonik"
            ispace = (q, q) if c == 1 else (q, q, c)
            want = O.map_launch(parse(HIER_MAPPERS), task, ("GPU", *ex.machine), ispace)
            got = [ex.owner[(a, b, 0)] for a in range(q) for b in range(q)] if c == 1 else \
                [ex.owner[(a, b, d)] for a in range(q) for b in range(q) for d in range(c)]
            out.append({"c": c, "dtype": dtype, "N": N, "graph": graph, "rank": rank, "err": err,
                        "moves": sum(moves), "want_moves": cannon_moves(q, c),
                        "owners_ok": got == want})
            if world > 1:
                dist.barrier()
            ex.close()
    if world == 4:
        # BASELINE configs[0] exactly as the reference states it: the corpus' own
        # `cannon_mm` (matmul_mappers.mapper, hierarchical_block2D) on
        # MachineShape(GPU, 2, 2), fp32 N=1024; owners == the reference's
        # assignment table (tests/golden/mappings.json, produced by running the
        # reference), 12 block moves, full C vs float64
        gold = json.loads((ROOT / "tests" / "golden" / "mappings.json").read_text())
        case = next(c for c in gold["cases"] if c["name"] == "matmul_mappers:cannon_mm"
                    and c["machine"] == [2, 2] and c["ispace"] == [2, 2])
        ref_ids = [n * 2 + p for n, p in case["table"]]
        for graph in (False, True):
            ex = MappedCannon(1024, layers=1, rank=rank, world=world, dtype="fp32", seed=21,
                              graph=graph, machine=(2, 2), program=gold["sources"][case["src"]],
                              task="cannon_mm")
            for _ in range(5):
                ex.step()
            C = ex.result()
            torch.cuda.synchronize()
            i, j, _ = ex.coord
            nb = ex.nb
            A = synth((i * nb, (i + 1) * nb), (0, 1024), 1024, 21, "cuda").double()
            Bt = synth((j * nb, (j + 1) * nb), (0, 1024), 1024, 22, "cuda").double()
            R = A @ Bt.T
            err = float((C.double() - R).abs().max() / R.abs().max())
            moves = [None] * world
            dist.all_gather_object(moves, ex.moved_blocks)
            got = [ex.owner[(a, b, 0)] for a in range(2) for b in range(2)]
            out.append({"c": 1, "dtype": "fp32", "N": 1024, "graph": graph, "rank": rank,
                        "err": err, "moves": sum(moves), "want_moves": 12,
                        "owners_ok": got == ref_ids, "configs0_reference_owners": ref_ids,
                        "owners": got})
            dist.barrier()
            ex.close()
    allr = [out]
    if world > 1:
        allr = [None] * world
        dist.all_gather_object(allr, out)
    if rank == 0:
        flat = [r for rs in allr for r in rs]
        ok = all(r["err"] < 1e-2 and r["moves"] == r["want_moves"] and r["owners_ok"]
                 for r in flat)
        print(json.dumps({"ok": ok, "world": world, "results": flat}))
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
