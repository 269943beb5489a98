"""Multi-GPU check of the mapped circuit executor (torchrun, one rank per GPU):
node voltages and wire currents vs the float64 oracle (oracle/circuit.py),
the piece owners vs the oracle's evaluation of the same Mapple mappers, and
the cross-GPU wire count (the communication model) vs a host count."""

import json
import os
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))

import numpy as np  # noqa: E402
import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402

from oracle import circuit as OC  # noqa: E402
from oracle import mapple_oracle as O  # noqa: E402
from paper_2507_17087_b200.dsl import parse  # noqa: E402
from paper_2507_17087_b200.executors.circuit import (CIRCUIT_MAPPERS, CircuitSpec,  # noqa: E402
                                                     MappedCircuit)

TOL = 1e-4  # fp32 arithmetic vs float64, a few iterations


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
    res = []
    for spec, iters in ((CircuitSpec(12, 64, 256, pct_in=80, steps=20, seed=3), 4),
                        (CircuitSpec(5, 33, 100, pct_in=50, steps=7, seed=1), 3)):
        ref_v, ref_i = OC.simulate(spec.pieces, spec.nodes_per_piece, spec.wires_per_piece,
                                   spec.pct_in, spec.steps, spec.dt, spec.seed, iters)
        gen = OC.generate(spec.pieces, spec.nodes_per_piece, spec.wires_per_piece, spec.pct_in,
                          spec.seed)
        for mapping in ("block", "cyclic"):
            ex = MappedCircuit(spec, mapping=mapping, rank=rank, world=world)
            for _ in range(iters):
                ex.step()
            torch.cuda.synchronize()
            if world > 1:
                dist.barrier()
            ids = ex.node_ids.cpu().numpy()
            v = ex.volt[:ids.size].double().cpu().numpy()
            wids = ex.wire_ids.cpu().numpy()
            cur = ex.current[:, :wids.size].double().cpu().numpy().T
            ev = float(np.abs(v - ref_v[ids]).max() / np.abs(ref_v).max()) if ids.size else 0.0
            ei = float(np.abs(cur - ref_i[wids]).max() / max(np.abs(ref_i).max(), 1e-30)) \
                if wids.size else 0.0
            owners = O.map_launch(parse(CIRCUIT_MAPPERS), f"circuit_{mapping}", ("GPU", world, 1),
                                  (spec.pieces,))
            piece_in = gen["in_node"] // spec.nodes_per_piece
            piece_out = gen["out_node"] // spec.nodes_per_piece
            own_in = np.asarray(owners)[piece_in]
            own_out = np.asarray(owners)[piece_out]
            want_cross = int(((own_in == rank) & (own_out != rank)).sum())
            res.append({"spec": str(spec), "mapping": mapping, "rank": rank, "err_v": ev,
                        "err_i": ei, "owners_ok": ex.owner == owners,
                        "cross": ex.cross_gpu_wires, "want_cross": want_cross})
            ex.close()
            if world > 1:
                dist.barrier()
    allr = [res]
    if world > 1:
        allr = [None] * world
        dist.all_gather_object(allr, res)
    if rank == 0:
        flat = [r for rs in allr for r in rs]
        ok = all(r["err_v"] < TOL and r["err_i"] < TOL and r["owners_ok"]
                 and r["cross"] == r["want_cross"] for r in flat)
        print(json.dumps({"ok": ok, "world": world, "results": flat}))
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
