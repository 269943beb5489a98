"""Multi-GPU check of the mapped PENNANT-style hydro executor (torchrun, one
rank per GPU): point kinematics and zone energies vs the float64 oracle
(oracle/hydro.py), zone owners vs the oracle's evaluation of the same Mapple
mappers, and the cross-GPU corner count (the exchange model) vs a host count."""

import json
import os
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))

import numpy as np  # noqa: E402
import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402

from oracle import hydro as OH  # noqa: E402
from oracle import mapple_oracle as O  # noqa: E402
from paper_2507_17087_b200.dsl import parse  # noqa: E402
from paper_2507_17087_b200.executors.hydro import HydroSpec, MappedHydro  # noqa: E402
from paper_2507_17087_b200.executors.stencil import STENCIL_MAPPERS  # noqa: E402
from paper_2507_17087_b200.factorize import greedy_grid  # noqa: E402

TOL = 1e-3  # fp32 vs float64 after 20 steps, errors normalised by the field's max


def rel(a, b, full):
    """Max error normalised by the field's max over the WHOLE mesh (`full`), not over
    this rank's share: an 8-way split leaves ranks whose points barely move, and their
    own max made f32 rounding look like 1e-2 errors."""
    return float(np.abs(a - b).max() / max(np.abs(full).max(), 1e-30)) if a.size else 0.0


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
    steps = 20
    for Lx, Ly in ((48, 40), (37, 29)):
        ref = OH.simulate(Lx, Ly, steps)
        for mapping in ("decompose", "heuristic"):
            spec = HydroSpec(Lx, Ly)
            ex = MappedHydro(spec, mapping=mapping, rank=rank, world=world)
            for _ in range(steps):
                ex.step()
            torch.cuda.synchronize()
            if world > 1:
                dist.barrier()
            pid = ex.point_ids.cpu().numpy()
            zid = ex.zone_ids.cpu().numpy()
            n = pid.size
            errs = {k: rel(getattr(ex, a)[:n].double().cpu().numpy(), ref[k][pid], ref[k])
                    for k, a in (("x", "px"), ("y", "py"), ("u", "ux"), ("v", "uy"))}
            errs["e"] = rel(ex.ze.double().cpu().numpy(), ref["e"][zid], ref["e"])
            # owners and the exchange model from the oracle's mapping
            g0 = greedy_grid(world, 2)[0]
            zo = np.asarray(O.map_launch(parse(STENCIL_MAPPERS.format(g0=g0)),
                                         f"stencil_{mapping}", ("GPU", 1, world), (Ly, Lx)))
            zo2 = zo.reshape(Ly, Lx)
            po = zo2[np.minimum(np.arange(Ly + 1), Ly - 1)[:, None],
                     np.minimum(np.arange(Lx + 1), Lx - 1)[None, :]].ravel()
            mine = np.nonzero(zo == rank)[0]
            zj, zi = mine // Lx, mine % Lx
            W = Lx + 1
            corners = np.stack([zj * W + zi, zj * W + zi + 1, (zj + 1) * W + zi + 1,
                                (zj + 1) * W + zi])
            want_cross = int((po[corners] != rank).sum())
            res.append({"mesh": [Lx, Ly], "mapping": mapping, "rank": rank, "errs": errs,
                        "zones_ok": bool(np.array_equal(np.sort(zid), mine)),
                        "cross": ex.cross_corners, "want_cross": want_cross})
            ex.close()
            if world > 1:
                dist.barrier()
    allr = [res]
    if world > 1:
        allr = [None] * world
        dist.all_gather_object(allr, res)
    if rank == 0:
        flat = [r for rs in allr for r in rs]
        ok = all(max(r["errs"].values()) < TOL and r["zones_ok"] and r["cross"] == r["want_cross"]
                 for r in flat)
        print(json.dumps({"ok": ok, "world": world, "results": flat}))
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
