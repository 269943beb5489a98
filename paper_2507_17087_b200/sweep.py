"""Decompose-vs-heuristic sweep over the paper's Table-3 grid (host side).

Same records and grouping as the reference's `sweep_configs` / `sweep_groups`
(reference: cli.py:264-324): for every aspect ratio 1:r, per-node area A and GPU
count, the iteration space x = round(sqrt(A * nodes / r)), y = r * x is cut by
the `decompose` optimum and by the Algorithm-1 grid, and the model-predicted
boundary volumes (surface_volume, commvol.py:94-96) are compared.
"""

from __future__ import annotations

import math

from .commvol import BlockGrid, surface_volume
from .factorize import greedy_grid, search_optimal

TABLE3_RATIOS = (1, 2, 4, 8, 16, 32)
TABLE3_AREAS = (10**6, 10**7, 10**8, 2 * 10**8, 4 * 10**8)
TABLE3_GPUS = (4, 8, 16, 32, 64, 128)


def _join(values) -> str:
    return ";".join(str(v) for v in values)


def sweep_configs(ratios, areas, gpus_list, gpus_per_node):
    out = []
    for r in ratios:
        for area in areas:
            for g in gpus_list:
                nodes = max(1, g // gpus_per_node)
                x = max(1, round(math.sqrt(area * nodes / r)))
                ext = (x, x * r)
                opt = search_optimal(g, ext)[0]
                heur = greedy_grid(g, 2)
                v_opt = surface_volume(BlockGrid(ext, opt))
                v_heur = surface_volume(BlockGrid(ext, heur))
                ratio = float(v_heur / v_opt) if v_opt else 1.0
                pct = 100.0 * float((v_heur - v_opt) / v_heur) if v_heur else 0.0
                out.append({
                    "aspect_ratio": f"1:{r}", "area_per_node": area, "gpus": g, "nodes": nodes,
                    "extents": _join(ext), "optimal": _join(opt), "greedy": _join(heur),
                    "optimal_volume": str(v_opt), "greedy_volume": str(v_heur),
                    "volume_ratio": ratio, "improvement_pct": pct,
                })
    return out


def sweep_groups(records):
    """Geometric-mean volume ratio per value of each swept parameter."""
    groups = []
    for param in ("aspect_ratio", "area_per_node", "gpus"):
        seen = []
        for rec in records:
            if rec[param] not in seen:
                seen.append(rec[param])
        for value in seen:
            rs = [rec["volume_ratio"] for rec in records if rec[param] == value]
            gm = math.exp(sum(math.log(x) for x in rs) / len(rs))
            groups.append({"parameter": param, "value": value, "configs": len(rs),
                           "geomean_volume_ratio": gm,
                           "geomean_improvement_pct": 100.0 * (1.0 - 1.0 / gm)})
    return groups
