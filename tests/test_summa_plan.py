"""SUMMA / PUMMA per-GPU schedules (executors/summa.py: plan_panels), pure CPU: every
element of this GPU's C block receives every K exactly once, the first product touching an
element (row band x column band) writes it and later ones accumulate, and every product
waits for the pulls of the operand slices it reads -- on the BASELINE shapes at 2 / 4 / 8 GPUs, both mappings."""

import pytest

a_chunks_max = 4  # plan_panels' default chunk count (rows or columns)

from test_plans_gloo import _summa_plan


@pytest.mark.parametrize("world", [2, 4, 8])
@pytest.mark.parametrize("mnk", [(32768, 32768, 32768), (65536, 16384, 16384), (4096, 2048, 1024)])
@pytest.mark.parametrize("mapping", ["decompose", "heuristic"])
def test_plan_covers_k_once_per_row(world, mnk, mapping):
    M, N, K = mnk
    for rank in range(world):
        p = _summa_plan(rank, world, M, N, K, mapping)
        plan, lay = p["plan"], p["layout"]
        rc = lay.rects[rank]
        mr, nc = rc.r1 - rc.r0, rc.c1 - rc.c0
        # row / column boundaries of all GEMMs -> check each elementary C rectangle
        rows = sorted({0, mr} | {g[0] for g in plan.gemms} | {g[1] for g in plan.gemms})
        cols = sorted({0, nc} | {g[6] for g in plan.gemms} | {g[7] for g in plan.gemms})
        for lo, hi in zip(rows, rows[1:]):
            for clo, chi in zip(cols, cols[1:]):
                covering = [g for g in plan.gemms
                            if g[0] <= lo and hi <= g[1] and g[6] <= clo and chi <= g[7]]
                ks = sorted((g[2], g[3]) for g in covering)
                assert ks[0][0] == 0 and ks[-1][1] == K
                assert all(a[1] == b[0] for a, b in zip(ks, ks[1:])), (rank, ks)
                first = covering[0]
                assert not first[4]  # the first product writes C
                assert all(g[4] for g in covering if g is not first)
        # every GEMM waits for the pulls of the remote slices it reads
        pulled = set()
        for g in plan.gemms:
            r0, r1, k0, k1, _, evs, c0, c1 = g
            pulled |= set(evs)
            for i, (name, src, row0, nrows, p0, p1, _) in enumerate(plan.pulls):
                overlaps_k = p0 < k1 and k0 < p1
                span = (r0, r1) if name == "A" else (c0, c1)
                overlaps_rows = row0 < span[1] and span[0] < row0 + nrows
                if overlaps_k and overlaps_rows:
                    assert i in pulled, (rank, g, plan.pulls[i])
        # fewer launches than panels x chunks whenever runs merged
        assert len(plan.gemms) <= len(plan.panels) * max(1, len(plan.chunks), a_chunks_max)
