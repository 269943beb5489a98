"""Johnson / COSMA per-GPU schedules (executors/grid3d.py: plan_3d), pure CPU: every
element of every destination's C rows is produced exactly once per GPU, own rows first
(before the barrier) and the peers' after it, and every product waits for the pulls
of the A rows / Bt rows it reads -- on the BASELINE shapes at 2 / 4 / 8 GPUs."""

import pytest

from paper_2507_17087_b200.executors.grid3d import grid_for, plan_3d, split


@pytest.mark.parametrize("world", [2, 4, 8])
@pytest.mark.parametrize("mnk", [(32768, 32768, 32768), (65536, 16384, 16384), (4096, 2048, 1024)])
@pytest.mark.parametrize("mapping", ["decompose", "heuristic"])
def test_plan_3d_covers_and_waits(world, mnk, mapping):
    M, N, K = mnk
    grid = grid_for(world, M, N, K, mapping)
    pm, pn, pk = grid
    owner, lin = {}, 0
    for a in range(pm):
        for b in range(pn):
            for c in range(pk):
                owner[(a, b, c)] = lin
                lin += 1
    for (a, b, c), me in owner.items():
        mb = split(M, pm, a)[1] - split(M, pm, a)[0]
        nb = split(N, pn, b)[1] - split(N, pn, b)[0]
        plan = plan_3d(grid, (a, b, c), owner, mb, nb)
        gemms, pulls, bb = plan["gemms"], plan["pulls"], plan["barrier_before"]
        # own rows strictly first, then the barrier, then the peers'
        dsts = [g[2] for g in gemms]
        n_own = dsts.count(me)
        assert dsts[:n_own] == [me] * n_own
        assert bb == (n_own if pk > 1 else None)
        # each destination's rows x all columns covered exactly once
        for d in range(pk):
            R = split(mb, pk, d)
            dst = owner[(a, b, d)]
            cells = 0
            for (r0, r1), (c0, c1), g_dst, d0, _ in gemms:
                if g_dst == dst:
                    assert R[0] <= r0 < r1 <= R[1] and 0 <= c0 < c1 <= nb and d0 == R[0]
                    cells += (r1 - r0) * (c1 - c0)
            assert cells == (R[1] - R[0]) * nb, (grid, (a, b, c), d)
        # pairwise disjoint products per destination
        for i, g in enumerate(gemms):
            for h in gemms[i + 1:]:
                if g[2] == h[2]:
                    assert (g[0][1] <= h[0][0] or h[0][1] <= g[0][0] or
                            g[1][1] <= h[1][0] or h[1][1] <= g[1][0])
        # every product waits for the pulls of the remote rows it reads
        own_a = split(mb, pn, b)
        own_b = split(nb, pm, a)
        waited = set()
        for (r0, r1), (c0, c1), _, _, evs in gemms:
            waited |= set(evs)
            for i, (name, src, (p0, p1)) in enumerate(pulls):
                lo, hi = (r0, r1) if name == "A" else (c0, c1)
                if p0 < hi and lo < p1:
                    assert i in waited
            assert not (r0 < own_a[0] or r1 > own_a[1]) or any(
                pulls[e][0] == "A" for e in evs) or pn == 1
        # the pulls are exactly the remote parts
        a_bytes = sum(p1 - p0 for name, _, (p0, p1) in pulls if name == "A")
        b_bytes = sum(p1 - p0 for name, _, (p0, p1) in pulls if name == "Bt")
        assert a_bytes == mb - (own_a[1] - own_a[0])
        assert b_bytes == nb - (own_b[1] - own_b[0])
