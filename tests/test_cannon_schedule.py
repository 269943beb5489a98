"""CPU check of the Cannon / 2.5D schedule the executor runs (executors/cannon.py):
a lock-step symbolic simulation of every GPU's op list, with the tile owners
taken from the oracle's evaluation of the same Mapple mappers.  Checks that
every C block receives each A(i,k) B(k,j) product exactly once, that no pull
reads a buffer another GPU writes in the same barrier phase, and that the
block-move count equals cannon_moves()."""

import pytest

from oracle import mapple_oracle as O
from paper_2507_17087_b200.dsl import parse
from paper_2507_17087_b200.executors.cannon import HIER_MAPPERS, cannon_moves, cannon_schedule


def _owners(q, c, machine):
    prog = parse(HIER_MAPPERS)
    if c == 1:
        ranks = O.map_launch(prog, "cannon", ("GPU", *machine), (q, q))
        coords = [(i, j, 0) for i in range(q) for j in range(q)]
    else:
        ranks = O.map_launch(prog, "solomonik", ("GPU", *machine), (q, q, c))
        coords = [(i, j, l) for i in range(q) for j in range(q) for l in range(c)]
    return dict(zip(coords, ranks))


def _simulate(q, c, owner):
    world = q * q * c
    assert sorted(owner.values()) == list(range(world))
    coord_of = {r: xyz for xyz, r in owner.items()}
    # buffer state: rank -> name -> block label
    state = {}
    for r, (i, j, l) in coord_of.items():
        state[r] = {"A0": ("A", i, j), "B0": ("B", i, j)}
    ops = {r: cannon_schedule(q, c, coord_of[r]) for r in range(world)}
    # split every op list into barrier-separated phases
    phases = {}
    for r, lst in ops.items():
        ph, cur = [], []
        for op in lst:
            if op[0] == "barrier":
                ph.append(cur)
                cur = []
            else:
                cur.append(op)
        ph.append(cur)
        phases[r] = ph
    nph = {len(p) for p in phases.values()}
    assert len(nph) == 1, "every GPU joins the same number of barriers"
    products = {}
    moves = 0
    for p in range(nph.pop()):
        snap = {r: dict(s) for r, s in state.items()}
        reads, writes = set(), set()
        for r in range(world):
            for op in phases[r][p]:
                if op[0] == "pull":
                    _, name, src, (kind, slot) = op
                    s = owner[src]
                    bname = ("Acur" if kind == "A" else "Bcur") + str(slot)
                    reads.add((s, name))
                    writes.add((r, bname))
                    state[r][bname] = snap[s][name]
                    moves += s != r
                else:
                    _, slot, d = op
                    a, b = state[r][f"Acur{slot}"], state[r][f"Bcur{slot}"]
                    reads.update({(r, f"Acur{slot}"), (r, f"Bcur{slot}")})
                    assert a[0] == "A" and b[0] == "B" and a[2] == b[1], (a, b)
                    i, j, _ = coord_of[r]
                    assert (a[1], b[2]) == (i, j)
                    key = (i, j, d)
                    products.setdefault(key, []).append(a[2])
        assert not (reads & writes), f"read/write race in phase {p}: {reads & writes}"
    for i in range(q):
        for j in range(q):
            for d in range(c):
                assert sorted(products[(i, j, d)]) == list(range(q)), (i, j, d)
    return moves


@pytest.mark.parametrize("q,c,machine", [(1, 1, (1, 1)), (2, 1, (2, 2)), (2, 1, (4, 1)),
                                         (3, 1, (9, 1)), (4, 1, (2, 8)), (2, 2, (8, 1)),
                                         (4, 2, (4, 8)), (4, 4, (8, 8))])
def test_cannon_schedule(q, c, machine):
    owner = _owners(q, c, machine)
    assert _simulate(q, c, owner) == cannon_moves(q, c)
