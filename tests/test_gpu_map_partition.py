"""K1+K2 fused (map_partition.cu) on the B200: the two-pass map + partition
must equal K1 followed by K2 -- which the golden tests pin to the reference's
assignments and shard trees -- on every golden mapping, in implicit and
explicit mode, on sub-ranges, with failing points, and on the full 32768^2
stencil launch."""

import pytest

from conftest import golden, mapping_cases
from paper_2507_17087_b200.dsl import compile_mapper, parse
from paper_2507_17087_b200.ownership import partition, shard_leaves
from paper_2507_17087_b200.spaces import MachineShape

pytestmark = pytest.mark.gpu

CASES = [c for c in mapping_cases() if isinstance(c["table"], list)]


def _same(own, ref):
    import torch

    return (torch.equal(own.counts, ref.counts) and torch.equal(own.offsets, ref.offsets)
            and torch.equal(own.perm, ref.perm))


def test_fused_equals_k1_k2_on_golden_cases(cuda):
    torch = cuda
    done = 0
    for c in CASES[::3]:
        machine = MachineShape("GPU", *c["machine"])
        fn = compile_mapper(parse(c["source"]), c["task"], machine)
        ispace = tuple(c["ispace"])
        P = machine.nodes * machine.procs_per_node
        fails = any(isinstance(r, dict) for r in c["table"])
        if fails:
            with pytest.raises(Exception) as e1:
                fn.map_ispace(ispace)
            with pytest.raises(Exception) as e2:
                fn.map_partition(ispace)
            assert type(e1.value) is type(e2.value) and str(e1.value) == str(e2.value)
            continue
        ids = fn.map_ispace(ispace)
        ref = partition(ids, P)
        own, ids2 = fn.map_partition(ispace, with_ids=True)
        assert _same(own, ref), c["name"]
        assert torch.equal(ids, ids2)
        # explicit points
        pts = torch.cartesian_prod(*[torch.arange(e, dtype=torch.int32) for e in ispace])
        pts = pts.view(-1, len(ispace)).to("cuda", torch.int32)
        assert _same(fn.map_partition(ispace, points=pts), ref), c["name"]
        done += 1
    assert done > 50


def test_fused_shard_trees_match_reference(cuda):
    torch = cuda
    for case in golden("shards"):
        machine = MachineShape("GPU", *case["machine"])
        fn = compile_mapper(parse(case["source"]), case["task"], machine)
        ispace = tuple(case["ispace"])
        own = fn.map_partition(ispace)
        leaves = shard_leaves(case["task"], own, machine.procs_per_node)
        pts = torch.cartesian_prod(*[torch.arange(e) for e in ispace]).view(-1, len(ispace))
        got = [{"id": lid, "target": list(tgt), "points": pts[idx.cpu().long()].tolist()}
               for lid, tgt, idx in leaves]
        assert got == case["leaves"], case["task"]


CYCLIC = """
m = Machine(GPU)
def cyc(Tuple p, Tuple s):
    q = m.merge(0, 1)
    return q[(p[0] * 7 + p[1] * 13 + p[0] * p[1]) % q.size[0]]
def blk(Tuple p, Tuple s):
    q = m.merge(0, 1).decompose(0, s)
    return q[*(p * q.size / s)]
IndexTaskMap cyc cyc
IndexTaskMap blk blk
"""


@pytest.mark.parametrize("task,machine,ispace,first,count", [
    ("cyc", (1, 8), (1000, 999), 0, None), ("cyc", (4, 16), (3001, 777), 12345, 1_000_000),
    ("blk", (2, 4), (4097, 4099), 4095, 5_000_000), ("blk", (1, 64), (8192, 8192), 0, None),
    ("cyc", (3, 5), (7, 5), 3, 20), ("blk", (1, 1), (10, 10), 0, None)])
def test_fused_ranges(cuda, task, machine, ispace, first, count):
    torch = cuda
    fn = compile_mapper(parse(CYCLIC), task, MachineShape("GPU", *machine))
    P = machine[0] * machine[1]
    ids = fn.map_ispace(ispace, first, count)
    ref = partition(ids, P)
    own, ids2 = fn.map_partition(ispace, first, count, with_ids=True)
    assert torch.equal(ids, ids2)
    assert _same(own, ref)


def test_fused_full_stencil_launch(cuda):
    """configs[4]: the 1.07e9-point launch, 8 processors."""
    torch = cuda
    L = 32768
    fn = compile_mapper(parse(CYCLIC), "blk", MachineShape("GPU", 1, 8))
    ref = partition(fn.map_ispace((L, L)), 8)
    own = fn.map_partition((L, L))
    assert torch.equal(own.counts, ref.counts)
    assert torch.equal(own.perm, ref.perm)


def _scaled(ispace, min_points=3 * 4096 + 123):
    """The golden launch shape stretched to several 4096-point tiles."""
    n = 1
    for e in ispace:
        n *= e
    f = 1
    while n * f ** len(ispace) < min_points:
        f += 1
    return tuple(e * f + (i % 2) for i, e in enumerate(ispace))


def test_tile_proofs_on_multi_tile_launches(cuda):
    """Pass 1 proves whole tiles uniform by interval arithmetic over each tile's
    coordinate box (mapping.cpp pm_tile_bin); only tiles before the last are
    eligible, so the golden launches (one tile) never exercise it.  Stretch the
    golden programs -- corpus mappers and the seeded random programs with
    ternaries, negative operands, division / modulo by zero, helper calls -- to
    multi-tile launches and hold the fused partition to K1 then K2, errors
    included."""
    torch = cuda
    done = 0
    for c in CASES[1::13]:
        machine = MachineShape("GPU", *c["machine"])
        fn = compile_mapper(parse(c["source"]), c["task"], machine)
        ispace = _scaled(tuple(c["ispace"]))
        P = machine.nodes * machine.procs_per_node
        try:
            ids = fn.map_ispace(ispace)
        except Exception as e1:  # noqa: BLE001
            with pytest.raises(Exception) as e2:
                fn.map_partition(ispace)
            assert type(e1) is type(e2.value) and str(e1) == str(e2.value), c["name"]
            continue
        own = fn.map_partition(ispace)
        assert _same(own, partition(ids, P)), (c["name"], ispace)
        done += 1
    assert done > 20


PROOF_EDGES = """
m = Machine(GPU)
def blk(Tuple p, Tuple s):
    q = m.merge(0, 1).decompose(0, s)
    return q[*(p * q.size / s)]
def tern(Tuple p, Tuple s):
    q = m.merge(0, 1)
    return q[(p[0] > 50 ? 1 : (p[1] < 4000 ? 0 : 2))]
def divp(Tuple p, Tuple s):
    q = m.merge(0, 1)
    return q[(1000 / (p[0] - 97)) % q.size[0]]
def neg(Tuple p, Tuple s):
    q = m.merge(0, 1)
    return q[((p[1] - 5000) / 777) % q.size[0]]
def rowmod(Tuple p, Tuple s):
    q = m.merge(0, 1)
    return q[(p[0] / 3 + p[1] / 4096) % q.size[0]]
IndexTaskMap blk blk
IndexTaskMap tern tern
IndexTaskMap divp divp
IndexTaskMap neg neg
IndexTaskMap rowmod rowmod
"""


@pytest.mark.parametrize("task", ["blk", "tern", "divp", "neg", "rowmod"])
@pytest.mark.parametrize("ispace", [(200, 8192), (150, 10007), (3, 4096 * 5 + 1)])
def test_tile_proof_edges(cuda, task, ispace):
    """Tiles straddling block edges, decided / undecided ternaries, a divisor
    that is zero on one row (an error at the lowest failing point, as K1),
    floor division of negative values, and row-periodic modulo."""
    machine = MachineShape("GPU", 2, 3)
    fn = compile_mapper(parse(PROOF_EDGES), task, machine)
    try:
        ids = fn.map_ispace(ispace)
    except Exception as e1:  # noqa: BLE001
        with pytest.raises(Exception) as e2:
            fn.map_partition(ispace)
        assert type(e1) is type(e2.value) and str(e1) == str(e2.value)
        return
    assert _same(fn.map_partition(ispace), partition(ids, 6))
    f0, cnt = 4096 * 3 + 5, 4096 * 7 + 9  # a sub-range: tiles start off the launch's grid
    assert _same(fn.map_partition(ispace, first=f0, count=cnt),
                 partition(ids[f0:f0 + cnt].contiguous(), 6))
