"""K3 on the B200: halo transfer lists vs the oracle's per-cell enumeration,
and totals vs the reference's oracle_boundary_count / surface_volume."""

import itertools
import random

import pytest

from oracle import mapple_oracle as O
from paper_2507_17087_b200 import commvol as cv
from paper_2507_17087_b200.dsl import compile_mapper, parse
from paper_2507_17087_b200.spaces import MachineShape
from paper_2507_17087_b200.transfer import halo_lists

pytestmark = pytest.mark.gpu

BLOCK = """
m = Machine(GPU)
def block(Tuple p, Tuple s):
    q = m.merge(0, 1).decompose(0, s)
    idx = p * q.size / s
    return q[*idx]
IndexTaskMap t block
"""


def _entries(tl):
    out = {}
    counts = tl.pair_counts.tolist()
    offs = tl.pair_offsets.tolist()
    cells = tl.cells.tolist()
    dims = tl.dims.tolist()
    for key, c in enumerate(counts):
        if c:
            src, dst = divmod(key, tl.nprocs)
            out[(src, dst)] = list(zip(cells[offs[key]:offs[key] + c], dims[offs[key]:offs[key] + c]))
    return out


def test_random_owners_match_oracle(cuda):
    torch = cuda
    rng = random.Random(3)
    for _ in range(30):
        rank = rng.choice([1, 2, 3])
        ext = tuple(rng.randint(1, 9) for _ in range(rank))
        halo = tuple(rng.randint(0, 3) for _ in range(rank))
        P = rng.randint(1, 6)
        cells = list(itertools.product(*map(range, ext)))
        owner = {c: rng.randrange(P) for c in cells}
        t = torch.tensor([owner[c] for c in cells], dtype=torch.int32, device="cuda")
        tl = halo_lists(t, ext, halo, P)
        assert _entries(tl) == O.halo_entries(owner.__getitem__, ext, halo)


@pytest.mark.parametrize("ext,machine,halo", [((12, 18), (1, 6), (1, 1)), ((18, 12), (1, 6), (1, 1)),
                                              ((37, 23), (2, 3), (2, 1)), ((16, 64), (1, 8), (1, 1)),
                                              ((9, 10, 11), (2, 4), (1, 2, 1))])
def test_block_partition_totals_match_reference_models(cuda, ext, machine, halo):
    fn = compile_mapper(parse(BLOCK), "t", MachineShape("GPU", *machine))
    ids = fn.map_ispace(ext)
    tl = halo_lists(ids, ext, halo, machine[0] * machine[1])
    from paper_2507_17087_b200.factorize import search_optimal

    grid, _ = search_optimal(machine[0] * machine[1], ext)
    g = cv.BlockGrid(ext, grid)
    assert tl.total == cv.oracle_boundary_count(g, halo, cap=1 << 40)
    if all(h == 1 for h in halo):
        assert tl.total == cv.surface_volume(g)
    # per pair: every send list has a mirror receive of the same size (block grids)
    counts = tl.pair_counts.view(tl.nprocs, tl.nprocs)
    assert (counts == counts.T).all()


def test_stencil_32768_counts(cuda):
    """Config 5: 32768^2 on 8 GPUs, decompose grid (2,4): 262,144 halo cells (h=1)."""
    fn = compile_mapper(parse(BLOCK), "t", MachineShape("GPU", 1, 8))
    ext = (32768, 32768)
    ids = fn.map_ispace(ext)
    tl = halo_lists(ids, ext, (1, 1), 8, counts_only=True)
    g = cv.BlockGrid(ext, (2, 4))
    assert tl.total == cv.oracle_boundary_count(g, (1, 1), cap=1 << 40) == 262144


@pytest.mark.parametrize("ext,halo,P", [((37, 53), (1, 1), 4), ((64, 48), (2, 1), 3),
                                        ((9, 10, 11), (1, 2, 1), 5), ((200,), (3,), 8),
                                        ((33, 40), (1, 1), 12)])
def test_single_call_abi_matches_compaction(cuda, ext, halo, P):
    """pm_halo_lists (one call, partition of all slots) == the compaction path."""
    import ctypes

    from paper_2507_17087_b200 import native

    torch = cuda
    g = torch.Generator(device="cuda").manual_seed(sum(ext) + P)
    n = 1
    for e in ext:
        n *= e
    owner = torch.randint(0, P, (n,), device="cuda", dtype=torch.int32, generator=g)
    want = halo_lists(owner, ext, halo, P)
    lib = native.lib()
    r = len(ext)
    ext_c = (ctypes.c_int64 * r)(*ext)
    halo_c = (ctypes.c_int32 * r)(*halo)
    counts = torch.empty(P * P, dtype=torch.int64, device="cuda")
    offsets = torch.empty(P * P, dtype=torch.int64, device="cuda")
    nb = lib.pm_halo_scratch_bytes(ext_c, r, P)
    scratch = torch.empty(nb, dtype=torch.uint8, device="cuda")
    total = want.total
    cells = torch.empty(max(total, 1), dtype=torch.int64, device="cuda")
    dims = torch.empty(max(total, 1), dtype=torch.int8, device="cuda")
    native.check(lib.pm_halo_lists(owner.data_ptr(), ext_c, r, halo_c, P, counts.data_ptr(),
                                   offsets.data_ptr(), cells.data_ptr(), dims.data_ptr(),
                                   scratch.data_ptr(), nb, None), "pm_halo_lists")
    assert torch.equal(counts, want.pair_counts)
    assert torch.equal(offsets, want.pair_offsets)
    assert torch.equal(cells[:total], want.cells) and torch.equal(dims[:total], want.dims)


def _block_owner(rng, rows, cols, P):
    """Random rectangular ownership: random row / column cuts, random owner per block."""
    rc = sorted(rng.sample(range(1, rows), min(rows - 1, rng.randint(0, 3)))) if rows > 1 else []
    cc = sorted(rng.sample(range(1, cols), min(cols - 1, rng.randint(0, 4)))) if cols > 1 else []
    rb = [0] + rc + [rows]
    cb = [0] + cc + [cols]
    ids = {(a, b): rng.randrange(P) for a in range(len(rb) - 1) for b in range(len(cb) - 1)}
    import bisect

    return [[ids[(bisect.bisect_right(rb, r) - 1, bisect.bisect_right(cb, c) - 1)]
             for c in range(cols)] for r in range(rows)]


@pytest.mark.parametrize("rows,cols", [(37, 1028), (65, 2048), (3, 4), (1, 8), (40, 1036),
                                       (33, 3072), (70, 516)])
def test_strip_2d_unit_halo_matches_oracle(cuda, rows, cols):
    """The 2-D h=(1,1) strip kernels (cols % 4 == 0): partial strips, partial row
    blocks, single rows / columns, block and cell-level noise ownership."""
    torch = cuda
    rng = random.Random(rows * 7919 + cols)
    for trial in range(2):
        P = rng.randint(2, 8)
        grid = _block_owner(rng, rows, cols, P)
        if trial:  # sprinkle cell-level noise
            for _ in range(rows * cols // 50 + 1):
                grid[rng.randrange(rows)][rng.randrange(cols)] = rng.randrange(P)
        flat = [v for row in grid for v in row]
        t = torch.tensor(flat, dtype=torch.int32, device="cuda")
        tl = halo_lists(t, (rows, cols), (1, 1), P)
        assert _entries(tl) == O.halo_entries(lambda c: grid[c[0]][c[1]], (rows, cols), (1, 1))


@pytest.mark.parametrize("ext,P", [((300, 4100), 7), ((129, 1024), 64), ((64, 2052), 3)])
def test_strip_2d_out_of_range_owners_match_single_call(cuda, ext, P):
    """Cells owned by no processor (ids < 0 or >= P) emit and receive nothing: the
    strip kernels agree with the single-call partition of every slot."""
    import ctypes

    from paper_2507_17087_b200 import native

    torch = cuda
    g = torch.Generator(device="cuda").manual_seed(ext[1] + P)
    n = ext[0] * ext[1]
    owner = torch.randint(-1, P + 1, (n,), device="cuda", dtype=torch.int32, generator=g)
    # mostly blocky: coarsen to 16x16 blocks, keep 1% noise
    r = torch.arange(ext[0], device="cuda") // 16
    c = torch.arange(ext[1], device="cuda") // 16
    blk = owner.view(ext)[(r * 16).clamp(max=ext[0] - 1)][:, (c * 16).clamp(max=ext[1] - 1)]
    noise = torch.rand(ext, device="cuda", generator=g) < 0.01
    owner = torch.where(noise, owner.view(ext), blk).contiguous().view(-1)
    want = halo_lists(owner, ext, (1, 1), P)
    lib = native.lib()
    ext_c = (ctypes.c_int64 * 2)(*ext)
    halo_c = (ctypes.c_int32 * 2)(1, 1)
    counts = torch.empty(P * P, dtype=torch.int64, device="cuda")
    offsets = torch.empty(P * P, dtype=torch.int64, device="cuda")
    nb = lib.pm_halo_scratch_bytes(ext_c, 2, P)
    scratch = torch.empty(nb, dtype=torch.uint8, device="cuda")
    total = want.total
    cells = torch.empty(max(total, 1), dtype=torch.int64, device="cuda")
    dims = torch.empty(max(total, 1), dtype=torch.int8, device="cuda")
    native.check(lib.pm_halo_lists(owner.data_ptr(), ext_c, 2, halo_c, P, counts.data_ptr(),
                                   offsets.data_ptr(), cells.data_ptr(), dims.data_ptr(),
                                   scratch.data_ptr(), nb, None), "pm_halo_lists")
    assert total > 0
    assert torch.equal(counts, want.pair_counts)
    assert torch.equal(offsets, want.pair_offsets)
    assert torch.equal(cells[:total], want.cells) and torch.equal(dims[:total], want.dims)


@pytest.mark.parametrize("ext,P", [((256, 1024), 8), ((77, 96), 6), ((9, 10, 11), 5)])
def test_capacity_mode_matches_exact(cuda, ext, P):
    """capacity= (no host round trip inside the call) gives the exact lists when the
    capacity suffices, and raises on access when it does not; repeated calls on one
    stream share the workspace without corrupting earlier results."""
    from paper_2507_17087_b200.errors import ProcMapError

    torch = cuda
    g = torch.Generator(device="cuda").manual_seed(sum(ext) * 7 + P)
    n = 1
    for e in ext:
        n *= e
    halo = (1,) * len(ext)
    owner = torch.randint(0, P, (n,), device="cuda", dtype=torch.int32, generator=g)
    owner2 = torch.randint(0, P, (n,), device="cuda", dtype=torch.int32, generator=g)
    want = halo_lists(owner, ext, halo, P)
    want2 = halo_lists(owner2, ext, halo, P)
    a = halo_lists(owner, ext, halo, P, capacity=want.total + 17)
    b = halo_lists(owner2, ext, halo, P, capacity=max(want.total, want2.total))
    for got, ref in ((a, want), (b, want2)):
        assert got.total == ref.total
        assert torch.equal(got.pair_counts, ref.pair_counts)
        assert torch.equal(got.pair_offsets, ref.pair_offsets)
        assert torch.equal(got.cells, ref.cells) and torch.equal(got.dims, ref.dims)
    small = halo_lists(owner, ext, halo, P, capacity=max(0, want.total - 1))
    with pytest.raises(ProcMapError):
        small.total
