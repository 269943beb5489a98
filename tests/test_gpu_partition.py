"""K2 on the B200: stable ownership partition vs the reference's shard trees
and vs a stable sort at scale."""

import pytest

from conftest import golden
from paper_2507_17087_b200.dsl import compile_mapper, parse
from paper_2507_17087_b200.ownership import partition, proc_counts, shard_leaves
from paper_2507_17087_b200.spaces import MachineShape
from paper_2507_17087_b200.errors import ProcMapError

pytestmark = pytest.mark.gpu


def test_shard_trees_match_reference(cuda):
    torch = cuda
    for case in golden("shards"):
        machine = MachineShape("GPU", *case["machine"])
        fn = compile_mapper(parse(case["source"]), case["task"], machine)
        ispace = tuple(case["ispace"])
        ids = fn.map_ispace(ispace)
        own = partition(ids, machine.size)
        leaves = shard_leaves(case["task"], own, machine.procs_per_node)
        pts = torch.cartesian_prod(*[torch.arange(e) for e in ispace]).view(-1, len(ispace))
        got = [{"id": lid, "target": list(tgt), "points": pts[idx.cpu().long()].tolist()}
               for lid, tgt, idx in leaves]
        assert got == case["leaves"], case["task"]
        counts = proc_counts(own, machine.procs_per_node)
        assert sum(r["points"] for r in counts) == ids.numel()


@pytest.mark.parametrize("n,nbins", [(1, 1), (1000, 3), (10_000_000, 8), (3_000_001, 100),
                                     (2_000_000, 4096), (65536, 257)])
def test_partition_is_a_stable_sort(cuda, n, nbins):
    torch = cuda
    g = torch.Generator(device="cuda").manual_seed(n + nbins)
    ids = torch.randint(0, nbins, (n,), device="cuda", dtype=torch.int32, generator=g)
    own = partition(ids, nbins)
    assert torch.equal(own.counts, torch.bincount(ids.long(), minlength=nbins))
    want = torch.sort(ids, stable=True).indices.to(torch.int32)
    assert torch.equal(own.perm, want)
    assert torch.equal(own.offsets, torch.cumsum(own.counts, 0) - own.counts)


def test_partition_rejects_bad_ids(cuda):
    torch = cuda
    ids = torch.zeros(5000, dtype=torch.int32, device="cuda")
    ids[1234] = 9
    with pytest.raises(ProcMapError):
        partition(ids, 8)
    empty = partition(torch.zeros(0, dtype=torch.int32, device="cuda"), 4)
    assert empty.counts.tolist() == [0, 0, 0, 0]


@pytest.mark.parametrize("n", [4096 * 300 + 17, 10_000_003])
def test_partition_block_ids_uniform_tiles(cuda, n):
    """Block-structured ids (the mapped-launch case: most 4096-id tiles hold one
    processor, so the scatter writes them as runs and the warp-per-tile histogram
    classifies them) mixed with a random stretch, also through an unaligned view (no
    16-byte loads), against a stable sort."""
    torch = cuda
    nbins = 8
    ids = (torch.arange(n, device="cuda", dtype=torch.int64) * nbins // n).to(torch.int32)
    g = torch.Generator(device="cuda").manual_seed(n)
    ids[n // 3: n // 3 + 50_000] = torch.randint(0, nbins, (50_000,), device="cuda",
                                                 dtype=torch.int32, generator=g)
    for view in (ids, ids[1:]):
        own = partition(view, nbins)
        assert torch.equal(own.counts, torch.bincount(view.long(), minlength=nbins))
        assert torch.equal(own.perm, torch.sort(view, stable=True).indices.to(torch.int32))


def test_partition_flags_bad_id_in_uniform_region(cuda):
    torch = cuda
    n = 4096 * 64
    ids = (torch.arange(n, device="cuda", dtype=torch.int64) * 4 // n).to(torch.int32)
    ids[4096 * 10 + 123] = -3  # inside an otherwise uniform tile: the vector path checks it
    with pytest.raises(ProcMapError):
        partition(ids, 4)
