"""The repo's MappingFunction plugged into the reference's own consumers.

The reference (installed unmodified into baseline/_ref) is the
caller here, not the checker of a restatement: its `expand_shards` /
`shard_policy` (tasksim/sim.py:67-120) and its `cmd_map` (cli.py:149-170) run
with this repo's `compile_mapper` result as the `MappingFn` plugin
(tasksim/sim.py:44), and what they produce must equal what they produce with
the reference's own mapper -- and equal the batched K1/K2 ownership lists.
"""

import io
import itertools
import json
import sys
import time
from contextlib import redirect_stdout

import pytest

from conftest import ROOT, golden

REF = ROOT / "baseline" / "_ref"
pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def procmap():
    if not (REF / "procmap").is_dir():
        pytest.skip("baseline/_ref (the pip-installed reference) is absent")
    sys.path.insert(0, str(REF))
    import procmap as pm  # noqa: F401
    import procmap.cli  # noqa: F401
    import procmap.dsl  # noqa: F401
    import procmap.tasksim.sim  # noqa: F401

    yield pm
    sys.path.remove(str(REF))


def _source(name):
    doc = golden("mappings")
    case = next(c for c in doc["cases"] if c["name"] == name)
    return doc["sources"][case["src"]]


CASES = [("matmul_mappers:cannon_mm", "cannon_mm", (1, 8), (16, 16)),
         ("matmul_mappers:cannon_mm", "cannon_mm", (2, 2), (6, 6)),
         ("matmul_mappers:solomonik_mm", "solomonik_mm", (2, 4), (4, 4, 4)),
         ("matmul_mappers:solomonik_shift", "solomonik_shift", (2, 4), (3, 5, 2)),
         ("matmul_mappers:cosma_mm", "cosma_mm", (8, 1), (2, 2, 2))]


@pytest.mark.parametrize("name,task,machine,ispace", CASES)
def test_reference_expand_shards_with_repo_mapper(procmap, cuda, name, task, machine, ispace):
    from paper_2507_17087_b200.dsl import compile_mapper, parse
    from paper_2507_17087_b200.ownership import shard_leaves
    from paper_2507_17087_b200.spaces import MachineShape

    src = _source(name)
    ours = compile_mapper(parse(src), task, MachineShape("GPU", *machine))
    import procmap.dsl as rdsl

    theirs = rdsl.compile_mapper(rdsl.parse(src), task, procmap.MachineShape("GPU", *machine))
    from procmap.tasksim.graph import IndexTask
    from procmap.tasksim.sim import expand_shards

    pts = tuple(itertools.product(*(range(e) for e in ispace)))
    t0 = time.perf_counter()
    tree_ours = expand_shards(IndexTask("t", pts), ours, ispace)
    t1 = time.perf_counter()
    tree_ref = expand_shards(IndexTask("t", pts), theirs, ispace)
    t2 = time.perf_counter()
    assert tree_ours.leaves == tree_ref.leaves
    assert tree_ours.targets == tree_ref.targets
    for leaf in tree_ref.leaves:
        assert tree_ours.subtasks[leaf].points == tree_ref.subtasks[leaf].points
    assert tree_ours.decisions == tree_ref.decisions
    # the batched path (K1 + K2 in one fused pass pair) gives the same leaves
    own = ours.map_partition(ispace)
    batched = shard_leaves("t", own, machine[1])
    assert [b[0] for b in batched] == list(tree_ref.leaves)
    for leaf, target, idx in batched:
        assert target == tree_ref.targets[leaf]
        assert tuple(pts[i] for i in idx.tolist()) == tree_ref.subtasks[leaf].points
    print(f"{name} {machine} {ispace}: expand_shards {len(pts)} points, repo mapper "
          f"{t1 - t0:.4f} s, reference mapper {t2 - t1:.4f} s")


def test_reference_cmd_map_with_repo_mapper(procmap, cuda, tmp_path, monkeypatch):
    """`procmap map` (the reference CLI) with the repo's parse/validate/
    compile_mapper patched in: byte-identical report to the stock run, and
    proc_counts equal to the K2 counts."""
    import procmap.cli as rcli

    from paper_2507_17087_b200 import dsl
    from paper_2507_17087_b200.ownership import partition, proc_counts
    from paper_2507_17087_b200.spaces import MachineShape

    mapper = tmp_path / "matmul.mapper"
    mapper.write_text(_source("matmul_mappers:cannon_mm"))
    argv = ["map", str(mapper), "--task", "cannon_mm", "--ispace", "12,10",
            "--machine", "2x4", "--format", "json"]

    def run():
        buf = io.StringIO()
        with redirect_stdout(buf):
            assert rcli.main(argv) == 0
        return buf.getvalue()

    stock = run()

    def load(path):
        program = dsl.parse(open(path).read())
        return program

    def compile_ours(program, task, machine):
        return dsl.compile_mapper(program, task, MachineShape(machine.kind, machine.nodes,
                                                              machine.procs_per_node))

    monkeypatch.setattr(rcli, "_load_mapper", load)
    monkeypatch.setattr(rcli, "compile_mapper", compile_ours)
    patched = run()
    assert patched == stock
    rep = json.loads(stock)
    fn = compile_ours(dsl.parse(mapper.read_text()), "cannon_mm", MachineShape("GPU", 2, 4))
    own = partition(fn.map_ispace((12, 10)), 8)
    assert proc_counts(own, 4) == rep["proc_counts"]
