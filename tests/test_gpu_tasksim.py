"""The lifecycle simulator fed by batched ownership on the B200.

Every task's shard tree comes from one fused K1 + K2 launch over its points
(tasksim.expand_shards with a repo MappingFunction); the traces must equal the
reference simulator's (tests/golden/tasksim.json) and be accepted by the
reference's own trace checker (check_trace, tasksim/check.py:29-248, from the
unmodified reference in baseline/_ref) driven with the same repo mapper.
"""

import sys

import pytest

from conftest import ROOT, golden
from paper_2507_17087_b200 import tasksim as T
from paper_2507_17087_b200.dsl import compile_mapper, parse
from paper_2507_17087_b200.spaces import MachineShape

pytestmark = pytest.mark.gpu
DOC = golden("tasksim")
REF = ROOT / "baseline" / "_ref"


def _fn(machine):
    return compile_mapper(parse(DOC["mapper"]), DOC["task"], MachineShape("GPU", *machine))


def test_batched_shard_trees_equal_per_point_trees(cuda):
    for doc in DOC["graphs"][:12]:
        graph = T.load_taskgraph(doc)
        for machine in ((2, 2), (1, 4), (2, 3)):
            fn = _fn(machine)
            for tid, task in graph.tasks.items():
                if tid == graph.root:
                    continue
                ispace = graph.ispaces[tid]
                batched = T.expand_shards(task, fn, ispace)               # K1 + K2
                per_point = T.shard_tree(task, [fn(p, ispace) for p in task.points])
                assert batched == per_point, (tid, machine)


def test_traces_equal_reference_with_batched_trees(cuda):
    for case in DOC["cases"][::7]:
        graph = T.load_taskgraph(DOC["graphs"][case["graph"]])
        machine = tuple(case["machine"])
        args = dict(scheduler=case["scheduler"], seed=case["seed"])
        if "error" in case:
            with pytest.raises(Exception) as info:
                T.run_to_quiescence(graph, _fn(machine), MachineShape("GPU", *machine), **args)
            assert [type(info.value).__name__, str(info.value)] == case["error"]
            continue
        tr = T.run_to_quiescence(graph, _fn(machine), MachineShape("GPU", *machine), **args)
        assert tr.records() == case["records"]
        assert [[list(k), v] for k, v in sorted(tr.proc_stats.items())] == case["stats"]


def test_reference_check_trace_accepts_the_traces(cuda):
    if not (REF / "procmap").is_dir():
        pytest.skip("baseline/_ref (the pip-installed reference) is absent")
    sys.path.insert(0, str(REF))
    try:
        from procmap.tasksim import check_trace
        from procmap.tasksim import load_taskgraph as ref_load
    finally:
        sys.path.remove(str(REF))
    for case in DOC["cases"][::11]:
        if "error" in case:
            continue
        doc = DOC["graphs"][case["graph"]]
        machine = tuple(case["machine"])
        fn = _fn(machine)
        tr = T.run_to_quiescence(T.load_taskgraph(doc), fn, MachineShape("GPU", *machine),
                                 scheduler=case["scheduler"], seed=case["seed"])
        diags = check_trace(tr.records(), ref_load(doc), fn)
        assert not diags, [str(d) for d in diags][:5]
