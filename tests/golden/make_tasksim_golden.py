"""Generate tests/golden/tasksim.json by running the REFERENCE's lifecycle simulator.

Run in the build container (the reference is at /root/reference, read-only):

    python tests/golden/make_tasksim_golden.py

Records, for the corpus graph (tests/corpus/fghk.json) and seeded random task
graphs, the reference's trace records, per-processor statistics (or the Stuck
diagnosis) under the deterministic scheduler and the random scheduler with
several seeds, for the 2-D block mapping `block2d` (the corpus mapper
block2d_full.mapper: point * machine.size / ispace) on a few machine shapes;
plus load_taskgraph's error class on malformed documents.  The GPU box never
needs /root/reference.
"""

from __future__ import annotations

import itertools
import json
import random
import sys
from pathlib import Path

REF = Path("/root/reference/pkg")
sys.path.insert(0, str(REF / "src"))

from procmap.dsl import compile_mapper, parse  # noqa: E402
from procmap.errors import ProcMapError  # noqa: E402
from procmap.spaces import MachineShape  # noqa: E402
from procmap.tasksim import load_taskgraph, run_to_quiescence  # noqa: E402

OUT = Path(__file__).resolve().parent
BLOCK2D = (REF / "tests" / "corpus" / "block2d_full.mapper").read_text()
MACHINES = [(2, 2), (1, 4), (2, 3)]


def random_doc(rng: random.Random, n_max: int = 24) -> dict:
    """A random single-root forest: tasks with explicit points (subsets of a 2-D
    ispace) or ispace shorthands, random parents, sibling orders and acyclic
    sibling dependences (every dependence points forward in a shuffled order)."""
    n = rng.randint(2, n_max)
    ids = [f"t{i}" for i in range(n)]
    tasks, parents = [], []
    kids = {t: [] for t in ids}
    for i, tid in enumerate(ids):
        ext = [rng.randint(1, 4), rng.randint(1, 4)]
        r = rng.random()
        if r < 0.4:
            tasks.append({"id": tid, "ispace": ext})
        else:
            pts = [list(p) for p in itertools.product(range(ext[0]), range(ext[1]))]
            rng.shuffle(pts)
            pts = pts[:rng.randint(1, len(pts))]
            tasks.append({"id": tid, "points": pts, "ispace": ext})
        if i:
            p = rng.choice([ids[0]] + [t for t in ids[1:i] if rng.random() < 0.2])
            parents.append({"parent": p, "child": tid})
            kids[p].append(tid)
    deps, siblings = [], {}
    for p, group in kids.items():
        if len(group) > 1:
            order = group[:]
            rng.shuffle(order)
            if rng.random() < 0.5:
                siblings[p] = order[:]
            for a, b in itertools.combinations(range(len(order)), 2):
                if rng.random() < 0.25:
                    deps.append({"before": order[a], "after": order[b]})
    doc = {"tasks": tasks, "parent": parents, "deps": deps}
    if siblings:
        doc["siblings"] = siblings
    return doc


BAD_DOCS = [
    "not json",
    [],
    {"tasks": []},
    {"tasks": [{"id": "a/b", "ispace": [2]}]},
    {"tasks": [{"id": "a", "ispace": [2]}, {"id": "a", "ispace": [2]}]},
    {"tasks": [{"id": "a", "points": []}]},
    {"tasks": [{"id": "a", "points": [[0, 1], [0]]}]},
    {"tasks": [{"id": "a", "points": [[0, 1], [0, 1]]}]},
    {"tasks": [{"id": "a", "ispace": [0]}]},
    {"tasks": [{"id": "a"}]},
    {"tasks": [{"id": "a", "ispace": [1]}, {"id": "b", "ispace": [1]}]},
    {"tasks": [{"id": "a", "ispace": [1]}, {"id": "b", "ispace": [1]}],
     "parent": [{"parent": "a", "child": "b"}, {"parent": "b", "child": "a"}]},
    {"tasks": [{"id": "r", "ispace": [1]}, {"id": "a", "ispace": [1]}, {"id": "b", "ispace": [1]}],
     "parent": [{"parent": "r", "child": "a"}, {"parent": "r", "child": "b"}],
     "deps": [{"before": "a", "after": "b"}, {"before": "b", "after": "a"}]},
    {"tasks": [{"id": "r", "ispace": [1]}, {"id": "a", "ispace": [1]}],
     "parent": [{"parent": "r", "child": "a"}], "deps": [{"before": "a", "after": "a"}]},
    {"tasks": [{"id": "r", "ispace": [1]}, {"id": "a", "ispace": [1]}],
     "parent": [{"parent": "r", "child": "a"}], "siblings": {"r": ["a", "x"]}},
]


def main():
    rng = random.Random(20251019)
    docs = [json.loads((REF / "tests" / "corpus" / "fghk.json").read_text())]
    docs += [random_doc(rng) for _ in range(40)]
    # a graph that cannot finish (Stuck): a waits for its child x, x for b, b for a
    docs.append({"tasks": [{"id": "r", "ispace": [1]}, {"id": "a", "ispace": [2, 2]},
                           {"id": "b", "ispace": [2, 2]}, {"id": "x", "ispace": [2, 2]}],
                 "parent": [{"parent": "r", "child": "a"}, {"parent": "r", "child": "b"},
                            {"parent": "a", "child": "x"}],
                 "deps": [{"before": "a", "after": "b"}, {"before": "b", "after": "x"}]})
    cases = []
    for gi, doc in enumerate(docs):
        graph = load_taskgraph(doc)
        for machine in MACHINES:
            fn = compile_mapper(parse(BLOCK2D), "loop0", MachineShape("GPU", *machine))
            for scheduler, seed in [("deterministic", None), ("random", 1), ("random", 7),
                                    ("random", 12345)]:
                case = {"graph": gi, "machine": list(machine), "scheduler": scheduler,
                        "seed": seed}
                try:
                    tr = run_to_quiescence(graph, fn, MachineShape("GPU", *machine),
                                           scheduler=scheduler, seed=seed)
                    case["records"] = tr.records()
                    case["stats"] = [[list(k), v] for k, v in sorted(tr.proc_stats.items())]
                except ProcMapError as exc:
                    case["error"] = [type(exc).__name__, str(exc)]
                cases.append(case)
    bad = []
    for d in BAD_DOCS:
        try:
            load_taskgraph(d if not isinstance(d, str) else d)
            bad.append({"doc": d, "error": None})
        except ProcMapError as exc:
            bad.append({"doc": d, "error": [type(exc).__name__, str(exc)]})
    out = {"mapper": BLOCK2D, "task": "loop0", "graphs": docs, "cases": cases,
           "bad_docs": bad}
    (OUT / "tasksim.json").write_text(json.dumps(out, separators=(",", ":")))
    print(f"{len(cases)} simulator cases, {len(bad)} malformed documents")


if __name__ == "__main__":
    main()
