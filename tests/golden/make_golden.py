"""Generate the golden fixtures in tests/golden/ by running the REFERENCE.

Run in the build container (the reference is at /root/reference, read-only):

    python tests/golden/make_golden.py

It imports the reference package `procmap` (pkg/src) and records its outputs
on seeded inputs; the GPU box never needs /root/reference.  Fixtures:

* mappings.json  -- corpus mappers (tests/corpus copies are not needed: the
                    sources are embedded) and seeded random mapper programs:
                    per launch point the reference's (node, proc) or the
                    exception class it raised, via compile_mapper (cmd_map
                    semantics) and eval_mapping;
* parse.json     -- reference to_source() canonical text, validate() codes,
                    syntax-error positions;
* models.json    -- search_optimal / greedy_grid / surface_volume /
                    halo_volume / transpose_volume / oracle_boundary_count;
* shards.json    -- expand_shards leaves (ids, targets, point order).
"""

from __future__ import annotations

import itertools
import json
import random
import sys
from pathlib import Path

REF = Path("/root/reference/pkg")
sys.path.insert(0, str(REF / "src"))

from procmap import commvol as cv  # noqa: E402
from procmap import factorize as fz  # noqa: E402
from procmap.dsl import compile_mapper, eval_mapping, parse, to_source, validate  # noqa: E402
from procmap.errors import MapperSyntaxError  # noqa: E402
from procmap.spaces import MachineShape  # noqa: E402
from procmap.tasksim.graph import IndexTask  # noqa: E402
from procmap.tasksim.sim import expand_shards  # noqa: E402

OUT = Path(__file__).resolve().parent
CORPUS = REF / "tests" / "corpus"
MACHINES = [(2, 2), (2, 4), (1, 8), (8, 1), (4, 2), (3, 2), (1, 1)]


def points(ispace):
    return list(itertools.product(*(range(e) for e in ispace)))


def run_table(fn, ispace):
    """Per point: proc id (node * ppn + proc) or [error class name]."""
    rows = []
    for pt in points(ispace):
        try:
            node, proc = fn(pt, ispace)
            rows.append([node, proc])
        except Exception as exc:  # noqa: BLE001 - record the reference's behaviour
            rows.append({"error": type(exc).__name__, "message": str(exc)})
    return rows


# -- random mapper programs ------------------------------------------------------


class Gen:
    def __init__(self, rng: random.Random, rank: int):
        self.r = rng
        self.rank = rank

    def const(self):
        return str(self.r.choice([0, 1, 1, 2, 2, 3, 4, 5, 7, -1, -2, -3]))

    def int_atom(self):
        c = self.r.random()
        k = self.rank
        if c < 0.35:
            return f"p[{self.r.randrange(-k, k)}]"
        if c < 0.5:
            return f"s[{self.r.randrange(k)}]"
        if c < 0.65:
            return f"m.size[{self.r.randrange(2)}]"
        return self.const()

    def int_expr(self, d):
        if d <= 0:
            return self.int_atom()
        c = self.r.random()
        if c < 0.55:
            op = self.r.choice(["+", "-", "*", "/", "%", "/", "%", "+", ">", "<", "=="])
            return f"({self.int_expr(d - 1)} {op} {self.int_expr(d - 1)})"
        if c < 0.7:
            return (f"({self.int_expr(d - 1)} ? {self.int_expr(d - 1)} : "
                    f"{self.int_expr(d - 1)})")
        if c < 0.8:
            return f"{self.tuple_expr(d - 1)}[{self.r.randrange(-self.rank, self.rank)}]"
        if c < 0.88:
            return f"h({self.int_expr(d - 1)}, {self.int_expr(d - 1)})"
        if c < 0.94:
            # dynamic tuple index (bounded so it is mostly in range)
            return f"p[(({self.int_expr(d - 1)}) % {self.rank})]"
        return self.int_atom()

    def tuple_expr(self, d):
        c = self.r.random()
        k = self.rank
        if d <= 0 or c < 0.3:
            return self.r.choice(["p", "s", "p", "(p * 1)"])
        if c < 0.55:
            op = self.r.choice(["+", "-", "*", "/", "%"])
            rhs = self.tuple_expr(d - 1) if self.r.random() < 0.5 else self.int_expr(d - 1)
            return f"({self.tuple_expr(d - 1)} {op} {rhs})"
        if c < 0.7:
            items = ", ".join(self.int_expr(d - 1) for _ in range(k))
            return f"({items},)" if k == 1 else f"({items})"
        if c < 0.8:
            idx = ", ".join(map(str, range(k))) + ("," if k == 1 else "")
            return f"tuple(p[i] + {self.const()} for i in ({idx}))"
        if c < 0.9:
            return (f"(({self.int_expr(d - 1)}) ? {self.tuple_expr(d - 1)} : "
                    f"{self.tuple_expr(d - 1)})")
        return "s"

    def space_global(self, nodes, ppn):
        """A global transformed space `q` plus its rank."""
        opts = [("m", 2)]
        if ppn > 1:
            f = self.r.choice([d for d in range(1, ppn + 1) if ppn % d == 0])
            opts.append((f"m.split(1, {f})", 3))
        if nodes > 1:
            f = self.r.choice([d for d in range(1, nodes + 1) if nodes % d == 0])
            opts.append((f"m.split(0, {f}).swap(0, 2)", 3))
        tot = nodes * ppn
        f = self.r.choice([d for d in range(1, tot + 1) if tot % d == 0])
        opts.append((f"m.merge(0, 1).split(0, {f})", 2))
        opts.append(("m.swap(0, 1)", 2))
        opts.append(("m.merge(0, 1)", 1))
        if ppn > 1:
            opts.append((f"m.slice(1, 1, {ppn - 1})", 2))
        opts.append((f"m.merge(0, 1).decompose(0, {'(' + ', '.join(['4'] * self.rank) + (',)' if self.rank == 1 else ')')})",
                     self.rank))
        return self.r.choice(opts)

    def program(self, nodes, ppn):
        q, qrank = self.space_global(nodes, ppn)
        lines = ["m = Machine(GPU)", f"q = {q}",
                 "def h(a, b):", f"    return (a * 3 + b) % {self.r.randrange(1, 9)}",
                 "def f(Tuple p, Tuple s):"]
        nstmt = self.r.randrange(0, 3)
        for i in range(nstmt):
            if self.r.random() < 0.5:
                lines.append(f"    v{i} = {self.int_expr(2)}")
            else:
                lines.append(f"    v{i} = s[0] + {self.const()}")
        style = self.r.random()
        if qrank == 1:
            idx = self.int_expr(2)
            if style < 0.8:
                idx = f"({idx}) % q.size[0]"
            ret = f"q[{idx}]"
        else:
            if style < 0.45:
                parts = [f"({self.int_expr(2)}) % q.size[{i}]" for i in range(qrank)]
                ret = f"q[{', '.join(parts)}]"
            elif style < 0.75 and qrank == self.rank:
                ret = f"q[*(({self.tuple_expr(2)}) % q.size)]"
            elif style < 0.9:
                parts = [f"{self.int_expr(1)}" for _ in range(qrank)]
                ret = f"q[{', '.join(parts)}]"
            else:
                ret = f"(({self.int_expr(1)}) ? q[{', '.join(['0'] * qrank)}] : m[0, 0])"
        lines.append(f"    return {ret}")
        lines.append("IndexTaskMap t f")
        return "\n".join(lines) + "\n"


def mapping_cases():
    cases = []
    # corpus mappers, every bound task, several machines and launch shapes
    shapes2 = [(2, 2), (4, 4), (6, 6), (5, 3), (1, 7), (3, 8)]
    shapes3 = [(2, 2, 2), (4, 4, 4), (3, 3, 3), (2, 1, 3), (3, 1, 2), (4, 2, 1)]
    for path in sorted(CORPUS.glob("*.mapper")):
        src = path.read_text()
        prog = parse(src)
        for task, fname in sorted(prog.bindings().items()):
            func = prog.functions[fname]
            rank = 3 if "3D" in fname or "3d" in fname or fname in (
                "linearize_cyclic",) else 2
            for machine in MACHINES:
                m = MachineShape("GPU", *machine)
                for ispace in (shapes3 if rank == 3 else shapes2):
                    try:
                        fn = compile_mapper(prog, task, m)
                        table = run_table(fn, ispace)
                    except Exception as exc:  # noqa: BLE001
                        table = {"compile_error": type(exc).__name__}
                    cases.append({"name": f"{path.stem}:{task}", "source": src, "task": task,
                                  "func": func.name, "machine": list(machine),
                                  "ispace": list(ispace), "table": table})
    # the paper's/SPEC's named examples with eval_mapping semantics
    rng = random.Random(2507_17087)
    for n in range(260):
        rank = rng.choice([1, 2, 2, 3])
        machine = rng.choice(MACHINES[:6])
        g = Gen(rng, rank)
        src = g.program(*machine)
        try:
            prog = parse(src)
        except MapperSyntaxError as exc:
            raise SystemExit(f"generator produced unparsable source:\n{src}\n{exc}")
        ispace = tuple(rng.randrange(1, 5) for _ in range(rank))
        m = MachineShape("GPU", *machine)
        try:
            fn = compile_mapper(prog, "t", m)
            table = run_table(fn, ispace)
        except Exception as exc:  # noqa: BLE001
            table = {"compile_error": type(exc).__name__}
        ev_table = run_table(lambda pt, isp: eval_mapping(prog, "f", pt, isp, m), ispace)
        cases.append({"name": f"random{n}", "source": src, "task": "t", "func": "f",
                      "machine": list(machine), "ispace": list(ispace), "table": table,
                      "eval_table": ev_table})
    return cases


def parse_cases(mapping):
    srcs = sorted({c["source"] for c in mapping})
    out = {"programs": [], "errors": []}
    for src in srcs:
        prog = parse(src)
        out["programs"].append({
            "source": src,
            "canonical": to_source(prog),
            "diagnostics": [[d.severity, d.code, d.line, d.col] for d in validate(prog)],
        })
    bad = [
        "def f(:\n    return 1\n", "x = 1 @ 2\n", "Remap loop0 f\n", "def f(a, b):\nIndexTaskMap t f\n",
        "def return(a, b):\n    return a\n", "tuple = Machine(GPU)\n",
        "def f(a, b):\n    return a[b ? 1 : 2]\n", "x = (1, 2\n", "x = -y\n", "x = 1 +\n",
        "m = Machine(GPU)\ndef f(a, b):\n    return m[a[0] a[1]]\n",
        "def f(a, b):\n    return 0\ndef f(a, b):\n    return 1\n",
        "IndexTaskMap t\n", "Backpressure t x\n", "Layout t r GPU Align == \n",
        "x = tuple(i for i in (1, y))\n", "x = 3; y = 4\n", "x = a.b.c(1, )\n",
        "def g(a, b):\n  x = 1\n    return x\n",
    ]
    for src in bad:
        try:
            parse(src)
            out["errors"].append({"source": src, "ok": True})
        except MapperSyntaxError as exc:
            out["errors"].append({"source": src, "ok": False, "line": exc.line, "col": exc.col})
    return out


def model_cases():
    rng = random.Random(99)
    out = {"search": [], "greedy": [], "volumes": []}
    shapes = [(6, (12, 18)), (72, (8, 9)), (16, (4, 8, 4)), (2, (4, 4)), (8, (32768, 32768)),
              (8, (32768, 32768, 32768)), (4, (65536, 16384)), (8, (65536, 16384)),
              (4, (65536, 16384, 16384)), (8, (65536, 16384, 16384)), (8, (16384, 65536)),
              (1, (5,)), (12, (7, 7)), (48, (3, 5, 7)), (30, (100, 1, 10))]
    for _ in range(120):
        k = rng.randint(1, 3)
        shapes.append((rng.randint(1, 96), tuple(rng.randint(1, 300) for _ in range(k))))
    for d, ext in shapes:
        best, sc = fz.search_optimal(d, ext)
        out["search"].append({"d": d, "extents": list(ext), "best": list(best),
                              "score": [sc.numerator, sc.denominator]})
    for d in range(1, 130):
        for k in (1, 2, 3, 4):
            out["greedy"].append({"d": d, "k": k, "grid": list(fz.greedy_grid(d, k))})
    grids = [((12, 18), (3, 2), (1, 1)), ((18, 12), (3, 2), (1, 1)), ((5, 7), (2, 3), (2, 1)),
             ((32768, 32768), (2, 4), (1, 1)), ((32768, 32768), (4, 2), (1, 1)),
             ((4, 8, 4), (2, 4, 2), (1, 1, 1))]
    for _ in range(150):
        k = rng.choice([1, 2, 3])
        ext = tuple(rng.randint(1, 40) for _ in range(k))
        grid = tuple(rng.randint(1, e) for e in ext)
        halo = tuple(rng.randint(0, 4) for _ in range(k))
        grids.append((ext, grid, halo))
    for ext, grid, halo in grids:
        g = cv.BlockGrid(ext, grid)
        rec = {"extents": list(ext), "grid": list(grid), "halo": list(halo)}
        for name, val in (("surface", cv.surface_volume(g)), ("halo_volume", cv.halo_volume(g, halo))):
            rec[name] = [val.numerator, val.denominator]
        rec["transpose"] = [[v.numerator, v.denominator]
                            for v in (cv.transpose_volume(g, n) for n in range(len(ext)))]
        rec["oracle"] = cv.oracle_boundary_count(g, halo, cap=1 << 40)
        out["volumes"].append(rec)
    return out


def shard_cases():
    out = []
    progs = {
        "block2d": (CORPUS / "block2d_full.mapper").read_text(),
        "matmul": (CORPUS / "matmul_mappers.mapper").read_text(),
        "dist": (CORPUS / "distributions.mapper").read_text(),
    }
    plan = [("block2d", "loop0", (2, 2), (6, 6)), ("block2d", "loop0", (1, 8), (16, 16)),
            ("matmul", "cannon_mm", (1, 8), (4, 4)), ("matmul", "cannon_mm", (2, 4), (8, 8)),
            ("dist", "t_cyclic2D", (2, 2), (5, 7)), ("dist", "t_blockcyclic", (2, 2), (8, 8)),
            ("matmul", "solomonik_mm", (2, 4), (4, 4, 4))]
    for key, task, machine, ispace in plan:
        prog = parse(progs[key])
        fn = compile_mapper(prog, task, MachineShape("GPU", *machine))
        pts = points(ispace)
        tree = expand_shards(IndexTask(task, tuple(pts)), fn, ispace)
        out.append({"source": progs[key], "task": task, "machine": list(machine),
                    "ispace": list(ispace),
                    "leaves": [{"id": leaf, "target": list(tree.targets[leaf]),
                                "points": [list(p) for p in tree.subtasks[leaf].points]}
                               for leaf in tree.leaves]})
    return out


def cli_cases():
    """The reference CLI's exact stdout and exit code (cli.py:358-435)."""
    import contextlib
    import io
    import tempfile

    from procmap.cli import main as ref_main

    corpus = {p.stem: p.read_text() for p in CORPUS.glob("*.mapper")}
    plans = [
        ("map", "block2d_full", ["--task", "loop0", "--ispace", "6,6", "--machine", "2x2"]),
        ("map", "matmul_mappers", ["--task", "cannon_mm", "--ispace", "4,4", "--machine", "2x4"]),
        ("map", "matmul_mappers", ["--task", "solomonik_mm", "--ispace", "4,4,4", "--machine",
                                   "2x4"]),
        ("map", "distributions", ["--task", "t_cyclic2D", "--ispace", "5,3", "--format", "csv"]),
        ("map", "linear_cyclic", ["--task", "loop0", "--ispace", "7,2", "--machine", "1x8"]),
        ("map", "block2d_full", ["--task", "nosuchtask", "--ispace", "2,2"]),
        ("parse", "matmul_mappers", []),
        ("parse", "block2d_full", ["--format", "csv"]),
        ("decompose", None, ["6", "--extents", "12,18"]),
        ("decompose", None, ["8", "--extents", "65536,16384,16384"]),
        ("decompose", None, ["16", "--extents", "4,8,4", "--objective", "halo", "--halo", "1,2,1"]),
        ("decompose", None, ["8", "--extents", "12,18", "--strict"]),
        ("commvol", None, ["--extents", "12,18", "--grid", "3,2"]),
        ("commvol", None, ["--extents", "4,8,4", "--grid", "2,4,2", "--transpose-dims", "1",
                           "--halo", "1,0,2"]),
        ("sweep", None, []),
        ("sweep", None, ["--ratios", "1,4", "--areas", "1000000", "--gpus", "8,16",
                         "--format", "csv"]),
    ]
    out = []
    for cmd, mapper, rest in plans:
        argv = [cmd]
        path = None
        if mapper:
            fh = tempfile.NamedTemporaryFile("w", suffix=".mapper", delete=False)
            fh.write(corpus[mapper])
            fh.close()
            path = fh.name
            argv.append(path)
        argv += rest
        buf, err = io.StringIO(), io.StringIO()
        with contextlib.redirect_stdout(buf), contextlib.redirect_stderr(err):
            code = ref_main(argv)
        text = buf.getvalue()
        if path:
            text = text.replace(path, "@MAPPER@")
        out.append({"cmd": cmd, "mapper": mapper, "source": corpus.get(mapper), "args": rest,
                    "stdout": text, "exit": code})
    return out


def main():
    (OUT / "cli.json").write_text(json.dumps(cli_cases(), separators=(",", ":")))
    mapping = mapping_cases()
    sources = sorted({c["source"] for c in mapping})
    index = {s: i for i, s in enumerate(sources)}
    slim = [dict({k: v for k, v in c.items() if k != "source"}, src=index[c["source"]])
            for c in mapping]
    (OUT / "mappings.json").write_text(
        json.dumps({"sources": sources, "cases": slim}, separators=(",", ":")))
    (OUT / "parse.json").write_text(json.dumps(parse_cases(mapping), separators=(",", ":")))
    (OUT / "models.json").write_text(json.dumps(model_cases(), separators=(",", ":")))
    (OUT / "shards.json").write_text(json.dumps(shard_cases(), separators=(",", ":")))
    n_err = sum(1 for c in mapping if isinstance(c["table"], list)
                for r in c["table"] if isinstance(r, dict))
    n_pts = sum(len(c["table"]) for c in mapping if isinstance(c["table"], list))
    print(f"{len(mapping)} mapping cases, {n_pts} points ({n_err} reference errors)")


if __name__ == "__main__":
    main()
