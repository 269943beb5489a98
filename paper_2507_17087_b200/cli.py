"""Command line with the reference's report formats (reference: cli.py:1-435).

`python -m paper_2507_17087_b200 map MAPPER --task T --ispace a,b --machine NxP`
writes the same JSON/CSV report as `procmap map` (records in row-major point
order, cli.py:155-161; proc_counts sorted by (node, proc), cli.py:162-164) but
the per-point work runs on the GPU: K1 maps the launch, K2 counts points per
processor.  `decompose`, `commvol`, `sweep` and `parse` are host reports (the
same analytic models as the reference).  Exit codes: 0 ok, 1 domain error,
2 usage error (cli.py:10,422-431).
"""

from __future__ import annotations

import argparse
import csv
import json
import sys

from . import commvol as cv
from . import factorize as fz
from . import sweep as sw
from .dsl import ast as dsl_ast
from .dsl import compile_mapper, parse as parse_mapper, validate
from .dsl.validate import errors_of
from .errors import ProcMapError
from .spaces import MachineShape


def _ints(text: str) -> tuple:
    try:
        return tuple(int(x) for x in text.replace(";", ",").split(","))
    except ValueError:
        raise argparse.ArgumentTypeError(f"expected comma-separated integers, got {text!r}")


def _join(values) -> str:
    return ";".join(str(v) for v in values)


def _machine(args) -> MachineShape:
    kind, nodes, procs = "GPU", 2, 2
    if args.machine_config:
        try:
            with open(args.machine_config) as fh:
                doc = json.load(fh)
            kind = doc.get("kind", kind)
            nodes, procs = int(doc["nodes"]), int(doc["procs_per_node"])
        except (OSError, ValueError, KeyError, TypeError) as exc:
            raise ProcMapError(f"bad machine config {args.machine_config!r}: {exc}") from exc
    if args.machine is not None:
        try:
            a, b = args.machine.lower().split("x")
            nodes, procs = int(a), int(b)
        except (ValueError, TypeError) as exc:
            raise ProcMapError(f"bad --machine value {args.machine!r}: {exc}") from exc
    if args.kind is not None:
        kind = args.kind
    try:
        return MachineShape(kind, nodes, procs)
    except ValueError as exc:
        raise ProcMapError(str(exc)) from exc


def write_report(records, extras, args) -> None:
    """{"records": [...], **extras} as indented JSON, or the records as CSV (cli.py:74-94)."""
    out = open(args.out, "w") if args.out else sys.stdout
    try:
        if args.format == "json":
            doc = {"records": records}
            doc.update(extras)
            json.dump(doc, out, indent=2)
            out.write("\n")
        else:
            fields = []
            for r in records:
                fields += [k for k in r if k not in fields]
            w = csv.DictWriter(out, fieldnames=fields)
            w.writeheader()
            for r in records:
                w.writerow({k: "" if v is None else v for k, v in r.items()})
    finally:
        if args.out:
            out.close()


def _load(path):
    with open(path) as fh:
        program = parse_mapper(fh.read())
    diags = validate(program)
    for d in diags:
        print(f"{path}:{d}", file=sys.stderr)
    if errors_of(diags):
        raise ProcMapError(f"mapper {path!r} has validation errors")
    return program


def cmd_map(args) -> int:
    """Index-launch mapping on the GPU with cmd_map's report (cli.py:149-170)."""
    from .ownership import partition, proc_counts

    program = _load(args.mapper)
    machine = _machine(args)
    fn = compile_mapper(program, args.task, machine)
    ispace = tuple(args.ispace)
    ids = fn.map_ispace(ispace)                       # K1 (raises the reference's errors)
    own = partition(ids, machine.size)                # K2
    ppn = machine.procs_per_node
    host = ids.tolist()
    records = []
    npts = len(host)
    idx = [0] * len(ispace)
    for k in range(npts):
        node, proc = divmod(host[k], ppn)
        records.append({"point": _join(idx), "node": node, "proc": proc})
        for d in range(len(ispace) - 1, -1, -1):  # row-major successor, last dim fastest
            idx[d] += 1
            if idx[d] < ispace[d]:
                break
            idx[d] = 0
    write_report(records, {"task": args.task, "ispace": _join(ispace),
                           "proc_counts": proc_counts(own, ppn)}, args)
    return 0


def _objective(args, k):
    if args.objective == "isotropic":
        return fz.Isotropic()
    halo = args.halo if args.halo is not None else (1,) * k
    if args.objective == "halo":
        return fz.AnisotropicHalo(halo)
    return fz.WithTranspose(halo, frozenset(args.transpose_dims or ()))


def cmd_decompose(args) -> int:
    ext = args.extents
    obj = _objective(args, len(ext))
    best, s_best = fz.search_optimal(args.processors, ext, obj, strict=args.strict)
    heur = fz.greedy_grid(args.processors, len(ext))
    s_heur = fz.score(heur, ext, obj)
    rec = {
        "processors": args.processors, "extents": _join(ext), "objective": args.objective,
        "optimal": _join(best), "optimal_score": str(s_best), "optimal_score_float": float(s_best),
        "optimal_workload": _join(fz.workload_vector(best, ext)), "greedy": _join(heur),
        "greedy_score": str(s_heur), "greedy_score_float": float(s_heur),
        "amgm_bound": fz.amgm_lower_bound(args.processors, ext),
        "improvement_ratio": float(s_heur / s_best) if s_best else 1.0,
    }
    write_report([rec], {}, args)
    return 0


def cmd_commvol(args) -> int:
    grid = cv.BlockGrid(args.extents, args.grid)
    halo = args.halo if args.halo is not None else (1,) * grid.rank
    rec = {"extents": _join(args.extents), "grid": _join(args.grid), "halo": _join(halo),
           "surface_volume": str(cv.surface_volume(grid)),
           "halo_volume": str(cv.halo_volume(grid, halo))}
    if args.transpose_dims:
        rec["transpose_dims"] = _join(args.transpose_dims)
        rec["transpose_volumes"] = _join(str(cv.transpose_volume(grid, n))
                                         for n in args.transpose_dims)
    if not args.no_oracle:
        rec["oracle_count"] = cv.oracle_boundary_count(grid, halo)
    write_report([rec], {}, args)
    return 0


def cmd_sweep(args) -> int:
    recs = sw.sweep_configs(args.ratios or sw.TABLE3_RATIOS, args.areas or sw.TABLE3_AREAS,
                            args.gpus or sw.TABLE3_GPUS, args.gpus_per_node)
    write_report(recs, {"volumes": "model-predicted boundary element counts, not wall-clock",
                        "groups": sw.sweep_groups(recs)}, args)
    return 0


def cmd_parse(args) -> int:
    program = _load(args.mapper)
    recs = []
    for it in program.items:
        kind = type(it).__name__
        if isinstance(it, dsl_ast.GlobalBinding):
            recs.append({"kind": kind, "name": it.name})
        elif isinstance(it, dsl_ast.FuncDef):
            recs.append({"kind": kind, "name": it.name, "params": _join(p.name for p in it.params)})
        elif isinstance(it, dsl_ast.IndexTaskMap):
            recs.append({"kind": kind, "task": it.task, "func": it.func})
        elif isinstance(it, dsl_ast.TaskMap):
            recs.append({"kind": kind, "task": it.task, "procs": _join(it.procs)})
        elif isinstance(it, dsl_ast.DataMap):
            recs.append({"kind": kind, "task": it.task, "region": it.region, "proc": it.proc,
                         "memories": _join(it.memories)})
        elif isinstance(it, dsl_ast.DataLayout):
            parts = [f"{c.name}=={c.value}" if isinstance(c, dsl_ast.AlignConstraint) else c
                     for c in it.constraints]
            recs.append({"kind": kind, "task": it.task, "region": it.region, "proc": it.proc,
                         "constraints": _join(parts)})
        elif isinstance(it, dsl_ast.GarbageCollect):
            recs.append({"kind": kind, "task": it.task, "arg": it.arg})
        elif isinstance(it, dsl_ast.Backpressure):
            recs.append({"kind": kind, "task": it.task, "depth": it.depth})
    write_report(recs, {"mapper": args.mapper}, args)
    return 0


def build_parser() -> argparse.ArgumentParser:
    ap = argparse.ArgumentParser(prog="paper_2507_17087_b200",
                                 description="Mapple mapping on B200 (procmap-compatible reports)")
    sub = ap.add_subparsers(dest="cmd", required=True)

    def common(p):
        p.add_argument("--format", choices=["json", "csv"], default="json")
        p.add_argument("--out")

    def machine(p):
        p.add_argument("--machine")
        p.add_argument("--kind", choices=["CPU", "GPU", "OMP"])
        p.add_argument("--machine-config")

    p = sub.add_parser("parse")
    p.add_argument("mapper")
    common(p)
    p.set_defaults(fn=cmd_parse)
    p = sub.add_parser("map")
    p.add_argument("mapper")
    p.add_argument("--task", required=True)
    p.add_argument("--ispace", type=_ints, required=True)
    machine(p)
    common(p)
    p.set_defaults(fn=cmd_map)
    p = sub.add_parser("decompose")
    p.add_argument("processors", type=int)
    p.add_argument("--extents", type=_ints, required=True)
    p.add_argument("--objective", choices=["isotropic", "halo", "transpose"], default="isotropic")
    p.add_argument("--halo", type=_ints)
    p.add_argument("--transpose-dims", type=_ints)
    p.add_argument("--strict", action="store_true")
    common(p)
    p.set_defaults(fn=cmd_decompose)
    p = sub.add_parser("commvol")
    p.add_argument("--extents", type=_ints, required=True)
    p.add_argument("--grid", type=_ints, required=True)
    p.add_argument("--halo", type=_ints)
    p.add_argument("--transpose-dims", type=_ints)
    p.add_argument("--no-oracle", action="store_true")
    common(p)
    p.set_defaults(fn=cmd_commvol)
    p = sub.add_parser("sweep")
    p.add_argument("--ratios", type=_ints)
    p.add_argument("--areas", type=_ints)
    p.add_argument("--gpus", type=_ints)
    p.add_argument("--gpus-per-node", type=int, default=4)
    common(p)
    p.set_defaults(fn=cmd_sweep)
    return ap


def main(argv=None) -> int:
    ap = build_parser()
    try:
        args = ap.parse_args(argv)
    except SystemExit as exc:
        return int(exc.code or 0)
    try:
        return args.fn(args)
    except (ProcMapError, OSError) as exc:
        print(f"error: {exc}", file=sys.stderr)
        return 1
