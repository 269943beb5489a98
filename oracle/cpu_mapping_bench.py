"""ORACLE (test / bench-baseline infrastructure only): the CPU mapping baseline.

Times the reference's own per-point mapping (kind "reference": the unmodified
reference pip-installed into baseline/_ref) or the oracle's restatement of it
(kind "port") over the reference's index-launch loop
(cmd_map, cli.py:149-161: compile_mapper once, then fn(point, ispace) for the
row-major points of the launch; interp.py:366-433 for the per-ispace prefix
cache and the per-point suffix) on the host cores, as SURVEY.md §8(d) asks:
one core, and every core of the affinity mask with one worker process per core
each mapping its own contiguous slice of the launch.  Each worker maps for a
bounded wall time and reports how many points it mapped; the full launch time
is extrapolated linearly from the measured rate (labelled as such).

Only bench.py's cpu_baseline leg calls this; nothing in the product imports it.
"""

from __future__ import annotations

import multiprocessing as mp
import os
import sys
import time
from pathlib import Path


REF_PATH = Path(__file__).resolve().parents[1] / "baseline" / "_ref"


def reference_available() -> bool:
    """The unmodified reference, pip-installed into baseline/_ref."""
    return (REF_PATH / "procmap").is_dir()


def _mapper(kind, src, task, machine):
    """A per-point callable (point, ispace) -> anything, built once per worker."""
    if kind == "reference":
        # the reference itself: compile_mapper + MappingFunction.__call__
        # (dsl/interp.py:401-433), exactly what cmd_map calls per point (cli.py:158-161)
        if str(REF_PATH) not in sys.path:
            sys.path.insert(0, str(REF_PATH))
        from procmap.dsl import compile_mapper, parse
        from procmap.spaces import MachineShape

        return compile_mapper(parse(src), task, MachineShape(*machine))
    from oracle.mapple_oracle import OracleMapper
    from paper_2507_17087_b200.dsl import parse

    return OracleMapper(parse(src), task, machine).proc_id


def _worker(job):
    src, task, machine, ispace, first, seconds, kind = job
    fn = _mapper(kind, src, task, machine)
    strides = [1] * len(ispace)
    for m in range(len(ispace) - 2, -1, -1):
        strides[m] = strides[m + 1] * ispace[m + 1]
    total = 1
    for e in ispace:
        total *= e
    i = first
    done = 0
    t0 = time.perf_counter()
    while True:
        for _ in range(256):
            rem, pt = i % total, []
            for s in strides:
                q, rem = divmod(rem, s)
                pt.append(q)
            fn(tuple(pt), ispace)  # row-major, last dimension fastest (cli.py:155-157)
            i += 1
        done += 256
        dt = time.perf_counter() - t0
        if dt >= seconds:
            return done, dt


def cpu_mapping_rate(src: str, task: str, machine: tuple, ispace: tuple, *, seconds: float = 3.0,
                     procs: int | None = None, kind: str = "port") -> dict:
    """Points/s of per-point mapping on the host: 1 core, then `procs` cores
    (default: the affinity mask), each on a contiguous slice of the launch.
    kind "reference": the reference itself (baseline/_ref); "port": the oracle."""
    total = 1
    for e in ispace:
        total *= e
    n1, t1 = _worker((src, task, machine, ispace, 0, seconds, kind))
    ncores = procs or len(os.sched_getaffinity(0))
    jobs = [(src, task, machine, ispace, total * k // ncores, seconds, kind)
            for k in range(ncores)]
    ctx = mp.get_context("spawn")  # the parent holds a CUDA context: never fork it
    with ctx.Pool(ncores) as pool:
        res = pool.map(_worker, jobs)
    # aggregate rate: every worker ran concurrently for ~`seconds`
    rate_all = sum(n / t for n, t in res)
    return {"kind": kind, "points_per_s_1core": n1 / t1, "points_per_s_all": rate_all, "cores": ncores,
            "sample_points_1core": n1, "sample_points_all": sum(n for n, _ in res),
            "seconds_per_worker": seconds, "launch_points": total,
            "extrapolated_launch_s_1core": total / (n1 / t1),
            "extrapolated_launch_s_all": total / rate_all}
