"""Pin the oracle (CPU restatement) against the reference's own outputs.

The golden vectors were produced by running the reference itself
(tests/golden/make_golden.py); the oracle must reproduce every assignment and
every exception class, so it can stand in for the reference on the GPU box.
"""

import itertools
from fractions import Fraction

import pytest

from conftest import golden, mapping_cases
from oracle import mapple_oracle as O
from paper_2507_17087_b200.dsl import parse


def _points(ispace):
    return list(itertools.product(*(range(e) for e in ispace)))


def _check_table(fn, ispace, table):
    for pt, want in zip(_points(ispace), table):
        if isinstance(want, dict):
            with pytest.raises(Exception) as info:
                fn(pt, ispace)
            assert type(info.value).__name__ == want["error"], (pt, want)
        else:
            assert list(fn(pt, ispace)) == want, pt


CASES = mapping_cases()


@pytest.mark.parametrize("case", CASES, ids=[f"{c['name']}-{c['machine']}-{c['ispace']}"
                                             for c in CASES])
def test_oracle_mapping_tables(case):
    prog = parse(case["source"])
    machine = ("GPU", *case["machine"])
    ispace = tuple(case["ispace"])
    if isinstance(case["table"], dict):
        with pytest.raises(Exception) as info:
            O.OracleMapper(prog, case["task"], machine)
        assert type(info.value).__name__ == case["table"]["compile_error"]
        return
    fn = O.OracleMapper(prog, case["task"], machine)
    _check_table(fn, ispace, case["table"])
    if "eval_table" in case:
        _check_table(lambda p, s: O.eval_point(prog, case["func"], p, s, machine), ispace,
                     case["eval_table"])


def test_oracle_models():
    doc = golden("models")
    for rec in doc["search"]:
        assert list(O.search_optimal(rec["d"], rec["extents"])) == rec["best"]
    for rec in doc["greedy"]:
        assert list(O.greedy_grid(rec["d"], rec["k"])) == rec["grid"]
    for rec in doc["volumes"]:
        ext, grid, halo = rec["extents"], rec["grid"], rec["halo"]
        assert O.surface_volume(ext, grid) == Fraction(*rec["surface"])
        if sum(ext) < 400:
            assert O.boundary_count(ext, grid, halo) == rec["oracle"]


def test_oracle_shards():
    for case in golden("shards"):
        prog = parse(case["source"])
        machine = ("GPU", *case["machine"])
        ispace = tuple(case["ispace"])
        fn = O.OracleMapper(prog, case["task"], machine)
        pts = O.row_major(ispace)
        targets = [tuple(fn(p, ispace)) for p in pts]
        leaves = O.shard_leaves(case["task"], pts, targets)
        want = {l["id"]: (tuple(l["target"]), [tuple(p) for p in l["points"]])
                for l in case["leaves"]}
        assert leaves == want
