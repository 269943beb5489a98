"""Host-side drop-in surface vs the reference's goldens (CPU only).

Covers the parts of the plan that stay on the host: the Mapple front-end
(parser / printer / validator), the processor-space algebra, the decompose
optimizer and heuristic, and the communication-volume models
(reference tests: test_spaces.py, test_factorize.py, test_commvol.py,
test_dsl_parse.py).
"""

import itertools
from fractions import Fraction

import pytest
from hypothesis import given, settings, strategies as st

from conftest import golden
from paper_2507_17087_b200 import commvol as cv
from paper_2507_17087_b200 import factorize as fz
from paper_2507_17087_b200.dsl import ast, parse, to_source, validate
from paper_2507_17087_b200.dsl.validate import errors_of
from paper_2507_17087_b200.errors import (
    BadDimOrder,
    BadSliceBounds,
    DimOutOfRange,
    IndexOutOfRange,
    MapperSyntaxError,
    NonDivisibleSplit,
    ProductMismatch,
    ShapeMismatch,
    TooLarge,
)
from paper_2507_17087_b200.spaces import machine_space

# -- front-end ------------------------------------------------------------------


def test_canonical_text_matches_reference():
    for rec in golden("parse")["programs"]:
        prog = parse(rec["source"])
        assert to_source(prog) == rec["canonical"]
        assert parse(to_source(prog)) == prog


def test_diagnostics_match_reference():
    for rec in golden("parse")["programs"]:
        got = [[d.severity, d.code, d.line, d.col] for d in validate(parse(rec["source"]))]
        assert got == rec["diagnostics"]


def test_syntax_error_positions_match_reference():
    for rec in golden("parse")["errors"]:
        if rec["ok"]:
            parse(rec["source"])
            continue
        with pytest.raises(MapperSyntaxError) as info:
            parse(rec["source"])
        assert (info.value.line, info.value.col) == (rec["line"], rec["col"]), rec["source"]


def test_statement_details():
    task, region, layout = parse(
        "Task sweep GPU CPU\nRegion sweep r0 GPU FBMEM ZCMEM\nLayout sweep r0 GPU SOA Align == 128\n"
    ).statements
    assert task == ast.TaskMap("sweep", ("GPU", "CPU"))
    assert region == ast.DataMap("sweep", "r0", "GPU", ("FBMEM", "ZCMEM"))
    assert layout.constraints == ("SOA", ast.AlignConstraint("Align", 128))
    assert parse("").items == ()
    assert parse("t = (1, 2,)\n").globals[0].expr == ast.TupleLit((ast.IntLit(1), ast.IntLit(2)))


def test_validator_codes():
    src = ("def f(Tuple a, Tuple b):\n    return a[missing]\n"
           "def g(Tuple a, Tuple b):\n    c = f(a)\n    return c\n")
    assert sorted(d.code for d in errors_of(validate(parse(src)))) == [
        "ArityMismatch", "UndefinedVariable"]
    src = "m = Machine(GPU)\ndef f(Tuple a, Tuple b):\n    x = m.rotate(0, 1)\n    return a[m.rank]\n"
    assert sorted(d.code for d in errors_of(validate(parse(src)))) == [
        "UnknownMember", "UnknownPrimitive"]


_atoms = st.one_of(st.sampled_from([ast.Var("a"), ast.Var("b"), ast.Var("m")]),
                   st.integers(-9, 99).map(ast.IntLit))


def _exprs(children):
    ops = st.sampled_from(["+", "-", "*", "/", "%", ">", "<", "=="])
    index_arg = st.one_of(children, children.map(ast.Splat),
                          st.tuples(st.none() | children, st.none() | children).map(
                              lambda t: ast.SliceArg(t[0], t[1])))
    return st.one_of(
        st.tuples(ops, children, children).map(lambda t: ast.BinOp(*t)),
        st.tuples(children, children, children).map(lambda t: ast.Ternary(*t)),
        children.map(lambda e: ast.Member(e, "size")),
        st.tuples(children, st.lists(children, min_size=1, max_size=2)).map(
            lambda t: ast.MethodCall(t[0], "split", tuple(t[1]))),
        st.tuples(children, st.lists(index_arg, min_size=1, max_size=3)).map(
            lambda t: ast.Index(t[0], tuple(t[1]))),
        st.lists(children, min_size=1, max_size=3).map(lambda xs: ast.TupleLit(tuple(xs))),
        st.tuples(children, st.lists(st.integers(-3, 3), min_size=1, max_size=3)).map(
            lambda t: ast.TupleComprehension(t[0], "i", tuple(t[1]))),
    )


@settings(max_examples=200, deadline=None)
@given(st.recursive(_atoms, _exprs, max_leaves=25))
def test_generated_expression_round_trip(expr):
    program = ast.MapperProgram((ast.GlobalBinding("x", expr),))
    assert parse(to_source(program)) == program


# -- processor spaces (reference: test_spaces.py) --------------------------------


def test_space_goldens_and_errors():
    m = machine_space("GPU", 2, 4)
    assert m.split(1, 2).shape == (2, 2, 2)
    assert m.merge(0, 1).shape == (8,)
    assert m.merge(0, 1).resolve((5,)) == (1, 2)
    assert m.swap(0, 1).resolve((3, 1)) == (1, 3)
    assert m.slice(1, 1, 2).resolve((0, 1)) == (0, 2)
    assert m.decompose(1, (2, 2)).resolve((1, 1, 1)) == (1, 3)
    for bad, exc in [(lambda: m.split(1, 3), NonDivisibleSplit), (lambda: m.merge(1, 0), BadDimOrder),
                     (lambda: m.slice(1, 2, 1), BadSliceBounds), (lambda: m.split(5, 1), DimOutOfRange),
                     (lambda: m.decompose(1, (3, 2)), ProductMismatch),
                     (lambda: m.resolve((2, 0)), IndexOutOfRange),
                     (lambda: m.resolve((0,)), IndexOutOfRange)]:
        with pytest.raises(exc):
            bad()


def test_space_algebra_laws_exhaustive():
    for n, p in itertools.product((1, 2, 3, 4, 6, 8), repeat=2):
        m = machine_space("GPU", n, p)
        pts = list(m.indices())
        for i in range(2):
            for d in (x for x in range(1, m.shape[i] + 1) if m.shape[i] % x == 0):
                rt = m.split(i, d).merge(i, i + 1)
                assert all(rt.resolve(ix) == m.resolve(ix) for ix in pts)
        sw = m.swap(0, 1)
        assert all(sw.resolve((b, a)) == m.resolve((a, b)) for a, b in pts)
        assert len(set(m.materialize().values())) == m.size


# -- optimizer and volume models (reference: test_factorize.py, test_commvol.py) ---


def test_factorize_goldens():
    doc = golden("models")
    for rec in doc["search"]:
        best, score = fz.search_optimal(rec["d"], tuple(rec["extents"]))
        assert list(best) == rec["best"]
        assert score == Fraction(*rec["score"])
    for rec in doc["greedy"]:
        assert list(fz.greedy_grid(rec["d"], rec["k"])) == rec["grid"]
    for d in range(1, 200):
        for k in (1, 2, 3):
            fs = fz.enumerate_factorizations(d, k)
            assert len(fs) == fz.count_factorizations(d, k) == len(set(fs))
            assert fs == sorted(fs)


def test_volume_goldens():
    for rec in golden("models")["volumes"]:
        g = cv.BlockGrid(rec["extents"], rec["grid"])
        assert cv.surface_volume(g) == Fraction(*rec["surface"])
        assert cv.halo_volume(g, rec["halo"]) == Fraction(*rec["halo_volume"])
        for n, t in enumerate(rec["transpose"]):
            assert cv.transpose_volume(g, n) == Fraction(*t)
        assert cv.oracle_boundary_count(g, rec["halo"], cap=1 << 40) == rec["oracle"]
    big = cv.BlockGrid((32768, 32768), (2, 4))
    with pytest.raises(TooLarge):
        cv.oracle_boundary_count(big, (1, 1))
    with pytest.raises(ShapeMismatch):
        cv.BlockGrid((4, 4), (5, 1))


def test_paper_examples():
    assert cv.surface_volume(cv.BlockGrid((12, 18), (3, 2))) == 96
    assert cv.surface_volume(cv.BlockGrid((18, 12), (3, 2))) == 84
    assert fz.search_optimal(6, (12, 18))[0] == (2, 3)
    assert fz.greedy_grid(6, 2) == (3, 2)
