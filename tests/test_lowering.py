"""The lowered point programs reproduce the reference on every golden case.

Runs the lowering (dsl/lower.py) for every golden mapper x machine x launch
shape, in both the implicit (row-major ispace) and explicit (int32 points)
modes and in eval_mapping order, executes the program with the test-only IR
executor (tests/irsim.py, which also proves the register widths exact), and
compares per point with the reference's (node, proc) or exception class.
CPU only: the sm_100a kernels are checked against the same goldens in
test_gpu_mapping.py.
"""

import itertools

import pytest

import irsim
from conftest import mapping_cases
from paper_2507_17087_b200.dsl import compile_mapper, parse
from paper_2507_17087_b200.dsl.interp import Evaluator
from paper_2507_17087_b200.dsl.lower import Lowerer, lower_mapping
from paper_2507_17087_b200.spaces import MachineShape

CASES = mapping_cases()


def _points(ispace):
    return list(itertools.product(*(range(e) for e in ispace)))


def _compare(lowered, ispace, table, ppn):
    for pt, want in zip(_points(ispace), table):
        try:
            got = irsim.run(lowered, pt)
        except irsim.Fail as f:
            assert isinstance(want, dict), (pt, "kernel failed", lowered.program.sites[f.site], want)
            assert type(lowered.program.sites[f.site]).__name__ == want["error"], pt
            # the reference's exact message, point-specific values included
            assert irsim.message(lowered, f) == want["message"], (pt, want)
            continue
        assert not isinstance(want, dict), (pt, got, want)
        assert list(divmod(got, ppn)) == want, pt


@pytest.mark.parametrize("case", CASES, ids=[f"{c['name']}-{c['machine']}-{c['ispace']}"
                                             for c in CASES])
def test_lowered_program_matches_reference(case):
    prog = parse(case["source"])
    machine = MachineShape("GPU", *case["machine"])
    ispace = tuple(case["ispace"])
    if isinstance(case["table"], dict):
        with pytest.raises(Exception) as info:
            compile_mapper(prog, case["task"], machine)
        assert type(info.value).__name__ == case["table"]["compile_error"]
        return
    fn = compile_mapper(prog, case["task"], machine)
    ppn = machine.procs_per_node
    for implicit in (True, False):
        low = Lowerer(prog, machine, globals_env=fn.evaluator.globals)
        lowered = lower_mapping(low, fn.func, ispace, implicit=implicit,
                                n_coords=len(ispace), plan_mode=True)
        _compare(lowered, ispace, case["table"], ppn)
    if "eval_table" in case:
        ev = Evaluator(prog, machine)
        low = Lowerer(prog, machine, globals_env=ev.globals)
        lowered = lower_mapping(low, prog.functions[case["func"]], ispace, implicit=False,
                                n_coords=len(ispace), plan_mode=False)
        _compare(lowered, ispace, case["eval_table"], ppn)


def test_lazy_ternary_and_recursion_guard():
    src = ("m = Machine(GPU)\n"
           "def f(Tuple p, Tuple s):\n"
           "    return p[0] > 0 ? m[p[0] / p[0] - 1, 0] : m[1 / p[0], 0]\n"
           "def loop(Tuple p, Tuple s):\n"
           "    return loop(p, s)\n"
           "IndexTaskMap a f\nIndexTaskMap b loop\n")
    prog = parse(src)
    machine = MachineShape("GPU", 2, 2)
    fn = compile_mapper(prog, "a", machine)
    low = Lowerer(prog, machine, globals_env=fn.evaluator.globals)
    lowered = lower_mapping(low, fn.func, (3, 1), implicit=True, n_coords=2, plan_mode=True)
    with pytest.raises(irsim.Fail):
        irsim.run(lowered, (0, 0))           # untaken branch is fine, taken one divides by 0
    assert irsim.run(lowered, (1, 0)) == 0   # (1/1 - 1, 0)
    fn = compile_mapper(prog, "b", machine)
    low = Lowerer(prog, machine, globals_env=fn.evaluator.globals)
    lowered = lower_mapping(low, fn.func, (2, 2), implicit=True, n_coords=2, plan_mode=True)
    assert lowered.dead
    assert "call depth" in str(lowered.program.sites[0])


def test_wide_values_use_int128():
    src = ("m = Machine(GPU)\n"
           "def f(Tuple p, Tuple s):\n"
           "    x = p[0] * 1000000000000 * 1000000000000\n"
           "    return m[(x / 1000000000000 / 1000000000000) % 2, 0]\n"
           "IndexTaskMap a f\n")
    prog = parse(src)
    machine = MachineShape("GPU", 2, 2)
    fn = compile_mapper(prog, "a", machine)
    low = Lowerer(prog, machine, globals_env=fn.evaluator.globals)
    lowered = lower_mapping(low, fn.func, (1,), implicit=False, n_coords=1, plan_mode=True)
    assert 2 in lowered.program.widths()
    for v in (-5, 0, 3, 2**31 - 1, -(2**31)):
        assert irsim.run(lowered, (v,)) == (v % 2) * 2
