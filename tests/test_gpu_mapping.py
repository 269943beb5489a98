"""K1 on the B200: the JIT-compiled point kernels vs the reference goldens,
plus the full 32768^2 stencil launch checked against its closed form and a
sampled oracle run."""

import itertools
import random
from concurrent.futures import ThreadPoolExecutor

import pytest

from conftest import mapping_cases
from oracle import mapple_oracle as O
from paper_2507_17087_b200.dsl import compile_mapper, eval_mapping, parse
from paper_2507_17087_b200.spaces import MachineShape

pytestmark = pytest.mark.gpu

CASES = [c for c in mapping_cases() if isinstance(c["table"], list)]


def _points(ispace):
    return list(itertools.product(*(range(e) for e in ispace)))


def _expect(table, ppn):
    ids, errs, msgs = [], [], []
    for row in table:
        if isinstance(row, dict):
            ids.append(-1)
            errs.append(row["error"])
            msgs.append(row["message"])
        else:
            ids.append(row[0] * ppn + row[1])
            errs.append(None)
            msgs.append(None)
    return ids, errs, msgs


@pytest.fixture(scope="module")
def built(cuda):
    dev = cuda.cuda.current_device()
    work = []
    for c in CASES:
        fn = compile_mapper(parse(c["source"]), c["task"], MachineShape("GPU", *c["machine"]))
        for implicit in (True, False):
            work.append((c, fn, fn.program_for(c["ispace"], implicit=implicit,
                                               k=len(c["ispace"]))))
    with ThreadPoolExecutor(8) as ex:
        list(ex.map(lambda w: w[2].plan(dev), work))
    return work


def test_golden_tables_implicit_and_explicit(built, cuda):
    torch = cuda
    for case, fn, pp in built:
        ispace = tuple(case["ispace"])
        ppn = case["machine"][1]
        want, errs, msgs = _expect(case["table"], ppn)
        n = len(want)
        status = torch.full((1,), -1, dtype=torch.int64, device="cuda")
        pts = None
        if pp.lowered.implicit:
            got = fn.map_ispace(ispace, check=False, status=status)
        else:
            pts = torch.tensor(_points(ispace), dtype=torch.int32, device="cuda").reshape(n, -1)
            got = fn.map_points(pts, ispace, check=False, status=status)
        assert got.tolist() == want, (case["name"], case["machine"], ispace)
        word = int(status.item())
        first_bad = next((i for i, e in enumerate(errs) if e), None)
        assert pp.failing_index(word) == first_bad
        if first_bad is not None:
            with pytest.raises(Exception) as info:
                pp.raise_for(word, pts)
            # the reference's class and exact message (point values from the probe)
            assert type(info.value).__name__ == errs[first_bad]
            assert str(info.value) == msgs[first_bad], (case["name"], first_bad)


def test_single_point_api_and_eval_mapping(cuda):
    picked = [c for c in CASES if "eval_table" in c][:40] + CASES[::25]
    for c in picked:
        prog = parse(c["source"])
        machine = MachineShape("GPU", *c["machine"])
        fn = compile_mapper(prog, c["task"], machine)
        ispace = tuple(c["ispace"])
        pts = _points(ispace)
        for i in sorted({0, len(pts) // 2, len(pts) - 1}):
            want = c["table"][i]
            if isinstance(want, dict):
                with pytest.raises(Exception) as info:
                    fn(pts[i], ispace)
                assert type(info.value).__name__ == want["error"]
                assert str(info.value) == want["message"]
            else:
                assert list(fn(pts[i], ispace)) == want
            if "eval_table" in c:
                want = c["eval_table"][i]
                if isinstance(want, dict):
                    with pytest.raises(Exception) as info:
                        eval_mapping(prog, c["func"], pts[i], ispace, machine)
                    assert type(info.value).__name__ == want["error"]
                    assert str(info.value) == want["message"]
                else:
                    assert list(eval_mapping(prog, c["func"], pts[i], ispace, machine)) == want


STENCIL = """
m = Machine(GPU)
def stencil_decompose(Tuple p, Tuple s):
    q = m.merge(0, 1).decompose(0, s)
    idx = p * q.size / s
    return q[*idx]
def stencil_heuristic(Tuple p, Tuple s):
    q = m.merge(0, 1).split(0, 4)
    idx = p * q.size / s
    return q[*idx]
IndexTaskMap stencil_d stencil_decompose
IndexTaskMap stencil_h stencil_heuristic
"""


@pytest.mark.parametrize("task,grid", [("stencil_d", (2, 4)), ("stencil_h", (4, 2))])
def test_full_stencil_launch_closed_form(cuda, task, grid):
    """1.07e9-point launch vs floor(x * d / l) (the block mapping's closed form)."""
    torch = cuda
    L = 32768
    fn = compile_mapper(parse(STENCIL), task, MachineShape("GPU", 1, 8))
    ids = fn.map_ispace((L, L))
    assert ids.numel() == L * L
    rows = L // 64
    for r0 in range(0, L, rows):
        x = torch.arange(r0, r0 + rows, device="cuda", dtype=torch.int64).view(-1, 1)
        y = torch.arange(L, device="cuda", dtype=torch.int64).view(1, -1)
        want = (x * grid[0] // L) + grid[0] * (y * grid[1] // L)
        got = ids[r0 * L:(r0 + rows) * L].view(rows, L).to(torch.int64)
        assert torch.equal(got, want), r0
    # sampled check against the CPU restatement of the reference evaluator
    rng = random.Random(5)
    prog = parse(STENCIL)
    ofn = O.OracleMapper(prog, task, ("GPU", 1, 8))
    idx = [rng.randrange(L * L) for _ in range(2000)]
    host = ids[torch.tensor(idx, device="cuda")].tolist()
    for i, got in zip(idx, host):
        assert got == ofn.proc_id(divmod(i, L), (L, L))


def test_sharded_launch_concatenates(cuda):
    """Contiguous chunks of the linear point range reproduce the whole launch."""
    torch = cuda
    c = next(c for c in CASES if c["name"].startswith("matmul_mappers:cannon_mm")
             and c["machine"] == [2, 4] and c["ispace"] == [6, 6])
    fn = compile_mapper(parse(c["source"]), "cannon_mm", MachineShape("GPU", 2, 4))
    whole = fn.map_ispace((6, 6))
    parts = torch.cat([fn.map_ispace((6, 6), first=f, count=n)
                       for f, n in ((0, 7), (7, 13), (20, 16))])
    assert torch.equal(whole, parts)
