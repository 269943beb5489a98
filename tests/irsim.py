"""Test-only reference executor of a lowered point program (pm_program).

Executes the flat instruction list with Python ints exactly as the generated
CUDA does (floor division/modulo, 0/1 comparisons, structured if/else,
fail sites), and asserts that every value written to a register lies inside
that register's proven interval -- i.e. that the int32/int64/int128 widths
the code generator uses are exact.  Lets the lowering be checked against the
reference goldens on machines without a GPU.
"""

from paper_2507_17087_b200.dsl import lower as L


class Fail(Exception):
    def __init__(self, site, regs=None):
        super().__init__(site)
        self.site = site
        self.regs = list(regs or [])


def message(lowered, fail: "Fail") -> str:
    """The exception message the product formats for a failure (the registers a
    site's message quotes come from pm_map_probe on the GPU; here from the run)."""
    fmt = lowered.program.site_fmts.get(fail.site)
    if fmt is None:
        return str(lowered.program.sites[fail.site])
    return L.format_site(fmt, fail.regs)


def run(lowered, point):
    prog = lowered.program
    flat = prog.flat()
    ranges = prog.regs
    regs = [None] * len(ranges)

    def put(d, v):
        lo, hi = ranges[d]
        assert lo <= v <= hi, f"r{d}={v} outside proven range [{lo}, {hi}]"
        regs[d] = v

    # structured control flow: precompute matching ELSE/ENDIF
    match, stack = {}, []
    for i, ins in enumerate(flat):
        if ins[0] == L.OP_IF:
            stack.append([i, None])
        elif ins[0] == L.OP_ELSE:
            stack[-1][1] = i
        elif ins[0] == L.OP_ENDIF:
            start, els = stack.pop()
            match[start] = (els, i)
            if els is not None:
                match[els] = (None, i)
    pc = 0
    while pc < len(flat):
        op, d, a, b, c, site, lo, hi = flat[pc]
        if op == L.OP_CONST:
            v = (hi << 64) | (lo & ((1 << 64) - 1)) if prog.width_of(*ranges[d]) == 2 else lo
            if prog.width_of(*ranges[d]) == 2 and v >= 1 << 127:
                v -= 1 << 128
            put(d, v)
        elif op == L.OP_COORD:
            put(d, point[lo])
        elif op in (L.OP_ADD, L.OP_SUB, L.OP_MUL):
            x, y = regs[a], regs[b]
            put(d, x + y if op == L.OP_ADD else x - y if op == L.OP_SUB else x * y)
        elif op in (L.OP_DIV, L.OP_MOD):
            x, y = regs[a], regs[b]
            if y == 0:
                assert site >= 0, "unchecked division by zero"
                raise Fail(site, regs)
            if c & 1:
                assert x >= 0 and y > 0
            put(d, x // y if op == L.OP_DIV else x % y)
        elif op in (L.OP_GT, L.OP_LT, L.OP_EQ):
            x, y = regs[a], regs[b]
            put(d, int(x > y) if op == L.OP_GT else int(x < y) if op == L.OP_LT else int(x == y))
        elif op == L.OP_SELECT:
            put(d, regs[b] if regs[a] else regs[c])
        elif op == L.OP_MOV:
            put(d, regs[a])
        elif op == L.OP_CHECK:
            if not lo <= regs[a] < hi:
                raise Fail(site, regs)
        elif op == L.OP_FAIL:
            raise Fail(site, regs)
        elif op == L.OP_IF:
            els, end = match[pc]
            if regs[a] == 0:
                pc = (els if els is not None else end) + 1
                continue
        elif op == L.OP_ELSE:
            pc = match[pc][1] + 1
            continue
        elif op == L.OP_ENDIF:
            pass
        elif op == L.OP_RET:
            return regs[a]
        pc += 1
    raise AssertionError("program ended without RET")
