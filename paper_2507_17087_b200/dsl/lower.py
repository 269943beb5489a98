"""Symbolic evaluation of a Mapple mapping function into a GPU point program.

This is the host half of the batched mapping plan.  It runs the reference
evaluator's semantics (reference: dsl/interp.py:47-309, the per-ispace
prefix/suffix plan of dsl/interp.py:366-418) once per (mapper, ispace), with
the iteration point *symbolic*:

* point-independent values (globals, the prefix, `decompose` via
  `search_optimal`, every processor space) fold to concrete Python values on
  the host, exactly as the reference computes them;
* point-dependent integers become registers of a straight-line program
  (`Program`) with an interval per register, so the CUDA code generator
  (csrc/codegen.cpp) can pick int32 / int64 / int128 arithmetic that is exact
  for every possible input (Python ints are unbounded);
* `space[idx]` with a symbolic index becomes range checks plus the inverse of
  the space's transform chain as integer arithmetic (spaces.py:185-213), and
  the result is the linear processor id `node * procs_per_node + proc`;
* every error the reference would raise becomes a FAIL site at the same
  place in evaluation order, inside the branch that would raise it, so a lazy
  ternary (interp.py:134-139) never fires an error of the untaken branch.
  The host re-raises the site's exception (same class, same message) for the
  lowest failing point, as the reference's row-major loop would
  (cli.py:155-161).

Values during lowering: Python `int`; `Reg` (symbolic int); `tuple` of those;
`ProcSpace`; `ProcRef` (concrete processor); `DynProc` (symbolic processor
id); `Choice` (a ternary whose two branches produced values that cannot be
merged into registers, e.g. two different spaces).  Operations that inspect a
value's type fork on a `Choice` (`split_on`), duplicating the rest of that
expression's evaluation into both branches.
"""

from __future__ import annotations

import sys
from dataclasses import dataclass

from ..errors import EvalError, LoweringError, ProcMapError
from ..factorize import search_optimal
from ..spaces import Merge, ProcSpace, Slice, Split, Swap
from . import ast as A

MAX_CALL_DEPTH = 64          # reference: dsl/interp.py:24,81-82
MAX_INSNS = 200_000          # lowering budget (recursion / fan-out blow-up guard)
MAX_FANOUT = 64              # symbolic value enumerated into concrete cases

INT32 = (-(1 << 31), (1 << 31) - 1)
INT64 = (-(1 << 63), (1 << 63) - 1)
INT128 = (-(1 << 127), (1 << 127) - 1)

# opcodes: keep in sync with include/mapple_b200.h (PM_OP_*)
(OP_CONST, OP_COORD, OP_ADD, OP_SUB, OP_MUL, OP_DIV, OP_MOD, OP_GT, OP_LT, OP_EQ,
 OP_SELECT, OP_MOV, OP_CHECK, OP_FAIL, OP_IF, OP_ELSE, OP_ENDIF, OP_RET) = range(18)
OP_NAMES = ("CONST COORD ADD SUB MUL DIV MOD GT LT EQ SELECT MOV CHECK FAIL IF ELSE "
            "ENDIF RET").split()


@dataclass(frozen=True)
class ProcRef:
    """A resolved processor (reference: dsl/interp.py:27-33)."""

    node: int
    proc: int


class Reg:
    """A symbolic integer: register id plus a value interval [lo, hi]."""

    __slots__ = ("id", "lo", "hi")

    def __init__(self, rid: int, lo: int, hi: int):
        self.id, self.lo, self.hi = rid, lo, hi

    def __repr__(self):
        return f"r{self.id}[{self.lo},{self.hi}]"


class DynProc:
    """A symbolic processor reference: `reg` holds node * ppn + proc."""

    __slots__ = ("reg",)

    def __init__(self, reg: Reg):
        self.reg = reg


class Choice:
    """`a` if cond != 0 else `b`, for values that cannot share registers."""

    __slots__ = ("cond", "a", "b")

    def __init__(self, cond: Reg, a, b):
        self.cond, self.a, self.b = cond, a, b


class _Bottom:
    __slots__ = ()

    def __repr__(self):
        return "BOTTOM"


BOTTOM = _Bottom()


class _Dead(Exception):
    """Evaluation of the current control path ended at a FAIL site."""


def _is_int(v) -> bool:
    return isinstance(v, (int, Reg)) and not isinstance(v, bool)


def _tuple_pieces(vals) -> list:
    """Message pieces printing a tuple of ints / registers as Python does."""
    out = ["("]
    for k, v in enumerate(vals):
        if k:
            out.append(", ")
        out.append(v)
    out.append(",)" if len(vals) == 1 else ")")
    return out


def format_site(fmt: tuple, regs) -> str:
    """The message of a site from its pieces and the failing point's registers."""
    return "".join(p if isinstance(p, str) else str(regs[p[1]]) if isinstance(p, tuple)
                   else str(p) for p in fmt)


def type_name(v) -> str:
    if isinstance(v, (bool, int, Reg)):
        return "Int"
    if isinstance(v, tuple):
        return "Tuple"
    if isinstance(v, ProcSpace):
        return "Space"
    if isinstance(v, (ProcRef, DynProc)):
        return "ProcessorRef"
    return type(v).__name__


def _floordiv(a: int, b: int) -> int:
    return a // b


def _range_of(op: str, a: tuple, b: tuple) -> tuple[int, int]:
    """Exact value range of `a op b` for a, b ranging over intervals."""
    (alo, ahi), (blo, bhi) = a, b
    if op == "+":
        return alo + blo, ahi + bhi
    if op == "-":
        return alo - bhi, ahi - blo
    if op == "*":
        c = (alo * blo, alo * bhi, ahi * blo, ahi * bhi)
        return min(c), max(c)
    if op in ("/", "%"):
        divs = [x for x in {blo, bhi, 1, -1} if x != 0 and blo <= x <= bhi]
        if not divs:  # divisor is always zero: no value survives
            return 0, 0
        if op == "/":
            c = [x // d for x in (alo, ahi) for d in divs]
            return min(c), max(c)
        lo = 0 if blo > 0 else min(blo + 1, 0)
        hi = 0 if bhi < 0 else max(bhi - 1, 0)
        if alo >= 0 and blo > 0 and ahi < blo:  # remainder is the dividend itself
            return alo, ahi
        return lo, hi
    return 0, 1  # comparisons


class Program:
    """The lowered point program in structured form."""

    def __init__(self):
        self.regs: list[list[int]] = []    # per register [lo, hi] (union of assignments)
        self.consts: dict[int, Reg] = {}
        self.const_insns: list[tuple] = []
        self.body: list = []                # insn tuples and ("if", cond, then, else)
        self.sites: list[Exception] = []
        self.site_fmts: dict[int, tuple] = {}   # site -> message pieces (str / int / ("r", id))
        self._site_keys: dict = {}
        self.n_insns = 0
        self.coords: list[Reg] = []

    def new_reg(self, lo: int, hi: int) -> Reg:
        self.regs.append([lo, hi])
        return Reg(len(self.regs) - 1, lo, hi)

    def site(self, exc: Exception, fmt: tuple | None = None) -> int:
        """A failure site.  `fmt` (for messages that quote per-point values) is a
        sequence of str pieces and Reg / int operands: the host formats the
        reference's message from the registers of the failing point (probed on
        the device, PointProgram.raise_for)."""
        key = (type(exc), str(exc), None if fmt is None else tuple(
            ("r", x.id) if isinstance(x, Reg) else x for x in fmt))
        sid = self._site_keys.get(key)
        if sid is None:
            sid = len(self.sites)
            self.sites.append(exc)
            if fmt is not None:
                self.site_fmts[sid] = key[2]
            self._site_keys[key] = sid
        return sid

    # -- serialisation ---------------------------------------------------------

    @staticmethod
    def width_of(lo: int, hi: int) -> int:
        if INT32[0] <= lo and hi <= INT32[1]:
            return 0
        if INT64[0] <= lo and hi <= INT64[1]:
            return 1
        if INT128[0] <= lo and hi <= INT128[1]:
            return 2
        raise LoweringError(
            f"intermediate value range [{lo}, {hi}] exceeds 128-bit integers")

    def widths(self) -> list[int]:
        return [self.width_of(lo, hi) for lo, hi in self.regs]

    def flat(self) -> list[tuple]:
        """Insns as (op, dst, a, b, c, site, lo, hi) with IF/ELSE/ENDIF markers."""
        out = list(self.const_insns)

        def walk(items):
            for it in items:
                if it[0] == "if":
                    _, cond, then, other = it
                    out.append((OP_IF, -1, cond, -1, -1, -1, 0, 0))
                    walk(then)
                    if other:
                        out.append((OP_ELSE, -1, -1, -1, -1, -1, 0, 0))
                        walk(other)
                    out.append((OP_ENDIF, -1, -1, -1, -1, -1, 0, 0))
                else:
                    out.append(it)

        walk(self.body)
        return out

    def dump(self) -> str:
        ws = self.widths()
        lines, ind = [], 0
        for op, d, a, b, c, s, lo, hi in self.flat():
            if op in (OP_ELSE, OP_ENDIF):
                ind -= 1
            args = [f"r{x}" for x in (a, b, c) if x >= 0]
            extra = f" site={s}" if s >= 0 else ""
            if op in (OP_CONST, OP_CHECK, OP_COORD):
                extra += f" imm=({lo},{hi})"
            dst = f"r{d}:i{32 << ws[d]} = " if d >= 0 else ""
            lines.append("  " * ind + f"{dst}{OP_NAMES[op]} {', '.join(args)}{extra}")
            if op in (OP_IF, OP_ELSE):
                ind += 1
        return "\n".join(lines)


class Lowerer:
    """Evaluator over concrete and symbolic values.

    With `program=None` it is a plain concrete evaluator (used for globals,
    which the reference evaluates eagerly when the mapper is compiled,
    interp.py:50-56): errors raise immediately.  With a `Program`, errors
    become FAIL sites and the current control path is abandoned.
    """

    def __init__(self, program: A.MapperProgram, machine, globals_env=None):
        self.mapper = program
        self.machine = machine
        self.functions = program.functions
        self.prog: Program | None = None
        self.block: list | None = None
        self.globals: dict = {}
        if globals_env is None:
            for g in program.globals:
                self.globals[g.name] = self.eval(g.expr, {}, 0)
        else:
            self.globals = dict(globals_env)

    # -- emission helpers ----------------------------------------------------------

    def fail(self, exc: Exception, fmt: tuple | None = None):
        if self.prog is None:
            raise exc
        self._emit((OP_FAIL, -1, -1, -1, -1, self.prog.site(exc, fmt), 0, 0))
        raise _Dead()

    def _emit(self, insn):
        self.prog.n_insns += 1
        if self.prog.n_insns > MAX_INSNS:
            raise LoweringError("mapper too large to lower (instruction budget exceeded)")
        self.block.append(insn)

    def const(self, v: int) -> Reg:
        r = self.prog.consts.get(v)
        if r is None:
            r = self.prog.new_reg(v, v)
            self.prog.consts[v] = r
            Program.width_of(v, v)
            mask = (1 << 64) - 1
            lo64 = v & mask
            hi64 = (v >> 64) & mask
            if lo64 >= 1 << 63:
                lo64 -= 1 << 64
            if hi64 >= 1 << 63:
                hi64 -= 1 << 64
            self.prog.const_insns.append((OP_CONST, r.id, -1, -1, -1, -1, lo64, hi64))
        return r

    def as_reg(self, v) -> Reg:
        return v if isinstance(v, Reg) else self.const(v)

    def _op(self, op, rng, a=-1, b=-1, c=-1, site=-1, lo=0, hi=0) -> Reg:
        Program.width_of(*rng)
        r = self.prog.new_reg(*rng)
        self._emit((op, r.id, a, b, c, site, lo, hi))
        return r

    def branch(self, cond: Reg, then_fn, else_fn):
        """Evaluate both arms lazily under `cond`; merge or wrap the results."""
        outer = self.block
        t_blk, e_blk = [], []
        self.block = t_blk
        try:
            a = then_fn()
        except _Dead:
            a = BOTTOM
        self.block = e_blk
        try:
            b = else_fn()
        except _Dead:
            b = BOTTOM
        self.block = outer
        merged = self._merge(cond, a, b, t_blk, e_blk)
        self._emit(("if", cond.id, t_blk, e_blk))
        if merged is BOTTOM:
            raise _Dead()
        return merged

    def _merge(self, cond, a, b, t_blk, e_blk):
        if a is BOTTOM:
            return b
        if b is BOTTOM:
            return a
        if _is_int(a) and _is_int(b):
            if isinstance(a, int) and isinstance(b, int) and a == b:
                return a
            lo = min(a.lo if isinstance(a, Reg) else a, b.lo if isinstance(b, Reg) else b)
            hi = max(a.hi if isinstance(a, Reg) else a, b.hi if isinstance(b, Reg) else b)
            Program.width_of(lo, hi)
            phi = self.prog.new_reg(lo, hi)
            t_blk.append((OP_MOV, phi.id, self.as_reg(a).id, -1, -1, -1, 0, 0))
            e_blk.append((OP_MOV, phi.id, self.as_reg(b).id, -1, -1, -1, 0, 0))
            return phi
        procs = (ProcRef, DynProc)
        if isinstance(a, procs) and isinstance(b, procs):
            r = self._merge(cond, self._pid(a), self._pid(b), t_blk, e_blk)
            return DynProc(self.as_reg(r)) if isinstance(r, Reg) else self._ref(r)
        if isinstance(a, tuple) and isinstance(b, tuple) and len(a) == len(b):
            return tuple(self._merge(cond, x, y, t_blk, e_blk) for x, y in zip(a, b))
        if isinstance(a, ProcSpace) and isinstance(b, ProcSpace) and a == b:
            return a
        return Choice(cond, a, b)

    def _pid(self, p):
        if isinstance(p, DynProc):
            return p.reg
        return p.node * self.machine.procs_per_node + p.proc

    def _ref(self, pid: int) -> ProcRef:
        return ProcRef(*divmod(pid, self.machine.procs_per_node))

    def split_on(self, v, k):
        """Apply continuation k to every non-Choice alternative of v."""
        if isinstance(v, Choice):
            return self.branch(v.cond, lambda: self.split_on(v.a, k),
                               lambda: self.split_on(v.b, k))
        return k(v)

    def collect(self, n, produce, k, acc=()):
        """Evaluate produce(0..n-1) in order, forking on each Choice, then k(values)."""
        if len(acc) == n:
            return k(acc)
        return self.split_on(produce(len(acc)),
                             lambda x: self.collect(n, produce, k, acc + (x,)))

    def concrete(self, v, k, clamp=None):
        """Run k with v as a concrete int, enumerating a register's values.

        With `clamp=(lo, hi)`, values below lo behave like lo and above hi like
        hi (Python slice-bound semantics), which bounds the fan-out.
        """
        if isinstance(v, int):
            return k(v)
        lo, hi = v.lo, v.hi
        if clamp is not None:
            lo, hi = max(lo, clamp[0]), min(hi, clamp[1])
            lo, hi = min(lo, clamp[1]), max(hi, clamp[0])
        if hi - lo + 1 > MAX_FANOUT:
            raise LoweringError(
                f"a point-dependent value in [{v.lo}, {v.hi}] selects a processor "
                "space or shape; too many cases to enumerate")
        vals = list(range(lo, hi + 1))

        def rec(i):
            x = vals[i]
            if i == len(vals) - 1:
                return k(x)
            if clamp is not None and x == clamp[0]:
                cond = self.compare("<", v, x + 1)
            else:
                cond = self.compare("==", v, x)
            if isinstance(cond, int):
                return k(x) if cond else rec(i + 1)
            return self.branch(cond, lambda: k(x), lambda: rec(i + 1))

        return rec(0)

    # -- integer arithmetic (reference: dsl/interp.py:268-309) ----------------------

    def compare(self, op, x, y):
        if isinstance(x, int) and isinstance(y, int):
            return int(x > y) if op == ">" else int(x < y) if op == "<" else int(x == y)
        xl, xh = (x.lo, x.hi) if isinstance(x, Reg) else (x, x)
        yl, yh = (y.lo, y.hi) if isinstance(y, Reg) else (y, y)
        if op == ">":
            if xl > yh:
                return 1
            if xh <= yl:
                return 0
        elif op == "<":
            if xh < yl:
                return 1
            if xl >= yh:
                return 0
        else:
            if xl == xh == yl == yh:
                return 1
            if xh < yl or yh < xl:
                return 0
        code = {">": OP_GT, "<": OP_LT, "==": OP_EQ}[op]
        return self._op(code, (0, 1), self.as_reg(x).id, self.as_reg(y).id)

    def scalar(self, op, x, y):
        if op in (">", "<", "=="):
            return self.compare(op, x, y)
        if isinstance(x, int) and isinstance(y, int):
            if op == "+":
                return x + y
            if op == "-":
                return x - y
            if op == "*":
                return x * y
            if y == 0:
                self.fail(EvalError("division by zero" if op == "/" else "modulo by zero"))
            return x // y if op == "/" else x % y
        if op == "*" and (x == 0 or y == 0):
            return 0
        if op in ("+", "-") and y == 0:
            return x
        if op == "+" and x == 0:
            return y
        if op in ("*", "/") and y == 1:
            return x
        if op == "*" and x == 1:
            return y
        xr = (x.lo, x.hi) if isinstance(x, Reg) else (x, x)
        yr = (y.lo, y.hi) if isinstance(y, Reg) else (y, y)
        site, fast = -1, 0
        if op in ("/", "%"):
            if yr == (0, 0):
                self.fail(EvalError("division by zero" if op == "/" else "modulo by zero"))
            if yr[0] <= 0 <= yr[1]:
                site = self.prog.site(
                    EvalError("division by zero" if op == "/" else "modulo by zero"))
            fast = int(xr[0] >= 0 and yr[0] > 0)
        rng = _range_of(op, xr, yr)
        code = {"+": OP_ADD, "-": OP_SUB, "*": OP_MUL, "/": OP_DIV, "%": OP_MOD}[op]
        return self._op(code, rng, self.as_reg(x).id, self.as_reg(y).id, fast, site)

    def binop(self, op, a, b):
        if isinstance(a, tuple) or isinstance(b, tuple):
            if isinstance(a, tuple) and isinstance(b, tuple):
                if len(a) != len(b):
                    self.fail(EvalError(f"rank mismatch: {len(a)} vs {len(b)}"))
                pairs = list(zip(a, b))
            elif isinstance(a, tuple):
                if not _is_int(b):
                    self.fail(EvalError(f"cannot combine Tuple with {type_name(b)}"))
                pairs = [(x, b) for x in a]
            else:
                if not _is_int(a):
                    self.fail(EvalError(f"cannot combine {type_name(a)} with Tuple"))
                pairs = [(a, y) for y in b]
            return tuple(self.scalar(op, x, y) for x, y in pairs)
        if _is_int(a) and _is_int(b):
            return self.scalar(op, a, b)
        self.fail(EvalError(
            f"operator {op!r} undefined on {type_name(a)} and {type_name(b)}"))

    def require_int(self, v, what):
        if not _is_int(v):
            self.fail(EvalError(f"{what} is {type_name(v)}, expected Int"))
        return v

    # -- expressions (reference: dsl/interp.py:100-259) ------------------------------

    def eval(self, e, env: dict, depth: int):
        t = type(e)
        if t is A.Var:
            if e.name in env:
                return env[e.name]
            if e.name in self.globals:
                return self.globals[e.name]
            self.fail(EvalError(f"undefined variable {e.name!r}"))
        if t is A.IntLit:
            return e.value
        if t is A.BinOp:
            lhs = self.eval(e.lhs, env, depth)
            rhs = self.eval(e.rhs, env, depth)
            return self.split_on(lhs, lambda a: self.split_on(
                rhs, lambda b: self.binop(e.op, a, b)))
        if t is A.Index:
            obj = self.eval(e.obj, env, depth)
            return self.split_on(obj, lambda o: self._index(e, o, env, depth))
        if t is A.Member:
            obj = self.eval(e.obj, env, depth)
            return self.split_on(obj, lambda o: self._member(e, o))
        if t is A.MethodCall:
            obj = self.eval(e.obj, env, depth)
            return self.split_on(obj, lambda o: self._primitive(e, o, env, depth))
        if t is A.MachineExpr:
            if e.kind != self.machine.kind:
                self.fail(EvalError(
                    f"machine provides {self.machine.kind}, mapper asks for {e.kind}"))
            return ProcSpace.of(self.machine)
        if t is A.Call:
            fn = self.functions.get(e.name)
            if fn is None:
                self.fail(EvalError(f"call to undefined function {e.name!r}"))
            args = [self.eval(a, env, depth) for a in e.args]
            return self.call(fn, args, depth + 1)
        if t is A.Ternary:
            c = self.eval(e.cond, env, depth)
            return self.split_on(c, lambda cv: self._ternary(e, cv, env, depth))
        if t is A.TupleComprehension:
            def item(i):
                inner = dict(env)
                inner[e.var] = e.values[i]
                return self.eval(e.body, inner, depth)
            return self.collect(len(e.values), item, lambda xs: self._int_tuple(
                xs, "comprehension element"))
        if t is A.TupleLit:
            return self.collect(len(e.items), lambda i: self.eval(e.items[i], env, depth),
                                lambda xs: self._int_tuple(xs, "tuple element"))
        self.fail(EvalError(f"cannot evaluate {t.__name__}"))

    def _int_tuple(self, xs, what):
        # the reference checks each element right after evaluating it; collect()
        # forks per element, so checking here in order is equivalent
        for x in xs:
            if not _is_int(x):
                self.fail(EvalError(f"{what} is {type_name(x)}, expected Int"))
        return tuple(xs)

    def _ternary(self, e, c, env, depth):
        if not _is_int(c):
            self.fail(EvalError(f"ternary condition is {type_name(c)}, expected Int"))
        if isinstance(c, Reg):
            if c.lo > 0 or c.hi < 0:
                c = 1
            elif c.lo == c.hi == 0:
                c = 0
        if isinstance(c, int):
            return self.eval(e.then if c != 0 else e.other, env, depth)
        return self.branch(c, lambda: self.eval(e.then, env, depth),
                           lambda: self.eval(e.other, env, depth))

    def _member(self, e, obj):
        if e.name == "size" and isinstance(obj, ProcSpace):
            return obj.shape
        self.fail(EvalError(f"no member {e.name!r} on {type_name(obj)}"))

    def _primitive(self, e, obj, env, depth):
        if not isinstance(obj, ProcSpace):
            self.fail(EvalError(
                f"transformation {e.name!r} applies to a Space, got {type_name(obj)}"))
        args = [self.eval(a, env, depth) for a in e.args]
        arity = {"split": 2, "merge": 2, "swap": 2, "reorder": 2, "slice": 3, "decompose": 2}
        if e.name not in arity:
            self.fail(EvalError(f"unknown primitive {e.name!r}"))
        if len(args) != arity[e.name]:
            self.fail(EvalError(f"primitive {e.name!r} takes {arity[e.name]} arguments"))
        return self.collect(len(args), lambda i: args[i],
                            lambda vals: self._apply_primitive(e.name, obj, vals))

    def _host_call(self, fn, *args):
        """Run a host-side space/optimizer call, turning its errors into sites.

        ProcMapErrors other than EvalError are re-wrapped as EvalError like the
        reference (interp.py:192-195); other exceptions pass through as is.
        """
        try:
            return fn(*args)
        except _Dead:
            raise
        except EvalError as exc:
            self.fail(exc)
        except ProcMapError as exc:
            self.fail(EvalError(f"{self._prim_name}: {exc}"))
        except Exception as exc:  # noqa: BLE001 - the reference propagates these
            self.fail(exc)

    def _apply_primitive(self, name, obj, vals):
        self._prim_name = name
        if name == "decompose":
            dim = self.require_int(vals[0], "decompose dimension")
            ext = vals[1]
            if not isinstance(ext, tuple):
                self.fail(EvalError(f"decompose extents must be a Tuple, got {type_name(ext)}"))

            def with_dim(d):
                if not 0 <= d < obj.rank:
                    self.fail(EvalError(f"dimension {d} out of range for rank {obj.rank}"))

                def with_ext(ex):
                    self._prim_name = name
                    factors, _ = self._host_call(search_optimal, obj.shape[d], ex)
                    return self._host_call(obj.decompose, d, factors)

                return self._concrete_tuple(ext, with_ext)

            return self.concrete(dim, with_dim)
        ints = [self.require_int(v, f"argument of {name}") for v in vals]
        method = {"split": obj.split, "merge": obj.merge, "slice": obj.slice,
                  "swap": obj.swap, "reorder": obj.swap}[name]

        def go(i, acc):
            if i == len(ints):
                self._prim_name = name
                return self._host_call(method, *acc)
            return self.concrete(ints[i], lambda x: go(i + 1, acc + (x,)))

        return go(0, ())

    def _concrete_tuple(self, t, k, i=0, acc=()):
        if i == len(t):
            return k(acc)
        return self.concrete(t[i], lambda x: self._concrete_tuple(t, k, i + 1, acc + (x,)))

    def _index(self, e, obj, env, depth):
        if len(e.args) == 1 and isinstance(e.args[0], A.SliceArg):
            sl = e.args[0]
            lo = self._bound(sl.lo, env, depth)
            hi = self._bound(sl.hi, env, depth)
            seq = obj.shape if isinstance(obj, ProcSpace) else obj
            if not isinstance(seq, tuple):
                self.fail(EvalError(f"cannot slice {type_name(obj)}"))
            n = len(seq)

            def with_lo(a):
                if hi is None:
                    return seq[a:]
                return self.concrete(hi, lambda b: seq[a:b], clamp=(-n, n))

            if lo is None:
                return with_lo(None)
            return self.concrete(lo, with_lo, clamp=(-n, n))
        if isinstance(obj, tuple):
            if len(e.args) != 1:
                self.fail(EvalError("tuples take a single index"))
            i = self.eval(e.args[0], env, depth)
            return self.split_on(i, lambda iv: self._tuple_item(
                obj, self.require_int(iv, "tuple index")))
        if isinstance(obj, ProcSpace):
            return self._index_space(obj, e, env, depth)
        self.fail(EvalError(f"cannot index {type_name(obj)}"))

    def _bound(self, b, env, depth):
        if b is None:
            return None
        v = self.eval(b, env, depth)
        return self.split_on(v, lambda x: self.require_int(x, "slice bound"))

    def _tuple_item(self, tup, i):
        n = len(tup)
        if isinstance(i, int):
            if not -n <= i < n:
                self.fail(EvalError(f"index {i} out of range for tuple of rank {n}"))
            return tup[i]
        if i.lo < -n or i.hi >= n:
            site = self.prog.site(EvalError(f"index out of range for tuple of rank {n}"),
                                  ("index ", i, f" out of range for tuple of rank {n}"))
            self._emit((OP_CHECK, -1, i.id, -1, -1, site, -n, n))
            i = Reg(i.id, max(i.lo, -n), min(i.hi, n - 1))
        cands = list(range(i.lo, i.hi + 1))
        if all(_is_int(tup[j]) for j in cands):
            return self._select(i, [(j, tup[j]) for j in cands])
        return self.concrete(i, lambda j: tup[j])

    def _select(self, key: Reg, cases):
        """Select the value paired with key's value among int cases."""
        vals = [v for _, v in cases]
        if all(isinstance(v, int) for v in vals) and len(set(vals)) == 1:
            return vals[0]
        acc = cases[-1][1]
        for j, v in reversed(cases[:-1]):
            c = self.compare("==", key, j)
            if isinstance(c, int):
                if c:
                    acc = v
                continue
            lo = min(_lo(v), _lo(acc))
            hi = max(_hi(v), _hi(acc))
            acc = self._op(OP_SELECT, (lo, hi), c.id, self.as_reg(v).id, self.as_reg(acc).id)
        return acc

    def _index_space(self, space, e, env, depth):
        nargs = len(e.args)

        def step(i, coords, single):
            if i == nargs:
                return self._index_space_done(space, nargs, coords, single)
            a = e.args[i]
            if isinstance(a, A.Splat):
                v = self.eval(a.value, env, depth)

                def splat(x):
                    if not isinstance(x, tuple):
                        self.fail(EvalError(f"splat needs a Tuple, got {type_name(x)}"))
                    return step(i + 1, coords + list(x), single)
                return self.split_on(v, splat)
            if isinstance(a, A.SliceArg):
                self.fail(EvalError("slice cannot be combined with other index arguments"))
            v = self.eval(a, env, depth)

            def plain(x):
                s = x if nargs == 1 else single
                if isinstance(x, tuple):
                    if nargs != 1:
                        self.fail(EvalError("a Tuple index must be the only index argument"))
                    return step(i + 1, coords + list(x), s)
                return step(i + 1, coords + [self.require_int(x, "space index")], s)
            return self.split_on(v, plain)

        return step(0, [], None)

    def _index_space_done(self, space, nargs, coords, single):
        if nargs == 1 and _is_int(single) and space.rank > 1:
            # partial scalar index reads an extent (reference: interp.py:245-250)
            r = space.rank
            if isinstance(single, int):
                if not 0 <= single < r:
                    self.fail(EvalError(f"dimension {single} out of range for rank {r}"))
                return space.shape[single]
            if single.lo < 0 or single.hi >= r:
                site = self.prog.site(EvalError(f"dimension out of range for rank {r}"),
                                      ("dimension ", single, f" out of range for rank {r}"))
                self._emit((OP_CHECK, -1, single.id, -1, -1, site, 0, r))
                single = Reg(single.id, max(single.lo, 0), min(single.hi, r - 1))
            return self._select(single, [(j, space.shape[j])
                                         for j in range(single.lo, single.hi + 1)])
        if len(coords) != space.rank:
            self.fail(EvalError(
                f"space of rank {space.rank} indexed with {len(coords)} coordinates"))
        return self.resolve(space, coords)

    def resolve(self, space: ProcSpace, coords):
        """`space[coords]` -> ProcRef / DynProc (reference: spaces.py:185-213)."""
        if all(isinstance(c, int) for c in coords):
            try:
                node, proc = space.resolve(tuple(coords))
            except ProcMapError as exc:
                self.fail(EvalError(str(exc)))
            return ProcRef(node, proc)
        # the reference's message quotes the whole index tuple (spaces.py:215-221)
        msg = ["index ", *_tuple_pieces(coords), f" out of range for shape {space.shape}"]
        for c, s in zip(coords, space.shape):
            if isinstance(c, int) and not 0 <= c < s:
                self.fail(EvalError(f"index out of range for shape {space.shape}"), tuple(msg))
        site = None
        cur = []
        for c, s in zip(coords, space.shape):
            if isinstance(c, Reg) and (c.lo < 0 or c.hi >= s):
                if site is None:
                    site = self.prog.site(EvalError(
                        f"index out of range for shape {space.shape}"), tuple(msg))
                self._emit((OP_CHECK, -1, c.id, -1, -1, site, 0, s))
                c = Reg(c.id, max(c.lo, 0), min(c.hi, s - 1))
            cur.append(c)
        for link in reversed(space.chain):
            t, src = link.transform, link.source_shape
            if isinstance(t, Split):
                i = t.dim
                cur[i:i + 2] = [self.scalar("+", cur[i], self.scalar("*", cur[i + 1], t.factor))]
            elif isinstance(t, Merge):
                v = cur[t.p]
                lo, hi = self.scalar("%", v, src[t.p]), self.scalar("/", v, src[t.p])
                cur[t.p] = lo
                cur.insert(t.q, hi)
            elif isinstance(t, Swap):
                cur[t.p], cur[t.q] = cur[t.q], cur[t.p]
            elif isinstance(t, Slice):
                cur[t.dim] = self.scalar("+", cur[t.dim], t.low)
        node, proc = cur
        pid = self.scalar("+", self.scalar("*", node, self.machine.procs_per_node), proc)
        if isinstance(pid, int):
            return self._ref(pid)
        return DynProc(pid)

    # -- functions (reference: dsl/interp.py:60-96) ----------------------------------

    def call(self, fn: A.FuncDef, args, depth: int):
        if depth > MAX_CALL_DEPTH:
            self.fail(EvalError(f"call depth exceeded in {fn.name!r}"))
        if len(args) != len(fn.params):
            self.fail(EvalError(f"{fn.name!r} takes {len(fn.params)} arguments, got {len(args)}"))
        env = {p.name: a for p, a in zip(fn.params, args)}
        return self.body(fn.body, env, depth)

    def body(self, stmts, env, depth):
        for st in stmts:
            if isinstance(st, A.Assign):
                env[st.target] = self.eval(st.expr, env, depth)
            else:
                return self.eval(st.expr, env, depth)
        self.fail(EvalError("function body ended without a return"))

    def as_processor(self, result, func_name):
        def check(r):
            if not isinstance(r, (ProcRef, DynProc)):
                self.fail(EvalError(
                    f"mapping function {func_name!r} returned {type_name(r)}, "
                    "expected a processor reference"))
            return r
        return self.split_on(result, check)


def _lo(v):
    return v.lo if isinstance(v, Reg) else v


def _hi(v):
    return v.hi if isinstance(v, Reg) else v


# -- plan analysis (reference: dsl/interp.py:323-399) ------------------------------


def free_vars(e, bound=frozenset()) -> set:
    """Names an expression reads that are not bound inside it."""
    out: set = set()

    def go(x, b):
        if x is None:
            return
        t = type(x)
        if t is A.Var:
            if x.name not in b:
                out.add(x.name)
        elif t in (A.IntLit, A.MachineExpr):
            pass
        elif t is A.Call:
            for a in x.args:
                go(a, b)
        elif t is A.Member:
            go(x.obj, b)
        elif t is A.MethodCall:
            go(x.obj, b)
            for a in x.args:
                go(a, b)
        elif t is A.BinOp:
            go(x.lhs, b)
            go(x.rhs, b)
        elif t is A.Index:
            go(x.obj, b)
            for a in x.args:
                if isinstance(a, A.Splat):
                    go(a.value, b)
                elif isinstance(a, A.SliceArg):
                    go(a.lo, b)
                    go(a.hi, b)
                else:
                    go(a, b)
        elif t is A.Ternary:
            go(x.cond, b)
            go(x.then, b)
            go(x.other, b)
        elif t is A.TupleComprehension:
            go(x.body, b | {x.var})
        elif t is A.TupleLit:
            for i in x.items:
                go(i, b)
        else:
            raise TypeError(f"unhandled expression {x!r}")

    go(e, set(bound))
    return out


def split_plan(func: A.FuncDef):
    """(prefix, suffix, return expr) or None when the body has early returns.

    A statement joins the per-point suffix when it reads the point parameter
    or a name already tainted, or re-assigns a tainted name
    (reference: interp.py:380-399).
    """
    body = func.body
    if not body or not isinstance(body[-1], A.Return):
        return None
    if any(isinstance(s, A.Return) for s in body[:-1]):
        return None
    tainted = {func.params[0].name}
    prefix, suffix = [], []
    for st in body[:-1]:
        if free_vars(st.expr) & tainted or st.target in tainted:
            tainted.add(st.target)
            suffix.append(st)
        else:
            prefix.append(st)
    return prefix, suffix, body[-1].expr


# -- entry point -------------------------------------------------------------------


@dataclass
class Lowered:
    program: Program
    n_coords: int
    implicit: bool
    extents: tuple
    ppn: int
    constant: int | None      # proc id if the map is point-independent
    dead: bool                # every point fails at a static site


def lower_mapping(lowerer: Lowerer, func: A.FuncDef, ispace: tuple, *,
                  implicit: bool, n_coords: int, plan_mode: bool,
                  coord_range=INT32) -> Lowered:
    """Lower `func` for one iteration space.

    implicit: points are the row-major enumeration of `ispace` (cli.py:155-157),
              generated on the device from the linear index;
    otherwise: points are explicit int32 rows of length `n_coords`.
    plan_mode: follow MappingFunction.__call__ (prefix, then suffix) rather
               than eval_mapping's in-order evaluation.
    """
    prog = Program()
    lowerer.prog, lowerer.block = prog, prog.body
    old_limit = sys.getrecursionlimit()
    sys.setrecursionlimit(max(old_limit, 20000))
    try:
        coords = []
        for i in range(n_coords):
            lo, hi = (0, ispace[i] - 1) if implicit else coord_range
            r = prog.new_reg(lo, hi)
            prog.coords.append(r)
            coords.append(r)
        for i, r in enumerate(coords):
            lowerer._emit((OP_COORD, r.id, -1, -1, -1, -1, i, 0))
        point = tuple(coords)
        dead = False
        result = None
        try:
            plan = split_plan(func) if plan_mode else None
            if plan is None:
                if len(func.params) != 2:
                    lowerer.fail(EvalError(
                        f"mapping function {func.name!r} must take (ipoint, ispace)"))
                res = lowerer.call(func, [point, tuple(ispace)], 0)
            else:
                prefix, suffix, ret = plan
                env = {func.params[1].name: tuple(ispace)}
                for st in prefix:
                    env[st.target] = lowerer.eval(st.expr, env, 0)
                env = dict(env)
                env[func.params[0].name] = point
                for st in suffix:
                    env[st.target] = lowerer.eval(st.expr, env, 0)
                res = lowerer.eval(ret, env, 0)
            result = lowerer.as_processor(res, func.name)
        except _Dead:
            dead = True
        constant = None
        if not dead:
            pid = lowerer._pid(result)
            if isinstance(pid, int):
                constant = pid
            lowerer._emit((OP_RET, -1, lowerer.as_reg(pid).id, -1, -1, -1, 0, 0))
        prog.widths()  # validates every register range
        return Lowered(prog, n_coords, implicit, tuple(ispace),
                       lowerer.machine.procs_per_node, constant, dead)
    finally:
        sys.setrecursionlimit(old_limit)
        lowerer.prog, lowerer.block = None, None
