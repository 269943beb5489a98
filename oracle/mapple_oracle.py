"""ORACLE (test infrastructure only): CPU restatement of the Mapple hot path.

Restates, per point and in plain Python (unbounded ints, floor semantics),
the reference's mapping evaluation and its neighbours; every function cites
the reference (paths relative to /root/reference/pkg/src/procmap/):

* processor spaces and index resolution ........ spaces.py:116-221
* decompose optimizer / Algorithm-1 heuristic ... factorize.py:166-206
* boundary volume closed form + counting oracle . commvol.py:65-168
* DSL evaluation, prefix/suffix plan ............ dsl/interp.py:47-433
* index-launch driver + proc_counts ............. cli.py:149-170
* shard-policy ownership leaves ................. tasksim/sim.py:67-120

It consumes ASTs from the product parser (the parser is pinned separately
against the reference's own ASTs in tests/golden/parse_*.json); evaluation,
spaces and the optimizer are independent re-implementations.  Pinned against
the reference's outputs in tests/golden/ (tests/test_oracle_golden.py).
"""

from __future__ import annotations

import itertools
import math
from fractions import Fraction

from paper_2507_17087_b200.dsl import ast as A
from paper_2507_17087_b200.errors import (
    BadDimOrder,
    BadSliceBounds,
    DimOutOfRange,
    EvalError,
    IndexOutOfRange,
    NoBinding,
    NonDivisibleSplit,
    ProcMapError,
    ProductMismatch,
)

# ----------------------------------------------------------------------------
# processor spaces (spaces.py:95-221)
# ----------------------------------------------------------------------------


class OSpace:
    """Immutable space: base (kind, nodes, ppn), links, shape."""

    __slots__ = ("base", "links", "shape")

    def __init__(self, base, links, shape):
        self.base, self.links, self.shape = base, links, tuple(shape)

    def __eq__(self, other):
        return isinstance(other, OSpace) and (self.base, self.links, self.shape) == (
            other.base, other.links, other.shape)

    def __hash__(self):
        return hash((self.base, self.links, self.shape))

    @property
    def rank(self):
        return len(self.shape)

    def _dim(self, i):  # spaces.py:86-88
        if not 0 <= i < len(self.shape):
            raise DimOutOfRange(f"dimension {i} out of range")

    def _add(self, link, shape):
        return OSpace(self.base, self.links + ((link, self.shape),), shape)

    def split(self, i, d):  # spaces.py:116-125
        self._dim(i)
        if d < 1 or self.shape[i] % d:
            raise NonDivisibleSplit(f"bad split {d} of {self.shape[i]}")
        s = list(self.shape)
        s[i:i + 1] = [d, self.shape[i] // d]
        return self._add(("split", i, d), s)

    def merge(self, p, q):  # spaces.py:127-139
        self._dim(p)
        self._dim(q)
        if p >= q:
            raise BadDimOrder(f"merge({p},{q})")
        s = list(self.shape)
        s[p] = s[p] * s[q]
        del s[q]
        return self._add(("merge", p, q), s)

    def swap(self, p, q):  # spaces.py:141-147
        self._dim(p)
        self._dim(q)
        s = list(self.shape)
        s[p], s[q] = s[q], s[p]
        return self._add(("swap", p, q), s)

    def slice(self, i, lo, hi):  # spaces.py:149-157
        self._dim(i)
        if not (0 <= lo <= hi < self.shape[i]):
            raise BadSliceBounds(f"slice({lo},{hi})")
        s = list(self.shape)
        s[i] = hi - lo + 1
        return self._add(("slice", i, lo), s)

    def decompose(self, i, factors):  # spaces.py:159-177
        self._dim(i)
        factors = tuple(factors)
        if not factors or any(f < 1 for f in factors) or math.prod(factors) != self.shape[i]:
            raise ProductMismatch(f"decompose {factors} of {self.shape[i]}")
        sp = self
        for n, f in enumerate(factors[:-1]):
            sp = sp.split(i + n, f)
        return sp

    def resolve(self, idx):  # spaces.py:185-221
        c = list(idx)
        _in(c, self.shape)
        for link, src in reversed(self.links):
            kind = link[0]
            if kind == "split":
                _, i, d = link
                c = c[:i] + [c[i] + d * c[i + 1]] + c[i + 2:]
            elif kind == "merge":
                _, p, q = link
                v = c[p]
                c[p] = v % src[p]
                c.insert(q, v // src[p])
            elif kind == "swap":
                _, p, q = link
                c[p], c[q] = c[q], c[p]
            else:
                _, i, lo = link
                c[i] += lo
            _in(c, src)
        return c[0], c[1]


def _in(c, shape):
    if len(c) != len(shape) or not all(0 <= x < s for x, s in zip(c, shape)):
        raise IndexOutOfRange(f"index {tuple(c)} out of range for shape {tuple(shape)}")


def machine_space(kind, nodes, ppn):
    return OSpace((kind, nodes, ppn), (), (nodes, ppn))


# ----------------------------------------------------------------------------
# decompose optimizer (factorize.py:134-206), by brute force over divisors
# ----------------------------------------------------------------------------


def factorizations(d, k):
    if k < 1:
        raise ValueError("k >= 1")
    if d < 1:
        raise ValueError("d >= 1")
    divs = [x for x in range(1, d + 1) if d % x == 0]
    return sorted(t for t in itertools.product(divs, repeat=k) if math.prod(t) == d)


def search_optimal(d, extents):
    """Isotropic argmin of (sum d_m / l_m, factors) (factorize.py:166-188)."""
    extents = tuple(extents)
    best = min(factorizations(d, len(extents)),
               key=lambda f: (sum(Fraction(x, l) for x, l in zip(f, extents)), f))
    return best


def greedy_grid(d, k):  # factorize.py:191-206
    g = [1] * k
    n, p = d, 2
    primes = []
    while n > 1:
        while n % p == 0:
            primes.append(p)
            n //= p
        p += 1
    for p in primes:
        j = min(range(k), key=lambda i: (g[i], i))
        g[j] *= p
    return tuple(sorted(g, reverse=True))


# ----------------------------------------------------------------------------
# communication volume (commvol.py:65-168)
# ----------------------------------------------------------------------------


def surface_volume(extents, grid):  # commvol.py:90-96
    w = [Fraction(l, d) for l, d in zip(extents, grid)]
    sa = lambda x: 2 * math.prod(x) * sum(Fraction(1) / v for v in x)  # noqa: E731
    return sa(w) * math.prod(grid) - sa([Fraction(l) for l in extents])


def boundary_count(extents, grid, halo):
    """Per-cell enumeration like oracle_boundary_count (commvol.py:136-168)."""
    total = 0
    for n, (l, d) in enumerate(zip(extents, grid)):
        h = halo[n]
        if h == 0:
            continue
        cuts = [l * b // d for b in range(d + 1)]
        line = 0
        for b in range(1, d):
            line += sum(1 for x in range(cuts[b - 1], cuts[b]) if x >= cuts[b] - h)
            line += sum(1 for x in range(cuts[b], cuts[b + 1]) if x < cuts[b] + h)
        total += line * math.prod(e for m, e in enumerate(extents) if m != n)
    return total


def halo_entries(owner_of, extents, halo):
    """Per-(cell, dim, dir) transfer entries of a cell-owned grid (K3 contract).

    owner_of(cell_tuple) -> proc id.  Returns {(src, dst): [(lin, 2n+dir)]}
    with cells ascending -- the grouping pm_halo_lists produces.
    """
    out = {}
    strides = [math.prod(extents[m + 1:]) for m in range(len(extents))]
    for cell in itertools.product(*map(range, extents)):
        o = owner_of(cell)
        lin = sum(c * s for c, s in zip(cell, strides))
        for n in range(len(extents)):
            for sgn, dd in ((-1, 2 * n), (1, 2 * n + 1)):
                for j in range(1, halo[n] + 1):
                    y = cell[n] + sgn * j
                    if not 0 <= y < extents[n]:
                        break
                    nb = cell[:n] + (y,) + cell[n + 1:]
                    q = owner_of(nb)
                    if q != o:
                        out.setdefault((o, q), []).append((lin, dd))
                        break
    return out


# ----------------------------------------------------------------------------
# DSL evaluation (dsl/interp.py:47-309)
# ----------------------------------------------------------------------------


class ORef(tuple):
    """A resolved processor (node, proc)."""


def _tn(v):
    if isinstance(v, int):
        return "Int"
    if isinstance(v, ORef):
        return "ProcessorRef"
    if isinstance(v, tuple):
        return "Tuple"
    if isinstance(v, OSpace):
        return "Space"
    return type(v).__name__


def _int(v, what):
    if not isinstance(v, int):
        raise EvalError(f"{what} is {_tn(v)}, expected Int")
    return v


def _arith(op, a, b):  # interp.py:288-309
    if op == "+":
        return a + b
    if op == "-":
        return a - b
    if op == "*":
        return a * b
    if op in "/%":
        if b == 0:
            raise EvalError("division by zero")
        return a // b if op == "/" else a % b
    return int(a > b) if op == ">" else int(a < b) if op == "<" else int(a == b)


def _binop(op, a, b):  # interp.py:268-285
    ta, tb = isinstance(a, tuple) and not isinstance(a, ORef), \
        isinstance(b, tuple) and not isinstance(b, ORef)
    if ta and tb:
        if len(a) != len(b):
            raise EvalError("rank mismatch")
        return tuple(_arith(op, x, y) for x, y in zip(a, b))
    if ta:
        if not isinstance(b, int):
            raise EvalError("cannot combine")
        return tuple(_arith(op, x, b) for x in a)
    if tb:
        if not isinstance(a, int):
            raise EvalError("cannot combine")
        return tuple(_arith(op, a, y) for y in b)
    if isinstance(a, int) and isinstance(b, int):
        return _arith(op, a, b)
    raise EvalError(f"operator {op} undefined")


class OracleEval:
    """Tree-walking evaluator with the reference's semantics (interp.py:47-259)."""

    def __init__(self, program, machine):
        self.prog = program
        self.kind, self.nodes, self.ppn = machine
        self.funcs = {f.name: f for f in program.items if isinstance(f, A.FuncDef)}
        self.glob = {}
        for g in program.items:
            if isinstance(g, A.GlobalBinding):
                self.glob[g.name] = self.ev(g.expr, {}, 0)

    def call(self, fn, args, depth):  # interp.py:80-96
        if depth > 64:
            raise EvalError("call depth exceeded")
        if len(args) != len(fn.params):
            raise EvalError("arity")
        env = {p.name: a for p, a in zip(fn.params, args)}
        for st in fn.body:
            if isinstance(st, A.Assign):
                env[st.target] = self.ev(st.expr, env, depth)
            else:
                return self.ev(st.expr, env, depth)
        raise EvalError("function body ended without a return")

    def ev(self, e, env, depth):  # interp.py:100-160
        t = type(e)
        if t is A.Var:
            if e.name in env:
                return env[e.name]
            if e.name in self.glob:
                return self.glob[e.name]
            raise EvalError(f"undefined variable {e.name}")
        if t is A.IntLit:
            return e.value
        if t is A.BinOp:
            return _binop(e.op, self.ev(e.lhs, env, depth), self.ev(e.rhs, env, depth))
        if t is A.Index:
            return self.index(e, env, depth)
        if t is A.Member:
            o = self.ev(e.obj, env, depth)
            if e.name == "size" and isinstance(o, OSpace):
                return o.shape
            raise EvalError("no member")
        if t is A.MethodCall:
            return self.prim(e, env, depth)
        if t is A.MachineExpr:
            if e.kind != self.kind:
                raise EvalError("machine kind mismatch")
            return machine_space(self.kind, self.nodes, self.ppn)
        if t is A.Call:
            fn = self.funcs.get(e.name)
            if fn is None:
                raise EvalError("undefined function")
            return self.call(fn, [self.ev(a, env, depth) for a in e.args], depth + 1)
        if t is A.Ternary:
            c = self.ev(e.cond, env, depth)
            if not isinstance(c, int) or isinstance(c, ORef):
                raise EvalError("ternary condition")
            return self.ev(e.then if c != 0 else e.other, env, depth)
        if t is A.TupleComprehension:
            out = []
            for v in e.values:
                inner = dict(env)
                inner[e.var] = v
                x = self.ev(e.body, inner, depth)
                out.append(_int(x, "comprehension element"))
            return tuple(out)
        if t is A.TupleLit:
            return tuple(_int(self.ev(x, env, depth), "tuple element") for x in e.items)
        raise EvalError(f"cannot evaluate {t.__name__}")

    def prim(self, e, env, depth):  # interp.py:162-195
        o = self.ev(e.obj, env, depth)
        if not isinstance(o, OSpace):
            raise EvalError("transformation applies to a Space")
        args = [self.ev(a, env, depth) for a in e.args]
        ar = {"split": 2, "merge": 2, "swap": 2, "reorder": 2, "slice": 3, "decompose": 2}
        if e.name not in ar or len(args) != ar[e.name]:
            raise EvalError("bad primitive")
        try:
            if e.name == "decompose":
                dim = _int(args[0], "decompose dimension")
                if not isinstance(args[1], tuple) or isinstance(args[1], ORef):
                    raise EvalError("decompose extents must be a Tuple")
                if not 0 <= dim < o.rank:
                    raise EvalError("dimension out of range")
                return o.decompose(dim, search_optimal(o.shape[dim], args[1]))
            ints = [_int(a, "argument") for a in args]
            name = "swap" if e.name == "reorder" else e.name
            return getattr(o, name)(*ints)
        except EvalError:
            raise
        except ProcMapError as exc:
            raise EvalError(str(exc)) from exc

    def index(self, e, env, depth):  # interp.py:197-259
        o = self.ev(e.obj, env, depth)
        if len(e.args) == 1 and isinstance(e.args[0], A.SliceArg):
            sl = e.args[0]
            lo = None if sl.lo is None else _int(self.ev(sl.lo, env, depth), "slice bound")
            hi = None if sl.hi is None else _int(self.ev(sl.hi, env, depth), "slice bound")
            seq = o.shape if isinstance(o, OSpace) else o
            if not isinstance(seq, tuple) or isinstance(seq, ORef):
                raise EvalError("cannot slice")
            return tuple(seq[lo:hi])
        if isinstance(o, tuple) and not isinstance(o, ORef):
            if len(e.args) != 1:
                raise EvalError("tuples take a single index")
            i = _int(self.ev(e.args[0], env, depth), "tuple index")
            if not -len(o) <= i < len(o):
                raise EvalError("tuple index out of range")
            return o[i]
        if not isinstance(o, OSpace):
            raise EvalError("cannot index")
        coords, single = [], None
        for a in e.args:
            if isinstance(a, A.Splat):
                v = self.ev(a.value, env, depth)
                if not isinstance(v, tuple) or isinstance(v, ORef):
                    raise EvalError("splat needs a Tuple")
                coords.extend(v)
            elif isinstance(a, A.SliceArg):
                raise EvalError("slice cannot be combined")
            else:
                v = self.ev(a, env, depth)
                if len(e.args) == 1:
                    single = v
                if isinstance(v, tuple) and not isinstance(v, ORef):
                    if len(e.args) != 1:
                        raise EvalError("a Tuple index must be the only index argument")
                    coords.extend(v)
                else:
                    coords.append(_int(v, "space index"))
        if len(e.args) == 1 and isinstance(single, int) and o.rank > 1:
            if not 0 <= single < o.rank:
                raise EvalError("dimension out of range")
            return o.shape[single]
        if len(coords) != o.rank:
            raise EvalError("space rank mismatch")
        try:
            return ORef(o.resolve(coords))
        except ProcMapError as exc:
            raise EvalError(str(exc)) from exc


def _free(e, bound=frozenset()):
    """Free variable names of an expression (interp.py:323-363)."""
    out = set()
    stack = [(e, frozenset(bound))]
    while stack:
        x, b = stack.pop()
        if x is None:
            continue
        t = type(x)
        if t is A.Var:
            if x.name not in b:
                out.add(x.name)
        elif t is A.TupleComprehension:
            stack.append((x.body, b | {x.var}))
        elif t in (A.Splat,):
            stack.append((x.value, b))
        elif t is A.SliceArg:
            stack += [(x.lo, b), (x.hi, b)]
        elif t in (A.IntLit, A.MachineExpr):
            pass
        else:
            for f in ("obj", "lhs", "rhs", "cond", "then", "other"):
                if hasattr(x, f):
                    stack.append((getattr(x, f), b))
            for f in ("args", "items"):
                if hasattr(x, f):
                    stack += [(y, b) for y in getattr(x, f)]
    return out


class OracleMapper:
    """compile_mapper + MappingFunction.__call__ semantics (interp.py:366-433)."""

    def __init__(self, program, task, machine):
        binds = {i.task: i.func for i in program.items if isinstance(i, A.IndexTaskMap)}
        if task not in binds:
            raise NoBinding(task)
        self.ev = OracleEval(program, machine)
        self.fn = self.ev.funcs.get(binds[task])
        if self.fn is None or len(self.fn.params) != 2:
            raise EvalError("bad mapping function")
        self.ppn = machine[2]
        body = self.fn.body
        self.plan = None
        if isinstance(body[-1], A.Return) and not any(isinstance(s, A.Return) for s in body[:-1]):
            taint = {self.fn.params[0].name}
            pre, suf = [], []
            for s in body[:-1]:
                if _free(s.expr) & taint or s.target in taint:
                    taint.add(s.target)
                    suf.append(s)
                else:
                    pre.append(s)
            self.plan = (pre, suf, body[-1].expr)
        self.cache = {}

    def __call__(self, pt, ispace):
        pt, ispace = tuple(pt), tuple(ispace)
        if self.plan is None:
            r = self.ev.call(self.fn, [pt, ispace], 0)
        else:
            pre, suf, ret = self.plan
            base = self.cache.get(ispace)
            if base is None:
                base = {self.fn.params[1].name: ispace}
                for s in pre:
                    base[s.target] = self.ev.ev(s.expr, base, 0)
                self.cache[ispace] = base
            env = dict(base)
            env[self.fn.params[0].name] = pt
            for s in suf:
                env[s.target] = self.ev.ev(s.expr, env, 0)
            r = self.ev.ev(ret, env, 0)
        if not isinstance(r, ORef):
            raise EvalError("mapping function must return a processor")
        return r

    def proc_id(self, pt, ispace):
        n, p = self(pt, ispace)
        return n * self.ppn + p


def eval_point(program, func, pt, ispace, machine):
    """eval_mapping (interp.py:312-320): fresh evaluator, in-order body."""
    ev = OracleEval(program, machine)
    fn = ev.funcs.get(func)
    if fn is None or len(fn.params) != 2:
        raise EvalError("bad mapping function")
    r = ev.call(fn, [tuple(pt), tuple(ispace)], 0)
    if not isinstance(r, ORef):
        raise EvalError("mapping function must return a processor")
    return tuple(r)


def row_major(ispace):
    """Launch points, last dimension fastest (cli.py:155-157)."""
    pts = [()]
    for e in ispace:
        pts = [p + (i,) for p in pts for i in range(e)]
    return pts


def map_launch(program, task, machine, ispace, first=0, count=None):
    """cmd_map's loop (cli.py:149-161): proc ids of row-major points."""
    fn = OracleMapper(program, task, machine)
    pts = row_major(ispace)
    if count is None:
        count = len(pts) - first
    return [fn.proc_id(p, ispace) for p in pts[first:first + count]]


def proc_counts(ids, ppn):
    """cli.py:162-164: sorted (node, proc) -> count."""
    c = {}
    for i in ids:
        c[divmod(i, ppn)] = c.get(divmod(i, ppn), 0) + 1
    return dict(sorted(c.items()))


def shard_leaves(task_id, points, targets):
    """expand_shards fixpoint (tasksim/sim.py:67-120): leaf id -> (target, points).

    The smallest target splits off as `/0`, the rest recurse as `/1`; point
    order inside every leaf is the launch order.
    """
    leaves = {}
    pending = [(task_id, list(zip(points, targets)))]
    while pending:
        tid, items = pending.pop()
        distinct = sorted({t for _, t in items})
        if len(distinct) == 1:
            leaves[tid] = (distinct[0], [p for p, _ in items])
            continue
        low = distinct[0]
        pending.append((tid + "/1", [(p, t) for p, t in items if t != low]))
        pending.append((tid + "/0", [(p, t) for p, t in items if t == low]))
    return dict(sorted(leaves.items()))
