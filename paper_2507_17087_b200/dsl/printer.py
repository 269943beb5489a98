"""Source printer for the Mapple AST.

Round-trip contract of the reference printer (reference: dsl/ast.py:227-311):
`parse(to_source(p)) == p`.  Parentheses are inserted from binding strength:
ternary < comparison < additive < multiplicative < postfix; a ternary or
comparison inside `[...]` is parenthesised because `:` separates slice
bounds there.
"""

from __future__ import annotations

from . import ast as A

# binding strength of each operator class
_STRENGTH = {"?": 1, ">": 2, "<": 2, "==": 2, "+": 3, "-": 3, "*": 4, "/": 4, "%": 4}
_POSTFIX = 5


def _wrap(text: str, mine: int, ctx: int) -> str:
    return f"({text})" if mine < ctx else text


def expr(e, ctx: int = 0) -> str:
    t = type(e)
    if t is A.IntLit:
        return str(e.value)
    if t is A.Var:
        return e.name
    if t is A.MachineExpr:
        return f"Machine({e.kind})"
    if t is A.Call:
        return f"{e.name}({', '.join(expr(a) for a in e.args)})"
    if t is A.Member:
        return f"{expr(e.obj, _POSTFIX)}.{e.name}"
    if t is A.MethodCall:
        return f"{expr(e.obj, _POSTFIX)}.{e.name}({', '.join(expr(a) for a in e.args)})"
    if t is A.BinOp:
        s = _STRENGTH[e.op]
        return _wrap(f"{expr(e.lhs, s)} {e.op} {expr(e.rhs, s + 1)}", s, ctx)
    if t is A.Ternary:
        body = f"{expr(e.cond, 2)} ? {expr(e.then, 1)} : {expr(e.other, 1)}"
        return _wrap(body, 1, ctx)
    if t is A.Index:
        return f"{expr(e.obj, _POSTFIX)}[{', '.join(_index_arg(a) for a in e.args)}]"
    if t is A.TupleComprehension:
        vals = ", ".join(map(str, e.values))
        return f"tuple({expr(e.body)} for {e.var} in ({vals}))"
    if t is A.TupleLit:
        if len(e.items) == 1:
            return f"({expr(e.items[0])},)"
        return "(" + ", ".join(expr(i) for i in e.items) + ")"
    raise TypeError(f"cannot print {e!r}")


def _index_arg(a) -> str:
    if isinstance(a, A.Splat):
        return "*" + expr(a.value, _POSTFIX)
    if isinstance(a, A.SliceArg):
        lo = "" if a.lo is None else expr(a.lo, 2)
        hi = "" if a.hi is None else expr(a.hi, 2)
        return f"{lo}:{hi}"
    return expr(a, 2)


def _constraint(c) -> str:
    return f"{c.name} == {c.value}" if isinstance(c, A.AlignConstraint) else c


def _item_lines(item):
    if isinstance(item, A.GlobalBinding):
        yield f"{item.name} = {expr(item.expr)}"
    elif isinstance(item, A.FuncDef):
        ps = ", ".join(f"{p.type_name} {p.name}" if p.type_name else p.name for p in item.params)
        yield f"def {item.name}({ps}):"
        for st in item.body:
            if isinstance(st, A.Assign):
                yield f"    {st.target} = {expr(st.expr)}"
            else:
                yield f"    return {expr(st.expr)}"
    elif isinstance(item, A.IndexTaskMap):
        yield f"IndexTaskMap {item.task} {item.func}"
    elif isinstance(item, A.TaskMap):
        yield " ".join(("Task", item.task) + tuple(item.procs))
    elif isinstance(item, A.DataMap):
        yield " ".join(("Region", item.task, item.region, item.proc) + tuple(item.memories))
    elif isinstance(item, A.DataLayout):
        cs = tuple(_constraint(c) for c in item.constraints)
        yield " ".join(("Layout", item.task, item.region, item.proc) + cs)
    elif isinstance(item, A.GarbageCollect):
        yield f"GarbageCollect {item.task} {item.arg}"
    elif isinstance(item, A.Backpressure):
        yield f"Backpressure {item.task} {item.depth}"
    else:
        raise TypeError(f"cannot print {item!r}")


def to_source(program: A.MapperProgram) -> str:
    lines = [ln for item in program.items for ln in _item_lines(item)]
    return "\n".join(lines) + "\n"
