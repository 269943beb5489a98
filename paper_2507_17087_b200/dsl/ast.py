"""Mapple AST.

Node classes, field names and field order are the reference's public AST
(reference: pkg/src/procmap/dsl/ast.py:13-223) so programs built by hand or
compared structurally stay interchangeable.  Source positions ride along as
keyword-only fields excluded from equality.  The printer lives in
`printer.py`; `to_source` is re-exported here for API parity.
"""

from __future__ import annotations

from dataclasses import dataclass, field


def _pos():
    return field(default=0, compare=False, kw_only=True)


@dataclass(frozen=True)
class Node:
    line: int = _pos()
    col: int = _pos()


# expressions ------------------------------------------------------------------

@dataclass(frozen=True)
class IntLit(Node):
    value: int


@dataclass(frozen=True)
class Var(Node):
    name: str


@dataclass(frozen=True)
class TupleLit(Node):
    items: tuple


@dataclass(frozen=True)
class TupleComprehension(Node):
    body: object
    var: str
    values: tuple


@dataclass(frozen=True)
class MachineExpr(Node):
    kind: str


@dataclass(frozen=True)
class Call(Node):
    name: str
    args: tuple


@dataclass(frozen=True)
class Member(Node):
    obj: object
    name: str


@dataclass(frozen=True)
class MethodCall(Node):
    obj: object
    name: str
    args: tuple


@dataclass(frozen=True)
class BinOp(Node):
    op: str
    lhs: object
    rhs: object


@dataclass(frozen=True)
class Ternary(Node):
    cond: object
    then: object
    other: object


@dataclass(frozen=True)
class Splat(Node):
    value: object


@dataclass(frozen=True)
class SliceArg(Node):
    lo: object
    hi: object


@dataclass(frozen=True)
class Index(Node):
    obj: object
    args: tuple


Expr = (
    Var | IntLit | Call | MachineExpr | Member | MethodCall | BinOp
    | Index | Ternary | TupleComprehension | TupleLit
)


# function bodies -----------------------------------------------------------------

@dataclass(frozen=True)
class Param(Node):
    type_name: str | None
    name: str


@dataclass(frozen=True)
class Assign(Node):
    target: str
    expr: object


@dataclass(frozen=True)
class Return(Node):
    expr: object


FuncStmt = Assign | Return


# top-level statements ---------------------------------------------------------------

@dataclass(frozen=True)
class FuncDef(Node):
    name: str
    params: tuple
    body: tuple


@dataclass(frozen=True)
class IndexTaskMap(Node):
    task: str
    func: str


@dataclass(frozen=True)
class TaskMap(Node):
    task: str
    procs: tuple


@dataclass(frozen=True)
class DataMap(Node):
    task: str
    region: str
    proc: str
    memories: tuple


@dataclass(frozen=True)
class AlignConstraint(Node):
    name: str
    value: int


Constraint = str | AlignConstraint


@dataclass(frozen=True)
class DataLayout(Node):
    task: str
    region: str
    proc: str
    constraints: tuple


@dataclass(frozen=True)
class GarbageCollect(Node):
    task: str
    arg: str


@dataclass(frozen=True)
class Backpressure(Node):
    task: str
    depth: int


Statement = (
    FuncDef | IndexTaskMap | TaskMap | DataMap | DataLayout | GarbageCollect | Backpressure
)


@dataclass(frozen=True)
class GlobalBinding(Node):
    name: str
    expr: object


TopLevel = Statement | GlobalBinding


@dataclass(frozen=True)
class MapperProgram:
    """Top-level items in source order (reference: dsl/ast.py:199-223)."""

    items: tuple

    @property
    def statements(self) -> tuple:
        return tuple(x for x in self.items if not isinstance(x, GlobalBinding))

    @property
    def globals(self) -> tuple:
        return tuple(x for x in self.items if isinstance(x, GlobalBinding))

    @property
    def functions(self) -> dict:
        return {x.name: x for x in self.items if isinstance(x, FuncDef)}

    def bindings(self) -> dict:
        """task -> mapping function name (IndexTaskMap statements)."""
        return {x.task: x.func for x in self.items if isinstance(x, IndexTaskMap)}


def to_source(program: MapperProgram) -> str:
    from .printer import to_source as _print

    return _print(program)
