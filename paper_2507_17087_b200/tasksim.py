"""Task-lifecycle simulator fed by batched ownership.

The reference's lifecycle simulator (tasksim/sim.py:174-514) runs the
operational semantics of the paper's Figs 10-11 -- ENQUEUE, DISTRIBUTE,
LOCAL, MAP, LAUNCH, EXECUTE -- over a task graph, and builds every task's
shard tree up front with `expand_shards` (sim.py:199-205), which re-maps the
task's points point by point at every level of the tree (O(points x
processors) mapping calls, sim.py:78).  Here the shard tree of a task comes
from ONE batched launch: the fused K1 + K2 kernels (`map_partition`) map the
task's points and stably partition them by processor, and the whole tree --
every decision, subtask and leaf -- is read off the per-processor lists
(leaf k of D distinct targets is task + "/1" * k + "/0", the last
task + "/1" * (D - 1); sim.py:83-120).  Any other `MappingFn` still works,
mapped point by point as in the reference.

The graph format, validation errors, rule set, schedulers (deterministic:
lowest rule, then smallest task id; random: `random.Random(seed)` over the
candidate pool), log entries, statistics and `Stuck` diagnoses follow the
reference, so a trace produced here is accepted by the reference's
`check_trace` (check.py:29-248) and equals the reference simulator's trace
for the same graph, mapping, scheduler and seed (tests/test_tasksim.py,
tests/test_gpu_tasksim.py).
"""

from __future__ import annotations

import heapq
import json
import random
from collections import deque
from dataclasses import dataclass, field
from typing import Callable

from .errors import CyclicDependence, EmptyTask, MultipleRoots, SchemaError, Stuck

MappingFn = Callable[[tuple, tuple], tuple]

ENQUEUED, MAPPED, LAUNCHED, EXECUTED = "enqueued", "mapped", "launched", "executed"
STAGES = (ENQUEUED, MAPPED, LAUNCHED, EXECUTED)


# -- graphs (reference: tasksim/graph.py) -----------------------------------------------


@dataclass(frozen=True)
class IndexTask:
    id: str
    points: tuple


@dataclass
class TaskGraph:
    tasks: dict
    root: str
    parent: dict
    children: dict            # parent id -> tuple of child ids in program order
    deps: frozenset           # (before, after)
    ispaces: dict
    deps_before: dict = field(default_factory=dict)
    deps_after: dict = field(default_factory=dict)
    sibling_deps_before: dict = field(default_factory=dict)

    def __post_init__(self):
        before = {t: [] for t in self.tasks}
        after = {t: [] for t in self.tasks}
        sib = {t: [] for t in self.tasks}
        for b, a in sorted(self.deps):
            before[a].append(b)
            after[b].append(a)
            pa = self.parent.get(a)
            if pa is not None and pa == self.parent.get(b):
                sib[a].append(b)
        self.deps_before = {t: tuple(v) for t, v in before.items()}
        self.deps_after = {t: tuple(v) for t, v in after.items()}
        self.sibling_deps_before = {t: tuple(v) for t, v in sib.items()}

    def earlier_siblings(self, tid: str) -> tuple:
        p = self.parent.get(tid)
        if p is None:
            return ()
        order = self.children[p]
        return order[:order.index(tid)]


def _parse_points(tid, item):
    raw = item["points"]
    if not isinstance(raw, list) or not raw:
        raise SchemaError(f"task {tid!r} has no points")
    pts = []
    for p in raw:
        if not isinstance(p, list) or any(not isinstance(c, int) or c < 0 for c in p):
            raise SchemaError(f"bad point {p!r} in task {tid!r}")
        pts.append(tuple(p))
    ranks = {len(p) for p in pts}
    if len(ranks) != 1:
        raise SchemaError(f"task {tid!r} mixes point ranks {ranks}")
    if len(set(pts)) != len(pts):
        raise SchemaError(f"task {tid!r} repeats points")
    if item.get("ispace") is not None:
        ispace = tuple(item["ispace"])
    else:
        ispace = tuple(max(p[d] for p in pts) + 1 for d in range(len(pts[0])))
    return tuple(pts), ispace


def _parse_ispace(tid, item):
    ext = item["ispace"]
    if not isinstance(ext, list) or not ext or any(not isinstance(e, int) or e < 1 for e in ext):
        raise SchemaError(f"task {tid!r} has bad ispace {ext!r}")
    pts = [()]
    for e in ext:
        pts = [p + (i,) for p in pts for i in range(e)]
    return tuple(pts), tuple(ext)


def _acyclic(edges, group, parent_id):
    """Kahn's algorithm over one sibling group's dependences."""
    indeg = {t: 0 for t in group}
    succs = {t: [] for t in group}
    for b, a in edges:
        succs[b].append(a)
        indeg[a] += 1
    ready = [t for t in group if not indeg[t]]
    n = 0
    while ready:
        t = ready.pop()
        n += 1
        for s in succs[t]:
            indeg[s] -= 1
            if not indeg[s]:
                ready.append(s)
    if n != len(group):
        raise CyclicDependence(f"dependences among children of {parent_id!r} form a cycle")


def load_taskgraph(document) -> TaskGraph:
    """Parse and validate a task-graph document (reference: tasksim/graph.py:73-191)."""
    if isinstance(document, (str, bytes)):
        try:
            document = json.loads(document)
        except json.JSONDecodeError as exc:
            raise SchemaError(f"not valid JSON: {exc}") from exc
    if not isinstance(document, dict):
        raise SchemaError("task graph document must be a JSON object")
    raw = document.get("tasks")
    if not isinstance(raw, list) or not raw:
        raise SchemaError("'tasks' must be a non-empty list")
    tasks, ispaces = {}, {}
    for item in raw:
        if not isinstance(item, dict) or not isinstance(item.get("id"), str):
            raise SchemaError(f"task entries need a string 'id': {item!r}")
        tid = item["id"]
        if not tid or "/" in tid:
            raise SchemaError(f"task id {tid!r} is empty or contains '/'")
        if tid in tasks:
            raise SchemaError(f"duplicate task id {tid!r}")
        if "points" in item:
            pts, ispaces[tid] = _parse_points(tid, item)
        elif "ispace" in item:
            pts, ispaces[tid] = _parse_ispace(tid, item)
        else:
            raise SchemaError(f"task {tid!r} needs 'points' or 'ispace'")
        tasks[tid] = IndexTask(tid, pts)

    parent = {}
    for edge in document.get("parent", []):
        p, c = edge.get("parent"), edge.get("child")
        if p not in tasks or c not in tasks:
            raise SchemaError(f"parent edge references unknown task: {edge!r}")
        if c in parent:
            raise SchemaError(f"task {c!r} has two parents")
        parent[c] = p
    roots = [t for t in tasks if t not in parent]
    if len(roots) > 1:
        raise MultipleRoots(f"multiple root tasks: {sorted(roots)}")
    if not roots:
        raise SchemaError("parent relation has a cycle (no root task)")
    for tid in tasks:
        seen, cur = {tid}, tid
        while cur in parent:
            cur = parent[cur]
            if cur in seen:
                raise SchemaError(f"parent relation has a cycle through {cur!r}")
            seen.add(cur)

    children = {t: [c for c in tasks if parent.get(c) == t] for t in tasks}
    spec = document.get("siblings", {})
    if not isinstance(spec, dict):
        raise SchemaError("'siblings' must map parent id to an ordered id list")
    for p, order in spec.items():
        if p not in tasks:
            raise SchemaError(f"siblings entry for unknown task {p!r}")
        if sorted(order) != sorted(children[p]):
            raise SchemaError(
                f"siblings of {p!r} must be a permutation of its children {children[p]}")
        children[p] = list(order)

    deps = set()
    for edge in document.get("deps", []):
        b, a = edge.get("before"), edge.get("after")
        if b not in tasks or a not in tasks:
            raise SchemaError(f"dep references unknown task: {edge!r}")
        if b == a:
            raise CyclicDependence(f"task {b!r} depends on itself")
        deps.add((b, a))
    for p, group in children.items():
        members = set(group)
        _acyclic([(b, a) for b, a in deps if b in members and a in members], group, p)
    return TaskGraph(tasks=tasks, root=roots[0], parent=parent,
                     children={p: tuple(c) for p, c in children.items()},
                     deps=frozenset(deps), ispaces=ispaces)


# -- shard trees (reference: tasksim/sim.py:50-120) -------------------------------------


@dataclass(frozen=True)
class ShardLocal:
    node: int


@dataclass(frozen=True)
class ShardDistribute:
    left: IndexTask
    right: IndexTask
    left_node: int
    right_node: int


@dataclass(frozen=True)
class ShardTree:
    decisions: dict
    subtasks: dict
    leaves: tuple
    targets: dict   # leaf id -> (node, proc)


def shard_policy(task: IndexTask, mapping: MappingFn, ispace):
    """One SHARD decision (reference semantics, point by point): the points of the
    smallest (node, proc) split off as task/0, the rest as task/1."""
    if not task.points:
        raise EmptyTask(f"task {task.id!r} has no points")
    ispace = tuple(ispace)
    return _decide(task, [tuple(mapping(p, ispace)) for p in task.points])


def _decide(task, targets):
    distinct = sorted(set(targets))
    if len(distinct) == 1:
        return ShardLocal(distinct[0][0])
    low = distinct[0]
    left = tuple(p for p, t in zip(task.points, targets) if t == low)
    right = tuple(p for p, t in zip(task.points, targets) if t != low)
    return ShardDistribute(IndexTask(task.id + "/0", left), IndexTask(task.id + "/1", right),
                           low[0], distinct[1][0])


def shard_tree(task: IndexTask, targets) -> ShardTree:
    """The complete shard tree from every point's target (node, proc): the policy's
    fixpoint in closed form -- the k-th smallest target's points are leaf
    task + "/1" * k + "/0", and node task + "/1" * k holds the points of targets
    >= k in task order."""
    if not task.points:
        raise EmptyTask(f"task {task.id!r} has no points")
    targets = [tuple(t) for t in targets]
    order = sorted(set(targets))
    rank = {t: k for k, t in enumerate(order)}
    ranks = [rank[t] for t in targets]
    decisions, subtasks, leaves, leaf_target = {}, {}, [], {}
    cur = task
    for k, t in enumerate(order):
        subtasks[cur.id] = cur
        if k == len(order) - 1:
            decisions[cur.id] = ShardLocal(t[0])
            leaves.append(cur.id)
            leaf_target[cur.id] = t
            break
        left = IndexTask(cur.id + "/0", tuple(p for p, r in zip(task.points, ranks) if r == k))
        right = IndexTask(cur.id + "/1", tuple(p for p, r in zip(task.points, ranks) if r > k))
        decisions[cur.id] = ShardDistribute(left, right, t[0], order[k + 1][0])
        subtasks[left.id] = left
        decisions[left.id] = ShardLocal(t[0])
        leaves.append(left.id)
        leaf_target[left.id] = t
        cur = right
    return ShardTree(decisions, subtasks, tuple(sorted(leaves)), leaf_target)


def expand_shards(task: IndexTask, mapping: MappingFn, ispace) -> ShardTree:
    """The shard tree of `task` (reference: sim.py:101-120).  A repo
    `MappingFunction` maps and partitions all of the task's points in one fused
    K1 + K2 launch; any other callable is mapped point by point."""
    from .dsl.interp import MappingFunction

    if not task.points:
        raise EmptyTask(f"task {task.id!r} has no points")
    ispace = tuple(ispace)
    k = len(task.points[0])
    if isinstance(mapping, MappingFunction) and k > 0:
        return shard_tree(task, _batched_targets(task, mapping, ispace))
    return shard_tree(task, [tuple(mapping(p, ispace)) for p in task.points])


def _batched_targets(task, fn, ispace):
    """Every point's (node, proc) from one map + partition launch (K1 + K2)."""
    from . import native

    torch = native.require_cuda()
    pts = torch.tensor(task.points, dtype=torch.int32).to("cuda", non_blocking=True)
    own = fn.map_partition(ispace, points=pts)
    ppn = fn.machine.procs_per_node
    targets = [None] * len(task.points)
    counts = own.counts.tolist()
    offsets = own.offsets.tolist()
    perm = own.perm.tolist()
    for pid, (o, c) in enumerate(zip(offsets, counts)):
        if c:
            t = divmod(pid, ppn)
            for i in perm[o:o + c]:
                targets[i] = t
    return targets


# -- traces (reference: tasksim/trace.py) -------------------------------------------------


@dataclass(frozen=True)
class LogEntry:
    stage: str
    task: str
    node: int | None
    proc: int | None
    step: int

    def record(self) -> dict:
        return {"stage": self.stage, "task": self.task, "node": self.node, "proc": self.proc,
                "step": self.step}


@dataclass
class Trace:
    entries: tuple
    proc_stats: dict = field(default_factory=dict)

    def records(self) -> list:
        return [e.record() for e in self.entries]

    @staticmethod
    def from_records(records) -> "Trace":
        return Trace(tuple(LogEntry(r["stage"], r["task"], r.get("node"), r.get("proc"),
                                    r["step"]) for r in records))

    def stages_of(self, task: str) -> list:
        return [e.stage for e in self.entries if e.task == task]


# -- the semantics (reference: tasksim/sim.py:174-514) ----------------------------------

RULES = ("EXECUTE", "LAUNCH", "MAP", "LOCAL", "DISTRIBUTE", "ENQUEUE")  # priority order
EXECUTE, LAUNCH, MAP, LOCAL, DISTRIBUTE, ENQUEUE = range(6)


@dataclass
class ExecState:
    enqueued_queues: dict
    mapped_queues: dict
    log: tuple


class _Fragment:
    """A (sub)task instance moving through the pipeline."""

    __slots__ = ("task", "origin", "decision", "target", "node", "in_eq", "in_mq", "mapped",
                 "launched", "executed")

    def __init__(self, task, origin, decision, target, node=None):
        self.task, self.origin, self.decision, self.target = task, origin, decision, target
        self.node = node
        self.in_eq = self.in_mq = self.mapped = self.launched = self.executed = False


class _Task:
    """Per graph task: leaf counters and the premises its fragments wait on."""

    __slots__ = ("leaves", "unmapped", "unlaunched", "unexecuted", "map_deps", "exec_deps",
                 "children", "next_child", "waiting_map", "waiting_launch", "waiting_exec")

    def __init__(self, leaves, map_deps, exec_deps, children):
        self.leaves = self.unmapped = self.unlaunched = self.unexecuted = leaves
        self.map_deps, self.exec_deps, self.children = map_deps, exec_deps, children
        self.next_child = 0
        self.waiting_map, self.waiting_launch, self.waiting_exec = set(), set(), set()


class Simulator:
    """One run of the lifecycle semantics over a task graph and a mapping; the
    shard trees are built by `expand_shards` (batched for repo mappers)."""

    def __init__(self, graph: TaskGraph, mapping: MappingFn, machine,
                 scheduler: str = "deterministic", seed: int | None = None):
        if scheduler not in ("deterministic", "random"):
            raise ValueError(f"unknown scheduler {scheduler!r}")
        self.graph, self.mapping, self.machine = graph, mapping, machine
        self.scheduler = scheduler
        self.rng = random.Random(seed)
        self.step_no = 0
        self.log: list = []
        self.e_queues: dict = {}
        self.m_queues: dict = {}
        self.trees = {tid: expand_shards(t, mapping, graph.ispaces[tid])
                      for tid, t in graph.tasks.items() if tid != graph.root}
        self.enqueue_node = {tid: min(tr.targets.values())[0] for tid, tr in self.trees.items()}
        self.enqueue_node[graph.root] = 0
        self.state_of = {
            tid: _Task(1 if tid == graph.root else len(self.trees[tid].leaves),
                       len(graph.sibling_deps_before[tid]), len(graph.deps_before[tid]),
                       len(graph.children[tid]))
            for tid in graph.tasks}
        self.frags: dict = {}
        self._heaps = [[] for _ in RULES]   # deterministic scheduler
        self._pool: list = []               # random scheduler (swap-remove pool)
        self._in_pool: set = set()
        self._start()

    # candidates -------------------------------------------------------------------------

    def _offer(self, rule, tid):
        if self.scheduler == "deterministic":
            heapq.heappush(self._heaps[rule], tid)
        elif (rule, tid) not in self._in_pool:
            self._in_pool.add((rule, tid))
            self._pool.append((rule, tid))

    def _applicable(self, rule, tid) -> bool:
        g = self.graph
        if rule == ENQUEUE:
            if tid not in self.state_of or tid == g.root:
                return False
            p = g.parent[tid]
            ps = self.state_of[p]
            order = g.children[p]
            return ps.unlaunched == 0 and ps.next_child < len(order) and order[ps.next_child] == tid
        f = self.frags.get(tid)
        if f is None:
            return False
        st = self.state_of[f.origin]
        if rule == DISTRIBUTE:
            return f.in_eq and isinstance(f.decision, ShardDistribute)
        if rule == LOCAL:
            return f.in_eq and isinstance(f.decision, ShardLocal)
        if rule == MAP:
            return f.in_mq and st.map_deps == 0
        if rule == LAUNCH:
            return f.mapped and not f.launched and st.exec_deps == 0
        if rule == EXECUTE:
            return f.launched and not f.executed and st.children == 0
        return False

    def _next(self):
        if self.scheduler == "deterministic":
            for rule, heap in enumerate(self._heaps):
                while heap:
                    tid = heapq.heappop(heap)
                    if self._applicable(rule, tid):
                        return rule, tid
            return None
        while self._pool:
            i = self.rng.randrange(len(self._pool))
            cand = self._pool[i]
            self._pool[i] = self._pool[-1]
            self._pool.pop()
            self._in_pool.discard(cand)
            if self._applicable(*cand):
                return cand
        return None

    # effects ----------------------------------------------------------------------------

    def _log(self, stage, tid, node, proc):
        self.log.append(LogEntry(stage, tid, node, proc, self.step_no))

    def _offer_next_child(self, parent):
        order = self.graph.children[parent]
        k = self.state_of[parent].next_child
        if k < len(order):
            self._offer(ENQUEUE, order[k])

    def _start(self):
        root = self.graph.root
        f = _Fragment(self.graph.tasks[root], root, ShardLocal(0), (0, 0))
        f.mapped = f.launched = True
        self.frags[root] = f
        st = self.state_of[root]
        st.unmapped = st.unlaunched = 0
        st.waiting_exec.add(root)
        self._log(LAUNCHED, root, 0, 0)
        self.step_no = 1
        if st.children == 0:
            self._offer(EXECUTE, root)
        else:
            self._offer_next_child(root)

    def _enqueue_fragment(self, task, origin, node):
        tree = self.trees[origin]
        dec = tree.decisions[task.id]
        f = _Fragment(task, origin, dec, tree.targets.get(task.id), node)
        f.in_eq = True
        self.frags[task.id] = f
        self.e_queues.setdefault(node, deque()).append(task.id)
        self._offer(LOCAL if isinstance(dec, ShardLocal) else DISTRIBUTE, task.id)

    def _release(self, rule, members):
        for m in sorted(members):
            self._offer(rule, m)

    def _fire(self, rule, tid):
        g = self.graph
        if rule == ENQUEUE:
            p = g.parent[tid]
            node = self.enqueue_node[p]
            self._log(ENQUEUED, tid, node, None)
            self._enqueue_fragment(g.tasks[tid], tid, node)
            self.state_of[p].next_child += 1
            self._offer_next_child(p)
            return
        f = self.frags[tid]
        st = self.state_of[f.origin]
        if rule == DISTRIBUTE:
            self.e_queues[f.node].remove(tid)
            f.in_eq = False
            d = f.decision
            self._enqueue_fragment(d.left, f.origin, d.left_node)
            self._enqueue_fragment(d.right, f.origin, d.right_node)
        elif rule == LOCAL:
            self.e_queues[f.node].remove(tid)
            f.in_eq = False
            f.node = f.decision.node
            f.in_mq = True
            self.m_queues.setdefault(f.node, deque()).append(tid)
            st.waiting_map.add(tid)
            if st.map_deps == 0:
                self._offer(MAP, tid)
        elif rule == MAP:
            self.m_queues[f.node].remove(tid)
            f.in_mq = False
            f.mapped = True
            self._log(MAPPED, tid, *f.target)
            st.waiting_map.discard(tid)
            st.waiting_launch.add(tid)
            st.unmapped -= 1
            if st.exec_deps == 0:
                self._offer(LAUNCH, tid)
            if st.unmapped == 0:  # the task is mapped: its mapped-after siblings may map
                for succ in g.deps_after[f.origin]:
                    if f.origin in g.sibling_deps_before[succ]:
                        s = self.state_of[succ]
                        s.map_deps -= 1
                        if s.map_deps == 0:
                            self._release(MAP, s.waiting_map)
        elif rule == LAUNCH:
            f.launched = True
            self._log(LAUNCHED, tid, *f.target)
            st.waiting_launch.discard(tid)
            st.waiting_exec.add(tid)
            st.unlaunched -= 1
            if st.children == 0:
                self._offer(EXECUTE, tid)
            if st.unlaunched == 0:
                self._offer_next_child(f.origin)
        elif rule == EXECUTE:
            f.executed = True
            self._log(EXECUTED, tid, *f.target)
            st.waiting_exec.discard(tid)
            st.unexecuted -= 1
            if st.unexecuted == 0:  # successors may launch, the parent may execute
                for succ in g.deps_after[f.origin]:
                    s = self.state_of[succ]
                    s.exec_deps -= 1
                    if s.exec_deps == 0:
                        self._release(LAUNCH, s.waiting_launch)
                p = g.parent.get(f.origin)
                if p is not None:
                    ps = self.state_of[p]
                    ps.children -= 1
                    if ps.children == 0:
                        self._release(EXECUTE, ps.waiting_exec)
        else:
            raise AssertionError(f"unknown rule {rule}")

    # driving ----------------------------------------------------------------------------

    def step(self) -> bool:
        """Apply one rule; False when none applies."""
        move = self._next()
        if move is None:
            return False
        self._fire(*move)
        self.step_no += 1
        return True

    @property
    def done(self) -> bool:
        return all(s.unexecuted == 0 for s in self.state_of.values())

    def state(self) -> ExecState:
        return ExecState({n: list(q) for n, q in self.e_queues.items() if q},
                         {n: list(q) for n, q in self.m_queues.items() if q}, tuple(self.log))

    def run(self) -> Trace:
        while self.step():
            pass
        if not self.done:
            raise Stuck(self._diagnose(), blocked=self._blocked())
        stats = {}
        for tid, f in self.frags.items():
            if tid == self.graph.root or f.target is None or not f.executed:
                continue
            e = stats.setdefault(f.target, {"tasks": 0, "points": 0})
            e["tasks"] += 1
            e["points"] += len(f.task.points)
        return Trace(tuple(self.log), stats)

    def _blocked(self) -> list:
        return sorted(t for t, s in self.state_of.items() if s.unexecuted)

    def _diagnose(self) -> str:
        g = self.graph
        for tid in self._blocked():
            st = self.state_of[tid]
            if tid not in self.frags:
                p = g.parent[tid]
                if self.state_of[p].unlaunched:
                    return f"stuck: ENQUEUE of {tid!r} needs parent {p!r} launched"
                return f"stuck: ENQUEUE of {tid!r} waits on an earlier sibling"
            if st.unmapped and st.map_deps > 0:
                miss = [d for d in g.sibling_deps_before[tid] if self.state_of[d].unmapped]
                return f"stuck: MAP of {tid!r} needs mapped siblings {miss}"
            if st.unlaunched and st.exec_deps > 0:
                miss = [d for d in g.deps_before[tid] if self.state_of[d].unexecuted]
                return f"stuck: LAUNCH of {tid!r} needs executed predecessors {miss}"
            if st.children > 0:
                miss = [c for c in g.children[tid] if self.state_of[c].unexecuted]
                return f"stuck: EXECUTE of {tid!r} needs executed children {miss}"
        return "stuck: no applicable rule"


def step(sim: Simulator) -> bool:
    return sim.step()


def run_to_quiescence(graph: TaskGraph, mapping: MappingFn, machine,
                      scheduler: str = "deterministic", seed: int | None = None) -> Trace:
    """Run the semantics until no rule applies; raises Stuck if unfinished."""
    return Simulator(graph, mapping, machine, scheduler=scheduler, seed=seed).run()
