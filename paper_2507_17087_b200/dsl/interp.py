"""Drop-in mapping API: `compile_mapper`, `MappingFunction`, `eval_mapping`.

Same names, signatures and error behaviour as the reference
(reference: dsl/interp.py:27-433), re-built around the batched GPU plan:

* `Evaluator(program, machine)` evaluates global bindings on the host at
  construction, like the reference (interp.py:50-56);
* `compile_mapper(program, task, machine)` binds a task to its IndexTaskMap
  function (interp.py:421-433) and returns a `MappingFunction`;
* a `MappingFunction` keeps one lowered point program per iteration space
  (its `_prefix_cache`, interp.py:378,407-412); the per-point work always
  runs in the JIT-compiled sm_100a kernel (K1, csrc/mapping.cpp):
    - `fn(ipoint, ispace)`            one point -> (node, proc)
    - `fn.map_ispace(ispace, ...)`    every row-major point of the launch
                                      (cli.py:155-161 order) -> int32 ids
    - `fn.map_points(points, ispace)` explicit int32 [n, k] points -> ids
  where id = node * procs_per_node + proc.  Failures raise the reference's
  exception (class and message) for the lowest failing point.
"""

from __future__ import annotations

import copy
import ctypes
import threading
from collections import OrderedDict

from ..errors import EvalError, LoweringError, NativeError, NoBinding
from ..spaces import MachineShape
from . import ast as A
from .lower import INT32, Lowerer, ProcRef, format_site, lower_mapping, split_plan

__all__ = ["Evaluator", "MappingFunction", "PointProgram", "ProcRef", "compile_mapper",
           "eval_mapping"]


class PointProgram:
    """A lowered point program and its lazily created device plan."""

    def __init__(self, lowered):
        from .. import native

        self.lowered = lowered
        prog = lowered.program
        flat = prog.flat()
        widths = prog.widths()
        self._insns = (native.PmInsn * max(1, len(flat)))(*[native.PmInsn(*t) for t in flat])
        self._widths = (ctypes.c_uint8 * max(1, len(widths)))(*widths)
        ext = [int(e) for e in lowered.extents] if lowered.implicit else []
        self._ext = (ctypes.c_int64 * max(1, len(ext)))(*ext)
        self.c_program = native.PmProgram(len(flat), self._insns, len(widths), self._widths,
                                          lowered.n_coords, int(lowered.implicit), self._ext)
        self.sites = prog.sites
        self._plans: dict[int, int] = {}
        self._lock = threading.Lock()

    @property
    def n_coords(self) -> int:
        return self.lowered.n_coords

    def source(self) -> str:
        from .. import native

        n = ctypes.c_size_t(0)
        native.check(native.lib().pm_codegen(ctypes.byref(self.c_program), None, 0,
                                             ctypes.byref(n)), "pm_codegen")
        buf = ctypes.create_string_buffer(n.value + 1)
        native.check(native.lib().pm_codegen(ctypes.byref(self.c_program), buf, n.value + 1,
                                             ctypes.byref(n)), "pm_codegen")
        return buf.value.decode()

    def compile_check(self) -> None:
        from .. import native

        native.check(native.lib().pm_compile_check(ctypes.byref(self.c_program)),
                     "pm_compile_check")

    def compile_check_probe(self) -> None:
        """NVRTC-compile the failure probe of this program (no GPU)."""
        from .. import native

        native.check(native.lib().pm_compile_check_probe(ctypes.byref(self.c_program)),
                     "pm_compile_check_probe")

    def compile_check_fused(self) -> None:
        """NVRTC-compile the fused map + partition kernels of this program (no GPU)."""
        from .. import native

        native.check(native.lib().pm_compile_check_fused(ctypes.byref(self.c_program)),
                     "pm_compile_check_fused")

    def plan(self, device: int) -> int:
        from .. import native

        with self._lock:
            h = self._plans.get(device)
            if h is None:
                out = ctypes.c_void_p()
                native.check(native.lib().pm_plan_create(ctypes.byref(self.c_program),
                                                         ctypes.byref(out)), "pm_plan_create")
                h = self._plans[device] = out.value
        return h

    def launch(self, points, n: int, first: int, out, status, stream=None) -> None:
        """Stream-ordered launch; `status` must hold UINT64_MAX beforehand."""
        from .. import native

        torch = native.require_cuda()
        dev = out.device.index if out.device.index is not None else torch.cuda.current_device()
        with torch.cuda.device(dev):
            plan = self.plan(dev)
            pts = 0 if points is None else points.data_ptr()
            native.check(native.lib().pm_map_batch(plan, pts, n, first, out.data_ptr(),
                                                   status.data_ptr(), native.stream_ptr(stream)),
                         "pm_map_batch")

    def map_hist(self, points, n: int, first: int, nbins: int, counts, offsets, status, scratch,
                 stream=None) -> None:
        """Fused pass 1 (pm_map_hist): per-processor counts of points [first, first+n)."""
        from .. import native

        torch = native.require_cuda()
        dev = counts.device.index if counts.device.index is not None else \
            torch.cuda.current_device()
        with torch.cuda.device(dev):
            plan = self.plan(dev)
            native.check(native.lib().pm_map_hist(
                plan, 0 if points is None else points.data_ptr(), n, first, nbins,
                counts.data_ptr(), offsets.data_ptr(), status.data_ptr(), scratch.data_ptr(),
                scratch.numel(), native.stream_ptr(stream)), "pm_map_hist")

    def map_scatter(self, points, n: int, first: int, nbins: int, *, out=None, perm=None,
                    bin_dst=None, index_base: int = 0, status, scratch, stream=None) -> None:
        """Fused pass 2 (pm_map_scatter): stable slots of every point (after map_hist)."""
        from .. import native

        torch = native.require_cuda()
        dev = status.device.index if status.device.index is not None else \
            torch.cuda.current_device()
        ptr = (lambda t: 0 if t is None else t.data_ptr())
        with torch.cuda.device(dev):
            plan = self.plan(dev)
            native.check(native.lib().pm_map_scatter(
                plan, ptr(points), n, first, nbins, ptr(out), ptr(perm), ptr(bin_dst),
                index_base, status.data_ptr(), scratch.data_ptr(), scratch.numel(),
                native.stream_ptr(stream)), "pm_map_scatter")

    def raise_for(self, status_word: int, points=None) -> None:
        """Re-raise the failure a status word encodes (no-op for 'no failure'):
        the reference's exception for the lowest failing point, with its exact
        message -- a site whose message quotes per-point values (an index tuple,
        a tuple index, a dimension) is formatted from that point's registers,
        read back by the failure probe (pm_map_probe).  `points`: the explicit
        int32 points of the failing launch (None in implicit mode)."""
        if status_word in (-1, (1 << 64) - 1):
            return
        status_word &= (1 << 64) - 1
        site = status_word & 0xFFFF
        if site >= len(self.sites):
            raise EvalError("mapping function evaluation failed")
        exc = copy.copy(self.sites[site])
        fmt = self.lowered.program.site_fmts.get(site)
        if fmt is not None:
            regs, got = self.probe(status_word >> 16, points)
            if got != site:
                raise NativeError(f"failure probe reached site {got}, the launch site {site}")
            exc = type(exc)(format_site(fmt, regs))
        raise exc

    def probe(self, index: int, points=None):
        """(registers, site) of point `index` evaluated by the failure probe."""
        from .. import native

        torch = native.require_cuda()
        dev = points.device if points is not None else \
            torch.device("cuda", torch.cuda.current_device())
        with torch.cuda.device(dev):
            plan = self.plan(dev.index)
            nregs = native.lib().pm_plan_regs(plan)
            dump = torch.zeros(2 * max(nregs, 1), dtype=torch.int64, device=dev)
            site = torch.full((2,), -1, dtype=torch.int32, device=dev)
            native.check(native.lib().pm_map_probe(
                plan, 0 if points is None else points.data_ptr(), int(index), dump.data_ptr(),
                site.data_ptr(), native.stream_ptr(None)), "pm_map_probe")
            words = dump.cpu().tolist()
            got = int(site[0].item())
        regs = []
        for r in range(nregs):
            v = (words[2 * r] & ((1 << 64) - 1)) | (words[2 * r + 1] << 64)
            regs.append(v)
        return regs, got

    @staticmethod
    def failing_index(status_word: int) -> int | None:
        if status_word in (-1, (1 << 64) - 1):
            return None
        return (status_word & ((1 << 64) - 1)) >> 16

    def __del__(self):
        try:
            from .. import native

            for h in self._plans.values():
                native.lib().pm_plan_destroy(h)
        except Exception:  # noqa: BLE001 - interpreter shutdown
            pass


_CACHE_LIMIT = 256
_cache: "OrderedDict[tuple, PointProgram]" = OrderedDict()
_cache_lock = threading.Lock()


def _lowered(evaluator: "Evaluator", func: A.FuncDef, ispace, implicit, k, plan_mode):
    key = (evaluator.program, evaluator.machine, func.name, ispace, implicit, k, plan_mode)
    with _cache_lock:
        hit = _cache.get(key)
        if hit is not None:
            _cache.move_to_end(key)
            return hit
    low = Lowerer(evaluator.program, evaluator.machine, globals_env=evaluator.globals)
    pp = PointProgram(lower_mapping(low, func, ispace, implicit=implicit, n_coords=k,
                                    plan_mode=plan_mode))
    with _cache_lock:
        _cache[key] = pp
        while len(_cache) > _CACHE_LIMIT:
            _cache.popitem(last=False)
    return pp


def _run_points(pp: PointProgram, pts_list) -> list[tuple[int, int]]:
    """Map explicit host points through the device kernel (used by __call__)."""
    from .. import native

    torch = native.require_cuda()
    k = pp.n_coords
    for pt in pts_list:
        for c in pt:
            if not INT32[0] <= c <= INT32[1]:
                raise LoweringError(f"point coordinate {c} does not fit the int32 point layout")
    n = len(pts_list)
    dev = torch.device("cuda", torch.cuda.current_device())
    pts = torch.tensor(pts_list, dtype=torch.int32).reshape(n, k).to(dev) if k else None
    out = torch.empty(max(n, 1), dtype=torch.int32, device=dev)
    status = torch.full((1,), -1, dtype=torch.int64, device=dev)
    pp.launch(pts, n, 0, out, status)
    word = int(status.item())
    pp.raise_for(word, pts)
    return out[:n].tolist()


class Evaluator:
    """Host-side state of one program on one machine (reference: interp.py:47-56)."""

    def __init__(self, program: A.MapperProgram, machine: MachineShape):
        self.program = program
        self.machine = machine
        self.functions = program.functions
        self.globals = Lowerer(program, machine).globals

    def run_mapping(self, func_name: str, ipoint, ispace) -> tuple[int, int]:
        """One point through the device kernel (reference: interp.py:60-69)."""
        func = self.functions.get(func_name)
        if func is None:
            raise EvalError(f"undefined mapping function {func_name!r}")
        if len(func.params) != 2:
            raise EvalError(f"mapping function {func_name!r} must take (ipoint, ispace)")
        ipoint, ispace = tuple(ipoint), tuple(ispace)
        pp = _lowered(self, func, ispace, False, len(ipoint), False)
        pid = _run_points(pp, [ipoint])[0]
        return divmod(pid, self.machine.procs_per_node)


def eval_mapping(program, func: str, ipoint, ispace, machine) -> tuple[int, int]:
    """Evaluate one mapping function at one point (reference: interp.py:312-320)."""
    return Evaluator(program, machine).run_mapping(func, ipoint, ispace)


class _PrefixCache(dict):
    """ispace -> {(implicit, k): PointProgram}; mirrors the reference's cache keys."""


class MappingFunction:
    """Compiled point -> (node, proc) map for one task (reference: interp.py:366-418)."""

    def __init__(self, evaluator: Evaluator, func: A.FuncDef):
        self.evaluator = evaluator
        self.func = func
        self._plan = split_plan(func)
        self._prefix_cache = _PrefixCache()
        self._lock = threading.Lock()

    @property
    def machine(self) -> MachineShape:
        return self.evaluator.machine

    def program_for(self, ispace, *, implicit: bool, k: int | None = None) -> PointProgram:
        ispace = tuple(int(e) for e in ispace)
        k = len(ispace) if implicit else int(k)
        with self._lock:
            per = self._prefix_cache.setdefault(ispace, {})
            pp = per.get((implicit, k))
            if pp is None:
                pp = per[(implicit, k)] = _lowered(self.evaluator, self.func, ispace, implicit,
                                                   k, True)
        return pp

    # launches up to this many points are mapped whole on the first single-point
    # call and answered from the host copy of their ids afterwards
    LOOKUP_MAX_POINTS = 1 << 22
    LOOKUP_LAUNCHES = 8

    def __call__(self, ipoint, ispace) -> tuple[int, int]:
        """One point -> (node, proc): the reference's per-point plugin call
        (MappingFn, tasksim/sim.py:44), as driven point by point by cmd_map
        (cli.py:158-161) and shard_policy (tasksim/sim.py:78).

        The first call for a launch maps every point of it on the GPU (K1,
        implicit row-major mode) and keeps the ids on the host, so the
        reference's O(points x depth) call pattern costs one launch plus
        lookups.  A point that failed in that launch, a point outside the
        launch and launches above LOOKUP_MAX_POINTS take the single-point
        device path, which raises the reference's exception for it."""
        ipoint, ispace = tuple(ipoint), tuple(ispace)
        ids = self._launch_ids(ispace)
        if ids is not None and len(ipoint) == len(ispace):
            lin = 0
            for c, e in zip(ipoint, ispace):
                if not (type(c) is int and 0 <= c < e):
                    break
                lin = lin * e + c
            else:
                pid = ids[lin]
                if pid >= 0:
                    return divmod(pid, self.machine.procs_per_node)
        pp = self.program_for(ispace, implicit=False, k=len(ipoint))
        pid = _run_points(pp, [ipoint])[0]
        return divmod(pid, self.machine.procs_per_node)

    def _launch_ids(self, ispace):
        """Host copy (array of int32, -1 = failing point) of the whole launch's
        processor ids, computed by K1; None for launches too large to keep."""
        cache = self.__dict__.setdefault("_ids_cache", OrderedDict())
        with self._lock:
            hit = cache.get(ispace)
            if hit is not None:
                cache.move_to_end(ispace)
                return hit
        total = 1
        for e in ispace:
            if type(e) is not int or e <= 0:
                return None
            total *= e
        if total > self.LOOKUP_MAX_POINTS:
            return None
        from array import array

        try:
            dev_ids = self.map_ispace(ispace, check=False)
        except LoweringError:
            return None  # the single-point path reports it
        ids = array("i")
        ids.frombytes(dev_ids.cpu().numpy().tobytes())
        with self._lock:
            cache[ispace] = ids
            while len(cache) > self.LOOKUP_LAUNCHES:
                cache.popitem(last=False)
        return ids

    # -- batched device API -----------------------------------------------------

    def map_ispace(self, ispace, first: int = 0, count: int | None = None, *, out=None,
                   status=None, check: bool = True, stream=None):
        """Processor ids of row-major points [first, first + count) of `ispace`.

        Returns an int32 CUDA tensor (id = node * procs_per_node + proc).  With
        `check`, synchronises on the 8-byte status word and raises the
        reference's exception for the lowest failing point.
        """
        from .. import native

        torch = native.require_cuda()
        ispace = tuple(int(e) for e in ispace)
        total = 1
        for e in ispace:
            total *= max(e, 0)
        if count is None:
            count = total - first
        if first < 0 or count < 0 or first + count > total:
            raise ValueError(f"points [{first}, {first + count}) outside the launch of {total}")
        dev = torch.device("cuda", torch.cuda.current_device())
        if out is None:
            out = torch.empty(max(count, 1), dtype=torch.int32, device=dev)
        own_status = status is None
        if own_status:
            status = torch.full((1,), -1, dtype=torch.int64, device=out.device)
        if count:
            pp = self.program_for(ispace, implicit=True)
            pp.launch(None, count, first, out, status, stream)
            if check:
                pp.raise_for(int(status.item()))
        return out[:count]

    def map_partition(self, ispace, first: int = 0, count: int | None = None, *,
                      points=None, with_ids: bool = False, check: bool = True, stream=None):
        """Ownership lists of a launch in one fused pass pair (K1 + K2 without the
        id array): the stable partition of points [first, first + count) of
        `ispace` -- or of the explicit int32 [n, k] `points` -- by processor.

        Same result as `ownership.partition(self.map_ispace(...), P)` (perm holds
        indices relative to `first`); `with_ids` also returns the processor ids.
        Launches of more than 64 processors use the unfused K1 + K2 path."""
        from .. import native
        from ..ownership import Ownership, partition

        torch = native.require_cuda()
        ispace = tuple(int(e) for e in ispace)
        nprocs = self.machine.nodes * self.machine.procs_per_node
        if points is not None:
            if points.dtype != torch.int32 or not points.is_cuda or points.dim() != 2:
                raise ValueError("points must be an int32 CUDA tensor of shape [n, k]")
            points = points.contiguous()
            first, count = 0, points.shape[0]
            dev = points.device
        else:
            total = 1
            for e in ispace:
                total *= max(e, 0)
            if count is None:
                count = total - first
            if first < 0 or count < 0 or first + count > total:
                raise ValueError(f"points [{first}, {first + count}) outside the launch of {total}")
            dev = torch.device("cuda", torch.cuda.current_device())
        if nprocs > 64:
            ids = (self.map_points(points, ispace, check=check, stream=stream) if points is not None
                   else self.map_ispace(ispace, first, count, check=check, stream=stream))
            own = partition(ids, nprocs, stream=stream, check=check)
            return (own, ids) if with_ids else own
        pp = (self.program_for(ispace, implicit=False, k=points.shape[1]) if points is not None
              else self.program_for(ispace, implicit=True))
        counts = torch.empty(nprocs, dtype=torch.int64, device=dev)
        offsets = torch.empty(nprocs, dtype=torch.int64, device=dev)
        perm = torch.empty(max(count, 1), dtype=torch.int32, device=dev)
        ids = torch.empty(max(count, 1), dtype=torch.int32, device=dev) if with_ids else None
        status = torch.full((1,), -1, dtype=torch.int64, device=dev)
        nbytes = native.lib().pm_map_partition_scratch_bytes(count, nprocs)
        scratch = torch.empty(nbytes, dtype=torch.uint8, device=dev)
        pfirst = 0 if points is not None else first
        pp.map_hist(points, count, pfirst, nprocs, counts, offsets, status, scratch, stream)
        pp.map_scatter(points, count, pfirst, nprocs, out=ids, perm=perm, status=status,
                       scratch=scratch, stream=stream)
        if check:
            pp.raise_for(int(status.item()), points)
        own = Ownership(counts, offsets, perm[:count])
        return (own, ids[:count]) if with_ids else own

    def map_points(self, points, ispace, *, out=None, status=None, check: bool = True,
                   stream=None):
        """Processor ids of explicit points (int32 CUDA tensor [n, k], row-major)."""
        from .. import native

        torch = native.require_cuda()
        if points.dtype != torch.int32 or not points.is_cuda or points.dim() != 2:
            raise ValueError("points must be an int32 CUDA tensor of shape [n, k]")
        points = points.contiguous()
        n, k = points.shape
        if out is None:
            out = torch.empty(max(n, 1), dtype=torch.int32, device=points.device)
        if status is None:
            status = torch.full((1,), -1, dtype=torch.int64, device=points.device)
        if n:
            pp = self.program_for(tuple(ispace), implicit=False, k=k)
            pp.launch(points, n, 0, out, status, stream)
            if check:
                pp.raise_for(int(status.item()), points)
        return out[:n]


def compile_mapper(program: A.MapperProgram, task: str, machine: MachineShape) -> MappingFunction:
    """Bind `task` to its IndexTaskMap function (reference: interp.py:421-433)."""
    binds = program.bindings()
    if task not in binds:
        raise NoBinding(f"task {task!r} has no IndexTaskMap statement")
    func = program.functions.get(binds[task])
    if func is None:
        raise EvalError(f"task {task!r} is bound to undefined function {binds[task]!r}")
    if len(func.params) != 2:
        raise EvalError(f"mapping function {func.name!r} must take (ipoint, ispace)")
    return MappingFunction(Evaluator(program, machine), func)


_ = NativeError  # re-exported error class used by callers of this module
