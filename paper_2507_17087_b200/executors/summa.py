"""Mapped SUMMA: C = A @ B on the GPUs of one box, distributed by a Mapple
block mapper (the paper's matmul workloads).

Planning (once per problem, like the reference's per-ispace prefix,
dsl/interp.py:407-412):
  1. the C block launch (M/bs x N/bs points) is mapped to GPUs by a Mapple
     program on the machine (G GPUs, 1 per node) -- the decompose
     mapper `m.merge(0,1).decompose(0, ispace)` or the Algorithm-1 heuristic
     `m.merge(0,1).split(0, g0)` -- with the K1 kernel;
  2. the K2 kernel partitions the launch into per-GPU ownership lists, from
     which every GPU's C rectangle, its row group and its column group follow;
  3. A row-panels and B column-panels are distributed SUMMA style: the GPU
     owning C rectangle (rows R, cols C) holds A[R, K-slice] and B[K-slice, C],
     the K-slice being its position inside its row (column) group.
Execution (one step = one full multiply):
  * every GPU pulls the A slices of its row group and the B slices of its
    column group straight from the peers' memory over NVLink with the copy
    engines (no SM cost, no NCCL kernel competing with the GEMM);
  * B first, then A in row chunks, so the tcgen05 GEMM (K4) of chunk r runs
    while chunk r+1 is still in flight (a run whose A is local but B remote is
    chunked along C's columns instead, so its first GEMM waits for one B chunk,
    not all of B); C accumulates in TMEM over each run's K.
"""

from __future__ import annotations

from dataclasses import dataclass

from .. import native
from ..dsl import compile_mapper, parse
from ..factorize import greedy_grid, search_optimal
from ..spaces import MachineShape

TILE_MAPPERS = """
m = Machine(GPU)
def tiles_decompose(Tuple ipoint, Tuple ispace):
    q = m.merge(0, 1).decompose(0, ispace)
    return q[*(ipoint * q.size / ispace)]
def tiles_heuristic(Tuple ipoint, Tuple ispace):
    q = m.merge(0, 1).split(0, {g0})
    return q[*(ipoint * q.size / ispace)]
IndexTaskMap gemm_decompose tiles_decompose
IndexTaskMap gemm_heuristic tiles_heuristic
"""


@dataclass(frozen=True)
class Rect:
    r0: int
    r1: int
    c0: int
    c1: int


def rectangles(owner_ids, nbi: int, nbj: int, world: int, block_m: int, block_n: int,
               M: int, N: int) -> list[Rect]:
    """Per-rank C rectangle (element coordinates) from the block owner table.

    Fails unless every rank owns one full rectangle of blocks (a block
    mapping); the SUMMA executor needs a 2D grid.
    """
    spans = {}
    for b, r in enumerate(owner_ids):
        i, j = divmod(b, nbj)
        s = spans.setdefault(r, [i, i, j, j, 0])
        s[0], s[1] = min(s[0], i), max(s[1], i)
        s[2], s[3] = min(s[2], j), max(s[3], j)
        s[4] += 1
    out = []
    for r in range(world):
        if r not in spans:
            raise ValueError(f"GPU {r} owns no C blocks")
        i0, i1, j0, j1, n = spans[r]
        if n != (i1 - i0 + 1) * (j1 - j0 + 1):
            raise ValueError(f"GPU {r} does not own a rectangle of C blocks")
        out.append(Rect(i0 * block_m, min(M, (i1 + 1) * block_m),
                        j0 * block_n, min(N, (j1 + 1) * block_n)))
    return out


@dataclass(frozen=True)
class Layout:
    rects: list
    row_group: list        # per rank: ranks sharing its rows, sorted by column start
    col_group: list        # per rank: ranks sharing its columns, sorted by row start
    a_slice: list          # per rank: (k0, k1) of the A slice it holds
    b_slice: list          # per rank: (k0, k1) of the B slice it holds
    grid: tuple            # (rows of GPUs, cols of GPUs)


def summa_layout(rects: list, K: int) -> Layout:
    world = len(rects)
    row_group, col_group = [], []
    for me in rects:
        rg = sorted((q for q in range(world) if (rects[q].r0, rects[q].r1) == (me.r0, me.r1)),
                    key=lambda q: rects[q].c0)
        cg = sorted((q for q in range(world) if (rects[q].c0, rects[q].c1) == (me.c0, me.c1)),
                    key=lambda q: rects[q].r0)
        row_group.append(rg)
        col_group.append(cg)
    for r in range(world):
        covered = sum(rects[q].c1 - rects[q].c0 for q in row_group[r])
        width = max(x.c1 for x in rects) - min(x.c0 for x in rects)
        if covered != width:
            raise ValueError("row groups do not tile C: not a 2D processor grid")
    a_slice, b_slice = [], []
    for r in range(world):
        pc, a = len(row_group[r]), row_group[r].index(r)
        pr, b = len(col_group[r]), col_group[r].index(r)
        a_slice.append((K * a // pc, K * (a + 1) // pc))
        b_slice.append((K * b // pr, K * (b + 1) // pr))
    grid = (len(col_group[0]), len(row_group[0]))
    return Layout(rects, row_group, col_group, a_slice, b_slice, grid)


def comm_bytes(layout: Layout, K: int, elem: int = 2) -> list[int]:
    """Bytes each GPU receives per multiply (A panels of its row group + B of its column group)."""
    out = []
    for r, rc in enumerate(layout.rects):
        a = (rc.r1 - rc.r0) * sum(layout.a_slice[q][1] - layout.a_slice[q][0]
                                  for q in layout.row_group[r] if q != r)
        b = (rc.c1 - rc.c0) * sum(layout.b_slice[q][1] - layout.b_slice[q][0]
                                  for q in layout.col_group[r] if q != r)
        out.append((a + b) * elem)
    return out


def mapper_grid(world: int, M: int, N: int, mapping: str) -> tuple:
    if mapping == "decompose":
        return search_optimal(world, (M, N))[0]
    if mapping == "heuristic":
        return greedy_grid(world, 2)
    raise ValueError(f"unknown mapping {mapping!r}")


def tile_mapper(world: int, mapping: str):
    g0 = greedy_grid(world, 2)[0]
    prog = parse(TILE_MAPPERS.format(g0=g0))
    return compile_mapper(prog, f"gemm_{mapping}", MachineShape("GPU", world, 1))


def synth(rows: tuple, cols: tuple, ld: int, seed: int, device, dtype=None):
    """Deterministic U(-1, 1) block (bf16 unless `dtype`) of a virtual [*, ld] matrix.

    Element (i, k) depends only on (i * ld + k, seed), so every rank can
    materialise exactly its own slice of the global operands.
    """
    if dtype is not None:
        return synth_f32(rows, cols, ld, seed, device).to(dtype)
    return synth_f32(rows, cols, ld, seed, device).to(native.require_cuda().bfloat16)


def synth_f32(rows: tuple, cols: tuple, ld: int, seed: int, device):
    torch = native.require_cuda()
    i = torch.arange(rows[0], rows[1], device=device, dtype=torch.int64).view(-1, 1)
    k = torch.arange(cols[0], cols[1], device=device, dtype=torch.int64).view(1, -1)
    x = (i * ld + k) % (1 << 31)
    x = (x * 1103515245 + 12345 + seed * 7919) % (1 << 31)
    x = x ^ (x >> 13)
    x = (x * 69069 + 1) % (1 << 31)
    return (x.to(torch.float32) / float(1 << 30)) - 1.0


@dataclass(frozen=True)
class PanelPlan:
    panels: list      # (k0, k1, A source rank, B source rank), in execution order
    chunks: list      # A row chunks of remote panels
    pulls: list       # (operand, source rank, row0, rows, k0, k1, stream index); k in
                      # this GPU's rotated buffer positions (as the gemms' k0, k1)
    gemms: list       # (r0, r1, k0, k1, accumulate, [indices into pulls to wait for], c0, c1)
    n_streams: int
    rot: int = 0      # K rotation of this GPU's A / Bt buffers: global k sits at (k - rot) % K


def plan_panels(layout: Layout, me: int, K: int, mr: int, nc: int, block: int = 128,
                a_chunks: int = 4, copy_streams: int = 1) -> PanelPlan:
    """The per-GPU SUMMA schedule (pure; CPU-testable).

    K is cut at every slice boundary of my row group (A) and column group (B),
    so on each panel both operands come from single GPUs.  The least-remote
    panel (plus the fully local panels next to it in K) runs first -- no or
    little waiting -- while the copy engines bring in the others; the remaining
    panels merge with their K neighbours into runs (one launch per run and
    A-row chunk: fewer accumulate passes over C, longer-K launches); runs that
    pull A are split into row chunks of A so the GEMM of chunk c overlaps the
    pull of chunk c+1.  The first run writes C, later ones accumulate (TMA
    reduce-add epilogue).
    """
    cuts = {0, K}
    for q in layout.row_group[me]:
        cuts.update(layout.a_slice[q])
    for q in layout.col_group[me]:
        cuts.update(layout.b_slice[q])
    cuts = sorted(cuts)
    ranked = []
    for k0, k1 in zip(cuts, cuts[1:]):
        if k1 <= k0:
            continue
        a_src = next(q for q in layout.row_group[me]
                     if layout.a_slice[q][0] <= k0 and k1 <= layout.a_slice[q][1])
        b_src = next(q for q in layout.col_group[me]
                     if layout.b_slice[q][0] <= k0 and k1 <= layout.b_slice[q][1])
        remote = (a_src != me) * mr * (k1 - k0) + (b_src != me) * nc * (k1 - k0)
        ranked.append((remote, k0, k1, a_src, b_src))
    ranked.sort()
    # runs: one GEMM per run and A-row chunk -- fewer accumulate passes over C and
    # longer-K launches.  The first run is the least-remote panel (with the fully
    # local panels K-adjacent to it, which cost no waiting); every other panel merges
    # with its K neighbours, and those runs' pulls overlap the first run's GEMM.
    head = [ranked[0]]
    if ranked[0][0] == 0:
        for r in sorted(ranked[1:], key=lambda r: r[1]):
            if r[0] == 0 and r[1] == head[-1][2]:
                head.append(r)
        for r in sorted(ranked[1:], key=lambda r: -r[1]):
            if r[0] == 0 and r[2] == head[0][1]:
                head.insert(0, r)
    # K rotation: this GPU stores global k at buffer position (k - rot) % K with rot = the
    # head's first K, so the head sits at [0, h) and everything after it is ONE contiguous
    # range -- the remaining panels merge into as few runs (launches) as adjacency allows
    # (the K order of a product's terms is free).  Panels never wrap: rot is a cut.
    rot = head[0][1]
    rp = lambda r: (r[0], (r[1] - rot) % K, (r[1] - rot) % K + (r[2] - r[1]), r[3], r[4])  # noqa: E731
    head = [rp(r) for r in head]
    ranked = [rp(r) for r in ranked]
    runs = []
    for r in sorted((r for r in ranked if r not in head), key=lambda r: r[1]):
        if runs and runs[-1][-1][2] == r[1]:
            runs[-1].append(r)
        else:
            runs.append([r])
    runs.sort(key=lambda run: (sum(r[0] for r in run), run[0][1]))
    runs.insert(0, head)
    def cut(extent):
        nb = -(-extent // block)
        n = max(1, min(a_chunks, nb))
        out = [(min(extent, nb * c // n * block), min(extent, nb * (c + 1) // n * block))
               for c in range(n)]
        return [(a, b) for a, b in out if b > a]

    chunks = cut(mr)        # A-row chunks (C rows) of runs that pull A
    col_chunks = cut(nc)    # B-row chunks (C columns) of runs that pull only B
    n_streams = copy_streams if any(r[0] for r in ranked) else 0
    pulls, gemms = [], []
    rr = 0

    def pull(name, q, row0, rows, k0, k1):
        nonlocal rr
        idx = []
        pieces = min(n_streams, max(1, rows // block))
        for i in range(pieces):
            a = row0 + rows * i // pieces
            b = row0 + rows * (i + 1) // pieces
            pulls.append((name, q, a, b - a, k0, k1, rr % n_streams))
            idx.append(len(pulls) - 1)
            rr += 1
        return idx

    # a run is chunked only when its pulls may still be in flight when it starts:
    # every pull is issued at the step's start, so compare the bytes pulled up to and
    # including this run (at a conservative 500 GB/s) with the GEMM time ahead of it
    # (at 1.2 PFLOP/s); a run whose operands surely landed runs as one launch
    pulled_bytes, prior_flops = 0, 0
    first = True
    for run in runs:
        k0, k1 = run[0][1], run[-1][2]
        a_remote = any(a_src != me for _, _, _, a_src, _ in run)
        b_remote = any(b_src != me for _, _, _, _, b_src in run)
        pulled_bytes += 2 * sum(r[0] for r in run)
        landed = pulled_bytes / 500e9 < prior_flops / 1.2e15
        prior_flops += 2 * mr * nc * (k1 - k0)
        if landed and (a_remote or b_remote):
            evs = [i for _, p0, p1, a_src, b_src in run
                   for i in ((pull("Bt", b_src, 0, nc, p0, p1) if b_src != me else []) +
                             (pull("A", a_src, 0, mr, p0, p1) if a_src != me else []))]
            gemms.append((0, mr, k0, k1, not first, evs, 0, nc))
            first = False
            continue
        if b_remote and not a_remote:
            # only B arrives over NVLink: chunk the run along C's columns, so the GEMM
            # of column chunk c starts once that chunk's B rows landed (not all of B)
            for c0, c1 in col_chunks:
                b_evs = [i for _, p0, p1, _, b_src in run if b_src != me
                         for i in pull("Bt", b_src, c0, c1 - c0, p0, p1)]
                gemms.append((0, mr, k0, k1, not first, b_evs, c0, c1))
            first = False
            continue
        b_evs = [i for _, p0, p1, _, b_src in run if b_src != me
                 for i in pull("Bt", b_src, 0, nc, p0, p1)]
        for r0, r1 in (chunks if a_remote else [(0, mr)]):
            a_evs = [i for _, p0, p1, a_src, _ in run if a_src != me
                     for i in pull("A", a_src, r0, r1 - r0, p0, p1)]
            gemms.append((r0, r1, k0, k1, not first, b_evs + a_evs, 0, nc))
            b_evs = []  # later chunks of this run follow the first on one stream
        first = False
    ranked = [r for run in runs for r in run]
    return PanelPlan([((k0 + rot) % K, (k0 + rot) % K + (k1 - k0), a, b)
                      for _, k0, k1, a, b in ranked], chunks, pulls, gemms, n_streams, rot)


def rotated_segments(k0: int, k1: int, rot: int, K: int) -> list:
    """Global K range [k0, k1) -> [(buffer position, global k, length)] in a buffer rotated
    by `rot` (1 piece, or 2 when the range crosses the rotation point)."""
    p0 = (k0 - rot) % K
    n = k1 - k0
    if p0 + n <= K:
        return [(p0, k0, n)]
    first = K - p0
    return [(p0, k0, first), (0, k0 + first, n - first)]


class MappedGemm:
    """One GPU's share of a mapped SUMMA multiply (see module docstring)."""

    def __init__(self, M: int, N: int, K: int, *, mapping: str = "decompose", rank: int = 0,
                 world: int = 1, group=None, block: int = 128, a_chunks: int = 4,
                 seed: int = 0, out_dtype=None, copy_streams: int = 1):
        torch = native.require_cuda()
        from ..gemm import tile_gemm  # noqa: F401  (fail early if the library is missing)
        from ..ownership import partition
        from ..peer import PeerBuffers

        self.M, self.N, self.K = M, N, K
        self.rank, self.world, self.mapping = rank, world, mapping
        self.device = torch.device("cuda", torch.cuda.current_device())
        nbi, nbj = -(-M // block), -(-N // block)
        # 1-2: map the C block launch with the Mapple program (K1) and take
        # the per-GPU ownership lists (K2)
        self.mapper = tile_mapper(world, mapping)
        owners = self.mapper.map_ispace((nbi, nbj))
        own = partition(owners, world)
        self.block_counts = own.counts.tolist()
        self.owner_table = owners.tolist()
        self.layout = summa_layout(
            rectangles(self.owner_table, nbi, nbj, world, block, block, M, N), K)
        rc = self.layout.rects[rank]
        self.rows, self.cols = (rc.r0, rc.r1), (rc.c0, rc.c1)
        mr, nc = rc.r1 - rc.r0, rc.c1 - rc.c0
        # 3: operand buffers with full K, K-rotated per GPU (plan_panels: global k at
        # (k - rot) % K); this GPU's own slices live in place
        mrs = [(r.r1 - r.r0, r.c1 - r.c0) for r in self.layout.rects]
        self.rots = [plan_panels(self.layout, q, K, mrs[q][0], mrs[q][1], block, a_chunks,
                                 copy_streams).rot for q in range(world)]
        rot = self.rots[rank]
        self.A = torch.empty(mr, K, dtype=torch.bfloat16, device=self.device)
        self.Bt = torch.empty(nc, K, dtype=torch.bfloat16, device=self.device)
        self.C = torch.empty(mr, nc, dtype=out_dtype or torch.float32, device=self.device)
        ka, kb = self.layout.a_slice[rank], self.layout.b_slice[rank]
        # own slices as (buffer position, global k, length) pieces
        self.own_a = rotated_segments(ka[0], ka[1], rot, K)
        self.own_b = rotated_segments(kb[0], kb[1], rot, K)
        for p0, k0, n in self.own_a:
            self.A[:, p0:p0 + n] = synth(self.rows, (k0, k0 + n), K, seed, self.device)
        for p0, k0, n in self.own_b:
            self.Bt[:, p0:p0 + n] = synth(self.cols, (k0, k0 + n), K, seed + 1, self.device)
        # the own slices are complete before any peer can learn their address (the
        # handle exchange is collective): a peer's first pull never reads them early
        torch.cuda.synchronize(self.device)
        self.peers = PeerBuffers({"A": self.A, "Bt": self.Bt}, rank, world, group)
        self._plan(block, a_chunks, copy_streams)
        self.done = torch.cuda.Event()
        self.done.record()
        self.recv_bytes = comm_bytes(self.layout, K)[rank]
        self.flops = 2 * mr * nc * K
        self.gemm_launches = len(self.gemms)

    # -- schedule (built once) -------------------------------------------------------

    def _plan(self, block, a_chunks, copy_streams):
        """Bind the pure schedule (`plan_panels`) to CUDA streams and events."""
        torch = native.require_cuda()
        mr, nc = self.rows[1] - self.rows[0], self.cols[1] - self.cols[0]
        plan = plan_panels(self.layout, self.rank, self.K, mr, nc, block, a_chunks, copy_streams)
        self.copy_streams = [torch.cuda.Stream(device=self.device)
                             for _ in range(plan.n_streams)]
        events = [torch.cuda.Event() for _ in plan.pulls]
        self.pulls = [p + (events[i],) for i, p in enumerate(plan.pulls)]
        self.gemms = [(r0, r1, k0, k1, acc, [events[i] for i in evs], c0, c1)
                      for r0, r1, k0, k1, acc, evs, c0, c1 in plan.gemms]
        self.panels = plan.panels
        self.chunks = plan.chunks

    # -- one multiply ---------------------------------------------------------------

    def _pieces(self, q, k0, k1):
        """A pull of my buffer positions [k0, k1) (one panel: a global K range that does not
        wrap) from GPU q, which stores global k at its own rotation: [(my position, q's
        position, length)], 1 piece or 2 when the range crosses q's rotation point."""
        K, rm = self.K, self.rots[self.rank]
        g0 = (k0 + rm) % K
        if g0 + (k1 - k0) > K:
            raise AssertionError("a pulled panel crossed the end of K")
        return [((gk - rm) % K, pq, n)
                for pq, gk, n in rotated_segments(g0, g0 + (k1 - k0), self.rots[q], K)]

    def _copy(self, name, q, row0, nrows, k0, k1, stream):
        from ..peer import copy2d

        esz = 2
        pitch = self.K * esz
        for pm, pq, n in self._pieces(q, k0, k1):
            src = self.peers.ptrs[name][q] + (row0 * self.K + pq) * esz
            dst = self.peers.ptrs[name][self.rank] + (row0 * self.K + pm) * esz
            copy2d(dst, pitch, src, pitch, n * esz, nrows, stream)

    def _program(self):
        """The step as a StepProgram (csrc/steps.cpp): the same pulls on the same copy
        lanes, waits and GEMM launches as step_python, replayed by one C call.  Bound
        to the current A / Bt / C tensors (cached per binding)."""
        from ..peer import StepProgram

        key = (self.A.data_ptr(), self.Bt.data_ptr(), self.C.data_ptr())
        progs = self.__dict__.setdefault("_programs", {})
        prog = progs.get(key)
        if prog is not None:
            return prog
        prog = StepProgram()
        esz, K = 2, self.K
        pitch = K * esz
        at = {}
        for i, (name, q, row0, rows, k0, k1, si, _ev) in enumerate(self.pulls):
            at[i] = []
            for pm, pq, n in self._pieces(q, k0, k1):
                src = self.peers.ptrs[name][q] + (row0 * K + pq) * esz
                dst = (self.A if name == "A" else self.Bt).data_ptr() + (row0 * K + pm) * esz
                at[i].append(prog.pull(dst, pitch, src, pitch, n * esz, rows, lane=si % 4))
        ev_index = {id(p[-1]): i for i, p in enumerate(self.pulls)}
        c_bf16 = int(self.C.dtype != native.require_cuda().float32)
        csz = self.C.element_size()
        nc = self.C.shape[1]
        for r0, r1, k0, k1, acc, evs, c0, c1 in self.gemms:
            for ev in evs:
                for a in at[ev_index[id(ev)]]:
                    prog.wait(a)
            prog.gemm_bf16(self.A.data_ptr() + (r0 * K + k0) * esz, K,
                           self.Bt.data_ptr() + (c0 * K + k0) * esz, K,
                           self.C.data_ptr() + (r0 * nc + c0) * csz, nc, r1 - r0, c1 - c0,
                           k1 - k0, c_bf16, int(acc))
        progs[key] = prog.build()
        return prog

    def step(self, stream=None, ready=None):
        """One full multiply, stream-ordered (no host synchronisation), as one
        step-program call.  `ready`: an optional event the pulls also wait for (e.g.
        every GPU's operands landed)."""
        torch = native.require_cuda()
        cs = stream or torch.cuda.current_stream()
        if ready is not None:
            cs.wait_event(ready)  # the lanes fork from cs after it
        self._program().run(cs)
        self.done.record(cs)
        return self.C

    def step_python(self, stream=None, ready=None):
        """The same multiply issued op by op from Python (tile_gemm per launch, e.g.
        for per-launch timing)."""
        torch = native.require_cuda()
        from ..gemm import tile_gemm

        cs = stream or torch.cuda.current_stream()
        for s in self.copy_streams:
            s.wait_event(self.done)  # the previous multiply no longer reads A / Bt
            if ready is not None:
                s.wait_event(ready)
        if ready is not None:
            cs.wait_event(ready)
        for name, q, row0, rows, k0, k1, si, ev in self.pulls:
            s = self.copy_streams[si]
            self._copy(name, q, row0, rows, k0, k1, s)
            ev.record(s)
        for r0, r1, k0, k1, acc, evs, c0, c1 in self.gemms:
            for ev in evs:
                cs.wait_event(ev)
            tile_gemm(self.A[r0:r1, k0:k1], self.Bt[c0:c1, k0:k1], self.C[r0:r1, c0:c1],
                      accumulate=acc, stream=cs)
        self.done.record(cs)
        return self.C

    def close(self):
        for prog in self.__dict__.get("_programs", {}).values():
            prog.close()
        self.peers.close()
