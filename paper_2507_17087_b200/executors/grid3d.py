"""Mapped 3-D matmul (Johnson 3D, COSMA; BASELINE configs[2] and [3]) with the
depth reduction fused into the GEMM epilogue over NVLink.

The processor grid (pm, pn, pk) splits M, N and K.  It comes from the
`decompose` optimizer over the matrix extents (search_optimal(G, (M, N, K)),
reference factorize.py:166-188) or from the Algorithm-1 heuristic
(greedy_grid(G, 3), factorize.py:191-206); the grid launch is then mapped
onto the GPUs by a Mapple program (K1) -- the same role the paper's
`johnson_mm` / `cosma_mm` mappers play.

GPU (a, b, c) computes the partial product A[a, c] * B[c, b] over K block c:
  * initial layout (3-D): it holds rows-part b of A[a, c] and cols-part a of
    B[c, b]; the rest of both blocks is pulled from the peers of its
    n-group / m-group by the copy engines (all-gather, no SMs);
  * reduce-scatter over c: C[a, b] rows are split among the pk GPUs of the
    k-group; the GEMM is launched per destination row range (cut further where
    operands arrive separately, plan_3d) and its
    epilogue reduce-adds the tile straight into the owner's C buffer over
    NVLink (TMA `cp.reduce.async.bulk.tensor .add` on an IPC-mapped pointer) --
    the collective is fused into the GEMM, there is no separate NCCL call.
The launch for this GPU's own rows goes first and overwrites them (plain TMA
stores: C is never zeroed, never read back); one stream-ordered barrier per step
(through peer memory, csrc/barrier.cu -- no NCCL) then lets the peers' launches
reduce-add into them.  C is double-buffered.
"""

from __future__ import annotations

from math import prod

from .. import native
from ..dsl import compile_mapper, parse
from ..factorize import greedy_grid, search_optimal
from ..spaces import MachineShape
from .summa import synth

GRID3D_MAPPER = """
m = Machine(GPU)
def grid3d(Tuple ipoint, Tuple ispace):
    q = m.merge(0, 1).decompose(0, ispace)
    return q[*ipoint]
IndexTaskMap gemm3d grid3d
"""


def grid_for(world: int, M: int, N: int, K: int, mapping: str) -> tuple:
    if mapping == "decompose":
        return tuple(search_optimal(world, (M, N, K))[0])
    if mapping == "heuristic":
        return tuple(greedy_grid(world, 3))
    raise ValueError(mapping)


def split(n: int, parts: int, i: int) -> tuple:
    return (n * i // parts, n * (i + 1) // parts)


def comm_bytes_3d(M, N, K, grid) -> dict:
    """Per-GPU bytes: A/B all-gathers (bf16) and the C reduce-scatter (fp32)."""
    pm, pn, pk = grid
    Mb, Nb, Kb = M / pm, N / pn, K / pk
    a = Mb * Kb * (1 - 1 / pn) * 2
    b = Kb * Nb * (1 - 1 / pm) * 2
    c = Mb * Nb * (1 - 1 / pk) * 4
    return {"a_gather": int(a), "b_gather": int(b), "c_reduce_scatter": int(c),
            "total": int(a + b + c)}


def plan_3d(grid, coord, owner, mb: int, nb: int, a_chunks: int = 4) -> dict:
    """This GPU's step schedule (pure; CPU-testable).

    Pulls: the A row parts of the n-group (each cut into `a_chunks` pieces) and the Bt
    row parts (C columns) of the m-group, issued on ONE copy lane in the order the GEMMs
    need them (peer copies on several lanes ran one lane after another, not at once).
    GEMMs: every destination's rows (own first, then the peers') cut into sub-products
    at the edges of what arrives separately -- A rows at the local part / pull chunks,
    C columns at the Bt parts -- so the first product needs only operands already here
    or the first pull, not the whole all-gather.  Returns {"pulls": [(name, src rank,
    (r0, r1))], "gemms": [(rows, cols, dst rank, dst row0, [pull indices])],
    "barrier_before": index of the first reduce-adding product (or None)}."""
    pm, pn, pk = grid
    a, b, c = coord
    me = owner[(a, b, c)]
    a_parts = []  # (rows, src) ; src None = local
    for b2 in range(pn):
        r = split(mb, pn, b2)
        if b2 == b:
            a_parts.append((r, None))
        else:
            n = max(1, min(a_chunks, (r[1] - r[0]) // 128))
            for i in range(n):
                a_parts.append(((r[0] + (r[1] - r[0]) * i // n, r[0] + (r[1] - r[0]) * (i + 1) // n),
                                owner[(a, b2, c)]))
    b_parts = [(split(nb, pm, a2), None if a2 == a else owner[(a2, b, c)]) for a2 in range(pm)]
    local_first = sorted(range(len(a_parts)), key=lambda i: (a_parts[i][1] is not None, i))
    col_order = sorted(range(len(b_parts)), key=lambda i: (b_parts[i][1] is not None, i))
    pulls, pull_of = [], {}

    def need(kind, i):
        key = (kind, i)
        if key not in pull_of:
            rows, src = (a_parts if kind == "A" else b_parts)[i]
            pull_of[key] = len(pulls)
            pulls.append(("A" if kind == "A" else "Bt", src, rows))
        return pull_of[key]

    gemms, barrier_before = [], None
    for d in [(c + i) % pk for i in range(pk)]:
        R = split(mb, pk, d)
        dst = owner[(a, b, d)]
        if dst != me and barrier_before is None:
            barrier_before = len(gemms)
        for ai in local_first:
            (r0, r1), asrc = a_parts[ai]
            lo, hi = max(r0, R[0]), min(r1, R[1])
            if lo >= hi:
                continue
            for bi in col_order:
                (c0, c1), bsrc = b_parts[bi]
                evs = ([need("A", ai)] if asrc is not None else []) + \
                      ([need("B", bi)] if bsrc is not None else [])
                gemms.append(((lo, hi), (c0, c1), dst, R[0], evs))
    # merge column neighbours that wait for nothing new (fewer launches): a product over
    # local columns right after another over the same rows and local columns
    merged = []
    for g in gemms:
        if merged:
            p = merged[-1]
            if (p[0] == g[0] and p[2] == g[2] and p[1][1] == g[1][0] and
                    set(g[4]) <= set(p[4])):
                merged[-1] = (p[0], (p[1][0], g[1][1]), p[2], p[3], p[4])
                continue
        merged.append(g)
    if barrier_before is not None:
        barrier_before = next(i for i, g in enumerate(merged) if g[2] != me)
    return {"pulls": pulls, "gemms": merged, "barrier_before": barrier_before}


class MappedGemm3D:
    def __init__(self, M, N, K, *, mapping="decompose", rank=0, world=1, group=None, seed=0,
                 grid=None, block=256):
        torch = native.require_cuda()
        import torch.distributed as dist

        from ..peer import PeerBuffers

        self.M, self.N, self.K = M, N, K
        self.rank, self.world, self.group = rank, world, group
        self.grid = tuple(grid) if grid else grid_for(world, M, N, K, mapping)
        if prod(self.grid) != world:
            raise ValueError(f"grid {self.grid} does not cover {world} GPUs")
        pm, pn, pk = self.grid
        self.device = torch.device("cuda", torch.cuda.current_device())
        # map the (pm, pn, pk) launch onto the GPUs with the Mapple program (K1)
        fn = compile_mapper(parse(GRID3D_MAPPER), "gemm3d", MachineShape("GPU", world, 1))
        owners = fn.map_ispace(self.grid).tolist()
        if sorted(owners) != list(range(world)):
            raise ValueError("the grid mapping is not a bijection onto the GPUs")
        self.owner = {}
        for lin, r in enumerate(owners):
            a, rem = divmod(lin, pn * pk)
            b, c = divmod(rem, pk)
            self.owner[(a, b, c)] = r
        self.coord = next(k for k, v in self.owner.items() if v == rank)
        a, b, c = self.coord
        self.rows = split(M, pm, a)
        self.cols = split(N, pn, b)
        self.ks = split(K, pk, c)
        mb, nb, kb = (self.rows[1] - self.rows[0], self.cols[1] - self.cols[0],
                      self.ks[1] - self.ks[0])
        self.mb, self.nb, self.kb = mb, nb, kb
        # A[a, c] (mb x kb) and Bt[b, c] (nb x kb); my parts in place
        self.A = torch.empty(mb, kb, dtype=torch.bfloat16, device=self.device)
        self.Bt = torch.empty(nb, kb, dtype=torch.bfloat16, device=self.device)
        ar = split(mb, pn, b)   # rows of A[a, c] I hold
        bc = split(nb, pm, a)   # rows of Bt[b, c] (columns of B) I hold
        self.A[ar[0]:ar[1]] = synth((self.rows[0] + ar[0], self.rows[0] + ar[1]), self.ks, K,
                                    seed, self.device)
        self.Bt[bc[0]:bc[1]] = synth((self.cols[0] + bc[0], self.cols[0] + bc[1]), self.ks, K,
                                     seed + 1, self.device)
        # C[a, b] rows owned after the reduce-scatter: k-group position c
        self.my_rows = split(mb, pk, c)
        crows = self.my_rows[1] - self.my_rows[0]
        self.C = [torch.zeros(crows, nb, dtype=torch.float32, device=self.device)
                  for _ in range(2)]
        self.peers = PeerBuffers({"A": self.A, "Bt": self.Bt, "C0": self.C[0],
                                  "C1": self.C[1]}, rank, world, group)
        # the schedule: pulls on one copy lane in need order, sub-products that wait
        # only for what they read (plan_3d); the own rows of C first, written with plain
        # (TMA) stores -- they initialise this GPU's rows, so C is never zeroed nor read
        # back -- then, after a barrier, the peers' rows with TMA reduce-adds over NVLink
        self.plan = plan_3d(self.grid, self.coord, self.owner, mb, nb)
        self.pulls = self.plan["pulls"]
        self.gemms = self.plan["gemms"]
        self.done = torch.cuda.Event()
        self.done.record()
        from ..peer import PeerBarrier

        self._bar = PeerBarrier(rank, world, group) if world > 1 else None
        self.step_i = 0
        self.reduce = pk > 1
        self.flops = 2 * mb * nb * kb
        self.gemm_launches = len(self.gemms)
        cb = comm_bytes_3d(M, N, K, self.grid)
        self.recv_bytes = cb["total"]
        self.comm = cb
        self._dist = dist if world > 1 else None
        torch.cuda.synchronize()
        if self._dist:
            dist.barrier(group=group)

    def _barrier(self, stream=None):
        if self._bar is not None:  # stream-ordered: runs after the queued GEMMs
            self._bar(stream)

    def _program(self, buf):
        """One step into C[buf] as a StepProgram (csrc/steps.cpp): the all-gather pulls
        on copy lanes, the compute stream waiting for them, the local-rows GEMM
        (plain stores), a barrier, the peers' rows (TMA reduce-adds over NVLink)."""
        from ..peer import StepProgram

        progs = self.__dict__.setdefault("_programs", {})
        if buf in progs:
            return progs[buf]
        prog = StepProgram()
        at = []
        for name, q, (r0, r1) in self.pulls:
            t = self.A if name == "A" else self.Bt
            pitch = t.shape[1] * 2
            off = r0 * pitch
            at.append(prog.pull(self.peers.ptrs[name][self.rank] + off, pitch,
                                self.peers.ptrs[name][q] + off, pitch, pitch, r1 - r0, lane=0))
        kb, nb = self.kb, self.nb
        for i, ((r0, r1), (c0, c1), dst, d0, evs) in enumerate(self.gemms):
            for e in evs:
                prog.wait(at[e])
            if i == self.plan["barrier_before"] and self._bar is not None:
                prog.barrier(self._bar)  # every GPU has written its own rows of C[buf]
            prog.gemm_bf16(self.A.data_ptr() + r0 * kb * 2, kb,
                           self.Bt.data_ptr() + c0 * kb * 2, kb,
                           self.peers.ptrs[f"C{buf}"][dst] + ((r0 - d0) * nb + c0) * 4, nb,
                           r1 - r0, c1 - c0, kb, 0, 0 if dst == self.rank else 2)
        progs[buf] = prog.build()
        return progs[buf]

    def step(self, stream=None):
        torch = native.require_cuda()
        cs = stream or torch.cuda.current_stream()
        buf = self.step_i % 2
        self.step_i += 1
        # C[buf] was last added into by the peers two steps ago, before each of them
        # joined the previous step's barrier, which we passed: the local GEMM may
        # overwrite it now; the peers add into it only after this step's barrier.
        # C[1-buf] -- the previous step's result -- stays intact during this step.
        self._program(buf).run(cs)
        self.done.record(cs)
        return self.C[buf]

    def result(self):
        """This GPU's rows of C[a, b] after the last step (synchronises the peers)."""
        if self.reduce:
            self._barrier()
        return self.C[(self.step_i - 1) % 2]

    def close(self):
        for prog in self.__dict__.get("_programs", {}).values():
            prog.close()
        if self._bar is not None:
            self._bar.close()
        self.peers.close()
