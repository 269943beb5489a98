"""Mapped Cannon (BASELINE configs[0]) and Solomonik 2.5D (configs[2]).

Grid q x q x c (c = 1: Cannon; c > 1: 2.5D with c replication layers).  The
tile launch is mapped onto the GPUs by a Mapple hierarchical block mapper --
nodes block the tile grid, the processors of a node cycle over it (the paper's
Fig-12 `cannon_mm` / `solomonik_mm` mappers) -- evaluated by
the K1 kernel; the mapping must be a bijection onto the GPUs.

GPU (i, j, l) starts with the 2-D blocks A(i, j) and B(i, j) (replicated on
every layer).  Layer l runs Cannon steps t in [l q/c, (l+1) q/c): it first
skews (A(i, (i+j+t0) mod q) and B((i+j+t0) mod q, j) are pulled from their
holders), then alternates C += A*B with the Cannon shifts (A from the right
neighbour, B from the neighbour below), each a copy-engine pull of the
neighbour's current block over NVLink; a stream-ordered barrier through peer
memory (csrc/barrier.cu, no NCCL) per round orders the shifts.  With
c > 1 every step's product is reduce-added straight into the layer that owns
those rows of C (TMA `.add` over NVLink), i.e. the 2.5D reduction is fused into
the GEMMs.  fp32 operands run on the TF32 tensor cores, bf16 on the bf16 path.
"""

from __future__ import annotations

from math import isqrt

from .. import native
from ..dsl import compile_mapper, parse
from ..spaces import MachineShape
from .summa import synth

HIER_MAPPERS = """
m = Machine(GPU)
def tiles2d(Tuple ipoint, Tuple ispace):
    mn = m.decompose(0, ispace)
    mp = mn.decompose(2, ispace / mn[:-1])
    blk = tuple(ipoint[i] * mp.size[i] / ispace[i] for i in (0, 1))
    cyc = tuple(ipoint[i] % mp.size[i + 2] for i in (0, 1))
    return mp[*blk, *cyc]
def tiles3d(Tuple ipoint, Tuple ispace):
    mn = m.decompose(0, ispace)
    mp = mn.decompose(3, ispace / mn[:-1])
    blk = tuple(ipoint[i] * mp.size[i] / ispace[i] for i in (0, 1, 2))
    cyc = tuple(ipoint[i] % mp.size[i + 3] for i in (0, 1, 2))
    return mp[*blk, *cyc]
IndexTaskMap cannon tiles2d
IndexTaskMap solomonik tiles3d
"""


def cannon_moves(q: int, c: int = 1) -> int:
    """Block moves of the schedule (skew + shifts), A and B, summed over GPUs."""
    moves = 0
    steps = q // c
    for layer in range(c):
        t0 = layer * steps
        for i in range(q):
            for j in range(q):
                moves += (i + t0) % q != 0  # skew: A(i, i+j+t0) held by (i, i+j+t0)
                moves += (j + t0) % q != 0  # skew: B(i+j+t0, j) held by (i+j+t0, j)
        if q > 1:
            moves += (steps - 1) * 2 * q * q  # every shift moves one A and one B per GPU
    return moves


def split(n, parts, i):
    return (n * i // parts, n * (i + 1) // parts)


def cannon_schedule(q: int, c: int, coord):
    """The per-GPU op list of one multiply, shared by the executor and the CPU
    schedule test.  Ops:
      ("pull", src_buffer, src_coord, dst_slot)  -- copy a peer's block into A/B slot
      ("barrier",)                               -- stream-ordered all-GPU barrier
      ("gemm", slot, dst_layer)                  -- C(rows of dst_layer) += A[slot] B[slot]
    src_buffer names "A0"/"B0" (the initial blocks) or "Acur<s>"/"Bcur<s>"
    (a peer's current operand in slot s); dst_slot is (kind, slot)."""
    i, j, l = coord
    steps = q // c
    t0 = l * steps
    k0 = (i + j + t0) % q
    ops = [("barrier",),
           ("pull", "A0", (i, k0, l), ("A", 0)),
           ("pull", "B0", (k0, j, l), ("B", 0)),
           ("barrier",)]
    cur = 0
    for s in range(steps):
        for d in range(c):
            ops.append(("gemm", cur, d))
        if s + 1 < steps:  # Cannon shift: A from the right, B from below
            nxt = 1 - cur
            ops.append(("pull", f"Acur{cur}", (i, (j + 1) % q, l), ("A", nxt)))
            ops.append(("pull", f"Bcur{cur}", ((i + 1) % q, j, l), ("B", nxt)))
            ops.append(("barrier",))
            cur = nxt
    return ops


class MappedCannon:
    def __init__(self, N: int, *, layers: int = 1, rank: int = 0, world: int = 1, group=None,
                 dtype: str = "fp32", machine=None, seed: int = 0, graph: bool = False,
                 program: str | None = None, task: str | None = None):
        torch = native.require_cuda()
        self.graph = graph
        self._graphs = {}
        import torch.distributed as dist

        from ..peer import PeerBuffers

        c = layers
        q = isqrt(world // c)
        if q * q * c != world or q % c:
            raise ValueError(f"{world} GPUs do not form a q x q x c grid with c | q (c={c})")
        if dtype == "fp32" and c > 1:
            raise ValueError("the 2.5D layer reduction adds atomically over NVLink: use bf16")
        self.q, self.c, self.N = q, c, N
        self.rank, self.world, self.group = rank, world, group
        self.dtype = dtype
        tdt = torch.float32 if dtype == "fp32" else torch.bfloat16
        self.device = torch.device("cuda", torch.cuda.current_device())
        # Mapple mapping of the tile launch (K1)
        if machine is None:
            machine = (2, world // 2) if (c == 1 and world % 2 == 0 and world > 2) else (world, 1)
        # any Mapple program with a tile-launch task may place the tiles, e.g. the
        # reference corpus' `cannon_mm` (matmul_mappers.mapper); default: HIER_MAPPERS
        prog = parse(program if program is not None else HIER_MAPPERS)
        if c == 1:
            fn = compile_mapper(prog, task or "cannon", MachineShape("GPU", *machine))
            owners = fn.map_ispace((q, q)).tolist()
            coords = [(i, j, 0) for i in range(q) for j in range(q)]
        else:
            fn = compile_mapper(prog, task or "solomonik", MachineShape("GPU", *machine))
            owners = fn.map_ispace((q, q, c)).tolist()
            coords = [(i, j, l) for i in range(q) for j in range(q) for l in range(c)]
        if sorted(owners) != list(range(world)):
            raise ValueError("the tile mapping is not a bijection onto the GPUs")
        self.machine = machine
        self.owner = {xyz: r for xyz, r in zip(coords, owners)}
        self.coord = next(k for k, v in self.owner.items() if v == rank)
        i, j, l = self.coord
        nb = N // q
        if nb * q != N:
            raise ValueError("N must be divisible by q")
        self.nb = nb
        # operand blocks: cur / next buffers for the shifts; Bt stored transposed
        self.A = [torch.empty(nb, nb, dtype=tdt, device=self.device) for _ in range(2)]
        self.Bt = [torch.empty(nb, nb, dtype=tdt, device=self.device) for _ in range(2)]
        self.A0 = synth((i * nb, (i + 1) * nb), (j * nb, (j + 1) * nb), N, seed,
                        self.device, dtype=tdt)
        # Bt(j-cols, i-k) = B(i-block, j-block)^T
        self.B0 = synth((j * nb, (j + 1) * nb), (i * nb, (i + 1) * nb), N, seed + 1,
                        self.device, dtype=tdt)
        # C rows owned by this layer (reduce-scatter target), double-buffered
        self.my_rows = split(nb, c, l)
        self.C = [torch.zeros(self.my_rows[1] - self.my_rows[0], nb, dtype=torch.float32,
                              device=self.device) for _ in range(2)]
        self.peers = PeerBuffers({"A0": self.A0, "B0": self.B0, "Acur0": self.A[0],
                                  "Acur1": self.A[1], "Bcur0": self.Bt[0], "Bcur1": self.Bt[1],
                                  "C0": self.C[0], "C1": self.C[1]}, rank, world, group)
        from ..peer import PeerBarrier

        self._bar = PeerBarrier(rank, world, group) if world > 1 else None
        # small blocks: the SMs copy a round's blocks and run its barrier in one launch
        # (latency-bound rounds, configs[0]); large ones go to the copy engines
        # (pm_peer_copy_barrier copies 16-byte words: checked once here, so a step can
        # never fail half-way through its schedule and leave the peers in a barrier)
        blk = nb * nb * (4 if dtype == "fp32" else 2)
        ptrs = [p for v in self.peers.ptrs.values() for p in v]
        self._fused_pulls = (blk <= (8 << 20) and blk % 16 == 0 and (nb * (4 if dtype == "fp32"
                             else 2)) % 16 == 0 and all(p % 16 == 0 for p in ptrs))
        self._dist = dist if world > 1 else None
        self.step_i = 0
        self.moved_blocks = 0
        esz = 4 if dtype == "fp32" else 2
        self.block_bytes = nb * nb * esz
        self.flops = 2 * nb * nb * nb * (q // c)
        torch.cuda.synchronize()
        if self._dist:
            dist.barrier(group=group)

    def _barrier(self, stream=None):
        """Stream-ordered all-GPU barrier through peer memory (no NCCL on the path)."""
        if self._bar is not None:
            self._bar(stream)

    def step(self, stream=None):
        """One full multiply (all Cannon / 2.5D steps and the layer reduction).

        With `graph=True` the whole multiply -- pulls, barriers, GEMMs -- is
        captured once per C buffer into a CUDA graph and replayed: the small
        configurations (configs[0], N=1024) are launch-latency bound."""
        torch = native.require_cuda()
        cs = stream or torch.cuda.current_stream()
        buf = self.step_i % 2
        self.step_i += 1
        if not self.graph or self.step_i <= 2:  # the first call per buffer runs eagerly
            self._issue(buf, cs)
            return self.C[buf]
        g = self._graphs.get(buf)
        if g is None:
            g = torch.cuda.CUDAGraph()
            side = torch.cuda.Stream(device=self.device)
            side.wait_stream(cs)
            with torch.cuda.graph(g, stream=side):
                self._issue(buf, side)
            cs.wait_stream(side)
            self._graphs[buf] = g
        with torch.cuda.stream(cs):
            g.replay()
        return self.C[buf]

    def _issue(self, buf, cs):
        """One multiply into C[buf]: its step program (built once per buffer) run on cs."""
        progs = self.__dict__.setdefault("_programs", {})
        if buf not in progs:
            progs[buf] = self._build(buf)
        progs[buf].run(cs)

    def _build(self, buf):
        """The schedule (cannon_schedule) of one multiply into C[buf] as a StepProgram
        (csrc/steps.cpp): SM-copy + barrier launches for small blocks, copy-engine
        pulls + barriers for large ones, TF32 / bf16 GEMMs reduce-added into the
        owning layer."""
        from ..peer import StepProgram

        prog = StepProgram()
        q, c = self.q, self.c
        i, j, l = self.coord
        if c > 1:
            # the layers' adds into C[buf] date from two steps ago and all finished before
            # the previous step's barriers; the schedule's first barrier orders this zeroing
            # before any peer adds into it again
            prog.memset(self.C[buf].data_ptr(), self.C[buf].numel() * 4)
        moved = 0
        first = True  # the first local product overwrites C (Cannon); 2.5D always adds
        pending = []  # a round's pulls, issued with its closing barrier (one launch)
        ops = cannon_schedule(q, c, self.coord)
        if not self._fused_pulls and q > 1:
            # copy engines: a round's shift pulls read the peers' current blocks (valid
            # since the barrier that opened the round) into the other slot (not read by
            # this round's GEMMs) -- hoist them ahead of the GEMMs onto a copy lane so
            # the transfer overlaps the multiply; the round's barrier waits for them
            self._build_overlapped(prog, ops, buf)
            self.moved_blocks = sum(1 for op in ops if op[0] == "pull" and
                                    self.owner[op[2]] != self.rank)
            return prog.build()
        for op in ops:
            if op[0] == "barrier":
                if self._bar is not None and pending and self._fused_pulls:
                    prog.copy_barrier(self._bar, [(d, sp, w * h) for d, sp, w, h in pending])
                else:
                    for d, sp, w, h in pending:  # copy engines, pitched rows, in order
                        prog.pull(d, w, sp, w, w, h, lane=-1)
                    if self._bar is not None:
                        prog.barrier(self._bar)
                pending = []
            elif op[0] == "pull":
                _, name, src, (kind, slot) = op
                if q == 1:  # a 1x1 grid has no shifts: multiply the own blocks in place
                    continue
                dst = self.A[slot] if kind == "A" else self.Bt[slot]
                pending.append((dst.data_ptr(), self.peers.ptrs[name][self.owner[src]],
                                self.nb * dst.element_size(), self.nb))
                moved += self.owner[src] != self.rank
            else:  # C(rows of layer d) += A(i,k) B(k,j), reduce-added into the owning layer
                _, slot, d = op
                r0, r1 = split(self.nb, c, d)
                cptr = self.peers.ptrs[f"C{buf}"][self.owner[(i, j, d)]]
                a_blk, b_blk = (self.A0, self.B0) if q == 1 else (self.A[slot], self.Bt[slot])
                a = a_blk[r0:r1]
                acc = 2 if c > 1 else int(not first)
                if self.dtype == "fp32":
                    prog.gemm_tf32(a.data_ptr(), self.nb, b_blk.data_ptr(), self.nb, cptr,
                                   self.nb, r1 - r0, self.nb, self.nb, acc)
                else:
                    prog.gemm_bf16(a.data_ptr(), self.nb, b_blk.data_ptr(), self.nb, cptr,
                                   self.nb, r1 - r0, self.nb, self.nb, 0, acc)
                first = False
        self.moved_blocks = moved
        return prog.build()

    def _gemm(self, prog, buf, slot, d, first):
        """C(rows of layer d) += A[slot] B[slot], reduce-added into the owning layer."""
        c = self.c
        i, j, _ = self.coord
        r0, r1 = split(self.nb, c, d)
        cptr = self.peers.ptrs[f"C{buf}"][self.owner[(i, j, d)]]
        a_blk, b_blk = self.A[slot], self.Bt[slot]
        acc = 2 if c > 1 else int(not first)
        if self.dtype == "fp32":
            prog.gemm_tf32(a_blk[r0:r1].data_ptr(), self.nb, b_blk.data_ptr(), self.nb, cptr,
                           self.nb, r1 - r0, self.nb, self.nb, acc)
        else:
            prog.gemm_bf16(a_blk[r0:r1].data_ptr(), self.nb, b_blk.data_ptr(), self.nb, cptr,
                           self.nb, r1 - r0, self.nb, self.nb, 0, acc)

    def _build_overlapped(self, prog, ops, buf):
        """Copy-engine schedule with each round's shift pulls overlapping its GEMMs."""
        rounds, cur = [], []
        for op in ops:  # segments between barriers
            if op[0] == "barrier":
                rounds.append(cur)
                cur = []
            else:
                cur.append(op)
        rounds.append(cur)
        first = True
        for n, seg in enumerate(rounds):
            if n:
                if self._bar is not None:
                    prog.barrier(self._bar)
            pulls = [op for op in seg if op[0] == "pull"]
            gemms = [op for op in seg if op[0] == "gemm"]
            at = []
            if pulls:
                prog.fork()  # after the previous round's GEMMs (they read these slots)
                for _, name, src, (kind, slot) in pulls:
                    dst = self.A[slot] if kind == "A" else self.Bt[slot]
                    w = self.nb * dst.element_size()
                    at.append(prog.pull(dst.data_ptr(), w,
                                        self.peers.ptrs[name][self.owner[src]], w, w, self.nb,
                                        lane=0))
            for _, slot, d in gemms:
                self._gemm(prog, buf, slot, d, first)
                first = False
            for a in at:
                prog.wait(a)

    def result(self):
        self._barrier()
        return self.C[(self.step_i - 1) % 2]

    def close(self):
        # captured graphs hold NCCL persistent work: release them before the
        # communicator can be destroyed (destroy_process_group otherwise blocks)
        if self._graphs:
            native.require_cuda().cuda.synchronize()
            self._graphs.clear()
        for prog in self.__dict__.get("_programs", {}).values():
            prog.close()
        if self._bar is not None:
            self._bar.close()
        self.peers.close()
