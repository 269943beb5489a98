"""Mapped 2-D 5-point Jacobi stencil with NVLink halo exchange (BASELINE
configs[4]; the paper's stencil workload).

Planning: the cell launch (rows x cols points) is mapped onto the GPUs by a
Mapple block mapper -- `decompose` (m.merge(0,1).decompose(0, ispace)) or the
Algorithm-1 heuristic (m.merge(0,1).split(0, g0)), SURVEY F5 -- with K1; K2
gives every GPU's cell count and K3 the halo transfer lists, whose total is
the reference's `surface_volume` / `oracle_boundary_count`
(commvol.py:94-96,136-168).  The owner table must be a 2-D block grid; each
GPU keeps its rectangle in three rotating fp32 buffers.

Execution: K5 (csrc/stencil.cu) sweeps the rectangle; cells outside it are read
directly from the neighbours' buffers over NVLink, ordered by sweep-done flags
the GPUs push into each other's memory -- one kernel per sweep, no halo
copies, no collectives, no host synchronisation.
"""

from __future__ import annotations

import ctypes

from .. import native
from ..commvol import BlockGrid, surface_volume
from ..dsl import compile_mapper, parse
from ..factorize import greedy_grid, search_optimal
from ..spaces import MachineShape

STENCIL_MAPPERS = """
m = Machine(GPU)
def stencil_decompose(Tuple p, Tuple s):
    q = m.merge(0, 1).decompose(0, s)
    return q[*(p * q.size / s)]
def stencil_heuristic(Tuple p, Tuple s):
    q = m.merge(0, 1).split(0, {g0})
    return q[*(p * q.size / s)]
IndexTaskMap stencil_decompose stencil_decompose
IndexTaskMap stencil_heuristic stencil_heuristic
"""


class PmStencilView(ctypes.Structure):
    _fields_ = [("out", ctypes.c_void_p), ("in_", ctypes.c_void_p),
                ("rows", ctypes.c_int64), ("cols", ctypes.c_int64), ("pitch", ctypes.c_int64),
                ("grow0", ctypes.c_int64), ("gcol0", ctypes.c_int64),
                ("grows", ctypes.c_int64), ("gcols", ctypes.c_int64),
                ("nbr", ctypes.c_void_p * 4), ("nbr_pitch", ctypes.c_int64 * 4),
                ("nbr_rows", ctypes.c_int64 * 4), ("nbr_cols", ctypes.c_int64 * 4),
                ("my_flags", ctypes.c_void_p), ("nbr_flag_slot", ctypes.c_void_p * 4),
                ("nbr_rank", ctypes.c_int32 * 4), ("ticket", ctypes.c_void_p),
                ("col_out", ctypes.c_void_p * 2), ("nbr_col", ctypes.c_void_p * 2)]


def stencil_mapper(world: int, mapping: str):
    g0 = greedy_grid(world, 2)[0]
    return compile_mapper(parse(STENCIL_MAPPERS.format(g0=g0)), f"stencil_{mapping}",
                          MachineShape("GPU", 1, world))


def grid_for(world, rows, cols, mapping):
    return tuple(search_optimal(world, (rows, cols))[0]) if mapping == "decompose" \
        else tuple(greedy_grid(world, 2))


def rectangles_from_owner(ids, rows: int, cols: int, world: int, counts):
    """Per GPU (r0, r1, c0, c1) from a device owner table; checks block shape."""
    torch = native.require_cuda()
    t = ids.view(rows, cols)
    rects = []
    for r in range(world):
        rr = (t == r).any(dim=1).nonzero().flatten()
        cc = (t == r).any(dim=0).nonzero().flatten()
        if rr.numel() == 0:
            raise ValueError(f"GPU {r} owns no cells")
        r0, r1 = int(rr[0]), int(rr[-1]) + 1
        c0, c1 = int(cc[0]), int(cc[-1]) + 1
        if (r1 - r0) * (c1 - c0) != counts[r]:
            raise ValueError(f"GPU {r}'s cells are not a rectangle: not a block mapping")
        rects.append((r0, r1, c0, c1))
    del torch
    return rects


def block_neighbors(rects, rank: int, rows: int, cols: int) -> list:
    """[up, down, left, right] neighbour ranks of a 2-D block grid (None at the
    global boundary); raises unless every internal edge has exactly one owner."""
    r0, r1, c0, c1 = rects[rank]
    nbrs = [None] * 4
    for q, (q0, q1, p0, p1) in enumerate(rects):
        if q == rank:
            continue
        if (p0, p1) == (c0, c1) and q1 == r0:
            nbrs[0] = q
        elif (p0, p1) == (c0, c1) and q0 == r1:
            nbrs[1] = q
        elif (q0, q1) == (r0, r1) and p1 == c0:
            nbrs[2] = q
        elif (q0, q1) == (r0, r1) and p0 == c1:
            nbrs[3] = q
    for d, (lo, hi) in enumerate(((r0, 0), (r1, rows), (c0, 0), (c1, cols))):
        if lo != hi and nbrs[d] is None:
            raise ValueError("the mapping is not a 2-D block grid (missing neighbour)")
    return nbrs


def init_grid(rows: tuple, cols: tuple, ld: int, seed: int, device):
    """Deterministic U(0, 1) fp32 block of a virtual [*, ld] grid."""
    torch = native.require_cuda()
    i = torch.arange(rows[0], rows[1], device=device, dtype=torch.int64).view(-1, 1)
    k = torch.arange(cols[0], cols[1], device=device, dtype=torch.int64).view(1, -1)
    x = (i * ld + k) % (1 << 31)
    x = (x * 1103515245 + 12345 + seed * 7919) % (1 << 31)
    x = x ^ (x >> 13)
    x = (x * 69069 + 1) % (1 << 31)
    return x.to(torch.float32) / float(1 << 31)


class MappedStencil:
    def __init__(self, rows: int, cols: int, *, mapping="decompose", rank=0, world=1, group=None,
                 seed=0, halo_check=True):
        torch = native.require_cuda()
        import torch.distributed as dist

        from ..ownership import partition
        from ..peer import PeerBuffers
        from ..transfer import halo_lists

        self.rows, self.cols, self.rank, self.world = rows, cols, rank, world
        self.device = torch.device("cuda", torch.cuda.current_device())
        self.mapping = mapping
        fn = stencil_mapper(world, mapping)
        ids = fn.map_ispace((rows, cols))                      # K1 over every cell
        own = partition(ids, world)                            # K2
        counts = own.counts.tolist()
        self.rects = rectangles_from_owner(ids, rows, cols, world, counts)
        if halo_check:                                         # K3: send lists' total
            tl = halo_lists(ids, (rows, cols), (1, 1), world, counts_only=True)
            self.halo_cells = tl.total
        else:
            self.halo_cells = None
        self.grid = grid_for(world, rows, cols, mapping)
        self.model_halo = int(surface_volume(BlockGrid((rows, cols), self.grid)))
        del ids, own
        torch.cuda.empty_cache()
        r0, r1, c0, c1 = self.rects[rank]
        self.mr, self.mc = r1 - r0, c1 - c0
        self.pitch = (self.mc + 3) // 4 * 4
        self.buf = [torch.zeros(self.mr, self.pitch, dtype=torch.float32, device=self.device)
                    for _ in range(3)]
        self.buf[0][:, :self.mc] = init_grid((r0, r1), (c0, c1), cols, seed, self.device)
        # column strips per buffer: [0] my first column, [1] my last column, contiguous
        # (the left / right neighbours read them with 16-byte NVLink loads)
        rp = (self.mr + 3) // 4 * 4
        self.strips = [torch.zeros(2, rp, dtype=torch.float32, device=self.device)
                       for _ in range(3)]
        self.strips[0][0, :self.mr] = self.buf[0][:, 0]
        self.strips[0][1, :self.mr] = self.buf[0][:, self.mc - 1]
        self.flags = torch.zeros(max(world, 1), dtype=torch.int32, device=self.device)
        self.ticket = torch.zeros(1, dtype=torch.int32, device=self.device)
        names = {f"b{i}": b for i, b in enumerate(self.buf)}
        names.update({f"s{i}": t for i, t in enumerate(self.strips)})
        names["flags"] = self.flags
        self.peers = PeerBuffers(names, rank, world, group)
        self.nbrs = block_neighbors(self.rects, rank, rows, cols)
        self.sweep = 0
        self.torch = torch
        self._dist = dist if world > 1 else None
        self.group = group
        torch.cuda.synchronize()
        if self._dist:
            dist.barrier(group=group)

    def _view(self, s: int) -> PmStencilView:
        v = PmStencilView()
        r0, r1, c0, c1 = self.rects[self.rank]
        v.out = self.buf[(s + 1) % 3].data_ptr()
        v.in_ = self.buf[s % 3].data_ptr()
        v.rows, v.cols, v.pitch = self.mr, self.mc, self.pitch
        v.grow0, v.gcol0, v.grows, v.gcols = r0, c0, self.rows, self.cols
        v.my_flags = self.flags.data_ptr()
        v.ticket = self.ticket.data_ptr()
        out_strip = self.strips[(s + 1) % 3]
        v.col_out[0], v.col_out[1] = out_strip[0].data_ptr(), out_strip[1].data_ptr()
        rp4 = 4 * self.strips[0].shape[1]  # bytes per strip row of the 2 x rp tensor
        for side, d in ((0, 2), (1, 3)):  # the left neighbour's last / right's first column
            q = self.nbrs[d]
            v.nbr_col[side] = None if q is None else \
                self.peers.ptrs[f"s{s % 3}"][q] + (rp4 if side == 0 else 0)
        for d, q in enumerate(self.nbrs):
            if q is None:
                v.nbr[d] = None
                continue
            q0, q1, p0, p1 = self.rects[q]
            v.nbr[d] = self.peers.ptrs[f"b{s % 3}"][q]
            v.nbr_pitch[d] = (p1 - p0 + 3) // 4 * 4
            v.nbr_rows[d], v.nbr_cols[d] = q1 - q0, p1 - p0
            v.nbr_flag_slot[d] = self.peers.ptrs["flags"][q] + 4 * self.rank
            v.nbr_rank[d] = q
        return v

    def run(self, sweeps: int, stream=None):
        """`sweeps` Jacobi sweeps, stream-ordered; returns this GPU's current block."""
        lib = native.lib()
        sp = native.stream_ptr(stream)
        if not hasattr(self, "_views"):  # the three buffer rotations, built once
            self._views = [ctypes.byref(self._keep(self._view(s))) for s in range(3)]
        fn = lib.pm_stencil_sweep
        for _ in range(sweeps):
            rc = fn(self._views[self.sweep % 3], self.sweep, sp)
            if rc:
                native.check(rc, "pm_stencil_sweep")
            self.sweep += 1
        return self.current()

    def _keep(self, v):
        self.__dict__.setdefault("_view_objs", []).append(v)
        return v

    def current(self):
        return self.buf[self.sweep % 3][:, :self.mc]

    def close(self):
        self.peers.close()
