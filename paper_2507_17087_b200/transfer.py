"""Halo transfer lists of a cell-owned grid on the GPU (K3).

Given the owner (processor id) of every cell of a 1-3D grid -- typically the
output of `MappingFunction.map_ispace` over the grid's cells -- builds, for
every ordered processor pair (src, dst), the cells src must send to dst for
a halo of width h_n along each dimension.  For block partitions the totals
equal the reference's ground-truth count `oracle_boundary_count`
(reference: commvol.py:136-168) and `surface_volume` (commvol.py:94-96) for
h = 1; tests/test_gpu_halo.py holds the kernel to both.  Built by compaction:
count entries per tile (plus a work list of the strips holding entries),
compact them in slot order, group them by pair with the K2 partition writing
the (cell, dim) lists directly (csrc/halo.cu).
"""

from __future__ import annotations

import ctypes
from . import native
from .errors import ProcMapError
from .ownership import partition


class TransferLists:
    """Send lists of every (src, dst) processor pair, grouped by key src * P + dst
    with cells ascending.  The device buffers may be longer than the entry count
    (`capacity` mode); every accessor slices to the device-computed total, which
    is read (one host synchronisation) on first use."""

    def __init__(self, nprocs, pair_counts, pair_offsets, cells, dims, capacity=None,
                 total_dev=None):
        self.nprocs = nprocs
        self._total_dev = total_dev       # device count of every entry (kept or dropped)
        self.pair_counts = pair_counts    # int64 [nprocs * nprocs], key = src * nprocs + dst
        self.pair_offsets = pair_offsets  # int64 [nprocs * nprocs]
        self._cells, self._dims = cells, dims
        self.capacity = capacity
        self._total = None

    @property
    def total(self) -> int:
        if self._total is None:
            self._total = int(self._total_dev if self._total_dev is not None
                              else self.pair_counts.sum())
            if self.capacity is not None and self._total > self.capacity:
                raise ProcMapError(
                    f"halo_lists: {self._total} entries exceed capacity={self.capacity}; "
                    "call again with a larger capacity (or capacity=None to size exactly)")
        return self._total

    @property
    def cells(self):  # int64 linear cell index, grouped by key, ascending
        return None if self._cells is None else self._cells[:self.total]

    @property
    def dims(self):   # int8 2 * dim + (direction > 0)
        return None if self._dims is None else self._dims[:self.total]

    def send_list(self, src: int, dst: int):
        k = src * self.nprocs + dst
        o, c = int(self.pair_offsets[k]), int(self.pair_counts[k])
        return self.cells[o:o + c], self.dims[o:o + c]


class _Workspace:
    """Grow-only device scratch per (device, stream): calls on one stream are
    ordered, so they can share it."""

    def __init__(self):
        self.bufs = {}

    def get(self, torch, name, nbytes, dev):
        b = self.bufs.get(name)
        if b is None or b.numel() < nbytes:
            b = self.bufs[name] = torch.empty(max(nbytes, 256), dtype=torch.uint8, device=dev)
        return b


_workspaces: dict = {}


def halo_lists(owner, extents, halo, nprocs: int, *, counts_only: bool = False,
               capacity: int | None = None, stream=None) -> TransferLists:
    """K3: count pass (+ tile offsets, work list), compaction of the entries in slot
    order, grouping by pair straight into (cell, dim) lists.

    capacity=None sizes the lists exactly (one host synchronisation after the count
    pass).  capacity=N skips it -- the whole call is stream-ordered with no host
    round trip, for pipelines that re-build lists of a known size (e.g. every
    sweep of a stencil whose ownership does not change); the result then holds
    buffers of N entries and raises on first access if the true total exceeded N."""
    torch = native.require_cuda()
    extents = tuple(int(e) for e in extents)
    halo = tuple(int(h) for h in halo)
    if owner.dtype != torch.int32 or not owner.is_cuda:
        raise ValueError("owner must be an int32 CUDA tensor")
    if len(extents) != len(halo) or not 1 <= len(extents) <= 3:
        raise ValueError("rank 1..3 with one halo width per dimension")
    owner = owner.contiguous().view(-1)
    rank = len(extents)
    dev = owner.device
    ext_c = (ctypes.c_int64 * rank)(*extents)
    halo_c = (ctypes.c_int32 * rank)(*halo)
    lib = native.lib()
    pairs = nprocs * nprocs
    counts = torch.empty(pairs, dtype=torch.int64, device=dev)
    s_obj = stream if stream is not None else torch.cuda.current_stream(dev)
    ws = _workspaces.setdefault((dev.index, s_obj.cuda_stream), _Workspace())
    tbytes = lib.pm_halo_tile_scratch_bytes(ext_c, rank)
    tiles = ws.get(torch, "tiles", tbytes, dev)
    if capacity is not None and nprocs > 8:
        capacity = None  # the > 64-pair grouping (K2 + gather) sizes exactly
    with torch.cuda.device(dev):
        s = native.stream_ptr(stream)
        # 1. per-tile entry counts (-> output offsets), per-pair totals, work list
        total_t = torch.empty(1, dtype=torch.int64, device=dev)
        native.check(lib.pm_halo_count(owner.data_ptr(), ext_c, rank, halo_c, nprocs,
                                       counts.data_ptr(), tiles.data_ptr(), tbytes,
                                       total_t.data_ptr(), s), "pm_halo_count")
        if counts_only:
            offsets = torch.cumsum(counts, 0) - counts
            return TransferLists(nprocs, counts, offsets, None, None, total_dev=total_t)
        cap = int(total_t.item()) if capacity is None else int(capacity)
        # 2. compaction of the entries in slot order (entries past cap dropped)
        keys = ws.get(torch, "keys", 4 * max(cap, 1), dev)
        slots = ws.get(torch, "slots", 8 * max(cap, 1), dev)
        native.check(lib.pm_halo_compact(owner.data_ptr(), ext_c, rank, halo_c, nprocs,
                                         tiles.data_ptr(), keys.data_ptr(), slots.data_ptr(), cap,
                                         s), "pm_halo_compact")
        if nprocs > 8:
            # 3'. > 64 pairs: K2 stable partition of the keys, then the (cell, dim) gather
            own = partition(keys.view(torch.int32)[:cap], pairs, stream=stream, check=False)
            cells = torch.empty(max(cap, 1), dtype=torch.int64, device=dev)
            dims = torch.empty(max(cap, 1), dtype=torch.int8, device=dev)
            native.check(lib.pm_halo_gather(own.perm.data_ptr() if cap else None,
                                            slots.data_ptr(), cap, rank, cells.data_ptr(),
                                            dims.data_ptr(), s), "pm_halo_gather")
            out = TransferLists(nprocs, own.counts, own.offsets, cells, dims, total_dev=total_t)
            out._total = cap
            return out
        # 3. stable grouping by (src, dst) pair, writing the (cell, dim) lists directly
        gbytes = lib.pm_halo_group_scratch_bytes(cap, nprocs)
        gscratch = ws.get(torch, "group", gbytes, dev)
        pc = torch.empty(pairs, dtype=torch.int64, device=dev)
        po = torch.empty(pairs, dtype=torch.int64, device=dev)
        cells = torch.empty(max(cap, 1), dtype=torch.int64, device=dev)
        dims = torch.empty(max(cap, 1), dtype=torch.int8, device=dev)
        native.check(lib.pm_halo_group(keys.data_ptr(), slots.data_ptr(), cap, total_t.data_ptr(),
                                       rank, nprocs, pc.data_ptr(), po.data_ptr(),
                                       cells.data_ptr(), dims.data_ptr(), gscratch.data_ptr(),
                                       gscratch.numel(), s), "pm_halo_group")
    out = TransferLists(nprocs, pc, po, cells, dims, capacity=None if capacity is None else cap,
                        total_dev=total_t)
    if capacity is None:
        out._total = cap
    return out
