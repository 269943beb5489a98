"""Halo transfer lists of a cell-owned grid on the GPU (K3).

Given the owner (processor id) of every cell of a 1-3D grid -- typically the
output of `MappingFunction.map_ispace` over the grid's cells -- builds, for
every ordered processor pair (src, dst), the cells src must send to dst for
a halo of width h_n along each dimension.  For block partitions the totals
equal the reference's ground-truth count `oracle_boundary_count`
(reference: commvol.py:136-168) and `surface_volume` (commvol.py:94-96) for
h = 1; tests/test_gpu_halo.py holds the kernel to both.  Built by compaction:
count entries per tile, compact them in slot order, group them by pair with
K2 (csrc/halo.cu).
"""

from __future__ import annotations

import ctypes
from dataclasses import dataclass

from . import native
from .ownership import partition


@dataclass
class TransferLists:
    nprocs: int
    pair_counts: "torch.Tensor"   # int64 [nprocs * nprocs], key = src * nprocs + dst
    pair_offsets: "torch.Tensor"  # int64 [nprocs * nprocs]
    cells: "torch.Tensor | None"  # int64 linear cell index, grouped by key, ascending
    dims: "torch.Tensor | None"   # int8 2 * dim + (direction > 0)

    @property
    def total(self) -> int:
        return int(self.pair_counts.sum())

    def send_list(self, src: int, dst: int):
        k = src * self.nprocs + dst
        o, c = int(self.pair_offsets[k]), int(self.pair_counts[k])
        return self.cells[o:o + c], self.dims[o:o + c]


def halo_lists(owner, extents, halo, nprocs: int, *, counts_only: bool = False,
               stream=None) -> TransferLists:
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
    tbytes = lib.pm_halo_tile_scratch_bytes(ext_c, rank)
    tiles = torch.empty(tbytes, dtype=torch.uint8, device=dev)
    with torch.cuda.device(dev):
        s = native.stream_ptr(stream)
        # 1. per-tile entry counts (-> output offsets) and per-pair totals
        native.check(lib.pm_halo_count(owner.data_ptr(), ext_c, rank, halo_c, nprocs,
                                       counts.data_ptr(), tiles.data_ptr(), tbytes, s),
                     "pm_halo_count")
        if counts_only:
            offsets = torch.cumsum(counts, 0) - counts
            return TransferLists(nprocs, counts, offsets, None, None)
        total = int(counts.sum())
        # 2. compaction of the entries in slot order
        keys = torch.empty(max(total, 1), dtype=torch.int32, device=dev)
        slots = torch.empty(max(total, 1), dtype=torch.int64, device=dev)
        native.check(lib.pm_halo_compact(owner.data_ptr(), ext_c, rank, halo_c, nprocs,
                                         tiles.data_ptr(), keys.data_ptr(), slots.data_ptr(), s),
                     "pm_halo_compact")
        # 3. stable grouping by (src, dst) pair (K2) and the (cell, dim) lists
        own = partition(keys[:total], pairs, stream=stream, check=False)
        cells = torch.empty(max(total, 1), dtype=torch.int64, device=dev)
        dims = torch.empty(max(total, 1), dtype=torch.int8, device=dev)
        native.check(lib.pm_halo_gather(own.perm.data_ptr() if total else None,
                                        slots.data_ptr(), total, rank, cells.data_ptr(),
                                        dims.data_ptr(), s), "pm_halo_gather")
    return TransferLists(nprocs, own.counts, own.offsets, cells[:total], dims[:total])
