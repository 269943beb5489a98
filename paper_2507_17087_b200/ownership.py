"""Ownership lists of an index launch on the GPU (K2).

`partition(proc_ids, nprocs)` is the stable partition of launch points by
processor: per processor, the points it owns in launch order.  That is the
shard tree of the reference's SHARD rule (reference: tasksim/sim.py:67-120,
`shard_policy` / `expand_shards`): with the D distinct targets sorted, leaf k
is `task + "/1" * k + "/0"` and the last leaf is `task + "/1" * (D - 1)`; the
enqueue node is the node of the smallest target (sim.py:204).  `proc_counts`
follows cli.py:154-164.
"""

from __future__ import annotations

from dataclasses import dataclass

from . import native
from .errors import ProcMapError


@dataclass
class Ownership:
    counts: "torch.Tensor"    # int64 [nprocs]
    offsets: "torch.Tensor"   # int64 [nprocs]
    perm: "torch.Tensor"      # int32 [n] point indices grouped by processor

    def points_of(self, proc: int):
        o, c = int(self.offsets[proc]), int(self.counts[proc])
        return self.perm[o:o + c]


def partition(proc_ids, nprocs: int, *, stream=None, check: bool = True) -> Ownership:
    """Stable partition of int32 processor ids (CUDA tensor) into nprocs bins."""
    torch = native.require_cuda()
    if proc_ids.dtype != torch.int32 or not proc_ids.is_cuda:
        raise ValueError("proc_ids must be an int32 CUDA tensor")
    ids = proc_ids.contiguous().view(-1)
    n = ids.numel()
    dev = ids.device
    counts = torch.empty(nprocs, dtype=torch.int64, device=dev)
    offsets = torch.empty(nprocs, dtype=torch.int64, device=dev)
    perm = torch.empty(max(n, 1), dtype=torch.int32, device=dev)
    bad = torch.empty(1, dtype=torch.int64, device=dev)
    lib = native.lib()
    nbytes = lib.pm_partition_scratch_bytes(n, nprocs)
    scratch = torch.empty(nbytes, dtype=torch.uint8, device=dev)
    with torch.cuda.device(dev):
        native.check(lib.pm_partition(ids.data_ptr() if n else 0, n, nprocs, counts.data_ptr(),
                                      offsets.data_ptr(), perm.data_ptr(), bad.data_ptr(),
                                      scratch.data_ptr(), nbytes, native.stream_ptr(stream)),
                     "pm_partition")
    if check:
        b = int(bad.item())
        if b >= 0:
            raise ProcMapError(f"point {b} has processor id {int(ids[b])} outside [0, {nprocs})")
    return Ownership(counts, offsets, perm[:n])


def proc_counts(own: Ownership, procs_per_node: int) -> list[dict]:
    """[{node, proc, points}] sorted by (node, proc), non-empty only (cli.py:162-164)."""
    out = []
    for pid, c in enumerate(own.counts.tolist()):
        if c:
            node, proc = divmod(pid, procs_per_node)
            out.append({"node": node, "proc": proc, "points": c})
    return out


def shard_leaves(task: str, own: Ownership, procs_per_node: int) -> list[tuple[str, tuple, object]]:
    """(leaf id, (node, proc), point-index tensor) per leaf, in leaf-id order."""
    targets = [pid for pid, c in enumerate(own.counts.tolist()) if c]
    leaves = []
    for k, pid in enumerate(targets):
        if len(targets) == 1:
            leaf = task
        elif k < len(targets) - 1:
            leaf = task + "/1" * k + "/0"
        else:
            leaf = task + "/1" * k
        leaves.append((leaf, divmod(pid, procs_per_node), own.points_of(pid)))
    return sorted(leaves, key=lambda t: t[0])
