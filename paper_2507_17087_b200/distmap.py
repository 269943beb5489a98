"""Sharded index-launch mapping across GPUs.

The reference maps a launch point by point on one host thread (cmd_map,
cli.py:149-170) and builds ownership lists by re-mapping every point per shard
level (shard_policy / expand_shards, tasksim/sim.py:67-120).  Points are
independent once the per-ispace prefix is fixed (interp.py:380-418), so here
the row-major point range is cut into `world` contiguous chunks, one per GPU:

  1. K1 maps the chunk (pm_map_batch with `first` = chunk start; no exchange);
  2. K2 stably partitions it by processor (local per-processor counts);
  3. one all-gather of the world x P count matrix gives every GPU the global
     layout: processor p's list is chunk 0's p-points, then chunk 1's, ...
     -- the reference's launch order, i.e. its shard-tree point order;
  4. optionally an all-to-all-v delivers each processor's list to the GPU that
     hosts it (processor p -> rank p * world // P, a monotone block map), so
     every GPU ends up holding exactly the points it executes.

For <= 64 processors steps 1-2 are the fused map + partition kernels
(map_partition.cu): pass 1 histograms the chunk without storing ids, the
counts (and the status word) are all-gathered, and pass 2 writes every point's
global index straight to its final place -- with the exchange, into the list
buffer of the GPU that hosts its processor (NVLink stores through CUDA IPC
pointers), so step 4 costs no extra pass or copy.  Measured at 32768^2 / 8
processors: the exchange is NVLink-bound (each GPU ships (world-1)/world of
its chunk), the non-exchanging layout scales with the GPU count.

A failing point raises on every rank: the 8-byte status words are
min-reduced, so all ranks re-raise the lowest failing point's exception, the
error the reference's row-major loop hits first.
"""

from __future__ import annotations

from dataclasses import dataclass, field

from . import native

_NO_FAIL = (1 << 63) - 1


def chunk(n: int, world: int, rank: int) -> tuple[int, int]:
    """[lo, hi) of rank's contiguous share of n row-major points."""
    return n * rank // world, n * (rank + 1) // world


def host_rank(p: int, nprocs: int, world: int) -> int:
    """GPU that receives processor p's ownership list (monotone in p)."""
    return p * world // nprocs


@dataclass
class ExchangePlan:
    """Sizes of one rank's all-to-all-v and the segment moves that restore
    per-processor launch order on the receiving side (pure host arithmetic)."""
    send_splits: list[int]
    recv_splits: list[int]
    procs: list[int]                       # processors this rank hosts
    lists_offsets: dict[int, int]          # proc -> offset of its list in the result
    lists_counts: dict[int, int]           # proc -> length of its list
    moves: list[tuple[int, int, int]] = field(default_factory=list)  # (src, dst, len)


def exchange_plan(counts_all, rank: int, world: int, nprocs: int) -> ExchangePlan:
    """counts_all[r][p] = #points of chunk r mapped to processor p (host ints)."""
    send = [0] * world
    for p in range(nprocs):
        send[host_rank(p, nprocs, world)] += counts_all[rank][p]
    procs = [p for p in range(nprocs) if host_rank(p, nprocs, world) == rank]
    recv = [sum(counts_all[r][p] for p in procs) for r in range(world)]
    # received buffer: source-major, each source's part grouped by proc ascending
    lists_counts = {p: sum(counts_all[r][p] for r in range(world)) for p in procs}
    lists_offsets, o = {}, 0
    for p in procs:
        lists_offsets[p] = o
        o += lists_counts[p]
    moves, src = [], 0
    fill = dict(lists_offsets)
    for r in range(world):
        for p in procs:
            c = counts_all[r][p]
            if c:
                moves.append((src, fill[p], c))
                fill[p] += c
                src += c
    return ExchangePlan(send, recv, procs, lists_offsets, lists_counts, moves)


def global_layout(counts_all, rank: int):
    """(totals[p], offsets[p], write_at[p]): processor p's global list length,
    its start in the processor-grouped launch order, and where this rank's
    chunk writes its p-points inside it."""
    world, nprocs = len(counts_all), len(counts_all[0])
    totals = [sum(counts_all[r][p] for r in range(world)) for p in range(nprocs)]
    offsets, o = [], 0
    for t in totals:
        offsets.append(o)
        o += t
    write_at = [offsets[p] + sum(counts_all[r][p] for r in range(rank)) for p in range(nprocs)]
    return totals, offsets, write_at


@dataclass
class ShardedOwnership:
    first: int                 # this rank's chunk [first, first + count) of the launch
    count: int
    proc_ids: object           # int32 [count] K1 output of the chunk
    counts_all: list           # world x P host ints
    totals: list               # per processor, whole launch
    offsets: list              # per processor, start in processor-grouped order
    write_at: list             # per processor, where this chunk's points go
    procs: list                # processors hosted by this rank (after exchange)
    lists: dict                # proc -> device tensor of its global point indices

    def points_of(self, proc: int):
        return self.lists[proc]


def _status_min(status, group):
    import torch.distributed as dist

    torch = native.require_cuda()
    s = status.clone()
    s[s == -1] = _NO_FAIL
    dist.all_reduce(s, op=dist.ReduceOp.MIN, group=group)
    s[s == _NO_FAIL] = -1
    return s


def shard_ownership(proc_ids, first: int, nprocs: int, rank: int, world: int, *, group=None,
                    partition_fn=None, exchange: bool = True, index_dtype=None):
    """Steps 2-4 for a chunk whose processor ids are already known.

    `partition_fn(ids, nprocs) -> (counts, perm)` defaults to K2 (the GPU);
    the CPU multi-rank tests pass a host partition to exercise the exchange
    over gloo."""
    import torch
    import torch.distributed as dist

    if partition_fn is None:
        from .ownership import partition

        def partition_fn(ids, P):
            own = partition(ids, P, check=True)
            return own.counts, own.perm

    count = proc_ids.numel()
    counts, perm = partition_fn(proc_ids, nprocs)
    dev = counts.device
    if world > 1:
        gathered = torch.empty(world * nprocs, dtype=torch.int64, device=dev)
        dist.all_gather_into_tensor(gathered, counts.to(torch.int64).contiguous(), group=group)
    else:
        gathered = counts.to(torch.int64)
    counts_all = gathered.view(world, nprocs).cpu().tolist()
    totals, offsets, write_at = global_layout(counts_all, rank)
    idt = index_dtype or (torch.int32 if first + count <= (1 << 31) - 1 and
                          sum(totals) <= (1 << 31) - 1 else torch.int64)
    gidx = perm.to(idt)  # K2's perm is ours: offset it in place
    if first:
        gidx.add_(first)
    lists = {}
    procs = list(range(nprocs))
    if exchange:
        plan = exchange_plan(counts_all, rank, world, nprocs)
        procs = plan.procs
        if world > 1:
            recv = torch.empty(sum(plan.recv_splits), dtype=idt, device=dev)
            dist.all_to_all_single(recv, gidx.contiguous(), plan.recv_splits, plan.send_splits,
                                   group=group)
        else:
            recv = gidx
        if len(plan.procs) == 1 or world == 1:
            merged = recv  # already processor-grouped in launch order
        else:
            merged = torch.empty_like(recv)
            for src, dst, c in plan.moves:
                merged[dst:dst + c].copy_(recv[src:src + c])
        for p in plan.procs:
            o = plan.lists_offsets[p]
            lists[p] = merged[o:o + plan.lists_counts[p]]
    else:
        o = 0
        for p in range(nprocs):
            c = counts_all[rank][p]
            lists[p] = gidx[o:o + c]
            o += c
    return ShardedOwnership(first, count, proc_ids, counts_all, totals, offsets, write_at,
                            procs, lists)


class _Workspace:
    """Grow-only receive buffer of the fused exchange, IPC-shared across the
    group (handles re-exchanged only when some rank's buffer must grow; every
    rank sees the same count matrix, so the decision is collective)."""

    def __init__(self):
        self.cap = 0
        self.buf = None
        self.peers = None

    def ensure(self, need_all, rank, world, group, device):
        torch = native.require_cuda()
        from .peer import PeerBuffers

        need = max(need_all)
        if need <= self.cap and self.buf is not None:
            return
        if self.peers is not None:
            self.peers.close()
        self.cap = max(need, int(self.cap * 1.25), 1024)
        self.buf = torch.empty(self.cap, dtype=torch.int32, device=device)
        self.peers = PeerBuffers({"lists": self.buf}, rank, world, group)


_workspaces: dict = {}


def map_launch_sharded(fn, ispace, *, rank: int = 0, world: int = 1, group=None,
                       exchange: bool = True, fused: bool | None = None,
                       stream=None) -> ShardedOwnership:
    """K1 + K2 over this rank's chunk of the launch, then the count all-gather
    (and the ownership exchange when `exchange`).  `fn` is a MappingFunction
    (compile_mapper); every rank must pass the same mapper and ispace.

    fused (default for <= 64 processors, `exchange` and int32 indices): the
    map + partition kernels of map_partition.cu -- pass 1 histograms the
    chunk, the counts are all-gathered, pass 2 writes every point's global
    index straight into the list buffer of the GPU hosting its processor
    (NVLink stores through CUDA IPC pointers), so no id array, no local
    permutation and no all-to-all copy exist.  The lists then alias a
    per-group workspace: valid until the next fused call on the group.
    Otherwise: K1 (ids) + K2 + NCCL all-to-all-v (shard_ownership)."""
    torch = native.require_cuda()
    import torch.distributed as dist

    if stream is not None and stream != torch.cuda.current_stream():
        # the kernels and the collectives (which join the current stream) on one stream
        with torch.cuda.stream(stream):
            return map_launch_sharded(fn, ispace, rank=rank, world=world, group=group,
                                      exchange=exchange, fused=fused, stream=None)
    ispace = tuple(int(e) for e in ispace)
    n = 1
    for e in ispace:
        n *= max(e, 0)
    lo, hi = chunk(n, world, rank)
    nprocs = fn.machine.nodes * fn.machine.procs_per_node
    if fused is None:
        fused = nprocs <= 64 and n <= (1 << 31) - 1
    if not fused:
        status = torch.full((1,), -1, dtype=torch.int64, device="cuda")
        ids = fn.map_ispace(ispace, lo, hi - lo, status=status, check=False, stream=stream)
        if world > 1:
            status = _status_min(status, group)
        word = int(status.item())
        if word != -1:
            fn.program_for(ispace, implicit=True).raise_for(word)
        return shard_ownership(ids, lo, nprocs, rank, world, group=group, exchange=exchange)
    dev = torch.device("cuda", torch.cuda.current_device())
    pp = fn.program_for(ispace, implicit=True)
    cnt = hi - lo
    # pass 1: histogram of the chunk; the status word rides along with the counts
    packed = torch.empty(nprocs + 1, dtype=torch.int64, device=dev)
    offsets = torch.empty(nprocs, dtype=torch.int64, device=dev)
    packed[nprocs:].fill_(-1)
    nbytes = native.lib().pm_map_partition_scratch_bytes(cnt, nprocs)
    scratch = torch.empty(max(nbytes, 1), dtype=torch.uint8, device=dev)
    status = packed[nprocs:]
    pp.map_hist(None, cnt, lo, nprocs, packed[:nprocs], offsets, status, scratch, stream)
    if world > 1:
        gathered = torch.empty(world * (nprocs + 1), dtype=torch.int64, device=dev)
        dist.all_gather_into_tensor(gathered, packed, group=group)
    else:
        gathered = packed
    rows = gathered.view(world, nprocs + 1).cpu().tolist()
    words = [r[nprocs] for r in rows if r[nprocs] != -1]
    if words:
        pp.raise_for(min(w & ((1 << 64) - 1) for w in words))
    counts_all = [r[:nprocs] for r in rows]
    totals, offs, write_at = global_layout(counts_all, rank)
    if not exchange:  # every GPU keeps its chunk's lists (global indices, write_at known)
        perm = torch.empty(max(cnt, 1), dtype=torch.int32, device=dev)
        pp.map_scatter(None, cnt, lo, nprocs, perm=perm, index_base=lo, status=status,
                       scratch=scratch, stream=stream)
        lists, o = {}, 0
        for p in range(nprocs):
            c = counts_all[rank][p]
            lists[p] = perm[o:o + c]
            o += c
        return ShardedOwnership(lo, cnt, None, counts_all, totals, offs, write_at,
                                list(range(nprocs)), lists)
    plans = [exchange_plan(counts_all, r, world, nprocs) for r in range(world)]
    need_all = [sum(pl.lists_counts.values()) for pl in plans]
    key = (id(group), dev.index)
    ws = _workspaces.get(key)
    if ws is None:
        ws = _workspaces[key] = _Workspace()
    ws.ensure(need_all, rank, world, group, dev)
    # pass 2: processor p's points go to host_rank(p)'s buffer at
    #   lists_offsets[p] + (points of p in lower chunks), relative to our local slot
    local_off = []
    o = 0
    for c in counts_all[rank]:
        local_off.append(o)
        o += c
    tab = []
    for p in range(nprocs):
        h = host_rank(p, nprocs, world)
        below = sum(counts_all[r][p] for r in range(rank))
        tab += [ws.peers.ptrs["lists"][h], plans[h].lists_offsets[p] + below - local_off[p]]
    tab_t = torch.tensor(tab, dtype=torch.int64).to(dev, non_blocking=True)
    pp.map_scatter(None, cnt, lo, nprocs, bin_dst=tab_t, index_base=lo, status=status,
                   scratch=scratch, stream=stream)
    if world > 1:  # every peer's stores into our buffer have landed
        flag = torch.zeros(1, dtype=torch.int32, device=dev)
        dist.all_reduce(flag, group=group)
    mine = plans[rank]
    lists = {p: ws.buf[mine.lists_offsets[p]:mine.lists_offsets[p] + mine.lists_counts[p]]
             for p in mine.procs}
    return ShardedOwnership(lo, cnt, None, counts_all, totals, offs, write_at, mine.procs, lists)
