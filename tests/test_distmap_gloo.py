"""Sharded launch mapping (distmap.py) over gloo on CPU.

Each rank takes its contiguous chunk of the launch, the processor ids come
from the oracle's evaluation of the Mapple mapper (the GPU path gets them from
K1), the stable partition is a host sort (K2 on the GPU) -- and the real
count all-gather + ownership all-to-all-v of `shard_ownership` run over gloo.
The lists every rank ends up with must equal the reference's shard-tree
leaves (oracle.shard_leaves: expand_shards, tasksim/sim.py:67-120): same
points, launch order, one list per processor, each on its host rank.
"""

import os
import socket

import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from oracle import mapple_oracle as O
from paper_2507_17087_b200 import distmap
from paper_2507_17087_b200.dsl import parse

MAPPERS = """
m = Machine(GPU)
def blk(Tuple p, Tuple s):
    q = m.merge(0, 1).decompose(0, s)
    return q[*(p * q.size / s)]
def cyc(Tuple p, Tuple s):
    q = m.merge(0, 1)
    return q[(p[0] * 7 + p[1] * 3) % q.size[0]]
def skew(Tuple p, Tuple s):
    q = m.merge(0, 1)
    return q[((p[0] < 3) ? 0 : (p[0] + p[1]) % q.size[0])]
IndexTaskMap blk blk
IndexTaskMap cyc cyc
IndexTaskMap skew skew
"""

CASES = [("blk", (2, 4), (12, 20)), ("blk", (1, 6), (9, 13)), ("cyc", (3, 2), (11, 7)),
         ("skew", (2, 3), (10, 10)), ("cyc", (1, 5), (1, 3))]


def host_partition(ids, P):
    counts = torch.bincount(ids.long(), minlength=P)
    perm = torch.sort(ids.long(), stable=True).indices.to(torch.int32)
    return counts, perm


def _worker(rank, world, port, out_q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        prog = parse(MAPPERS)
        res = []
        for task, machine, ispace in CASES:
            ids = O.map_launch(prog, task, ("GPU", *machine), ispace)
            n = len(ids)
            lo, hi = distmap.chunk(n, world, rank)
            P = machine[0] * machine[1]
            for exchange in (True, False):
                sh = distmap.shard_ownership(torch.tensor(ids[lo:hi], dtype=torch.int32), lo, P,
                                             rank, world, partition_fn=host_partition,
                                             exchange=exchange)
                mine = {p: sh.lists[p].tolist() for p in sh.lists}
                allr = [None] * world
                dist.all_gather_object(allr, (mine, sh.procs, sh.write_at, sh.totals))
                res.append((task, machine, ispace, exchange, ids, allr))
        out_q.put((rank, "ok", res if rank == 0 else None))
    except Exception as e:  # noqa: BLE001
        import traceback

        out_q.put((rank, "fail", traceback.format_exc() + repr(e)))
    finally:
        dist.destroy_process_group()


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


@pytest.mark.parametrize("world", [2, 3, 4, 8])
def test_sharded_ownership_matches_shard_tree(world):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    out = [q.get(timeout=300) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
    assert all(s == "ok" for _, s, _ in out), out
    res = next(r for _, _, r in out if r is not None)
    for task, machine, ispace, exchange, ids, allr in res:
        P = machine[0] * machine[1]
        pts = O.row_major(ispace)
        want = {p: [i for i, x in enumerate(ids) if x == p] for p in range(P)}
        totals = allr[0][3]
        assert totals == [len(want[p]) for p in range(P)]
        if exchange:
            got = {}
            for r, (mine, hosted, _, _) in enumerate(allr):
                assert hosted == [p for p in range(P) if distmap.host_rank(p, P, world) == r]
                for p in hosted:
                    got[p] = mine[p]
            assert got == want, (task, machine, ispace)
            # == the reference's shard-tree leaves, point order included
            leaves = O.shard_leaves(task, pts, [divmod(x, machine[1]) for x in ids])
            for _, (tgt, lpts) in leaves.items():
                p = tgt[0] * machine[1] + tgt[1]
                assert [pts[i] for i in got[p]] == list(lpts)
        else:
            # without the exchange every rank holds its chunk's lists at write_at
            for p in range(P):
                cat = []
                for r in range(world):
                    mine, _, write_at, _ = allr[r]
                    assert write_at[p] == sum(totals[:p]) + len(cat)
                    cat += mine[p]
                assert cat == want[p]
