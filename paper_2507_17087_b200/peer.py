"""Peer pointers over NVLink for the mapped executors.

Each rank exposes some of its device buffers to the other ranks of the box:
CUDA IPC handles are exchanged once through `torch.distributed`
(all_gather_object), then every rank can pull slices of a peer's buffer with
the copy engines (`copy2d`), leaving all SMs to the tensor-core kernels.
"""

from __future__ import annotations

import ctypes

from . import native


class PeerBuffers:
    """name -> [device pointer of that buffer on every rank]."""

    def __init__(self, tensors: dict, rank: int, world: int, group=None):
        torch = native.require_cuda()
        import torch.distributed as dist

        self.rank, self.world = rank, world
        self._opened = []
        mine = {}
        for name, t in tensors.items():
            h = (ctypes.c_char * 64)()
            off = ctypes.c_int64(0)
            native.check(native.lib().pm_ipc_handle(t.data_ptr(), h, ctypes.byref(off)),
                         "pm_ipc_handle")
            mine[name] = (bytes(h), off.value)
        gathered = [None] * world
        if world > 1:
            dist.all_gather_object(gathered, mine, group=group)
        else:
            gathered = [mine]
        self.ptrs = {name: [0] * world for name in tensors}
        cache = {}
        for r in range(world):
            for name, (h, off) in gathered[r].items():
                if r == rank:
                    self.ptrs[name][r] = tensors[name].data_ptr()
                    continue
                base = cache.get((r, h))
                if base is None:
                    out = ctypes.c_void_p()
                    native.check(native.lib().pm_ipc_open(h, ctypes.byref(out)), "pm_ipc_open")
                    base = cache[(r, h)] = out.value
                    self._opened.append(base)
                self.ptrs[name][r] = base + off
        _ = torch

    def close(self):
        for base in self._opened:
            native.lib().pm_ipc_close(base)
        self._opened = []


class PmPeerBarrierView(ctypes.Structure):
    _fields_ = [("my_flags", ctypes.c_void_p), ("peer_slot", ctypes.c_void_p * 16),
                ("epoch", ctypes.c_void_p), ("world", ctypes.c_int32), ("rank", ctypes.c_int32)]


class PmPeerCopy(ctypes.Structure):
    _fields_ = [("dst", ctypes.c_void_p), ("src", ctypes.c_void_p), ("bytes", ctypes.c_int64)]


class PeerBarrier:
    """Stream-ordered barrier of the box's ranks through peer memory (csrc/barrier.cu):
    a 32-thread kernel pushes the next epoch into every peer's flag slot and waits
    for theirs -- no NCCL, and capturable in a CUDA graph (the epoch advances on
    the device)."""

    def __init__(self, rank: int, world: int, group=None):
        torch = native.require_cuda()
        if world > 16:
            raise ValueError("pm_peer_barrier supports up to 16 ranks")
        dev = torch.device("cuda", torch.cuda.current_device())
        self.flags = torch.zeros(max(world, 1), dtype=torch.int32, device=dev)
        self.epoch = torch.zeros(1, dtype=torch.int32, device=dev)
        self.ticket = torch.zeros(1, dtype=torch.int32, device=dev)
        torch.cuda.synchronize()  # zeroed before any peer can push into them
        self.peers = PeerBuffers({"flags": self.flags}, rank, world, group)
        v = PmPeerBarrierView()
        v.my_flags = self.flags.data_ptr()
        for q in range(world):
            v.peer_slot[q] = self.peers.ptrs["flags"][q] + 4 * rank
        v.epoch = self.epoch.data_ptr()
        v.world, v.rank = world, rank
        self.view = v

    def __call__(self, stream=None) -> None:
        native.check(native.lib().pm_peer_barrier(ctypes.byref(self.view),
                                                  native.stream_ptr(stream)), "pm_peer_barrier")

    def copy_then_wait(self, copies, stream=None) -> None:
        """[(dst_ptr, src_ptr, bytes)] copied by the SMs (peer or local), then this
        barrier -- one launch (pm_peer_copy_barrier)."""
        if len(copies) > 4:
            raise ValueError("at most 4 copies per launch")
        arr = (PmPeerCopy * max(1, len(copies)))(*[PmPeerCopy(d, s, n) for d, s, n in copies])
        native.check(native.lib().pm_peer_copy_barrier(ctypes.byref(self.view), arr, len(copies),
                                                       self.ticket.data_ptr(),
                                                       native.stream_ptr(stream)),
                     "pm_peer_copy_barrier")

    def close(self):
        self.peers.close()


def copy2d(dst: int, dpitch: int, src: int, spitch: int, width: int, height: int, stream) -> None:
    """Pitched byte copy on the copy engines (peer or local), stream-ordered."""
    native.check(native.lib().pm_copy2d_async(dst, dpitch, src, spitch, width, height,
                                              native.stream_ptr(stream)), "pm_copy2d_async")
