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


class PmStepOp(ctypes.Structure):
    _fields_ = [("kind", ctypes.c_int32), ("lane", ctypes.c_int32), ("dst", ctypes.c_void_p),
                ("src", ctypes.c_void_p), ("b", ctypes.c_void_p), ("dpitch", ctypes.c_int64),
                ("spitch", ctypes.c_int64), ("width", ctypes.c_int64), ("height", ctypes.c_int64),
                ("lda", ctypes.c_int64), ("ldb", ctypes.c_int64), ("ldc", ctypes.c_int64),
                ("m", ctypes.c_int64), ("n", ctypes.c_int64), ("k", ctypes.c_int64),
                ("c_bf16", ctypes.c_int32), ("accumulate", ctypes.c_int32),
                ("barrier", ctypes.c_void_p), ("copies", ctypes.c_void_p),
                ("n_copies", ctypes.c_int32), ("ticket", ctypes.c_void_p)]


PULL, WAIT, GEMM_BF16, GEMM_TF32, MEMSET, BARRIER, COPY_BARRIER, FORK = range(8)
LANES = 4


class StepProgram:
    """One GPU's per-step schedule as data (csrc/steps.cpp, pm_steps_*): built once by
    an executor's planner over fixed device / peer pointers, replayed by one C call
    per step (`run`).  Ops: pull (copy-engine copy on a lane, or on the compute
    stream with lane=-1), wait (the compute stream on a lane pull), fork (the lanes
    restart after the compute stream's work so far), GEMMs, memset, peer barriers."""

    def __init__(self):
        self.ops = []
        self._keep = []   # ctypes objects the ops point to (barrier views, copy lists)
        self._handle = None

    def pull(self, dst, dpitch, src, spitch, width, height, lane=0) -> int:
        self.ops.append(PmStepOp(kind=PULL, lane=lane, dst=dst, src=src, dpitch=dpitch,
                                 spitch=spitch, width=width, height=height))
        return len(self.ops) - 1

    def wait(self, pull_index: int) -> None:
        self.ops.append(PmStepOp(kind=WAIT, lane=pull_index))

    def fork(self) -> None:
        """Later lane pulls start after everything issued so far on the compute stream."""
        self.ops.append(PmStepOp(kind=FORK))

    def gemm_bf16(self, A, lda, Bt, ldb, C, ldc, m, n, k, c_bf16=0, accumulate=0) -> None:
        self.ops.append(PmStepOp(kind=GEMM_BF16, src=A, lda=lda, b=Bt, ldb=ldb, dst=C, ldc=ldc,
                                 m=m, n=n, k=k, c_bf16=c_bf16, accumulate=accumulate))

    def gemm_tf32(self, A, lda, Bt, ldb, C, ldc, m, n, k, accumulate=0) -> None:
        self.ops.append(PmStepOp(kind=GEMM_TF32, src=A, lda=lda, b=Bt, ldb=ldb, dst=C, ldc=ldc,
                                 m=m, n=n, k=k, accumulate=accumulate))

    def memset(self, ptr, nbytes) -> None:
        self.ops.append(PmStepOp(kind=MEMSET, dst=ptr, width=nbytes))

    def barrier(self, bar: "PeerBarrier") -> None:
        self._keep.append(bar.view)
        self.ops.append(PmStepOp(kind=BARRIER, barrier=ctypes.addressof(bar.view)))

    def copy_barrier(self, bar: "PeerBarrier", copies) -> None:
        if len(copies) > 4:
            raise ValueError("at most 4 copies per launch")
        arr = (PmPeerCopy * max(1, len(copies)))(*[PmPeerCopy(d, s_, n) for d, s_, n in copies])
        self._keep += [bar.view, arr]
        self.ops.append(PmStepOp(kind=COPY_BARRIER, barrier=ctypes.addressof(bar.view),
                                 copies=ctypes.addressof(arr), n_copies=len(copies),
                                 ticket=bar.ticket.data_ptr()))

    def build(self) -> "StepProgram":
        arr = (PmStepOp * max(1, len(self.ops)))(*self.ops)
        out = ctypes.c_void_p()
        native.check(native.lib().pm_steps_create(arr, len(self.ops), ctypes.byref(out)),
                     "pm_steps_create")
        self._handle = out.value
        return self

    def run(self, stream=None) -> None:
        native.check(native.lib().pm_steps_run(self._handle, native.stream_ptr(stream)),
                     "pm_steps_run")

    def close(self) -> None:
        if self._handle:
            native.lib().pm_steps_destroy(self._handle)
            self._handle = None
