"""Mapped circuit simulation (the paper's Circuit workload).

The circuit is the Legion circuit benchmark's model (Bauer et al. 2012):
pieces of nodes joined by wires; each iteration runs calc_new_currents (an
implicit segment update solved by `steps` fixed-point iterations per wire),
distribute_charge (each wire deposits charge on its two end nodes) and
update_voltages (charge -> voltage, leakage).  The reference package has no
code for it (parity unpinned); oracle/circuit.py restates the
same model in float64.

Placement: the piece launch (ispace (pieces,)) is mapped onto the GPUs by a
Mapple mapper evaluated by K1, and every GPU takes its pieces from the fused
map + partition (K1+K2) ownership lists.  A wire belongs to the piece of its
in-node; its out-node is in the same piece (pct_in %) or in a neighbouring
piece (piece +- 1), so a block mapping keeps most cross-piece wires on one
GPU while a cyclic one sends them all over NVLink -- the mapping decides the
communication, as in the paper.  Cross-GPU wires read the remote node's
voltage and deposit charge with float atomics straight into the owning GPU's
arrays (csrc/circuit.cu); the communication volume is therefore exactly
8 bytes per cross-GPU wire end per iteration (4 B voltage read, 4 B charge).

The synthetic circuit is generated from a counter-based hash of (seed, field,
global index), so every GPU generates just its own pieces and the oracle
reproduces the same values.
"""

from __future__ import annotations

import ctypes
from dataclasses import dataclass

from .. import native
from ..dsl import compile_mapper, parse
from ..spaces import MachineShape

SEGMENTS = 10
MAX_RANKS = 16

CIRCUIT_MAPPERS = """
m = Machine(GPU)
def circuit_block(Tuple p, Tuple s):
    q = m.merge(0, 1)
    return q[p[0] * q.size[0] / s[0]]
def circuit_cyclic(Tuple p, Tuple s):
    q = m.merge(0, 1)
    return q[p[0] % q.size[0]]
IndexTaskMap circuit_block circuit_block
IndexTaskMap circuit_cyclic circuit_cyclic
"""

# hash fields
F_CAP, F_LEAK, F_V0, F_IN, F_LOC, F_DIR, F_OUT, F_R, F_L, F_C = range(10)


@dataclass(frozen=True)
class CircuitSpec:
    pieces: int
    nodes_per_piece: int
    wires_per_piece: int
    pct_in: int = 95        # % of wires whose out-node is in the same piece
    steps: int = 100        # fixed-point iterations of calc_new_currents
    dt: float = 1e-4
    seed: int = 0


def hash31(idx, salt: int):
    """Counter-based hash -> int64 in [0, 2^31) (same arithmetic as the oracle's)."""
    x = (idx * 2654435761 + salt * 40503 + 12345) % (1 << 31)
    x = x ^ (x >> 13)
    x = (x * 1103515245 + 12345) % (1 << 31)
    x = x ^ (x >> 16)
    x = (x * 69069 + 1) % (1 << 31)
    return x


def _salt(spec: CircuitSpec, field: int) -> int:
    return spec.seed * 64 + field


def _u(spec, idx, field):
    torch = native.require_cuda()
    return (hash31(idx, _salt(spec, field)).to(torch.float64) / float(1 << 31))


def node_values(spec: CircuitSpec, g):
    """(capacitance, leakage, initial voltage) of global node ids g (int64 tensor)."""
    torch = native.require_cuda()
    cap = (1.0 + _u(spec, g, F_CAP)).to(torch.float32)
    leak = (0.1 * _u(spec, g, F_LEAK)).to(torch.float32)
    v0 = (2.0 * _u(spec, g, F_V0) - 1.0).to(torch.float32)
    return cap, leak, v0


def wire_values(spec: CircuitSpec, gw):
    """(in node, out node, R, L, C) of global wire ids gw (int64 tensor)."""
    torch = native.require_cuda()
    P, npp, wpp = spec.pieces, spec.nodes_per_piece, spec.wires_per_piece
    piece = gw // wpp
    in_node = piece * npp + hash31(gw, _salt(spec, F_IN)) % npp
    local = hash31(gw, _salt(spec, F_LOC)) % 100 < spec.pct_in
    step = torch.where(hash31(gw, _salt(spec, F_DIR)) % 2 == 0, 1, P - 1)
    out_piece = torch.where(local, piece, (piece + step) % P)
    out_node = out_piece * npp + hash31(gw, _salt(spec, F_OUT)) % npp
    R = (1.0 + _u(spec, gw, F_R)).to(torch.float32)
    L = ((0.1 + _u(spec, gw, F_L)) * 1e-5).to(torch.float32)
    C = (1.0 + _u(spec, gw, F_C)).to(torch.float32)
    return in_node, out_node, R, L, C


class PmCircuitView(ctypes.Structure):
    _fields_ = [("n_wires", ctypes.c_int64), ("n_nodes", ctypes.c_int64),
                ("in_ref", ctypes.c_void_p), ("out_ref", ctypes.c_void_p),
                ("inductance", ctypes.c_void_p), ("resistance", ctypes.c_void_p),
                ("capacitance", ctypes.c_void_p), ("current", ctypes.c_void_p),
                ("wire_volt", ctypes.c_void_p), ("node_cap", ctypes.c_void_p),
                ("leakage", ctypes.c_void_p),
                ("volt", ctypes.c_void_p * MAX_RANKS), ("charge", ctypes.c_void_p * MAX_RANKS),
                ("rank", ctypes.c_int32), ("steps", ctypes.c_int32), ("dt", ctypes.c_float)]


class MappedCircuit:
    def __init__(self, spec: CircuitSpec, *, mapping: str = "block", rank: int = 0,
                 world: int = 1, group=None):
        torch = native.require_cuda()
        import torch.distributed as dist

        from ..peer import PeerBuffers

        if world > MAX_RANKS:
            raise ValueError(f"at most {MAX_RANKS} GPUs")
        self.spec, self.rank, self.world, self.group = spec, rank, world, group
        self.device = torch.device("cuda", torch.cuda.current_device())
        P, npp, wpp = spec.pieces, spec.nodes_per_piece, spec.wires_per_piece
        # Mapple placement of the piece launch (K1) and this GPU's pieces (K1+K2 fused)
        fn = compile_mapper(parse(CIRCUIT_MAPPERS), f"circuit_{mapping}",
                            MachineShape("GPU", world, 1))
        owner = fn.map_ispace((P,))
        own = fn.map_partition((P,))
        self.owner = owner.tolist()
        counts = own.counts.tolist()
        pos = [0] * P
        seen = [0] * world
        for p in range(P):  # position of each piece inside its GPU's list (launch order)
            pos[p] = seen[self.owner[p]]
            seen[self.owner[p]] += 1
        self.my_pieces = own.points_of(rank).to(torch.int64)
        self.n_pieces = int(counts[rank])
        dev = self.device
        owner_t = owner.to(torch.int64)
        pos_t = torch.tensor(pos, dtype=torch.int64, device=dev)
        # nodes of my pieces, piece-major
        j = torch.arange(npp, device=dev, dtype=torch.int64)
        g = (self.my_pieces.view(-1, 1) * npp + j.view(1, -1)).reshape(-1)
        self.node_ids = g
        self.node_cap, self.leakage, self.volt = node_values(spec, g)
        if g.numel() == 0:  # a GPU without pieces still exposes (1-element) node arrays
            self.node_cap, self.leakage, self.volt = (
                torch.ones(1, device=dev), torch.zeros(1, device=dev), torch.zeros(1, device=dev))
        self.charge = torch.zeros_like(self.volt)
        # wires of my pieces
        k = torch.arange(wpp, device=dev, dtype=torch.int64)
        gw = (self.my_pieces.view(-1, 1) * wpp + k.view(1, -1)).reshape(-1)
        self.wire_ids = gw
        in_node, out_node, self.R, self.L, self.C = wire_values(spec, gw)

        def ref(node):
            pc = node // npp
            return ((owner_t[pc] << 27) | (pos_t[pc] * npp + node % npp)).to(torch.int32)

        self.in_ref, self.out_ref = ref(in_node), ref(out_node)
        nw = gw.numel()
        self.current = torch.zeros(SEGMENTS, max(nw, 1), dtype=torch.float32, device=dev)
        self.wire_volt = torch.zeros(SEGMENTS - 1, max(nw, 1), dtype=torch.float32, device=dev)
        self.cross_gpu_wires = int(((self.out_ref.to(torch.int64) >> 27) != rank).sum())
        self.peers = PeerBuffers({"volt": self.volt, "charge": self.charge}, rank, world, group)
        v = PmCircuitView()
        v.n_wires, v.n_nodes = nw, g.numel()
        for name in ("in_ref", "out_ref"):
            setattr(v, name, getattr(self, name).data_ptr())
        v.inductance, v.resistance, v.capacitance = (self.L.data_ptr(), self.R.data_ptr(),
                                                     self.C.data_ptr())
        v.current, v.wire_volt = self.current.data_ptr(), self.wire_volt.data_ptr()
        v.node_cap, v.leakage = self.node_cap.data_ptr(), self.leakage.data_ptr()
        for r in range(world):
            v.volt[r] = self.peers.ptrs["volt"][r]
            v.charge[r] = self.peers.ptrs["charge"][r]
        v.rank, v.steps, v.dt = rank, spec.steps, spec.dt
        self.view = v
        from ..peer import PeerBarrier

        self._bar = PeerBarrier(rank, world, group) if world > 1 else None
        self._dist = dist if world > 1 else None
        self.iterations = 0
        torch.cuda.synchronize()
        if self._dist:
            dist.barrier(group=group)

    def _barrier(self, stream=None):
        """Stream-ordered all-GPU barrier through peer memory (csrc/barrier.cu)."""
        if self._bar is not None:
            self._bar(stream)

    def step(self, stream=None):
        """One iteration: calc_new_currents + distribute_charge, update_voltages."""
        torch = native.require_cuda()
        lib = native.lib()
        cs = native.stream_ptr(stream or torch.cuda.current_stream())
        self._barrier(stream)  # every GPU's voltages are final
        native.check(lib.pm_circuit_step(ctypes.byref(self.view), 0, cs), "pm_circuit_step")
        self._barrier(stream)  # every GPU's charge deposits have landed
        native.check(lib.pm_circuit_step(ctypes.byref(self.view), 1, cs), "pm_circuit_step")
        self.iterations += 1

    # FP32 ops per wire per step of calc_new_currents (csrc/circuit.cu)
    OPS_PER_WIRE_STEP = 48

    def work(self) -> dict:
        nw = self.wire_ids.numel()
        return {"wires": nw, "nodes": self.node_ids.numel(),
                "wire_steps": nw * self.spec.steps,
                "fp32_ops": nw * self.spec.steps * self.OPS_PER_WIRE_STEP,
                "cross_gpu_wires": self.cross_gpu_wires,
                "nvlink_bytes_per_iteration": 8 * self.cross_gpu_wires}

    def close(self):
        if self._bar is not None:
            self._bar.close()
        self.peers.close()
