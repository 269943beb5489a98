"""Mapped PENNANT-style hydrodynamics (the paper's PENNANT workload).

A Lagrangian staggered-grid step in the PENNANT structure (Ferenbaugh 2015):
zone-centred thermodynamics (mass, energy, gamma-law pressure, artificial
viscosity), point-centred kinematics, zone -> corner -> point force
gathering.  The mesh is a quadrilateral mesh stored unstructured (zone ->
point references), generated as an Lx x Ly grid on [0,1]^2 with a smooth
energy pulse in the middle and reflecting walls.  The reference package has
no code for it (parity unpinned); oracle/hydro.py restates the
same model in float64.

Placement: the zone launch (ispace (Ly, Lx)) is mapped onto the GPUs by the
stencil workloads' Mapple block mappers (decompose or Algorithm-1 heuristic),
evaluated by K1; each GPU's zones come from the fused map + partition, a
point belongs to the GPU of the zone at its (clamped) coordinates, and K2
partitions the points.  Zones read their points through per-GPU pointer
tables and deposit corner forces with float atomics into the owning GPU's
array (csrc/hydro.cu): the shared points on GPU boundaries are the whole
exchange (16 B read + one 8-byte float2 atomic per cross-GPU corner per step).
"""

from __future__ import annotations

import ctypes
import math
from dataclasses import dataclass

from .. import native
from .stencil import stencil_mapper

MAX_RANKS = 16


@dataclass(frozen=True)
class HydroSpec:
    zones_x: int
    zones_y: int
    gamma: float = 5.0 / 3.0
    cq: float = 1.0          # artificial viscosity coefficient
    pulse: float = 10.0      # energy pulse amplitude (over a background of 1)
    cfl: float = 0.25


def hydro_dt(spec: HydroSpec) -> float:
    """Fixed time step from the initial maximum sound speed (the same on host and oracle)."""
    h = 1.0 / max(spec.zones_x, spec.zones_y)
    e_max = 1.0 + spec.pulse
    c = math.sqrt(spec.gamma * (spec.gamma - 1.0) * e_max)
    return spec.cfl * h / c


class PmHydroView(ctypes.Structure):
    _fields_ = [("n_zones", ctypes.c_int64), ("n_points", ctypes.c_int64),
                ("z2p", ctypes.c_void_p), ("zm", ctypes.c_void_p), ("ze", ctypes.c_void_p),
                ("za", ctypes.c_void_p), ("zpe", ctypes.c_void_p), ("pm", ctypes.c_void_p),
                ("pbc", ctypes.c_void_p)] + \
               [(n, ctypes.c_void_p * MAX_RANKS) for n in ("pst", "fxy")] + \
               [("rank", ctypes.c_int32), ("dt", ctypes.c_float), ("gamma", ctypes.c_float),
                ("cq", ctypes.c_float)]


class MappedHydro:
    def __init__(self, spec: HydroSpec, *, mapping: str = "decompose", rank: int = 0,
                 world: int = 1, group=None):
        torch = native.require_cuda()
        import torch.distributed as dist

        from ..ownership import partition
        from ..peer import PeerBuffers

        if world > MAX_RANKS:
            raise ValueError(f"at most {MAX_RANKS} GPUs")
        self.spec, self.rank, self.world, self.group = spec, rank, world, group
        dev = self.device = torch.device("cuda", torch.cuda.current_device())
        Lx, Ly = spec.zones_x, spec.zones_y
        i64 = torch.int64
        # zone placement (K1) and this GPU's zones (fused K1+K2), launch order
        fn = stencil_mapper(world, mapping)
        zparts, zown = fn.map_partition((Ly, Lx), with_ids=True)
        self.zone_ids = zparts.points_of(rank).to(i64)
        # point owner = owner of the zone at the clamped coordinates; K2 lists
        pj = torch.arange(Ly + 1, device=dev, dtype=i64).clamp(max=Ly - 1)
        pi = torch.arange(Lx + 1, device=dev, dtype=i64).clamp(max=Lx - 1)
        zids = zown.view(Ly, Lx)
        pown = zids[pj.view(-1, 1), pi.view(1, -1)].reshape(-1).contiguous()
        pp = partition(pown, world)
        npts = (Lx + 1) * (Ly + 1)
        # global point id -> slot on its owner
        perm = pp.perm.to(i64)
        slot = torch.empty(npts, dtype=i64, device=dev)
        slot[perm] = torch.arange(npts, device=dev, dtype=i64) - pp.offsets[pown[perm].to(i64)]
        pref = (pown.to(i64) << 27) | slot
        self.point_ids = pp.points_of(rank).to(i64)
        # zones: CCW point references
        zj, zi = self.zone_ids // Lx, self.zone_ids % Lx
        W = Lx + 1
        corners = [zj * W + zi, zj * W + zi + 1, (zj + 1) * W + zi + 1, (zj + 1) * W + zi]
        self.z2p = torch.stack([pref[c] for c in corners]).to(torch.int32).contiguous()
        h2 = 1.0 / (Lx * Ly)
        nz = self.zone_ids.numel()
        xc = (zi.to(torch.float64) + 0.5) / Lx
        yc = (zj.to(torch.float64) + 0.5) / Ly
        r2 = (xc - 0.5) ** 2 + (yc - 0.5) ** 2
        self.ze = (1.0 + spec.pulse * torch.exp(-r2 / 0.01)).to(torch.float32)
        self.zm = torch.full((nz,), h2, dtype=torch.float32, device=dev)
        self.za = torch.full((nz,), h2, dtype=torch.float32, device=dev)
        self.zpe = torch.zeros(nz, dtype=torch.float32, device=dev)
        # points
        gj, gi = self.point_ids // W, self.point_ids % W
        # point state (x, y, u, v) as one 16-byte record per point (a zone gathers each
        # corner with one vector load); px / py / ux / uy are strided views of it
        npl = self.point_ids.numel()
        self.pst = torch.zeros(max(npl, 1), 4, dtype=torch.float32, device=dev)
        self.pst[:npl, 0] = (gi.to(torch.float64) / Lx).to(torch.float32)
        self.pst[:npl, 1] = (gj.to(torch.float64) / Ly).to(torch.float32)
        self.px, self.py, self.ux, self.uy = (self.pst[:, c] for c in range(4))
        self.fxy = torch.zeros(2 * max(npl, 1), dtype=torch.float32, device=dev)
        nadj = ((gi > 0).to(i64) + (gi < Lx).to(i64)) * ((gj > 0).to(i64) + (gj < Ly).to(i64))
        self.pm = (nadj.to(torch.float64) * h2 / 4.0).to(torch.float32)
        self.pbc = (((gi == 0) | (gi == Lx)).to(torch.int8) +
                    2 * ((gj == 0) | (gj == Ly)).to(torch.int8)).contiguous()
        # the communication model: corners whose point lives on another GPU
        self.cross_corners = int(((self.z2p.to(i64) >> 27) != rank).sum())
        self.peers = PeerBuffers({n: getattr(self, n) for n in ("pst", "fxy")}, rank, world,
                                 group)
        v = PmHydroView()
        v.n_zones, v.n_points = nz, self.point_ids.numel()
        v.z2p, v.zm, v.ze, v.za, v.zpe = (self.z2p.data_ptr(), self.zm.data_ptr(),
                                          self.ze.data_ptr(), self.za.data_ptr(),
                                          self.zpe.data_ptr())
        v.pm, v.pbc = self.pm.data_ptr(), self.pbc.data_ptr()
        for n in ("pst", "fxy"):
            arr = getattr(v, n)
            for r in range(world):
                arr[r] = self.peers.ptrs[n][r]
        v.rank, v.dt, v.gamma, v.cq = rank, hydro_dt(spec), spec.gamma, spec.cq
        self.view = v
        from ..peer import PeerBarrier

        self._bar = PeerBarrier(rank, world, group) if world > 1 else None
        self._dist = dist if world > 1 else None
        torch.cuda.synchronize()
        if self._dist:
            dist.barrier(group=group)

    def _barrier(self, stream=None):
        """Stream-ordered all-GPU barrier through peer memory (csrc/barrier.cu)."""
        if self._bar is not None:
            self._bar(stream)

    def step(self, stream=None):
        """One Lagrangian step: zones (forces to points), then points (kinematics)."""
        torch = native.require_cuda()
        lib = native.lib()
        cs = native.stream_ptr(stream or torch.cuda.current_stream())
        self._barrier(stream)  # all points moved
        native.check(lib.pm_hydro_step(ctypes.byref(self.view), 0, cs), "pm_hydro_step")
        self._barrier(stream)  # all corner forces deposited
        native.check(lib.pm_hydro_step(ctypes.byref(self.view), 1, cs), "pm_hydro_step")

    # algorithmic HBM bytes per zone-step: zone kernel 16 (z2p) + 16 (zm, ze, za, zpe) +
    # 12 (ze, za, zpe) + 16 (point x, y, u, v) + 8 (force RMW); point kernel 29 read
    # (state 16, force 8, mass 4, wall flags 1) + 24 write (state 16, force reset 8)
    BYTES_PER_ZONE_STEP = 16 + 16 + 12 + 16 + 8 + 29 + 24

    def close(self):
        if self._bar is not None:
            self._bar.close()
        self.peers.close()
