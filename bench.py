#!/usr/bin/env python
"""Benchmark: mapped-GEMM TFLOP/s on 1/2/4/8 B200 (decompose vs heuristic) + comm bytes.

Workload (BASELINE.json configs[1]): SUMMA, bf16 inputs, fp32 accumulation,
M = N = K = 32768, C distributed over the GPUs by a Mapple block mapper
(`decompose` mapping = headline `value`; the Algorithm-1 heuristic mapping is
measured in the same run).  Synthetic operands (seeded), 2 GiB each, far
larger than L2, so no flush is needed between steps.  One step = one full
multiply: NVLink peer pulls of the SUMMA panels on the copy engines + the
tcgen05 GEMMs.  Time = CUDA events on the compute stream, max over ranks.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]

`--impl reference` times the reference's CPU path on the host cores (rank 0):
the unmodified reference (baseline/_ref) maps the launch with the same Mapple
program, numpy float32 multiplies a bounded sample of the same product (the
reference has no GEMM), and prints the same JSON line with "impl": "reference".
"""

from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

METRIC = "mapped-GEMM TFLOP/s at 1/2/4/8 B200 (decompose vs heuristic); comm bytes"
WORKLOAD = "SUMMA bf16 M=N=K=32768, Mapple block mapping (BASELINE configs[1])"


def peaks():
    p = ROOT / "MEASURED_PEAKS.json"
    if p.exists():
        d = json.loads(p.read_text())
        return d["bf16_tflops"], d["bf16_tflops_sustained"], d["hbm_gbs"], "measured"
    return 1590.0, 1400.0, 6650.0, "fallback"


class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled during the timed region."""

    Q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.proc = None
        self.lines = []
        self.window = None

    def start(self):
        """Start sampling (call before warm-up so samples exist in the timed window)."""
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--id={self.index}", f"--query-gpu={self.Q}",
                 "--format=csv,noheader,nounits", "-lms", "50"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except OSError:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append((time.time(), line.strip()))

    def mark(self, t0: float, t1: float):
        self.window = (t0, t1)

    def stop(self):
        if self.proc:
            time.sleep(0.12)
            self.proc.terminate()
            self.proc.wait(timeout=5)
            self.t.join(timeout=5)

    def summary(self):
        sm, mx, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        lines = self.lines
        if self.window:
            inside = [l for l in lines if self.window[0] - 0.06 <= l[0] <= self.window[1] + 0.06]
            lines = inside or lines[-3:]
        for _, ln in lines:
            parts = [x.strip() for x in ln.split(",")]
            if len(parts) < 6:
                continue
            try:
                sm.append(float(parts[0]))
                mx = float(parts[1])
            except ValueError:
                continue
            for n, v in zip(names, parts[2:]):
                if v.lower().startswith("active"):
                    reasons.add(n)
        if not sm:
            return {"sm_mhz": None, "sm_max_mhz": mx, "reasons": [], "samples": 0}
        loaded = [s for s in sm if s > 0.5 * max(sm)] or sm
        return {"sm_mhz": statistics.median(loaded), "sm_max_mhz": mx,
                "reasons": sorted(reasons), "samples": len(sm)}


# -- distributed plumbing -----------------------------------------------------------


def init_dist(n_gpus: int):
    import torch

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world != n_gpus:
        raise SystemExit(f"--gpus {n_gpus} but WORLD_SIZE={world}; launch with torchrun for N>1")
    # PM_BENCH_OVERSUB=1 (a code-path check, never a measurement): more ranks than GPUs,
    # ranks sharing a GPU through same-device IPC, gloo instead of NCCL (NCCL refuses two
    # ranks on one GPU) -- how an 8-rank run is exercised on a 4-GPU box
    oversub = os.environ.get("PM_BENCH_OVERSUB", "0") != "0"
    if oversub:
        local %= torch.cuda.device_count()
    torch.cuda.set_device(local)
    if world > 1:
        import torch.distributed as dist

        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        if oversub:
            dist.init_process_group("gloo")
        else:
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    return rank, world, local


def barrier(world):
    if world > 1:
        import torch.distributed as dist

        dist.barrier()


def max_over_ranks(x: float, world: int) -> float:
    if world == 1:
        return x
    import torch
    import torch.distributed as dist

    t = torch.tensor([x], dtype=torch.float64, device="cuda")
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def sum_over_ranks(x: float, world: int) -> float:
    if world == 1:
        return x
    import torch
    import torch.distributed as dist

    t = torch.tensor([x], dtype=torch.float64, device="cuda")
    dist.all_reduce(t)
    return float(t.item())


# -- our implementation -----------------------------------------------------------------


def run_mapping(args, rank, world, local, mapping, mnk=None):
    import torch

    from paper_2507_17087_b200.executors.summa import MappedGemm

    S = args.size
    M, N, K = mnk or (S, S, S)
    ex = MappedGemm(M, N, K, mapping=mapping, rank=rank, world=world, a_chunks=args.chunks,
                    seed=1234)
    cs = torch.cuda.current_stream()
    sampler = ClockSampler(local).start()
    for _ in range(args.warmup):
        ex.step()
    torch.cuda.synchronize()
    barrier(world)
    # the timed region: one event after every step on the compute stream, so each step's
    # own duration is known; with one GEMM launch per step (N=1) that IS the launch's
    # duration over the timed region (the roofline's `achieved`); multi-launch steps
    # (N>1) take per-launch durations from the instrumented pass below
    t0, t1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    step_ev = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]
    torch.cuda.synchronize()
    barrier(world)
    w0 = time.time()
    t0.record(cs)
    for i in range(args.steps):
        ex.step()
        step_ev[i].record(cs)
    t1.record(cs)
    torch.cuda.synchronize()
    step_ms = [t0.elapsed_time(step_ev[0])] + [step_ev[i - 1].elapsed_time(step_ev[i])
                                               for i in range(1, args.steps)]
    sampler.mark(w0, time.time())
    sampler.stop()
    barrier(world)
    ms = t0.elapsed_time(t1) / args.steps
    ms_max = max_over_ranks(ms, world)
    # instrumented pass: per-launch GEMM durations on the compute stream
    launch_ms = []
    for _ in range(max(2, min(args.steps, 5))):
        evs = []
        orig = ex.step_python  # op by op, so each tile_gemm launch can be bracketed

        from paper_2507_17087_b200 import gemm as G

        real = G.tile_gemm

        def timed_gemm(*a, **k):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(cs)
            out = real(*a, **k)
            e1.record(cs)
            evs.append((e0, e1))
            return out

        G.tile_gemm = timed_gemm
        try:
            orig()
        finally:
            G.tile_gemm = real
        torch.cuda.synchronize()
        launch_ms += [a.elapsed_time(b) for a, b in evs]
    instrumented_ms = statistics.mean(launch_ms)
    if ex.gemm_launches == 1:  # the step is the launch: use the timed region's own times
        launch_ms = step_ms
    res = {
        "grid": list(ex.layout.grid),
        "ms_per_step": ms_max,
        "tflops": 2 * M * N * K / (ms_max * 1e-3) / 1e12,
        "comm_bytes_per_gpu_max": int(max_over_ranks(ex.recv_bytes, world)),
        "comm_bytes_total": int(sum_over_ranks(ex.recv_bytes, world)),
        "gemm_launch_ms_avg": statistics.mean(launch_ms),
        "gemm_launch_ms_source": ("timed region (one launch per step)" if ex.gemm_launches == 1
                                  else "instrumented pass after the timed region"),
        "gemm_launch_ms_instrumented": instrumented_ms,
        "gemm_flops_per_launch": ex.flops / max(1, ex.gemm_launches),
        "gemm_launches_per_step": ex.gemm_launches,
        "clocks": sampler.summary(),
    }
    return ex, res


def run_3d_pair(args, rank, world, local, M, N, K, rounds=3):
    """Time one 3-D mapped multiply (Johnson / COSMA grid, fused GEMM + NVLink
    reduce-scatter) under the decompose AND the heuristic mapping: both executors live at
    once and their timed blocks alternate `rounds` times (the box's power state drifts by
    several % over a run, so back-to-back blocks would favour whichever runs first);
    per mapping the median block, each block's time the max over ranks of CUDA events."""
    import torch

    from paper_2507_17087_b200.executors.grid3d import MappedGemm3D

    cs = torch.cuda.current_stream()
    steps = max(3, args.steps // 2)
    exs = {m: MappedGemm3D(M, N, K, mapping=m, rank=rank, world=world, seed=99)
           for m in ("decompose", "heuristic")}
    for ex in exs.values():
        for _ in range(args.warmup):
            ex.step()
        ex.result()
    times = {m: [] for m in exs}
    for _ in range(rounds):
        for m, ex in exs.items():
            torch.cuda.synchronize()
            barrier(world)
            t0, t1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            t0.record(cs)
            for _ in range(steps):
                ex.step()
            ex.result()  # the last step's reduce-adds from the peers have landed
            t1.record(cs)
            torch.cuda.synchronize()
            times[m].append(max_over_ranks(t0.elapsed_time(t1) / steps, world))
    out = {}
    for m, ex in exs.items():
        ms = statistics.median(times[m])
        out[m] = {"grid": list(ex.grid), "ms_per_step": ms,
                  "tflops": 2.0 * M * N * K / (ms * 1e-3) / 1e12,
                  "ms_per_step_blocks": times[m],
                  "comm_bytes_per_gpu": ex.comm, "steps": steps, "rounds": rounds,
                  "gpu_launches_per_step": ex.gemm_launches}
        ex.close()
    del exs
    torch.cuda.empty_cache()
    return out["decompose"], out["heuristic"]


def run_2d_pair(args, rank, world, M, N, K, rounds=3):
    """SUMMA / PUMMA panels under both mappings, timed in alternating blocks (as
    run_3d_pair); per mapping the median block, max over ranks."""
    import torch

    from paper_2507_17087_b200.executors.summa import MappedGemm

    cs = torch.cuda.current_stream()
    exs = {m: MappedGemm(M, N, K, mapping=m, rank=rank, world=world, a_chunks=args.chunks,
                         seed=1234) for m in ("decompose", "heuristic")}
    for ex in exs.values():
        for _ in range(args.warmup):
            ex.step()
    times = {m: [] for m in exs}
    for _ in range(rounds):
        for m, ex in exs.items():
            torch.cuda.synchronize()
            barrier(world)
            t0, t1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            t0.record(cs)
            for _ in range(args.steps):
                ex.step()
            t1.record(cs)
            torch.cuda.synchronize()
            times[m].append(max_over_ranks(t0.elapsed_time(t1) / args.steps, world))
    out = {}
    for m, ex in exs.items():
        ms = statistics.median(times[m])
        out[m] = {"grid": list(ex.layout.grid), "ms_per_step": ms,
                  "tflops": 2.0 * M * N * K / (ms * 1e-3) / 1e12, "ms_per_step_blocks": times[m],
                  "comm_bytes_per_gpu_max": int(max_over_ranks(ex.recv_bytes, world)),
                  "comm_bytes_total": int(sum_over_ranks(ex.recv_bytes, world)),
                  "gemm_launches_per_step": ex.gemm_launches, "rounds": rounds}
        ex.close()
    del exs
    torch.cuda.empty_cache()
    return out


def run_cannon(args, rank, world, N, layers, dtype, graph=False):
    """BASELINE configs[0] (Cannon fp32 N=1024 on 2x2) and the Cannon / 2.5D
    bf16 variants: Cannon skew + shifts as NVLink pulls, 2.5D layer reduction
    fused into the GEMM epilogue.  graph=True replays the whole multiply (pulls,
    peer-memory barriers, GEMMs) as one CUDA graph per C buffer."""
    import torch

    from paper_2507_17087_b200.executors.cannon import MappedCannon, cannon_moves

    ex = MappedCannon(N, layers=layers, rank=rank, world=world, dtype=dtype, seed=31,
                      graph=graph)
    cs = torch.cuda.current_stream()
    for _ in range(max(args.warmup, 4 if graph else 0)):  # graphs are captured in warm-up
        ex.step()
    ex.result()
    torch.cuda.synchronize()
    barrier(world)
    steps = max(3, args.steps // 2)
    t0, t1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    t0.record(cs)
    for _ in range(steps):
        ex.step()
    ex.result()
    t1.record(cs)
    torch.cuda.synchronize()
    ms = max_over_ranks(t0.elapsed_time(t1) / steps, world)
    moves = int(sum_over_ranks(ex.moved_blocks, world))
    res = {"N": N, "dtype": dtype, "graph": graph, "grid": [ex.q, ex.q, ex.c],
           "machine": list(ex.machine),
           "ms_per_multiply": ms, "tflops": 2.0 * N ** 3 / (ms * 1e-3) / 1e12,
           "block_moves": moves, "block_moves_schedule": cannon_moves(ex.q, ex.c),
           "bytes_moved": moves * ex.block_bytes}
    barrier(world)
    ex.close()
    del ex
    torch.cuda.empty_cache()
    return res


def run_circuit(args, rank, world, mapping, pieces_per_gpu=96, npp=5000, wpp=20000,
                steps=1000, iters=5):
    """The circuit workload, weak scaling: 96 pieces of 5000 nodes /
    20000 wires per GPU, 1000 calc_new_currents steps per iteration."""
    import torch

    from paper_2507_17087_b200.executors.circuit import CircuitSpec, MappedCircuit

    spec = CircuitSpec(pieces_per_gpu * world, npp, wpp, pct_in=95, steps=steps, seed=7)
    ex = MappedCircuit(spec, mapping=mapping, rank=rank, world=world)
    cs = torch.cuda.current_stream()
    ex.step()
    torch.cuda.synchronize()
    barrier(world)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(cs)
    for _ in range(iters):
        ex.step()
    e1.record(cs)
    torch.cuda.synchronize()
    ms = max_over_ranks(e0.elapsed_time(e1) / iters, world)
    w = ex.work()
    wires = sum_over_ranks(w["wires"], world)
    cross = sum_over_ranks(w["cross_gpu_wires"], world)
    ops = wires * steps * ex.OPS_PER_WIRE_STEP
    barrier(world)
    ex.close()
    return {"mapping": mapping, "pieces": spec.pieces, "wires": int(wires),
            "ms_per_iteration": ms, "wire_steps_per_s": wires * steps / (ms * 1e-3),
            "fp32_ops_per_s": ops / (ms * 1e-3), "cross_gpu_wires": int(cross),
            "nvlink_bytes_per_iteration": int(8 * cross)}


def run_hydro(args, rank, world, mapping, zx=16384, zy=4096, steps=10):
    """PENNANT-style hydro, strong scaling on a fixed 16384 x 4096-zone
    mesh (aspect 4:1, where the decompose and heuristic grids differ)."""
    import torch

    from paper_2507_17087_b200.executors.hydro import HydroSpec, MappedHydro

    ex = MappedHydro(HydroSpec(zx, zy), mapping=mapping, rank=rank, world=world)
    cs = torch.cuda.current_stream()
    for _ in range(2):
        ex.step()
    torch.cuda.synchronize()
    barrier(world)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(cs)
    for _ in range(steps):
        ex.step()
    e1.record(cs)
    torch.cuda.synchronize()
    ms = max_over_ranks(e0.elapsed_time(e1) / steps, world)
    cross = int(sum_over_ranks(ex.cross_corners, world))
    zones = zx * zy
    _, _, hbm, _ = peaks()
    gbs = ex.BYTES_PER_ZONE_STEP * zones / world / (ms * 1e-3) / 1e9
    barrier(world)
    ex.close()
    del ex
    torch.cuda.empty_cache()
    return {"mapping": mapping, "zones": zones, "ms_per_step": ms,
            "zone_steps_per_s": zones / (ms * 1e-3), "cross_gpu_corners": cross,
            "bytes_per_zone_step": 121, "achieved_gbs_per_gpu": gbs, "frac_hbm": gbs / hbm}


def run_stencil(args, rank, world, rows, cols, mapping, sweeps=20):
    """BASELINE configs[4]: 5-point Jacobi fp32 with the fused NVLink halo exchange."""
    import torch

    from paper_2507_17087_b200.executors.stencil import MappedStencil

    ex = MappedStencil(rows, cols, mapping=mapping, rank=rank, world=world, seed=7)
    cs = torch.cuda.current_stream()
    ex.run(3 * max(1, args.warmup))
    torch.cuda.synchronize()
    barrier(world)
    t0, t1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    t0.record(cs)
    ex.run(sweeps)
    t1.record(cs)
    torch.cuda.synchronize()
    ms = max_over_ranks(t0.elapsed_time(t1) / sweeps, world)
    _, _, hbm, _ = peaks()
    cells = rows * cols
    per_gpu_gbs = 8.0 * cells / world / (ms * 1e-3) / 1e9
    res = {"grid": list(ex.grid), "ms_per_sweep": ms, "cells_per_s": cells / (ms * 1e-3),
           "sweeps": sweeps, "bytes_per_cell": 8, "achieved_gbs_per_gpu": per_gpu_gbs,
           "frac_hbm": per_gpu_gbs / hbm, "halo_cells_per_sweep": ex.halo_cells,
           "halo_model_surface_volume": ex.model_halo,
           "halo_bytes_per_sweep": 4 * (ex.halo_cells or 0)}
    barrier(world)
    ex.close()
    del ex
    torch.cuda.empty_cache()
    return res


def run_e2e_pipelined(args, ex):
    """N=1 end to end: every step copies its operands in from pinned host memory
    and its C out; the copies run on their own streams (copy engines) with
    double-buffered device operands so step s+1's H2D and step s's D2H overlap
    step s's GEMM.  CUDA events from the first H2D to the last D2H."""
    import torch

    hA = ex.A.cpu().pin_memory()
    hB = ex.Bt.cpu().pin_memory()
    hC = [torch.empty(ex.C.shape, dtype=ex.C.dtype).pin_memory() for _ in range(2)]
    bufs = [(ex.A, ex.Bt, ex.C), (torch.empty_like(ex.A), torch.empty_like(ex.Bt),
                                  torch.empty_like(ex.C))]
    cs = torch.cuda.current_stream()
    h2d, d2h = torch.cuda.Stream(), torch.cuda.Stream()
    ev_in = [torch.cuda.Event() for _ in range(2)]
    ev_comp = [torch.cuda.Event() for _ in range(2)]
    ev_out = [torch.cuda.Event() for _ in range(2)]
    for e in ev_comp + ev_out:
        e.record(cs)

    def run(n, t0=None, t1=None):
        if t0 is not None:
            t0.record(h2d)
        for s in range(n):
            b = s % 2
            A, Bt, C = bufs[b]
            h2d.wait_event(ev_comp[b])          # the GEMM two steps ago is done with A, Bt
            with torch.cuda.stream(h2d):
                A.copy_(hA, non_blocking=True)
                Bt.copy_(hB, non_blocking=True)
            ev_in[b].record(h2d)
            cs.wait_event(ev_in[b])
            cs.wait_event(ev_out[b])            # C of two steps ago has been read out
            ex.A, ex.Bt, ex.C = A, Bt, C
            ex.step()
            ev_comp[b].record(cs)
            d2h.wait_event(ev_comp[b])
            with torch.cuda.stream(d2h):
                hC[b].copy_(C, non_blocking=True)
            ev_out[b].record(d2h)
        if t1 is not None:
            t1.record(d2h)

    run(2)
    torch.cuda.synchronize()
    # the timed window includes the pipeline's fill (first H2D) and drain (last D2H)
    n = min(max(24, args.steps), 32)  # fill + drain amortised over >= 24 pipelined steps
    t0, t1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    run(n, t0, t1)
    torch.cuda.synchronize()
    ex.A, ex.Bt, ex.C = bufs[0]
    ms = t0.elapsed_time(t1) / n
    # the PCIe floor: one step's H2D and D2H timed alone
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(h2d)
    with torch.cuda.stream(h2d):
        bufs[1][0].copy_(hA, non_blocking=True)
        bufs[1][1].copy_(hB, non_blocking=True)
    e1.record(h2d)
    torch.cuda.synchronize()
    h2d_ms = e0.elapsed_time(e1)
    e0.record(d2h)
    with torch.cuda.stream(d2h):
        hC[0].copy_(bufs[1][2], non_blocking=True)
    e1.record(d2h)
    torch.cuda.synchronize()
    d2h_ms = e0.elapsed_time(e1)
    # both directions at once, no GEMM: the PCIe / host-memory floor of a pipelined step
    e2 = torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    e0.record(h2d)
    d2h.wait_event(e0)
    with torch.cuda.stream(h2d):
        bufs[1][0].copy_(hA, non_blocking=True)
        bufs[1][1].copy_(hB, non_blocking=True)
    with torch.cuda.stream(d2h):
        hC[0].copy_(bufs[1][2], non_blocking=True)
    e1.record(h2d)
    e2.record(d2h)
    torch.cuda.synchronize()
    both_ms = max(e0.elapsed_time(e1), e0.elapsed_time(e2))
    S = args.size
    return {"value": 2 * S ** 3 / (ms * 1e-3) / 1e12, "unit": "TFLOP/s", "ms_per_step": ms,
            "steps": n, "h2d_ms_alone": h2d_ms, "d2h_ms_alone": d2h_ms,
            "h2d_d2h_concurrent_ms": both_ms,
            "h2d_bytes_per_step": int(hA.numel() * 2 + hB.numel() * 2),
            "d2h_bytes_per_step": int(hC[0].numel() * hC[0].element_size()),
            "pipelined": "H2D(s+1) / GEMM(s) / D2H(s-1) on separate streams"}


def run_e2e(args, ex, rank, world):
    """Same multiply through the public API with host buffers: H2D of this GPU's
    operand slices from pinned memory, the mapped multiply, D2H of its C block."""
    if world == 1:
        return run_e2e_pipelined(args, ex)
    return run_e2e_pipelined_multi(args, ex, rank, world)


def run_e2e_pipelined_multi(args, ex, rank, world):
    """N > 1 end to end, pipelined like N=1 across two operand sets (two executors
    with their own peer-shared buffers): step s loads this GPU's A / B slices into
    set s % 2 from pinned memory (H2D stream), a stream-ordered 4-byte NCCL
    all-reduce on a comm stream says "every GPU's slices landed" before any pull
    of step s, the mapped multiply runs, a second all-reduce says "every GPU is
    done pulling from set s % 2" before step s + 2 overwrites it, and C goes out
    on the D2H stream.  No host synchronisation inside the window; CUDA events
    from the first H2D to the last D2H, max over ranks."""
    import torch
    import torch.distributed as dist

    from paper_2507_17087_b200.executors.summa import MappedGemm

    ex2 = MappedGemm(ex.M, ex.N, ex.K, mapping=ex.mapping, rank=rank, world=world,
                     a_chunks=args.chunks)
    sets = [ex, ex2]
    # this GPU's own slices in its K-rotated buffers: 1 or 2 column pieces each
    hA = [ex.A[:, p0:p0 + n].contiguous().cpu().pin_memory() for p0, _, n in ex.own_a]
    hB = [ex.Bt[:, p0:p0 + n].contiguous().cpu().pin_memory() for p0, _, n in ex.own_b]
    hC = [torch.empty(ex.C.shape, dtype=ex.C.dtype).pin_memory() for _ in range(2)]
    cs = torch.cuda.current_stream()
    h2d, d2h, comm = torch.cuda.Stream(), torch.cuda.Stream(), torch.cuda.Stream()
    flag = torch.zeros(2, dtype=torch.int32, device=cs.device)
    ev = {k: [torch.cuda.Event() for _ in range(2)] for k in ("in", "ready", "comp", "free", "out")}
    for b in range(2):
        for k in ("comp", "free", "out"):
            ev[k][b].record(cs)

    trace = [] if os.environ.get("PM_E2E_TRACE") else None

    def mark(stream):
        if trace and trace[-1] is not None:
            e = torch.cuda.Event(enable_timing=True)
            e.record(stream)
            trace[-1].append(e)

    def run(n, t0=None, t1=None):
        if t0 is not None:
            t0.record(h2d)
        for s in range(n):
            b = s % 2
            E = sets[b]
            if trace is not None:
                trace.append([] if t0 is not None else None)
            h2d.wait_event(ev["free"][b])      # every GPU done pulling from set b
            mark(h2d)
            with torch.cuda.stream(h2d):
                for (p0, _, n), h in zip(E.own_a, hA):
                    E.A[:, p0:p0 + n].copy_(h, non_blocking=True)
                for (p0, _, n), h in zip(E.own_b, hB):
                    E.Bt[:, p0:p0 + n].copy_(h, non_blocking=True)
            ev["in"][b].record(h2d)
            mark(h2d)
            comm.wait_event(ev["in"][b])
            with torch.cuda.stream(comm):     # every GPU's slices of set b landed
                dist.all_reduce(flag[0:1])
            ev["ready"][b].record(comm)
            cs.wait_event(ev["out"][b])        # C of two steps ago has been read out
            cs.wait_event(ev["ready"][b])
            mark(cs)
            E.step(stream=cs, ready=ev["ready"][b])
            ev["comp"][b].record(cs)
            mark(cs)
            comm.wait_event(ev["comp"][b])
            with torch.cuda.stream(comm):
                dist.all_reduce(flag[1:2])
            ev["free"][b].record(comm)
            d2h.wait_event(ev["comp"][b])
            mark(d2h)
            with torch.cuda.stream(d2h):
                hC[b].copy_(E.C, non_blocking=True)
            ev["out"][b].record(d2h)
            mark(d2h)
        if t1 is not None:
            t1.record(d2h)

    run(2)
    torch.cuda.synchronize()
    barrier(world)
    n = min(max(24, args.steps), 32)  # fill + drain amortised over >= 24 pipelined steps
    t0, t1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    run(n, t0, t1)
    torch.cuda.synchronize()
    ms = max_over_ranks(t0.elapsed_time(t1) / n, world)
    if trace is not None and rank == 0:  # per step: h2d, compute, d2h (start, end) in ms
        tr = [[round(t0.elapsed_time(e), 2) for e in st] for st in trace if st is not None]
        print(json.dumps({"e2e_trace": tr[:12]}), file=sys.stderr)
    barrier(world)
    ex2.close()
    del ex2
    torch.cuda.empty_cache()
    h2d_b = sum_over_ranks(sum(h.numel() * 2 for h in hA + hB), world)
    d2h_b = sum_over_ranks(hC[0].numel() * hC[0].element_size(), world)
    S = args.size
    return {"value": 2 * S ** 3 / (ms * 1e-3) / 1e12, "unit": "TFLOP/s", "ms_per_step": ms,
            "steps": n, "h2d_bytes_per_step": int(h2d_b), "d2h_bytes_per_step": int(d2h_b),
            "pipelined": "two operand sets: H2D(s+1) / mapped multiply(s) / D2H(s-1) on "
                         "separate streams, stream-ordered NCCL flags between GPUs"}


def cpu_sample(args, threads=None, seconds=None):
    """The oracle port on the host: numpy float64 C[0:r, 0:c] of the same product."""
    import numpy as np
    import torch

    from oracle.numerics import sample_rows_cols
    from paper_2507_17087_b200.executors.summa import synth

    S = args.size
    r, c = args.cpu_rows, args.cpu_cols
    dev = torch.device("cuda", torch.cuda.current_device()) if torch.cuda.is_available() else None
    A = synth((0, r), (0, S), S, 1234, dev).float().cpu().numpy().astype(np.float64)
    Bt = synth((0, c), (0, S), S, 1235, dev).float().cpu().numpy().astype(np.float64)
    lim, used = blas_threads()
    # repeat the bounded sample until ~10 s of host work (contract: 10-30 s)
    t = time.perf_counter()
    C = sample_rows_cols(A, Bt)
    reps = 1
    while time.perf_counter() - t < (args.cpu_seconds if seconds is None else seconds):
        sample_rows_cols(A, Bt)
        reps += 1
    dt = (time.perf_counter() - t) / reps
    return C, dt, 2.0 * r * c * S, used


def run_sharded_mapping(args, rank, world):
    """The 32768^2 stencil launch (configs[4]) mapped + partitioned across the
    GPUs (distmap.py, fused kernels): with the ownership exchange over NVLink
    and with each GPU keeping its chunk's lists.  Strong scaling (fixed launch)."""
    import torch

    from paper_2507_17087_b200 import distmap
    from paper_2507_17087_b200.dsl import compile_mapper, parse
    from paper_2507_17087_b200.spaces import MachineShape

    src = ("m = Machine(GPU)\ndef blk(Tuple p, Tuple s):\n"
           "    q = m.merge(0, 1).decompose(0, s)\n    return q[*(p * q.size / s)]\n"
           "IndexTaskMap t blk\n")
    fn = compile_mapper(parse(src), "t", MachineShape("GPU", 1, 8))
    L = 32768
    out = {"workload": "32768^2 launch, decompose block mapper, 8 processors, sharded over "
                       f"{world} GPU(s)", "points": L * L}
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    for exchange in (True, False):
        for _ in range(2):
            distmap.map_launch_sharded(fn, (L, L), rank=rank, world=world, exchange=exchange)
        torch.cuda.synchronize()
        barrier(world)
        e0.record()
        reps = 5
        for _ in range(reps):
            distmap.map_launch_sharded(fn, (L, L), rank=rank, world=world, exchange=exchange)
        e1.record()
        torch.cuda.synchronize()
        ms = max_over_ranks(e0.elapsed_time(e1) / reps, world)
        key = "exchange_to_host_gpu" if exchange else "lists_stay_on_chunk_gpu"
        out[key] = {"ms": ms, "points_per_s": L * L / (ms * 1e-3)}
    barrier(world)
    return out


def hot_path_kernels(args):
    """K1 / K2 throughput on config 5 (32768^2 stencil launch, 8-way block mapping)."""
    import torch

    from paper_2507_17087_b200.dsl import compile_mapper, parse
    from paper_2507_17087_b200.ownership import partition
    from paper_2507_17087_b200.spaces import MachineShape

    src = ("m = Machine(GPU)\ndef blk(Tuple p, Tuple s):\n"
           "    q = m.merge(0, 1).decompose(0, s)\n    return q[*(p * q.size / s)]\n"
           "IndexTaskMap t blk\n")
    fn = compile_mapper(parse(src), "t", MachineShape("GPU", 1, 8))
    L = 32768
    n = L * L
    out = torch.empty(n, dtype=torch.int32, device="cuda")
    st = torch.full((1,), -1, dtype=torch.int64, device="cuda")
    for _ in range(3):
        fn.map_ispace((L, L), out=out, status=st, check=False)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    reps = 20
    e0.record()
    for _ in range(reps):
        fn.map_ispace((L, L), out=out, status=st, check=False)
    e1.record()
    torch.cuda.synchronize()
    k1_ms = e0.elapsed_time(e1) / reps
    partition(out, 8)
    torch.cuda.synchronize()
    e0.record()
    for _ in range(5):
        partition(out, 8, check=False)
    e1.record()
    torch.cuda.synchronize()
    k2_ms = e0.elapsed_time(e1) / 5
    # K3: halo transfer lists of the same 8-way block ownership (h = 1)
    from paper_2507_17087_b200.transfer import halo_lists

    tl = halo_lists(out, (L, L), (1, 1), 8)
    cap = tl.total  # the lists of an unchanged ownership: sized once, no host round trip
    for _ in range(2):
        halo_lists(out, (L, L), (1, 1), 8, capacity=cap)
    torch.cuda.synchronize()
    e0.record()
    reps = 10
    for _ in range(reps):
        tl = halo_lists(out, (L, L), (1, 1), 8, capacity=cap)
    e1.record()
    torch.cuda.synchronize()
    k3_ms = e0.elapsed_time(e1) / reps
    k3_entries = tl.total
    tl_exact = halo_lists(out, (L, L), (1, 1), 8)
    torch.cuda.synchronize()
    e0.record()
    for _ in range(3):
        tl_exact = halo_lists(out, (L, L), (1, 1), 8)
    e1.record()
    torch.cuda.synchronize()
    k3_exact_ms = e0.elapsed_time(e1) / 3
    assert tl_exact.total == k3_entries
    # K1+K2 fused: two passes over the launch, ids never stored (4 B/pt: the perm write)
    fn.map_partition((L, L), check=False)
    torch.cuda.synchronize()
    e0.record()
    for _ in range(5):
        fn.map_partition((L, L), check=False)
    e1.record()
    torch.cuda.synchronize()
    k12_ms = e0.elapsed_time(e1) / 5
    _, _, hbm, _ = peaks()
    # write ceiling of this box, live: fill_ of the same 4 B/pt id array (a pure store
    # stream runs above the copy peak: ~7.5 vs ~6.6 TB/s; reads alike)
    out.fill_(0)
    torch.cuda.synchronize()
    e0.record()
    for _ in range(5):
        out.fill_(0)
    e1.record()
    torch.cuda.synchronize()
    fill_gbs = 4 * n / (e0.elapsed_time(e1) / 5 * 1e-3) / 1e9
    fn.map_ispace((L, L), out=out, check=False)  # restore the ids for anything after
    k1_gbs = 4 * n / (k1_ms * 1e-3) / 1e9
    k1_cpu = None
    if not args.no_cpu:
        # the reference's CPU path for this launch (oracle port of cmd_map's per-point
        # loop) on 1 core and on every core, bounded samples, extrapolated
        from oracle.cpu_mapping_bench import cpu_mapping_rate, reference_available

        kind = "reference" if reference_available() else "port"
        k1_cpu = cpu_mapping_rate(src, "t", ("GPU", 1, 8), (L, L), seconds=3.0, kind=kind)
        k1_cpu.update({"unit": "points/s",
                       "sample": "contiguous row-major slices of the 32768^2 launch, 3 s per "
                                 "worker (full-launch time extrapolated); kind reference = the "
                                 "unmodified reference in baseline/_ref (compile_mapper + "
                                 "per-point fn, cmd_map's loop)",
                       "k1_speedup_vs_all_cores": (n / (k1_ms * 1e-3)) /
                                                  k1_cpu["points_per_s_all"]})
        if kind == "reference":  # the oracle port beside it
            port = cpu_mapping_rate(src, "t", ("GPU", 1, 8), (L, L), seconds=2.0, kind="port")
            k1_cpu["port"] = {k: port[k] for k in ("points_per_s_1core", "points_per_s_all",
                                                   "cores")}
    # K2 reads the ids twice and writes the permutation; the scatter skips the read for
    # tiles whose 4096 ids are all equal (uniform): 8 + 4 * (non-uniform fraction) B/pt
    t = out.view(-1, 4096)
    uniform = float((t.amin(dim=1) == t.amax(dim=1)).float().mean())
    k2_bpp = 8 + 4 * (1 - uniform)
    k2_gbs = k2_bpp * n / (k2_ms * 1e-3) / 1e9
    k12_gbs = 4 * n / (k12_ms * 1e-3) / 1e9
    return {"workload": "stencil 32768^2 launch, decompose block mapper, 1x8 GPUs (configs[4])",
            "write_ceiling_gbs": fill_gbs,
            "k1_map": {"points_per_s": n / (k1_ms * 1e-3), "ms": k1_ms, "bytes_per_point": 4,
                       "achieved_gbs": k1_gbs, "frac_hbm": k1_gbs / hbm,
                       "frac_write_ceiling": k1_gbs / fill_gbs,
                       "cpu_baseline": k1_cpu},
            "k2_partition": {"ms": k2_ms, "bytes_per_point": k2_bpp,
                             "uniform_tile_fraction": uniform, "achieved_gbs": k2_gbs,
                             "frac_hbm": k2_gbs / hbm},
            "k3_halo_lists": {"ms": k3_ms, "entries": k3_entries,
                              "mode": "capacity= (stream-ordered, no host round trip)",
                              "ms_exact_sizing": k3_exact_ms,
                              "bytes": 4 * n + 9 * k3_entries,
                              "achieved_gbs": (4 * n + 9 * k3_entries) / (k3_ms * 1e-3) / 1e9,
                              "frac_hbm": (4 * n + 9 * k3_entries) / (k3_ms * 1e-3) / 1e9 / hbm},
            "k12_fused_map_partition": {"ms": k12_ms, "points_per_s": n / (k12_ms * 1e-3),
                                        "bytes_per_point": 4, "achieved_gbs": k12_gbs,
                                        "frac_hbm": k12_gbs / hbm,
                                        "frac_write_ceiling": k12_gbs / fill_gbs,
                                        "vs_k1_then_k2": (k1_ms + k2_ms) / k12_ms}}


def cublas_same_shape(ex, rounds=3):
    """cuBLAS (torch.matmul, bf16 in / bf16 out) beside K4 (bf16 in / fp32 out) on the same
    32768^3 operands, interleaved launch by launch so both see the same clocks / power
    state; median CUDA-event time of each."""
    import torch

    from paper_2507_17087_b200.gemm import tile_gemm

    A, Bt, C = ex.A, ex.Bt, ex.C
    out = torch.empty(A.shape[0], Bt.shape[0], dtype=torch.bfloat16, device=A.device)
    ours, theirs = [], []
    for _ in range(rounds):
        for fn, acc in ((lambda: tile_gemm(A, Bt, C), ours),
                        (lambda: torch.matmul(A, Bt.t(), out=out), theirs)):
            fn()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            fn()
            e1.record()
            torch.cuda.synchronize()
            acc.append(e0.elapsed_time(e1))
    flops = 2.0 * A.shape[0] * Bt.shape[0] * A.shape[1]
    o, t = statistics.median(ours), statistics.median(theirs)
    del out
    return {"k4_ms": o, "k4_tflops": flops / (o * 1e-3) / 1e12, "cublas_ms": t,
            "cublas_tflops": flops / (t * 1e-3) / 1e12, "k4_vs_cublas": t / o,
            "note": "interleaved single launches on the headline operands; K4 writes fp32 C "
                    "(4 GiB), cuBLAS bf16 C (2 GiB)"}


def main_ours(args):
    import torch

    rank, world, local = init_dist(args.gpus)
    burst, sustained, hbm, peak_src = peaks()
    ex, dec = run_mapping(args, rank, world, local, "decompose")
    e2e = run_e2e(args, ex, rank, world) if not args.no_e2e else None
    cublas = cublas_same_shape(ex) if world == 1 and not args.no_kernels else None
    ex.close()
    del ex
    torch.cuda.empty_cache()
    heur = None
    if not args.decompose_only:
        ex, heur = run_mapping(args, rank, world, local, "heuristic")
        ex.close()
        del ex
        torch.cuda.empty_cache()
    extra = {}
    errors = {}

    def guarded(name, fn):
        """An extra workload must not take the headline line down with it: its
        failure is recorded in the JSON line instead (same on every rank)."""
        try:
            return fn()
        except Exception as e:  # noqa: BLE001
            errors[name] = f"{type(e).__name__}: {e}"[:300]
            torch.cuda.synchronize()
            return None

    if not args.no_3d:
        # BASELINE configs[2] (Johnson 3D, square) and configs[3] (COSMA, rectangular)
        def w3d():
            wl = {}
            for name, (M, N, K) in (("johnson3d", (args.size,) * 3),
                                    ("cosma", (2 * args.size, args.size // 2, args.size // 2))):
                d, h = run_3d_pair(args, rank, world, local, M, N, K)
                wl[name] = {"M": M, "N": N, "K": K, "decompose": d, "heuristic": h,
                            "speedup": d["tflops"] / h["tflops"],
                            "comm_ratio": h["comm_bytes_per_gpu"]["total"] /
                            max(1, d["comm_bytes_per_gpu"]["total"])}
            return wl
        extra["workloads_3d"] = guarded("workloads_3d", w3d)

        def pumma():
            # configs[3]'s 2-D algorithm: SUMMA / PUMMA panels on the rectangular shape,
            # where the decompose grid differs from Algorithm 1's (e.g. (4,1) vs (2,2))
            mnk = (2 * args.size, args.size // 2, args.size // 2)
            out = {"M": mnk[0], "N": mnk[1], "K": mnk[2]}
            out.update(run_2d_pair(args, rank, world, *mnk))
            out["speedup"] = out["decompose"]["tflops"] / out["heuristic"]["tflops"]
            out["comm_ratio"] = (out["heuristic"]["comm_bytes_total"] /
                                 max(1, out["decompose"]["comm_bytes_total"]))
            return out
        extra["pumma"] = guarded("pumma", pumma)
    if not args.no_cannon:
        cn = {}
        if world in (1, 4):  # q x q grids: configs[0] is Cannon fp32 N=1024 on 2x2
            cn["cannon_fp32_N1024"] = guarded(
                "cannon_fp32", lambda: run_cannon(args, rank, world, 1024, 1, "fp32"))
            # configs[0] is launch-latency bound: the same multiply replayed as a CUDA graph
            cn["cannon_fp32_N1024_graph"] = guarded(
                "cannon_fp32_graph",
                lambda: run_cannon(args, rank, world, 1024, 1, "fp32", graph=True))
            cn["cannon_bf16"] = guarded(
                "cannon_bf16", lambda: run_cannon(args, rank, world, args.size, 1, "bf16"))
        if world == 8:       # configs[2]: Solomonik 2.5D on 2x2x2
            cn["solomonik_2p5d_bf16"] = guarded(
                "solomonik_2p5d", lambda: run_cannon(args, rank, world, args.size, 2, "bf16"))
        extra["cannon"] = cn
    if not args.no_stencil:
        def stencil():
            st = {}
            for name, (r, c) in (("square", (args.size, args.size)),
                                 ("aspect_1x4", (args.size // 2, 2 * args.size))):
                d = run_stencil(args, rank, world, r, c, "decompose")
                h = run_stencil(args, rank, world, r, c, "heuristic")
                st[name] = {"rows": r, "cols": c, "decompose": d, "heuristic": h,
                            "speedup": h["ms_per_sweep"] / d["ms_per_sweep"],
                            "halo_ratio": (h["halo_cells_per_sweep"] or 1) /
                            max(1, d["halo_cells_per_sweep"] or 1)}
            return {"workload": "5-point Jacobi fp32, Mapple block mapping, fused NVLink "
                                "halo exchange (BASELINE configs[4])", **st}
        extra["stencil"] = guarded("stencil", stencil)
    if not args.no_circuit:
        extra["circuit"] = guarded("circuit", lambda: {
            "workload": "circuit simulation (configs[4] 'plus circuit sim'), weak scaling, "
                        "node exchange fused over NVLink",
            "block": run_circuit(args, rank, world, "block"),
            "cyclic": run_circuit(args, rank, world, "cyclic")})
    if not args.no_hydro:
        def hydro():
            d = run_hydro(args, rank, world, "decompose")
            h = run_hydro(args, rank, world, "heuristic")
            return {"workload": "PENNANT-style Lagrangian hydro, 16384x4096 quad zones, "
                                "shared points fused over NVLink",
                    "decompose": d, "heuristic": h, "speedup": h["ms_per_step"] / d["ms_per_step"]}
        extra["pennant_hydro"] = guarded("pennant_hydro", hydro)
    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu:
        # the reference's CPU path of this workload (same as the --impl reference arm)
        h = host_reference_step(args, world, args.cpu_seconds)
        cpu = {"value": h["tflops"], "unit": "TFLOP/s", "cores": h["cores"],
               "kind": h["mapping_kind"],
               "sample": f"the reference (baseline/_ref) maps all {h['mapping_points']} C-block "
                         f"points (every core), then {h['gemm_sample']} extrapolated to the "
                         "full product (the reference has no GEMM, SURVEY F9)",
               "parts": h}
        C64, dt, fl, used = cpu_sample(args, seconds=0.0)
        # parity on the same sample: the GPU's C block starts at row/col 0 here
        from paper_2507_17087_b200.executors.summa import MappedGemm

        exc = MappedGemm(args.size, args.size, args.size, mapping="decompose", seed=1234)
        exc.step()
        torch.cuda.synchronize()
        got = exc.C[:args.cpu_rows, :args.cpu_cols].double().cpu().numpy()
        err = float(abs(got - C64).max() / abs(C64).max())
        extra["parity"] = {"sample": "C[0:%d, 0:%d] vs numpy float64" % (args.cpu_rows, args.cpu_cols),
                           "max_rel_err": err, "tolerance": 1e-2, "ok": err <= 1e-2}
        exc.close()
        del exc
        torch.cuda.empty_cache()
    if rank == 0 and world == 1 and not args.no_kernels:
        extra["hot_path_kernels"] = guarded("hot_path_kernels", lambda: hot_path_kernels(args))
    if not args.no_kernels:
        extra["sharded_mapping"] = guarded("sharded_mapping",
                                           lambda: run_sharded_mapping(args, rank, world))
    if errors:
        extra["errors"] = errors
    if rank != 0:
        return
    # burst peak unless the timed region lasted > 1 s (the conservative denominator);
    # the sustained figure (measured under the 1 kW power cap, as our timed region
    # runs when clocks show sw_power_cap) is reported beside it
    capped = "sw_power_cap" in (dec.get("clocks") or {}).get("reasons", [])
    peak = sustained if dec["ms_per_step"] * args.steps > 1000 else burst
    achieved = dec["gemm_flops_per_launch"] / (dec["gemm_launch_ms_avg"] * 1e-3) / 1e12
    traffic = None
    tf = ROOT / "profiles" / "gemm_traffic.json"
    if tf.exists():
        traffic = json.loads(tf.read_text()).get("bytes_per_launch")
    line = {
        "metric": METRIC,
        "value": dec["tflops"],
        "unit": "TFLOP/s",
        "n_gpus": world,
        "steps": args.steps,
        "warmup": args.warmup,
        "ms_per_step": dec["ms_per_step"],
        "higher_is_better": True,
        "scaling": "strong",
        "vs_baseline": None,
        "dtype": "bf16",
        "data": "synthetic (seeded U(-1,1) operands generated on device)",
        "config": {"workload": WORKLOAD, "M": args.size, "N": args.size, "K": args.size,
                   "mapping": "decompose", "grid": dec["grid"], "accumulate": "fp32",
                   "l2": "operands 2 GiB each, larger than L2 (no flush needed)",
                   "parallelism": f"summa{dec['grid'][0]}x{dec['grid'][1]}"},
        "e2e": None if e2e is None else {k: e2e[k] for k in
                                         ("value", "unit", "h2d_bytes_per_step",
                                          "d2h_bytes_per_step", "ms_per_step", "steps",
                                          "h2d_ms_alone", "d2h_ms_alone",
                                          "h2d_d2h_concurrent_ms", "pipelined")
                                         if k in e2e},
        "roofline": {"bound": "tensor", "achieved": achieved, "peak": peak,
                     "unit": "TFLOP/s", "frac": achieved / peak,
                     "peak_source": f"{peak_src} {'sustained' if peak == sustained else 'burst'} "
                                    "bf16 (MEASURED_PEAKS.json)",
                     "frac_of_burst": achieved / burst,
                     "frac_of_sustained": achieved / sustained,
                     "power_capped": capped,
                     "kernel": "pm::gemm::wide::k_gemm_bf16_wide (tcgen05 cta_group::2, pair "
                               "tile 512x256, TMA ring, TMEM, dynamic tile scheduler)",
                     "traffic": traffic,
                     "achieved_from": dec["gemm_launch_ms_source"],
                     "achieved_instrumented_pass": dec["gemm_flops_per_launch"] /
                     (dec["gemm_launch_ms_instrumented"] * 1e-3) / 1e12,
                     "cublas_same_shape": cublas},
        "cpu_baseline": cpu,
        "clocks": dec["clocks"],
        "gpu_launches": dec["gemm_launches_per_step"] * args.steps,
        "comm": {"decompose": {"grid": dec["grid"],
                               "bytes_per_gpu_max": dec["comm_bytes_per_gpu_max"],
                               "bytes_total": dec["comm_bytes_total"]}},
        "decompose_vs_heuristic": None,
    }
    if heur is not None:
        line["comm"]["heuristic"] = {"grid": heur["grid"],
                                     "bytes_per_gpu_max": heur["comm_bytes_per_gpu_max"],
                                     "bytes_total": heur["comm_bytes_total"]}
        line["decompose_vs_heuristic"] = {
            "heuristic_tflops": heur["tflops"], "heuristic_ms_per_step": heur["ms_per_step"],
            "speedup": dec["tflops"] / heur["tflops"],
            "comm_ratio": heur["comm_bytes_total"] / max(1, dec["comm_bytes_total"])}
    line.update(extra)
    print(json.dumps(line), flush=True)


def blas_threads():
    """Every host core of the affinity mask for numpy's BLAS, whatever OMP_NUM_THREADS
    torchrun set (it pins each rank to 1 thread); returns (limiter, threads in use)."""
    from threadpoolctl import threadpool_info, threadpool_limits

    cores = len(os.sched_getaffinity(0))
    lim = threadpool_limits(limits=cores, user_api="blas")
    used = max([p.get("num_threads", 1) for p in threadpool_info()
                if p.get("user_api") == "blas"] or [1])
    return lim, used


def host_reference_step(args, world: int, seconds: float):
    """One step of the reference's CPU path for the headline workload, on the host
    cores: (1) the reference itself (baseline/_ref, unmodified) maps the SUMMA C-block
    launch -- compile_mapper + the per-point loop of cmd_map (cli.py:149-161,
    dsl/interp.py:401-433) over all (S/128)^2 points of the same Mapple program and
    machine (G, 1) our arm uses, on every host core (contiguous slices, one worker
    per core); (2) the block products, which the reference does not implement
    (SURVEY F9), as numpy float32 GEMMs on every core -- a bounded sample
    C[0:r, 0:c] with the full K, repeated for ~`seconds`, extrapolated to the whole
    product.  Returns the step time and its parts."""
    import numpy as np

    from oracle.cpu_mapping_bench import cpu_mapping_rate, reference_available
    from paper_2507_17087_b200.executors.summa import TILE_MAPPERS
    from paper_2507_17087_b200.factorize import greedy_grid

    S = args.size
    nb = -(-S // 128)
    src = TILE_MAPPERS.format(g0=greedy_grid(world, 2)[0])
    kind = "reference" if reference_available() else "port"
    m = cpu_mapping_rate(src, "gemm_decompose", ("GPU", world, 1), (nb, nb),
                         seconds=min(3.0, seconds / 4), kind=kind)
    t_map = nb * nb / m["points_per_s_all"]
    lim, cores = blas_threads()
    r, c = args.cpu_rows, args.cpu_cols
    rng = np.random.default_rng(1234)
    A = rng.uniform(-1, 1, (r, S)).astype(np.float32)
    Bt = rng.uniform(-1, 1, (c, S)).astype(np.float32)
    A[:64] @ Bt[:64].T  # BLAS warm-up
    t = time.perf_counter()
    reps = 0
    while reps == 0 or time.perf_counter() - t < seconds:
        A @ Bt.T
        reps += 1
    t_sample = (time.perf_counter() - t) / reps
    t_gemm = t_sample * (S / r) * (S / c)
    return {"ms_per_step": (t_map + t_gemm) * 1e3, "tflops": 2.0 * S ** 3 / (t_map + t_gemm) / 1e12,
            "cores": max(cores, m["cores"]), "mapping_kind": kind,
            "mapping_points": nb * nb, "mapping_points_per_s_all_cores": m["points_per_s_all"],
            "mapping_points_per_s_1core": m["points_per_s_1core"], "mapping_s": t_map,
            "gemm_sample": f"numpy float32 C[0:{r}, 0:{c}] (full K = {S}), {t_sample:.3f} s",
            "gemm_sample_tflops": 2.0 * r * c * S / t_sample / 1e12, "gemm_s_extrapolated": t_gemm}


def main_reference(args):
    """Reference arm: the reference's CPU path on the host cores, rank 0 only
    (host_reference_step: the reference maps the launch, numpy multiplies)."""
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    world = int(os.environ.get("WORLD_SIZE", "1"))
    nsteps = max(1, min(args.steps, 3))
    steps = [host_reference_step(args, world, args.cpu_seconds / nsteps) for _ in range(nsteps)]
    ms = statistics.mean(s["ms_per_step"] for s in steps)
    v = 2.0 * args.size ** 3 / (ms * 1e-3) / 1e12
    last = steps[-1]
    S = args.size
    print(json.dumps({
        "impl": "reference", "metric": METRIC, "value": v, "unit": "TFLOP/s",
        "n_gpus": world, "steps": nsteps, "warmup": args.warmup, "ms_per_step": ms,
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f32",
        "data": "synthetic",
        "config": {"workload": WORKLOAD, "M": S, "N": S, "K": S, "mapping": "decompose",
                   "machine": [world, 1]},
        "cpu_baseline": {"value": v, "unit": "TFLOP/s", "cores": last["cores"],
                         "kind": last["mapping_kind"],
                         "sample": f"per step: the reference (baseline/_ref) maps all "
                                   f"{last['mapping_points']} C-block points of the launch "
                                   f"(compile_mapper + cmd_map's per-point loop, every core), "
                                   f"then {last['gemm_sample']} extrapolated to the full product "
                                   "(the reference has no GEMM, SURVEY F9)",
                         "parts": last},
        "e2e": {"value": v, "unit": "TFLOP/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }), flush=True)


def main():
    ap = argparse.ArgumentParser(description=__doc__.splitlines()[0])
    ap.add_argument("--gpus", type=int, default=int(os.environ.get("WORLD_SIZE", "1")))
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--size", type=int, default=32768)
    ap.add_argument("--chunks", type=int, default=4)
    ap.add_argument("--cpu-rows", type=int, default=2048)
    ap.add_argument("--cpu-cols", type=int, default=8192)
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--no-kernels", action="store_true")
    ap.add_argument("--decompose-only", action="store_true")
    ap.add_argument("--no-3d", action="store_true", help="skip the Johnson / COSMA workloads")
    ap.add_argument("--no-stencil", action="store_true", help="skip the stencil workload")
    ap.add_argument("--no-cannon", action="store_true", help="skip the Cannon / 2.5D workloads")
    ap.add_argument("--no-circuit", action="store_true", help="skip the circuit workload")
    ap.add_argument("--no-hydro", action="store_true", help="skip the PENNANT-style workload")
    ap.add_argument("--cpu-seconds", type=float, default=10.0,
                    help="host seconds spent on the CPU baseline sample")
    args = ap.parse_args()
    if args.warmup < 3 and args.impl == "ours":
        print("note: the contract needs >= 3 warm-up steps", file=sys.stderr)
    if args.impl == "reference":
        main_reference(args)
    else:
        main_ours(args)
        if int(os.environ.get("WORLD_SIZE", "1")) > 1:
            import torch.distributed as dist

            dist.barrier()
            dist.destroy_process_group()


if __name__ == "__main__":
    main()
