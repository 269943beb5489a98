"""NVLink bytes moved by the fused peer-memory kernels, against their algorithmic
exchange bytes (torchrun, one rank per GPU; no profiler, so no kernel replay --
the ranks' peer barriers would not survive one).

Each rank reads its GPU's NVLink data counters (NVML field values
NVLINK_THROUGHPUT_DATA_TX / RX, KiB, summed over links) before and after K
iterations of a workload and reports bytes per iteration beside the executor's
own count of what it must move:
  * grid3d  -- Johnson / COSMA multiply: A / B all-gathers by copy-engine pulls
               plus the C reduce-scatter fused into the GEMM epilogue (TMA .add into
               the owner's C over NVLink): comm_bytes_3d per GPU;
  * stencil -- column strips / peer rows read by the sweep kernel: 4 B per halo cell;
  * circuit -- peer loads + peer float atomics of the cross-GPU wires: 8 B per wire;
  * hydro   -- cross-GPU corners: 16 B point-state load + 8 B force atomic.
Pulls show up as RX on the pulling GPU; a peer atomic / store as TX on the issuing one.

    torchrun --nproc-per-node 2 tools/nvlink_probe.py > gpurun_out/nvlink.json
"""

import json
import os
import sys
import time

sys.path.insert(0, ".")
import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402


def counters(handle):
    import pynvml

    vals = pynvml.nvmlDeviceGetFieldValues(
        handle, [pynvml.NVML_FI_DEV_NVLINK_THROUGHPUT_DATA_TX,
                 pynvml.NVML_FI_DEV_NVLINK_THROUGHPUT_DATA_RX])
    out = []
    for v in vals:
        if v.nvmlReturn != 0:
            return None
        out.append(int(v.value.ullVal) * 1024)  # KiB -> bytes
    return out


def measure(handle, fn, iters):
    torch.cuda.synchronize()
    dist.barrier()
    time.sleep(0.2)
    c0 = counters(handle)
    for _ in range(iters):
        fn()
    torch.cuda.synchronize()
    dist.barrier()
    time.sleep(1.2)  # the counters are refreshed by the driver, not instantaneously
    c1 = counters(handle)
    if c0 is None or c1 is None:
        return None
    return {"tx_per_iter": (c1[0] - c0[0]) / iters, "rx_per_iter": (c1[1] - c0[1]) / iters}


def main():
    rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
    torch.cuda.set_device(int(os.environ.get("LOCAL_RANK", rank)))
    dist.init_process_group("nccl", device_id=torch.device("cuda", torch.cuda.current_device()))
    import pynvml

    pynvml.nvmlInit()
    uuid = torch.cuda.get_device_properties(torch.cuda.current_device()).uuid
    handle = None
    for i in range(pynvml.nvmlDeviceGetCount()):
        h = pynvml.nvmlDeviceGetHandleByIndex(i)
        u = pynvml.nvmlDeviceGetUUID(h)
        u = u.decode() if isinstance(u, bytes) else u
        if u.replace("GPU-", "") == str(uuid).replace("GPU-", ""):
            handle = h
    if handle is None:
        handle = pynvml.nvmlDeviceGetHandleByIndex(torch.cuda.current_device())
    res = {"rank": rank, "world": world}

    from paper_2507_17087_b200.executors.grid3d import MappedGemm3D

    for name, (M, N, K) in (("johnson3d_16384", (16384, 16384, 16384)),
                            ("cosma_32768x8192x8192", (32768, 8192, 8192))):
        ex = MappedGemm3D(M, N, K, mapping="decompose", rank=rank, world=world, seed=1)
        for _ in range(2):
            ex.step()
        ex.result()
        m = measure(handle, ex.step, 10)
        ex.result()
        res[name] = {"grid": list(ex.grid), "algorithmic_per_gpu": ex.comm, "nvlink": m}
        dist.barrier()
        ex.close()
        del ex
        torch.cuda.empty_cache()

    from paper_2507_17087_b200.executors.stencil import MappedStencil

    for mapping in ("decompose", "heuristic"):
        ex = MappedStencil(32768, 32768, mapping=mapping, rank=rank, world=world, seed=1)
        ex.run(5)
        m = measure(handle, lambda: ex.run(1), 200)
        r0, r1, c0, c1 = ex.rects[rank]
        halo_in = sum((c1 - c0) if d < 2 else (r1 - r0)
                      for d, q in enumerate(ex.nbrs) if q is not None)
        res[f"stencil_{mapping}"] = {"grid": list(ex.grid), "halo_cells_read_per_sweep": halo_in,
                                     "algorithmic_bytes_per_sweep": 4 * halo_in, "nvlink": m}
        dist.barrier()
        ex.close()
        del ex
        torch.cuda.empty_cache()

    from paper_2507_17087_b200.executors.circuit import CircuitSpec, MappedCircuit

    spec = CircuitSpec(96 * world, 5000, 20000, pct_in=95, steps=100, seed=7)
    for mapping in ("block", "cyclic"):
        ex = MappedCircuit(spec, mapping=mapping, rank=rank, world=world)
        ex.step()
        m = measure(handle, ex.step, 5)
        w = ex.work()
        res[f"circuit_{mapping}"] = {"cross_gpu_wires": w["cross_gpu_wires"],
                                     "algorithmic_bytes_per_iteration": 8 * w["cross_gpu_wires"],
                                     "nvlink": m}
        dist.barrier()
        ex.close()
        del ex

    from paper_2507_17087_b200.executors.hydro import HydroSpec, MappedHydro

    ex = MappedHydro(HydroSpec(16384, 4096), mapping="decompose", rank=rank, world=world)
    ex.step()
    m = measure(handle, ex.step, 20)
    res["hydro"] = {"cross_gpu_corners": ex.cross_corners,
                    "algorithmic_bytes_per_step": 24 * ex.cross_corners, "nvlink": m}
    dist.barrier()
    ex.close()

    allr = [None] * world
    dist.all_gather_object(allr, res)
    if rank == 0:
        print(json.dumps(allr))
    dist.barrier()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
