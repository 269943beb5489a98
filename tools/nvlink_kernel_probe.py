"""Single-process, two-GPU NVLink probe of the fused peer kernels (ncu target).

One process drives GPU 0 and GPU 1 with peer access enabled, so ncu can replay
every kernel (no cross-process barriers) and report its NVLink bytes
(nvlrx__bytes / nvltx__bytes, user data) beside the algorithmic bytes:
  gemm_peer_add   pm_gemm_bf16 on GPU 0 reduce-adding its fp32 C tile straight
                  into GPU 1's memory (TMA .add epilogue; the 3-D / 2.5D
                  executors' fused reduce-scatter): M * N * 4 bytes;
  copy2d_pull     pm_copy2d_async of a panel from GPU 1 into GPU 0 (the SUMMA /
                  3-D all-gather pulls, copy engines -- no kernel, shown by the
                  stencil/gemm counters only; timed here);
  stencil_peer    pm_stencil_sweep on GPU 0 whose down neighbour's rows and right
                  neighbour's column strip live on GPU 1 (sweep 0: no flag waits):
                  4 B per halo cell read;
  hydro_peer_zones the zone kernel on GPU 0 with every point on GPU 1: 16-byte
                  point-state loads and 2 x 4-byte force atomics per corner.

    ncu --metrics nvlrx__bytes_data_user.sum,nvltx__bytes_data_user.sum,gpu__time_duration.sum \
        python tools/nvlink_kernel_probe.py
"""

import ctypes
import json
import sys

sys.path.insert(0, ".")
import torch  # noqa: E402

from paper_2507_17087_b200 import native  # noqa: E402
from paper_2507_17087_b200.executors.stencil import PmStencilView  # noqa: E402


def enable_peer(a, b):
    rt = ctypes.CDLL("libcudart.so")
    with torch.cuda.device(a):
        rc = rt.cudaDeviceEnablePeerAccess(b, 0)
        if rc not in (0, 704):  # 704: already enabled
            raise RuntimeError(f"cudaDeviceEnablePeerAccess({a}->{b}) = {rc}")


def main():
    assert torch.cuda.device_count() >= 2, "needs 2 GPUs"
    enable_peer(0, 1)
    enable_peer(1, 0)
    lib = native.lib()
    out = {}
    # 1. GEMM with the C tile reduce-added into the peer GPU
    M = N = 8192
    K = 4096
    A = torch.randn(M, K, device="cuda:0").to(torch.bfloat16)
    Bt = torch.randn(N, K, device="cuda:0").to(torch.bfloat16)
    C1 = torch.zeros(M, N, device="cuda:1")
    torch.cuda.synchronize(0)
    torch.cuda.synchronize(1)
    with torch.cuda.device(0):
        s = native.stream_ptr(torch.cuda.current_stream(0))
        for _ in range(2):
            native.check(lib.pm_gemm_bf16(A.data_ptr(), K, Bt.data_ptr(), K, C1.data_ptr(), N,
                                          M, N, K, 0, 2, s), "pm_gemm_bf16")
        torch.cuda.synchronize(0)
    ref = 2 * (A.float() @ Bt.float().T).to("cuda:1")
    err = float((C1 - ref).abs().max() / ref.abs().max())
    out["gemm_peer_add"] = {"M": M, "N": N, "K": K, "algorithmic_nvlink_bytes": M * N * 4,
                            "rel_err": err}
    # 2. copy-engine pull GPU 1 -> GPU 0
    src = torch.randn(8192, 8192, device="cuda:1").to(torch.bfloat16)
    dst = torch.empty_like(src, device="cuda:0")
    with torch.cuda.device(0):
        st = torch.cuda.current_stream(0)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(st)
        native.check(lib.pm_copy2d_async(dst.data_ptr(), 8192 * 2, src.data_ptr(), 8192 * 2,
                                         8192 * 2, 8192, native.stream_ptr(st)), "pm_copy2d")
        e1.record(st)
        torch.cuda.synchronize(0)
        ms = e0.elapsed_time(e1)
    out["copy2d_pull"] = {"bytes": 8192 * 8192 * 2, "ms": ms,
                          "gbs": 8192 * 8192 * 2 / ms / 1e6, "ok": bool(torch.equal(dst.cpu(), src.cpu()))}
    # 3. stencil sweep with peer neighbours (down rows, right column strip) on GPU 1
    R = Cc = 16384
    pitch = Cc
    inb = torch.rand(R, pitch, device="cuda:0")
    outb = torch.zeros(R, pitch, device="cuda:0")
    down = torch.rand(R, pitch, device="cuda:1")       # down neighbour's rectangle
    rstrip = torch.rand(2, R, device="cuda:1")         # right neighbour's column strips
    mystrips = torch.zeros(2, R, device="cuda:0")
    flags = torch.zeros(4, dtype=torch.int32, device="cuda:0")
    pflags = torch.zeros(4, dtype=torch.int32, device="cuda:1")
    v = PmStencilView()
    v.out, v.in_ = outb.data_ptr(), inb.data_ptr()
    v.rows, v.cols, v.pitch = R, Cc, pitch
    v.grow0, v.gcol0, v.grows, v.gcols = 0, 0, 2 * R, 2 * Cc
    v.nbr[1], v.nbr_pitch[1], v.nbr_rows[1], v.nbr_cols[1] = down.data_ptr(), pitch, R, Cc
    v.nbr[3], v.nbr_pitch[3], v.nbr_rows[3], v.nbr_cols[3] = down.data_ptr(), pitch, R, Cc
    v.nbr_rank[1], v.nbr_rank[3] = 1, 2
    v.nbr_flag_slot[1] = pflags.data_ptr()
    v.nbr_flag_slot[3] = pflags.data_ptr() + 4
    v.my_flags = flags.data_ptr()
    v.col_out[0], v.col_out[1] = mystrips[0].data_ptr(), mystrips[1].data_ptr()
    v.nbr_col[1] = rstrip[0].data_ptr()
    torch.cuda.synchronize(1)
    with torch.cuda.device(0):
        s = native.stream_ptr(torch.cuda.current_stream(0))
        for _ in range(2):
            native.check(lib.pm_stencil_sweep(ctypes.byref(v), 0, s), "pm_stencil_sweep")
        torch.cuda.synchronize(0)
    out["stencil_peer"] = {"rect": [R, Cc], "halo_cells_read": 2 * R,
                           "algorithmic_nvlink_bytes": 4 * 2 * R}
    # 4. hydro zones on GPU 0 whose points all live on GPU 1: every corner is a 16-byte
    #    peer load of the point state and two 4-byte peer float atomics of its force
    from paper_2507_17087_b200.executors.hydro import PmHydroView

    Lx = Ly = 1024
    nz, npt = Lx * Ly, (Lx + 1) * (Ly + 1)
    zi = torch.arange(nz, device="cuda:0") % Lx
    zj = torch.arange(nz, device="cuda:0") // Lx
    W = Lx + 1
    corners = [zj * W + zi, zj * W + zi + 1, (zj + 1) * W + zi + 1, (zj + 1) * W + zi]
    z2p = torch.stack([(1 << 27) | c for c in corners]).to(torch.int32).contiguous()
    zm = torch.full((nz,), 1.0 / nz, device="cuda:0")
    ze = torch.ones(nz, device="cuda:0")
    za = torch.full((nz,), 1.0 / nz, device="cuda:0")
    zpe = torch.zeros(nz, device="cuda:0")
    pst = torch.zeros(npt, 4, device="cuda:1")
    pst[:, 0] = (torch.arange(npt, device="cuda:1") % W).float() / Lx
    pst[:, 1] = (torch.arange(npt, device="cuda:1") // W).float() / Ly
    fxy = torch.zeros(2 * npt, device="cuda:1")
    hv = PmHydroView()
    hv.n_zones, hv.n_points = nz, 0
    hv.z2p, hv.zm, hv.ze, hv.za, hv.zpe = (z2p.data_ptr(), zm.data_ptr(), ze.data_ptr(),
                                           za.data_ptr(), zpe.data_ptr())
    hv.pm = hv.pbc = None
    hv.pst[1], hv.fxy[1] = pst.data_ptr(), fxy.data_ptr()
    hv.rank, hv.dt, hv.gamma, hv.cq = 0, 1e-6, 5.0 / 3.0, 1.0
    torch.cuda.synchronize(1)
    with torch.cuda.device(0):
        s = native.stream_ptr(torch.cuda.current_stream(0))
        for _ in range(2):
            native.check(lib.pm_hydro_step(ctypes.byref(hv), 0, s), "pm_hydro_step")
        torch.cuda.synchronize(0)
    out["hydro_peer_zones"] = {"zones": nz, "points_on_peer": npt,
                               "algorithmic_rx_bytes": 16 * 4 * nz,
                               "algorithmic_rx_bytes_unique_points": 16 * npt,
                               "algorithmic_tx_atomic_bytes": 8 * 4 * nz}
    print(json.dumps(out))


if __name__ == "__main__":
    main()
