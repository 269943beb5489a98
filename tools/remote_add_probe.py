"""Cost of the reduce-adding epilogue into a PEER GPU's C (the 3-D / 2.5D fused
reduce-scatter) against the same GEMM storing / adding locally: one process, GPUs 0 and 1
with peer access, CUDA events on GPU 0."""
import ctypes
import json
import sys

sys.path.insert(0, ".")
import torch  # noqa: E402

from paper_2507_17087_b200 import native  # noqa: E402


def main():
    rt = ctypes.CDLL("libcudart.so")
    for a, b in ((0, 1), (1, 0)):
        with torch.cuda.device(a):
            rc = rt.cudaDeviceEnablePeerAccess(b, 0)
            assert rc in (0, 704), rc
    lib = native.lib()
    out = {}
    for (M, N, K) in ((16384, 32768, 16384), (16384, 16384, 16384)):
        A = torch.randn(M, K, device="cuda:0").to(torch.bfloat16)
        Bt = torch.randn(N, K, device="cuda:0").to(torch.bfloat16)
        C0 = torch.zeros(M, N, device="cuda:0")
        C1 = torch.zeros(M, N, device="cuda:1")
        torch.cuda.synchronize(0)
        torch.cuda.synchronize(1)
        res = {}
        with torch.cuda.device(0):
            s = native.stream_ptr(torch.cuda.current_stream(0))
            seq = [("store_local", C0, 0), ("add_local", C0, 2), ("add_peer", C1, 2),
                   ("add_peer_nowave", C1, 2)] * 4
            import os
            for name, C, acc in seq:
                if name.endswith("_nowave"):
                    os.environ["PM_GEMM_WAVESYNC"] = "0"
                else:
                    os.environ.pop("PM_GEMM_WAVESYNC", None)
                for _ in range(2):
                    native.check(lib.pm_gemm_bf16(A.data_ptr(), K, Bt.data_ptr(), K, C.data_ptr(),
                                                  N, M, N, K, 0, acc, s), "gemm")
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record()
                for _ in range(5):
                    native.check(lib.pm_gemm_bf16(A.data_ptr(), K, Bt.data_ptr(), K, C.data_ptr(),
                                                  N, M, N, K, 0, acc, s), "gemm")
                e1.record()
                torch.cuda.synchronize(0)
                ms = e0.elapsed_time(e1) / 5
                res.setdefault(name, []).append(round(ms, 3))
        out[f"{M}x{N}x{K}"] = res
    print(json.dumps(out))


if __name__ == "__main__":
    main()
