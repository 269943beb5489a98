"""K4 variants vs cuBLAS at one shape, interleaved launch by launch (same power state),
median of ROUNDS: default (wave barrier, raster group 4), group 2 / 8, no wave barrier.
python tools/gemm_vs_cublas.py M N K [ROUNDS]"""
import json
import os
import statistics
import sys

sys.path.insert(0, ".")
import torch  # noqa: E402

from paper_2507_17087_b200.gemm import tile_gemm  # noqa: E402

M, N, K = (int(x) for x in sys.argv[1:4])
rounds = int(sys.argv[4]) if len(sys.argv) > 4 else 5
A = torch.randn(M, K, device="cuda").to(torch.bfloat16)
Bt = torch.randn(N, K, device="cuda").to(torch.bfloat16)
C = torch.empty(M, N, device="cuda")
Cb = torch.empty(M, N, device="cuda", dtype=torch.bfloat16)
variants = {"k4": {}, "k4_nowave": {"PM_GEMM_WAVESYNC": "0"},
            "k4_pair256": {"PM_GEMM_KERNEL": "1"}, "k4_pair256_g4": {"PM_GEMM_KERNEL": "1", "PM_GEMM_GROUP": "4"},
            "cublas": None}
times = {k: [] for k in variants}
for _ in range(rounds):
    for name, env in variants.items():
        for k in ("PM_GEMM_GROUP", "PM_GEMM_WAVESYNC", "PM_GEMM_KERNEL"):
            os.environ.pop(k, None)
        if env:
            os.environ.update(env)
        if name == "cublas":
            fn = lambda: torch.matmul(A, Bt.t(), out=Cb)  # noqa: E731
        elif name == "k4_bf16out":
            fn = lambda: tile_gemm(A, Bt, Cb)  # noqa: E731
        else:
            fn = lambda: tile_gemm(A, Bt, C)  # noqa: E731
        fn()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        fn()
        e1.record()
        torch.cuda.synchronize()
        times[name].append(e0.elapsed_time(e1))
fl = 2.0 * M * N * K
print(json.dumps({"shape": [M, N, K], "rounds": rounds,
                  **{k: {"ms": round(statistics.median(v), 3),
                         "tflops": round(fl / statistics.median(v) / 1e9)} for k, v in times.items()}}))
