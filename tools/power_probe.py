"""Sustained GEMM probe: TFLOP/s, SM clock and board power for pm_gemm vs torch.matmul
(back-to-back launches for a few seconds each, nvidia-smi sampled meanwhile)."""
import subprocess
import statistics
import sys
import threading
import time

sys.path.insert(0, ".")
import torch  # noqa: E402

from paper_2507_17087_b200.gemm import tile_gemm  # noqa: E402


def sample(stop, out):
    p = subprocess.Popen(["nvidia-smi", "--id=0", "--query-gpu=clocks.sm,power.draw",
                          "--format=csv,noheader,nounits", "-lms", "100"],
                         stdout=subprocess.PIPE, text=True)
    while not stop.is_set():
        line = p.stdout.readline()
        if line:
            out.append([float(x) for x in line.split(",")])
    p.terminate()


def run(name, fn, flops, secs):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    stop, out = threading.Event(), []
    t = threading.Thread(target=sample, args=(stop, out))
    t.start()
    time.sleep(0.3)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    n = 0
    e0.record()
    t0 = time.time()
    while time.time() - t0 < secs:
        fn()
        n += 1
        if n % 4 == 0:
            torch.cuda.synchronize()
    e1.record()
    torch.cuda.synchronize()
    stop.set()
    t.join()
    ms = e0.elapsed_time(e1) / n
    load = out[len(out) // 4:] or out
    clk = statistics.median(x[0] for x in load)
    pw = statistics.mean(x[1] for x in load)
    print(f"{name}: {flops / ms / 1e9:.1f} TF/s  sm {clk:.0f} MHz  {pw:.0f} W  "
          f"({flops / ms / 1e9 / clk:.3f} TF/s per MHz)", flush=True)


n = int(sys.argv[1]) if len(sys.argv) > 1 else 16384
secs = float(sys.argv[2]) if len(sys.argv) > 2 else 4
A = torch.randn(n, n, device="cuda").to(torch.bfloat16)
Bt = torch.randn(n, n, device="cuda").to(torch.bfloat16)
C = torch.empty(n, n, device="cuda")
Cb = torch.empty(n, n, device="cuda", dtype=torch.bfloat16)
fl = 2 * n ** 3
run("pm_gemm fp32-out", lambda: tile_gemm(A, Bt, C), fl, secs)
run("torch.matmul bf16-out", lambda: torch.matmul(A, Bt.T, out=Cb), fl, secs)
run("pm_gemm bf16-out", lambda: tile_gemm(A, Bt, Cb), fl, secs)
run("pm_gemm fp32-out", lambda: tile_gemm(A, Bt, C), fl, secs)
