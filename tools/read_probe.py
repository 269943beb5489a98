"""HBM read ceiling on this box (pure 16-byte streaming loads over 4.29 GB) at several grid
shapes, beside the fill_ write ceiling: what K2's histogram and K3's count pass can reach."""
import ctypes
import os
import sys

sys.path.insert(0, ".")
import torch  # noqa: E402

so = os.path.join(os.path.dirname(__file__), "probe_src", "read_probe.so")
lib = ctypes.CDLL(so)
lib.launch.argtypes = [ctypes.c_int, ctypes.c_void_p, ctypes.c_longlong, ctypes.c_void_p,
                       ctypes.c_longlong, ctypes.c_void_p]
n = 1 << 30
x = torch.randint(0, 8, (n,), dtype=torch.int32, device="cuda")
out = torch.zeros(1 << 22, dtype=torch.int32, device="cuda")
n4 = n // 4
sms = torch.cuda.get_device_properties(0).multi_processor_count
s = torch.cuda.current_stream().cuda_stream


def t(fn, reps=5):
    for _ in range(2):
        fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps


for which in (0, 1):
    for label, blocks in (("8/SM", sms * 8), ("32/SM", sms * 32), ("iters4", n4 // (256 * 4)),
                          ("iters16", n4 // (256 * 16)), ("iters1", n4 // 256)):
        ms = t(lambda: lib.launch(which, x.data_ptr(), n4, out.data_ptr(), blocks, s))
        print(f"read{'_unroll4' if which else ''} {label:8s} {ms:.4f} ms {4 * n / ms / 1e6:.0f} GB/s")
ms = t(lambda: x.fill_(3))
print(f"fill_ {ms:.4f} ms {4 * n / ms / 1e6:.0f} GB/s")
ms = t(lambda: x.sum())
print(f"torch sum {ms:.4f} ms {4 * n / ms / 1e6:.0f} GB/s")
