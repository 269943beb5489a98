"""N=1 SUMMA: the step-program step vs the bare GEMM launch vs per-launch events, back to
back on the same operands (where does the bench's value-vs-roofline gap come from?)."""
import json
import sys

sys.path.insert(0, ".")
import torch  # noqa: E402

from paper_2507_17087_b200.executors.summa import MappedGemm  # noqa: E402
from paper_2507_17087_b200.gemm import tile_gemm  # noqa: E402

ex = MappedGemm(32768, 32768, 32768, mapping="decompose", seed=1234)
cs = torch.cuda.current_stream()
out = {}


def loop(name, fn, n=10):
    for _ in range(2):
        fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(cs)
    for _ in range(n):
        fn()
    e1.record(cs)
    torch.cuda.synchronize()
    out[name] = round(e0.elapsed_time(e1) / n, 3)


def per_launch(n=10):
    evs = []
    for _ in range(n):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(cs)
        tile_gemm(ex.A, ex.Bt, ex.C)
        b.record(cs)
        evs.append((a, b))
    torch.cuda.synchronize()
    out["per_launch_events"] = round(sum(a.elapsed_time(b) for a, b in evs) / n, 3)


for rep in range(2):
    loop(f"step_{rep}", ex.step)
    loop(f"tile_gemm_{rep}", lambda: tile_gemm(ex.A, ex.Bt, ex.C))
    per_launch()
    out[f"per_launch_{rep}"] = out.pop("per_launch_events")
print(json.dumps(out))
