"""Single-GPU stencil ms/sweep for several rectangle shapes (the per-GPU rectangles of
the multi-GPU mappings), to separate shape effects from the exchange."""
import json
import sys

sys.path.insert(0, ".")
import torch
from paper_2507_17087_b200.executors.stencil import MappedStencil

out = {}
for shape in sys.argv[1:]:
    r, c = (int(x) for x in shape.split("x"))
    ex = MappedStencil(r, c, halo_check=False)
    ex.run(10)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    ex.run(40)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / 40
    out[shape] = {"ms": round(ms, 4), "gbs": round(8 * r * c / ms / 1e6, 1)}
    ex.close()
    del ex
    torch.cuda.empty_cache()
print(json.dumps(out))
