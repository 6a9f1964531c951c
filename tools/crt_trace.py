"""CUPTI timeline (torch.profiler) of one modular integer sketch (RID_SKETCH_CRT=1): each kernel's
start, duration and stream, to see how the column-block pipeline overlaps.

    python tools/crt_trace.py C4
"""
import os
import sys

sys.path.insert(0, os.getcwd())
os.environ.setdefault("RID_SKETCH_CRT", "1")
import torch  # noqa: E402
from torch.profiler import ProfilerActivity, profile  # noqa: E402

import paper_1205_3830_b200 as rid  # noqa: E402
from paper_1205_3830_b200.configs import CONFIGS  # noqa: E402

c = CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "C4"]
ctx = rid.Context(0, torch.cuda.current_stream())
A = rid.generate(1, c.m, c.n, c.k, c.noise, ctx=ctx)
Y = rid.sketch(A, 1, c.l, ctx=ctx)
torch.cuda.synchronize()
with profile(activities=[ProfilerActivity.CUDA]) as prof:
    rid.sketch(A, 1, c.l, out=Y, ctx=ctx)
    torch.cuda.synchronize()
ev = sorted([e for e in prof.events() if e.device_type.name == "CUDA"],
            key=lambda e: e.time_range.start)
t0 = ev[0].time_range.start
for e in ev:
    print(f"{e.name[:44]:44s} start {(e.time_range.start - t0) / 1e3:8.3f} ms  dur "
          f"{e.time_range.elapsed_us() / 1e3:7.3f} ms")
print(f"span {(ev[-1].time_range.end - t0) / 1e3:.3f} ms")
