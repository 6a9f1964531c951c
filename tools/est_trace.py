"""Per-kernel device timeline of one error estimate (torch.profiler / CUPTI, no nsys needed):
kernel durations and the idle gaps between them in a real back-to-back run.
    python tools/est_trace.py [C4] [q]"""
import os
import sys

sys.path.insert(0, os.getcwd())
import torch  # noqa: E402
from torch.profiler import ProfilerActivity, profile  # noqa: E402

import paper_1205_3830_b200 as rid  # noqa: E402
from paper_1205_3830_b200.configs import CONFIGS  # noqa: E402

c = CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "C4"]
q = int(sys.argv[2]) if len(sys.argv) > 2 else 3
A = rid.generate(1, c.m, c.n, c.k, c.noise)
r = rid.decompose(A, c.k, c.l, 1)
rid.error_estimate(A, r.J, r.P, q, 1)
torch.cuda.synchronize()
with profile(activities=[ProfilerActivity.CUDA]) as prof:
    rid.error_estimate(A, r.J, r.P, q, 1)
    torch.cuda.synchronize()
ev = sorted([e for e in prof.events() if e.device_type.name == "CUDA"],
            key=lambda e: e.time_range.start)
prev = None
for e in ev:
    gap = (e.time_range.start - prev) if prev is not None else 0
    print(f"{e.name[:44]:44s} start {e.time_range.start:12.1f} dur {e.time_range.elapsed_us():9.1f} us"
          f"  gap {gap:8.1f} us")
    prev = e.time_range.end
