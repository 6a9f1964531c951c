"""CUPTI timeline (torch.profiler) of one rid_decompose at a config: kernels and the idle gaps
between them.    python tools/decompose_trace.py C1"""
import os
import sys

sys.path.insert(0, os.getcwd())
import torch  # noqa: E402
from torch.profiler import ProfilerActivity, profile  # noqa: E402

import paper_1205_3830_b200 as rid  # noqa: E402
from paper_1205_3830_b200.configs import CONFIGS  # noqa: E402

c = CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "C1"]
A = rid.generate(1, c.m, c.n, c.k, c.noise)
for _ in range(3):
    rid.decompose(A, c.k, c.l, 1)
torch.cuda.synchronize()
with profile(activities=[ProfilerActivity.CUDA]) as prof:
    r = rid.decompose(A, c.k, c.l, 1)
    torch.cuda.synchronize()
ev = sorted([e for e in prof.events() if e.device_type.name == "CUDA"],
            key=lambda e: e.time_range.start)
t0 = ev[0].time_range.start
prev = None
busy = 0.0
for e in ev:
    gap = (e.time_range.start - prev) if prev is not None else 0
    busy += e.time_range.elapsed_us()
    print(f"{e.name[:50]:50s} at {e.time_range.start - t0:9.1f} dur {e.time_range.elapsed_us():8.1f} us"
          f"  gap {gap:7.1f}")
    prev = e.time_range.end
span = ev[-1].time_range.end - t0
print(f"span {span:.1f} us, busy {busy:.1f} us, diag t_total {r.diag['t_total'] * 1e6:.1f} us")
