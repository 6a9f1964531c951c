"""Sketch kernel timing: cp.async kernel (RID_Z3_TMA=0) vs the TMA/mbarrier kernel at 2/3/4 stages.
    python tools/tma_sketch_time.py [C3 C4 ...]
Device time of rid.sketch (R fill + the sketch launches) with CUDA events, best and mean of reps."""
import os
import sys

sys.path.insert(0, os.getcwd())
import torch  # noqa: E402

import paper_1205_3830_b200 as rid  # noqa: E402
from paper_1205_3830_b200.configs import CONFIGS  # noqa: E402

VARIANTS = [("cp.async", {"RID_Z3_TMA": "0"}), ("tma3", {"RID_Z3_TMA": "1"}),
            ("tma2", {"RID_Z3_TMA": "1", "RID_Z3T_VARIANT": "2"}),
            ("tma4", {"RID_Z3_TMA": "1", "RID_Z3T_VARIANT": "4"})]
if os.environ.get("ORDER_VARIANTS"):
    VARIANTS = [("tma3", {"RID_Z3_TMA": "1"})] + [
        (f"ord{v}", {"RID_Z3_TMA": "1", "RID_Z3T_VARIANT": str(v)}) for v in (11, 12, 13)]

if os.environ.get("RS_VARIANTS"):  # 48-row tiles: sums in registers (3 stages) vs the Rs plane
    VARIANTS = [("regs3", {"RID_Z3_TMA": "1", "RID_Z3T_VARIANT": "3"}),
                ("rs3", {"RID_Z3_TMA": "1", "RID_Z3T_VARIANT": "30"}),
                ("rs2", {"RID_Z3_TMA": "1"})]
if os.environ.get("ROWS_VARIANTS"):
    VARIANTS = [("rows40", {"RID_Z3_TMA": "1", "RID_Z3_ROWS": "40"}),
                ("rows48", {"RID_Z3_TMA": "1", "RID_Z3_ROWS": "48"})]
names = sys.argv[1:] or ["C4"]
for name in names:
    c = CONFIGS[name]
    A = rid.generate(1, c.m, c.n, c.k, c.noise)
    Y = rid.colmajor_empty(c.l, c.n, device="cuda")
    reps = 5 if c.m * c.n >= 1 << 28 else 20
    for label, env in VARIANTS:
        for key in ("RID_Z3_TMA", "RID_Z3T_VARIANT", "RID_Z3_ROWS"):
            os.environ.pop(key, None)
        os.environ.update(env)
        for _ in range(2):
            rid.sketch(A, 1, c.l, out=Y)
        ts = []
        for _ in range(reps):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            rid.sketch(A, 1, c.l, out=Y)
            e1.record()
            torch.cuda.synchronize()
            ts.append(e0.elapsed_time(e1) * 1e-3)
        f8 = 8.0 * c.l * c.m * c.n
        best, mean = min(ts), sum(ts) / len(ts)
        print(f"{name} {label:9s} best {best * 1e3:8.3f} ms mean {mean * 1e3:8.3f} ms  "
              f"{f8 / best / 1e12:6.2f} TF/s (8lmn)  {0.75 * f8 / best / 1e12:6.2f} executed "
              f"({0.75 * f8 / best / 1e12 / 37.11:.3f} of DMMA peak)", flush=True)
