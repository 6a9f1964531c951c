"""Time the error estimate (q iterations) at configs: s per iteration and GB/s over 2 passes."""
import os
import sys
import time

sys.path.insert(0, os.getcwd())
import torch  # noqa: E402

import paper_1205_3830_b200 as rid  # noqa: E402
from paper_1205_3830_b200.configs import CONFIGS  # noqa: E402

for name in sys.argv[1:]:
    c = CONFIGS[name]
    A = rid.generate(1, c.m, c.n, c.k, c.noise)
    r = rid.decompose(A, c.k, c.l, 1)
    for var in ("1", "0"):
      os.environ["RID_EST_TMA"] = var
      rid.error_estimate(A, r.J, r.P, 2, 1)
      for q in (5, 15):
        torch.cuda.synchronize()
        ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        t0 = time.perf_counter()
        ev0.record()
        e = rid.error_estimate(A, r.J, r.P, q, 1)
        ev1.record()
        torch.cuda.synchronize()
        dt = time.perf_counter() - t0
        dd = ev0.elapsed_time(ev1) * 1e-3
        if q == 5:
            t5, d5 = dt, dd
        else:
            per = (dt - t5) / 10
            print(f"  device time per iteration {(dd - d5) / 10 * 1e3:.3f} ms "
                  f"(wall {per * 1e3:.3f} ms)", flush=True)
            print(f"{name} RID_EST_TMA={var}: est {e:.15e}  {per*1e3:.3f} ms per iteration  "
                  f"{2 * 16 * c.m * c.n / per / 1e12:.2f} TB/s over the two passes", flush=True)
    del A, r
    torch.cuda.empty_cache()
