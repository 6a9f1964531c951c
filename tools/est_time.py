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
    rid.error_estimate(A, r.J, r.P, 2, 1)
    for q in (5, 15):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        e = rid.error_estimate(A, r.J, r.P, q, 1)
        dt = time.perf_counter() - t0
        if q == 5:
            t5 = dt
        else:
            per = (dt - t5) / 10
            print(f"{name}: est {e:.6e}  {per*1e3:.3f} ms per iteration  "
                  f"{2 * 16 * c.m * c.n / per / 1e12:.2f} TB/s over the two passes", flush=True)
    del A, r
    torch.cuda.empty_cache()
