"""3M (Gauss) vs 4M (ordered real embedding) sketch: accuracy against the oracle on the parity
shapes, and TFLOP/s (8 l m n convention and executed flops) on the configs.
    python tools/sketch3m_check.py [C4 C5 ...]"""
import os
import sys

sys.path.insert(0, os.getcwd())
import numpy as np  # noqa: E402
import torch  # noqa: E402

import oracle  # noqa: E402
import paper_1205_3830_b200 as rid  # noqa: E402
from paper_1205_3830_b200.configs import CONFIGS  # noqa: E402

oracle.build()
for (seed, m, n, k, noise, l) in [(1, 1024, 512, 16, 0.0, 24), (2, 2048, 300, 64, 1e-10, 80),
                                  (5, 2048, 270, 256, 1e-10, 272), (6, 1024, 540, 512, 1e-8, 528),
                                  (3, 8192, 200, 128, 1e-12, 144), (7, 3000, 9, 3, 0.0, 1)]:
    A = rid.generate(seed, m, n, k, noise)
    Yo = oracle.sketch(oracle.generate(seed, m, n, k, noise), seed, l)
    out = []
    for env in ("0", "1"):
        os.environ["RID_SKETCH_4M"] = env
        Y = rid.sketch(A, seed, l).cpu().numpy()
        out.append(np.linalg.norm(Y - Yo) / np.linalg.norm(Yo))
        out.append(np.abs(Y - Yo).max() / np.abs(Yo).max())
    print(f"m={m} n={n} l={l}: 3M rel fro {out[0]:.2e} max {out[1]:.2e} | 4M rel fro {out[2]:.2e} max {out[3]:.2e}",
          flush=True)

for name in sys.argv[1:]:
    c = CONFIGS[name]
    A = rid.generate(1, c.m, c.n, c.k, c.noise)
    Y = rid.colmajor_empty(c.l, c.n, device="cuda")
    st = torch.cuda.current_stream()
    for env in ("1", "0"):
        os.environ["RID_SKETCH_4M"] = env
        rid.sketch(A, 1, c.l, out=Y)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        reps = 5
        torch.cuda.synchronize()
        e0.record(st)
        for _ in range(reps):
            rid.sketch(A, 1, c.l, out=Y)
        e1.record(st)
        torch.cuda.synchronize()
        dt = e0.elapsed_time(e1) / reps * 1e-3
        f8 = 8.0 * c.l * c.m * c.n
        mults = 4 if env == "1" else 3
        print(f"{name} {mults}M: {dt*1e3:8.2f} ms  {f8/dt/1e12:6.2f} TF/s (8lmn)  "
              f"{f8*mults/4/dt/1e12:6.2f} TF/s executed  S={rid.sketch_splits(c.m, c.l, c.n)}", flush=True)
    os.environ.pop("RID_SKETCH_4M")
    del A, Y
    torch.cuda.empty_cache()
