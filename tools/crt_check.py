"""The modular integer sketch (k_crt.cu, RID_SKETCH_CRT=1) against the default DMMA sketch and
the oracle: accuracy (relative Frobenius difference, sampled oracle columns) and device time.

    python tools/crt_check.py small C2 C3 C4 [--reps 3] [--T 14]
"""
import json
import os
import sys

sys.path.insert(0, os.getcwd())
import numpy as np  # noqa: E402
import torch  # noqa: E402

import oracle  # noqa: E402
import paper_1205_3830_b200 as rid  # noqa: E402
from paper_1205_3830_b200.configs import CONFIGS  # noqa: E402

args = sys.argv[1:]
reps = int(args[args.index("--reps") + 1]) if "--reps" in args else 3
if "--T" in args:
    os.environ["RID_CRT_MODULI"] = args[args.index("--T") + 1]
names = [a for a in args if not a.startswith("--") and not a.isdigit()] or ["small"]
ctx = rid.Context(0, torch.cuda.current_stream())


def timed(A, l, seed, crt):
    os.environ["RID_SKETCH_CRT"] = "1" if crt else "0"
    Y = rid.sketch(A, seed, l, ctx=ctx)
    torch.cuda.synchronize()
    ts = []
    for _ in range(reps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        rid.sketch(A, seed, l, out=Y, ctx=ctx)
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    os.environ.pop("RID_SKETCH_CRT", None)
    return Y, min(ts)


SHAPES = {"small": (1024, 512, 16, 24, 0.0), "tiny": (256, 128, 4, 16, 0.0),
          "ragged": (1000, 300, 10, 40, 1e-10)}
for name in names:
    if name in SHAPES:
        m, n, k, l, noise = SHAPES[name]
    else:
        c = CONFIGS[name]
        m, n, k, l, noise = c.m, c.n, c.k, c.l, c.noise
    A = rid.generate(1, m, n, k, noise, ctx=ctx)
    Yc, tc = timed(A, l, 1, True)
    Yd, td = timed(A, l, 1, False)
    d = torch.linalg.norm(Yc - Yd).item() / torch.linalg.norm(Yd).item()
    cols = sorted(set([0, 1, 127, 128, n // 2 + 5, n - 1]))
    errs = []
    for j in cols:
        a = oracle.generate(1, m, n, k, noise, j, 1)
        y = oracle.sketch(a, 1, l)[:, 0]
        errs.append(float(np.linalg.norm(Yc[:, j].cpu().numpy() - y) / np.linalg.norm(y)))
    f8 = 8.0 * l * m * n
    print(json.dumps({"shape": name, "m": m, "n": n, "l": l, "crt_ms": tc, "dmma_ms": td,
                      "crt_tflops_8lmn": f8 / tc / 1e9, "dmma_tflops_8lmn": f8 / td / 1e9,
                      "rel_frob_crt_vs_dmma": d, "oracle_col_rel_max": max(errs)}), flush=True)
