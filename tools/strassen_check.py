"""The Strassen sketch (k_strassen.cu) against the plain 3M sketch and the oracle: accuracy and
device time per config.

    python tools/strassen_check.py C4 C5 [--reps 5]
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

names = [a for a in sys.argv[1:] if not a.startswith("--")] or ["C4"]
reps = 5
ctx = rid.Context(0, torch.cuda.current_stream())


def timed(A, l, seed, env):
    old = os.environ.get("RID_SKETCH_STRASSEN")
    if env is None:
        os.environ.pop("RID_SKETCH_STRASSEN", None)
    else:
        os.environ["RID_SKETCH_STRASSEN"] = env
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
    if old is None:
        os.environ.pop("RID_SKETCH_STRASSEN", None)
    else:
        os.environ["RID_SKETCH_STRASSEN"] = old
    return Y, min(ts)


for name in names:
    c = CONFIGS[name]
    A = rid.generate(1, c.m, c.n, c.k, c.noise, ctx=ctx)
    Ys, ts = timed(A, c.l, 1, None)
    Y3, t3 = timed(A, c.l, 1, "0")
    d = torch.linalg.norm(Ys - Y3).item() / torch.linalg.norm(Y3).item()
    cols = [0, 31, 32, 63, 64, c.n // 2 + 5, c.n - 1]
    errs = []
    for j in cols:
        a = oracle.generate(1, c.m, c.n, c.k, c.noise, j, 1)
        y = oracle.sketch(a, 1, c.l)[:, 0]
        errs.append(float(np.linalg.norm(Ys[:, j].cpu().numpy() - y) / np.linalg.norm(y)))
    f8 = 8.0 * c.l * c.m * c.n
    print(json.dumps({"config": name, "strassen_ms": ts, "plain3m_ms": t3,
                      "strassen_tflops_8lmn": f8 / ts / 1e9, "plain3m_tflops_8lmn": f8 / t3 / 1e9,
                      "strassen_exec_frac": 5.25 * c.l * c.m * c.n / ts / 1e9 / 37.08,
                      "rel_fro_vs_3m": d, "rel_col_vs_oracle_max": max(errs)}), flush=True)
    del A, Ys, Y3
    torch.cuda.empty_cache()
