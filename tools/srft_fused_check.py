"""The single-pass SRFT (k_srft_fused) against the two-pass one (RID_SRFT_FUSED=0) and the oracle's
direct sums: device time of rid.sketch_srft and accuracy per config.
    python tools/srft_fused_check.py C2 C3 C4 C5"""
import json
import os
import sys

sys.path.insert(0, os.getcwd())
import numpy as np  # noqa: E402
import torch  # noqa: E402

import oracle  # noqa: E402
import paper_1205_3830_b200 as rid  # noqa: E402
from paper_1205_3830_b200.configs import CONFIGS  # noqa: E402


def timed(A, l, env, reps=3):
    if env is None:
        os.environ.pop("RID_SRFT_FUSED", None)
    else:
        os.environ["RID_SRFT_FUSED"] = env
    Y = rid.sketch_srft(A, 1, l)
    torch.cuda.synchronize()
    ts = []
    for _ in range(reps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        rid.sketch_srft(A, 1, l, out=Y)
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    os.environ.pop("RID_SRFT_FUSED", None)
    return Y, min(ts)


for name in [a for a in sys.argv[1:] if not a.startswith("-")] or ["C4"]:
    c = CONFIGS[name]
    A = rid.generate(1, c.m, c.n, c.k, c.noise)
    Yf, tf = timed(A, c.l, None)
    Y2, t2 = timed(A, c.l, "0")
    d, s = oracle.srft_plan(1, c.m, c.l)
    errs = []
    for j in (0, 1, c.n // 2, c.n - 1):
        a = oracle.generate(1, c.m, c.n, c.k, c.noise, j, 1)
        y = oracle.srft_apply(d, s, a)[:, 0]
        errs.append(float(np.linalg.norm(Yf[:, j].cpu().numpy() - y) / np.linalg.norm(y)))
    rel = (torch.linalg.norm(Yf - Y2) / torch.linalg.norm(Y2)).item()
    print(json.dumps({"config": name, "fused_ms": tf, "two_pass_ms": t2,
                      "fused_hbm_frac": 16.0 * c.m * c.n / (tf * 1e-3) / 6536.7e9,
                      "rel_fused_vs_two_pass": rel, "rel_col_vs_oracle_max": max(errs)}), flush=True)
    del A, Yf, Y2
    torch.cuda.empty_cache()
