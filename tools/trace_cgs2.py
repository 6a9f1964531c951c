"""Per-phase timing of the persistent CGS2 kernel (k_cgs2_fused, RID_QRCP_TRACE) on a config.

    python tools/trace_cgs2.py C4
Stamps per step j (CTA 0, %globaltimer): 0 start, 1/2 coef/update pass 0 done, 3/4 pass 1 done,
5 q_j normalised, 6 own projection done, 7 candidates reduced (p_{j+1} known)."""
import os
import sys

sys.path.insert(0, os.getcwd())
import numpy as np  # noqa: E402

import paper_1205_3830_b200 as rid  # noqa: E402
from paper_1205_3830_b200.configs import CONFIGS  # noqa: E402

c = CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "C4"]
A = rid.generate(1, c.m, c.n, c.k, c.noise)
rid.decompose(A, c.k, c.l, 1, qr="cgs2")  # warm
path = f"gpurun_out/cgs2_trace_{c.name}.txt"
os.environ["RID_QRCP_TRACE"] = path
r = rid.decompose(A, c.k, c.l, 1, qr="cgs2")
del os.environ["RID_QRCP_TRACE"]
t = np.loadtxt(path, dtype=np.float64)[:, 1:]
t = t[1:-1]  # step 0 has no reorthogonalisation, the last step no projection
ph = {"coef0": t[:, 1] - t[:, 0], "upd0": t[:, 2] - t[:, 1], "coef1": t[:, 3] - t[:, 2],
      "upd1": t[:, 4] - t[:, 3], "normalise": t[:, 5] - t[:, 4], "project": t[:, 6] - t[:, 5],
      "choose": t[:, 7] - t[:, 6]}
tot = sum(v.sum() for v in ph.values()) / 1e6
print(f"{c.name}: t_qrcp {r.diag['t_qrcp']*1e3:.2f} ms; traced steps 1..k-2 {tot:.2f} ms")
print("  ".join(f"{k} {v.mean()/1e3:.2f} us" for k, v in ph.items()))
for a, b in [(1, 64), (64, 256), (256, 511)]:
    b = min(b, len(t))
    if a >= b:
        break
    print(f" steps {a}-{b}: " + "  ".join(f"{k} {v[a:b].mean()/1e3:.2f}" for k, v in ph.items()))
