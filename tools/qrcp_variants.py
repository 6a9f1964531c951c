"""Compare the QRCP variants on a config's sketch: 0 = exact recompute every step (one persistent
kernel), 1 = blocked panels with norm downdating + tensor-core trailing update (default).
Reports t_qrcp (device events) per variant and checks J equal and P agreement.

    python tools/qrcp_variants.py C4 [nb ...]
"""
import os
import sys

sys.path.insert(0, os.getcwd())
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_1205_3830_b200 as rid  # noqa: E402
from paper_1205_3830_b200.configs import CONFIGS  # noqa: E402

c = CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "C4"]
nbs = [int(x) for x in sys.argv[2:]] or [16]
A = rid.generate(1, c.m, c.n, c.k, c.noise)


def run(variant, nb=None, reps=3):
    os.environ["RID_QRCP_VARIANT"] = str(variant)
    if nb:
        os.environ["RID_QRCP_NB"] = str(nb)
    ts = []
    for _ in range(reps):
        r = rid.decompose(A, c.k, c.l, 1)
        ts.append(r.diag["t_qrcp"])
    return r, min(ts)


r0, t0 = run(0)
J0, P0 = r0.J.cpu().numpy(), r0.P
print(f"{c.name}: exact-recompute qrcp {t0*1e3:.3f} ms  step {r0.diag['t_total']*1e3:.2f} ms")
for nb in nbs:
    r1, t1 = run(1, nb)
    J1 = r1.J.cpu().numpy()
    same = np.array_equal(J0, J1)
    dp = (torch.linalg.norm(r1.P - P0) / torch.linalg.norm(P0)).item() if same else float("nan")
    print(f"{c.name}: blocked nb={nb:2d} qrcp {t1*1e3:.3f} ms  step {r1.diag['t_total']*1e3:.2f} ms"
          f"  J equal {same}  |dP|/|P| {dp:.2e}  launches {r1.diag['launches']}")
