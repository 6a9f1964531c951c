"""Device time of the pivoted QR inside rid.decompose (diag t_qrcp, median of 20 calls) per
config or shape, for QR variant comparisons.   python tools/qr_time.py C1 C2 [m,n,k,l,noise ...]
RID_QRCP_VARIANT selects the kernel (tests/test_gpu_qrcp_variants.py lists them)."""
import os
import sys

sys.path.insert(0, os.getcwd())
import numpy as np  # noqa: E402

import paper_1205_3830_b200 as rid  # noqa: E402
from paper_1205_3830_b200.configs import CONFIGS  # noqa: E402

for arg in sys.argv[1:]:
    if arg in CONFIGS:
        c = CONFIGS[arg]
        m, n, k, l, noise = c.m, c.n, c.k, c.l, c.noise
    else:
        m, n, k, l = (int(x) for x in arg.split(",")[:4])
        noise = float(arg.split(",")[4])
    A = rid.generate(1, m, n, k, noise)
    for _ in range(3):
        rid.decompose(A, k, l, 1)
    tq, tt = [], []
    for _ in range(20):
        r = rid.decompose(A, k, l, 1)
        tq.append(r.diag["t_qrcp"] * 1e3)
        tt.append(r.diag["t_total"] * 1e3)
    print(f"{arg} variant {os.environ.get('RID_QRCP_VARIANT', 'default')}: qr median "
          f"{np.median(tq):.4f} ms (min {min(tq):.4f}), decompose device span median "
          f"{np.median(tt):.4f} ms", flush=True)
