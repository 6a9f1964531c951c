"""Debug helper: run rid_qrcp (variant from RID_QRCP_VARIANT) on a Philox sketch-like Y of shape
l x n and compare J with variant 0. Usage: python tools/dbg_qrcp.py l n k"""
import os
import sys

sys.path.insert(0, os.getcwd())
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_1205_3830_b200 as rid  # noqa: E402

l, n, k = (int(x) for x in sys.argv[1:4])
Y = rid.normal_fill(7, 9, l, n)
# low-rank-ish: scale rows so the spectrum decays
Y.mul_(torch.logspace(0, -6, l, dtype=torch.float64, device="cuda")[:, None])
os.environ["RID_QRCP_VARIANT"] = "0"
J0 = rid.qrcp(Y, k)[0]
os.environ["RID_QRCP_VARIANT"] = "1"
J1 = rid.qrcp(Y, k)[0]
torch.cuda.synchronize()
J0 = np.asarray(J0.cpu() if hasattr(J0, "cpu") else J0)
J1 = np.asarray(J1.cpu() if hasattr(J1, "cpu") else J1)
print(f"l={l} n={n} k={k}: J equal {np.array_equal(J0, J1)}", flush=True)
