"""Debug helper: the decompose of a config with the blocked QRCP (RID_QRCP_VARIANT=1), checked
against variant 0 (J equal, P close). python tools/dbg_qrcp_cfg.py C4"""
import os
import sys

sys.path.insert(0, os.getcwd())
import torch  # noqa: E402

import paper_1205_3830_b200 as rid  # noqa: E402
from paper_1205_3830_b200.configs import CONFIGS  # noqa: E402

c = CONFIGS[sys.argv[1]]
A = rid.generate(1, c.m, c.n, c.k, c.noise)
os.environ["RID_QRCP_VARIANT"] = "1"
r1 = rid.decompose(A, c.k, c.l, 1)
torch.cuda.synchronize()
print(f"{c.name}: blocked ok t_qrcp {r1.diag['t_qrcp']*1e3:.2f} ms", flush=True)
os.environ["RID_QRCP_VARIANT"] = "0"
r0 = rid.decompose(A, c.k, c.l, 1)
same = torch.equal(r0.J, r1.J)
print(f"{c.name}: J equal {same}; |dP|/|P| "
      f"{(torch.linalg.norm(r1.P - r0.P) / torch.linalg.norm(r0.P)).item():.2e}", flush=True)
