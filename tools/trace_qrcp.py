"""Per-step timing of the QRCP kernel (RID_QRCP_TRACE) on a config's sketch."""
import os, sys
sys.path.insert(0, os.getcwd())
import numpy as np, torch
import paper_1205_3830_b200 as rid
from paper_1205_3830_b200.configs import CONFIGS
c = CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "C4"]
A = rid.generate(1, c.m, c.n, c.k, c.noise)
path = f"gpurun_out/qrcp_trace_{c.name}.txt"
os.environ["RID_QRCP_TRACE"] = path
r = rid.decompose(A, c.k, c.l, 1)
t = np.loadtxt(path, dtype=np.float64)
t0 = t[0, 1]
d_piv = (t[:, 2] - t[:, 1]) / 1e3  # pivot reduce + Householder (us)
d_upd = (t[:, 3] - t[:, 2]) / 1e3  # update pass + publish
d_bar = (t[:, 4] - t[:, 3]) / 1e3  # grid barrier
tot = (t[-1, 4] - t[0, 1]) / 1e6
print(f"{c.name}: qrcp total {tot:.2f} ms (diag {r.diag['t_qrcp']*1e3:.2f} ms)")
for a, b in [(0, 64), (64, 128), (128, 256), (256, 384), (384, c.k)]:
    if a >= c.k: break
    b = min(b, c.k)
    print(f" steps {a:4d}-{b:4d}: pivot+hh {d_piv[a:b].mean():7.2f} us  update {d_upd[a:b].mean():8.2f} us  barrier {d_bar[a:b].mean():6.2f} us  (rows {c.l-a}..{c.l-b+1})")
