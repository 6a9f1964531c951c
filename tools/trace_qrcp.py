"""Per-step timing of the QRCP kernels (RID_QRCP_TRACE) on a config's sketch.

    python tools/trace_qrcp.py C4 [variant]      variant: 1 blocked (default), 0 exact recompute
Stamps per step (CTA 0, %globaltimer): start, reflector ready, own pass + publish done, barrier
passed. For the blocked variant the time between the last step of a panel and the first of the
next (the tensor-core trailing update + launch) is reported as "panel gap"."""
import os
import sys

sys.path.insert(0, os.getcwd())
import numpy as np  # noqa: E402

import paper_1205_3830_b200 as rid  # noqa: E402
from paper_1205_3830_b200.configs import CONFIGS  # noqa: E402

c = CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "C4"]
variant = sys.argv[2] if len(sys.argv) > 2 else "1"
os.environ["RID_QRCP_VARIANT"] = variant
A = rid.generate(1, c.m, c.n, c.k, c.noise)
rid.decompose(A, c.k, c.l, 1)  # warm
path = f"gpurun_out/qrcp_trace_{c.name}_v{variant}.txt"
os.environ["RID_QRCP_TRACE"] = path
r = rid.decompose(A, c.k, c.l, 1)
del os.environ["RID_QRCP_TRACE"]
t = np.loadtxt(path, dtype=np.float64)
d_piv = (t[:, 2] - t[:, 1]) / 1e3  # pivot reduce + Householder (us)
d_upd = (t[:, 3] - t[:, 2]) / 1e3  # pass + publish
d_bar = (t[:, 4] - t[:, 3]) / 1e3  # grid barrier
gap = (t[1:, 1] - t[:-1, 4]) / 1e3  # between steps (kernel boundary for the blocked variant)
tot = (t[-1, 4] - t[0, 1]) / 1e6
print(f"{c.name} variant {variant}: qrcp traced span {tot:.2f} ms (diag t_qrcp {r.diag['t_qrcp']*1e3:.2f} ms)"
      f"; sum pivot+hh {d_piv.sum()/1e3:.2f} ms, pass {d_upd.sum()/1e3:.2f} ms, barrier {d_bar.sum()/1e3:.2f} ms,"
      f" gaps {gap.sum()/1e3:.2f} ms")
lazy = t.shape[1] > 8 and t[:, 7].any()
if t.shape[1] > 5 and t[:, 5].any() and not lazy:  # ring kernel: pivot | x-build | zlarfg + sv | G
    d_a = (t[:, 5] - t[:, 1]) / 1e3
    d_b = (t[:, 6] - t[:, 5]) / 1e3
    d_c = (t[:, 7] - t[:, 6]) / 1e3
    d_d = (t[:, 2] - t[:, 7]) / 1e3
    print(f" reflector phase split (mean us): pivot reduce {d_a.mean():.2f}, x-build {d_b.mean():.2f},"
          f" zlarfg+v {d_c.mean():.2f}, G {d_d.mean():.2f}")
edges = [0, 16, 64, 128, 256, 384, 512, 1024]
for a, b in zip(edges[:-1], edges[1:]):
    if a >= c.k:
        break
    b = min(b, c.k)
    print(f" steps {a:4d}-{b:4d}: pivot+hh {d_piv[a:b].mean():7.2f} us  pass {d_upd[a:b].mean():8.2f} us"
          f"  barrier {d_bar[a:b].mean():6.2f} us  gap {gap[a:b-1].mean() if b - 1 > a else 0:7.2f} us"
          f"  (rows {c.l-a}..{c.l-b+1})")
if lazy:  # lazy kernel: columns refreshed per step (all CTAs), retries; CTA 0's phase A / B ns
    print(f" lazy: CTA 0 grid-barrier wait {t[:, 5].sum()/1e6:.2f} ms, reading the candidates"
          f" {t[:, 6].sum()/1e6:.2f} ms (of the exchange, all passes of a step)")
    print(f" lazy: columns refreshed {t[:, 7].sum():.0f} (full refresh would be "
          f"{sum(c.n - j for j in range(c.k))}), retried steps {int((t[:, 8] > 0).sum())}")
    for a, b in zip(edges[:-1], edges[1:]):
        if a >= c.k:
            break
        b = min(b, c.k)
        print(f"  steps {a:4d}-{b:4d}: refreshed/step {t[a:b, 7].mean():9.1f}  retries {int(t[a:b, 8].sum())}")
