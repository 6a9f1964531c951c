"""One C-config sketch through the modular integer path (RID_SKETCH_CRT=1) after one warm-up call:
the command the ncu launch list / full set of the CRT kernels are taken on.

    RID_SKETCH_CRT=1 python tools/crt_one.py C4
"""
import os
import sys

sys.path.insert(0, os.getcwd())
import torch  # noqa: E402

import paper_1205_3830_b200 as rid  # noqa: E402
from paper_1205_3830_b200.configs import CONFIGS  # noqa: E402

c = CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "C4"]
ctx = rid.Context(0, torch.cuda.current_stream())
A = rid.generate(1, c.m, c.n, c.k, c.noise, ctx=ctx)
Y = rid.sketch(A, 1, c.l, ctx=ctx)
torch.cuda.synchronize()
rid.sketch(A, 1, c.l, out=Y, ctx=ctx)
torch.cuda.synchronize()
print("ok", float(Y.abs().max()))
