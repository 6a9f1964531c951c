"""Sketch time against the K-slice count S (RID_SKETCH_SPLIT) at a config: wave quantisation of
the small configs.    python tools/split_sweep.py C2 [S ...]"""
import os
import sys

sys.path.insert(0, os.getcwd())
import torch  # noqa: E402

import paper_1205_3830_b200 as rid  # noqa: E402
from paper_1205_3830_b200.configs import CONFIGS  # noqa: E402

c = CONFIGS[sys.argv[1]]
A = rid.generate(1, c.m, c.n, c.k, c.noise)
Y = rid.colmajor_empty(c.l, c.n, device="cuda")
print(c.name, "default S =", rid.sketch_splits(c.m, c.l, c.n), flush=True)
for S in ["0"] + sys.argv[2:]:
    if S == "0":
        os.environ.pop("RID_SKETCH_SPLIT", None)
    else:
        os.environ["RID_SKETCH_SPLIT"] = S
    for _ in range(3):
        rid.sketch(A, 1, c.l, out=Y)
    ts = []
    for _ in range(20):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        rid.sketch(A, 1, c.l, out=Y)
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    f = 6.0 * c.l * c.m * c.n
    print(f"{c.name} S={S:>3s} best {min(ts):.4f} ms  executed {f / min(ts) / 1e9:.2f} TF/s "
          f"({f / min(ts) / 1e9 / 37.11:.3f})", flush=True)
