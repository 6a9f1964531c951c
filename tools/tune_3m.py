"""Time the 3M sketch kernel variants (RID_Z3_VARIANT, k_zgemm3m.cu) on configs.
    python tools/tune_3m.py C4,C5 1,2,3"""
import json
import os
import sys

sys.path.insert(0, os.getcwd())
import torch  # noqa: E402

import paper_1205_3830_b200 as rid  # noqa: E402
from paper_1205_3830_b200.configs import CONFIGS  # noqa: E402

cfgs = sys.argv[1].split(",")
variants = [int(x) for x in sys.argv[2].split(",")]
for cname in cfgs:
    c = CONFIGS[cname]
    A = rid.generate(1, c.m, c.n, c.k, c.noise)
    Y = rid.colmajor_empty(c.l, c.n, device="cuda")
    ref = None
    for v in variants:
        os.environ["RID_Z3_VARIANT"] = str(v)
        rid.sketch(A, 1, c.l, out=Y)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        reps = 3
        e0.record()
        for _ in range(reps):
            rid.sketch(A, 1, c.l, out=Y)
        e1.record()
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / reps
        if ref is None:
            ref = Y.clone()
            err = 0.0
        else:
            err = float(torch.linalg.norm(Y - ref) / torch.linalg.norm(ref))
        f8 = 8.0 * c.l * c.m * c.n
        print(json.dumps({"cfg": cname, "variant": v, "ms": round(ms, 3),
                          "tflops_8lmn": round(f8 / ms / 1e9, 2),
                          "tflops_exec": round(0.75 * f8 / ms / 1e9, 2), "rel_vs_first": err}),
              flush=True)
    os.environ.pop("RID_Z3_VARIANT")
    del A, Y
    torch.cuda.empty_cache()
