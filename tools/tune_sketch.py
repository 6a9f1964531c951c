"""Time the DMMA sketch GEMM under the tile variants of k_zgemm.cu (RID_ZGEMM_VARIANT)."""
import os, sys, json
sys.path.insert(0, os.getcwd())
import torch
import paper_1205_3830_b200 as rid
from paper_1205_3830_b200.configs import CONFIGS
cfgs = sys.argv[1].split(",") if len(sys.argv) > 1 else ["C4"]
variants = [int(x) for x in sys.argv[2].split(",")] if len(sys.argv) > 2 else [0] + list(range(1, 11))
for cname in cfgs:
    c = CONFIGS[cname]
    A = rid.generate(1, c.m, c.n, c.k, c.noise)
    ref = None
    for v in variants:
        if v: os.environ["RID_ZGEMM_VARIANT"] = str(v)
        else: os.environ.pop("RID_ZGEMM_VARIANT", None)
        Y = rid.sketch(A, 1, c.l); torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        reps = 3
        e0.record()
        for _ in range(reps): rid.sketch(A, 1, c.l, out=Y)
        e1.record(); torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / reps
        same = True
        if ref is None: ref = Y.clone()
        else: same = bool(torch.equal(torch.view_as_real(Y), torch.view_as_real(ref)))
        print(json.dumps({"cfg": cname, "variant": v, "ms": round(ms, 3), "tflops": round(c.sketch_flops / ms / 1e9, 2), "bitequal": same}), flush=True)
