"""Time the DMMA generation GEMM (A = X Y0 + eps E) under the tile variants (RID_ZGEMM_VARIANT)."""
import os, sys, json
sys.path.insert(0, os.getcwd())
import torch
import paper_1205_3830_b200 as rid
from paper_1205_3830_b200.configs import CONFIGS
cname = sys.argv[1]; variants = [int(x) for x in sys.argv[2].split(",")]
c = CONFIGS[cname]
A = rid.colmajor_empty(c.m, c.n)
ref = None
for v in variants:
    if v: os.environ["RID_ZGEMM_VARIANT"] = str(v)
    else: os.environ.pop("RID_ZGEMM_VARIANT", None)
    rid.generate(1, c.m, c.n, c.k, c.noise, out=A); torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(); rid.generate(1, c.m, c.n, c.k, c.noise, out=A); e1.record(); torch.cuda.synchronize()
    ms = e0.elapsed_time(e1)
    if ref is None: ref = A.clone(); same = True
    else: same = bool(torch.equal(torch.view_as_real(A), torch.view_as_real(ref)))
    print(json.dumps({"cfg": cname, "gen_variant": v, "ms": round(ms, 3), "tflops": round(8.0*c.m*c.n*c.k/ms/1e9, 2), "bitequal": same}), flush=True)
