import os, sys
sys.path.insert(0, os.getcwd())
import torch
import paper_1205_3830_b200 as rid
from paper_1205_3830_b200.configs import CONFIGS
for name in sys.argv[1:]:
    c = CONFIGS[name]
    A = rid.colmajor_empty(c.m, c.n, device="cuda")
    for label, env in [("cp.async", {"RID_ZGEMM_TMA": "0"}), ("tma6", {"RID_ZGEMM_TMA": "1"}),
                       ("tma4", {"RID_ZGEMM_TMA": "1", "RID_ZGEMM_TMA_STAGES": "4"}),
                       ("tma8", {"RID_ZGEMM_TMA": "1", "RID_ZGEMM_TMA_STAGES": "8"})]:
        for kk in ("RID_ZGEMM_TMA", "RID_ZGEMM_TMA_STAGES"):
            os.environ.pop(kk, None)
        os.environ.update(env)
        rid.generate(1, c.m, c.n, c.k, c.noise, out=A)
        ts = []
        for _ in range(3):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(); rid.generate(1, c.m, c.n, c.k, c.noise, out=A); e1.record()
            torch.cuda.synchronize(); ts.append(e0.elapsed_time(e1))
        f = 8.0 * c.m * c.n * c.k
        print(f"{name} gen {label:8s} {min(ts):8.2f} ms  {f / min(ts) / 1e9:6.2f} TF/s ({f / min(ts) / 1e9 / 37.11:.3f} of DMMA peak)", flush=True)
    del A
    torch.cuda.empty_cache()
