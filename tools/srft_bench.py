"""NEXT-1 measurement: the paper's SRFT randomisation Y = S F D A against the
Gaussian sketch on the same configs: sketch time, whole-ID time, and the error estimate of each
ID (different randomisations give different, equally valid IDs).
    python tools/srft_bench.py C4 [C5 ...]"""
import json
import os
import sys

sys.path.insert(0, os.getcwd())
import torch  # noqa: E402

import paper_1205_3830_b200 as rid  # noqa: E402
from paper_1205_3830_b200.configs import CONFIGS  # noqa: E402


def timed(fn, reps=3):
    fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps * 1e-3


for name in sys.argv[1:]:
    c = CONFIGS[name]
    A = rid.generate(1, c.m, c.n, c.k, c.noise)
    Y = rid.colmajor_empty(c.l, c.n, device="cuda")
    t_g = timed(lambda: rid.sketch(A, 1, c.l, out=Y))
    t_s = timed(lambda: rid.sketch_srft(A, 1, c.l, out=Y))
    out = {"cfg": name, "gauss_sketch_ms": t_g * 1e3, "srft_sketch_ms": t_s * 1e3,
           "srft_hbm_bytes": 3 * 16 * c.m * c.n, "srft_flops": 8 * c.l * c.m * c.n / 16}
    for kind in ("gaussian", "srft"):
        r = rid.decompose(A, c.k, c.l, 1, sketch=kind)
        t = timed(lambda: rid.decompose(A, c.k, c.l, 1, sketch=kind), reps=2)
        est = rid.error_estimate(A, r.J, r.P, 10, 1)
        out[f"{kind}_id_ms"] = t * 1e3
        out[f"{kind}_err_est"] = est
        out[f"{kind}_tie_margin"] = r.diag["tie_margin_min"]
        out[f"{kind}_diag"] = {k: r.diag[k] for k in ("t_sketch", "t_qrcp", "t_solve", "t_total")}
    Js = set(rid.decompose(A, c.k, c.l, 1, sketch="srft").J.cpu().tolist())
    Jg = set(rid.decompose(A, c.k, c.l, 1).J.cpu().tolist())
    out["J_overlap"] = len(Js & Jg) / c.k
    print(json.dumps(out), flush=True)
    del A, Y
    torch.cuda.empty_cache()
