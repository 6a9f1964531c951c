"""NEXT-2 measurement: the paper's QR (CGS2, k_cgs2.cu) beside the Householder kernels on the
north-star configs, same sketch. Per config: t_qrcp of both (device events, median of 3 after a
warm-up), and for CGS2 the HBM roofline of its dominant kernel (k_cgs_project): each step reads
and writes every unchosen column of W once, 2*16*l*(n - j) bytes at step j, so the k steps move
16*l*k*(2n - k + 1) bytes (plus the norm pass of step 0, 16 l n); the rest of a step is the two
reorthogonalisation passes (4 small launches, latency-bound).

    python tools/cgs2_bench.py [--configs C2,C3,C4,C5]
"""
import argparse
import json
import os
import statistics
import sys

sys.path.insert(0, os.getcwd())
import torch  # noqa: E402

import paper_1205_3830_b200 as rid  # noqa: E402
from paper_1205_3830_b200.configs import CONFIGS, HEADLINE_SEED  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--configs", default="C2,C3,C4,C5")
ap.add_argument("--reps", type=int, default=3)
args = ap.parse_args()
peaks = json.load(open("MEASURED_PEAKS.json")) if os.path.exists("MEASURED_PEAKS.json") else {}
for name in args.configs.split(","):
    cfg = CONFIGS[name]
    m, n, k, l = cfg.m, cfg.n, cfg.k, cfg.l
    A = rid.generate(HEADLINE_SEED, m, n, k, cfg.noise)
    out = {"config": name, "m": m, "n": n, "k": k, "l": l}
    Js = {}
    for qr in ("householder", "cgs2"):
        rid.decompose(A, k, l, HEADLINE_SEED, qr=qr)
        ts, tot = [], []
        for _ in range(args.reps):
            r = rid.decompose(A, k, l, HEADLINE_SEED, qr=qr)
            ts.append(r.diag["t_qrcp"])
            tot.append(r.diag["t_total"])
        Js[qr] = r.J.clone()
        out[qr] = {"t_qr_ms": statistics.median(ts) * 1e3, "t_total_ms": statistics.median(tot) * 1e3,
                   "launches": r.diag["launches"]}
    bytes_proj = 16.0 * l * k * (2 * n - k + 1) + 16.0 * l * n
    out["cgs2"]["project_bytes"] = bytes_proj
    out["cgs2"]["GBps_if_all_time_project"] = bytes_proj / (out["cgs2"]["t_qr_ms"] * 1e-3) / 1e9
    out["same_J"] = bool(torch.equal(Js["householder"], Js["cgs2"]))
    out["ratio_cgs2_over_householder"] = out["cgs2"]["t_qr_ms"] / out["householder"]["t_qr_ms"]
    print(json.dumps(out), flush=True)
    del A
    torch.cuda.empty_cache()
