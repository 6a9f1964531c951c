"""NEXT-4: the paper's own experiment grid on one B200 (Tables 1-4 and the
error table): exact-rank A = B P with B, P complex Gaussian (
noise 0), l = 2k (PAPER.md:69 / the figure captions), for the eight (k, m, n) of the tables.
Each shape runs the whole ID with the paper's randomisation (SRFT, Y = S F D A) and with the
Gaussian sketch of the north star, timing the phases the paper tabulates — randomisation
("FFT", Table 2 in source order), the pivoted QR ("Gram-Schmidt"), the factorisation of R and P
(the R11^-1 R12 solve) and the total — and estimating ||A - BP||_2 (q = 10, compensated).
The paper's 4-processor XMT numbers are printed beside ours as context (different hardware).
Each also runs with the paper's own QR (--qrs cgs2: classical Gram-Schmidt with one
reorthogonalisation, k_cgs2.cu); srft + cgs2 is the paper's algorithm exactly.
Writes one JSON line per (shape, randomisation, QR).

    python tools/paper_sweep.py [--shapes 0,1,2] [--kinds srft,gaussian] [--qrs householder,cgs2]
"""
import argparse
import json
import os
import sys

sys.path.insert(0, os.getcwd())
import torch  # noqa: E402

import paper_1205_3830_b200 as rid  # noqa: E402

# (k, log2 m, log2 n), and the paper's 4-processor seconds: total, FFT, GS, factor R/P; error
SHAPES = [
    (100, 14, 14, 56.0, 43.0, 0.23, 12.5, 5e-11),
    (100, 16, 14, 188.6, 176.0, 0.23, 12.4, 1e-10),
    (400, 16, 14, 381.1, 175.4, 6.80, 198.9, 2e-10),
    (400, 18, 14, 923.9, 718.0, 6.86, 199.0, 4e-10),
    (100, 16, 16, 732.8, 684.3, 0.22, 48.3, 2e-10),
    (1000, 16, 16, 5657, 687.8, 83.2, 4886, 6e-10),
    (400, 14, 18, 3780, 683.6, 6.66, 3090, 3e-10),
    (1000, 14, 18, 20167, 691, 82.02, 19394, 6e-10),
]
ap = argparse.ArgumentParser()
ap.add_argument("--shapes", default=",".join(str(i) for i in range(len(SHAPES))))
ap.add_argument("--kinds", default="srft,gaussian")
ap.add_argument("--qrs", default="householder")
ap.add_argument("--q", type=int, default=10)
args = ap.parse_args()
for si in [int(x) for x in args.shapes.split(",")]:
    k, lm, ln, p_tot, p_fft, p_gs, p_fac, p_err = SHAPES[si]
    m, n, l = 1 << lm, 1 << ln, 2 * k
    A = rid.generate(1, m, n, k, 0.0)
    # ||A||_2 by the same estimator with P = 0 (||A - A[:, J] 0||_2), for relative errors
    J0 = torch.arange(k, dtype=torch.int64, device="cuda")
    P0 = rid.colmajor_empty(k, n, device="cuda")
    P0.zero_()
    normA = rid.error_estimate(A, J0, P0, args.q, 1)
    del P0
    for kind, qr in [(a, b) for a in args.kinds.split(",") for b in args.qrs.split(",")]:
        rid.decompose(A, k, l, 1, sketch=kind, qr=qr)  # warm (workspace, plan)
        torch.cuda.synchronize()
        r = rid.decompose(A, k, l, 1, sketch=kind, qr=qr)
        d = r.diag
        est = rid.error_estimate(A, r.J, r.P, args.q, 1)
        print(json.dumps({
            "shape": f"k={k} m=2^{lm} n=2^{ln} l={l}", "randomisation": kind, "qr": qr,
            "t_total_s": d["t_total"], "t_randomise_s": d["t_rgen"] + d["t_sketch"],
            "t_qr_s": d["t_qrcp"], "t_factor_s": d["t_solve"],
            "err_2norm_est": est, "norm_A_2_est": normA, "rel_err": est / normA,
            "tie_margin_min": d["tie_margin_min"],
            "paper_xmt_4proc_s": {"total": p_tot, "fft": p_fft, "gram_schmidt": p_gs,
                                  "factor_R_P": p_fac, "error": p_err},
            "speedup_vs_paper_4proc_total": p_tot / d["t_total"]}), flush=True)
    del A
    torch.cuda.empty_cache()
