"""Repeatability of the TMA-fed kernels: the ordered GEMM (generation) against the cp.async kernel,
and the three-product sketch run to run.
    python tools/gen_tma_check.py [reps]"""
import os
import sys

sys.path.insert(0, os.getcwd())
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_1205_3830_b200 as rid  # noqa: E402

REPS = int(sys.argv[1]) if len(sys.argv) > 1 else 6
bad = 0

for (seed, m, n, k, noise) in [(3, 2500, 1000, 512, 0.0), (1, 2048, 300, 64, 1e-10),
                               (2, 4099, 77, 13, 1e-8)]:
    os.environ["RID_ZGEMM_TMA"] = "0"
    ref = rid.generate(seed, m, n, k, noise).cpu().numpy()
    os.environ["RID_ZGEMM_TMA"] = "1"
    for rep in range(REPS):
        A = rid.generate(seed, m, n, k, noise).cpu().numpy()
        d = np.ascontiguousarray(A).view(np.uint64) != np.ascontiguousarray(ref).view(np.uint64)
        if d.any():
            idx = np.argwhere(d)
            rows = sorted(set((i[0]) for i in idx))[:10]
            cols = sorted(set((i[1] // 2) for i in idx))[:10]
            bad += 1
            print(m, n, k, "rep", rep, "DIFF count", int(d.sum()), "rows", rows, "cols", cols,
                  "max abs", float(np.abs(A - ref).max()), flush=True)

for (seed, m, n, l) in [(1, 2048, 2048, 528), (2, 4096, 700, 80), (3, 1001, 333, 47)]:
    A = rid.generate(seed, m, n, 16, 1e-9)
    ref = np.ascontiguousarray(rid.sketch(A, seed, l).cpu().numpy()).view(np.uint64)
    for rep in range(REPS):
        Y = np.ascontiguousarray(rid.sketch(A, seed, l).cpu().numpy()).view(np.uint64)
        if not np.array_equal(Y, ref):
            bad += 1
            print("sketch", m, n, l, "rep", rep, "DIFFERS", int((Y != ref).sum()), flush=True)
print("differing runs:", bad, flush=True)
