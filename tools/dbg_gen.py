import sys, os
sys.path.insert(0, os.getcwd())
import numpy as np, torch
import oracle, paper_1205_3830_b200 as rid
for (seed, m, n, k, noise) in [(3, 2048, 130, 64, 0.0), (3, 2048, 130, 16, 0.0), (3, 2048, 128, 16, 0.0),
                               (3, 1024, 130, 64, 0.0), (3, 2048, 130, 64, 1e-10), (3, 4096, 64, 32, 0.0)]:
    g = rid.generate(seed, m, n, k, noise).cpu().numpy()
    o = oracle.generate(seed, m, n, k, noise)
    bad = (g != o)
    rel = np.abs(g - o).max() / np.abs(o).max()
    rows, cols = np.nonzero(bad)
    print(f"m={m} n={n} k={k} noise={noise}: mismatches {bad.sum()} of {bad.size}, max rel {rel:.2e}",
          "rows%128:", np.unique(rows % 128)[:10], "cols:", np.unique(cols)[:10], "rows:", np.unique(rows)[:10])
