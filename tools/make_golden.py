"""Write tests/golden/<cfg>_oracle.json: the CPU ORACLE's own results at full config size.

Calls only oracle/ (no CUDA path): A is generated and sketched block by block (A itself is never
held: C5's A is 64 GiB), then the oracle's pivoted CGS2 and back-substitution run on the full Y.
Stored: J, the pivot residual norms and tie margins, sampled columns of Y and P (exact hex), and
checksums — the expected values of tests/test_gpu_fullsize.py.

    python tools/make_golden.py C2 C3 C4 C5     (minutes to tens of minutes on 8 cores)
"""
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import oracle  # noqa: E402
from paper_1205_3830_b200.configs import CONFIGS, HEADLINE_SEED  # noqa: E402  (shapes only)


def hexz(z):
    return [float(z.real).hex(), float(z.imag).hex()]


def sample_cols(n, count=6):
    rng = np.random.default_rng(12345)
    cols = sorted(set([0, n - 1] + rng.choice(n, size=count, replace=False).tolist()))
    return cols


def main(names):
    oracle.set_threads(int(os.environ.get("ORACLE_THREADS", os.cpu_count() or 1)))
    for name in names:
        c = CONFIGS[name]
        seed = HEADLINE_SEED
        t0 = time.time()
        Y = np.zeros((c.l, c.n), np.complex128, order="F")
        blk = max(64, min(c.n, (2 << 30) // (16 * c.m)))  # ~2 GiB of A per block
        for col0 in range(0, c.n, blk):
            nb = min(blk, c.n - col0)
            A = oracle.generate(seed, c.m, c.n, c.k, c.noise, col0, nb)
            Y[:, col0:col0 + nb] = oracle.sketch(A, seed, c.l)
            del A
            print(f"{name}: sketched columns {col0 + nb}/{c.n} ({time.time() - t0:.0f} s)",
                  flush=True)
        qr = oracle.pivoted_qr(Y, c.k)
        assert qr.status == 0, f"{name}: oracle rank failure"
        P = oracle.backsolve(qr.R, qr.J, c.k)
        cols = sample_cols(c.n)
        out = {
            "config": name, "seed": seed, "m": c.m, "n": c.n, "k": c.k, "l": c.l,
            "noise": c.noise,
            "source": "tools/make_golden.py (oracle/ only: orc_generate, orc_sketch, "
                      "orc_pivoted_cgs2, orc_backsolve)",
            "J": qr.J.tolist(),
            "resid_norms": [float(x).hex() for x in qr.resid_norms],
            "tie_margin_min": float(qr.tie_margins[:-1].min()),
            "sample_cols": cols,
            "Y_cols": {str(j): [hexz(z) for z in Y[:, j]] for j in cols},
            "P_cols": {str(j): [hexz(z) for z in P[:, j]] for j in cols},
            "Y_fro": float(np.linalg.norm(Y)),
            "P_fro": float(np.linalg.norm(P)),
            "seconds": time.time() - t0,
        }
        path = os.path.join(ROOT, "tests", "golden", f"{name}_oracle.json")
        with open(path, "w") as f:
            json.dump(out, f)
        print(f"{name}: wrote {path} in {out['seconds']:.0f} s; min tie margin "
              f"{out['tie_margin_min']:.3e}", flush=True)


if __name__ == "__main__":
    main(sys.argv[1:] or ["C2", "C3", "C4", "C5"])
