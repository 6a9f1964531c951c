"""Randomised parity sweep of the whole CUDA path against the oracle on small random shapes
(every kernel variant the shapes select: 24/40/48-row sketch tiles, K tails, split-K, the
small and blocked QR, both solves), seeded and reproducible.
    python tools/fuzz_parity.py [count] [seed] [gaussian|srft] [householder|cgs2]
(srft: m is drawn as a power of two, the paper's randomisation Y = S F D A)"""
import os
import sys

sys.path.insert(0, os.getcwd())
import numpy as np  # noqa: E402

import oracle  # noqa: E402
import paper_1205_3830_b200 as rid  # noqa: E402

count = int(sys.argv[1]) if len(sys.argv) > 1 else 40
rng = np.random.default_rng(int(sys.argv[2]) if len(sys.argv) > 2 else 12345)
kind = sys.argv[3] if len(sys.argv) > 3 else "gaussian"
qr = sys.argv[4] if len(sys.argv) > 4 else "householder"
oracle.build()
bad = 0
for it in range(count):
    m = int(2 ** rng.integers(5, 12)) if kind == "srft" else int(rng.integers(16, 3000))
    n = int(rng.integers(1, 1500))
    k = int(rng.integers(1, min(m, n, 300) + 1))
    l = int(min(m, k + rng.integers(0, 40)))
    noise = float(rng.choice([0.0, 1e-12, 1e-9, 1e-6]))
    seed = int(rng.integers(1, 1 << 30))
    A = rid.generate(seed, m, n, k, noise)
    A_o = oracle.generate(seed, m, n, k, noise)
    ok_a = np.array_equal(np.ascontiguousarray(A.cpu().numpy()).view(np.uint64),
                          np.ascontiguousarray(A_o).view(np.uint64))
    if kind == "srft":
        Y = rid.sketch_srft(A, seed, l).cpu().numpy()
        Y_o = oracle.srft_sketch(A_o, seed, l)
    else:
        Y = rid.sketch(A, seed, l).cpu().numpy()
        Y_o = oracle.sketch(A_o, seed, l)
    ry = np.linalg.norm(Y - Y_o) / max(np.linalg.norm(Y_o), 1e-300)
    msg = ""
    try:
        try:
            d = oracle.decompose(A_o, k, l, seed, sketch_kind=kind)
        except oracle.OracleError as oe:  # rank-deficient sketch: the GPU must say so as well
            try:
                rid.decompose(A, k, l, seed, sketch=kind, qr=qr)
                raise RuntimeError(f"oracle failed ({oe}) but the GPU path did not")
            except rid.RidError as ge:
                raise ge from None
        r = rid.decompose(A, k, l, seed, sketch=kind, qr=qr)
        J, P = r.J.cpu().numpy(), r.P.cpu().numpy()
        same_j = J.tolist() == list(d.J)
        rp = np.linalg.norm(P - d.P) / max(np.linalg.norm(d.P), 1e-300) if same_j else float("nan")
        margin = float(np.min(d.tie_margins)) if len(d.tie_margins) else float("nan")
        ok = ok_a and ry <= 1e-12 and same_j and rp <= 1e-10
        msg = f"J {'equal' if same_j else 'DIFF'} P {rp:.1e} margin {margin:.1e}"
    except rid.RidError as e:
        ok = ok_a and ry <= 1e-12 and "RANK" in str(e).upper()
        msg = f"RidError {e}"
    except Exception as e:  # noqa: BLE001 (the oracle raises on rank deficiency too)
        ok = False
        msg = f"{type(e).__name__} {e}"
    bad += 0 if ok else 1
    print(f"{'ok ' if ok else 'BAD'} m={m} n={n} k={k} l={l} noise={noise:g}: A "
          f"{'bitwise' if ok_a else 'DIFF'} Y {ry:.1e} {msg}", flush=True)
print(f"{count - bad}/{count} ok", flush=True)
