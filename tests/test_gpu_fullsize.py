"""GPU parity at the FULL BASELINE.json configs (C1–C5), in the launch configuration bench.py
times, against values the CPU oracle computed on its own (tests/golden/<cfg>_oracle.json, written
by tools/make_golden.py which calls only oracle/):

- J identical to the oracle's J (reading R18; the oracle's min top-2 gap is stored and > 1e-10);
- sampled columns of Y bit-identical (the DMMA chain is the oracle's fused ascending order);
- sampled columns of P within 1e-10 relative (reading R17), P[:, J] = I bitwise;
- residual norms nu_p per pivot step within 1e-10 relative;
- sampled columns of A recomputed by the oracle one by one: bit-identical;
- the error estimate: finite, below the Eq. (3) right-hand side with sigma_{k+1} from the Weyl
  bracket (reading R20), and exact-rank C1 at rho <= 1e-13.
"""
import json
import math
import os

import numpy as np
import pytest

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")

HERE = os.path.dirname(os.path.abspath(__file__))


@pytest.fixture(scope="module")
def rid():
    if not torch.cuda.is_available():
        pytest.skip("no GPU")
    from paper_1205_3830_b200 import build

    build.build()
    import paper_1205_3830_b200 as rid

    return rid


def load_golden(name):
    path = os.path.join(HERE, "golden", f"{name}_oracle.json")
    if not os.path.exists(path):
        pytest.skip(f"{path} not generated yet (tools/make_golden.py {name})")
    with open(path) as f:
        return json.load(f)


def unhex(col):
    return np.array([complex(float.fromhex(a), float.fromhex(b)) for a, b in col])


def bits(a):
    return np.ascontiguousarray(np.asarray(a, dtype=np.complex128)).view(np.uint64)


@pytest.mark.parametrize("name", ["C2", "C3", "C4", "C5"])
def test_fullsize_against_oracle_golden(rid, orc, name):
    from paper_1205_3830_b200.configs import CONFIGS

    g = load_golden(name)
    c = CONFIGS[name]
    assert (g["m"], g["n"], g["k"], g["l"], g["noise"]) == (c.m, c.n, c.k, c.l, c.noise)
    seed = g["seed"]
    free = torch.cuda.mem_get_info()[0]
    if free < 1.2 * c.a_bytes + (2 << 30):
        pytest.skip(f"{name}: needs {c.a_bytes / 2**30:.0f} GiB of free HBM")
    A = rid.generate(seed, c.m, c.n, c.k, c.noise)
    cols = g["sample_cols"]
    # sampled A columns, recomputed one by one by the oracle: bitwise
    for j in cols[:3]:
        a_o = orc.generate(seed, c.m, c.n, c.k, c.noise, j, 1)
        assert np.array_equal(bits(A[:, j].cpu().numpy()), bits(a_o[:, 0])), f"A[:, {j}]"
    # sketch: sampled columns bitwise, Frobenius norm
    Y = rid.sketch(A, seed, c.l)
    S = rid.sketch_splits(c.m, c.l, c.n)
    # per-column bar: DMMA (3M / Strassen / K slices) to rounding, 1e-13; the INT8_CRT engine
    # (R33) rounds each operand to b bits of its row / column maximum (~3.6 2^-b, 3e-15 at b = 50):
    # there the oracle's own fp64 accumulation error (~1e-14) dominates, so the same 1e-13
    tol = 1e-13
    if rid.sketch_engine(c.m, c.l, c.n) == "int8_crt":
        tol = max(tol, 8.0 * 2.0 ** -rid.crt_plan(c.l, c.m)["b"])
    for j in cols:
        y_o = unhex(g["Y_cols"][str(j)])
        y_g = Y[:, j].cpu().numpy()
        if S == 1 and rid.sketch_mults() == 4:  # one ascending fused chain: bit-identical
            assert np.array_equal(bits(y_g), bits(y_o)), f"Y[:, {j}]"
        else:  # Gauss's three products (R31) and/or S fixed-order slice sums: to rounding
            assert np.linalg.norm(y_g - y_o) <= tol * np.linalg.norm(y_o), f"Y[:, {j}]"
    yf = float(torch.linalg.norm(Y))
    assert abs(yf - g["Y_fro"]) <= 1e-12 * g["Y_fro"]
    del Y
    # the ID
    r = rid.decompose(A, c.k, c.l, seed)
    J = r.J.cpu().numpy()
    assert g["tie_margin_min"] > 1e-10
    assert J.tolist() == g["J"]
    P = r.P
    assert np.array_equal(bits(P[:, r.J].cpu().numpy()), bits(np.eye(c.k)))
    for j in cols:
        p_o = unhex(g["P_cols"][str(j)])
        p_g = P[:, j].cpu().numpy()
        assert np.linalg.norm(p_g - p_o) <= 1e-10 * max(np.linalg.norm(p_o), 1.0), f"P[:, {j}]"
    pf = float(torch.linalg.norm(P))
    assert abs(pf - g["P_fro"]) <= 1e-10 * g["P_fro"]
    assert abs(r.diag["tie_margin_min"] - g["tie_margin_min"]) <= 1e-6 * g["tie_margin_min"]
    # error estimate vs Eq. (3) with sigma_{k+1} <= noise * sigma_1(E) ~ noise (sqrt m + sqrt n)
    est = rid.error_estimate(A, r.J, r.P, 3, seed)
    sig = c.noise * (math.sqrt(c.m) + math.sqrt(c.n)) * 1.05
    assert math.isfinite(est) and 0 < est <= rid.error_bound(c.m, c.n, c.k, 1e-20, sig)
    assert est >= c.noise * (math.sqrt(c.m) - math.sqrt(c.n)) * 0.5 if c.m > c.n else est > 0


def test_fullsize_c1_exact_rank(rid, orc):
    """C1 = the paper's noiseless A = BP: full oracle, J equal, rho <= 1e-13."""
    from paper_1205_3830_b200.configs import CONFIGS

    c = CONFIGS["C1"]
    A_o = orc.generate(1, c.m, c.n, c.k, 0.0)
    d = orc.decompose(A_o, c.k, c.l, 1)
    A = rid.generate(1, c.m, c.n, c.k, 0.0)
    r = rid.decompose(A, c.k, c.l, 1)
    assert r.J.cpu().numpy().tolist() == d.J.tolist()
    P = r.P.cpu().numpy()
    assert np.linalg.norm(P - d.P) <= 1e-10 * np.linalg.norm(d.P)
    est = rid.error_estimate(A, r.J, r.P, 20, 1)
    nA = np.linalg.svd(A_o, compute_uv=False)[0]
    assert est / nA <= 1e-13


@pytest.mark.parametrize("name", ["C2", "C3"])
def test_fullsize_live_oracle(rid, orc, name):
    """C2 and C3 at full size against the oracle run LIVE on the box's host (no stored values):
    A bitwise, every element of P within 1e-10 relative (reading R17) and J equal, the estimator
    on the oracle's (A, J, P) within 1e-10 of the oracle's Dot2 estimator (R16 (i), q = 3), and
    each side's own P within 1e-10 in rho = est / ||A||_2 (R16 (ii); ||A||_2 from the oracle's
    power iteration with P = 0, q = 5: a lower bound of ||A||_2, so the check is conservative)."""
    from paper_1205_3830_b200.configs import CONFIGS

    c = CONFIGS[name]
    seed, q = 1, 3
    free = torch.cuda.mem_get_info()[0]
    if free < 1.5 * c.a_bytes + (2 << 30):
        pytest.skip(f"{name}: needs {c.a_bytes / 2**30:.0f} GiB of free HBM")
    A_o = orc.generate(seed, c.m, c.n, c.k, c.noise)
    d = orc.decompose(A_o, c.k, c.l, seed)
    assert d.tie_margins[:-1].min() > 1e-10
    A = rid.generate(seed, c.m, c.n, c.k, c.noise)
    assert np.array_equal(bits(A.cpu().numpy()), bits(A_o)), "A"
    r = rid.decompose(A, c.k, c.l, seed)
    assert r.J.cpu().numpy().tolist() == d.J.tolist()
    P = r.P.cpu().numpy()
    assert np.array_equal(bits(P[:, d.J]), bits(np.eye(c.k)))
    assert np.linalg.norm(P - d.P) <= 1e-10 * np.linalg.norm(d.P)
    # per column as well: no column of P may hide behind the Frobenius norm
    colerr = np.linalg.norm(P - d.P, axis=0) / np.maximum(np.linalg.norm(d.P, axis=0), 1.0)
    assert colerr.max() <= 1e-10, (int(colerr.argmax()), float(colerr.max()))
    # (i) estimator parity on the same (A, J, P)
    e_o = orc.error_estimate(A_o, d.J, d.P, q, seed)
    Jt = torch.from_numpy(d.J.copy()).cuda()
    Pt = torch.from_numpy(d.P.T.copy()).T.cuda()
    e_g = rid.error_estimate(A, Jt, Pt, q, seed)
    assert abs(e_g - e_o) <= 1e-10 * e_o, (e_g, e_o)
    # (ii) each side's own P, relative to ||A||_2
    e_g2 = rid.error_estimate(A, r.J, r.P, q, seed)
    nA = orc.error_estimate(A_o, np.zeros(1, np.int64), np.zeros((1, c.n), np.complex128,
                                                                   order="F"), 5, seed)
    assert abs(e_g2 - e_o) / nA <= 1e-10
