"""Pins for the oracle's method layer, each against something other than the oracle itself.

| oracle step | pinned by |
|---|---|
| generate (docs/RNG.md §5) | numpy X@Y0 (BLAS); dense SVD rank; exact-fma
  recomputation in pure Python for a few entries; noise term ε·E |
| sketch (Y = R·A; north_star) | numpy R@A (BLAS ZGEMM); exact ascending-fma pure
  Python for a few entries; (R X) Y0 + ε R E identity; column-shard invariance |
| pivoted CGS2 | LAPACK ZGEQP3 pivots; scipy interp_decomp(rand=False);
  SPEC.md:246-248 examples; Q^H Q / R11 triangularity; non-increasing residual norms |
| backsolve (Eqs. 10–11) | numpy lstsq; SPEC.md:311-313 and :320-322 examples;
  singular diagonal; P[:, J] = I bitwise |
| whole ID | brute force over all column subsets on tiny inputs; exact-rank reconstruction
  (north star); Eq. (3) bound with the dense σ_{k+1} |
| error estimate (Table 5) | SPEC.md:66-68 examples; dense SVD of the residual
  formed in double-double (Dekker TwoProd) |
| bound / noise floor (Eq. 3) | SPEC.md:346, :354 closed forms |
| threads | bitwise thread-count invariance |
"""
import itertools
import math
import os

import numpy as np
import pytest
import scipy.linalg as sla
from scipy.linalg import interpolative as sli

HERE = os.path.dirname(os.path.abspath(__file__))


def relf(a, b):
    return np.linalg.norm(a - b) / np.linalg.norm(b)


def fma_exact(a, b, c):
    """Correctly rounded a*b + c through exact rationals (independent of libm's fma)."""
    from fractions import Fraction

    return float(Fraction(a) * Fraction(b) + Fraction(c))


def cmac_ref(acc, x, y):
    """docs/RNG.md §5 MAC in exact-rational fma arithmetic."""
    re = fma_exact(x.real, y.real, acc.real)
    re = fma_exact(-x.imag, y.imag, re)
    im = fma_exact(x.imag, y.real, acc.imag)
    im = fma_exact(x.real, y.imag, im)
    return complex(re, im)


# ----------------------------------------------------------------------------- generation ---
def test_generate_matches_blas_and_exact_fma(orc):
    seed, m, n, k, eps = 11, 40, 30, 5, 1e-10
    A = orc.generate(seed, m, n, k, eps)
    X = orc.normal_matrix(seed, 1, m, k)
    Y0 = orc.normal_matrix(seed, 2, k, n)
    E = orc.normal_matrix(seed, 3, m, n)
    assert relf(A, X @ Y0 + eps * E) <= 1e-14
    for (i, j) in [(0, 0), (7, 29), (39, 13)]:
        acc = complex(0.0, 0.0)
        for t in range(k):
            acc = cmac_ref(acc, X[i, t], Y0[t, j])
        want = complex(fma_exact(eps, E[i, j].real, acc.real), fma_exact(eps, E[i, j].imag, acc.imag))
        assert A[i, j] == want  # bitwise


def test_generate_exact_rank(orc):
    A = orc.generate(5, 64, 64, 8, 0.0)  # 64x64, k=8 -> s9/s1 <= 1e-13
    s = np.linalg.svd(A, compute_uv=False)
    assert s[8] / s[0] <= 1e-13
    assert s[7] / s[0] >= 1e-3
    A1 = orc.generate(5, 30, 20, 1, 0.0)  # k = 1 -> collinear columns
    col0 = A1[:, 0]
    for j in range(1, 20):
        c = np.vdot(col0, A1[:, j]) / np.vdot(col0, col0)
        assert np.linalg.norm(A1[:, j] - c * col0) <= 1e-12 * np.linalg.norm(A1[:, j])


def test_generate_noise_spectrum(orc):
    # A = X Y0 + eps E: sigma_{k+1} sits inside the Weyl bracket [eps s_{2k+1}(E), eps s_1(E)]
    m, n, k, eps = 120, 100, 6, 1e-6
    A = orc.generate(3, m, n, k, eps)
    E = orc.normal_matrix(3, 3, m, n)
    s = np.linalg.svd(A, compute_uv=False)
    sE = np.linalg.svd(E, compute_uv=False)
    assert eps * sE[2 * k] * (1 - 1e-6) <= s[k] <= eps * sE[0] * (1 + 1e-6)


def test_generate_sharding_bitwise(orc):
    A = orc.generate(2, 50, 40, 4, 1e-8)
    for col0, nl in [(0, 13), (13, 14), (27, 13)]:
        assert np.array_equal(orc.generate(2, 50, 40, 4, 1e-8, col0, nl), A[:, col0:col0 + nl])


# --------------------------------------------------------------------------------- sketch ---
def test_sketch_matches_blas_and_exact_fma(orc):
    seed, m, n, k, l = 4, 60, 25, 4, 9
    A = orc.generate(seed, m, n, k, 1e-9)
    Y = orc.sketch(A, seed, l)
    R = orc.normal_matrix(seed, 4, l, m)
    assert relf(Y, R @ A) <= 1e-14
    for (r, j) in [(0, 0), (8, 24), (3, 11)]:
        acc = complex(0.0, 0.0)
        for i in range(m):
            acc = cmac_ref(acc, R[r, i], A[i, j])
        assert Y[r, j] == acc


def test_sketch_identity_and_shards(orc):
    seed, m, n, k, l, eps = 8, 100, 40, 3, 7, 1e-6
    A = orc.generate(seed, m, n, k, eps)
    X, Y0 = orc.normal_matrix(seed, 1, m, k), orc.normal_matrix(seed, 2, k, n)
    E, R = orc.normal_matrix(seed, 3, m, n), orc.normal_matrix(seed, 4, l, m)
    Y = orc.sketch(A, seed, l)
    assert relf(Y, (R @ X) @ Y0 + eps * (R @ E)) <= 1e-13
    assert np.array_equal(orc.sketch(A[:, 10:25], seed, l), Y[:, 10:25])
    assert not np.array_equal(orc.sketch(A, seed, l, stream=20), Y)


# ----------------------------------------------------------------------------- pivoted QR ---
def test_qr_spec_examples(orc):
    qr = orc.pivoted_qr(np.eye(4), 4)  # tie-break -> 0,1,2,3
    assert qr.J.tolist() == [0, 1, 2, 3]
    assert np.allclose(np.abs(qr.R), np.eye(4), atol=1e-15)
    Y = np.zeros((3, 2), complex)
    Y[0, 0], Y[1, 1] = 2, 1  # (2 e1, e2) -> diag(2, 1)
    qr = orc.pivoted_qr(Y, 2)
    assert qr.J.tolist() == [0, 1]
    assert np.allclose(np.abs(np.diag(qr.R)), [2, 1], atol=1e-15)
    assert qr.resid_norms.tolist() == [2.0, 1.0]


def _rand_lowrank(rng, l, n, r, noise=0.0):
    G = lambda *s: rng.standard_normal(s) + 1j * rng.standard_normal(s)
    return G(l, r) @ G(r, n) + noise * G(l, n)


def test_qr_matches_zgeqp3_and_interp_decomp(orc):
    rng = np.random.default_rng(0)
    for (l, n, k, noise) in [(24, 512, 16, 0.0), (48, 300, 32, 1e-9), (80, 400, 64, 1e-6),
                             (20, 50, 20, 0.0)]:
        Y = np.asfortranarray(_rand_lowrank(rng, l, n, k, noise) if noise or k < l else
                              _rand_lowrank(rng, l, n, l))
        qr = orc.pivoted_qr(Y, k)
        assert qr.status == 0
        _, _, piv = sla.qr(Y, pivoting=True, mode="economic")  # LAPACK ZGEQP3
        assert qr.J.tolist() == piv[:k].tolist()
        idx, _ = sli.interp_decomp(Y.copy(), k, rand=False)
        assert sorted(qr.J.tolist()) == sorted(idx[:k].tolist())
        # R11 = R[:, J] upper triangular up to rounding; |diag| = residual norms, non-increasing
        R11 = qr.R[:, qr.J]
        assert np.linalg.norm(np.tril(R11, -1)) <= 1e-13 * np.linalg.norm(R11)
        assert np.allclose(np.abs(np.diag(R11)), qr.resid_norms, rtol=1e-12)
        assert np.all(np.diff(qr.resid_norms) <= 1e-12 * qr.resid_norms[0])
        assert np.all(qr.tie_margins[:-1] >= 0)


def test_qr_reconstruction_and_orthonormality(orc):
    rng = np.random.default_rng(1)
    Y = np.asfortranarray(_rand_lowrank(rng, 6, 10, 3))  # SPEC.md:248 rank-3 6x10
    qr = orc.pivoted_qr(Y, 3)
    # Q = Y_J R11^{-1}: orthonormal, and Q R reproduces Y (exact rank)
    Q = Y[:, qr.J] @ np.linalg.inv(qr.R[:, qr.J])
    assert np.linalg.norm(Q.conj().T @ Q - np.eye(3)) <= 1e-12 * math.sqrt(3)
    assert np.linalg.norm(Y - Q @ qr.R) <= 1e-12 * np.linalg.norm(Y)


def test_qr_rank_failure(orc):
    rng = np.random.default_rng(2)
    Y = np.asfortranarray(_rand_lowrank(rng, 10, 30, 3))
    qr = orc.pivoted_qr(Y, 5)  # rank 3 < k = 5 -> ERANK with the achieved rank
    assert qr.status == orc.RID_ERANK and qr.rank_achieved == 3


# ------------------------------------------------------------------------------ backsolve ---
def test_backsolve_spec_examples(orc):
    # r1 = I -> t = r2 ; R = [I | r2] in columns (0, 1 | 2)
    r2 = np.array([[2 + 1j], [3 - 1j]])
    R = np.hstack([np.eye(2), r2])
    P = orc.backsolve(R, [0, 1], 2)
    assert np.array_equal(P, np.hstack([np.eye(2), r2]))  # also SPEC.md:321 [[1,0,a],[0,1,b]]
    # [[2,1],[0,1]] t = (3,1)^T -> t = (1,1)^T
    R = np.array([[2, 1, 3], [0, 1, 1]], dtype=complex)
    P = orc.backsolve(R, [0, 1], 2)
    assert np.allclose(P[:, 2], [1, 1], atol=0)
    # zero diagonal -> singular
    R = np.array([[2, 1, 3], [0, 0, 1]], dtype=complex)
    with pytest.raises(orc.OracleError) as e:
        orc.backsolve(R, [0, 1], 2)
    assert e.value.status == orc.RID_ESINGULAR
    # n = k with pivots [1, 0] -> permutation matrix
    R = np.array([[0, 1], [1, 0]], dtype=complex)
    P = orc.backsolve(R, [1, 0], 2)
    assert np.array_equal(P, np.array([[0, 1], [1, 0]], dtype=complex))


def test_backsolve_matches_lstsq(orc):
    rng = np.random.default_rng(3)
    for (l, n, k, noise) in [(24, 200, 16, 0.0), (40, 150, 24, 1e-8)]:
        Y = np.asfortranarray(_rand_lowrank(rng, l, n, k, noise))
        qr = orc.pivoted_qr(Y, k)
        P = orc.backsolve(qr.R, qr.J, k)
        Jc = np.setdiff1d(np.arange(n), qr.J)
        T, *_ = np.linalg.lstsq(Y[:, qr.J], Y[:, Jc], rcond=None)
        assert relf(P[:, Jc], T) <= 1e-12
        assert np.array_equal(P[:, qr.J], np.eye(k))  # identity block bitwise


# ------------------------------------------------------------------------------ whole ID ----
def _spec2(M):
    return np.linalg.svd(M, compute_uv=False)[0]


def test_brute_force_tiny(orc):
    rng = np.random.default_rng(4)
    for trial in range(6):
        m, n, k = 8, 9, 2 + trial % 2
        A = _rand_lowrank(rng, m, n, k, 1e-3 * (trial + 1))
        d = orc.decompose(A, k, k + 3, seed=trial + 1)
        e_id = _spec2(A - A[:, d.J] @ d.P)
        best = min(_spec2(A - A[:, list(J)] @ np.linalg.lstsq(A[:, list(J)], A, rcond=None)[0])
                   for J in itertools.combinations(range(n), k))
        J = list(d.J)
        e_ls = _spec2(A - A[:, J] @ np.linalg.lstsq(A[:, J], A, rcond=None)[0])
        s = np.linalg.svd(A, compute_uv=False)
        assert s[k] * (1 - 1e-12) <= best <= e_ls * (1 + 1e-12) <= e_id * (1 + 1e-9)
        assert e_id <= orc.error_bound(m, n, k, 1e-20, s[k])  # Eq. (3)


def test_exact_rank_reconstruction(orc):
    # C1's shape (m=1024, n=512, k=16, l=24, no noise): exact reconstruction (north star)
    m, n, k, l = 1024, 512, 16, 24
    A = orc.generate(1, m, n, k, 0.0)
    d = orc.decompose(A, k, l, seed=1)
    assert d.retries == 0 and len(set(d.J.tolist())) == k
    res = A.astype(np.clongdouble) - A[:, d.J].astype(np.clongdouble) @ d.P.astype(np.clongdouble)
    rho = np.linalg.norm(res.astype(np.complex128), "fro") / np.linalg.norm(A, "fro")
    assert rho <= 1e-13
    assert np.array_equal(d.P[:, d.J], np.eye(k))
    assert d.tie_margins[:-1].min() > 1e-10  # well-separated (reading R18)


def test_decompose_thread_invariance(orc):
    A = orc.generate(3, 300, 200, 10, 1e-9)
    orc.set_threads(1)
    d1 = orc.decompose(A, 10, 18, seed=3)
    e1 = orc.error_estimate(A, d1.J, d1.P, 5, 3)
    orc.set_threads(os.cpu_count() or 4)
    d2 = orc.decompose(A, 10, 18, seed=3)
    e2 = orc.error_estimate(A, d2.J, d2.P, 5, 3)
    assert np.array_equal(d1.J, d2.J) and np.array_equal(d1.P, d2.P) and np.array_equal(d1.Y, d2.Y)
    assert e1 == e2



def _two_sum(a, b):
    s = a + b
    bb = s - a
    return s, (a - (s - bb)) + (b - bb)


def _split(a):
    c = 134217729.0 * a  # Veltkamp split, 2^27 + 1
    hi = c - (c - a)
    return hi, a - hi


def _two_prod(a, b):
    p = a * b
    ah, al = _split(a)
    bh, bl = _split(b)
    return p, ((ah * bh - p) + ah * bl + al * bh) + al * bl


def dd_residual(A, J, P):
    """A - A[:, J] P to ~106-bit precision (Dekker TwoProd + TwoSum; no fma, no libm)."""
    B = A[:, J]
    out = []
    for part in ("re", "im"):
        s = (A.real if part == "re" else A.imag).copy()
        c = np.zeros_like(s)
        for t in range(len(J)):
            b = B[:, t:t + 1]
            p = P[t:t + 1, :]
            terms = ((b.real, p.real, -1.0), (b.imag, p.imag, 1.0)) if part == "re" else \
                    ((b.real, p.imag, -1.0), (b.imag, p.real, -1.0))
            for x, y, sg in terms:
                ph, pl = _two_prod(sg * x, np.broadcast_to(y, s.shape))
                s, e = _two_sum(s, ph)
                c = c + (e + pl)
        out.append(s + c)
    return out[0] + 1j * out[1]

# ---------------------------------------------------------------------------- estimator ----
def test_estimator_spec_examples(orc):
    # ||A - A_J P||_2 with J = [0], P = 0 except P[0, 0] = 1: residual = A with column 0 zeroed.
    A = np.zeros((3, 3), complex)
    A[1, 1], A[2, 2] = 3, -4j  # SPEC.md:66 diag(3, -4i) -> 4 (column 0 is the pivot, zero)
    A[0, 0] = 1.0
    P = np.zeros((1, 3), complex)
    P[0, 0] = 1
    assert abs(orc.error_estimate(A, [0], P, 60, 1) - 4.0) <= 1e-12
    rng = np.random.default_rng(5)  # SPEC.md:67 rank-1 u v^H -> |u| |v|
    u = rng.standard_normal(6) + 1j * rng.standard_normal(6)
    v = rng.standard_normal(5) + 1j * rng.standard_normal(5)
    A = np.hstack([np.zeros((6, 1)), np.outer(u, v.conj())])
    P = np.zeros((1, 6), complex)
    P[0, 0] = 1
    assert abs(orc.error_estimate(A, [0], P, 3, 2) - np.linalg.norm(u) * np.linalg.norm(v)) <= 1e-12 * np.linalg.norm(u) * np.linalg.norm(v)


@pytest.mark.parametrize("eps", [0.0, 1e-12, 1e-8])
def test_estimator_vs_dd_residual_svd(orc, eps):
    m, n, k, l = 200, 120, 8, 16
    A = orc.generate(7, m, n, k, eps)
    d = orc.decompose(A, k, l, seed=7)
    sv = np.linalg.svd(dd_residual(A, d.J, d.P), compute_uv=False)
    est = orc.error_estimate(A, d.J, d.P, 200, 7)
    assert est <= sv[0] * (1 + 1e-9)
    assert est >= sv[0] * (1 - 1e-6)


def test_estimator_compensation_beats_plain(orc):
    # exact rank: the residual is pure rounding; plain fp64 A x - B (P x) loses most digits
    m, n, k, l = 256, 256, 10, 20  # SPEC.md:336's shape
    A = orc.generate(2, m, n, k, 0.0)
    d = orc.decompose(A, k, l, seed=2)
    est = orc.error_estimate(A, d.J, d.P, 100, 2)
    s1 = np.linalg.svd(dd_residual(A, d.J, d.P), compute_uv=False)[0]
    assert abs(est - s1) <= 1e-6 * s1
    assert est / np.linalg.svd(A, compute_uv=False)[0] <= 1e-13


# ------------------------------------------------------------------------------- bound -----
def _golden():
    out = {}
    with open(os.path.join(HERE, "golden", "spec_examples.txt")) as f:
        for line in f:
            if line.startswith("#") or not line.strip():
                continue
            name, val = line.split()[:2]
            out[name] = float(val)
    return out


def test_bound_and_noise_floor(orc):
    g = _golden()
    b = orc.error_bound(2**14, 2**14, 100, 1e-20, 1e-14)
    assert abs(b - g["error_bound_2^14_2^14_k100_eps1e-20_sigma1e-14"]) <= 1e-4 * b
    f = orc.noise_floor(2**14, 2**14, 1e-16)
    assert abs(f - g["noise_floor_2^14_2^14_delta1e-16"]) <= 1e-4 * f
    assert abs(orc.noise_floor(2, 5, 1e-16) - g["noise_floor_min2_delta1e-16"]) <= 1e-30
    assert orc.error_bound(10, 40, 3, 1.0, 2.0) == 50 * 20 * 2.0  # eps = 1: factor exactly 1
    ks = [orc.error_bound(100, 100, k, 1e-20, 1.0) for k in (5, 10, 50, 100)]
    assert all(a > b for a, b in zip(ks, ks[1:]))
