"""Pins for the oracle's SRFT randomisation Y = S F D A (§2, Eqs. 4–7;
docs/RNG.md §7) — NEXT-1 of SURVEY.md §8(f) — each against something other than the oracle:

- numpy's FFT (pocketfft): S F D A == fft(D A)[s] to rounding;
- a dense materialisation of S, F (Eq. 6 entries from numpy exp), D (m = 8);
- SPEC.md:196-198 examples: m = 1; phases 0 and S = I -> the plain FFT of the columns;
- plan statistics: |D_ii| = 1, sample indices uniform (chi-square), phases uniform (KS);
- E||Y||_F^2 = l ||A||_F^2 over plans, rank preservation for exact rank k, l = 2k.
"""
import math

import numpy as np
import pytest
from scipy import stats


def crandn(rng, *shape):
    return rng.standard_normal(shape) + 1j * rng.standard_normal(shape)


def relf(a, b):
    return np.linalg.norm(a - b) / np.linalg.norm(b)


def test_srft_matches_numpy_fft(orc):
    rng = np.random.default_rng(0)
    for m, l, n in [(8, 5, 3), (256, 40, 7), (4096, 24, 5)]:
        A = np.asfortranarray(crandn(rng, m, n))
        d, s = orc.srft_plan(11, m, l)
        Y = orc.srft_apply(d, s, A)
        Yn = np.fft.fft(d[:, None] * A, axis=0)[s, :]
        assert relf(Y, Yn) <= 1e-13
        assert np.array_equal(orc.srft_sketch(A, 11, l), Y)


def test_srft_dense_materialisation(orc):
    rng = np.random.default_rng(1)
    m, n, l = 8, 5, 6
    A = np.asfortranarray(crandn(rng, m, n))
    d, s = orc.srft_plan(3, m, l)
    S = np.zeros((l, m))
    S[np.arange(l), s] = 1.0  # Eq. (5)
    jj, kk = np.meshgrid(np.arange(m), np.arange(m), indexing="ij")
    F = np.exp(-2j * np.pi * jj * kk / m)  # Eq. (6), 0-based
    D = np.diag(d)  # Eq. (7)
    assert relf(orc.srft_apply(d, s, A), S @ F @ D @ A) <= 1e-13


def test_srft_spec_examples(orc):
    rng = np.random.default_rng(2)
    a = np.asfortranarray(crandn(rng, 1, 4))
    d, s = orc.srft_plan(5, 1, 1)  # m = 1 -> Y = e^{2 pi i phi_0} a
    assert s.tolist() == [0]
    assert relf(orc.srft_apply(d, s, a), d[0] * a) <= 1e-15
    m = 16  # phases 0, S = identity (l = m) -> fft_columns(a)
    A = np.asfortranarray(crandn(rng, m, 3))
    Y = orc.srft_apply(np.ones(m, complex), np.arange(m), A)
    assert relf(Y, np.fft.fft(A, axis=0)) <= 1e-14
    e0 = np.zeros((4, 1), complex)
    e0[0] = 1  # (1,0,0,0) -> (1,1,1,1)
    assert np.allclose(orc.srft_apply(np.ones(4, complex), np.arange(4), e0)[:, 0], 1)


def test_srft_plan_statistics(orc):
    m, l = 1024, 1024 * 40
    d, s = orc.srft_plan(7, m, l)
    assert np.max(np.abs(np.abs(d) - 1)) <= 2e-16 * 4
    counts = np.bincount(s, minlength=m)
    chi2 = ((counts - l / m) ** 2 / (l / m)).sum()
    assert stats.chi2.sf(chi2, m - 1) > 1e-4
    phi = (np.angle(d) / (2 * np.pi)) % 1.0
    assert stats.kstest(phi, stats.uniform.cdf).pvalue > 1e-4
    d2, s2 = orc.srft_plan(7, m, 64, retry=True)
    assert not np.array_equal(d2, d) and not np.array_equal(s2, s[:64])


def test_srft_norm_and_rank(orc):
    rng = np.random.default_rng(3)
    m, n, l = 256, 20, 32
    A = np.asfortranarray(crandn(rng, m, n))
    ratios = [np.linalg.norm(orc.srft_sketch(A, seed, l)) ** 2 / (l * np.linalg.norm(A) ** 2)
              for seed in range(50)]
    assert abs(np.mean(ratios) - 1) <= 0.2
    k = 6  # exact rank k, l = 2k: Y keeps rank k
    B = np.asfortranarray(crandn(rng, m, k) @ crandn(rng, k, 40))
    sv = np.linalg.svd(orc.srft_sketch(B, 1, 2 * k), compute_uv=False)
    assert sv[k - 1] >= 1e-8 * sv[0] and sv[k] <= 1e-12 * sv[0]


def test_srft_decompose_exact_rank(orc):
    A = orc.generate(4, 512, 300, 10, 0.0)
    d = orc.decompose(A, 10, 20, 4, sketch_kind="srft")
    res = A - A[:, d.J] @ d.P
    assert np.linalg.norm(res) <= 1e-11 * np.linalg.norm(A)
    assert np.array_equal(d.P[:, d.J], np.eye(10))
