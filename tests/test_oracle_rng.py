"""Pins for the oracle's random-number layer (docs/RNG.md), independent of the oracle itself.

- Philox4x32-10 against published known-answer vectors and against the CUDA toolkit's own
  implementation (curand_philox4x32_x.h, host branch), PAPER.md:110 / docs/RNG.md §1.
- The RID-libm ln / sincos(2π·) against the platform libm to ≤ 2 ulp on dense sweeps (§4.1, §4.3).
- The normal transform against the distribution the configs state: parts N(0, 1/2), E|z|^2 = 1
  (BASELINE.json:configs; SPEC.md:76-77 statistics), plus a Kolmogorov–Smirnov test.
- The uniform mapping's exactness and range (§3).
"""
import math
import os
import subprocess

import numpy as np
import pytest
from scipy import stats

HERE = os.path.dirname(os.path.abspath(__file__))


def _kat():
    rows = []
    with open(os.path.join(HERE, "golden", "philox4x32_10_kat.txt")) as f:
        for line in f:
            if line.startswith("#") or not line.strip():
                continue
            v = [int(x, 16) for x in line.split()]
            rows.append((v[:4], v[4:6], v[6:10]))
    return rows


def test_philox_known_answers(orc):
    for ctr, key, want in _kat():
        assert orc.philox4x32_10(ctr, key).tolist() == want


@pytest.fixture(scope="module")
def curand_host(tmp_path_factory):
    exe = tmp_path_factory.mktemp("curand") / "curand_host"
    src = os.path.join(HERE, "helpers", "curand_philox_host.cpp")
    try:
        subprocess.check_call(["g++", "-O1", "-I/usr/local/cuda/include", "-o", str(exe), src])
    except (OSError, subprocess.CalledProcessError) as e:  # pragma: no cover
        pytest.skip(f"cannot build curand host helper: {e}")
    return str(exe)


def test_philox_matches_curand(orc, curand_host):
    rng = np.random.default_rng(7)
    cases = rng.integers(0, 2**32, size=(2000, 6), dtype=np.uint64)
    cases[:10, 3] = 0  # our counter layout (i, j, s, 0)
    inp = "\n".join(" ".join(str(int(x)) for x in row) for row in cases) + "\n"
    out = subprocess.run([curand_host], input=inp, capture_output=True, text=True, check=True)
    want = [list(map(int, l.split())) for l in out.stdout.strip().splitlines()]
    for row, w in zip(cases, want):
        got = orc.philox4x32_10(row[:4].astype(np.uint32), row[4:6].astype(np.uint32))
        assert got.tolist() == w


def _ulp_err(a, b):
    return abs(a - b) / math.ulp(b) if b != 0 else abs(a)


def test_rid_ln_accuracy(orc):
    rng = np.random.default_rng(1)
    us = list(rng.uniform(0, 1, 20000)) + list(2.0 ** -rng.uniform(0, 53, 5000))
    us += [2.0**-53, 1 - 2.0**-53, 0.5, 0.25, 1 / math.sqrt(2), math.sqrt(0.5) * (1 + 2**-52),
           0.7071067811865476, 0.7071067811865475, 0.99999, 1e-10]
    worst = 0.0
    for u in us:
        worst = max(worst, _ulp_err(orc.rid_ln(u), math.log(u)))
    assert worst <= 2.0, worst


def test_rid_ln_exact_points(orc):
    # ln(2^-e) = -e ln 2: the split of step 1 makes f = 1, s = 0, and only LN2_HI + LN2_LO remain.
    for e in range(1, 54):
        assert _ulp_err(orc.rid_ln(2.0**-e), -e * math.log(2)) <= 1.0


def test_rid_sincos_accuracy(orc):
    rng = np.random.default_rng(2)
    us = list(rng.uniform(0, 1, 20000)) + [2.0**-53, 1 - 2.0**-53, 0.125, 0.25, 0.375, 0.5,
                                           0.625, 0.75, 0.875, 1 / 3]
    twopi = np.longdouble("6.28318530717958647692528676655900577")
    for u in us:
        c, s = orc.rid_sincos2pi(u)
        th = twopi * np.longdouble(u)  # 64-bit-mantissa angle: reference error ~1e-19
        rc, rs = float(np.cos(th)), float(np.sin(th))
        # <= 2 ulp of the unit-magnitude result (absolute 2^-52 covers values near zeros)
        assert abs(c - rc) <= 2 * 2.0**-53 + 2 * math.ulp(rc), (u, c, rc)
        assert abs(s - rs) <= 2 * 2.0**-53 + 2 * math.ulp(rs), (u, s, rs)
        assert abs(c * c + s * s - 1) <= 4e-16


def test_rid_sincos_quadrant_points(orc):
    assert orc.rid_sincos2pi(0.25) == (0.0, 1.0) or orc.rid_sincos2pi(0.25)[1] == 1.0
    c, s = orc.rid_sincos2pi(0.5)
    assert c == -1.0 and abs(s) == 0.0
    c, s = orc.rid_sincos2pi(0.125)  # angle pi/4
    assert abs(c - math.sqrt(0.5)) <= 2.3e-16 and abs(s - math.sqrt(0.5)) <= 2.3e-16


def test_uniform_range_and_exactness(orc):
    # w = 0 -> u = 0.5 * 2^-52 = 2^-53; w = 2^64-1 -> (2^52 - 1 + 0.5) 2^-52 = 1 - 2^-53 (§3).
    # Recover u1 from the normal: rho = sqrt(-ln u1) — checked on the extreme counters through
    # the formula applied to the Philox output of a counter whose x0, x1 we know.
    for ctr, key, want in _kat():
        w = (want[1] << 32) | want[0]
        u = ((w >> 12) + 0.5) * 2.0**-52
        assert 2.0**-53 <= u <= 1 - 2.0**-53
        assert u == float((w >> 12) + 0.5) / 2**52  # exact


def test_normal_bits_from_uniforms(orc):
    # N(seed, s, i, j) = sqrt(-ln u1) (cos, sin)(2 pi u2) with u from the Philox words (§4).
    for seed, s, i, j in [(1, 4, 0, 0), (2**40 + 3, 1, 17, 99), (5, 20, 123456, 7)]:
        key = [seed & 0xFFFFFFFF, seed >> 32]
        x = orc.philox4x32_10([i, j, s, 0], key)
        u1 = (((int(x[1]) << 32 | int(x[0])) >> 12) + 0.5) * 2.0**-52
        u2 = (((int(x[3]) << 32 | int(x[2])) >> 12) + 0.5) * 2.0**-52
        z = orc.normal(seed, s, i, j)
        rho = math.sqrt(-math.log(u1))
        assert abs(z.real - rho * math.cos(2 * math.pi * u2)) <= 1e-15 * max(1, rho)
        assert abs(z.imag - rho * math.sin(2 * math.pi * u2)) <= 1e-15 * max(1, rho)


def test_normal_statistics(orc):
    Z = orc.normal_matrix(1, 4, 256, 256).ravel()
    N = Z.size
    assert abs(Z.mean()) <= 4 / math.sqrt(N)
    assert 0.95 <= np.mean(np.abs(Z) ** 2) <= 1.05
    Zb = orc.normal_matrix(3, 1, 400, 500).ravel()
    for part in (Zb.real, Zb.imag):
        v = part.var()
        se = 0.5 * math.sqrt(2 / part.size)
        assert abs(v - 0.5) <= 5 * se
        assert stats.kstest(part / math.sqrt(0.5), stats.norm.cdf).pvalue > 1e-4
    assert abs(np.corrcoef(Zb.real, Zb.imag)[0, 1]) <= 5 / math.sqrt(Zb.size)


def test_streams_and_indices_independent(orc):
    a = orc.normal_matrix(1, 1, 64, 64)
    b = orc.normal_matrix(1, 2, 64, 64)
    c = orc.normal_matrix(2, 1, 64, 64)
    assert not np.any(a == b) and not np.any(a == c)
    # pure function of (seed, s, i, j): an offset block equals the block of a larger fill
    big = orc.normal_matrix(9, 3, 50, 40)
    sub = orc.normal_matrix(9, 3, 20, 10, row0=13, col0=25)
    assert np.array_equal(big[13:33, 25:35], sub)
    assert orc.normal(9, 3, 13, 25) == big[13, 25]
