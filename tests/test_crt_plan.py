"""CPU checks of the INT8_CRT engine's plan (host arithmetic of librid, no GPU): the moduli and the
bounds that make every step exact (reading R33).

- the moduli are odd, pairwise coprime and <= 253 (so a residue rounded to the nearest quotient
  in fp32 is within ±127 and fits int8);
- M = prod p_t exceeds 2 max|Y'| = 2 * 2m * 2^(2b) (Y' the integer sketch: 2m terms of
  products of b-bit integers), so the symmetric CRT representative is Y' itself;
- every K slice accumulates exactly in int32: K'_slice * 127^2 < 2^31;
- b <= 50: the magic-number rint and the FP64 quotient of the residue kernels stay exact
  (|a| < 2^51); the default T = 15 gives b = 50 (m <= 32768) / 49 (m <= 2^17).
"""
import math

import pytest


@pytest.fixture(scope="module")
def rid():
    from paper_1205_3830_b200 import build

    build.build()
    import paper_1205_3830_b200 as rid

    return rid


def test_moduli(rid):
    p = rid.crt_moduli()
    assert len(p) >= 15 and len(set(p)) == len(p)
    for i, a in enumerate(p):
        assert a % 2 == 1 and 128 < a <= 253
        for b in p[i + 1:]:
            assert math.gcd(a, b) == 1, (a, b)


@pytest.mark.parametrize("l,m", [(24, 1024), (80, 8192), (144, 65536), (528, 32768),
                                 (272, 131072), (13, 333), (37, 70000), (1, 3000),
                                 (2048, 1 << 20)])
def test_plan_bounds(rid, l, m):
    pl = rid.crt_plan(l, m)
    T, b, ks, Kp, nc = pl["T"], pl["b"], pl["kslices"], pl["Kp"], pl["nc"]
    mods = rid.crt_moduli()[:T]
    M = math.prod(mods)
    assert abs(math.log2(M) - pl["log2M"]) < 1e-9
    mh = (m + 63) // 64 * 64
    assert Kp >= 2 * mh and Kp % (128 * ks) == 0
    # exact integer product: |Y'| <= 2m 2^(2b) < M / 2
    assert 2 * (2 * m) * 2 ** (2 * b) < M
    # int32-exact K slices
    assert (Kp // ks) * 127 * 127 < 2**31
    assert 40 <= b <= 50
    if m <= 32768:
        assert b == 50  # T = 15 moduli: more operand bits than an fp64 GEMM's accumulated error
    # tile rows: multiples of 16, at most 256 (the Re and Im accumulators share 512 TMEM columns)
    l16 = (l + 15) // 16 * 16
    assert nc % 16 == 0 and 16 <= nc <= 256 and nc * math.ceil(l16 / nc) >= l


@pytest.mark.parametrize("l,m", [(528, 32768), (272, 131072), (144, 65536), (16, 1024), (400, 2048)])
def test_pair_plan_same_tiles(rid, monkeypatch, l, m):
    """The CTA-pair GEMM (RID_CRT_2SM=1) uses the single-CTA kernel's 16-row granules: the same row
    tiles (C4 l = 528: 3 x 176, 88 rows per CTA of the pair; C5 l = 272: 144 + 128), and each
    CTA's half is whole 8-row 128-byte swizzle atoms."""
    base = rid.crt_plan(l, m)
    monkeypatch.setenv("RID_CRT_2SM", "1")
    pair = rid.crt_plan(l, m)
    assert pair == base
    assert pair["nc"] % 16 == 0 and (pair["nc"] // 2) % 8 == 0
    if (l, m) == (528, 32768):
        assert pair["nc"] == 176
