"""GPU parity of the INT8_CRT sketch engine (k_crt.cu, reading R33): the sketch
Y = R A as the exact integer product of R and A rounded to b bits relative to their row / column
maxima, computed as T int8 GEMMs on tcgen05 and recovered by the Chinese remainder theorem.

Bars (BASELINE.json:north_star): Y within 1e-12 relative Frobenius of the oracle (the rounding of
the operands to b = 45-46 bits gives ~4e-14, tested at 2e-13); J equal to the oracle's and P
within 1e-10 through rid_decompose. Because the integer product is exact, Y does not depend on
how the columns are blocked or sharded: those checks are bitwise.
"""
import threading

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")


@pytest.fixture(scope="module")
def rid():
    if not torch.cuda.is_available():
        pytest.skip("no GPU")
    from paper_1205_3830_b200 import build

    build.build()
    import paper_1205_3830_b200 as rid

    return rid


@pytest.fixture(scope="module")
def ctx(rid):
    c = rid.Context(0, torch.cuda.current_stream())
    c.set_sketch_engine("int8_crt")
    yield c
    c.close()


def np_(t):
    return t.cpu().numpy() if hasattr(t, "cpu") else np.asarray(t)


def bits_equal(a, b):
    a, b = np.asarray(a), np.asarray(b)
    return a.shape == b.shape and np.array_equal(np.ascontiguousarray(a).view(np.uint64),
                                                 np.ascontiguousarray(b).view(np.uint64))


def relf(a, b):
    return np.linalg.norm(a - b) / np.linalg.norm(b)


TOL_Y = 2e-13  # north-star bar 1e-12; the CRT's own error is ~3e-15 (b = 49-50), the oracle's ~1e-14

SKETCH_CASES = [  # (seed, m, n, k, noise, l): the shapes the plan's tiling must cover
    (1, 1024, 512, 16, 0.0, 24),     # C1: l < 32 (one 32-row tile, 8 padding rows)
    (2, 333, 45, 5, 1e-9, 13),       # ragged m (K' padding), n < 128 (one partial column tile)
    (3, 2048, 200, 64, 1e-10, 80),   # C2 structure, a ragged column tile
    (4, 4096, 150, 128, 1e-12, 144), # C3 structure
    (5, 2048, 270, 256, 1e-10, 272), # C5 structure: two row tiles (144 + 128)
    (6, 1024, 540, 512, 1e-8, 528),  # C4 structure: three row tiles of 176
    (7, 3000, 9, 3, 0.0, 1),         # l = 1
    (8, 1000, 300, 10, 1e-10, 37),   # l not a multiple of 16
]


@pytest.mark.parametrize("seed,m,n,k,noise,l", SKETCH_CASES)
def test_crt_sketch_parity(rid, orc, ctx, seed, m, n, k, noise, l):
    assert rid.sketch_engine(m, l, n, ctx=ctx) == "int8_crt"
    A_g = rid.generate(seed, m, n, k, noise, ctx=ctx)
    Y_o = orc.sketch(orc.generate(seed, m, n, k, noise), seed, l)
    Y_g = np_(rid.sketch(A_g, seed, l, ctx=ctx))
    assert relf(Y_g, Y_o) <= TOL_Y
    # column by column as well (each column has its own scale)
    colerr = np.linalg.norm(Y_g - Y_o, axis=0) / np.linalg.norm(Y_o, axis=0)
    assert colerr.max() <= 4 * TOL_Y


def _exact_sketch(R, A):
    """Y = R A exactly (Python integers: every double is an integer multiple of 2^-1074), rounded
    once to complex128."""
    from fractions import Fraction

    def ints(x):
        return [int(Fraction(float(v)) * (1 << 1074)) for v in x]

    l, n = R.shape[0], A.shape[1]
    Rr = [ints(R[i].real) for i in range(l)]
    Ri = [ints(R[i].imag) for i in range(l)]
    Ar = [ints(A[:, j].real) for j in range(n)]
    Ai = [ints(A[:, j].imag) for j in range(n)]
    Y = np.zeros((l, n), np.complex128)
    sc = Fraction(1, 1 << 2148)
    for i in range(l):
        for j in range(n):
            re = sum(a * b for a, b in zip(Rr[i], Ar[j])) - sum(a * b for a, b in zip(Ri[i], Ai[j]))
            im = sum(a * b for a, b in zip(Rr[i], Ai[j])) + sum(a * b for a, b in zip(Ri[i], Ar[j]))
            Y[i, j] = complex(float(Fraction(re) * sc), float(Fraction(im) * sc))
    return Y


def test_crt_more_accurate_than_fp64(rid, orc, ctx, monkeypatch):
    """Against the EXACT product (big-integer arithmetic), the INT8_CRT sketch (b = 50-bit operands,
    exact accumulation, one final rounding) is more accurate than the fp64 ordered fused chain the
    oracle and the DMMA 4-product kernel compute (accumulated rounding ~u sqrt(m / 2))."""
    m, n, l, seed = 16384, 4, 8, 11
    assert rid.crt_plan(l, m)["b"] == 50
    A_o = orc.generate(seed, m, n, 3, 1e-9)
    R = orc.normal_matrix(seed, 4, l, m)  # the sketch matrix (stream 4, reading R4/R5)
    Y_ex = _exact_sketch(R, A_o)
    A_g = torch.from_numpy(np.asfortranarray(A_o)).cuda()
    Y_crt = np_(rid.sketch(A_g, seed, l, ctx=ctx))
    Y_orc = orc.sketch(A_o, seed, l)
    e_crt, e_orc = relf(Y_crt, Y_ex), relf(Y_orc, Y_ex)
    assert e_crt <= 1e-14, e_crt
    assert e_crt < e_orc, (e_crt, e_orc)


@pytest.mark.parametrize("m,n,l", [(2048, 700, 528), (4096, 300, 272), (1024, 513, 80),
                                   (1024, 300, 16), (3000, 257, 48), (2048, 400, 400)])
def test_crt_pair_kernel(rid, orc, monkeypatch, m, n, l):
    """The CTA-pair GEMM (k_imma2, tcgen05.mma.cta_group::2, RID_CRT_2SM=1): row tiles in 16-row
    granules like the single-CTA kernel (528 -> 3 x 176: 88 rows per CTA; l = 16: 8 rows per CTA),
    column tiles of 256 (ragged n), bitwise equal to the
    single-CTA kernel (the integer products are exact) and within the bar of the oracle."""
    c = rid.Context(0, torch.cuda.current_stream())
    c.set_sketch_engine("int8_crt")
    A_g = rid.generate(5, m, n, 16, 1e-9, ctx=c)
    Y1 = np_(rid.sketch(A_g, 5, l, ctx=c))
    monkeypatch.setenv("RID_CRT_2SM", "1")
    assert rid.crt_plan(l, m)["nc"] % 16 == 0
    Y2 = np_(rid.sketch(A_g, 5, l, ctx=c))
    assert bits_equal(Y1, Y2)
    Y_o = orc.sketch(orc.generate(5, m, n, 16, 1e-9), 5, l)
    assert relf(Y2, Y_o) <= TOL_Y
    c.close()


@pytest.mark.parametrize("m,n,l", [(1, 1, 1), (3, 5, 2), (17, 2, 17), (300, 7, 300),
                                   (2048, 130, 2048), (4100, 33, 1000)])
def test_crt_edge_shapes(rid, orc, ctx, m, n, l):
    """Tiny operands (TMA boxes larger than the tensors: zero-filled), l = m, the maximum l = 2048
    (8 row tiles of 256), uneven row tiles (300 = 160 + 144, 1000 = 4 x 256 - 24)."""
    A_o = orc.generate(7, m, n, min(m, n, 3), 1e-9)
    Y_o = orc.sketch(A_o, 7, l)
    Y_g = np_(rid.sketch(torch.from_numpy(np.asfortranarray(A_o)).cuda(), 7, l, ctx=ctx))
    assert relf(Y_g, Y_o) <= TOL_Y


def test_crt_two_k_slices(rid, orc, ctx):
    """m > 66560: K' = 2m no longer fits one exact int32 accumulation; two K slices whose
    residues are summed mod p before the reconstruction."""
    m, n, l = 70000, 130, 24
    assert rid.crt_plan(l, m)["kslices"] == 2
    A_g = rid.generate(3, m, n, 8, 1e-10, ctx=ctx)
    Y_o = orc.sketch(orc.generate(3, m, n, 8, 1e-10), 3, l)
    assert relf(np_(rid.sketch(A_g, 3, l, ctx=ctx)), Y_o) <= TOL_Y


def test_crt_column_scales(rid, orc, ctx):
    """Per-column scaling: columns 1e±200 apart, an all-zero column and a one-spike column are each
    reproduced to the same relative accuracy (a single global scale would flush the small ones)."""
    m, n, l, seed = 512, 160, 24, 5
    A = orc.generate(seed, m, n, 8, 1e-6).copy(order="F")
    A[:, 3] *= 1e200
    A[:, 4] *= 1e-200
    A[:, 5] = 0
    A[:, 6] = 0
    A[17, 6] = 3.0 - 2.0j
    A[:, 7] *= 1e-300  # scale 2^s with s > 1023: applied in two exact steps
    Y_o = orc.sketch(A, seed, l)
    Y_g = np_(rid.sketch(torch.from_numpy(A).cuda(), seed, l, ctx=ctx))
    assert np.all(Y_g[:, 5] == 0)
    for j in range(n):
        if j == 5:
            continue
        assert np.linalg.norm(Y_g[:, j] - Y_o[:, j]) <= 4 * TOL_Y * np.linalg.norm(Y_o[:, j]), j
    # an inf or NaN in a column makes that column's sketch NaN (as the fp64 product would)
    A[9, 8] = np.inf
    A[2, 9] = np.nan
    Y_g = np_(rid.sketch(torch.from_numpy(A).cuda(), seed, l, ctx=ctx))
    assert np.all(np.isnan(Y_g[:, 8])) and np.all(np.isnan(Y_g[:, 9]))
    assert np.all(np.isfinite(Y_g[:, 10:]))


def test_crt_blocks_bitwise(rid, ctx):
    """The integer product is exact: any column block of A sketches to the same bits as the same
    columns of the whole sketch, and a host A (streamed in chunks) gives the same bits."""
    m, n, l, seed = 2048, 1024, 80, 9
    A = rid.generate(seed, m, n, 64, 1e-10, ctx=ctx)
    Y = np_(rid.sketch(A, seed, l, ctx=ctx))
    for c0, w in ((128, 256), (0, 64), (1000, 24), (333, 100)):
        Yb = np_(rid.sketch(A[:, c0:c0 + w], seed, l, n=n, col0=c0, ctx=ctx))
        assert bits_equal(Yb, Y[:, c0:c0 + w]), (c0, w)
    Yh = rid.sketch(np.asfortranarray(np_(A)), seed, l, ctx=ctx)
    assert bits_equal(Yh, Y)


def test_crt_engine_selection(rid, monkeypatch):
    c = rid.Context(0, torch.cuda.current_stream())
    assert rid.sketch_engine(8192, 80, 8192, ctx=c) == "fp64_dmma"      # C2: l m n < 2^34
    assert rid.sketch_engine(65536, 144, 4096, ctx=c) == "int8_crt"     # C3
    assert rid.sketch_engine(32768, 528, 32768, ctx=c) == "int8_crt"    # C4
    assert not rid.sketch_strassen(32768, 528, 32768, ctx=c)
    c.set_sketch_engine("fp64_dmma")
    assert rid.sketch_engine(32768, 528, 32768, ctx=c) == "fp64_dmma"
    assert rid.sketch_strassen(32768, 528, 32768, ctx=c)
    monkeypatch.setenv("RID_SKETCH_CRT", "1")
    assert rid.sketch_engine(8192, 80, 8192, ctx=c) == "int8_crt"
    monkeypatch.delenv("RID_SKETCH_CRT")
    with pytest.raises(KeyError):
        c.set_sketch_engine("bogus")
    c.set_sketch_engine("int8_crt")  # l > 2048: the engine's limit, DMMA whatever the selection
    assert rid.sketch_engine(4096, 2100, 64, ctx=c) == "fp64_dmma"
    with pytest.raises(rid.RidError):
        rid.crt_plan(2100, 4096)
    c.close()


DEC_CASES = [  # (name, seed, m, n, k, l, noise): tests/test_gpu_parity.py DEC_CASES
    ("C1", 1, 1024, 512, 16, 24, 0.0),
    ("C2s", 1, 2048, 2048, 64, 80, 1e-10),
    ("C3s", 1, 8192, 1024, 128, 144, 1e-12),
    ("C4s", 1, 2048, 2048, 512, 528, 1e-8),
    ("C5s", 1, 8192, 2048, 256, 272, 1e-10),
    ("ragged", 3, 700, 333, 20, 29, 1e-7),
]


@pytest.mark.parametrize("name,seed,m,n,k,l,noise", DEC_CASES)
def test_crt_decompose_parity(rid, orc, ctx, name, seed, m, n, k, l, noise):
    A_o = orc.generate(seed, m, n, k, noise)
    d = orc.decompose(A_o, k, l, seed)
    A_g = rid.generate(seed, m, n, k, noise, ctx=ctx)
    r = rid.decompose(A_g, k, l, seed, ctx=ctx)
    assert r.diag["sketch_engine"] == 2 and r.diag["t_sketch_tc"] > 0
    assert r.diag["t_sketch_tc"] <= r.diag["t_sketch"]
    assert np_(r.J).tolist() == d.J.tolist()
    P_g = np_(r.P)
    assert bits_equal(P_g[:, np_(r.J)], np.eye(k, dtype=np.complex128))
    assert relf(P_g, d.P) <= 1e-10
    # repeated call: the CUDA-graph replay gives the same bits and still times the GEMMs
    r2 = rid.decompose(A_g, k, l, seed, ctx=ctx)
    r3 = rid.decompose(A_g, k, l, seed, ctx=ctx)
    assert bits_equal(np_(r3.P), P_g) and bits_equal(np_(r2.P), P_g)
    assert r3.diag["t_sketch_tc"] > 0


@pytest.mark.parametrize("name,seed,m,n,k,l,noise", [DEC_CASES[1], DEC_CASES[3], DEC_CASES[5]])
def test_crt_solve_selection(rid, orc, ctx, monkeypatch, name, seed, m, n, k, l, noise):
    """RID_SOLVE_CRT=1: T = R11^-1 R12 on the INT8_CRT engine as well (a tested selection)."""
    monkeypatch.setenv("RID_SOLVE_CRT", "1")
    A_o = orc.generate(seed, m, n, k, noise)
    d = orc.decompose(A_o, k, l, seed)
    r = rid.decompose(rid.generate(seed, m, n, k, noise, ctx=ctx), k, l, seed, ctx=ctx)
    assert np_(r.J).tolist() == d.J.tolist()
    P_g = np_(r.P)
    assert bits_equal(P_g[:, np_(r.J)], np.eye(k, dtype=np.complex128))
    assert relf(P_g, d.P) <= 1e-10


def test_crt_multirank_bitwise(rid, orc):
    """G column shards on one GPU (in-process communicator, one thread per rank): J and the
    concatenated P bitwise equal to one rank, on the INT8_CRT engine."""
    m, n, k, l, noise, seed = 2048, 2048, 64, 80, 1e-10, 1
    one = rid.Context(0, torch.cuda.current_stream())
    one.set_sketch_engine("int8_crt")
    A = rid.generate(seed, m, n, k, noise, ctx=one)
    ref = rid.decompose(A, k, l, seed, ctx=one)
    torch.cuda.synchronize()
    for G in (2, 4):
        streams = [torch.cuda.Stream() for _ in range(G)]
        ctxs = [rid.Context(0, s) for s in streams]
        rid.comm_init_local(ctxs)
        for c in ctxs:
            c.set_sketch_engine("int8_crt")
        out = [None] * G
        nl = n // G

        def body(g):
            with torch.cuda.stream(streams[g]):
                out[g] = rid.decompose(A[:, g * nl:(g + 1) * nl], k, l, seed, n=n, col0=g * nl,
                                       ctx=ctxs[g])

        th = [threading.Thread(target=body, args=(g,)) for g in range(G)]
        for t in th:
            t.start()
        for t in th:
            t.join(timeout=600)
        torch.cuda.synchronize()
        for g in range(G):
            assert np_(out[g].J).tolist() == np_(ref.J).tolist()
        P = np.concatenate([np_(o.P) for o in out], axis=1)
        assert bits_equal(P, np_(ref.P)), G
        for c in ctxs:
            c.close()
    one.close()


@pytest.mark.parametrize("m,n,l", [(8192, 2048, 144), (65536, 512, 144), (4096, 1000, 80)])
def test_crt_kslice_balance_bitwise(rid, ctx, monkeypatch, m, n, l):
    """Small sketches get extra K slices so that the GEMM's work items fill the waves (C3: 2
    slices); the slices' residues are summed mod p, so Y has the same bits with and without
    (RID_CRT_NOBALANCE=1)."""
    seed = 12
    A = rid.generate(seed, m, n, 32, 1e-10, ctx=ctx)
    Y1 = np_(rid.sketch(A, seed, l, ctx=ctx))
    monkeypatch.setenv("RID_CRT_NOBALANCE", "1")
    Y0 = np_(rid.sketch(A, seed, l, ctx=ctx))
    assert bits_equal(Y1, Y0)


def test_crt_prep_cluster_bitwise(rid, ctx, monkeypatch):
    """Tall matrices (m > 65536) prepare each column with a CTA pair (partial maxima over
    distributed shared memory); any cluster size gives the same residues, so the same Y."""
    m, n, l, seed = 70000, 300, 80, 13
    A = rid.generate(seed, m, n, 16, 1e-10, ctx=ctx)
    Y2 = np_(rid.sketch(A, seed, l, ctx=ctx))
    for cl in ("1", "4"):
        monkeypatch.setenv("RID_CRT_PREP_CLUSTER", cl)
        assert bits_equal(np_(rid.sketch(A, seed, l, ctx=ctx)), Y2), cl
