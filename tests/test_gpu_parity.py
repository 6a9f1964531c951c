"""GPU parity: the CUDA path (through the C ABI) against the CPU oracle, element by element.

Bars (BASELINE.json:north_star):
- generated inputs, Philox normals, and — because the DMMA K-chain is the oracle's ascending fused
  order — the sketch Y: BIT-EXACT (checked on the uint64 bit patterns);
- J: identical arrays (the oracle logs the smallest top-2 gap; all cases here are well separated);
- P: relative Frobenius error <= 1e-10 (reading R17); P[:, J] = I bitwise;
- error estimate on the same (A, J, P): relative <= 1e-10 (reading R16 (i));
  |rho_gpu - rho_oracle| <= 1e-10 for each side's own P (R16 (ii)); exact rank: rho <= 1e-13 (iii).
Sizes are reduced copies of C1–C5 (same k/l structure and noise) that the oracle finishes in
seconds while still spanning several tiles and a ragged tail; tests/test_gpu_fullsize.py covers
the full configs.
"""
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


def np_(t):
    return t.cpu().numpy() if hasattr(t, "cpu") else np.asarray(t)


def bits_equal(a, b):
    a, b = np.asarray(a), np.asarray(b)
    return a.shape == b.shape and np.array_equal(np.ascontiguousarray(a).view(np.uint64),
                                                 np.ascontiguousarray(b).view(np.uint64))


def relf(a, b):
    return np.linalg.norm(a - b) / np.linalg.norm(b)


# ------------------------------------------------------------------------- RNG / generation ---
@pytest.mark.parametrize("seed,s,rows,cols,row0,col0", [
    (1, 1, 37, 29, 0, 0), (1, 4, 24, 1000, 0, 0), (2**40 + 7, 20, 13, 7, 5, 100000),
    (3, 5, 1000, 1, 0, 0), (0, 3, 64, 64, 2**31, 7)])
def test_normal_fill_bitexact(rid, orc, seed, s, rows, cols, row0, col0):
    g = np_(rid.normal_fill(seed, s, rows, cols, row0, col0))
    o = orc.normal_matrix(seed, s, rows, cols, row0, col0)
    assert bits_equal(g, o)


GEN_CASES = [  # (seed, m, n, k, noise, col0, n_loc)
    (1, 1024, 512, 16, 0.0, 0, 512),         # C1 exactly
    (2, 300, 77, 7, 1e-8, 0, 77),            # ragged m, n, odd k
    (2, 300, 77, 7, 1e-8, 50, 27),           # a column shard
    (3, 2048, 130, 64, 1e-10, 0, 130),       # C2 structure, ragged n
    (4, 4100, 196, 128, 1e-12, 0, 196),      # C3 structure, ragged m
    (5, 64, 64, 1, 0.0, 0, 64),              # k = 1
]


@pytest.mark.parametrize("seed,m,n,k,noise,col0,n_loc", GEN_CASES)
def test_generate_bitexact(rid, orc, seed, m, n, k, noise, col0, n_loc):
    g = np_(rid.generate(seed, m, n, k, noise, col0, n_loc))
    o = orc.generate(seed, m, n, k, noise, col0, n_loc)
    assert bits_equal(g, o)


def test_generate_host_buffer_and_empty(rid, orc):
    out = np.zeros((200, 33), np.complex128, order="F")
    rid.generate(9, 200, 40, 5, 1e-6, 7, 33, out=out)
    assert bits_equal(out, orc.generate(9, 200, 40, 5, 1e-6, 7, 33))
    rid.generate(9, 200, 40, 5, 1e-6, 40, 0, out=np.zeros((200, 0), np.complex128, order="F"))
    with pytest.raises(rid.RidError):
        rid.generate(9, 200, 40, 50, 1e-6, 0, 40)  # k > n


# ------------------------------------------------------------------------------- sketch -------
SKETCH_CASES = [  # (seed, m, n, k, noise, l)
    (1, 1024, 512, 16, 0.0, 24),     # C1
    (2, 333, 45, 5, 1e-9, 13),       # ragged everything, odd l
    (3, 2048, 200, 64, 1e-10, 80),   # C2 structure (FR = 10)
    (4, 4096, 150, 128, 1e-12, 144), # C3 structure (FR = 9)
    (5, 2048, 270, 256, 1e-10, 272), # C5 structure (FR = 17)
    (6, 1024, 540, 512, 1e-8, 528),  # C4 structure (FR = 11)
    (7, 3000, 9, 3, 0.0, 1),         # l = 1
]


@pytest.mark.parametrize("seed,m,n,k,noise,l", SKETCH_CASES)
def test_sketch_bitexact(rid, orc, seed, m, n, k, noise, l, monkeypatch):
    A_g = rid.generate(seed, m, n, k, noise)
    A_o = orc.generate(seed, m, n, k, noise)
    Y_o = orc.sketch(A_o, seed, l)
    # the default launch: Gauss's three products (reading R31), K split into S slices when the
    # tile count is small: the north-star bar, and in practice a few ulps
    assert rid.sketch_mults() == 3
    Y_g = np_(rid.sketch(A_g, seed, l))
    assert relf(Y_g, Y_o) <= 1e-12
    # random-walk rounding of an m-term sum, ~u·sqrt(m), times the ~4x cancellation of
    # Im = P3 - P1 - P2: <= 5e-14 for m <= 8192 (measured 2e-15 .. 1e-14 on these shapes)
    tol3 = 5e-14
    assert relf(Y_g, Y_o) <= tol3
    monkeypatch.setenv("RID_SKETCH_SPLIT", "1")
    assert relf(np_(rid.sketch(A_g, seed, l)), Y_o) <= tol3
    # the ordered real embedding (4 products): one slice is the single ascending fused chain,
    # bit-identical to the oracle's naive loop
    monkeypatch.setenv("RID_SKETCH_4M", "1")
    assert rid.sketch_mults() == 4
    Y_1 = np_(rid.sketch(A_g, seed, l))
    assert bits_equal(Y_1, Y_o)
    # an explicit 3-slice split: fixed-order slice sums, within rounding
    monkeypatch.setenv("RID_SKETCH_SPLIT", "3")
    Y_3 = np_(rid.sketch(A_g, seed, l))
    assert relf(Y_3, Y_o) <= 1e-14
    monkeypatch.setenv("RID_SKETCH_4M", "0")
    Y_33 = np_(rid.sketch(A_g, seed, l))
    assert relf(Y_33, Y_o) <= tol3


def test_sketch_retry_stream_and_ld(rid, orc):
    A = orc.generate(11, 500, 30, 4, 1e-9)
    big = np.zeros((520, 30), np.complex128, order="F")
    big[:500] = A  # lda = 520 > m: the view A_view has stride 520
    At = torch.from_numpy(big).T.contiguous().T.cuda()[:500]
    assert At.stride() == (1, 520)
    Y = np_(rid.sketch(At, 11, 9, stream=20))
    Y_o = orc.sketch(A, 11, 9, stream=20)
    assert relf(Y, Y_o) <= 5e-14  # Gauss's three products (default), see test_sketch_bitexact
    with pytest.MonkeyPatch.context() as mp:  # the ordered chain: bitwise
        mp.setenv("RID_SKETCH_4M", "1")
        assert bits_equal(np_(rid.sketch(At, 11, 9, stream=20)), Y_o)


# ------------------------------------------------------------------------------ decompose ----
DEC_CASES = [  # (name, seed, m, n, k, l, noise)
    ("C1", 1, 1024, 512, 16, 24, 0.0),
    ("C2s", 1, 2048, 2048, 64, 80, 1e-10),
    ("C3s", 1, 8192, 1024, 128, 144, 1e-12),
    ("C4s", 1, 2048, 2048, 512, 528, 1e-8),
    ("C5s", 1, 8192, 2048, 256, 272, 1e-10),
    ("ragged", 3, 700, 333, 20, 29, 1e-7),
    ("n=k", 4, 64, 12, 12, 16, 0.0),
]


@pytest.fixture(scope="module")
def oracle_dec(orc):
    cache = {}

    def get(seed, m, n, k, l, noise):
        key = (seed, m, n, k, l, noise)
        if key not in cache:
            A = orc.generate(seed, m, n, k, noise)
            cache[key] = (A, orc.decompose(A, k, l, seed))
        return cache[key]

    return get


@pytest.mark.parametrize("name,seed,m,n,k,l,noise", DEC_CASES)
def test_decompose_parity(rid, orc, oracle_dec, name, seed, m, n, k, l, noise):
    A_o, d = oracle_dec(seed, m, n, k, l, noise)
    A_g = rid.generate(seed, m, n, k, noise)
    r = rid.decompose(A_g, k, l, seed)
    J_g, P_g = np_(r.J), np_(r.P)
    margin = d.tie_margins[:-1].min() if k > 1 else np.inf
    assert margin > 1e-10, f"{name}: tie-ambiguous case (min margin {margin})"
    assert J_g.tolist() == d.J.tolist()
    assert bits_equal(P_g[:, J_g], np.eye(k, dtype=np.complex128))
    assert relf(P_g, d.P) <= 1e-10
    assert r.diag["retries"] == 0 and r.diag["rank_achieved"] == k
    assert abs(r.diag["tie_margin_min"] - margin) <= 1e-6 * max(margin, 1e-300) + 1e-12


def test_decompose_host_path_matches_device(rid):
    m, n, k, l = 1500, 400, 24, 40
    A_g = rid.generate(8, m, n, k, 1e-9)
    r_dev = rid.decompose(A_g, k, l, 8)
    A_h = np_(A_g)  # numpy, column-major -> host staging inside librid
    r_host = rid.decompose(np.asfortranarray(A_h), k, l, 8)
    assert np.array_equal(np_(r_dev.J), r_host.J)
    assert bits_equal(np_(r_dev.P), r_host.P)
    assert r_host.diag["t_h2d"] > 0


def test_g_emulation_bitwise(rid):
    """G column shards on one GPU (sketch per shard, concatenated Y, factor + solve per shard):
    J and P bitwise equal to the single-GPU call (the data path of bench.py --gpus G)."""
    m, n, k, l, noise, seed = 2048, 1024, 48, 64, 1e-10, 2
    A = rid.generate(seed, m, n, k, noise)
    ref = rid.decompose(A, k, l, seed)
    for G in (2, 4, 8):
        Ys, Ps = [], []
        for g in range(G):
            col0, nl = rid.shard_range(n, g, G)
            A_g = rid.generate(seed, m, n, k, noise, col0, nl)
            assert torch.equal(A_g.contiguous(), A[:, col0:col0 + nl].contiguous())
            Ys.append(rid.sketch(A_g, seed, l, n=n, col0=col0))  # the whole matrix's plan
        Y = torch.cat([y.T for y in Ys]).T  # column-major concatenation
        for g in range(G):
            col0, nl = rid.shard_range(n, g, G)
            J, P, _ = rid.factor_solve(Y, k, col0, nl)
            assert torch.equal(J, ref.J)
            Ps.append(P)
        P = torch.cat([p.T for p in Ps]).T
        assert bits_equal(np_(P), np_(ref.P))


def test_qrcp_on_oracle_sketch(rid, orc):
    """GPU Householder QRCP fed the oracle's Y: same J as the oracle's CGS2 and LAPACK ZGEQP3."""
    import scipy.linalg as sla

    A = orc.generate(5, 3000, 700, 40, 1e-9)
    Y = orc.sketch(A, 5, 56)
    qr_o = orc.pivoted_qr(Y, 40)
    J, R, resid, margin, _ = rid.qrcp(torch.from_numpy(Y.T.copy()).T.cuda(), 40)
    assert np_(J).tolist() == qr_o.J.tolist()
    assert np_(J).tolist() == sla.qr(Y, pivoting=True, mode="economic")[2][:40].tolist()
    np.testing.assert_allclose(np_(resid), qr_o.resid_norms, rtol=1e-12)
    R = np_(R)
    R11 = R[:, np_(J)]
    assert np.all(np.tril(R11, -1) == 0)
    assert np.allclose(np.abs(np.diag(R11)), qr_o.resid_norms, rtol=1e-12)
    # R = Q^H Y up to a diagonal unitary: |R| rows agree with the oracle's R
    assert relf(np.abs(R), np.abs(qr_o.R)) <= 1e-11


def test_rank_failure_raises(rid):
    m, n, k = 400, 200, 3
    A = rid.generate(1, m, n, k, 0.0)  # exact rank 3
    with pytest.raises(rid.RidError) as e:
        rid.decompose(A, 6, 10, 1)
    assert e.value.status == rid.RID_ERANK


def test_bad_arguments(rid):
    A = rid.generate(1, 100, 50, 4, 0.0)
    with pytest.raises(rid.RidError) as e:
        rid.decompose(A, 8, 4, 1)  # l < k
    assert e.value.status == rid.RID_EINVAL
    with pytest.raises(rid.RidError):
        rid.decompose(A, 4, 2000, 1)  # l > m
    with pytest.raises(rid.RidError) as e:
        rid.sketch(A, 1, 8, n=60, col0=20)  # columns [20, 70) outside n = 60
    assert e.value.status == rid.RID_EINVAL
    with pytest.raises(rid.RidError):
        rid.sketch(A, 1, 8, n=50, col0=-1)
    B = rid.generate(1, 3000, 40, 4, 0.0)
    with pytest.raises(rid.RidError):
        rid.decompose(B, 4, 2100, 1)  # l > 2048 (QR limit)


# ------------------------------------------------------------------------------ estimator ----
EST_CASES = [("C1", 1, 1024, 512, 16, 24, 0.0), ("C2s", 1, 2048, 2048, 64, 80, 1e-10),
             ("C3s", 1, 8192, 1024, 128, 144, 1e-12), ("C4s", 1, 2048, 2048, 512, 528, 1e-8),
             ("ragged", 3, 700, 333, 20, 29, 1e-7)]


@pytest.mark.parametrize("name,seed,m,n,k,l,noise", EST_CASES)
def test_estimator_parity(rid, orc, oracle_dec, name, seed, m, n, k, l, noise):
    q = 12
    A_o, d = oracle_dec(seed, m, n, k, l, noise)
    A_g = rid.generate(seed, m, n, k, noise)
    # (i) same (A, J, P): the oracle's J and P fed to both estimators
    Jt = torch.from_numpy(d.J.copy()).cuda()
    Pt = torch.from_numpy(d.P.T.copy()).T.cuda()
    e_o = orc.error_estimate(A_o, d.J, d.P, q, seed)
    e_g = rid.error_estimate(A_g, Jt, Pt, q, seed)
    assert abs(e_g - e_o) <= 1e-10 * e_o, (e_g, e_o)
    # (ii) each side's own P: |rho_gpu - rho_orc| <= 1e-10 with rho = est / ||A||_2
    r = rid.decompose(A_g, k, l, seed)
    e_g2 = rid.error_estimate(A_g, r.J, r.P, q, seed)
    # ||A||_2: dense SVD (every EST_CASES shape has m n <= 2^23: C3s is 8192 x 1024)
    assert m * n <= 2**23
    nA = np.linalg.svd(A_o, compute_uv=False)[0]
    assert abs(e_g2 - e_o) / nA <= 1e-10
    if noise == 0.0:
        assert e_g2 / nA <= 1e-13 and e_o / nA <= 1e-13  # (iii) exact rank


def test_estimator_host_path(rid, orc):
    A_o = orc.generate(2, 500, 120, 6, 1e-6)
    d = orc.decompose(A_o, 6, 12, 2)
    e_h = rid.error_estimate(A_o, d.J, d.P, 5, 2)  # all host buffers
    e_o = orc.error_estimate(A_o, d.J, d.P, 5, 2)
    assert abs(e_h - e_o) <= 1e-10 * e_o


def test_sketch_wave_tail_split(rid, orc, monkeypatch):
    """The trailing global columns of a nearly empty last wave are computed with a K split
    (rid_sketch_cols, reading R30): those columns agree with the oracle to rounding, every other
    column is bitwise the unsplit kernel's, and the plan is a function of the global column index
    — shards reproduce the whole matrix bit for bit."""
    seed, m, n, k, l, noise = 4, 1024, 13824, 64, 528, 1e-9  # 11 x 216 tiles = 8 over 8 waves
    monkeypatch.setenv("RID_SKETCH_STRASSEN", "0")  # this shape's default plan is Strassen's
    A = rid.generate(seed, m, n, k, noise)
    Y = np_(rid.sketch(A, seed, l))
    monkeypatch.setenv("RID_SKETCH_NOTAIL", "1")
    Y0 = np_(rid.sketch(A, seed, l))
    monkeypatch.delenv("RID_SKETCH_NOTAIL")
    tail = n - 64
    assert bits_equal(Y[:, :tail], Y0[:, :tail])
    assert not bits_equal(Y[:, tail:], Y0[:, tail:])  # the split path ran
    assert relf(Y[:, tail:], Y0[:, tail:]) <= 5e-14
    A_o = orc.generate(seed, m, n, k, noise, tail, 64)
    assert relf(Y[:, tail:], orc.sketch(A_o, seed, l)) <= 5e-14
    for G in (2, 8):
        parts = []
        for g in range(G):
            col0, nl = rid.shard_range(n, g, G)
            parts.append(np_(rid.sketch(A[:, col0:col0 + nl], seed, l, n=n, col0=col0)))
        assert bits_equal(np.concatenate(parts, axis=1), Y)
