"""The paper's own QR on the GPU: column-pivoted classical Gram-Schmidt
with one reorthogonalisation ("CGS with iteration"), k_cgs2.cu, selected by
rid_set_qr(ctx, RID_QR_CGS2) — against the oracle's orc_pivoted_cgs2, which is the same algorithm
step by step (pinned in test_oracle.py against LAPACK ZGEQP3, brute force and closed forms).

Bar (the same as the Householder path's): J equal to the oracle's unless the step is
tie-ambiguous (reading R18), R = Q^H Y and P within 1e-10 relative, resid norms within 1e-10, the
identity block exact, rank failure reported with the oracle's rank.
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


def relf(a, b):
    return np.linalg.norm(a - b) / np.linalg.norm(b)


CASES = [  # (name, seed, m, n, k, l, noise): the configs' k/l structure reduced, and edge shapes
    ("C1", 1, 1024, 512, 16, 24, 0.0),
    ("C2s", 1, 2048, 2048, 64, 80, 1e-10),
    ("C4s", 1, 2048, 2048, 512, 528, 1e-8),
    ("C5s", 1, 8192, 2048, 256, 272, 1e-10),
    ("k=l", 1, 500, 300, 24, 24, 1e-9),
    ("k=n", 2, 300, 40, 40, 48, 0.0),
    ("k=1", 4, 256, 100, 1, 9, 1e-6),
    ("one column", 5, 128, 1, 1, 4, 0.0),
    ("ragged", 6, 1001, 777, 13, 29, 1e-8),
    ("l=1100", 3, 1500, 1300, 600, 1100, 1e-9),
    ("l=2000", 4, 2100, 700, 640, 2000, 0.0),
]


@pytest.mark.parametrize("fused", ["1", "0"])
@pytest.mark.parametrize("name,seed,m,n,k,l,noise", CASES)
def test_cgs2_qr_parity(rid, orc, monkeypatch, fused, name, seed, m, n, k, l, noise):
    """rid_qrcp with CGS2 on the oracle's own sketch: J, R = Q^H Y, resid norms and margins —
    the persistent kernel (default; columns in registers up to l = 544, chunked beyond) and the
    multi-launch path (RID_CGS2_FUSED=0)."""
    monkeypatch.setenv("RID_CGS2_FUSED", fused)
    Y_o = orc.sketch(orc.generate(seed, m, n, k, noise), seed, l)
    q = orc.pivoted_qr(Y_o, k)
    Yd = torch.from_numpy(Y_o.T.copy()).T.cuda()
    J, R, resid, margin, diag = rid.qrcp(Yd, k, qr="cgs2")
    if k > 1 and q.tie_margins[:-1].min() < 1e-10:
        pytest.skip(f"{name}: tie-ambiguous (margin {q.tie_margins[:-1].min():.2e})")
    J = np_(J)
    assert J.tolist() == q.J.tolist()
    R, R_o = np_(R), q.R
    nonpiv = np.setdiff1d(np.arange(n), J)
    if nonpiv.size:
        assert relf(R[:, nonpiv], R_o[:, nonpiv]) <= 1e-10
    T, T_o = R[:, J], R_o[:, J]
    iu = np.triu_indices(k)
    assert relf(T[iu], T_o[iu]) <= 1e-10
    assert np.all(np.tril(T, -1) == 0)  # the dense triangle rid_qrcp reports for pivot columns
    assert np.max(np.abs(np_(resid) - q.resid_norms) / q.resid_norms) <= 1e-10
    mg, mg_o = np_(margin)[:-1], q.tie_margins[:-1]
    assert np.all(np.abs(mg - mg_o) <= 1e-9)
    assert diag["rank_achieved"] == k


@pytest.mark.parametrize("name,seed,m,n,k,l,noise", CASES[:6])
def test_cgs2_decompose_parity(rid, orc, name, seed, m, n, k, l, noise):
    """The whole ID with the paper's QR: J and P against the oracle's decompose (CGS2 too)."""
    A_o = orc.generate(seed, m, n, k, noise)
    d = orc.decompose(A_o, k, l, seed)
    r = rid.decompose(rid.generate(seed, m, n, k, noise), k, l, seed, qr="cgs2")
    if k > 1 and d.tie_margins[:-1].min() < 1e-10:
        pytest.skip(f"{name}: tie-ambiguous (margin {d.tie_margins[:-1].min():.2e})")
    J, P = np_(r.J), np_(r.P)
    assert J.tolist() == d.J.tolist()
    assert np.array_equal(P[:, J], np.eye(k, dtype=complex))
    assert relf(P, d.P) <= 1e-10
    assert r.diag["rank_achieved"] == k and r.diag["retries"] == 0


def test_cgs2_paper_pipeline_srft(rid, orc):
    """The paper's algorithm end to end (SRFT randomisation + CGS with iteration + factor R)."""
    seed, m, n, k, l, noise = 1, 2048, 1024, 128, 256, 1e-9
    A_o = orc.generate(seed, m, n, k, noise)
    d = orc.decompose(A_o, k, l, seed, sketch_kind="srft")
    r = rid.decompose(rid.generate(seed, m, n, k, noise), k, l, seed, sketch="srft", qr="cgs2")
    assert d.tie_margins[:-1].min() >= 1e-10
    assert np_(r.J).tolist() == d.J.tolist()
    assert relf(np_(r.P), d.P) <= 1e-10


@pytest.mark.parametrize("fused", ["1", "0"])
def test_cgs2_matches_householder_and_is_deterministic(rid, monkeypatch, fused):
    """Same J as the Householder kernels, P to rounding; two CGS2 runs bitwise identical (a race
    canary for the grid barriers of the persistent kernel)."""
    monkeypatch.setenv("RID_CGS2_FUSED", fused)
    seed, m, n, k, l, noise = 9, 4096, 4100, 200, 216, 1e-9
    A = rid.generate(seed, m, n, k, noise)
    r1 = rid.decompose(A, k, l, seed, qr="cgs2")
    r2 = rid.decompose(A, k, l, seed, qr="cgs2")
    assert torch.equal(r1.J, r2.J)
    assert np.array_equal(np.ascontiguousarray(np_(r1.P)).view(np.uint64),
                          np.ascontiguousarray(np_(r2.P)).view(np.uint64))
    rh = rid.decompose(A, k, l, seed)
    assert torch.equal(rh.J, r1.J)
    assert relf(np_(r1.P), np_(rh.P)) <= 1e-11


def test_cgs2_rank_failure(rid, orc):
    """Exact rank 5 < k = 6: the failure flag stops every later kernel; RID_ERANK with rank 5
    after the re-randomisation; the context stays usable."""
    A = rid.generate(3, 300, 120, 5, 0.0)
    with pytest.raises(rid.RidError) as e:
        rid.decompose(A, 6, 12, 3, qr="cgs2")
    assert e.value.status == rid.RID_ERANK
    assert "rank 5" in str(e.value)
    Y_o = orc.sketch(orc.generate(3, 300, 120, 5, 0.0), 3, 12)
    assert orc.pivoted_qr(Y_o, 6).rank_achieved == 5
    r = rid.decompose(A, 5, 12, 3, qr="cgs2")
    assert r.diag["rank_achieved"] == 5


def test_set_qr_rejects_unknown_kind(rid):
    ctx = rid.default_context()
    assert rid.lib().rid_set_qr(ctx.h, 7) == rid.RID_EINVAL
    assert rid.lib().rid_set_qr(ctx.h, rid.QR_HOUSEHOLDER) == rid.RID_OK
