"""Both pivoted-QR kernels of the CUDA path against the oracle (through the C ABI).

librid picks the kernel by sketch size (k_qrcp.cu): the single persistent kernel that recomputes
every residual norm exactly (variant 0, small sketches) or the blocked panels with downdated norms
and a tensor-core trailing update (variant 1, sketches past 64 MB: C4, C5). Here RID_QRCP_VARIANT
forces each on small shapes, so both are held to the same bar as the default path: J equal to the
oracle's (reading R18), P within 1e-10 (R17), the identity block exact, rank failure reported, and
the result independent of the panel width nb (RID_QRCP_NB) and bitwise run-to-run deterministic.
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


CASES = [  # (name, seed, m, n, k, l, noise): the configs' k/l structure, reduced; edge shapes
    ("C1", 1, 1024, 512, 16, 24, 0.0),
    ("C2s", 1, 2048, 2048, 64, 80, 1e-10),
    ("C4s", 1, 2048, 2048, 512, 528, 1e-8),
    ("C5s", 1, 8192, 2048, 256, 272, 1e-10),
    ("k=l", 1, 500, 300, 24, 24, 1e-9),
    ("k=n", 2, 300, 40, 40, 48, 0.0),
    ("k=1", 4, 256, 100, 1, 9, 1e-6),
    ("one column", 5, 128, 1, 1, 4, 0.0),
    ("ragged", 6, 1001, 777, 13, 29, 1e-8),
    ("n not /32", 7, 3000, 1000, 70, 86, 1e-9),
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


@pytest.mark.parametrize("variant", ["0", "1", "2", "4"])
@pytest.mark.parametrize("name,seed,m,n,k,l,noise", CASES)
def test_variant_parity(rid, oracle_dec, monkeypatch, variant, name, seed, m, n, k, l, noise):
    monkeypatch.setenv("RID_QRCP_VARIANT", variant)
    A_o, d = oracle_dec(seed, m, n, k, l, noise)
    r = rid.decompose(rid.generate(seed, m, n, k, noise), k, l, seed)
    if k > 1 and d.tie_margins[:-1].min() < 1e-10:
        pytest.skip(f"{name}: tie-ambiguous (margin {d.tie_margins[:-1].min():.2e})")
    J, P = np_(r.J), np_(r.P)
    assert J.tolist() == d.J.tolist()
    assert np.array_equal(P[:, J], np.eye(k, dtype=complex))
    assert relf(P, d.P) <= 1e-10
    assert r.diag["rank_achieved"] == k and r.diag["retries"] == 0


@pytest.mark.parametrize("nb", ["1", "3", "7", "16"])
def test_blocked_panel_width_invariance(rid, oracle_dec, monkeypatch, nb):
    """Any panel width gives the oracle's J and P within the bar (the panel boundaries move the
    tensor-core update between steps; the downdated norms and f_s carry the rest)."""
    monkeypatch.setenv("RID_QRCP_VARIANT", "1")
    monkeypatch.setenv("RID_QRCP_NB", nb)
    seed, m, n, k, l, noise = 1, 2048, 1500, 100, 116, 1e-10
    A_o, d = oracle_dec(seed, m, n, k, l, noise)
    r = rid.decompose(rid.generate(seed, m, n, k, noise), k, l, seed)
    assert np_(r.J).tolist() == d.J.tolist()
    assert relf(np_(r.P), d.P) <= 1e-10


def test_blocked_rank_failure_and_retry(rid, monkeypatch):
    """Exact rank 5 < k = 6: the blocked kernel stops at the same step on every CTA, the later
    panels see the stop flag, the library retries once and reports RID_ERANK with rank 5."""
    monkeypatch.setenv("RID_QRCP_VARIANT", "1")
    monkeypatch.setenv("RID_QRCP_NB", "2")
    A = rid.generate(3, 300, 120, 5, 0.0)
    with pytest.raises(rid.RidError) as e:
        rid.decompose(A, 6, 12, 3)
    assert e.value.status == rid.RID_ERANK
    assert "rank 5" in str(e.value)
    # the context stays usable
    r = rid.decompose(A, 5, 12, 3)
    assert r.diag["rank_achieved"] == 5


def test_blocked_deterministic_and_matches_exact_variant(rid, monkeypatch):
    """Two blocked runs are bitwise identical (a race canary for the TMA ring and the grid
    barrier); J equals the exact-recompute kernel's and P agrees to rounding."""
    seed, m, n, k, l, noise = 9, 4096, 4100, 200, 216, 1e-9
    A = rid.generate(seed, m, n, k, noise)
    monkeypatch.setenv("RID_QRCP_VARIANT", "1")
    r1 = rid.decompose(A, k, l, seed)
    r2 = rid.decompose(A, k, l, seed)
    assert torch.equal(r1.J, r2.J)
    assert np.array_equal(np.ascontiguousarray(np_(r1.P)).view(np.uint64),
                          np.ascontiguousarray(np_(r2.P)).view(np.uint64))
    assert r1.diag["tie_margin_min"] == r2.diag["tie_margin_min"]
    monkeypatch.setenv("RID_QRCP_VARIANT", "0")
    r0 = rid.decompose(A, k, l, seed)
    assert torch.equal(r0.J, r1.J)
    assert relf(np_(r1.P), np_(r0.P)) <= 1e-12
    assert abs(r0.diag["tie_margin_min"] - r1.diag["tie_margin_min"]) <= 1e-9


@pytest.mark.parametrize("name,seed,m,n,k,l,noise", [
    ("l=1100 (MAXQ 48)", 3, 1500, 1300, 600, 1100, 1e-9),
    ("l=2000 (MAXQ 64)", 4, 2100, 700, 640, 2000, 0.0),
])
def test_large_l_blocked_only(rid, oracle_dec, name, seed, m, n, k, l, noise):
    """l > 1024 (the paper's l = 2k at k = 1000, NEXT-4) runs only on the blocked kernel (the
    exact kernel holds a segment in registers): same bar against the oracle."""
    A_o, d = oracle_dec(seed, m, n, k, l, noise)
    r = rid.decompose(rid.generate(seed, m, n, k, noise), k, l, seed)
    if d.tie_margins[:-1].min() < 1e-10:
        pytest.skip(f"{name}: tie-ambiguous (margin {d.tie_margins[:-1].min():.2e})")
    J, P = np_(r.J), np_(r.P)
    assert J.tolist() == d.J.tolist()
    assert np.array_equal(P[:, J], np.eye(k, dtype=complex))
    assert relf(P, d.P) <= 1e-10


CLUSTER_CASES = [  # sketches that fit one cluster's shared memory (16 CTAs)
    ("C1", 1, 1024, 512, 16, 24, 0.0),
    ("C2s", 1, 2048, 2048, 64, 80, 1e-10),
    ("C3s", 1, 8192, 1024, 128, 144, 1e-12),
    ("k=l", 1, 500, 300, 24, 24, 1e-9),
    ("k=n", 2, 300, 40, 40, 48, 0.0),
    ("k=1", 4, 256, 100, 1, 9, 1e-6),
    ("one column", 5, 128, 1, 1, 4, 0.0),
    ("ragged", 6, 1001, 777, 13, 29, 1e-8),
]


@pytest.mark.parametrize("name,seed,m,n,k,l,noise", CLUSTER_CASES)
def test_cluster_qr_bitwise_vs_grid_kernel(rid, oracle_dec, monkeypatch, name, seed, m, n, k, l,
                                           noise):
    """The one-cluster QR (variant 3: distributed-shared-memory exchange, cluster barrier) gives
    the same J and P bits as the grid-wide shared-memory kernel (variant 4), and the oracle's J."""
    A = rid.generate(seed, m, n, k, noise)
    monkeypatch.setenv("RID_QRCP_VARIANT", "4")
    r4 = rid.decompose(A, k, l, seed)
    monkeypatch.setenv("RID_QRCP_VARIANT", "3")
    r3 = rid.decompose(A, k, l, seed)
    assert np.array_equal(np_(r3.J), np_(r4.J))
    assert np.array_equal(np.ascontiguousarray(np_(r3.P)).view(np.uint64),
                          np.ascontiguousarray(np_(r4.P)).view(np.uint64))
    A_o, d = oracle_dec(seed, m, n, k, l, noise)
    if k == 1 or d.tie_margins[:-1].min() >= 1e-10:
        assert np_(r3.J).tolist() == d.J.tolist()
    assert relf(np_(r3.P), d.P) <= 1e-10


def test_cluster_qr_rank_failure(rid, monkeypatch):
    monkeypatch.setenv("RID_QRCP_VARIANT", "3")
    A = rid.generate(1, 400, 200, 3, 0.0)  # exact rank 3
    with pytest.raises(rid.RidError) as e:
        rid.decompose(A, 6, 10, 1)
    assert e.value.status == rid.RID_ERANK
