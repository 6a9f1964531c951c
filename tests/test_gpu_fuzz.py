"""Randomised parity of the whole CUDA path against the oracle (seeded, reproducible): random
(m, n, k, l, noise) pick every sketch tile height (24 / 40 / 48 rows), ragged K and column tails,
split-K, the small and the blocked QR and both R11^-1 kernels. Bars as everywhere: generated A
bitwise, Y <= 1e-12 relative (reading R31), J equal (R18), P <= 1e-10 (R17).
tools/fuzz_parity.py runs the same sweep at larger counts, also for the SRFT and the CGS2 QR (at
the round's end on B200: 150/150 Gaussian + Householder, 60/60 SRFT + Householder, 60/60 SRFT +
CGS2 — the paper's own algorithm — and 60/60 Gaussian + CGS2)."""
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


def _shapes(count, seed):
    rng = np.random.default_rng(seed)
    out = []
    for _ in range(count):
        m = int(rng.integers(16, 2500))
        n = int(rng.integers(1, 1200))
        k = int(rng.integers(1, min(m, n, 200) + 1))
        l = int(min(m, k + rng.integers(0, 40)))
        out.append((int(rng.integers(1, 1 << 30)), m, n, k, l,
                    float(rng.choice([0.0, 1e-12, 1e-9, 1e-6]))))
    return out


@pytest.mark.parametrize("seed,m,n,k,l,noise", _shapes(12, 2026))
def test_random_shape_parity(rid, orc, seed, m, n, k, l, noise):
    A = rid.generate(seed, m, n, k, noise)
    A_o = orc.generate(seed, m, n, k, noise)
    assert np.array_equal(np.ascontiguousarray(A.cpu().numpy()).view(np.uint64),
                          np.ascontiguousarray(A_o).view(np.uint64))
    Y = rid.sketch(A, seed, l).cpu().numpy()
    Y_o = orc.sketch(A_o, seed, l)
    assert np.linalg.norm(Y - Y_o) <= 1e-12 * np.linalg.norm(Y_o)
    r = rid.decompose(A, k, l, seed)
    d = orc.decompose(A_o, k, l, seed)
    assert r.J.cpu().numpy().tolist() == list(d.J)
    P = r.P.cpu().numpy()
    assert np.linalg.norm(P - d.P) <= 1e-10 * np.linalg.norm(d.P)


@pytest.mark.parametrize("seed,m,n,k,l,noise", _shapes(12, 2027))
def test_random_shape_parity_int8_crt(rid, orc, seed, m, n, k, l, noise):
    """The same sweep on the INT8_CRT sketch engine (tcgen05 int8 GEMMs + CRT, reading R33)."""
    ctx = rid.Context(0, torch.cuda.current_stream())
    ctx.set_sketch_engine("int8_crt")
    A = rid.generate(seed, m, n, k, noise, ctx=ctx)
    A_o = orc.generate(seed, m, n, k, noise)
    Y = rid.sketch(A, seed, l, ctx=ctx).cpu().numpy()
    Y_o = orc.sketch(A_o, seed, l)
    assert np.linalg.norm(Y - Y_o) <= 1e-12 * np.linalg.norm(Y_o)
    d = orc.decompose(A_o, k, l, seed)
    margin = d.tie_margins[:-1].min() if k > 1 else np.inf
    if margin > 1e-10:  # J is only defined on well-separated spectra (reading R18)
        r = rid.decompose(A, k, l, seed, ctx=ctx)
        assert r.J.cpu().numpy().tolist() == list(d.J)
        P = r.P.cpu().numpy()
        assert np.linalg.norm(P - d.P) <= 1e-10 * np.linalg.norm(d.P)
    ctx.close()


def _srft_shapes(count, seed):
    rng = np.random.default_rng(seed)
    out = []
    for _ in range(count):
        m = int(2 ** rng.integers(5, 12))
        n = int(rng.integers(1, 1000))
        k = int(rng.integers(1, min(m, n, 150) + 1))
        l = int(min(m, k + rng.integers(0, 40)))
        out.append((int(rng.integers(1, 1 << 30)), m, n, k, l,
                    float(rng.choice([0.0, 1e-12, 1e-9]))))
    return out


@pytest.mark.parametrize("seed,m,n,k,l,noise", _srft_shapes(6, 77))
def test_random_shape_parity_srft_cgs2(rid, orc, seed, m, n, k, l, noise):
    """The paper's own algorithm end to end (SRFT randomisation, Gram-Schmidt QR) on random
    shapes against the oracle's SRFT + CGS2."""
    A = rid.generate(seed, m, n, k, noise)
    A_o = orc.generate(seed, m, n, k, noise)
    Y = rid.sketch_srft(A, seed, l).cpu().numpy()
    Y_o = orc.srft_sketch(A_o, seed, l)
    assert np.linalg.norm(Y - Y_o) <= 1e-12 * np.linalg.norm(Y_o)
    # sampling rows with replacement can leave l <= m sampled rows rank-deficient
    # (duplicates): then both sides must report the rank failure after the one retry
    try:
        d = orc.decompose(A_o, k, l, seed, sketch_kind="srft")
    except orc.OracleError as e:
        assert e.status == orc.RID_ERANK
        with pytest.raises(rid.RidError, match="RANK"):
            rid.decompose(A, k, l, seed, sketch="srft", qr="cgs2")
        return
    r = rid.decompose(A, k, l, seed, sketch="srft", qr="cgs2")
    assert r.J.cpu().numpy().tolist() == list(d.J)
    P = r.P.cpu().numpy()
    assert np.linalg.norm(P - d.P) <= 1e-10 * np.linalg.norm(d.P)

