"""GPU parity of NEXT-1, the paper's SRFT randomisation Y = S F D A (Eqs. 4–7),
against the oracle's direct ascending sums (oracle.srft_sketch, pinned in test_oracle_srft.py):
Y within 1e-12 relative Frobenius (the north-star bar for sketches), the whole ID with the SRFT:
J identical and P within 1e-10; bad m rejected."""
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


@pytest.mark.parametrize("seed,m,n,k,noise,l", [
    (1, 16, 5, 2, 0.0, 4), (2, 64, 33, 4, 1e-9, 9), (3, 1024, 200, 16, 0.0, 24),
    (4, 4096, 130, 64, 1e-10, 80), (5, 2048, 300, 128, 1e-12, 144), (6, 8192, 64, 32, 1e-8, 600)])
def test_srft_sketch_parity(rid, orc, seed, m, n, k, noise, l):
    A = rid.generate(seed, m, n, k, noise)
    Y = np_(rid.sketch_srft(A, seed, l))
    Y_o = orc.srft_sketch(orc.generate(seed, m, n, k, noise), seed, l)
    assert relf(Y, Y_o) <= 1e-12
    Yr = np_(rid.sketch_srft(A, seed, l, retry=True))
    assert relf(Yr, orc.srft_sketch(orc.generate(seed, m, n, k, noise), seed, l, retry=True)) <= 1e-12


@pytest.mark.parametrize("name,seed,m,n,k,l,noise", [
    ("C1-srft", 1, 1024, 512, 16, 24, 0.0), ("C2s-srft", 1, 2048, 2048, 64, 80, 1e-10),
    # the paper's l = 2k: with row sampling WITH replacement, l = k + 16 out of only
    # m = 2048 rows loses ~18 rows to duplicates and the sketch is rank-deficient
    ("C4s-srft", 1, 2048, 1024, 256, 512, 1e-8)])
def test_srft_decompose_parity(rid, orc, name, seed, m, n, k, l, noise):
    A_o = orc.generate(seed, m, n, k, noise)
    d = orc.decompose(A_o, k, l, seed, sketch_kind="srft")
    A = rid.generate(seed, m, n, k, noise)
    r = rid.decompose(A, k, l, seed, sketch="srft")
    margin = d.tie_margins[:-1].min()
    assert margin > 1e-10, f"{name}: tie-ambiguous (margin {margin:.2e})"
    J, P = np_(r.J), np_(r.P)
    assert J.tolist() == d.J.tolist()
    assert relf(P, d.P) <= 1e-10
    assert np.array_equal(P[:, J], np.eye(k, dtype=complex))
    # the Gaussian path is still the default on the same context
    r2 = rid.decompose(A, k, l, seed)
    assert r2.J.cpu().numpy().tolist() == orc.decompose(A_o, k, l, seed).J.tolist()


def test_srft_rejects_bad_m(rid):
    A = rid.generate(1, 100, 20, 3, 0.0)
    with pytest.raises(rid.RidError):
        rid.sketch_srft(A, 1, 8)
    with pytest.raises(rid.RidError):
        rid.decompose(A, 3, 8, 1, sketch="srft")
