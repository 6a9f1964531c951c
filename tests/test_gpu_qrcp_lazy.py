"""The lazy-refresh pivoted QR (k_qrcp_lazy; the blocked default for l > 384 (C4), forced here).

A residual norm never grows, so a column whose last computed norm is below the step's threshold
is not re-read; the threshold is exact-checked after every pass. Held here:
- RID_QRCP_LAZY=1 (lazy) and RID_QRCP_LAZY=2 (every column refreshed at every step, the same
  kernel) give the SAME BITS: J, R, the residual norms and the tie margins. This is the property
  that makes the laziness invisible: a column's arithmetic does not depend on when it is refreshed;
- both agree with the ring kernel (RID_QRCP_LAZY=0, which streams every column every step): J
  equal, R to rounding;
- inputs that defeat the threshold (near-duplicate columns whose norm collapses when the twin is
  chosen, exact ties, geometric column scales) still give the exact greedy pivots;
- the lazy pass reads far fewer columns than the full one (RID_QRCP_TRACE refresh counts).
The oracle comparisons of the blocked path (tests/test_gpu_qrcp_variants.py, test_gpu_fullsize.py)
run on this kernel by default.
"""
import os

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


def bits(t):
    return np.ascontiguousarray(t.cpu().numpy()).view(np.uint64)


def lowrank_Y(seed, l, n, k, noise):
    """l x n sketch-like matrix: rank-k Gaussian product plus noise (the configs' structure)."""
    g = torch.Generator().manual_seed(seed)

    def cn(r, c):
        return torch.complex(torch.randn(r, c, generator=g, dtype=torch.float64),
                             torch.randn(r, c, generator=g, dtype=torch.float64)) / np.sqrt(2)

    Y = cn(l, k) @ cn(k, n) + noise * cn(l, n)
    return Y.T.contiguous().T.cuda()  # column-major


def twins_Y(seed, l, n):
    """Columns in near-duplicate pairs: choosing one collapses its twin's residual norm (a sharp
    drop of the top candidates that the threshold rule must catch by a second pass)."""
    g = torch.Generator().manual_seed(seed)
    h = n // 2
    B = torch.complex(torch.randn(l, h, generator=g, dtype=torch.float64),
                      torch.randn(l, h, generator=g, dtype=torch.float64))
    s = 1.0 - 1e-3 * torch.arange(h, dtype=torch.float64) / h
    E = 1e-6 * torch.complex(torch.randn(l, h, generator=g, dtype=torch.float64),
                             torch.randn(l, h, generator=g, dtype=torch.float64))
    Y = torch.cat([B, B * s + E], dim=1)
    return Y.T.contiguous().T.cuda()


def geometric_Y(seed, l, n):
    """Column scales 2^(-j/64): well separated pivots, many columns far below the top."""
    g = torch.Generator().manual_seed(seed)
    Y = torch.complex(torch.randn(l, n, generator=g, dtype=torch.float64),
                      torch.randn(l, n, generator=g, dtype=torch.float64))
    perm = torch.randperm(n, generator=g)
    Y = Y * (2.0 ** (-perm.to(torch.float64) / 64.0))
    return Y.T.contiguous().T.cuda()


def run(rid, monkeypatch, Y, k, lazy, nb=None):
    monkeypatch.setenv("RID_QRCP_VARIANT", "1")
    monkeypatch.setenv("RID_QRCP_LAZY", lazy)
    if nb is not None:
        monkeypatch.setenv("RID_QRCP_NB", nb)
    return rid.qrcp(Y.clone(), k)


CASES = [  # (name, builder, k)
    ("C4-like l=528", lambda: lowrank_Y(1, 528, 3000, 512, 1e-8), 512),
    ("C5-like l=272", lambda: lowrank_Y(2, 272, 4100, 256, 1e-10), 256),
    ("ragged l=97", lambda: lowrank_Y(3, 97, 1001, 81, 1e-9), 81),
    ("twins", lambda: twins_Y(4, 144, 2000), 128),
    ("geometric", lambda: geometric_Y(5, 200, 3000), 180),
    ("n < CTAs", lambda: lowrank_Y(6, 64, 100, 48, 1e-9), 48),
    # > 64 columns per CTA: the thread-per-column phase B of the full passes, and its handover
    # of the columns whose downdate needs the exact recompute (the twins) to the half-warp form
    ("twins wide", lambda: twins_Y(9, 144, 12000), 128),
    ("wide l=528", lambda: lowrank_Y(10, 528, 12000, 512, 1e-8), 512),
]


@pytest.mark.parametrize("name,builder,k", CASES)
def test_lazy_bitwise_equals_full_refresh(rid, monkeypatch, name, builder, k):
    Y = builder()
    J1, R1, res1, mar1, d1 = run(rid, monkeypatch, Y, k, "1")
    J2, R2, res2, mar2, d2 = run(rid, monkeypatch, Y, k, "2")
    assert torch.equal(J1, J2), name
    assert np.array_equal(bits(R1), bits(R2)), name
    assert np.array_equal(bits(res1), bits(res2)), name
    assert np.array_equal(bits(mar1), bits(mar2)), name
    # the ring kernel (every column streamed every step): same pivots, R to rounding
    J0, R0, res0, mar0, d0 = run(rid, monkeypatch, Y, k, "0")
    assert torch.equal(J0, J1), name
    assert float(torch.linalg.norm(R1 - R0) / torch.linalg.norm(R0)) <= 1e-12, name
    assert float((res1 - res0).abs().max() / res0.abs().max()) <= 1e-12, name


@pytest.mark.parametrize("nb", ["1", "5", "16"])
def test_lazy_panel_width(rid, monkeypatch, nb):
    """Any panel width: the same bits as the full refresh at that width, the ring kernel's J."""
    Y = lowrank_Y(7, 300, 2500, 280, 1e-9)
    J1, R1, _, _, _ = run(rid, monkeypatch, Y, 280, "1", nb)
    J2, R2, _, _, _ = run(rid, monkeypatch, Y, 280, "2", nb)
    J0, R0, _, _, _ = run(rid, monkeypatch, Y, 280, "0", nb)
    assert torch.equal(J1, J2) and np.array_equal(bits(R1), bits(R2))
    assert torch.equal(J1, J0)
    assert float(torch.linalg.norm(R1 - R0) / torch.linalg.norm(R0)) <= 1e-12


def test_lazy_exact_ties(rid, monkeypatch):
    """Columns in exactly equal pairs (bitwise identical columns): the greedy rule's ties go to the
    lowest index; the lazy pass must see them exactly like the full pass."""
    g = torch.Generator().manual_seed(8)
    B = torch.complex(torch.randn(64, 300, generator=g, dtype=torch.float64),
                      torch.randn(64, 300, generator=g, dtype=torch.float64))
    Y = torch.cat([B, B], dim=1).T.contiguous().T.cuda()
    J1, R1, _, mar1, _ = run(rid, monkeypatch, Y, 40, "1")
    J2, R2, _, mar2, _ = run(rid, monkeypatch, Y, 40, "2")
    assert torch.equal(J1, J2) and np.array_equal(bits(R1), bits(R2))
    assert np.array_equal(bits(mar1), bits(mar2))
    assert float(mar1[0]) == 0.0 and int(J1[0]) < 300  # the first pivot is a tie, lowest index


def test_lazy_reads_fewer_columns(rid, monkeypatch, tmp_path):
    """The point of the kernel: on the configs' structure most steps refresh a small fraction of
    the columns (RID_QRCP_TRACE column 7: columns refreshed per step, all CTAs)."""
    Y = lowrank_Y(1, 528, 6000, 512, 1e-8)
    path = str(tmp_path / "trace.txt")
    monkeypatch.setenv("RID_QRCP_TRACE", path)
    run(rid, monkeypatch, Y, 512, "1")
    t = np.loadtxt(path, dtype=np.float64)
    refreshed = t[:, 7]
    assert refreshed.sum() > 0
    # full refresh would be sum_j (n - j) column reads
    full = sum(6000 - j for j in range(512))
    assert refreshed.sum() < 0.25 * full, (refreshed.sum(), full)


def _fuzz_cases(count=16, seed=2026):
    rng = np.random.default_rng(seed)
    out = []
    for i in range(count):
        l = int(rng.integers(1, 545))
        n = int(rng.integers(1, 3000))
        k = int(rng.integers(1, min(l, n) + 1))
        kind = ["lowrank", "lowrank", "twins", "geometric"][i % 4]
        out.append((i, kind, l, n, k, int(rng.integers(1, 1 << 30))))
    return out


@pytest.mark.parametrize("i,kind,l,n,k,seed", _fuzz_cases())
def test_lazy_fuzz(rid, monkeypatch, i, kind, l, n, k, seed):
    """Random shapes (l up to the kernel's 544, any n and k) and structures: the lazy kernel is
    bitwise the full refresh and picks the ring kernel's pivots."""
    if kind == "twins" and n >= 2:
        Y = twins_Y(seed, l, n - n % 2)
        n = Y.shape[1]
    elif kind == "geometric":
        Y = geometric_Y(seed, l, n)
    else:
        Y = lowrank_Y(seed, l, n, max(1, min(l, n) - 3), 1e-9)
    k = min(k, l, n)
    try:
        J1, R1, res1, mar1, _ = run(rid, monkeypatch, Y, k, "1")
    except rid.RidError as e:  # rank failure must then be reported by the full refresh too
        with pytest.raises(rid.RidError) as e2:
            run(rid, monkeypatch, Y, k, "2")
        assert e2.value.status == e.status
        return
    J2, R2, res2, mar2, _ = run(rid, monkeypatch, Y, k, "2")
    assert torch.equal(J1, J2) and np.array_equal(bits(R1), bits(R2))
    assert np.array_equal(bits(res1), bits(res2)) and np.array_equal(bits(mar1), bits(mar2))
    J0, R0, _, mar0, _ = run(rid, monkeypatch, Y, k, "0")
    if float(mar0[:-1].min()) > 1e-9 if k > 1 else True:  # the ring downdates differently
        assert torch.equal(J0, J1)


def test_lazy_falls_back_to_ring_when_state_exceeds_shared_memory(rid, monkeypatch):
    """Per-column state (24 B per column of a CTA) beside the 140 KB reflector panel: beyond
    ≈ 700 columns per CTA the lazy kernel does not fit and the ring kernel runs instead — the
    same bits as forcing the ring kernel."""
    g = torch.Generator().manual_seed(11)
    l, n, k = 400, 120000, 40
    Y = torch.complex(torch.randn(l, n, generator=g, dtype=torch.float64),
                      torch.randn(l, n, generator=g, dtype=torch.float64)).T.contiguous().T.cuda()
    J1, R1, _, _, _ = run(rid, monkeypatch, Y, k, "1")
    J0, R0, _, _, _ = run(rid, monkeypatch, Y, k, "0")
    assert torch.equal(J1, J0) and np.array_equal(bits(R1), bits(R0))
