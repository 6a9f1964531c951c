"""The TMA-fed three-product sketch kernel (k_zgemm3m_tma.cu) against the cp.async kernel it
replaces (k_zgemm3m.cu) and against the oracle, through the C ABI.

Both kernels evaluate the same ascending fma chains per K slice (reading R31), only the
operand staging differs (TMA boxes with a 128-byte swizzle and mbarrier hand-over vs cp.async and
__syncthreads), so Y must be BITWISE equal (RID_Z3_TMA=0 selects the old kernel). The shapes put
each tile height (48, 40 and 24 rows) under every edge the TMA unit handles by
zero-filling: rows past l (l = 47, 143), K past m (m not a multiple of 16), columns past n, K
slices (split-K) and the wave-tail split; against the oracle Y holds the north-star bar (1e-12
relative Frobenius; measured 1e-15 .. 1e-14).
"""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")


def bits(a):
    return np.ascontiguousarray(a).view(np.uint64)


@pytest.fixture(scope="module")
def rid():
    if not torch.cuda.is_available():
        pytest.skip("no GPU")
    from paper_1205_3830_b200 import build

    build.build()
    import paper_1205_3830_b200 as rid

    return rid


SHAPES = [  # (seed, m, n, k, l, noise)
    (1, 2048, 2048, 512, 528, 1e-8),     # C4's k/l, reduced
    (2, 4096, 1024, 128, 144, 1e-12),    # C3's k/l, reduced
    (3, 1000, 777, 13, 47, 1e-8),        # ragged rows, K tail, ragged columns
    (4, 4099, 300, 100, 143, 0.0),       # ragged everything, exact rank
    (5, 65536, 64, 32, 144, 1e-12),      # narrow: K split into slices
    (6, 64, 5, 3, 48, 0.0),              # four stages, one tile
    (9, 2048, 1000, 64, 80, 1e-10),      # C2's k/l: the 40-row tile with the Re R + Im R plane
    (10, 4096, 600, 256, 272, 1e-10),    # C5's k/l: 40-row tiles, rows past l in the last one
    (11, 1003, 333, 20, 39, 1e-9),       # 40-row tile, ragged everything
    (12, 1024, 512, 16, 24, 0.0),        # C1: the 24-row tile
    (13, 777, 100, 5, 21, 1e-9),         # 24-row tile, ragged
]


@pytest.mark.parametrize("seed,m,n,k,l,noise", SHAPES)
def test_tma_sketch_bitwise_vs_cpasync_and_oracle(rid, orc, monkeypatch, seed, m, n, k, l, noise):
    monkeypatch.setenv("RID_SKETCH_STRASSEN", "0")  # the plain 3M kernels on both sides
    A = rid.generate(seed, m, n, k, noise)
    monkeypatch.setenv("RID_Z3_TMA", "0")
    Y_old = rid.sketch(A, seed, l).cpu().numpy()
    monkeypatch.setenv("RID_Z3_TMA", "1")
    Y_tma = rid.sketch(A, seed, l).cpu().numpy()
    torch.cuda.synchronize()
    assert np.array_equal(bits(Y_tma), bits(Y_old))
    if m * n * l <= 2048 * 2048 * 528:
        Y_o = orc.sketch(orc.generate(seed, m, n, k, noise), seed, l)
        rel = np.linalg.norm(Y_tma - Y_o) / np.linalg.norm(Y_o)
        assert rel <= 1e-12, rel


@pytest.mark.parametrize("variant,l", [("2", 96), ("4", 96), ("2", 80)])
def test_tma_pipeline_depths_bitwise(rid, monkeypatch, variant, l):
    """Two and four stages (RID_Z3T_VARIANT) give the same bits as the default three."""
    A = rid.generate(7, 3000, 700, 40, 1e-9)
    Y3 = rid.sketch(A, 7, l).cpu().numpy()
    monkeypatch.setenv("RID_Z3T_VARIANT", variant)
    Yv = rid.sketch(A, 7, l).cpu().numpy()
    assert np.array_equal(bits(Yv), bits(Y3))


def test_tma_wave_tail_and_shards_bitwise(rid, monkeypatch):
    """Column blocks of a matrix sketched as shards (different tensor maps, base pointers and the
    wave-tail split set) equal the whole-matrix sketch bit for bit, and equal the old kernel."""
    seed, m, n, k, l = 8, 2048, 4096, 64, 96
    monkeypatch.setenv("RID_SKETCH_STRASSEN", "0")  # the plain 3M kernels (this shape's default
    A = rid.generate(seed, m, n, k, 1e-10)            # plan is Strassen's, tests/test_gpu_strassen)
    Y = rid.sketch(A, seed, l).cpu().numpy()
    for G in (2, 8):
        w = n // G
        for g in range(G):
            Yg = rid.sketch(A[:, g * w:(g + 1) * w], seed, l, n=n, col0=g * w).cpu().numpy()
            assert np.array_equal(bits(Yg), bits(Y[:, g * w:(g + 1) * w]))
    monkeypatch.setenv("RID_Z3_TMA", "0")
    Y_old = rid.sketch(A, seed, l).cpu().numpy()
    assert np.array_equal(bits(Y), bits(Y_old))


@pytest.mark.parametrize("seed,m,n,l", [(1, 4096, 700, 80), (2, 2048, 333, 528), (3, 1024, 64, 47)])
def test_srft_residue_products_tma_bitwise(rid, monkeypatch, seed, m, n, l):
    """The SRFT's batched residue products on the TMA kernel equal the cp.async
    kernel's bit for bit (rows / columns a tile reads past its residue are discarded)."""
    A = rid.generate(seed, m, n, 8, 1e-9)
    Y_t = rid.sketch_srft(A, seed, l).cpu().numpy()
    monkeypatch.setenv("RID_Z3_TMA", "0")
    Y_o = rid.sketch_srft(A, seed, l).cpu().numpy()
    assert np.array_equal(bits(Y_t), bits(Y_o))


@pytest.mark.parametrize("seed,m,n,k,noise", [(1, 2048, 300, 64, 1e-10), (2, 4099, 77, 13, 1e-8),
                                               (3, 2500, 1000, 512, 0.0), (4, 8192, 64, 1, 1e-6)])
def test_generation_tma_bitwise(rid, orc, monkeypatch, seed, m, n, k, noise):
    """The TMA-fed ordered GEMM (k_zgemm_tma.cu, RID_ZGEMM_TMA=1) generates A = X·Y0 + ε·E bit for
    bit like the cp.async kernel (the default) and the oracle's ascending fma chains (RNG.md §5)."""
    monkeypatch.setenv("RID_ZGEMM_TMA", "1")
    A_t = rid.generate(seed, m, n, k, noise).cpu().numpy()
    monkeypatch.setenv("RID_ZGEMM_TMA", "0")
    A_c = rid.generate(seed, m, n, k, noise).cpu().numpy()
    assert np.array_equal(bits(A_t), bits(A_c))
    if m * n <= 2048 * 300:
        assert np.array_equal(bits(A_t), bits(orc.generate(seed, m, n, k, noise)))


def test_qr_update_tma_bitwise(rid, monkeypatch):
    """The QR's panel update on the TMA kernel (RID_ZGEMM_TMA_UPDATE=1) leaves J and P bitwise
    unchanged (a C4-shaped sketch, reduced: the blocked QR path)."""
    monkeypatch.setenv("RID_QRCP_VARIANT", "1")
    A = rid.generate(5, 2048, 3000, 256, 1e-9)
    r0 = rid.decompose(A, 256, 272, 5)
    monkeypatch.setenv("RID_ZGEMM_TMA", "1")
    monkeypatch.setenv("RID_ZGEMM_TMA_UPDATE", "1")
    r1 = rid.decompose(A, 256, 272, 5)
    assert torch.equal(r0.J, r1.J)
    assert np.array_equal(bits(r0.P.cpu().numpy()), bits(r1.P.cpu().numpy()))


def test_tma_rings_repeatable(rid, monkeypatch):
    """Run-to-run bitwise repeatability of the TMA rings (a slot refilled under a lagging warp's
    reads would show as a changed block in some run): sketch and, opt-in, the ordered GEMM."""
    A = rid.generate(3, 2500, 1000, 64, 1e-9)
    Y0 = bits(rid.sketch(A, 3, 528).cpu().numpy())
    for _ in range(8):
        assert np.array_equal(bits(rid.sketch(A, 3, 528).cpu().numpy()), Y0)
    monkeypatch.setenv("RID_ZGEMM_TMA", "1")
    G0 = bits(rid.generate(3, 2500, 1000, 512, 0.0).cpu().numpy())
    for _ in range(8):
        assert np.array_equal(bits(rid.generate(3, 2500, 1000, 512, 0.0).cpu().numpy()), G0)


@pytest.mark.parametrize("seed,m,n,l", [(1, 4096, 2048, 272), (2, 2048, 3000, 80), (3, 1500, 700, 88),
                                        (4, 1024, 333, 72), (5, 65536, 128, 272)])
def test_row_split_sketch_bitwise(rid, monkeypatch, seed, m, n, l):
    """l = 48 a + r with r in {24, 32, 40} runs as 48-row tiles plus r-row tiles (sketch_gemm's
    row split); every element is the same chain: Y equals the single-height plan bit for bit,
    with and without split-K, and the decomposition is unchanged."""
    monkeypatch.setenv("RID_SKETCH_STRASSEN", "0")  # the 3M row split (not Strassen's plan)
    A = rid.generate(seed, m, n, 16, 1e-9)
    Y_s = rid.sketch(A, seed, l).cpu().numpy()
    monkeypatch.setenv("RID_SKETCH_NOROWSPLIT", "1")
    Y_1 = rid.sketch(A, seed, l).cpu().numpy()
    assert np.array_equal(bits(Y_s), bits(Y_1))


@pytest.mark.parametrize("seed,m,n,k,l", [(6, 3000, 2500, 80, 96), (7, 2048, 4000, 128, 144),
                                          (8, 1200, 1500, 72, 88)])
def test_row_split_solve_bitwise(rid, monkeypatch, seed, m, n, k, l):
    """T = R11^-1 R12 with k = 48 a + r (r in {24, 32, 40}) runs its last r rows on r-row tiles
    beside the 48-row launch (solve_T through sketch_gemm on the aux stream): J and P equal the
    single-launch solve bit for bit."""
    A = rid.generate(seed, m, n, k, 1e-10)
    r_s = rid.decompose(A, k, l, seed)
    J_s, P_s = r_s.J.cpu().numpy(), r_s.P.cpu().numpy()
    monkeypatch.setenv("RID_SOLVE_NOAUX", "1")
    r_1 = rid.decompose(A, k, l, seed)
    assert np.array_equal(r_1.J.cpu().numpy(), J_s)
    assert np.array_equal(bits(r_1.P.cpu().numpy()), bits(P_s))
