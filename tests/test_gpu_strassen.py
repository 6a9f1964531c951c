"""The Strassen sketch (k_strassen.cu; reading R32): one level of Strassen's algorithm
over Gauss's three real products, the default plan for the unsplit shapes (C4, C5).

Bars: Y within 1e-13 relative per column of the oracle's ascending sums (north star 1e-12; the
reading derives 1e-13 from one Strassen level's error growth over the 3M kernel's ~1e-14, and
C4/C5 measure 1.6e-14 / 3.3e-14); every 64-aligned column sharding bitwise equal to the whole;
J equal to the oracle's and P within 1e-10 (R17, R18) — also with G ranks, replicated and sharded.
Shape: m = 1024, n = 13824, l = 528 (C4's l; enough column tiles that the 3M plan is unsplit).
"""
import threading

import numpy as np
import pytest

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")

SEED, M, N, L = 4, 1024, 13824, 528


@pytest.fixture(scope="module")
def rid():
    if not torch.cuda.is_available():
        pytest.skip("no GPU")
    from paper_1205_3830_b200 import build

    build.build()
    import paper_1205_3830_b200 as rid

    return rid


def bits(a):
    return np.ascontiguousarray(np.asarray(a)).view(np.uint64)


def test_plan(rid):
    assert rid.sketch_strassen(M, L, N)
    # C3-C5 run the INT8_CRT engine by default (rid_sketch_engine); on the DMMA engine they
    # take the Strassen plan
    assert not rid.sketch_strassen(32768, 528, 32768)
    dm = rid.Context(0, torch.cuda.current_stream())
    dm.set_sketch_engine("fp64_dmma")
    assert rid.sketch_strassen(32768, 528, 32768, ctx=dm)
    assert rid.sketch_strassen(131072, 272, 32768, ctx=dm)
    assert rid.sketch_strassen(8192, 80, 8192) and rid.sketch_strassen(65536, 144, 4096, ctx=dm)
    dm.close()
    assert not rid.sketch_strassen(1024, 24, 512)  # C1: l < 64
    assert not rid.sketch_strassen(M, L, N - 64)  # n not a multiple of 512
    assert not rid.sketch_strassen(M, 90, N)  # l not a multiple of 4


def test_sketch_vs_oracle_and_3m(rid, orc, monkeypatch):
    A = rid.generate(SEED, M, N, 64, 1e-9)
    Y = rid.sketch(A, SEED, L).cpu().numpy()
    monkeypatch.setenv("RID_SKETCH_STRASSEN", "0")
    Y3 = rid.sketch(A, SEED, L).cpu().numpy()
    monkeypatch.delenv("RID_SKETCH_STRASSEN")
    assert not np.array_equal(bits(Y), bits(Y3))  # the Strassen plan ran
    assert np.linalg.norm(Y - Y3) <= 1e-13 * np.linalg.norm(Y3)
    # columns of both halves of a 64-group, group edges, the last column
    for j in (0, 1, 31, 32, 33, 63, 64, 95, 96, 6900, N - 33, N - 32, N - 1):
        a = orc.generate(SEED, M, N, 64, 1e-9, j, 1)
        y = orc.sketch(a, SEED, L)[:, 0]
        assert np.linalg.norm(Y[:, j] - y) <= 1e-13 * np.linalg.norm(y), j


def test_shards_bitwise(rid):
    A = rid.generate(SEED, M, N, 64, 1e-9)
    Y = rid.sketch(A, SEED, L).cpu().numpy()
    for G in (2, 4, 8):  # n / G = 6912, 3456, 1728: multiples of 64
        w = N // G
        for g in range(G):
            Yg = rid.sketch(A[:, g * w:(g + 1) * w], SEED, L, n=N, col0=g * w).cpu().numpy()
            assert np.array_equal(bits(Yg), bits(Y[:, g * w:(g + 1) * w])), (G, g)
    with pytest.raises(rid.RidError) as e:  # a block that splits a 64-column group
        rid.sketch(A[:, 32:32 + 1024], SEED, L, n=N, col0=32)
    assert e.value.status == rid.RID_EINVAL


def _run_ranks(G, fn):
    out, errs = [None] * G, [None] * G

    def body(g):
        try:
            out[g] = fn(g)
        except BaseException as ex:  # noqa: BLE001
            errs[g] = ex

    th = [threading.Thread(target=body, args=(g,)) for g in range(G)]
    for t in th:
        t.start()
    for t in th:
        t.join(timeout=900)
    for ex in errs:
        if ex is not None:
            raise ex
    torch.cuda.synchronize()
    return out


def test_decompose_vs_oracle_and_ranks(rid, orc):
    k = 96
    A_o = orc.generate(SEED, M, N, k, 1e-9)
    d = orc.decompose(A_o, k, L, SEED)
    assert d.tie_margins[:-1].min() > 1e-10
    A = rid.generate(SEED, M, N, k, 1e-9)
    r = rid.decompose(A, k, L, SEED)
    assert r.J.cpu().numpy().tolist() == d.J.tolist()
    P = r.P.cpu().numpy()
    assert np.linalg.norm(P - d.P) <= 1e-10 * np.linalg.norm(d.P)
    for dist in ("replicated", "sharded"):
        G = 4
        streams = [torch.cuda.Stream() for _ in range(G)]
        ctxs = [rid.Context(0, s) for s in streams]
        rid.comm_init_local(ctxs)
        for c in ctxs:
            c.set_qr_dist(dist)
        w = N // G
        P_out = [rid.colmajor_empty(k, w) for _ in range(G)]
        J_out = [torch.empty(k, dtype=torch.int64, device="cuda") for _ in range(G)]
        torch.cuda.synchronize()

        def dec(g):
            return rid.decompose(A[:, g * w:(g + 1) * w], k, L, SEED, n=N, col0=g * w,
                                 J=J_out[g], P=P_out[g], ctx=ctxs[g])

        _run_ranks(G, dec)
        for g in range(G):
            assert J_out[g].cpu().numpy().tolist() == d.J.tolist(), (dist, g)
        Pc = np.concatenate([p.cpu().numpy() for p in P_out], axis=1)
        # the one-rank call runs the blocked QR here (16 l n >= 64 MB), as the sharded QR does,
        # and n / G = 3456 is a multiple of 32 (the batch alignment): the same bits either way
        assert np.array_equal(bits(Pc), bits(P)), dist
        assert np.linalg.norm(Pc - d.P) <= 1e-10 * np.linalg.norm(d.P)
        for c in ctxs:
            c.close()
