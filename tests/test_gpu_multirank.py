"""The G > 1 data path of librid, run on ONE GPU as G ranks of one process.

SURVEY.md §8(e) / rows a3 and a6: A is column-sharded, each rank sketches its shard, the sketch
blocks are all-gathered (a3), the QR runs replicated, each rank solves its own block of P; the
estimator replicates B = A[:, J] by an all-reduce and merges the compensated partials of every
iteration by all-gathers. Here the G ranks are G librid contexts joined by rid_comm_init_local
(include/rid.h): the same rid_decompose / rid_error_estimate code, with the communicator's two
collectives implemented as event-ordered device copies instead of NCCL calls, and every rank's
calls made concurrently from its own thread — exactly as G processes would call with NCCL.

Bars (BASELINE.json:north_star; R16–R18): J equal to the oracle's, P within 1e-10 of the
oracle's and BITWISE equal to the one-rank call (the sketch plan and every per-column chain are
independent of the sharding), the estimate on the same (A, J, P) within 1e-10 of the
oracle's. Shapes are the reduced configs of tests/test_gpu_parity.py (PAPER.md:112 workloads).
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


def np_(t):
    return t.cpu().numpy() if hasattr(t, "cpu") else np.asarray(t)


def bits_equal(a, b):
    a, b = np.asarray(a), np.asarray(b)
    return a.shape == b.shape and np.array_equal(np.ascontiguousarray(a).view(np.uint64),
                                                 np.ascontiguousarray(b).view(np.uint64))


def relf(a, b):
    return np.linalg.norm(a - b) / np.linalg.norm(b)


def make_ranks(rid, G):
    streams = [torch.cuda.Stream() for _ in range(G)]
    ctxs = [rid.Context(0, s) for s in streams]
    rid.comm_init_local(ctxs)
    for g, c in enumerate(ctxs):
        assert c.comm_info() == (g, G)
    return ctxs, streams


def run_ranks(G, fn):
    """fn(rank) on G threads at once (each rank's collective calls rendezvous with the others)."""
    out, errs = [None] * G, [None] * G

    def body(g):
        try:
            out[g] = fn(g)
        except BaseException as e:  # noqa: BLE001 - reported below
            errs[g] = e

    th = [threading.Thread(target=body, args=(g,)) for g in range(G)]
    for t in th:
        t.start()
    for t in th:
        t.join(timeout=900)
    for e in errs:
        if e is not None:
            raise e
    torch.cuda.synchronize()
    return out


CASES = [  # (name, seed, m, n, k, l, noise): tests/test_gpu_parity.py DEC_CASES
    ("C2s", 1, 2048, 2048, 64, 80, 1e-10),
    ("C3s", 1, 8192, 1024, 128, 144, 1e-12),
    ("C5s", 1, 8192, 2048, 256, 272, 1e-10),
]

_oracle_cache = {}


def oracle_case(orc, seed, m, n, k, l, noise, q):
    key = (seed, m, n, k, l, noise, q)
    if key not in _oracle_cache:
        A = orc.generate(seed, m, n, k, noise)
        d = orc.decompose(A, k, l, seed)
        e = orc.error_estimate(A, d.J, d.P, q, seed)
        _oracle_cache[key] = (d, e)
    return _oracle_cache[key]


@pytest.mark.parametrize("name,seed,m,n,k,l,noise", CASES)
def test_multirank_decompose_and_estimate(rid, orc, name, seed, m, n, k, l, noise):
    q = 6
    d, e_o = oracle_case(orc, seed, m, n, k, l, noise, q)
    A = rid.generate(seed, m, n, k, noise)
    ref = rid.decompose(A, k, l, seed)
    assert np_(ref.J).tolist() == d.J.tolist()
    Jo = torch.from_numpy(d.J.copy()).cuda()
    Po = torch.from_numpy(d.P.T.copy()).T.cuda()
    for G in (2, 4, 8):
        ctxs, streams = make_ranks(rid, G)
        shards = [rid.shard_range(n, g, G) for g in range(G)]
        # each rank's shard in its own buffer (as on its own GPU), generated for its columns
        A_loc = [rid.generate(seed, m, n, k, noise, c0, nl) for c0, nl in shards]
        J_out = [torch.empty(k, dtype=torch.int64, device="cuda") for _ in range(G)]
        P_out = [rid.colmajor_empty(k, nl) for _, nl in shards]
        torch.cuda.synchronize()

        def dec(g):
            c0, nl = shards[g]
            r = rid.decompose(A_loc[g], k, l, seed, n=n, col0=c0, J=J_out[g], P=P_out[g],
                              ctx=ctxs[g])
            return r.diag

        diags = run_ranks(G, dec)
        P_cat = np.concatenate([np_(p) for p in P_out], axis=1)
        for g in range(G):
            assert np_(J_out[g]).tolist() == d.J.tolist(), (name, G, g)
            assert diags[g]["t_gather"] > 0.0
        assert bits_equal(P_cat, np_(ref.P)), (name, G)
        assert relf(P_cat, d.P) <= 1e-10

        # estimator on the oracle's (A, J, P), each rank its own block of P
        P_o_loc = [Po[:, c0:c0 + nl] for c0, nl in shards]  # column-major views, ld = k
        torch.cuda.synchronize()

        def est(g):
            c0, nl = shards[g]
            return rid.error_estimate(A_loc[g], Jo, P_o_loc[g], q, seed, n=n, col0=c0,
                                      ctx=ctxs[g])

        ests = run_ranks(G, est)
        for g in range(G):
            assert ests[g] == ests[0]  # replicated result, same bits on every rank
        assert abs(ests[0] - e_o) <= 1e-10 * e_o, (name, G, ests[0], e_o)
        for c in ctxs:
            c.close()


@pytest.mark.parametrize("name,seed,m,n,k,l,noise", CASES)
def test_multirank_sharded_qr(rid, orc, name, seed, m, n, k, l, noise, monkeypatch):
    """NEXT-3: no all-gather of Y; the G ranks factor their sketch blocks
    together (one pivot-candidate exchange and one pivot-column read from its owner per step).
    J equal to the oracle's, P within 1e-10 of it and bitwise equal to the one-rank call of the
    same (blocked) kernel; every rank's outputs identical."""
    d, _ = oracle_case(orc, seed, m, n, k, l, noise, 6)
    A = rid.generate(seed, m, n, k, noise)
    monkeypatch.setenv("RID_QRCP_VARIANT", "1")  # the blocked kernel the sharded QR runs
    ref = rid.decompose(A, k, l, seed)
    monkeypatch.delenv("RID_QRCP_VARIANT")
    assert np_(ref.J).tolist() == d.J.tolist()
    assert relf(np_(ref.P), d.P) <= 1e-10
    for G in (1, 2, 4, 8):
        ctxs, _ = make_ranks(rid, G)
        for c in ctxs:
            c.set_qr_dist("sharded")
        shards = [rid.shard_range(n, g, G) for g in range(G)]
        A_loc = [A[:, c0:c0 + nl] for c0, nl in shards]
        J_out = [torch.empty(k, dtype=torch.int64, device="cuda") for _ in range(G)]
        P_out = [rid.colmajor_empty(k, nl) for _, nl in shards]
        torch.cuda.synchronize()

        def dec(g):
            c0, nl = shards[g]
            r = rid.decompose(A_loc[g], k, l, seed, n=n, col0=c0, J=J_out[g], P=P_out[g],
                              ctx=ctxs[g])
            return r.diag

        diags = run_ranks(G, dec)
        for g in range(G):
            assert np_(J_out[g]).tolist() == d.J.tolist(), (name, G, g)
            assert abs(diags[g]["tie_margin_min"] - diags[0]["tie_margin_min"]) == 0.0
        P_cat = np.concatenate([np_(p) for p in P_out], axis=1)
        assert bits_equal(P_cat, np_(ref.P)), (name, G)
        for c in ctxs:
            c.close()


def test_sharded_qr_refused_without_local_comm(rid):
    ctx = rid.Context(0, torch.cuda.current_stream())
    ctx.set_qr_dist("sharded")  # no communicator: the one-rank QR (G = 1), nothing to shard
    A = rid.generate(1, 300, 64, 4, 1e-9)
    r = rid.decompose(A, 4, 8, 1, ctx=ctx)
    assert r.J.numel() == 4
    with pytest.raises(KeyError):
        ctx.set_qr_dist("bogus")
    ctx.close()


def test_multirank_host_buffers(rid, orc):
    """The e2e path (host A streamed in chunks, host P) under a 2-rank communicator."""
    seed, m, n, k, l, noise = 5, 1500, 600, 24, 40, 1e-9
    A_o = orc.generate(seed, m, n, k, noise)
    d = orc.decompose(A_o, k, l, seed)
    G = 2
    ctxs, _ = make_ranks(rid, G)
    shards = [rid.shard_range(n, g, G) for g in range(G)]

    def dec(g):
        c0, nl = shards[g]
        A_h = np.asfortranarray(A_o[:, c0:c0 + nl])
        return rid.decompose(A_h, k, l, seed, n=n, col0=c0, ctx=ctxs[g])

    res = run_ranks(G, dec)
    for r in res:
        assert r.J.tolist() == d.J.tolist()
    P_cat = np.concatenate([r.P for r in res], axis=1)
    assert relf(P_cat, d.P) <= 1e-10
    for c in ctxs:
        c.close()


def test_multirank_rejects_bad_shard_before_collective(rid):
    """Argument errors are raised before anything is enqueued or any rendezvous is entered."""
    ctxs, _ = make_ranks(rid, 2)
    A = rid.generate(1, 200, 64, 4, 0.0)
    with pytest.raises(rid.RidError) as e:
        rid.decompose(A[:, :32], 4, 8, 1, n=64, col0=16, ctx=ctxs[1])  # rank 1 owns [32, 64)
    assert e.value.status == rid.RID_EINVAL
    for c in ctxs:
        c.close()


def test_estimate_rejects_out_of_range_pivot(rid):
    A = rid.generate(1, 300, 40, 4, 1e-9)
    r = rid.decompose(A, 4, 8, 1)
    J = r.J.clone()
    J[2] = 40  # outside [0, n)
    with pytest.raises(rid.RidError) as e:
        rid.error_estimate(A, J, r.P, 3, 1)
    assert e.value.status == rid.RID_EINVAL


def test_buffer_layout_checks(rid):
    A = rid.generate(1, 64, 8, 2, 0.0)
    bad = A[:, :1].expand(64, 8)  # stride(1) == 0: columns alias
    with pytest.raises(ValueError):
        rid.sketch(bad, 1, 4)
    with pytest.raises(ValueError):
        rid.sketch(np.zeros((64, 8), np.complex128, order="C"), 1, 4)


def test_default_context_follows_current_stream(rid):
    """Calls without ctx= run on torch's current stream at the time of the call."""
    m, n, k, l = 512, 256, 8, 16
    A = rid.generate(3, m, n, k, 1e-9)
    Y0 = rid.sketch(A, 3, l)
    s = torch.cuda.Stream()
    with torch.cuda.stream(s):
        Y1 = rid.sketch(A, 3, l)
        Y1c = Y1.clone()  # ordered after the sketch on s only if librid used s
    torch.cuda.synchronize()
    assert torch.equal(torch.view_as_real(Y1c), torch.view_as_real(Y0))


def _random_cases(count, seed):
    rng = np.random.default_rng(seed)
    out = []
    for _ in range(count):
        G = int(rng.choice([2, 3, 4, 5, 8]))
        n = G * int(rng.integers(8, 300))
        m = int(rng.integers(64, 3000))
        k = int(rng.integers(1, min(m, n, 120) + 1))
        l = int(min(m, k + rng.integers(0, 40)))
        out.append((int(rng.integers(1, 1 << 30)), G, m, n, k, l,
                    float(rng.choice([0.0, 1e-12, 1e-9, 1e-6]))))
    return out


@pytest.mark.parametrize("seed,G,m,n,k,l,noise", _random_cases(8, 2027))
def test_multirank_random_shapes(rid, orc, seed, G, m, n, k, l, noise):
    """Random shapes and rank counts (G = 3, 5 included): the replicated path bitwise equal to one
    rank, the sharded QR equal to it to rounding (bitwise when n / G is a multiple of 32), J equal
    to the oracle's on every rank (unless the oracle reports a tie-ambiguous step)."""
    A_o = orc.generate(seed, m, n, k, noise)
    try:
        d = orc.decompose(A_o, k, l, seed)
    except Exception:  # noqa: BLE001 - a rank-deficient random draw: not a parity case
        pytest.skip("oracle rank failure")
    tie = k > 1 and d.tie_margins[:-1].min() < 1e-10
    A = rid.generate(seed, m, n, k, noise)
    ref = rid.decompose(A, k, l, seed)
    shards = [rid.shard_range(n, g, G) for g in range(G)]
    for dist in ("replicated", "sharded"):
        ctxs, _ = make_ranks(rid, G)
        for c in ctxs:
            c.set_qr_dist(dist)
        J_out = [torch.empty(k, dtype=torch.int64, device="cuda") for _ in range(G)]
        P_out = [rid.colmajor_empty(k, nl) for _, nl in shards]
        torch.cuda.synchronize()

        def dec(g):
            c0, nl = shards[g]
            rid.decompose(A[:, c0:c0 + nl], k, l, seed, n=n, col0=c0, J=J_out[g], P=P_out[g],
                          ctx=ctxs[g])

        run_ranks(G, dec)
        P_cat = np.concatenate([np_(p) for p in P_out], axis=1)
        for g in range(G):
            assert np_(J_out[g]).tolist() == np_(J_out[0]).tolist()
        if not tie:
            assert np_(J_out[0]).tolist() == d.J.tolist(), dist
            assert relf(P_cat, d.P) <= 1e-10, dist
        if dist == "replicated":
            assert bits_equal(P_cat, np_(ref.P))
        for c in ctxs:
            c.close()
