"""The NCCL (multi-GPU) code path of librid, exercised on the one GPU this environment has.

With RID_FORCE_NCCL=1 a 1-rank NCCL communicator is created, so rid_decompose runs its in-place
all-gather of Y and rid_error_estimate its all-reduce of B = A[:, J] and all-gathers of the
compensated partials — the exact branches a G-GPU run takes — through real NCCL calls.
Results must equal the communicator-free call (J, P bitwise; the estimate to rounding, since
the collective path merges the partial accumulators in a different order).
The G > 1 data path itself (sharded sketch, concatenated Y, per-shard solve) is checked bitwise
by tests/test_gpu_parity.py::test_g_emulation_bitwise; the host plumbing by tests/test_abi.py.
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


def test_one_rank_nccl_path_matches(rid):
    m, n, k, l, noise, seed = 3000, 1200, 40, 56, 1e-9, 3
    ctx0 = rid.Context(0, torch.cuda.current_stream())
    A = rid.generate(seed, m, n, k, noise, ctx=ctx0)
    ref = rid.decompose(A, k, l, seed, ctx=ctx0)
    est0 = rid.error_estimate(A, ref.J, ref.P, 6, seed, ctx=ctx0)

    os.environ["RID_FORCE_NCCL"] = "1"
    try:
        ctx1 = rid.Context(0, torch.cuda.current_stream())
        ctx1.comm_init(rid.comm_get_id(), 0, 1)
        assert ctx1.comm_info() == (0, 1)
        r = rid.decompose(A, k, l, seed, ctx=ctx1)
        est1 = rid.error_estimate(A, r.J, r.P, 6, seed, ctx=ctx1)
    finally:
        del os.environ["RID_FORCE_NCCL"]
    assert torch.equal(r.J, ref.J)
    assert torch.equal(torch.view_as_real(r.P), torch.view_as_real(ref.P))
    assert abs(est1 - est0) <= 1e-12 * est0
    ctx1.close()
    ctx0.close()


def test_comm_rejects_bad_shards(rid):
    os.environ["RID_FORCE_NCCL"] = "1"
    try:
        ctx = rid.Context(0, torch.cuda.current_stream())
        ctx.comm_init(rid.comm_get_id(), 0, 1)
    finally:
        del os.environ["RID_FORCE_NCCL"]
    A = rid.generate(1, 200, 64, 4, 0.0, ctx=ctx)
    with pytest.raises(rid.RidError):
        rid.decompose(A[:, :32], 4, 8, 1, n=64, col0=0, ctx=ctx)  # 1 rank must own all columns
    ctx.close()
