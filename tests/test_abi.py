"""CPU-side checks of the C-ABI boundary and the host logic (no GPU compute calls).

- librid.so builds for sm_100a, loads, and exports every symbol include/rid.h declares;
- host-only entry points (rid_error_bound, rid_version, rid_comm_id_bytes) behave;
- without a GPU the library fails loudly (status, not a silent CPU fallback);
- shard bookkeeping; the NCCL-id exchange over a world-size-2 gloo process group.
"""
import ctypes
import os
import re
import socket
import subprocess
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def rid():
    from paper_1205_3830_b200 import build

    build.build()
    import paper_1205_3830_b200 as rid

    return rid


def header_symbols():
    with open(os.path.join(ROOT, "include", "rid.h")) as f:
        src = f.read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(rid_[a-z_0-9]+)\s*\(", src)))


def test_exports_every_header_symbol(rid):
    syms = header_symbols()
    assert len(syms) >= 14
    out = subprocess.check_output(["nm", "-D", "--defined-only", rid.LIB_PATH], text=True)
    exported = set(l.split()[-1] for l in out.splitlines())
    missing = [s for s in syms if s not in exported]
    assert not missing, missing
    assert set(rid.EXPORTS) == set(syms)
    L = rid.lib()
    for s in syms:
        assert getattr(L, s) is not None


def test_sass_is_sm100a_with_dmma(rid):
    out = subprocess.check_output(["/usr/local/cuda/bin/cuobjdump", "-lelf", rid.LIB_PATH], text=True)
    assert "sm_100a" in out
    sass = subprocess.check_output(["/usr/local/cuda/bin/cuobjdump", "-sass", rid.LIB_PATH], text=True)
    assert "DMMA" in sass  # the FP64 tensor pipe (mma.sync .f64 -> DMMA.8x8x4)
    assert "LDGSTS" in sass  # cp.async staging


def test_host_entry_points(rid):
    L = rid.lib()
    assert b"sm_100a" in L.rid_version()
    assert L.rid_comm_id_bytes() == 128  # NCCL_UNIQUE_ID_BYTES
    b = rid.error_bound(2**14, 2**14, 100, 1e-20, 1e-14)
    assert abs(b - 1.2983e-8) <= 1e-4 * b
    assert rid.error_bound(10, 40, 3, 1.0, 2.0) == 50 * 20 * 2.0
    assert np.isnan(rid.error_bound(10, 40, 3, 0.0, 2.0))


@pytest.mark.skipif(os.environ.get("CUDA_VISIBLE_DEVICES_FORCE_GPU") == "1", reason="gpu box")
def test_no_gpu_fails_loudly(rid):
    import torch

    if torch.cuda.is_available():
        pytest.skip("a GPU is visible")
    with pytest.raises(rid.RidError):
        rid.Context(0)


def test_shard_range():
    from paper_1205_3830_b200 import shard_range
    from paper_1205_3830_b200.dist import plan

    assert shard_range(32768, 3, 8) == (12288, 4096)
    with pytest.raises(ValueError):
        shard_range(10, 0, 3)
    p = plan(16, 4)
    assert [p.owner(c) for c in (0, 3, 4, 15)] == [0, 0, 1, 3]
    t, loc = p.local_pivots([5, 0, 9, 4], 1)
    assert t.tolist() == [0, 3] and loc.tolist() == [1, 0]


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def test_id_exchange_gloo_world2(rid, tmp_path):
    script = tmp_path / "w.py"
    script.write_text(
        "import os, sys\n"
        f"sys.path.insert(0, {ROOT!r})\n"
        "import torch.distributed as dist\n"
        "from paper_1205_3830_b200.dist import exchange_id, plan\n"
        "dist.init_process_group('gloo')\n"
        "r = dist.get_rank()\n"
        "idb = bytes(range(128)) if r == 0 else bytes(128)\n"
        "got = exchange_id(idb)\n"
        "assert got == bytes(range(128)), got[:8]\n"
        "p = plan(64, dist.get_world_size())\n"
        "col0, nl = p.ranges[r]\n"
        "import torch\n"
        "t = torch.tensor([col0, nl])\n"
        "out = [torch.zeros(2, dtype=t.dtype) for _ in range(2)]\n"
        "dist.all_gather(out, t)\n"
        "assert [o.tolist() for o in out] == [[0, 32], [32, 32]]\n"
        "dist.destroy_process_group()\n"
        "print('ok', r)\n")
    env = dict(os.environ, MASTER_ADDR="127.0.0.1", MASTER_PORT=str(_free_port()), WORLD_SIZE="2")
    procs = [subprocess.Popen([sys.executable, str(script)], env=dict(env, RANK=str(r)),
                              stdout=subprocess.PIPE, stderr=subprocess.STDOUT, text=True)
             for r in range(2)]
    outs = [p.communicate(timeout=120)[0] for p in procs]
    assert all(p.returncode == 0 for p in procs), outs


def test_buffer_layouts_rejected_on_host(rid):
    """_Buf refuses layouts librid cannot address as (pointer, ld >= rows) — before any call."""
    import torch

    col = np.zeros((64, 1), np.complex128, order="F")
    with pytest.raises(ValueError):
        rid._Buf(np.broadcast_to(col, (64, 8)), 64, 8, "A")  # column stride 0
    with pytest.raises(ValueError):
        rid._Buf(torch.zeros(64, 1, dtype=torch.complex128).expand(64, 8), 64, 8, "A")
    ok = rid._Buf(np.zeros((64, 8), np.complex128, order="F"), 64, 8, "A")
    assert ok.ld == 64
    sub = np.zeros((80, 8), np.complex128, order="F")[:64]  # ld 80 > rows: fine
    assert rid._Buf(sub, 64, 8, "A").ld == 80


def test_bench_reference_arm_runs_on_cpu():
    """bench.py --impl reference (the oracle arm the driver runs) prints one valid JSON line."""
    import json
    import subprocess
    import sys

    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    out = subprocess.run([sys.executable, os.path.join(root, "bench.py"), "--impl", "reference",
                          "--config", "C1", "--steps", "1", "--warmup", "0", "--ref-seconds", "0.5"],
                         capture_output=True, text=True, timeout=600, cwd=root)
    assert out.returncode == 0, out.stderr[-2000:]
    line = json.loads(out.stdout.strip().splitlines()[-1])
    assert line["impl"] == "reference" and line["value"] > 0 and line["dtype"] == "f64"
    assert line["config"]["workload"] == "C1" and line["e2e"]["h2d_bytes_per_step"] == 0
