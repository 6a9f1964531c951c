"""Host-side cost of one rid.decompose call at C1 (the GPU work is ~150 us): Python wall time per
call with and without the CUDA graph, the raw C call through ctypes with prepared arguments, and
the device span (diag t_total).   python tools/host_overhead.py"""
import ctypes
import os
import sys
import time

sys.path.insert(0, os.getcwd())
import torch  # noqa: E402

import paper_1205_3830_b200 as rid  # noqa: E402

os.environ["RID_GRAPH_DEBUG"] = "1"
A = rid.generate(1, 1024, 512, 16, 0.0)
J = torch.empty(16, dtype=torch.int64, device="cuda")
P = rid.colmajor_empty(16, 512, device="cuda")
for g in ("1", "0"):
    os.environ["RID_GRAPH"] = g
    for _ in range(5):
        rid.decompose(A, 16, 24, 1, J=J, P=P)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(200):
        r = rid.decompose(A, 16, 24, 1, J=J, P=P)
    torch.cuda.synchronize()
    dt = (time.perf_counter() - t0) / 200
    print(f"RID_GRAPH={g}: {dt * 1e6:.1f} us per decompose (wall), diag t_total "
          f"{r.diag['t_total'] * 1e6:.1f} us", flush=True)
os.environ["RID_GRAPH"] = "1"
ctx = rid.default_context()
L = rid.lib()
d = rid.Diag()
args = (ctx.h, A.data_ptr(), 1024, 512, 0, 512, 1024, 16, 24, 1, J.data_ptr(), P.data_ptr(), 16,
        ctypes.byref(d))
for _ in range(5):
    L.rid_decompose(*args)
t0 = time.perf_counter()
for _ in range(200):
    L.rid_decompose(*args)
dt = (time.perf_counter() - t0) / 200
print(f"raw C rid_decompose (graph replay, prepared args): {dt * 1e6:.1f} us per call", flush=True)
t0 = time.perf_counter()
for _ in range(1000):
    rid.sketch_mults()
print(f"trivial ctypes call: {(time.perf_counter() - t0) / 1000 * 1e6:.2f} us", flush=True)
