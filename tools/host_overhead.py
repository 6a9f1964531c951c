"""Host-side cost of one rid.decompose call at a small config: Python wall time per call (the
GPU work of C1 is ~150 us), with and without the CUDA graph.   python tools/host_overhead.py"""
import os
import sys
import time

sys.path.insert(0, os.getcwd())
import torch  # noqa: E402

import paper_1205_3830_b200 as rid  # noqa: E402

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
    # the ctypes call alone: time the C function through the binding with a trivial query
t0 = time.perf_counter()
for _ in range(1000):
    rid.sketch_mults()
print(f"trivial ctypes call: {(time.perf_counter() - t0) / 1000 * 1e6:.2f} us", flush=True)
