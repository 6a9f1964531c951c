"""The pipelined INT8_CRT sketch with an SM split (experiment build: RID_BUILD_EXPERIMENTS=1):
the residue preparation of block c+2 on RID_CRT_PIPE_SPLIT SMs of its own beside block c's GEMM
on the other SMs. Times the sketch of one config (median of 5 after a warm-up; CUDA events on the
context stream) for each setting and checks Y bitwise against the default.

    python tools/crt_split_exp.py C4 "PIPE=0" "PIPE=1" "PIPE=1,SPLIT=16,NB=8192" ...
"""
import os
import sys

sys.path.insert(0, os.getcwd())
import torch  # noqa: E402

import paper_1205_3830_b200 as rid  # noqa: E402
from paper_1205_3830_b200.configs import CONFIGS  # noqa: E402

name = sys.argv[1]
c = CONFIGS[name]
st = torch.cuda.current_stream()
ctx = rid.Context(0, st)
A = rid.generate(1, c.m, c.n, c.k, c.noise, ctx=ctx)
Y0 = rid.sketch(A, 1, c.l, ctx=ctx)
torch.cuda.synchronize()
Y = torch.empty_like(Y0)
for setting in sys.argv[2:]:
    for k in ("RID_CRT_PIPE", "RID_CRT_PIPE_SPLIT", "RID_CRT_PIPE_NB"):
        os.environ.pop(k, None)
    for kv in setting.split(","):
        k, v = kv.split("=")
        os.environ["RID_CRT_" + k] = v
    rid.sketch(A, 1, c.l, out=Y, ctx=ctx)
    torch.cuda.synchronize()
    ts = []
    for _ in range(5):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(st)
        rid.sketch(A, 1, c.l, out=Y, ctx=ctx)
        e1.record(st)
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    ts.sort()
    same = bool(torch.equal(torch.view_as_real(Y), torch.view_as_real(Y0)))
    print(f"{name} {setting:32s} sketch {ts[2]:8.3f} ms (min {ts[0]:.3f}) bitwise={same}", flush=True)
