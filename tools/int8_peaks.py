#!/usr/bin/env python
"""Measure the int8 tensor-core roofline denominator on this B200 (the INT8_CRT sketch's GEMM) and
record it with the clocks seen DURING the measurement: profiles/int8_peaks.json (read by bench.py).

    python tools/int8_peaks.py            (on the GPU box; ~15 s)

MEASURED_PEAKS.json (driver-written) has HBM and bf16 only. This times cuBLASLt's int8 x int8 ->
int32 GEMM through torch._int_mm (a library GEMM, the same kind of reference as the driver's bf16
figure) at 8192^3 and at the sketch's own shape class (K = 65536 = 2m at C4): burst = best of 10
launches, sustained = back to back for ~4 s. 2 M N K ops per GEMM. Clock samples (nvidia-smi,
200 ms) from bench.py's ClockSampler.
"""
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

from bench import ClockSampler  # noqa: E402


def timed(a, b, reps):
    torch._int_mm(a, b)
    torch.cuda.synchronize()
    best = float("inf")
    for _ in range(reps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        torch._int_mm(a, b)
        e1.record()
        torch.cuda.synchronize()
        best = min(best, e0.elapsed_time(e1) * 1e-3)
    return best


def main():
    clk = ClockSampler(int(os.environ.get("LOCAL_RANK", "0")))
    clk.start()
    clk.wait_first()
    n0 = len(clk.lines)
    res = {}
    for name, (M, N, K) in {"square_8192": (8192, 8192, 8192),
                            "sketch_like": (8192, 528, 65536)}.items():
        a = torch.randint(-127, 128, (M, K), dtype=torch.int8, device="cuda")
        b = torch.randint(-127, 128, (N, K), dtype=torch.int8, device="cuda").T  # K-major B
        ops = 2.0 * M * N * K
        t = timed(a, b, 10)
        res[name] = {"M": M, "N": N, "K": K, "burst_tops": ops / t / 1e12}
    a = torch.randint(-127, 128, (8192, 8192), dtype=torch.int8, device="cuda")
    b = torch.randint(-127, 128, (8192, 8192), dtype=torch.int8, device="cuda").T
    torch.cuda.synchronize()
    t0 = time.time()
    n = 0
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    while time.time() - t0 < 4.0:
        for _ in range(20):
            torch._int_mm(a, b)
        n += 20
        torch.cuda.synchronize()
    e1.record()
    torch.cuda.synchronize()
    res["square_8192"]["sustained_tops"] = n * 2.0 * 8192**3 / (e0.elapsed_time(e1) * 1e-3) / 1e12
    clocks = clk.stop(first=n0)
    out = {"int8_tops_burst": res["square_8192"]["burst_tops"],
           "int8_tops_sustained": res["square_8192"]["sustained_tops"],
           "shapes": res, "clocks": clocks,
           "when": time.strftime("%Y-%m-%dT%H:%M:%SZ", time.gmtime()),
           "how": "torch._int_mm (cuBLASLt int8 x int8 -> int32), 2MNK ops; burst best of 10, "
                  "sustained 4 s back to back; tools/int8_peaks.py"}
    print(json.dumps(out))
    with open(os.path.join(ROOT, "profiles", "int8_peaks.json"), "w") as f:
        json.dump(out, f, indent=1)


if __name__ == "__main__":
    main()
