#!/usr/bin/env python
"""Measure the FP64 tensor-pipe (DMMA) roofline denominators on this B200 and record them with the
clocks seen DURING the measurement: profiles/fp64_peaks.json (read by bench.py).

    python tools/fp64_peaks.py            (on the GPU box; ~10 s)

MEASURED_PEAKS.json (driver-written) has HBM and bf16 peaks only; the FP64 sketch needs the DMMA
peak. tools/microbench_fp64.cu `mb peaks` runs mma.sync.m8n8k4.f64 with 8 independent
accumulators per warp at 2 CTAs x 256 threads per SM: burst = best of 10 single ~10 ms launches,
sustained = back to back for ~4 s. Clock samples (nvidia-smi, 200 ms) come from bench.py's
ClockSampler; a run with a thermal/hw slowdown reason or SM clocks well below max is flagged.
"""
import json
import os
import subprocess
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from bench import ClockSampler  # noqa: E402


def main():
    mb = os.path.join(ROOT, "tools", "mb")
    src = os.path.join(ROOT, "tools", "microbench_fp64.cu")
    if not os.path.exists(mb) or os.path.getmtime(mb) < os.path.getmtime(src):
        subprocess.check_call(["/usr/local/cuda/bin/nvcc", "-gencode",
                               "arch=compute_100a,code=sm_100a", "-O3", "-o", mb, src])
    clk = ClockSampler(int(os.environ.get("LOCAL_RANK", "0")))
    clk.start()
    clk.wait_first()
    n0 = len(clk.lines)
    out = subprocess.check_output([mb, "peaks"], text=True)
    clocks = clk.stop(first=n0)
    res = json.loads(out.strip().splitlines()[-1])
    gpu = subprocess.run(["nvidia-smi", "--query-gpu=name,driver_version", "--format=csv,noheader"],
                         capture_output=True, text=True).stdout.strip()
    bad = [r for r in clocks.get("reasons", []) if r in ("hw_slowdown", "hw_thermal_slowdown",
                                                         "sw_thermal_slowdown")]
    low = (clocks.get("sm_mhz") and clocks.get("sm_max_mhz")
           and clocks["sm_mhz"] < 0.9 * clocks["sm_max_mhz"] and "sw_power_cap" not in
           clocks.get("reasons", []))
    res.update({"gpu": gpu, "when": time.strftime("%Y-%m-%dT%H:%M:%SZ", time.gmtime()),
                "clocks": clocks, "valid": not bad and not low,
                "how": "tools/microbench_fp64.cu `mb peaks` under tools/fp64_peaks.py (nvidia-smi "
                       "sampled every 200 ms during the run)"})
    path = os.path.join(ROOT, "profiles", "fp64_peaks.json")
    if len(sys.argv) > 1:
        path = sys.argv[1]
    with open(path, "w") as f:
        json.dump(res, f, indent=1)
    print(json.dumps(res))


if __name__ == "__main__":
    main()
