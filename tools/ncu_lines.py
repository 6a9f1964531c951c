"""Per-source-line instruction and stall-sample shares of one kernel in an ncu report.
    python tools/ncu_lines.py report.ncu-rep [N]"""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 40
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
hi = next(i for i, r in enumerate(rows) if r and r[0] == "Line No")
hdr = rows[hi]
i_ins = hdr.index("Instructions Executed")
i_samp = hdr.index("Warp Stall Sampling (All Samples)")
data = []
for r in rows[hi + 1:]:
    if len(r) <= i_samp or r[2] != "-":
        continue
    try:
        data.append((int(r[i_ins] or 0), int(r[i_samp] or 0), r[0], r[1][:110]))
    except ValueError:
        pass
ti = sum(d[0] for d in data) or 1
ts = sum(d[1] for d in data) or 1
print(f"instructions {ti}, stall samples {ts}")
for d in sorted(data, key=lambda x: -x[1])[:top]:
    print(f"{d[0] / ti * 100:5.1f}% ins {d[1] / ts * 100:5.1f}% samp  L{d[2]}: {d[3]}")
