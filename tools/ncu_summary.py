"""Summarise ncu outputs (launch list CSV + --set full reports) into profiles/ text files.

    python tools/ncu_summary.py <round-tag> <cfg>
reads gpurun_out/launches_<cfg>.csv, gpurun_out/prof_sketch*_<cfg>.ncu-rep (one per sketch
launch), prof_qrcp_<cfg>.ncu-rep, prof_update_<cfg>.ncu-rep
writes profiles/<tag>_<cfg>_launches.txt, profiles/<tag>_<cfg>_ncu_summary.txt and updates
profiles/traffic.json (dram bytes per launch of the sketch, read by bench.py's roofline.traffic).
"""
import csv
import glob
import io
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
OUT = os.path.join(ROOT, "gpurun_out")
PROF = os.path.join(ROOT, "profiles")

KEYS = [
    "gpu__time_duration.sum", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
    "sm__pipe_tensor_subpipe_dmma_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_tensor_subpipe_dmma.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active",
    "dram__bytes_read.sum", "dram__bytes_write.sum", "dram__throughput.avg.pct_of_peak_sustained_elapsed",
    "lts__t_sector_hit_rate.pct", "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum",
    "launch__registers_per_thread", "launch__grid_size", "launch__block_size",
    "launch__occupancy_limit_registers", "sm__warps_active.avg.pct_of_peak_sustained_active",
    "smsp__warp_issue_stalled_barrier_per_warp_active.pct",
    "dram__bytes.sum.per_second", "sm__inst_executed_pipe_tensor_subpipe_dmma.sum",
    "TPC.TriageCompute.sm__pipe_tensor_cycles_active_realtime.avg.pct_of_peak_sustained_elapsed",
    "sm__mem_tensor_cycles_active.avg.pct_of_peak_sustained_active",
    "l1tex__data_pipe_tc_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed",
    "smsp__issue_active.avg.pct_of_peak_sustained_active",
    "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active",
    "smsp__inst_executed.sum",
]


def raw(rep):
    txt = subprocess.check_output(["ncu", "-i", rep, "--page", "raw", "--csv"], text=True,
                                  stderr=subprocess.DEVNULL)
    rows = list(csv.reader(io.StringIO(txt)))
    h, units = rows[0], rows[1]
    out = []
    for r in rows[2:]:
        out.append({k: (v, u) for k, v, u in zip(h, r, units)})
    return out


def stalls(d):
    items = []
    for k, (v, u) in d.items():
        if "pcsamp_warps_issue_stalled" in k and not k.endswith("not_issued"):
            try:
                items.append((k.split("stalled_")[-1], float(v.replace(",", ""))))
            except ValueError:
                pass
    tot = sum(v for _, v in items) or 1.0
    return [(k, 100 * v / tot) for k, v in sorted(items, key=lambda x: -x[1])[:8]]


def main(tag, cfg):
    lines = []
    launches = os.path.join(OUT, f"launches_{cfg}.csv")
    if os.path.exists(launches):
        rows = list(csv.reader(open(launches)))
        hi = [i for i, r in enumerate(rows) if "Kernel Name" in r][0]
        h = rows[hi]
        ki, vi = h.index("Kernel Name"), h.index("Metric Value")
        ll = [f"# ncu --metrics gpu__time_duration.sum --clock-control none (cold-cache, serialised)",
              f"# bench.py --config {cfg} --steps 1 --warmup 1 --q 1 (generation, warm-up step, "
              "timed step, estimator)", "kernel,ms"]
        for r in rows[hi + 1:]:
            if len(r) > vi:
                ll.append(f"{r[ki].split('(')[0].strip()},{float(r[vi].replace(',', '')) / 1e6:.4f}")
        with open(os.path.join(PROF, f"{tag}_{cfg}_launches.txt"), "w") as f:
            f.write("\n".join(ll) + "\n")
    traffic_path = os.path.join(PROF, "traffic.json")
    traffic = json.load(open(traffic_path)) if os.path.exists(traffic_path) else {}
    seen = {}
    reps = [("sketch", p) for p in sorted(glob.glob(os.path.join(OUT, f"prof_sketch*_{cfg}.ncu-rep")))]
    reps += [(kind, os.path.join(OUT, f"prof_{kind}_{cfg}.ncu-rep"))
             for kind in ("crt_gemm", "crt_prep", "crt_rec", "qrcp", "update")]
    for kind, rep in reps:
        if not os.path.exists(rep):
            continue
        for d in raw(rep):
            name = d.get("Kernel Name", ("?", ""))[0]
            lines.append(f"== {kind}: {name}")
            for k in KEYS:
                if k in d:
                    lines.append(f"  {k:80s} {d[k][0]:>16s} {d[k][1]}")
            if "sm__inst_executed_pipe_tensor_subpipe_dmma.sum" in d:
                try:  # executed tensor work: one DMMA.8x8x4 = 8 x 8 x 4 FMA = 512 flop
                    cnt = float(d["sm__inst_executed_pipe_tensor_subpipe_dmma.sum"][0]
                                .replace(",", ""))
                    lines.append(f"  DMMA instructions x 512 flop = {cnt * 512:.4e} flop executed")
                except ValueError:
                    pass
            lines.append("  top stall reasons (% of samples): " +
                         ", ".join(f"{k} {v:.1f}" for k, v in stalls(d)))
            try:
                rd = float(d["dram__bytes_read.sum"][0].replace(",", ""))
                wr = float(d["dram__bytes_write.sum"][0].replace(",", ""))
                unit = d["dram__bytes_read.sum"][1]
                scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(unit, 1)
                scale_w = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(
                    d["dram__bytes_write.sum"][1], 1)
                if rd != rd or wr != wr:  # a replay that returned no counters (nan): skip
                    raise ValueError("nan")
                # the sketch phase = every launch in its report (the Strassen products: four)
                key = f"{cfg}/{kind}"
                prev = traffic.get(key, {}) if seen.get(key) else {}
                seen[key] = True
                traffic[key] = {"dram_bytes_per_launch":
                                prev.get("dram_bytes_per_launch", 0.0) + rd * scale + wr * scale_w,
                                "source": f"profiles/{tag}_{cfg}_ncu_summary.txt"}
            except (KeyError, ValueError):
                pass
    with open(os.path.join(PROF, f"{tag}_{cfg}_ncu_summary.txt"), "w") as f:
        f.write("\n".join(lines) + "\n")
    with open(traffic_path, "w") as f:
        json.dump(traffic, f, indent=1)
    print("\n".join(lines))


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2])
