#!/usr/bin/env python
"""Summarise ncu captures for profiles/: key counters of each .ncu-rep and the
per-kernel share of a launch-list CSV.

  python scripts/ncu_summary.py gpurun_out/X_fwd_kernel.ncu-rep ... [--launches gpurun_out/X_launches.csv]
"""
import csv
import io
import subprocess
import sys
from collections import defaultdict

KEYS = [
    "gpu__time_duration.sum", "launch__grid_size", "launch__block_size", "launch__registers_per_thread",
    "launch__shared_mem_per_block_dynamic", "launch__occupancy_limit_registers",
    "sm__warps_active.avg.pct_of_peak_sustained_active", "smsp__inst_executed.sum",
    "sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active",
    "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__pipe_shared_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__throughput.avg.pct_of_peak_sustained_elapsed",
    "dram__bytes_read.sum", "dram__bytes_write.sum", "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
    "lts__t_bytes.sum", "smsp__average_warp_latency_issue_stalled_barrier",
    "smsp__issue_active.avg.pct_of_peak_sustained_active",
]


def rep(path):
    out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    if len(rows) < 3:
        return f"{path}: no data\n"
    h, units = rows[0], rows[1]
    s = []
    for r in rows[2:]:
        d = dict(zip(h, r))
        s.append(f"### {d.get('Kernel Name', '?')[:90]}  ({path.split('/')[-1]})")
        for k in KEYS:
            if k in d:
                s.append(f"- {k}: {d[k]} {units[h.index(k)]}")
        stalls = sorted(((float(d[k] or 0), k) for k in h
                         if k.startswith("smsp__average_warp_latency_issue_stalled_") or
                         (k.startswith("smsp__pcsamp_warps_issue_stalled_") and not k.endswith("not_issued"))),
                        reverse=True)[:6]
        if stalls:
            s.append("- top stall counters: " + ", ".join(f"{k.split('stalled_')[-1]}={v:g}" for v, k in stalls))
    return "\n".join(s) + "\n"


def launches(path):
    txt = "".join(l for l in open(path) if not l.startswith("=="))
    tot = defaultdict(float)
    cnt = defaultdict(int)
    for d in csv.DictReader(io.StringIO(txt)):
        if d.get("Metric Name") != "gpu__time_duration.sum":
            continue
        name = d["Kernel Name"].split("(")[0]
        tot[name] += float(d["Metric Value"]) * (1e-6 if d["Metric Unit"] == "ns" else 1e-3 if d["Metric Unit"] == "us" else 1.0)
        cnt[name] += 1
    all_ms = sum(tot.values())
    s = [f"### launch list {path.split('/')[-1]} (ncu, serialised, cold-cache)", "| kernel | launches | total ms | share |", "|---|---|---|---|"]
    for k, v in sorted(tot.items(), key=lambda x: -x[1]):
        s.append(f"| {k} | {cnt[k]} | {v:.3f} | {v / all_ms:.1%} |")
    return "\n".join(s) + "\n"


if __name__ == "__main__":
    args = sys.argv[1:]
    out = []
    while args:
        a = args.pop(0)
        if a == "--launches":
            out.append(launches(args.pop(0)))
        else:
            out.append(rep(a))
    print("\n".join(out))
