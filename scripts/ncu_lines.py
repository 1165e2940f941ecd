#!/usr/bin/env python
"""Aggregate an ncu capture's per-SASS stall samples and executed instructions
by CUDA source line (needs -lineinfo): python scripts/ncu_lines.py REP [TOP] [STALL_COLUMN]"""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 30
col = sys.argv[3] if len(sys.argv) > 3 else None  # e.g. stall_no_inst: rank by that stall reason
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
agg = {}
fname = "?"
hdr = None
for r in csv.reader(io.StringIO(out)):
    if not r:
        continue
    if r[0] == "File Path":
        fname = r[1].split("/")[-1]
        continue
    if r[0] == "Line No":
        hdr = r
        continue
    if hdr is None or len(r) < len(hdr) or r[0] in ("Function Name",):
        continue
    try:
        line = int(r[0])
    except ValueError:
        continue
    f = lambda i: float(r[i]) if r[i] not in ("", "-") else 0.0
    try:
        sv, iv = f(hdr.index(col) if col else 4), f(7)
    except ValueError:
        continue
    key = (fname, line, r[1].strip()[:90])
    a = agg.setdefault(key, [0.0, 0.0])
    a[0] += sv
    a[1] += iv
ts = sum(v[0] for v in agg.values()) or 1
ti = sum(v[1] for v in agg.values()) or 1
print(f"total stall samples {ts:.0f}, warp instructions {ti:.3g}")
for (fn, ln, src), (s, i) in sorted(agg.items(), key=lambda x: -x[1][0])[:top]:
    print(f"{100*s/ts:5.1f}% stall {100*i/ti:5.1f}% inst {fn}:{ln} | {src}")
