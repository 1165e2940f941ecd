#!/usr/bin/env python
"""Executed warp instructions per SASS opcode from an ncu capture's source page:
python scripts/ncu_opcodes.py REP [TOP]"""
import csv
import io
import re
import subprocess
import sys

rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 30
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
agg, hdr = {}, None
for r in csv.reader(io.StringIO(out)):
    if not r:
        continue
    if "Address" in r and "Source" in r:
        hdr = r
        continue
    if hdr is None or len(r) < len(hdr):
        continue
    d = dict(zip(hdr, r))
    src = d.get("Source", "").strip()
    m = re.match(r"(?:@!?U?P\w+\s+)?([A-Z0-9_]+)(\.[A-Z0-9_.]+)?", src)
    if not m:
        continue
    try:
        n = float(d.get("Instructions Executed", "0") or 0)
    except ValueError:
        continue
    op = m.group(1) + ((m.group(2) or "")[:12] if m.group(1) in ("LDS", "STS", "LDG", "STG", "SHFL") else "")
    agg[op] = agg.get(op, 0) + n
tot = sum(agg.values()) or 1
print(f"total {tot:.4g} warp instructions")
for op, n in sorted(agg.items(), key=lambda x: -x[1])[:top]:
    print(f"{100 * n / tot:5.1f}% {n:12.4g} {op}")
