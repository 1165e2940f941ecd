#!/usr/bin/env python
"""Record DRAM traffic per launch from full ncu captures into profiles/traffic.json,
keyed the way bench.py looks it up: "<fwd_kernel|adj_kernel>:<solver>:<n_chunk>:<nb>:<nt>".

  python scripts/ncu_traffic.py fwd_kernel gpurun_out/X_fwd.ncu-rep adj_kernel gpurun_out/X_adj.ncu-rep \
      --config thomas:100:1000:10000 --tag r1v2
"""
import csv
import io
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def dram_bytes(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    h, units, v = rows[0], rows[1], rows[2]
    tot = 0.0
    for name in ("dram__bytes_read.sum", "dram__bytes_write.sum"):
        i = h.index(name)
        scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}[units[i]]
        tot += float(v[i]) * scale
    return tot


args = sys.argv[1:]
cfg = args[args.index("--config") + 1]
tag = args[args.index("--tag") + 1]
pairs = args[:args.index("--config")]
path = os.path.join(ROOT, "profiles", "traffic.json")
tab = json.load(open(path)) if os.path.exists(path) else {}
for k, rep in zip(pairs[0::2], pairs[1::2]):
    b = dram_bytes(rep)
    tab[f"{k}:{cfg}"] = {"bytes_per_launch": b, "source": f"ncu --set full, {os.path.basename(rep)} ({tag})"}
    print(k, cfg, f"{b:.4g} B")
json.dump(tab, open(path, "w"), indent=1, sort_keys=True)
