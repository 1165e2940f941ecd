"""Diagnostics: per-row timeline of CTA 0 in the first chunk of a v2 forward (CKO_TRACE)."""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
path = "/tmp/cko_trace.bin"
os.environ["CKO_TRACE"] = path
import paper_2310_08649_b200 as P  # noqa: E402
from paper_2310_08649_b200 import api  # noqa: E402

nb, nt, nc = int(sys.argv[1]), int(sys.argv[2]), int(sys.argv[3])
m = P.build_mass_damper_spring(10, nb)
grid = api.TimeGrid.uniform(nt, nb, nt * 1e-6)
for rep in range(2):
    api.integrate_backward_euler(m, np.zeros((nb, 20)), grid, nc, solver=api.SolverChoice(0))
t = np.fromfile(path, dtype=np.uint64).astype(np.int64)
k0 = t[0]
print("chunk markers (us from chunk-0 start): res0, [it: epoch-start, epoch-end, res+sync-end]")
for ch in range(4):
    row = t[ch * 16: ch * 16 + 16]
    print(ch, [(v - k0) / 1000 if v else None for v in row])
rows = t[64:].reshape(-1, 8)
print("row: prod(wait-start, acquired, lu-start, lu-end) cons(wait-start, acquired, done) [writer] in us")
for k in range(min(nc, int(os.environ.get("TRACE_ROWS", "24")))):
    r = rows[k]
    print(k, " ".join(f"{(v - k0) / 1000:8.2f}" if v else "       -" for v in r[:8]))
cons = rows[:, 6] - rows[:, 5]
lu = rows[:, 3] - rows[:, 2]
print("consumer solve us: median %.3f; producer LU us: median %.3f; producer load us: median %.3f" % (
    np.median(cons[cons > 0]) / 1000, np.median(lu[lu > 0]) / 1000, np.median((rows[:, 2] - rows[:, 1])[lu > 0]) / 1000))
ncx = min(nc, nt)
ctas = t[64 + 8 * ncx:].reshape(-1, 8)
ctas = ctas[ctas[:, 0] > 0]
if len(ctas):
    z = ctas[:, 0].min()
    rel = (ctas[:, :6] - z) / 1000
    print("per-CTA (us from earliest chunk start): start res0 bar1 epoch-end res bar2 ; spread / percentiles")
    for j, name in enumerate(["start", "res0", "bar1", "epoch_end", "res", "bar2"]):
        col = rel[:, j]
        print(f"  {name:9s} min {col.min():8.2f}  p50 {np.median(col):8.2f}  max {col.max():8.2f}")
    d = rel[:, 1:6] - rel[:, 0:5]
    for j, name in enumerate(["res0", "bar1-wait", "epoch", "res", "bar2-wait"]):
        print(f"  dur {name:10s} min {d[:, j].min():8.2f}  p50 {np.median(d[:, j]):8.2f}  max {d[:, j].max():8.2f}")
