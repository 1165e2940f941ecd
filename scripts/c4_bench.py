"""C4: neural ODE, state 8, hidden width 128 (18 824 parameters),
nb=256, nt=2000, one adjoint training step (forward + adjoint + parameter
gradient) through the public API on one GPU. One JSON line per (solver, n_chunk)."""
import json
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2310_08649_b200 as P  # noqa: E402
from paper_2310_08649_b200 import api  # noqa: E402

nb, nt = int(os.environ.get("C4_NB", 256)), int(os.environ.get("C4_NT", 2000))
m = P.build_node_wide(8, 128, nb)
grid = api.TimeGrid.uniform(nt, nb, 1.0)
y0 = np.zeros((nb, 8))
ctx = api.Context(0)
cfgs = [(0, 1), (0, 10), (0, 100), (1, 10)]
if len(sys.argv) > 1:
    cfgs = [tuple(int(v) for v in a.split(",")) for a in sys.argv[1:]]
for kind, nc in cfgs:
    sv = api.SolverChoice(kind, 1)
    api.gradient_adjoint(m, y0, grid, nc, solver=sv, ctx=ctx)
    t0 = time.perf_counter()
    r = api.gradient_adjoint(m, y0, grid, nc, solver=sv, ctx=ctx)
    dt = time.perf_counter() - t0
    print(json.dumps({"solver": ["thomas", "pcr", "hybrid"][kind], "n_chunk": nc, "seconds": dt,
                      "series_steps_per_s": nb * nt / dt, "newton_iterations": r.trajectory.work.newton_iterations,
                      "kernel_gen": ctx.kernel_generation_used(), "loss": r.loss,
                      "grad_norm": float(np.linalg.norm(r.gradient))}), flush=True)
