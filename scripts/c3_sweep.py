"""C3: stiff Chaboche, sparse batch (nb=50, nt=20000): chunked
solvers vs sequential (n_chunk=1) stepping on one GPU. Prints one JSON line per
(solver, n_chunk) with forward+adjoint wall time through the public API."""
import json
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2310_08649_b200 as P  # noqa: E402
from paper_2310_08649_b200 import api  # noqa: E402


def chaboche_plastic(n_unit, nb, scale=10.0):
    m = P.build_chaboche(n_unit, nb)
    p = m.params.copy()
    o = 6 + 2 * n_unit
    p[o:o + nb] *= scale
    return m.with_params(p)


nb, nt = int(os.environ.get("C3_NB", 50)), int(os.environ.get("C3_NT", 20000))
m = chaboche_plastic(3, nb)
grid = api.TimeGrid.uniform(nt, nb, 10.0)
y0 = np.zeros((nb, m.state_size))
ctx = api.Context(0)
cfgs = [(0, 1), (0, 16), (0, 128), (1, 16), (1, 64), (1, 256), (1, 1024), (2, 16), (2, 256)]
if len(sys.argv) > 1:
    cfgs = [tuple(int(v) for v in a.split(",")) for a in sys.argv[1:]]
for kind, nc in cfgs:
    sv = api.SolverChoice(kind, 2)
    api.gradient_adjoint(m, y0, grid, nc, solver=sv, ctx=ctx)  # warm-up
    reps = 2
    t0 = time.perf_counter()
    for _ in range(reps):
        r = api.gradient_adjoint(m, y0, grid, nc, solver=sv, ctx=ctx)
    dt = (time.perf_counter() - t0) / reps
    print(json.dumps({"solver": ["thomas", "pcr", "hybrid"][kind], "n_chunk": nc, "seconds": dt,
                      "series_steps_per_s": nb * nt / dt, "newton_iterations": r.trajectory.work.newton_iterations,
                      "kernel_gen": ctx.kernel_generation_used(), "loss": r.loss}), flush=True)
