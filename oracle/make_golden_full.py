"""Full-size golden summaries of the headline configurations, from the COMPILED
REFERENCE (oracle/_ref). TEST INFRASTRUCTURE ONLY.

    python oracle/make_golden_full.py [c2] [c3]

The full trajectories are GBs, so each fixture stores size-independent
summaries the GPU run can be checked against at full size:
  loss, gradient, forward/backward WorkCounters, the last trajectory row,
  per-row checksums sum_j states[i, j] (a "checksum of checksums" over every
  step) and per-row sums of squares.

  full_c2.npz : C2, MDS 10 units (n = 20), nb = 1000, nt = 10000, t_max = 0.01,
                Thomas n_chunk = 100 (the bench line's workload).
                The reference's MDS adjoint runs the Dual8 forward-AD VJP over
                1031 parameters (ode_model.hpp:154-182): ~70 min single thread.
  full_c3.npz : C3, Chaboche n_unit = 3 (eps_a x 10), nb = 50, nt = 20000,
                t_max = 10: Thomas n_chunk = 1 (sequential) and PCR n_chunk = 256.
"""
from __future__ import annotations

import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import paper_2310_08649_b200 as P  # noqa: E402
from oracle import load_ref  # noqa: E402
from tests.cases import chaboche_plastic  # noqa: E402
from tests.conftest import uniform_times  # noqa: E402

OUT = os.path.join(ROOT, "tests", "golden")
KEYS = ["newton_iterations", "rate_evals", "jacobian_evals", "linear_solves", "reduction_sweeps"]


def summary(prefix, r):
    return {
        f"{prefix}loss": np.array(r.loss),
        f"{prefix}grad": r.grad,
        f"{prefix}fwd": np.array([r.fwd[k] for k in KEYS]),
        f"{prefix}bwd": np.array([r.bwd[k] for k in KEYS]),
        f"{prefix}last_row": r.states[-1].copy(),
        f"{prefix}row_sum": r.states.sum(axis=1),
        f"{prefix}row_sumsq": (r.states * r.states).sum(axis=1),
    }


def c2():
    ref = load_ref()
    nb, nt, nc = 1000, 10000, 100
    m = P.build_mass_damper_spring(10, nb)
    y0 = np.zeros((nb, 20))
    t = uniform_times(nt, nb, 0.01)
    t0 = time.time()
    r = ref.gradient(m, y0, t, nc, solver=(0, 1))
    rec = dict(nb=nb, nt=nt, n_chunk=nc, t_max=0.01, n_unit=10, seconds=time.time() - t0, **summary("thomas_", r))
    np.savez_compressed(os.path.join(OUT, "full_c2.npz"), **rec)
    print(f"c2: loss {r.loss!r} in {time.time() - t0:.0f} s", flush=True)


def c3():
    ref = load_ref()
    nb, nt = 50, 20000
    m = chaboche_plastic(3, nb)
    y0 = np.zeros((nb, 5))
    t = uniform_times(nt, nb, 10.0)
    rec = dict(nb=nb, nt=nt, t_max=10.0, n_unit=3, eps_scale=10.0)
    for name, nc, sv in (("seq", 1, (0, 1)), ("pcr256", 256, (1, 1))):
        t0 = time.time()
        r = ref.gradient(m, y0, t, nc, solver=sv)
        rec.update(summary(f"{name}_", r))
        print(f"c3 {name}: loss {r.loss!r}, newton {r.fwd['newton_iterations']} in {time.time() - t0:.0f} s",
              flush=True)
    np.savez_compressed(os.path.join(OUT, "full_c3.npz"), **rec)


if __name__ == "__main__":
    which = sys.argv[1:] or ["c3", "c2"]
    for w in which:
        {"c2": c2, "c3": c3}[w]()
