"""Generate tests/golden/*.npz from the COMPILED REFERENCE (oracle/_ref).

TEST INFRASTRUCTURE ONLY. Run here, where /root/reference exists:
    python oracle/make_golden.py
The fixtures pin the C restatement (tests/test_oracle_golden.py, CPU) and
the CUDA path (tests/test_gpu_golden.py) to the reference's own outputs.
Contents:
  traj_<case>.npz  : model (kind, dims, params), y0, times, n_chunk, and for
                     each solver the reference states (thomas, pcr), loss,
                     gradient and forward/backward WorkCounters;
  solvers.npz      : make_random_system / make_random_rhs inputs
                     (verify.cpp:413-433) with solve_thomas / solve_pcr /
                     solve_hybrid(0,2,30) / solve_dense_oracle outputs and
                     sweep counts (acceptance.cpp:56-89 grid);
  model_<name>.npz : rate, Jacobian and parameter VJP at random points
                     (the MDS VJP is the reference's Dual8 sweep).
"""
from __future__ import annotations

import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from oracle import load_ref  # noqa: E402
from tests.cases import ALL_CASES, case  # noqa: E402

OUT = os.path.join(ROOT, "tests", "golden")
SOLVERS = {"thomas": (0, 1), "pcr": (1, 1), "hybrid1": (2, 1)}
KEYS = ["newton_iterations", "rate_evals", "jacobian_evals", "linear_solves", "reduction_sweeps"]


def model_meta(m):
    return dict(kind=m.kind, n_unit=m.n_unit, width=m.width, n_batch=m.n_batch, params=m.params)


def main():
    ref = load_ref()
    os.makedirs(OUT, exist_ok=True)
    for name in ALL_CASES:
        m, y0, t, nc = case(name)
        rec = dict(model_meta(m), y0=y0, times=t, n_chunk=nc)
        for sname, sv in SOLVERS.items():
            r = ref.gradient(m, y0, t, nc, solver=sv)
            if sname in ("thomas", "pcr"):
                rec[f"{sname}_states"] = r.states
            rec[f"{sname}_loss"] = r.loss
            rec[f"{sname}_grad"] = r.grad
            rec[f"{sname}_fwd"] = np.array([r.fwd[k] for k in KEYS])
            rec[f"{sname}_bwd"] = np.array([r.bwd[k] for k in KEYS])
        np.savez_compressed(os.path.join(OUT, f"traj_{name}.npz"), **rec)

    # solver equivalence grid (acceptance.cpp:56-89, n_size/n_batch subsampled)
    sol = {}
    seed = 2000
    idx = 0
    for nc in (1, 2, 3, 4, 5, 6, 7, 9, 12, 16, 17, 24, 31, 32, 33):
        for n in (1, 2, 3, 5):
            for nb in (1, 3):
                diag, off = ref.random_system(nc, nb, n, seed)
                rhs = ref.random_rhs(nc, nb, n, seed + 1)
                seed += 2
                p = f"s{idx}_"
                sol[p + "shape"] = np.array([nc, nb, n])
                sol[p + "diag"], sol[p + "off"], sol[p + "rhs"] = diag, off, rhs
                sol[p + "dense"] = ref.solve_dense(diag, off, rhs)
                for key, sv in {"thomas": (0, 1), "pcr": (1, 1), "h0": (2, 0), "h2": (2, 2), "h30": (2, 30)}.items():
                    x, sw = ref.solve(diag, off, rhs, sv)
                    sol[p + key] = x
                    sol[p + key + "_sweeps"] = np.array(sw)
                idx += 1
    sol["count"] = np.array(idx)
    np.savez_compressed(os.path.join(OUT, "solvers.npz"), **sol)

    # model kernels at random points
    rng = np.random.default_rng(20231008)
    for name in ("lin3", "mds", "chaboche", "node", "node_wide", "scalar", "constant"):
        m = case(name)[0]
        nb = max(m.n_batch, 2)
        c = 5
        n = m.state_size
        tt = rng.uniform(0.0, 1.0, (c, nb))
        scale = 0.05 if name == "mds" else (3.0 if name == "chaboche" else 1.0)
        yy = scale * rng.uniform(-1, 1, (c, nb, n))
        ww = rng.uniform(-1, 1, (c, nb, n))
        rec = dict(model_meta(m), t=tt, y=yy, w=ww,
                   rate=ref.model_eval(m, 0, tt, yy), jac=ref.model_eval(m, 1, tt, yy),
                   vjp=ref.model_eval(m, 2, tt, yy, ww))
        np.savez_compressed(os.path.join(OUT, f"model_{name}.npz"), **rec)
    print("golden fixtures written to", OUT)


if __name__ == "__main__":
    main()
