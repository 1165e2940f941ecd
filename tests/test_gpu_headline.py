"""GPU parity at the headline shapes, and directly against the reference's goldens.

* C2 (the bench line's workload: MDS, 10 units, n = 20, nb = 1000, Thomas
  n_chunk = 100, dt = 1e-6) on a shortened horizon (nt = 300 and a ragged
  nt = 250) against the C restatement, every state / loss / gradient /
  WorkCounter, with the warp-specialised kernels asserted to be the ones that
  ran;
* C2 at FULL size (nt = 10000) and C3 at full size (nb = 50, nt = 20000,
  sequential Thomas and PCR/256) against summaries of the COMPILED REFERENCE's
  own run (tests/golden/full_c*.npz, oracle/make_golden_full.py): loss,
  gradient, counters, the last trajectory row and per-step checksums;
* every tests/golden/traj_*.npz case straight against the reference's stored
  outputs (no restatement in between).

Bar (BASELINE.json north star): max-norm relative 1e-10 for
states, loss and gradient; Newton counters identical. Per-step checksums
(sums and sums of squares over a 20000-wide row) get 1e-9: a 1e-10 state
error summed over a row.
"""
import os

import numpy as np
import pytest

import paper_2310_08649_b200 as P
from paper_2310_08649_b200 import api
from tests.cases import ALL_CASES, case, chaboche_plastic
from tests.conftest import ROOT, rel_max, uniform_times

pytestmark = pytest.mark.gpu
TOL = 1e-10
TOL_SUM = 1e-9
GOLD = os.path.join(ROOT, "tests", "golden")
KEYS = ["newton_iterations", "rate_evals", "jacobian_evals", "linear_solves", "reduction_sweeps"]


def counters(w):
    return [w.as_dict()[k] for k in KEYS]


@pytest.mark.parametrize("nt", [300, 250])
def test_c2_headline_shape(port, nt):
    nb, nc = 1000, 100
    m = P.build_mass_damper_spring(10, nb)
    y0 = np.zeros((nb, 20))
    t = uniform_times(nt, nb, nt * 1e-6)  # dt of the full C2 grid (t_max = 0.01 over 10000 steps)
    want = port.gradient(m, y0, t, nc)
    ctx = api.Context(0)
    got = api.gradient_adjoint(m, y0, api.TimeGrid(t), nc, ctx=ctx)
    assert ctx.kernel_generation_used() == 2, "the warp-specialised Thomas kernels must run at the headline shape"
    assert got.trajectory.work.as_dict() == want.fwd
    assert got.backward_work.as_dict() == want.bwd
    assert rel_max(got.trajectory.states, want.states) <= TOL
    assert abs(got.loss - want.loss) <= TOL * abs(want.loss)
    assert rel_max(got.gradient, want.grad) <= TOL


def _check_summary(g, prefix, got):
    assert counters(got.trajectory.work) == list(g[prefix + "fwd"]), "forward WorkCounters differ"
    assert counters(got.backward_work) == list(g[prefix + "bwd"]), "backward WorkCounters differ"
    assert abs(got.loss - float(g[prefix + "loss"])) <= TOL * abs(float(g[prefix + "loss"]))
    assert rel_max(got.gradient, g[prefix + "grad"]) <= TOL
    s = got.trajectory.states
    assert rel_max(s[-1], g[prefix + "last_row"]) <= TOL
    assert rel_max(s.sum(axis=1), g[prefix + "row_sum"]) <= TOL_SUM
    assert rel_max((s * s).sum(axis=1), g[prefix + "row_sumsq"]) <= TOL_SUM


def test_c2_full_size_vs_reference():
    g = np.load(os.path.join(GOLD, "full_c2.npz"))
    nb, nt, nc = int(g["nb"]), int(g["nt"]), int(g["n_chunk"])
    m = P.build_mass_damper_spring(int(g["n_unit"]), nb)
    got = api.gradient_adjoint(m, np.zeros((nb, m.state_size)), api.TimeGrid.uniform(nt, nb, float(g["t_max"])), nc)
    _check_summary(g, "thomas_", got)


@pytest.mark.parametrize("prefix,nc,solver", [("seq_", 1, (0, 1)), ("pcr256_", 256, (1, 1))])
def test_c3_full_size_vs_reference(prefix, nc, solver):
    g = np.load(os.path.join(GOLD, "full_c3.npz"))
    nb, nt = int(g["nb"]), int(g["nt"])
    m = chaboche_plastic(int(g["n_unit"]), nb, float(g["eps_scale"]))
    got = api.gradient_adjoint(m, np.zeros((nb, m.state_size)), api.TimeGrid.uniform(nt, nb, float(g["t_max"])), nc,
                               solver=api.SolverChoice(*solver))
    _check_summary(g, prefix, got)


@pytest.mark.parametrize("name", ALL_CASES)
@pytest.mark.parametrize("sname,solver", [("thomas", (0, 1)), ("pcr", (1, 1)), ("hybrid1", (2, 1))])
def test_gpu_vs_reference_golden(name, sname, solver):
    """The CUDA path against the compiled reference's stored outputs (make_golden.py), no restatement."""
    g = np.load(os.path.join(GOLD, f"traj_{name}.npz"))
    m = case(name)[0]
    assert np.array_equal(m.params, g["params"])
    got = api.gradient_adjoint(m, g["y0"], api.TimeGrid(g["times"]), int(g["n_chunk"]),
                               solver=api.SolverChoice(*solver))
    assert counters(got.trajectory.work) == list(g[sname + "_fwd"])
    assert counters(got.backward_work) == list(g[sname + "_bwd"])
    if sname + "_states" in g:
        assert rel_max(got.trajectory.states, g[sname + "_states"]) <= TOL
    assert abs(got.loss - float(g[sname + "_loss"])) <= TOL * abs(float(g[sname + "_loss"]))
    assert rel_max(got.gradient, g[sname + "_grad"]) <= TOL
