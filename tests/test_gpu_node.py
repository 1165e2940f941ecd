"""GPU parity of the wide neural ODE (state 8, hidden width 128,
18 824 parameters): forward, adjoint and the outer-product parameter VJP
against the CPU oracle at reduced batch / steps."""
import numpy as np
import pytest

import paper_2310_08649_b200 as P
from paper_2310_08649_b200 import api
from tests.conftest import rel_max, uniform_times

pytestmark = pytest.mark.gpu
TOL = 1e-10


@pytest.mark.parametrize("solver", [(0, 1), (1, 1), (2, 1)])
@pytest.mark.parametrize("nc", [1, 7, 16])
def test_node_wide_128(port, solver, nc):
    nb, nt = 3, 24
    m = P.build_node_wide(8, 128, nb)
    assert m.params.size == 18824
    y0 = np.zeros((nb, 8))
    t = uniform_times(nt, nb, 1.0)
    want = port.gradient(m, y0, t, nc, solver=solver)
    got = api.gradient_adjoint(m, y0, api.TimeGrid(t), nc, solver=api.SolverChoice(*solver))
    assert got.trajectory.work.as_dict() == want.fwd
    assert got.backward_work.as_dict() == want.bwd
    assert rel_max(got.trajectory.states, want.states) <= TOL
    assert abs(got.loss - want.loss) <= TOL * abs(want.loss)
    assert rel_max(got.gradient, want.grad) <= TOL


def test_node_wide_random_start(port):
    nb, nt = 5, 12
    m = P.build_node_wide(8, 128, nb, seed=11)
    y0 = np.random.default_rng(2).uniform(-0.5, 0.5, (nb, 8))
    t = uniform_times(nt, nb, 2.0)
    want = port.gradient(m, y0, t, 4)
    got = api.gradient_adjoint(m, y0, api.TimeGrid(t), 4)
    assert got.trajectory.work.as_dict() == want.fwd
    assert rel_max(got.trajectory.states, want.states) <= TOL
    assert rel_max(got.gradient, want.grad) <= TOL
