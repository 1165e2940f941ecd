"""Forward Euler + its discrete adjoint on the GPU against the COMPILED REFERENCE
(integrate_forward_euler, adjoint_backward(Scheme::forward_euler): integrate.cpp:371-407,
adjoint.cpp:157-188). The reference's own law that FE is bitwise chunk-independent
(test_integrate.cpp:161-172) is replayed on the device."""
import numpy as np
import pytest

import paper_2310_08649_b200 as P
from paper_2310_08649_b200 import api
from tests.cases import case
from tests.conftest import rel_max, uniform_times

pytestmark = pytest.mark.gpu
TOL = 1e-10
FE = api.Scheme.forward_euler


@pytest.mark.parametrize("name", ["lin3", "mds", "chaboche", "node", "node_wide", "scalar", "constant"])
@pytest.mark.parametrize("nc", [1, 7])
def test_fe_parity(ref, name, nc):
    m, y0, t, _ = case(name)
    if name == "lin3":  # explicit Euler is unstable on the stiff 3-state system at this dt: stay short
        t = uniform_times(40, 10, 1e-6 * 40)
    want = ref.fe_gradient(m, y0, t, nc)
    got = api.gradient_adjoint(m, y0, api.TimeGrid(t), nc, scheme=FE)
    assert got.trajectory.work.as_dict() == want.fwd
    assert got.backward_work.as_dict() == want.bwd
    assert rel_max(got.trajectory.states, want.states) <= TOL
    assert abs(got.loss - want.loss) <= TOL * abs(want.loss)
    assert rel_max(got.gradient, want.grad) <= TOL


def test_fe_chunk_independent():
    m, y0, t, _ = case("chaboche")
    a = api.integrate_forward_euler(m, y0, api.TimeGrid(t), 1)
    b = api.integrate_forward_euler(m, y0, api.TimeGrid(t), 13)
    assert np.array_equal(a.states, b.states)


def test_fe_user_loss(ref):
    m, y0, t, _ = case("mds")
    tr = api.integrate_forward_euler(m, y0, api.TimeGrid(t), 4)
    dL = np.random.default_rng(5).uniform(-1, 1, tr.states.shape)
    loss = api.LossSpec(lambda tr: 0.0, lambda tr: dL)
    w = api.WorkCounters()
    _, g = api.adjoint_backward(m, tr, 4, loss, work=w, scheme=FE)
    want = ref.fe_gradient(m, y0, t, 4, dL=dL)
    assert rel_max(g, want.grad) <= TOL
    assert w.as_dict() == want.bwd


def test_fe_nonfinite_names_step():
    m = P.build_scalar_decay(-1e300)  # dy/dt = 1e300 y: overflows on the first steps
    with pytest.raises(P.NonFiniteOutput, match="step"):
        api.integrate_forward_euler(m, np.ones((2, 1)), api.TimeGrid.uniform(10, 2, 10.0))
