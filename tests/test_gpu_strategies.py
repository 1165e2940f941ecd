"""SURVEY §8 row f2 on the GPU: the Neuron device twin and the Jacobian strategies (analytic, forward-mode
dual numbers, central differences) against the COMPILED REFERENCE running the same strategy
(JacobianStrategy, ode_model.hpp:14; jacobian_forward_ad ode_model.hpp:132-151;
jacobian_finite_difference ode_model.cpp:44-66). The Neuron parameter product is forward-mode on both
sides (the model has no analytic VJP)."""
import numpy as np
import pytest

import paper_2310_08649_b200 as P
from paper_2310_08649_b200 import api
from tests.cases import case
from tests.conftest import rel_max, uniform_times

pytestmark = pytest.mark.gpu
TOL = 1e-10


def neuron_case():
    m = P.build_neuron(2, 3)
    return m, np.zeros((3, 8)), uniform_times(60, 3, 10.0), 6


def run_both(ref, m, y0, t, nc, solver, strategy):
    ref.set_jacobian_strategy(strategy)
    try:
        want = ref.gradient(m, y0, t, nc, solver=solver)
    finally:
        ref.set_jacobian_strategy("analytic")
    got = api.gradient_adjoint(m, y0, api.TimeGrid(t), nc, solver=api.SolverChoice(*solver), strategy=strategy)
    return got, want


def check(got, want, tol=TOL):
    assert got.trajectory.work.as_dict() == want.fwd
    assert got.backward_work.as_dict() == want.bwd
    assert rel_max(got.trajectory.states, want.states) <= tol
    assert abs(got.loss - want.loss) <= tol * abs(want.loss)
    assert rel_max(got.gradient, want.grad) <= tol


@pytest.mark.parametrize("solver", [(0, 1), (1, 1), (2, 2)])
def test_neuron_twin(ref, solver):
    m, y0, t, nc = neuron_case()
    got, want = run_both(ref, m, y0, t, nc, solver, "analytic")
    check(got, want)


@pytest.mark.parametrize("name", ["mds", "chaboche", "node", "lin3", "scalar", "neuron"])
@pytest.mark.parametrize("solver", [(0, 1), (1, 1)])
def test_forward_ad_strategy(ref, name, solver):
    m, y0, t, nc = neuron_case() if name == "neuron" else case(name)
    got, want = run_both(ref, m, y0, t, nc, solver, "forward_ad")
    check(got, want)


@pytest.mark.parametrize("name", ["mds", "chaboche", "neuron", "lin3"])
def test_finite_difference_strategy(ref, name):
    m, y0, t, nc = neuron_case() if name == "neuron" else case(name)
    got, want = run_both(ref, m, y0, t, nc, (0, 1), "finite_difference")
    check(got, want, tol=1e-8)  # difference quotients amplify the rate's last-bit differences by ~1/delta


@pytest.mark.parametrize("name", ["mds", "chaboche", "node", "neuron"])
def test_chunk_jacobian_strategies(ref, name):
    """The reference's criterion 5 on the device: forward mode vs analytic to 1e-12, vs differences to 1e-5."""
    m, y0, t, _ = neuron_case() if name == "neuron" else case(name)
    nb, n = y0.shape
    rng = np.random.default_rng(9)
    ys = rng.uniform(-0.5, 0.5, (nb, n))
    dy = np.zeros((3, nb, n))
    tc, dtc = t[1:4], t[1:4] - t[:3]
    an = api.chunk_jacobian(m, ys, dy, tc, dtc).diag
    ad = api.chunk_jacobian(m, ys, dy, tc, dtc, strategy="forward_ad").diag
    fd = api.chunk_jacobian(m, ys, dy, tc, dtc, strategy="finite_difference").diag
    assert np.max(np.abs(ad - an)) <= 1e-12 * max(1.0, np.max(np.abs(an)))
    assert np.max(np.abs(ad - fd)) <= 1e-5 * max(1.0, np.max(np.abs(ad)))
    ref.set_jacobian_strategy("forward_ad")
    try:
        diag_r, _ = ref.chunk_op(m, 1, ys, dy, tc, dtc)
    finally:
        ref.set_jacobian_strategy("analytic")
    assert rel_max(ad, diag_r) <= 1e-13
