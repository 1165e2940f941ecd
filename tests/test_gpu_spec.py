"""Initial-iterate edge cases of the generation-2 forward (integrate.cpp:208-231): chunks converged before
any iteration (0 iterations, and the fused Frobenius loss over their rows), lanes at rest beside moving
lanes, and a non-finite initial residual (divergence with 0 iterations)."""
import numpy as np
import pytest

import paper_2310_08649_b200 as P
from paper_2310_08649_b200 import api
from tests.conftest import rel_max, uniform_times

pytestmark = pytest.mark.gpu
TOL = 1e-10


@pytest.mark.parametrize("nb,nt,nc", [(1, 8, 4), (5, 40, 7), (300, 20, 20)])
def test_converged_initial_iterate_undone(port, nb, nt, nc):
    """Zero rate: every chunk is converged at its initial iterate (verify.cpp:363-375): 0 iterations,
    states, loss and gradient as the oracle, through both training-step entry points."""
    import torch
    m = P.build_constant_rate(0.0)
    y0 = np.full((nb, 1), 0.7)
    t = uniform_times(nt, nb, 1.0)
    want = port.gradient(m, y0, t, nc)
    assert want.fwd["newton_iterations"] == 0
    got = api.gradient_adjoint(m, y0, api.TimeGrid(t), nc)
    assert got.trajectory.work.as_dict() == want.fwd
    assert rel_max(got.trajectory.states, want.states) <= TOL
    assert abs(got.loss - want.loss) <= TOL * abs(want.loss)
    assert rel_max(got.gradient, want.grad) <= TOL
    loss, grad, d_states, wf, _ = api.gradient_adjoint_device(m, torch.from_numpy(y0).cuda(),
                                                             torch.from_numpy(t).cuda(), nc)
    assert wf.as_dict() == want.fwd
    assert abs(loss - want.loss) <= TOL * abs(want.loss)
    assert rel_max(grad, want.grad) <= TOL


def test_mixed_chunks(port):
    """Constant rate switched on by the grid: a chunk whose steps are all tiny after others that iterate."""
    m = P.build_scalar_decay(2.5)
    nb, nt, nc = 4, 60, 6
    y0 = np.zeros((nb, 1))
    y0[0, 0] = 1.0  # lanes at rest converge at once, the moving lane needs iterations
    t = uniform_times(nt, nb, 3.0)
    want = port.gradient(m, y0, t, nc)
    got = api.gradient_adjoint(m, y0, api.TimeGrid(t), nc)
    assert got.trajectory.work.as_dict() == want.fwd
    assert rel_max(got.trajectory.states, want.states) <= TOL
    assert rel_max(got.gradient, want.grad) <= TOL


@pytest.mark.parametrize("kind", ["mds", "scalar"])
def test_non_finite_initial_residual(port, kind):
    """A NaN start: the initial residual is not finite, NewtonDivergence with 0 iterations at the chunk."""
    if kind == "mds":
        m, n = P.build_mass_damper_spring(10, 6), 20
    else:
        m, n = P.build_scalar_decay(1.0), 1
    nb = 6 if kind == "mds" else 1
    y0 = np.zeros((nb, n))
    y0[nb - 1, 0] = np.nan
    t = uniform_times(40, nb, 0.01)
    with pytest.raises(P.NewtonDivergence) as want:
        port.gradient(m, y0, t, 10)
    with pytest.raises(P.NewtonDivergence) as got:
        api.gradient_adjoint(m, y0, api.TimeGrid(t), 10)
    assert got.value.chunk_start_step == want.value.chunk_start_step
    assert got.value.iterations == want.value.iterations == 0
