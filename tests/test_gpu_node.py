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


def test_node_wide_loop_modes_identical(port):
    """The device-driven Newton loop (nested CUDA-graph WHILE nodes) and the host-driven one
    (CKO_NODE_HOST_LOOP=1, another process: the switch is read once) run the same kernels: bitwise identical
    results, both equal to the oracle, with a ragged last chunk."""
    import os
    import subprocess
    import sys
    nb, nt, nc = 4, 30, 8
    m = P.build_node_wide(8, 128, nb)
    y0 = np.zeros((nb, 8))
    t = uniform_times(nt, nb, 1.0)
    want = port.gradient(m, y0, t, nc)
    got = api.gradient_adjoint(m, y0, api.TimeGrid(t), nc)
    assert got.trajectory.work.as_dict() == want.fwd
    assert rel_max(got.trajectory.states, want.states) <= TOL
    assert rel_max(got.gradient, want.grad) <= TOL
    code = ("import numpy as np, paper_2310_08649_b200 as P; from paper_2310_08649_b200 import api; "
            "from tests.conftest import uniform_times; m = P.build_node_wide(8, 128, 4); "
            "r = api.gradient_adjoint(m, np.zeros((4, 8)), api.TimeGrid(uniform_times(30, 4, 1.0)), 8); "
            "np.save('/tmp/cko_host_loop_states.npy', r.trajectory.states)")
    from tests.conftest import ROOT
    subprocess.run([sys.executable, "-c", code], check=True, cwd=ROOT, env=dict(os.environ, CKO_NODE_HOST_LOOP="1"))
    assert np.array_equal(np.load("/tmp/cko_host_loop_states.npy"), got.trajectory.states)


def test_node_wide_long_chunk_and_pivoting(port):
    """n_chunk > 128 (the lane-serial residual kernel) and a large dt whose blocks need row exchanges
    (the pivoting fallback of the thread LU)."""
    nb = 3
    m = P.build_node_wide(8, 128, nb)
    y0 = np.random.default_rng(4).uniform(-1, 1, (nb, 8))
    t = uniform_times(140, nb, 140.0)  # dt = 1: I - dt J far from diagonally dominant
    want = port.gradient(m, y0, t, 140)
    got = api.gradient_adjoint(m, y0, api.TimeGrid(t), 140)
    assert got.trajectory.work.as_dict() == want.fwd
    assert rel_max(got.trajectory.states, want.states) <= TOL
    assert rel_max(got.gradient, want.grad) <= TOL


def test_node_wide_divergence_on_device(port):
    """The iteration cap detected by the device control kernels: same NewtonDivergence payload as the oracle."""
    nb = 3
    m = P.build_node_wide(8, 128, nb)
    y0 = np.random.default_rng(5).uniform(-1, 1, (nb, 8))
    t = uniform_times(20, nb, 20.0)
    st = (1e-15, 1e-15, 1)
    with pytest.raises(P.NewtonDivergence) as want:
        port.gradient(m, y0, t, 5, settings=st)
    with pytest.raises(P.NewtonDivergence) as got:
        api.gradient_adjoint(m, y0, api.TimeGrid(t), 5, settings=api.NewtonSettings(*st))
    assert got.value.chunk_start_step == want.value.chunk_start_step
    assert got.value.batch_index == want.value.batch_index
    assert got.value.iterations == want.value.iterations
