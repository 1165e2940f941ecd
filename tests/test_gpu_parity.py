"""GPU parity: the sm_100a path through the C ABI vs the CPU oracle.

Bar (BASELINE.json north star): states, loss and gradient within
max-norm relative 1e-10; forward and backward WorkCounters identical (so the
Newton iteration counts match exactly).
"""
import numpy as np
import pytest

import paper_2310_08649_b200 as P
from paper_2310_08649_b200 import api
from tests.cases import ALL_CASES, case, chaboche_plastic
from tests.conftest import rel_max, uniform_times

pytestmark = pytest.mark.gpu

TOL = 1e-10
SOLVERS = [(0, 1), (1, 1), (2, 1), (2, 0), (2, 3)]


def run_gpu(m, y0, t, nc, solver, settings=(1e-8, 1e-6, 100)):
    return api.gradient_adjoint(m, y0, api.TimeGrid(t), nc, solver=api.SolverChoice(*solver),
                                settings=api.NewtonSettings(*settings))


@pytest.mark.parametrize("name", ALL_CASES)
@pytest.mark.parametrize("solver", SOLVERS)
def test_forward_adjoint_parity(port, name, solver):
    m, y0, t, nc = case(name)
    want = port.gradient(m, y0, t, nc, solver=solver)
    got = run_gpu(m, y0, t, nc, solver)
    assert got.trajectory.work.as_dict() == want.fwd, "forward WorkCounters differ"
    assert got.backward_work.as_dict() == want.bwd, "backward WorkCounters differ"
    assert rel_max(got.trajectory.states, want.states) <= TOL
    assert abs(got.loss - want.loss) <= TOL * abs(want.loss)
    assert rel_max(got.gradient, want.grad) <= TOL


@pytest.mark.parametrize("nc", [1, 2, 3, 5, 7, 8, 13, 16, 33, 64])
@pytest.mark.parametrize("solver", [(0, 1), (1, 1), (2, 2)])
def test_chunk_sweep_chaboche(port, nc, solver):
    """Nonlinear case across power-of-two and ragged chunk lengths (partitions 7 = 4+2+1 ...)."""
    m = chaboche_plastic(3, 4)
    y0 = np.zeros((4, 5))
    t = uniform_times(130, 4, 10.0)
    want = port.gradient(m, y0, t, nc, solver=solver)
    got = run_gpu(m, y0, t, nc, solver)
    assert got.trajectory.work.as_dict() == want.fwd
    assert rel_max(got.trajectory.states, want.states) <= TOL
    assert rel_max(got.gradient, want.grad) <= TOL


def test_mds_sequential_edge(port):
    """nc = 1 on MDS: early steps converge at iteration 0 (|r0| <= tol_a, SURVEY §7 hard parts)."""
    m = P.build_mass_damper_spring(10, 16)
    y0 = np.zeros((16, 20))
    t = uniform_times(300, 16, 3e-4)  # dt = 1e-6 as in C2 (nt = 10000, t_max = 0.01)
    want = port.gradient(m, y0, t, 1)
    got = run_gpu(m, y0, t, 1, (0, 1))
    assert got.trajectory.work.as_dict() == want.fwd
    assert want.fwd["newton_iterations"] < 300  # some chunks took zero iterations
    assert rel_max(got.trajectory.states, want.states) <= TOL
    assert rel_max(got.gradient, want.grad) <= TOL


@pytest.mark.parametrize("nb", [1, 2, 37, 149, 300])
def test_lane_partitions(port, nb):
    """Lane counts below, at and above the CTA count (uneven lane ranges per CTA)."""
    m = chaboche_plastic(2, nb)
    y0 = np.zeros((nb, 4))
    t = uniform_times(40, nb, 10.0)
    for solver in [(0, 1), (1, 1)]:
        want = port.gradient(m, y0, t, 8, solver=solver)
        got = run_gpu(m, y0, t, 8, solver)
        assert got.trajectory.work.as_dict() == want.fwd
        assert rel_max(got.trajectory.states, want.states) <= TOL
        assert rel_max(got.gradient, want.grad) <= TOL


@pytest.mark.parametrize("nc", [1, 2, 3, 5, 7, 8, 13, 16, 31, 32, 33])
@pytest.mark.parametrize("n", [1, 3, 5])
@pytest.mark.parametrize("nb", [1, 3])
def test_solver_general_offdiag(port, nc, n, nb):
    """Standalone solvers on random diagonally dominant systems (verify.cpp:413-433 fixture)."""
    rng = np.random.default_rng(1000 * nc + 10 * n + nb)
    diag = rng.uniform(-1, 1, (nc, nb, n, n)) + (n + 1.0) * np.eye(n)
    off = 0.5 * rng.uniform(-1, 1, (max(nc - 1, 0), nb, n, n))
    rhs = rng.uniform(-1, 1, (nc, nb, n))
    sys = api.BlockBidiagonalSystem(diag, off)
    for solver in [(0, 1), (1, 1), (2, 0), (2, 1), (2, 3)]:
        want, wsw = port.solve(diag, off, rhs, solver)
        got, gsw = api._solve(diag, off, rhs, api.SolverChoice(*solver), False, None)
        assert gsw == wsw
        assert rel_max(got, want) <= 1e-12
    x = api.solve_thomas(sys, rhs)
    assert rel_max(x, port.solve(diag, off, rhs, (0, 1))[0]) <= 1e-12


@pytest.mark.parametrize("nc", [1, 4, 6, 9])
def test_solver_unit_offdiag(port, nc):
    rng = np.random.default_rng(nc)
    n, nb = 4, 5
    diag = rng.uniform(-1, 1, (nc, nb, n, n)) + (n + 1.0) * np.eye(n)
    rhs = rng.uniform(-1, 1, (nc, nb, n))
    for solver in [(0, 1), (1, 1), (2, 1)]:
        want, wsw = port.solve(diag, None, rhs, solver)
        got, gsw = api.solve_unit_offdiag(diag, rhs, api.SolverChoice(*solver))
        assert gsw == wsw
        assert rel_max(got, want) <= 1e-12


def test_singular_block_location(port):
    """SingularBlock carries the chunk row and lane of the first singular block (test_linalg.cpp:120-131)."""
    nc, nb, n = 4, 3, 2
    diag = np.tile(np.eye(n), (nc, nb, 1, 1))
    diag[2, 1] = 0.0
    off = np.zeros((nc - 1, nb, n, n))
    rhs = np.ones((nc, nb, n))
    with pytest.raises(P.SingularBlock) as ei:
        api.solve_thomas(api.BlockBidiagonalSystem(diag, off), rhs)
    assert (ei.value.chunk_index, ei.value.batch_index) == (2, 1)


def test_newton_divergence_matches_oracle(port):
    """max_iter exhaustion: same exception payload as the oracle (integrate.cpp:247-254)."""
    m = chaboche_plastic(3, 4)
    y0 = np.zeros((4, 5))
    t = uniform_times(60, 4, 10.0)
    with pytest.raises(P.NewtonDivergence) as want:
        port.forward(m, y0, t, 30, settings=(1e-14, 1e-16, 1))
    with pytest.raises(P.NewtonDivergence) as got:
        api.integrate_backward_euler(m, y0, api.TimeGrid(t), 30, api.NewtonSettings(1e-14, 1e-16, 1))
    g, w = got.value, want.value
    assert (g.chunk_start_step, g.batch_index, g.iterations) == (w.chunk_start_step, w.batch_index, w.iterations)
    assert abs(g.residual_norm - w.residual_norm) <= 1e-10 * abs(w.residual_norm)


def test_divergence_nonfinite(port):
    """MDS at the paper horizon overflows: NewtonDivergence with a non-finite norm."""
    m = P.build_mass_damper_spring(10, 2)
    t = uniform_times(10000, 2, 1.0)
    with pytest.raises(P.NewtonDivergence) as want:
        port.forward(m, np.zeros((2, 20)), t, 100)
    with pytest.raises(P.NewtonDivergence) as got:
        api.integrate_backward_euler(m, np.zeros((2, 20)), api.TimeGrid(t), 100)
    assert got.value.chunk_start_step == want.value.chunk_start_step
    assert got.value.batch_index == want.value.batch_index


def test_user_loss_and_adjoint_host(port):
    m, y0, t, nc = case("mds_small")
    f = port.forward(m, y0, t, nc)
    rng = np.random.default_rng(3)
    dL = rng.uniform(-1, 1, f.states.shape)
    dL[0] = 0.0
    want = port.adjoint(m, f.states, t, nc, dL=dL)
    tr = api.Trajectory(f.states, api.TimeGrid(t), y0.shape[0], m.state_size)
    spec = api.LossSpec(lambda tr: 0.0, lambda tr: dL)
    bw = api.WorkCounters()
    _, g = api.adjoint_backward(m, tr, nc, spec, work=bw)
    assert rel_max(g, want.grad) <= TOL
    assert bw.as_dict() == want.bwd


def test_closed_form_scalar_decay():
    """y_1 = y_0 / (1 + p dt) to 1e-14 (test_integrate.cpp:99-113, acceptance.cpp:95-103)."""
    m = P.build_scalar_decay(2.5)
    tr = api.integrate_backward_euler(m, np.full((1, 1), 1.3), api.TimeGrid.uniform(1, 1, 0.1), 1)
    ref = 1.3 / (1.0 + 2.5 * 0.1)
    assert abs(tr.states[1, 0] - ref) <= 1e-14 * abs(ref)


def test_constant_rate_gradient_is_span():
    """dL/dp = T for L = y_N and dy/dt = p (test_adjoint.cpp:79-98)."""
    m = P.build_constant_rate(0.7)
    grid = api.TimeGrid.uniform(16, 1, 2.0)
    tr = api.integrate_backward_euler(m, np.zeros((1, 1)), grid, 4)

    def dL(tr):
        g = np.zeros_like(tr.states)
        g[-1] = 1.0
        return g
    _, g = api.adjoint_backward(m, tr, 4, api.LossSpec(lambda tr: tr.states[-1, 0], dL))
    assert abs(g[0] - 2.0) <= 1e-12


def test_zero_rate_converges_without_iterations():
    """Zero rate: converged before the first iteration (verify.cpp:363-375)."""
    m = P.build_constant_rate(0.0)
    tr = api.integrate_backward_euler(m, np.full((1, 1), 0.7), api.TimeGrid.uniform(8, 1, 1.0), 4)
    assert tr.work.newton_iterations == 0
    assert tr.states[8, 0] == 0.7


def test_linear_counter_laws():
    """One iteration per chunk; solves == iterations; rate evals = iterations + chunks (verify.cpp:377-390)."""
    m = P.build_scalar_decay(1.0)
    tr = api.integrate_backward_euler(m, np.ones((1, 1)), api.TimeGrid.uniform(4, 1, 1.0), 2)
    assert tr.work.newton_iterations == 2
    assert tr.work.linear_solves == tr.work.newton_iterations
    assert tr.work.rate_evals == tr.work.newton_iterations + 2


@pytest.mark.parametrize("entry", ["forward", "gradient"])
def test_time_grid_checked_on_device(entry):
    """The C ABI validates host grids after the copy (time_grid.cpp:7-19) and names the first non-increasing
    entry in the reference's scan order; the Python TimeGrid never gets here, so call the ABI directly."""
    import ctypes as C

    from paper_2310_08649_b200 import abi
    from paper_2310_08649_b200._native import lib
    from paper_2310_08649_b200.errors import raise_for

    nb, nt, n = 5, 40, 3
    m = P.build_lin3(nb)
    t = uniform_times(nt, nb, 1.0)
    t[17, 3] = t[16, 3]  # first violation in (step, lane) order ...
    t[30, 1] = t[29, 1] - 1.0  # ... not this later one
    t = np.ascontiguousarray(t)
    y0 = np.zeros((nb, n))
    ctx = api.Context(0)
    st, sv, w, w2, e = api.NewtonSettings().c(), api.SolverChoice().c(), abi.CkoWork(), abi.CkoWork(), abi.CkoError()
    dp = lambda a: a.ctypes.data_as(C.POINTER(C.c_double))
    states = np.zeros((nt + 1, nb * n))
    if entry == "forward":
        rc = lib().cko_be_forward(ctx.h, ctx.model(m), dp(y0), dp(t), nb, nt, 4, C.byref(st), C.byref(sv), dp(states),
                                  None, C.byref(w), C.byref(e))
    else:
        loss, grad = C.c_double(), np.zeros(m.params.size)
        rc = lib().cko_gradient_adjoint(ctx.h, ctx.model(m), dp(y0), dp(t), nb, nt, 4, C.byref(st), C.byref(sv),
                                        None, C.byref(loss), dp(grad), C.byref(w), C.byref(w2), C.byref(e))
    assert rc == abi.CKO_INVALID_TIME_GRID
    with pytest.raises(P.InvalidTimeGrid, match=r"step 17, batch 3"):
        raise_for(rc, e)
