"""Public single-chunk ops on the GPU against the COMPILED REFERENCE's own
functions (oracle/_ref): chunk_residual / chunk_jacobian / newton_solve_chunk (integrate.cpp:269-319),
adjoint_chunk_solve / adjoint_step_sequential (adjoint.cpp:223-261), plus the reference's own
chunked-reverse == sequential-reverse law (test_adjoint.cpp:130-180) replayed on the device."""
import numpy as np
import pytest

import paper_2310_08649_b200 as P
from paper_2310_08649_b200 import api
from tests.cases import case, chaboche_plastic
from tests.conftest import rel_max, uniform_times

pytestmark = pytest.mark.gpu
TOL = 1e-10
CASES = ["lin3", "mds", "chaboche", "node", "node_wide", "scalar"]


def chunk_inputs(name, c=6, seed=3):
    m, y0, t, _ = case(name)
    nb, n = y0.shape
    rng = np.random.default_rng(seed)
    y_start = y0 + 0.01 * rng.uniform(-1, 1, y0.shape)
    dy = 0.01 * rng.uniform(-1, 1, (c, nb, n))
    t_chunk = t[1:c + 1].copy()
    dt_chunk = (t[1:c + 1] - t[:c]) * rng.uniform(0.5, 1.5, (c, nb))  # independent of t_chunk on purpose
    return m, y_start, dy, t_chunk, dt_chunk


@pytest.mark.parametrize("name", CASES)
def test_chunk_residual_and_jacobian(ref, name):
    m, ys, dy, tc, dtc = chunk_inputs(name)
    r = api.chunk_residual(m, ys, dy, tc, dtc)
    assert rel_max(r, ref.chunk_op(m, 0, ys, dy, tc, dtc)) <= 1e-13
    sys = api.chunk_jacobian(m, ys, dy, tc, dtc)
    diag, off = ref.chunk_op(m, 1, ys, dy, tc, dtc)
    assert rel_max(sys.diag, diag) <= 1e-13
    assert np.array_equal(sys.offdiag, off)


@pytest.mark.parametrize("name", CASES)
@pytest.mark.parametrize("solver", [(0, 1), (1, 1), (2, 1)])
def test_newton_solve_chunk(ref, name, solver):
    m, ys, dy, tc, dtc = chunk_inputs(name)
    want_dy, want_it, want_w = ref.chunk_op(m, 2, ys, dy, tc, dtc, solver=solver)
    got = dy.copy()
    w = api.WorkCounters()
    it = api.newton_solve_chunk(m, ys, got, tc, dtc, solver=api.SolverChoice(*solver), work=w)
    assert it == want_it
    assert w.as_dict() == want_w
    assert rel_max(got, want_dy) <= TOL


@pytest.mark.parametrize("name", CASES)
@pytest.mark.parametrize("solver", [(0, 1), (1, 1)])
def test_adjoint_chunk_solve_and_step(ref, name, solver):
    m, y0, t, nc = case(name)
    tr = api.integrate_backward_euler(m, y0, api.TimeGrid(t), nc)
    rng = np.random.default_rng(11)
    dL = rng.uniform(-1, 1, tr.states.shape)
    dL[0] = 0.0
    nb, n = y0.shape
    lam0 = rng.uniform(-1, 1, (nb, n))
    g0 = rng.uniform(-1, 1, m.params.size)
    nt = tr.n_time
    step_hi, clen = nt - 3, min(5, nt - 3)
    st = api.AdjointState(lam0.copy(), g0.copy())
    w = api.WorkCounters()
    api.adjoint_chunk_solve(m, tr, step_hi, clen, dL, st, solver=api.SolverChoice(*solver), work=w)
    lam_r, g_r, w_r = ref.adjoint_chunk(m, 0, tr.states, t, step_hi, clen, dL, lam0, g0, solver)
    assert rel_max(st.lam, lam_r) <= TOL
    assert rel_max(st.grad, g_r) <= TOL
    assert w.as_dict() == w_r
    # one sequential step at step_hi
    st1 = api.AdjointState(lam0.copy(), g0.copy())
    yi, yp = tr.states[step_hi].reshape(nb, n), tr.states[step_hi - 1].reshape(nb, n)
    api.adjoint_step_sequential(m, yi, yp, t[step_hi], t[step_hi - 1], dL[step_hi].reshape(nb, n), st1,
                                solver=api.SolverChoice(*solver))
    lam_s, g_s, _ = ref.adjoint_chunk(m, 1, tr.states[step_hi - 1:step_hi + 1], t[step_hi - 1:step_hi + 1], 1, 1,
                                      dL[step_hi - 1:step_hi + 1], lam0, g0, solver)
    assert rel_max(st1.lam, lam_s) <= TOL
    assert rel_max(st1.grad, g_s) <= TOL


def test_chunked_reverse_equals_sequential():
    """test_adjoint.cpp:130-180 on the device: reversing a chunk in one coupled solve equals stepping it."""
    m = chaboche_plastic(3, 4)
    t = uniform_times(40, 4, 10.0)
    tr = api.integrate_backward_euler(m, np.zeros((4, 5)), api.TimeGrid(t), 8)
    dL = api.loss_frobenius().state_gradient(tr)
    a = api.AdjointState.zeros(m, 4)
    b = api.AdjointState.zeros(m, 4)
    api.adjoint_chunk_solve(m, tr, 40, 10, dL, a)
    for s in range(40, 30, -1):
        api.adjoint_step_sequential(m, tr.states[s].reshape(4, 5), tr.states[s - 1].reshape(4, 5), t[s], t[s - 1],
                                    dL[s].reshape(4, 5), b)
    assert rel_max(a.lam, b.lam) <= 1e-12
    assert rel_max(a.grad, b.grad) <= 1e-12


def test_step_rejects_nonpositive_dt():
    m = P.build_scalar_decay(1.0)
    st = api.AdjointState.zeros(m, 2)
    with pytest.raises(P.ShapeMismatch):
        api.adjoint_step_sequential(m, np.ones((2, 1)), np.ones((2, 1)), np.array([1.0, 1.0]),
                                    np.array([1.0, 0.5]), np.zeros((2, 1)), st)
