"""The device-buffer training step (cko_gradient_adjoint_device): the Frobenius loss
formed from per-CTA sums of y^2 left by the forward's residual passes (no separate
pass over the trajectory) and, for the Thomas / PCR generation-2 kernels, inside the
adjoint kernel. Parity against the oracle (adjoint.cpp:299-313) on every kernel
family the path can take: v2 Thomas, the n <= 8 and n = 20 PCR kernels, the generic
kernels (loss pass), the wide neural ODE (its own path)."""
import numpy as np
import pytest

import paper_2310_08649_b200 as P
from paper_2310_08649_b200 import api
from tests.conftest import rel_max, uniform_times

pytestmark = pytest.mark.gpu
TOL = 1e-10

CASES = [
    ("mds20-thomas", lambda nb: P.build_mass_damper_spring(10, nb), 37, 250, 100, (0, 1)),
    ("mds20-pcr", lambda nb: P.build_mass_damper_spring(10, nb), 9, 120, 16, (1, 1)),
    ("mds20-hybrid", lambda nb: P.build_mass_damper_spring(10, nb), 5, 64, 32, (2, 2)),
    ("mds4-pcr", lambda nb: P.build_mass_damper_spring(2, nb), 21, 300, 64, (1, 1)),
    ("chaboche-thomas", lambda nb: P.build_chaboche(3, nb), 7, 400, 50, (0, 1)),
    ("chaboche-pcr", lambda nb: P.build_chaboche(3, nb), 7, 400, 64, (1, 1)),
    ("lin3-thomas", lambda nb: P.build_lin3(nb), 4, 60, 7, (0, 1)),
    ("node-wide", lambda nb: P.build_node_wide(8, 128, nb), 3, 24, 8, (0, 1)),
]


@pytest.mark.parametrize("name,build,nb,nt,nc,solver", CASES, ids=[c[0] for c in CASES])
def test_gradient_adjoint_device(port, name, build, nb, nt, nc, solver):
    import torch
    m = build(nb)
    y0 = np.random.default_rng(3).uniform(-0.1, 0.1, (nb, m.state_size)) if name.startswith("mds") else \
        np.zeros((nb, m.state_size))
    t = uniform_times(nt, nb, 0.01 if name.startswith("mds") else 1.0)
    want = port.gradient(m, y0, t, nc, solver=solver)
    ctx = api.default_context()
    d_y0 = torch.from_numpy(y0).cuda()
    d_t = torch.from_numpy(t).cuda()
    for _ in range(2):  # a second call reuses the workspace (the partials are per call)
        loss, grad, d_states, wf, wb = api.gradient_adjoint_device(m, d_y0, d_t, nc, api.SolverChoice(*solver),
                                                                   ctx=ctx)
        assert wf.as_dict() == want.fwd
        assert wb.as_dict() == want.bwd
        assert rel_max(d_states.cpu().numpy(), want.states) <= TOL
        assert abs(loss - want.loss) <= TOL * abs(want.loss)
        assert rel_max(grad, want.grad) <= TOL
    # the host-buffer call agrees with the device one to rounding
    got = api.gradient_adjoint(m, y0, api.TimeGrid(t), nc, solver=api.SolverChoice(*solver), ctx=ctx)
    assert abs(got.loss - loss) <= 1e-13 * abs(loss)
    assert rel_max(got.gradient, grad) <= 1e-12


def test_adjoint_after_forward_does_not_reuse_partials(port):
    """A separate adjoint call over a trajectory (possibly modified since the forward) computes its own loss."""
    nb, nt, nc = 11, 200, 100
    m = P.build_mass_damper_spring(10, nb)
    y0 = np.random.default_rng(9).uniform(-0.1, 0.1, (nb, 20))
    t = uniform_times(nt, nb, 0.01)
    ctx = api.default_context()
    tr = api.integrate_backward_euler(m, y0, api.TimeGrid(t), nc, ctx=ctx)
    states = tr.states * 2.0  # not the forward's trajectory any more
    want_L = float(np.sqrt(np.sum(states[1:] ** 2)))
    L, g = api.adjoint_backward(m, api.Trajectory(states, tr.grid, nb, 20, tr.work), nc, ctx=ctx)
    assert abs(L - want_L) <= 1e-12 * want_L


STREAM_CASES = [
    ("mds20-thomas", lambda nb: P.build_mass_damper_spring(10, nb), 37, 1000, 50, (0, 1)),
    ("mds20-thomas-ragged", lambda nb: P.build_mass_damper_spring(10, nb), 13, 1003, 100, (0, 1)),
    ("mds4-pcr", lambda nb: P.build_mass_damper_spring(2, nb), 21, 2000, 64, (1, 1)),
    ("chaboche-thomas", lambda nb: P.build_chaboche(3, nb), 5, 2000, 100, (0, 1)),
]


@pytest.mark.parametrize("name,build,nb,nt,nc,solver", STREAM_CASES, ids=[c[0] for c in STREAM_CASES])
def test_streamed_grid(port, name, build, nb, nt, nc, solver):
    """gradient_adjoint with host buffers streams the time grid in pieces while the forward runs (the
    generation-2 kernels wait per chunk for their rows): same results as the oracle, odd batch widths
    included (piece boundaries on 128-byte lines)."""
    m = build(nb)
    y0 = np.zeros((nb, m.state_size))
    t = uniform_times(nt, nb, 0.01 if name.startswith("mds") else 2.0)
    want = port.gradient(m, y0, t, nc, solver=solver)
    for _ in range(2):
        got = api.gradient_adjoint(m, y0, api.TimeGrid(t), nc, solver=api.SolverChoice(*solver))
        assert got.trajectory.work.as_dict() == want.fwd
        assert got.backward_work.as_dict() == want.bwd
        assert rel_max(got.trajectory.states, want.states) <= TOL
        assert abs(got.loss - want.loss) <= TOL * abs(want.loss)
        assert rel_max(got.gradient, want.grad) <= TOL


@pytest.mark.parametrize("step", [1, 700, 1000])
def test_streamed_grid_invalid(step):
    """A bad grid found by the host check during the streamed forward: the first offending (step, batch),
    as the device check reports it, and no result (C ABI: the Python TimeGrid would refuse the grid)."""
    import ctypes as C

    from paper_2310_08649_b200 import abi
    from paper_2310_08649_b200._native import lib
    from paper_2310_08649_b200.errors import raise_for
    nb, nt, nc = 9, 1000, 50
    m = P.build_mass_damper_spring(10, nb)
    t = uniform_times(nt, nb, 0.01)
    t[step, 4] = t[step - 1, 4]
    t[min(step + 3, nt), 5] = -1.0  # a later (or same-step, higher-batch) fault: not the first
    ctx = api.Context(0)
    st, sv, w, w2, e = api.NewtonSettings().c(), api.SolverChoice().c(), abi.CkoWork(), abi.CkoWork(), abi.CkoError()
    dp = lambda a: a.ctypes.data_as(C.POINTER(C.c_double))
    y0 = np.zeros((nb, 20))
    loss, grad = C.c_double(), np.zeros(m.params.size)
    rc = lib().cko_gradient_adjoint(ctx.h, ctx.model(m), dp(y0), dp(t), nb, nt, nc, C.byref(st), C.byref(sv), None,
                                    C.byref(loss), dp(grad), C.byref(w), C.byref(w2), C.byref(e))
    assert rc == abi.CKO_INVALID_TIME_GRID
    with pytest.raises(P.InvalidTimeGrid, match=rf"step {step}, batch 4"):
        raise_for(rc, e)
    # the context stays usable
    r = api.gradient_adjoint(m, y0, api.TimeGrid(uniform_times(nt, nb, 0.01)), nc, ctx=ctx)
    assert np.isfinite(r.loss)
