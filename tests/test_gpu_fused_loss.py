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
