"""GPU parity of the structured-record Thomas kernels (cko_sparse.cuh) for the MDS chain.

M = I - dt J is [I B; C D] with diagonal bands B, C and tridiagonal D; the
structured kernels factor only its nonzeros. Whenever the reference's
lu_factor_block (linalg.cpp:13-44) would not exchange rows they must give its
results; any block it would pivot on (or call singular) must make the call
fall back to the group-LU kernels, reported through structured_used(). Every
case is checked against the CPU oracle (max-norm relative 1e-10, identical
WorkCounters) and against the same call with the structured kernels off.
"""
import numpy as np
import pytest

import paper_2310_08649_b200 as P
from paper_2310_08649_b200 import api
from tests.conftest import rel_max, uniform_times

pytestmark = pytest.mark.gpu

TOL = 1e-10
BOTH = api.Context.SP_FWD | api.Context.SP_ADJ


def _ctx(structured=True):
    c = api.Context(0)
    c.set_structured(structured)
    return c


def _check(got, want):
    assert got.trajectory.work.as_dict() == want.fwd, "forward WorkCounters differ"
    assert got.backward_work.as_dict() == want.bwd, "backward WorkCounters differ"
    assert rel_max(got.trajectory.states, want.states) <= TOL
    assert abs(got.loss - want.loss) <= TOL * abs(want.loss)
    assert rel_max(got.gradient, want.grad) <= TOL


def _mds(nu, nb, nt, dt, seed=3):
    m = P.build_mass_damper_spring(nu, nb)
    y0 = np.random.default_rng(seed).uniform(-1e-3, 1e-3, (nb, 2 * nu))
    return m, y0, uniform_times(nt, nb, nt * dt)


@pytest.mark.parametrize("nu", [10, 2])
@pytest.mark.parametrize("nb,nt,nc", [(1, 7, 3), (7, 64, 16), (33, 50, 50), (148, 40, 7), (300, 21, 5),
                                      (1000, 30, 10)])
def test_structured_parity(port, nu, nb, nt, nc):
    m, y0, t = _mds(nu, nb, nt, 1e-6)
    want = port.gradient(m, y0, t, nc)
    ctx = _ctx()
    got = api.gradient_adjoint(m, y0, api.TimeGrid(t), nc, ctx=ctx)
    assert ctx.kernel_generation_used() == 2
    assert ctx.structured_used() == BOTH, "structured kernels did not run (or fell back)"
    _check(got, want)


@pytest.mark.parametrize("nb,nt,nc", [(16, 300, 100), (64, 250, 100), (5000, 6, 3)])
def test_structured_matches_group_lu(port, nb, nt, nc):
    """Structured on / off on the same inputs: same counters, states and gradient to rounding."""
    m, y0, t = _mds(10, nb, nt, 1e-6, seed=nb)
    on, off = _ctx(True), _ctx(False)
    a = api.gradient_adjoint(m, y0, api.TimeGrid(t), nc, ctx=on)
    b = api.gradient_adjoint(m, y0, api.TimeGrid(t), nc, ctx=off)
    assert on.structured_used() == BOTH and off.structured_used() == 0
    assert a.trajectory.work.as_dict() == b.trajectory.work.as_dict()
    assert rel_max(a.trajectory.states, b.trajectory.states) <= 1e-12
    assert rel_max(a.gradient, b.gradient) <= 1e-12
    want = port.gradient(m, y0, t, nc)
    _check(a, want)


@pytest.mark.parametrize("dt", [5e-5, 5e-4])
def test_structured_falls_back_on_pivoting(port, dt):
    """Steps large enough that the reference exchanges rows in the forward blocks (|dt K_u / M_u| > 1 below
    the unit pivots): the forward must fall back. The adjoint's transposed blocks carry those entries in their
    rows, not below a pivot, so it stays structured. Everything must still match."""
    m, y0, t = _mds(10, 9, 40, dt, seed=11)
    want = port.gradient(m, y0, t, 8)
    ctx = _ctx()
    got = api.gradient_adjoint(m, y0, api.TimeGrid(t), 8, ctx=ctx)
    used = ctx.structured_used()
    assert used == api.Context.SP_FWD_FALLBACK | api.Context.SP_ADJ, used
    _check(got, want)


def test_structured_adjoint_falls_back(port):
    """dt > 1: the adjoint's unit pivots are beaten by -dt below them (M^T[NU+c][c]), so the adjoint falls back
    too."""
    m, y0, t = _mds(2, 3, 6, 2.0, seed=4)
    want = port.gradient(m, y0, t, 3)
    ctx = _ctx()
    got = api.gradient_adjoint(m, y0, api.TimeGrid(t), 3, ctx=ctx)
    used = ctx.structured_used()
    assert used == api.Context.SP_FWD_FALLBACK | api.Context.SP_ADJ_FALLBACK, used
    _check(got, want)


def test_structured_cross_lane_masses(port):
    """Alternating light / heavy masses: pivots in the velocity block's tridiagonal part (fallback)."""
    nb, nt = 7, 30
    m = P.build_mass_damper_spring(10, nb)
    p = np.array(m.params)
    p[20:30] = [1e-3 if u % 2 == 0 else 1e-8 for u in range(10)]
    m = m.with_params(p)
    y0 = np.zeros((nb, 20))
    t = uniform_times(nt, nb, nt * 1e-6)
    want = port.gradient(m, y0, t, 6)
    ctx = _ctx()
    got = api.gradient_adjoint(m, y0, api.TimeGrid(t), 6, ctx=ctx)
    assert ctx.structured_used() & api.Context.SP_FWD_FALLBACK
    _check(got, want)


def test_structured_one_lane_pivots(port):
    """Only one lane of many has a step that makes the reference pivot (per-lane time grids): the whole call
    falls back, every lane still matches."""
    nb, nt = 40, 24
    m = P.build_mass_damper_spring(10, nb)
    y0 = np.random.default_rng(2).uniform(-1e-3, 1e-3, (nb, 20))
    t = uniform_times(nt, nb, nt * 1e-6)
    t[:, 17] = np.linspace(0.0, nt * 5e-4, nt + 1)  # lane 17 only
    want = port.gradient(m, y0, t, 6)
    ctx = _ctx()
    got = api.gradient_adjoint(m, y0, api.TimeGrid(t), 6, ctx=ctx)
    assert ctx.structured_used() & api.Context.SP_FWD_FALLBACK
    _check(got, want)


def test_structured_forward_only(port):
    """integrate_backward_euler alone: only the forward bit."""
    m, y0, t = _mds(10, 20, 60, 1e-6, seed=9)
    ctx = _ctx()
    fw = api.integrate_backward_euler(m, y0, api.TimeGrid(t), 12, ctx=ctx)
    assert ctx.structured_used() == api.Context.SP_FWD
    want = port.forward(m, y0, t, 12)
    assert rel_max(fw.states, want.states) <= TOL
    assert fw.work.as_dict() == want.fwd
