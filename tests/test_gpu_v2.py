"""GPU parity of the warp-specialised (generation 2) Thomas kernels.

Every case runs through both kernel generations on fresh contexts and both are
checked against the CPU oracle at the north-star bar (max-norm relative 1e-10,
identical WorkCounters). The generation a call actually ran is asserted, so a
silent fallback to the generic kernels fails the test.
"""
import numpy as np
import pytest

import paper_2310_08649_b200 as P
from paper_2310_08649_b200 import api
from tests.cases import ALL_CASES, case, chaboche_plastic
from tests.conftest import rel_max, uniform_times

pytestmark = pytest.mark.gpu

TOL = 1e-10
V2_KINDS = {"lin3", "mds", "mds_small", "chaboche", "scalar", "constant"}


def _ctx(gen):
    c = api.Context(0)
    c.set_kernel_generation(gen)
    return c


def _check(got, want):
    assert got.trajectory.work.as_dict() == want.fwd, "forward WorkCounters differ"
    assert got.backward_work.as_dict() == want.bwd, "backward WorkCounters differ"
    assert rel_max(got.trajectory.states, want.states) <= TOL
    assert abs(got.loss - want.loss) <= TOL * abs(want.loss)
    assert rel_max(got.gradient, want.grad) <= TOL


PCR2_KINDS = {"lin3", "mds_small", "chaboche", "scalar", "constant",  # block size <= 8 (thread per point)
              "mds"}  # n = 20: warp-cooperative sweeps (cko_pcrw.cuh)


@pytest.mark.parametrize("name", ALL_CASES)
@pytest.mark.parametrize("gen", [1, 2])
@pytest.mark.parametrize("solver", [(0, 1), (1, 1), (2, 1), (2, 0), (2, 3)])
def test_generation_parity(port, name, gen, solver):
    m, y0, t, nc = case(name)
    want = port.gradient(m, y0, t, nc, solver=solver)
    ctx = _ctx(gen)
    got = api.gradient_adjoint(m, y0, api.TimeGrid(t), nc, solver=api.SolverChoice(*solver), ctx=ctx)
    _check(got, want)
    kinds = V2_KINDS if solver[0] == 0 else PCR2_KINDS
    expect = 2 if (gen == 2 and name in kinds) else 1
    assert ctx.kernel_generation_used() == expect


@pytest.mark.parametrize("nc", [1, 2, 3, 7, 16, 100, 256, 1000])
@pytest.mark.parametrize("solver", [(1, 1), (2, 2)])
def test_pcr2_chaboche_chunks(port, nc, solver):
    """Sparse-batch C3 shape (reduced): PCR / hybrid over ragged partitions, chunks in shared memory (<= 256
    rows) and in the global workspace (1000 rows)."""
    m = chaboche_plastic(3, 3)
    y0 = np.zeros((3, 5))
    t = uniform_times(1000, 3, 0.5)
    want = port.gradient(m, y0, t, nc, solver=solver)
    ctx = _ctx(2)
    got = api.gradient_adjoint(m, y0, api.TimeGrid(t), nc, solver=api.SolverChoice(*solver), ctx=ctx)
    assert ctx.kernel_generation_used() == 2
    _check(got, want)


@pytest.mark.parametrize("nb", [1, 7, 148, 149, 300, 1500])
@pytest.mark.parametrize("nc", [1, 3, 16, 64])
def test_mds_lane_tiles(port, nb, nc):
    """MDS n=20 across lane counts: < 1 lane per CTA, several lanes, more lanes than one tile (1500)."""
    m = P.build_mass_damper_spring(10, nb)
    nt = 64 if nb <= 300 else 24
    y0 = np.zeros((nb, 20))
    t = uniform_times(nt, nb, nt * 1e-6)
    want = port.gradient(m, y0, t, nc)
    ctx = _ctx(2)
    got = api.gradient_adjoint(m, y0, api.TimeGrid(t), nc, ctx=ctx)
    assert ctx.kernel_generation_used() == 2
    _check(got, want)


@pytest.mark.parametrize("nc", [1, 2, 5, 16, 130])
def test_chaboche_plastic_v2(port, nc):
    """Nonlinear Newton (1.5-11 iterations per chunk) through the generation-2 kernels."""
    m = chaboche_plastic(3, 6)
    y0 = np.zeros((6, 5))
    t = uniform_times(130, 6, 10.0)
    want = port.gradient(m, y0, t, nc)
    ctx = _ctx(2)
    got = api.gradient_adjoint(m, y0, api.TimeGrid(t), nc, ctx=ctx)
    assert ctx.kernel_generation_used() == 2
    _check(got, want)


def test_mds_nonzero_start(port):
    """Random initial state: every LU pivot path of the 20 x 20 blocks is exercised."""
    nb = 9
    m = P.build_mass_damper_spring(10, nb)
    rng = np.random.default_rng(5)
    y0 = rng.uniform(-1e-3, 1e-3, (nb, 20))
    t = uniform_times(50, nb, 5e-4)
    want = port.gradient(m, y0, t, 10)
    got = api.gradient_adjoint(m, y0, api.TimeGrid(t), 10, ctx=_ctx(2))
    _check(got, want)


def test_v2_divergence_payload(port):
    m = chaboche_plastic(3, 4)
    y0 = np.zeros((4, 5))
    t = uniform_times(60, 4, 10.0)
    with pytest.raises(P.NewtonDivergence) as want:
        port.forward(m, y0, t, 30, settings=(1e-14, 1e-16, 1))
    ctx = _ctx(2)
    with pytest.raises(P.NewtonDivergence) as got:
        api.integrate_backward_euler(m, y0, api.TimeGrid(t), 30, api.NewtonSettings(1e-14, 1e-16, 1), ctx=ctx)
    g, w = got.value, want.value
    assert (g.chunk_start_step, g.batch_index, g.iterations) == (w.chunk_start_step, w.batch_index, w.iterations)


@pytest.mark.parametrize("k", [-40, -9, -3, -1, 0, 1, 3, 9, 40])
def test_singularity_threshold_band(port, k):
    """Pivots straddling 1e-14 max|M| within the 2^-18 band where the kernels' high-word maximum defers to the
    exact test: M = I - dt A upper triangular (no elimination rounding), max|M| = |m_01| with low-word bits set,
    pivot m_22 = tiny (1 + k 2^-30). Singular or not, and where, must match the oracle."""
    m01 = 1e6 * (1.0 + 2.0 ** -40)
    tiny = 1e-14 * m01
    a22 = 1.0 - tiny * (1.0 + k * 2.0 ** -30)  # dt = 1: m_22 = 1 - a22 (exact, Sterbenz)
    p = np.array([0.0, -m01, 0.0, 0.0, 0.0, 0.0, 0.0, 0.0, a22, 1.0])
    nb, nt = 3, 6
    m = P.build_lin3(nb).with_params(p)
    y0 = np.zeros((nb, 3))
    t = uniform_times(nt, nb, float(nt))
    try:
        want = port.forward(m, y0, t, 2)
        werr = None
    except P.SingularBlock as e:
        want, werr = None, e
    ctx = _ctx(2)
    if werr is not None:
        with pytest.raises(P.SingularBlock) as got:
            api.integrate_backward_euler(m, y0, api.TimeGrid(t), 2, ctx=ctx)
        assert (got.value.chunk_index, got.value.batch_index) == (werr.chunk_index, werr.batch_index)
    else:
        got = api.integrate_backward_euler(m, y0, api.TimeGrid(t), 2, ctx=ctx)
        assert rel_max(got.states, want.states) <= TOL
    assert ctx.kernel_generation_used() == 2


@pytest.mark.parametrize("dt", [5e-6, 5e-5, 5e-4])
def test_mds_pivot_heavy(port, dt):
    """Larger steps: the reference's partial pivoting exchanges rows in most columns of the forward blocks
    (same-lane and cross-lane pairs of the 10-lane groups) — factors, pivots and parity must hold."""
    nb, nt = 9, 40
    m = P.build_mass_damper_spring(10, nb)
    rng = np.random.default_rng(11)
    y0 = rng.uniform(-1e-3, 1e-3, (nb, 20))
    t = uniform_times(nt, nb, nt * dt)
    want = port.gradient(m, y0, t, 8)
    ctx = _ctx(2)
    got = api.gradient_adjoint(m, y0, api.TimeGrid(t), 8, ctx=ctx)
    assert ctx.kernel_generation_used() == 2
    _check(got, want)


def test_mds_cross_lane_exchanges(port):
    """Alternating light / heavy masses: the pivot of column u is the velocity row of the NEXT unit, held by
    another lane of the 10-lane group (cross-lane row exchange)."""
    nb, nt = 7, 30
    m = P.build_mass_damper_spring(10, nb)
    p = np.array(m.params)
    p[20:30] = [1e-3 if u % 2 == 0 else 1e-8 for u in range(10)]  # M_u
    m = m.with_params(p)
    y0 = np.zeros((nb, 20))
    t = uniform_times(nt, nb, nt * 1e-6)
    want = port.gradient(m, y0, t, 6)
    ctx = _ctx(2)
    got = api.gradient_adjoint(m, y0, api.TimeGrid(t), 6, ctx=ctx)
    assert ctx.kernel_generation_used() == 2
    _check(got, want)


@pytest.mark.parametrize("nb,nt,nc", [(5000, 6, 3), (25000, 4, 4)])
def test_mds_wide_ctas(port, nb, nt, nc):
    """More lanes per CTA than one tile (nb = 5000: 2 lane tiles per CTA) and than the residual staging
    holds at once (nb = 25000: ~169 lanes per CTA, staged in lane tiles)."""
    m = P.build_mass_damper_spring(10, nb)
    y0 = np.random.default_rng(nb).uniform(-1e-3, 1e-3, (nb, 20))
    t = uniform_times(nt, nb, nt * 1e-6)
    want = port.gradient(m, y0, t, nc)
    assert want.loss > 0.0
    ctx = _ctx(2)
    got = api.gradient_adjoint(m, y0, api.TimeGrid(t), nc, ctx=ctx)
    assert ctx.kernel_generation_used() == 2
    _check(got, want)


@pytest.mark.parametrize("nc", [1, 2, 3, 5, 16, 33, 100, 128])
@pytest.mark.parametrize("solver", [(1, 1), (2, 1), (2, 3), (2, 0)])
def test_pcrw_mds20_chunks(port, nc, solver):
    """North-star block size (MDS, n = 20) under PCR / hybrid on the warp-cooperative generation-2 kernels:
    power-of-two and ragged partitions (100 = 64 + 32 + 4, 33 = 32 + 1), lanes below and above the CTA count."""
    for nb in (3, 200):
        m = P.build_mass_damper_spring(10, nb)
        y0 = np.zeros((nb, 20))
        t = uniform_times(256, nb, 256 * 1e-6)
        want = port.gradient(m, y0, t, nc, solver=solver)
        ctx = _ctx(2)
        got = api.gradient_adjoint(m, y0, api.TimeGrid(t), nc, solver=api.SolverChoice(*solver), ctx=ctx)
        _check(got, want)
        assert ctx.kernel_generation_used() == 2
