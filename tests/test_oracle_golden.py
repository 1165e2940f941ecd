"""Pin the C restatement oracle to the reference's own outputs (CPU).

The golden fixtures in tests/golden were produced by the unmodified
reference sources (oracle/make_golden.py over oracle/_ref). The restatement
must reproduce them: states/loss to 1e-13, gradients to 1e-12 (the MDS
gradient is analytic here vs the reference's Dual8 sweep), WorkCounters
exactly, solver outputs to 1e-12 and sweep counts exactly.
"""
import glob
import os

import numpy as np
import pytest

from paper_2310_08649_b200.models import Model
from tests.conftest import rel_max

GOLD = os.path.join(os.path.dirname(__file__), "golden")
KEYS = ["newton_iterations", "rate_evals", "jacobian_evals", "linear_solves", "reduction_sweeps"]
SOLVERS = {"thomas": (0, 1), "pcr": (1, 1), "hybrid1": (2, 1)}


def load_model(z):
    return Model(int(z["kind"]), np.array(z["params"]), n_unit=int(z["n_unit"]), width=int(z["width"]),
                 n_batch=int(z["n_batch"]))


TRAJ = sorted(glob.glob(os.path.join(GOLD, "traj_*.npz")))


@pytest.mark.parametrize("path", TRAJ, ids=[os.path.basename(p) for p in TRAJ])
@pytest.mark.parametrize("sname", list(SOLVERS))
def test_port_matches_reference_trajectory(port, path, sname):
    z = np.load(path)
    m = load_model(z)
    r = port.gradient(m, z["y0"], z["times"], int(z["n_chunk"]), solver=SOLVERS[sname])
    assert [r.fwd[k] for k in KEYS] == list(z[f"{sname}_fwd"])
    assert [r.bwd[k] for k in KEYS] == list(z[f"{sname}_bwd"])
    if f"{sname}_states" in z:
        assert rel_max(r.states, z[f"{sname}_states"]) <= 1e-13
    L = float(z[f"{sname}_loss"])
    assert abs(r.loss - L) <= 1e-13 * abs(L)
    assert rel_max(r.grad, z[f"{sname}_grad"]) <= 1e-12


def test_port_matches_reference_solvers(port):
    z = np.load(os.path.join(GOLD, "solvers.npz"))
    for i in range(int(z["count"])):
        p = f"s{i}_"
        diag, off, rhs = z[p + "diag"], z[p + "off"], z[p + "rhs"]
        assert rel_max(z[p + "thomas"], z[p + "dense"]) <= 1e-9  # the reference's own bar
        for key, sv in {"thomas": (0, 1), "pcr": (1, 1), "h0": (2, 0), "h2": (2, 2), "h30": (2, 30)}.items():
            x, sw = port.solve(diag, off, rhs, sv)
            assert rel_max(x, z[p + key]) <= 1e-12, (i, key)
            assert sw == int(z[p + key + "_sweeps"]), (i, key)


def expected_sweeps(n):
    """verify.cpp:39-45: sum of exponents of the power-of-two decomposition."""
    return sum(e for e in range(31) if n & (1 << e))


def test_sweep_counts_law(port):
    rng = np.random.default_rng(0)
    for nc in [1, 2, 3, 7, 8, 13, 16, 100, 1000]:
        diag = rng.uniform(-1, 1, (nc, 1, 2, 2)) + 3 * np.eye(2)
        _, sw = port.solve(diag, None, rng.uniform(-1, 1, (nc, 1, 2)), (1, 1))
        assert sw == expected_sweeps(nc)


MODELS = sorted(glob.glob(os.path.join(GOLD, "model_*.npz")))


@pytest.mark.parametrize("path", MODELS, ids=[os.path.basename(p) for p in MODELS])
def test_port_model_kernels(port, path):
    z = np.load(path)
    m = load_model(z)
    assert rel_max(port.model_eval(m, 0, z["t"], z["y"]), z["rate"]) <= 1e-14
    assert rel_max(port.model_eval(m, 1, z["t"], z["y"]), z["jac"]) <= 1e-14
    # MDS: analytic VJP vs the reference Dual8 sweep
    assert rel_max(port.model_eval(m, 2, z["t"], z["y"], z["w"]), z["vjp"]) <= 1e-12


def test_port_matches_reference_live(port, ref):
    """When the compiled reference is present, compare live on a fresh seeded case."""
    from tests.cases import chaboche_plastic
    from tests.conftest import uniform_times
    m = chaboche_plastic(2, 3, scale=7.0)
    t = uniform_times(90, 3, 10.0)
    for sv in [(0, 1), (1, 1), (2, 2)]:
        a = port.gradient(m, np.zeros((3, 4)), t, 11, solver=sv)
        b = ref.gradient(m, np.zeros((3, 4)), t, 11, solver=sv)
        assert a.fwd == b.fwd and a.bwd == b.bwd
        assert rel_max(a.states, b.states) <= 1e-13
        assert rel_max(a.grad, b.grad) <= 1e-12


@pytest.mark.parametrize("prefix,nc,solver", [("seq_", 1, (0, 1)), ("pcr256_", 256, (1, 1))])
def test_port_matches_reference_full_c3(port, prefix, nc, solver):
    """C3 at full size (nb = 50, nt = 20000): the restatement against the reference's own run
    (tests/golden/full_c3.npz), so the GPU's full-size check inherits a pinned chain."""
    from tests.cases import chaboche_plastic
    from tests.conftest import uniform_times
    g = np.load(os.path.join(GOLD, "full_c3.npz"))
    nb, nt = int(g["nb"]), int(g["nt"])
    m = chaboche_plastic(int(g["n_unit"]), nb, float(g["eps_scale"]))
    r = port.gradient(m, np.zeros((nb, m.state_size)), uniform_times(nt, nb, float(g["t_max"])), nc, solver=solver)
    assert [r.fwd[k] for k in KEYS] == list(g[prefix + "fwd"])
    assert [r.bwd[k] for k in KEYS] == list(g[prefix + "bwd"])
    assert abs(r.loss - float(g[prefix + "loss"])) <= 1e-13 * abs(float(g[prefix + "loss"]))
    assert rel_max(r.grad, g[prefix + "grad"]) <= 1e-12
    assert rel_max(r.states[-1], g[prefix + "last_row"]) <= 1e-13
