"""Shared model/problem cases for the parity tests (small sizes the CPU oracle finishes in seconds)."""
import numpy as np

import paper_2310_08649_b200 as P
from tests.conftest import uniform_times


def chaboche_plastic(n_unit, nb, scale=10.0):
    """Chaboche with eps_a scaled x10 so Newton leaves the elastic regime."""
    m = P.build_chaboche(n_unit, nb)
    p = m.params.copy()
    o = 6 + 2 * n_unit
    p[o:o + nb] *= scale
    return m.with_params(p)


def case(name):
    """(model, y0, times, default n_chunk) for a named case."""
    if name == "lin3":          # config C1 at full size
        m = P.build_lin3(10)
        return m, np.ones((10, 3)), uniform_times(1000, 10, 1.0), 10
    if name == "mds":           # config C2 shape, reduced batch / steps
        m = P.build_mass_damper_spring(10, 8)
        return m, np.zeros((8, 20)), uniform_times(200, 8, 0.01), 10
    if name == "mds_small":
        m = P.build_mass_damper_spring(2, 3)
        return m, np.zeros((3, 4)), uniform_times(64, 3, 2e-4), 8
    if name == "chaboche":      # config C3 shape, reduced
        m = chaboche_plastic(3, 5)
        return m, np.zeros((5, 5)), uniform_times(400, 5, 10.0), 16
    if name == "node":          # reference neural ODE (width n+1)
        m = P.build_neural_ode(4, 3)
        return m, np.zeros((3, 4)), uniform_times(100, 3, 1.0), 7
    if name == "node_wide":     # config C4 family, small width
        m = P.build_node_wide(3, 16, 3)
        return m, np.zeros((3, 3)), uniform_times(50, 3, 1.0), 8
    if name == "scalar":
        m = P.build_scalar_decay(2.5)
        return m, np.full((2, 1), 1.3), uniform_times(20, 2, 1.0), 4
    if name == "constant":
        m = P.build_constant_rate(0.7)
        return m, np.full((2, 1), 0.3), uniform_times(12, 2, 1.0), 5
    raise KeyError(name)


ALL_CASES = ["lin3", "mds", "mds_small", "chaboche", "node", "node_wide", "scalar", "constant"]
