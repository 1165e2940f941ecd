"""B200-native chunked backward-Euler integrator + discrete adjoint (arXiv 2310.08649).

Drop-in for the reference `chunkode` backward-Euler path. The compute runs in
hand-written sm_100a CUDA kernels behind the C ABI in include/chunkode_b200.h
(libchunkode_b200.so, built in-tree by __graft_entry__.build()); this package
is the Python mirror of the reference API used by the tests and bench.py.
"""
from . import abi, errors, models  # noqa: F401
from .errors import *  # noqa: F401,F403
from .models import (  # noqa: F401
    Model, build_chaboche, build_constant_rate, build_lin3, build_mass_damper_spring,
    build_neural_ode, build_neuron, build_node_wide, build_problem, build_scalar_decay, linspace,
)
