"""ctypes images of the C ABI types in include/chunkode_b200.h.

Pure type definitions: importing this module loads no native code.
"""
from __future__ import annotations

import ctypes as C

CKO_OK = 0
CKO_SHAPE_MISMATCH = 1
CKO_SINGULAR_BLOCK = 2
CKO_NEWTON_DIVERGENCE = 3
CKO_NON_FINITE = 4
CKO_STRATEGY_UNAVAILABLE = 5
CKO_SIZE_GUARD = 6
CKO_INVALID_TIME_GRID = 7
CKO_ERROR = 8
CKO_CUDA = 9
CKO_COMM = 10

CKO_SOLVER_THOMAS = 0
CKO_SOLVER_PCR = 1
CKO_SOLVER_HYBRID = 2

CKO_MODEL_SCALAR_DECAY = 0
CKO_MODEL_CONSTANT_RATE = 1
CKO_MODEL_LIN3 = 2
CKO_MODEL_MDS = 3
CKO_MODEL_CHABOCHE = 4
CKO_MODEL_NODE = 5
CKO_MODEL_NEURON = 6

CKO_JACOBIAN_ANALYTIC = 0
CKO_JACOBIAN_FORWARD_AD = 1
CKO_JACOBIAN_FINITE_DIFFERENCE = 2

CKO_LOSS_FROBENIUS = 0
CKO_LOSS_USER = 1


class CkoError(C.Structure):
    _fields_ = [
        ("code", C.c_int),
        ("chunk_index", C.c_int),
        ("batch_index", C.c_int),
        ("chunk_start_step", C.c_int),
        ("iterations", C.c_int),
        ("residual_norm", C.c_double),
        ("initial_norm", C.c_double),
        ("msg", C.c_char * 256),
    ]


class CkoWork(C.Structure):
    _fields_ = [
        ("newton_iterations", C.c_longlong),
        ("rate_evals", C.c_longlong),
        ("jacobian_evals", C.c_longlong),
        ("linear_solves", C.c_longlong),
        ("reduction_sweeps", C.c_longlong),
    ]


class CkoNewtonSettings(C.Structure):
    _fields_ = [("tol_a", C.c_double), ("tol_r", C.c_double), ("max_iter", C.c_int)]


class CkoSolverChoice(C.Structure):
    _fields_ = [("kind", C.c_int), ("n_switch", C.c_int)]


class CkoModelDesc(C.Structure):
    _fields_ = [
        ("kind", C.c_int),
        ("n_unit", C.c_int),
        ("width", C.c_int),
        ("n_batch_model", C.c_int),
        ("lane_offset", C.c_int),
        ("n_params", C.c_int),
        ("params", C.POINTER(C.c_double)),
    ]


def dptr(a):
    """double* of a C-contiguous float64 numpy array (or None)."""
    if a is None:
        return None
    return a.ctypes.data_as(C.POINTER(C.c_double))
