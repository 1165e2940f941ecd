"""Loader for the in-tree CUDA library libchunkode_b200.so.

There is no CPU fallback: if the library is missing or no CUDA device is
usable, every entry point raises. The library is built in-tree by
__graft_entry__.build() (make -C paper_2310_08649_b200/csrc).
"""
from __future__ import annotations

import ctypes as C
import os

from . import abi

HERE = os.path.dirname(os.path.abspath(__file__))
# CKO_LIB_PATH: an alternative build of the same library (kernel A/B experiments, scripts/build_variant.sh)
LIB_PATH = os.environ.get("CKO_LIB_PATH") or os.path.join(HERE, "libchunkode_b200.so")

_lib = None


class NativeLibraryMissing(RuntimeError):
    pass


def lib() -> C.CDLL:
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise NativeLibraryMissing(
            f"{LIB_PATH} not built; run `python -c 'import __graft_entry__ as g; g.build()'` "
            "(the B200 path has no CPU fallback)")
    L = C.CDLL(LIB_PATH)
    P, vp = C.POINTER, C.c_void_p
    E, W, S, N, D = abi.CkoError, abi.CkoWork, abi.CkoSolverChoice, abi.CkoNewtonSettings, abi.CkoModelDesc
    dp = P(C.c_double)
    sig = {
        "cko_abi_version": ([], C.c_int),
        "cko_model_state_size": ([P(D)], C.c_int),
        "cko_model_param_count": ([P(D)], C.c_int),
        "cko_ctx_create": ([C.c_int, P(vp), P(E)], C.c_int),
        "cko_ctx_destroy": ([vp], C.c_int),
        "cko_ctx_set_stream": ([vp, vp], C.c_int),
        "cko_comm_buffer_bytes": ([], C.c_size_t),
        "cko_ctx_set_group": ([vp, C.c_int, C.c_int, P(vp), P(E)], C.c_int),
        "cko_model_create": ([vp, P(D), P(vp), P(E)], C.c_int),
        "cko_model_destroy": ([vp], C.c_int),
        "cko_be_forward": ([vp, vp, dp, dp, C.c_int, C.c_int, C.c_int, P(N), P(S), dp, P(vp), P(W), P(E)], C.c_int),
        "cko_be_forward_device": ([vp, vp, vp, vp, C.c_int, C.c_int, C.c_int, P(N), P(S), vp, P(W), P(E)], C.c_int),
        "cko_be_adjoint": ([vp, vp, vp, C.c_int, P(S), C.c_int, dp, dp, dp, P(W), P(E)], C.c_int),
        "cko_be_adjoint_host": ([vp, vp, dp, dp, C.c_int, C.c_int, C.c_int, P(S), C.c_int, dp, dp, dp, P(W), P(E)],
                                C.c_int),
        "cko_be_adjoint_device": ([vp, vp, vp, vp, C.c_int, C.c_int, C.c_int, P(S), C.c_int, vp, dp, dp, P(W), P(E)],
                                  C.c_int),
        "cko_gradient_adjoint_device": ([vp, vp, vp, vp, C.c_int, C.c_int, C.c_int, P(N), P(S), vp, dp, dp, P(W), P(W),
                                         P(E)], C.c_int),
        "cko_gradient_adjoint": ([vp, vp, dp, dp, C.c_int, C.c_int, C.c_int, P(N), P(S), dp, dp, dp, P(W), P(W), P(E)],
                                 C.c_int),
        "cko_traj_states": ([vp, P(vp), P(C.c_int), P(C.c_int), P(C.c_int)], C.c_int),
        "cko_traj_destroy": ([vp], C.c_int),
        "cko_block_bidiag_solve": ([vp, P(S), C.c_int, C.c_int, C.c_int, dp, dp, dp, P(C.c_longlong), P(E)], C.c_int),
        "cko_comm_alloc": ([vp, P(vp), C.c_char_p, P(E)], C.c_int),
        "cko_comm_open": ([vp, C.c_char_p, P(vp), P(E)], C.c_int),
        "cko_ctx_enable_timing": ([vp, C.c_int], C.c_int),
        "cko_ctx_last_kernel_ms": ([vp, dp], C.c_int),
        "cko_ctx_last_launches": ([vp], C.c_int),
        "cko_probe_fp64_tflops": ([vp, dp, P(E)], C.c_int),
        "cko_ctx_set_kernel_generation": ([vp, C.c_int], C.c_int),
        "cko_ctx_kernel_generation_used": ([vp], C.c_int),
        "cko_ctx_set_structured": ([vp, C.c_int], C.c_int),
        "cko_ctx_structured_used": ([vp], C.c_int),
        "cko_newton_solve_chunk": ([vp, vp, dp, dp, dp, dp, C.c_int, C.c_int, P(N), P(S), C.c_int, P(C.c_int), P(W),
                                    P(E)], C.c_int),
        "cko_chunk_residual": ([vp, vp, dp, dp, dp, dp, C.c_int, C.c_int, dp, P(E)], C.c_int),
        "cko_chunk_jacobian": ([vp, vp, dp, dp, dp, dp, C.c_int, C.c_int, dp, dp, P(E)], C.c_int),
        "cko_adjoint_chunk_solve": ([vp, vp, dp, dp, C.c_int, C.c_int, C.c_int, C.c_int, dp, P(S), dp, dp, P(W),
                                     P(E)], C.c_int),
        "cko_adjoint_step_sequential": ([vp, vp, dp, dp, dp, dp, dp, C.c_int, P(S), dp, dp, P(E)], C.c_int),
        "cko_ctx_set_jacobian_strategy": ([vp, C.c_int], C.c_int),
        "cko_fe_forward": ([vp, vp, dp, dp, C.c_int, C.c_int, C.c_int, dp, P(W), P(E)], C.c_int),
        "cko_fe_adjoint_host": ([vp, vp, dp, dp, C.c_int, C.c_int, C.c_int, C.c_int, dp, dp, dp, P(W), P(E)],
                                C.c_int),
    }
    ab_build = bool(os.environ.get("CKO_LIB_PATH"))  # an A/B build may predate newer entry points
    for name, (args, res) in sig.items():
        if ab_build and not hasattr(L, name):
            continue
        f = getattr(L, name)
        f.argtypes = args
        f.restype = res
    if L.cko_abi_version() != 1:
        raise NativeLibraryMissing("libchunkode_b200.so ABI version mismatch")
    _lib = L
    return L


# The exported symbols every build must provide (checked by the CPU tests).
EXPORTS = [
    "cko_abi_version", "cko_model_state_size", "cko_model_param_count", "cko_ctx_create", "cko_ctx_destroy",
    "cko_ctx_set_stream", "cko_comm_buffer_bytes", "cko_ctx_set_group", "cko_model_create", "cko_model_destroy",
    "cko_be_forward", "cko_be_forward_device", "cko_be_adjoint", "cko_be_adjoint_host", "cko_be_adjoint_device",
    "cko_gradient_adjoint", "cko_gradient_adjoint_device", "cko_traj_states", "cko_traj_destroy", "cko_block_bidiag_solve",
    "cko_newton_solve_chunk", "cko_ctx_enable_timing", "cko_ctx_last_kernel_ms", "cko_ctx_last_launches",
    "cko_probe_fp64_tflops", "cko_comm_alloc", "cko_comm_open", "cko_ctx_set_kernel_generation",
    "cko_ctx_kernel_generation_used", "cko_chunk_residual", "cko_chunk_jacobian", "cko_adjoint_chunk_solve",
    "cko_adjoint_step_sequential", "cko_fe_forward", "cko_fe_adjoint_host", "cko_ctx_set_jacobian_strategy",
    "cko_ctx_set_structured", "cko_ctx_structured_used",
]
