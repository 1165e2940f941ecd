"""Test configuration: the `gpu` marker and shared helpers.

`-m "not gpu"` runs here on CPU (oracle vs golden vectors, host logic, ABI
exports, multi-process gloo); `-m gpu` runs on a B200 and calls the CUDA path
through the C ABI, checked against the CPU oracle.
"""
import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200); runs the sm_100a kernels")


def pytest_collection_modifyitems(config, items):
    have_gpu = _have_gpu()
    for it in items:
        if "gpu" in it.keywords and not have_gpu:
            it.add_marker(pytest.mark.skip(reason="no CUDA device"))


_GPU = None


def _have_gpu():
    global _GPU
    if _GPU is None:
        try:
            import torch
            _GPU = bool(torch.cuda.is_available())
        except Exception:
            _GPU = False
    return _GPU


def uniform_times(nt, nb, t_max):
    """TimeGrid::uniform (time_grid.cpp:21-29)."""
    ti = np.array([t_max * float(i) / float(nt) for i in range(nt + 1)])
    return np.repeat(ti[:, None], nb, axis=1)


def rel_max(a, ref):
    """SURVEY §8c parity metric: max|a - ref| / max|ref| (no floor)."""
    a, ref = np.asarray(a, np.float64), np.asarray(ref, np.float64)
    den = np.max(np.abs(ref)) if ref.size else 0.0
    num = np.max(np.abs(a - ref)) if ref.size else 0.0
    return num / den if den > 0 else num


@pytest.fixture(scope="session")
def port():
    from oracle import load_port
    return load_port()


@pytest.fixture(scope="session")
def ref():
    from oracle import load_ref, ref_available
    if not ref_available():
        pytest.skip("compiled reference (oracle/_ref) not built")
    return load_ref()
