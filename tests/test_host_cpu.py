"""CPU tests of the host side: model builders, time grid, ABI exports."""
import ctypes as C
import os
import re

import numpy as np
import pytest

import paper_2310_08649_b200 as P
from paper_2310_08649_b200 import _native, abi, api
from paper_2310_08649_b200.models import MT19937_64

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_mt19937_64_known_answer():
    """std::mt19937_64 default-seed 10000th output is 9981545732273789042 (C++11 [rand.predef])."""
    g = MT19937_64(5489)
    for _ in range(9999):
        g()
    assert g() == 9981545732273789042


@pytest.mark.parametrize("build,args", [
    (P.build_mass_damper_spring, (10, 7)), (P.build_chaboche, (3, 5)), (P.build_neural_ode, (8, 4)),
    (P.build_lin3, (6,)), (P.build_node_wide, (8, 128, 4)),
])
def test_default_params_match_reference(ref, build, args):
    m = build(*args)
    assert np.array_equal(ref.default_params(m), m.params)


def test_param_counts():
    from paper_2310_08649_b200.models import param_count
    for m in [P.build_mass_damper_spring(10, 1000), P.build_chaboche(3, 50), P.build_neural_ode(8, 3),
              P.build_node_wide(8, 128, 256), P.build_lin3(10)]:
        assert m.params.size == param_count(m.kind, m.n_unit, m.width, m.n_batch)
    assert P.build_node_wide(8, 128, 256).params.size == 18824


def test_time_grid_rules():
    g = api.TimeGrid.uniform(10, 3, 2.0)
    assert g.n_time == 10 and g.n_batch == 3 and g.time(10, 2) == 2.0
    with pytest.raises(P.InvalidTimeGrid):
        api.TimeGrid(np.array([[0.0], [0.0]]))
    with pytest.raises(P.InvalidTimeGrid):
        api.TimeGrid.uniform(0, 1, 1.0)


def test_with_params_keeps_count():
    m = P.build_chaboche(2, 2)
    with pytest.raises(P.ShapeMismatch):
        m.with_params(np.zeros(3))


def header_symbols():
    text = open(os.path.join(ROOT, "include", "chunkode_b200.h")).read()
    return sorted(set(re.findall(r"\b(cko_[a-z0-9_]+)\s*\(", text)))


def test_header_declares_python_exports():
    assert sorted(_native.EXPORTS) == header_symbols()


def test_library_loads_and_exports_every_symbol():
    """The in-tree sm_100a library loads on a CPU box and exports every ABI symbol."""
    if not os.path.exists(_native.LIB_PATH):
        pytest.skip("libchunkode_b200.so not built (run __graft_entry__.build())")
    L = C.CDLL(_native.LIB_PATH)
    for name in header_symbols():
        assert hasattr(L, name), name
    assert _native.lib().cko_abi_version() == 1


def test_no_cpu_fallback_without_gpu():
    """Without a CUDA device the product fails loudly instead of computing on the CPU."""
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    if not os.path.exists(_native.LIB_PATH):
        pytest.skip("library not built")
    h = C.c_void_p()
    e = abi.CkoError()
    rc = _native.lib().cko_ctx_create(0, C.byref(h), C.byref(e))
    assert rc == abi.CKO_CUDA
    with pytest.raises(P.DeviceError):
        api.Context(0)


def test_cuda_fatbin_is_sm100a():
    if not os.path.exists(_native.LIB_PATH):
        pytest.skip("library not built")
    import subprocess
    out = subprocess.run(["cuobjdump", "--list-elf", _native.LIB_PATH], capture_output=True, text=True).stdout
    assert "sm_100a" in out
