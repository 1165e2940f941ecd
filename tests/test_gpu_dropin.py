"""The C++ drop-in (paper_2310_08649_b200/shim): the reference's own C++ API, unchanged signatures,
served by the B200 path. tests/cpp/acceptance_b200 replays the reference's release gate
(acceptance.cpp criteria 1-5, 7, 8, plus the strategies through the device chunk_jacobian) through it; every integrate / adjoint / solve call runs on the GPU."""
import os
import subprocess

import pytest

from tests.conftest import ROOT

BIN = os.path.join(ROOT, "tests", "cpp", "_build", "acceptance_b200")


def test_dropin_exports_reference_signatures():
    lib = os.path.join(ROOT, "paper_2310_08649_b200", "shim", "_build", "libchunkode_b200_dropin.so")
    if not os.path.exists(lib):
        pytest.skip("drop-in not built (needs the reference headers)")
    out = subprocess.run(["nm", "-DC", lib], capture_output=True, text=True).stdout
    for sig in [
        "chunkode::integrate_backward_euler(chunkode::OdeModel const&, chunkode::Array2d const&, "
        "chunkode::TimeGrid const&, int, chunkode::NewtonSettings const&, chunkode::SolverChoice const&, "
        "chunkode::JacobianStrategy)",
        "chunkode::adjoint_backward(chunkode::OdeModel const&, chunkode::Trajectory const&, int, "
        "chunkode::LossSpec const&, chunkode::Scheme, chunkode::SolverChoice const&, chunkode::JacobianStrategy, "
        "chunkode::WorkCounters*)",
        "chunkode::gradient_adjoint(chunkode::OdeModel const&, chunkode::Array2d const&, chunkode::TimeGrid const&, "
        "int, chunkode::LossSpec const&, chunkode::Scheme, chunkode::SolverChoice const&, "
        "chunkode::JacobianStrategy, chunkode::NewtonSettings const&)",
        "chunkode::solve_pcr(chunkode::BlockBidiagonalSystem const&, chunkode::BatchedChunkVector const&, long*)",
    ]:
        assert f" T {sig}" in out, sig


@pytest.mark.gpu
def test_reference_acceptance_gate_through_the_dropin():
    assert os.path.exists(BIN), "tests/cpp/_build/acceptance_b200 not built (shim/Makefile)"
    r = subprocess.run([BIN], capture_output=True, text=True, timeout=600)
    print(r.stdout)
    assert r.returncode == 0, r.stdout + r.stderr
    assert r.stdout.count("PASS") == 8
