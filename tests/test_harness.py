"""The reference's benchmark harness (bench.hpp/bench.cpp, SURVEY §8 rows f1 + f4) over the GPU path.

CPU: grid parsing rules and error messages, canonical key order, the Cartesian product, and the CSV
header against the compiled reference's own output. GPU: run_study rows against the reference's
run_study rows (config columns and counters identical, loss / grad_norm within 1e-10, timing columns
excluded) and dump_trajectory against the reference's dump (time/batch/component identical, values
within 1e-10 max-norm relative)."""
import io

import numpy as np
import pytest

from paper_2310_08649_b200 import harness as H
from paper_2310_08649_b200.errors import Error

GRID = """# C2/C3-style study, small
problem = mds, chaboche
n_chunk = 1, 4
n_unit = 2
n_batch = 3
n_time = 8
solver = thomas, pcr
repeats = 2
t_max = 0.001
"""


def test_grid_canonical_order_and_product():
    g = H.parse_grid_file(GRID.splitlines())
    assert [k for k, _ in g.entries] == ["problem", "n_unit", "n_batch", "n_time", "n_chunk", "solver", "repeats",
                                         "t_max"]
    cfgs = H.expand_grid(g)
    assert len(cfgs) == 8
    # the last canonical key varies fastest
    assert [(c.problem, c.n_chunk, c.solver) for c in cfgs[:4]] == [("mds", 1, "thomas"), ("mds", 1, "pcr"),
                                                                    ("mds", 4, "thomas"), ("mds", 4, "pcr")]
    assert H.expand_grid(H.parse_grid_file(["n_unit = 1"])) == []


@pytest.mark.parametrize("text,msg", [
    ("problem mds", "has no '='"),
    ("colour = red", "unknown key 'colour'"),
    ("problem = mds\nproblem = node", "duplicate key 'problem'"),
    ("n_time = 4,", "empty value for key 'n_time'"),
    ("problem = mds\nn_time = x", "is not an integer"),
    ("problem = mds\nt_max = q", "is not a number"),
])
def test_grid_errors(text, msg):
    with pytest.raises(Error, match=msg):
        H.expand_grid(H.parse_grid_file(text.splitlines()))


def test_failed_trials_go_to_the_status_column():
    rows = H.run_trial(H.TrialConfig(problem="nope"))
    assert [r.repeat_label for r in rows] == ["1", "2", "3", "mean"]
    assert all(r.status == "unknown problem 'nope'" for r in rows)
    out = io.StringIO()
    H.write_csv_row(out, rows[0])
    assert out.getvalue().count(",") == H.CSV_HEADER.count(",")


def test_csv_header_is_the_reference_header(ref):
    text = ref.study_csv("problem = mds\nn_time = 2\nrepeats = 1\nt_max = 1e-4")
    assert text.splitlines()[0] == H.CSV_HEADER


def _rows(text):
    lines = text.strip().splitlines()
    hdr = lines[0].split(",")
    return hdr, [dict(zip(hdr, ln.split(","))) for ln in lines[1:]]


GRID2 = """problem = neuron, node
n_unit = 2
n_batch = 2
n_time = 12
n_chunk = 3
jacobian = analytic, forward_ad, finite_difference
repeats = 1
"""


@pytest.mark.gpu
@pytest.mark.parametrize("grid", [GRID, GRID2], ids=["mds_chaboche_solvers", "neuron_node_strategies"])
def test_study_matches_reference(ref, grid):
    buf = io.StringIO()
    failed = H.run_study(H.parse_grid_file(grid.splitlines()), buf)
    assert failed == 0
    hdr, got = _rows(buf.getvalue())
    _, want = _rows(ref.study_csv(grid))
    assert len(got) == len(want)
    timing = {"forward_s", "backward_s", "total_s"}
    for g, w in zip(got, want):
        for k in hdr:
            if k in timing:
                continue
            if k in ("loss", "grad_norm"):
                tol = 1e-8 if g["jacobian"] == "finite_difference" else 1e-10
                assert abs(float(g[k]) - float(w[k])) <= tol * abs(float(w[k])), (k, g, w)
            else:
                assert g[k] == w[k], (k, g, w)


@pytest.mark.gpu
@pytest.mark.parametrize("problem,n_unit,nc,solver,integ", [("mds", 3, 4, "thomas", "backward"),
                                                             ("chaboche", 2, 3, "pcr", "backward"),
                                                             ("node", 3, 2, "thomas", "forward")])
def test_dump_trajectory_matches_reference(ref, problem, n_unit, nc, solver, integ):
    t_max = 1e-3 if problem == "mds" else 0.0
    cfg = H.TrialConfig(problem=problem, n_unit=n_unit, n_batch=3, n_time=12, n_chunk=nc, solver=solver,
                        integration=integ, t_max=t_max)
    buf = io.StringIO()
    H.dump_trajectory(cfg, buf)
    want = ref.dump_trajectory(problem, n_unit, 3, 12, nc, solver, 1, integ, t_max)
    g = np.array([ln.split(",") for ln in buf.getvalue().strip().splitlines()[1:]], dtype=object)
    w = np.array([ln.split(",") for ln in want.strip().splitlines()[1:]], dtype=object)
    assert buf.getvalue().splitlines()[0] == want.splitlines()[0]
    assert g.shape == w.shape
    assert (g[:, :3] == w[:, :3]).all()
    gv, wv = g[:, 3].astype(float), w[:, 3].astype(float)
    assert np.max(np.abs(gv - wv)) <= 1e-10 * max(np.max(np.abs(wv)), 1e-300)
