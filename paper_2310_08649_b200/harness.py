"""Benchmark harness of the reference (bench.hpp / bench.cpp) over the GPU path.

Same API, CSV schema, grid-file format and error behaviour as
/root/reference/proj/core/include/chunkode/bench.hpp:16-90 and
src/bench.cpp:16-443, so GPU rows line up with the reference's rows:

  run_trial(cfg)                 one unmeasured warm-up, then `repeats` timed runs
                                 plus a "mean" row (bench.cpp:166-218); failures go
                                 to the status column, never raised
  write_csv_header / _row        the exact header and %.17g fields (bench.cpp:16-27, 222-231)
  parse_grid_file / run_study    `key = v1, v2` grids in canonical key order, the
                                 Cartesian product, streamed rows (bench.cpp:235-416)
  dump_trajectory(cfg, os)       long-format `time,batch,component,value` (bench.cpp:418-441)
  gradient_fd_oracle             the central-difference reference gradient
                                 (adjoint.cpp:315-342), on the device integrator

Every trial runs on the GPU through the C ABI (api.py), with the trial's
Jacobian strategy (analytic, forward_ad, finite_difference). Timings are
wall-clock around the synchronous calls, as the reference's steady_clock
timers (bench.cpp:87-111).
"""
from __future__ import annotations

import io
import math
import threading
import time
from dataclasses import dataclass, field, replace
from typing import Iterable

import numpy as np

from . import api
from .errors import Error, SizeGuardExceeded
from .models import build_problem

CSV_HEADER = ("problem,n_unit,n_size,n_batch,n_time,n_chunk,jacobian,gradient,solver,integration,repeat,"
              "forward_s,backward_s,total_s,loss,grad_norm,newton_iterations,rate_evals,jacobian_evals,"
              "linear_solves,status")

GRID_KEYS = ["problem", "n_unit", "n_batch", "n_time", "n_chunk", "jacobian", "gradient", "solver", "n_switch",
             "integration", "repeats", "seed", "t_max"]

DEFAULT_T_MAX = {"mds": 1.0, "chaboche": 10.0, "node": 1.0, "neuron": 10.0, "lin3": 1.0}


@dataclass
class TrialConfig:
    """bench.hpp:16-30."""
    problem: str = "mds"
    n_unit: int = 1
    n_batch: int = 1
    n_time: int = 16
    n_chunk: int = 1
    jacobian: str = "analytic"
    gradient: str = "adjoint"
    solver: str = "thomas"
    n_switch: int = 1
    integration: str = "backward"
    repeats: int = 3
    seed: int = 7
    t_max: float = 0.0


@dataclass
class TrialRecord:
    """bench.hpp:37-48."""
    config: TrialConfig
    n_size: int = 0
    repeat_label: str = ""
    forward_s: float = 0.0
    backward_s: float = 0.0
    total_s: float = 0.0
    loss: float = float("nan")
    grad_norm: float = float("nan")
    work: api.WorkCounters = field(default_factory=api.WorkCounters)
    status: str = "ok"


def fmt17(x: float) -> str:
    """printf("%.17g") (bench.cpp:23-27)."""
    return "%.17g" % x


def sanitize_status(s: str) -> str:
    """bench.cpp:29-37."""
    return s.replace(",", ";").replace("\n", " ").replace("\r", " ").replace('"', "'")


def _solver(cfg: TrialConfig) -> api.SolverChoice:
    if cfg.solver not in ("thomas", "pcr", "hybrid"):
        raise Error(f"unknown solver '{cfg.solver}'")
    return api.SolverChoice(cfg.solver, cfg.n_switch)


def _scheme(cfg: TrialConfig) -> str:
    if cfg.integration == "backward":
        return api.Scheme.backward_euler
    if cfg.integration == "forward":
        return api.Scheme.forward_euler
    raise Error(f"unknown integration scheme '{cfg.integration}'")


def _jacobian(cfg: TrialConfig) -> None:
    if cfg.jacobian not in ("analytic", "forward_ad", "finite_difference"):
        raise Error(f"unknown jacobian strategy '{cfg.jacobian}'")


def validate_trial_config(cfg: TrialConfig) -> None:
    """bench.cpp:141-162."""
    if cfg.problem not in ("mds", "neuron", "chaboche", "node"):
        raise Error(f"unknown problem '{cfg.problem}'")
    if cfg.n_unit < 1:
        raise Error("n_unit must be >= 1")
    if cfg.n_batch < 1:
        raise Error("n_batch must be >= 1")
    if cfg.n_time < 1:
        raise Error("n_time must be >= 1")
    if cfg.n_chunk < 1 or cfg.n_chunk > cfg.n_time:
        raise Error("n_chunk must be in [1, n_time]")
    if cfg.repeats < 1:
        raise Error("repeats must be >= 1")
    if cfg.n_switch < 0:
        raise Error("n_switch must be >= 0")
    _jacobian(cfg)
    _solver(cfg)
    _scheme(cfg)
    if cfg.gradient not in ("adjoint", "fd_oracle", "none"):
        raise Error(f"unknown gradient mode '{cfg.gradient}'")


def _model(cfg: TrialConfig):
    return build_problem(cfg.problem, cfg.n_unit, cfg.n_batch, cfg.seed)


def gradient_fd_oracle(model, y0, grid: api.TimeGrid, loss: api.LossSpec | None = None,
                       scheme: str = api.Scheme.backward_euler,
                       settings: api.NewtonSettings = api.NewtonSettings(1e-12, 1e-10, 100), ctx=None) -> np.ndarray:
    """adjoint.cpp:315-342: central differences with delta = 1e-6 (1 + |p_j|), sequential stepping
    (n_chunk = 1), tight Newton tolerances; guarded to 500 parameters."""
    loss = loss or api.loss_frobenius()
    p0 = np.array(model.params, dtype=np.float64)
    if p0.size > 500:
        raise SizeGuardExceeded(f"finite-difference gradient guarded to 500 parameters, got {p0.size}")
    g = np.zeros_like(p0)
    for j in range(p0.size):
        delta = 1e-6 * (1.0 + abs(p0[j]))
        L = []
        for side in (0, 1):
            p = p0.copy()
            p[j] = p0[j] + (delta if side == 0 else -delta)
            m = model.with_params(p)
            tr = (api.integrate_backward_euler(m, y0, grid, 1, settings, api.SolverChoice(), ctx)
                  if scheme == api.Scheme.backward_euler else api.integrate_forward_euler(m, y0, grid, 1, ctx))
            L.append(loss.value(tr))
        g[j] = (L[0] - L[1]) / (2.0 * delta)
    return g


def _run_once(model, cfg: TrialConfig, grid: api.TimeGrid, ctx):
    """bench.cpp:79-118."""
    nb, ns = cfg.n_batch, model.state_size
    solver, scheme = _solver(cfg), _scheme(cfg)
    y0 = np.zeros((nb, ns))  # every bundled problem starts from rest
    t0 = time.perf_counter()
    traj = (api.integrate_backward_euler(model, y0, grid, cfg.n_chunk, api.NewtonSettings(), solver, ctx,
                                         strategy=cfg.jacobian)
            if scheme == api.Scheme.backward_euler else api.integrate_forward_euler(model, y0, grid, cfg.n_chunk, ctx))
    fwd = time.perf_counter() - t0
    loss = api.loss_frobenius()
    bwd, L, gn = 0.0, float("nan"), 0.0
    if cfg.gradient == "adjoint":
        t0 = time.perf_counter()
        L, g = api.adjoint_backward(model, traj, cfg.n_chunk, loss, solver, None, ctx, scheme=scheme,
                                    strategy=cfg.jacobian)
        bwd = time.perf_counter() - t0
        gn = math.sqrt(float(np.sum(g * g)))
    elif cfg.gradient == "fd_oracle":
        L = loss.value(traj)
        t0 = time.perf_counter()
        g = gradient_fd_oracle(model, y0, grid, loss, scheme, ctx=ctx)
        bwd = time.perf_counter() - t0
        gn = math.sqrt(float(np.sum(g * g)))
    elif cfg.gradient == "none":
        L = loss.value(traj)
    else:
        raise Error(f"unknown gradient mode '{cfg.gradient}'")
    return fwd, bwd, L, gn, traj.work


def _failed_rows(cfg: TrialConfig, n_size: int, status: str):
    rows = [TrialRecord(cfg, n_size, str(r), status=status) for r in range(1, max(1, cfg.repeats) + 1)]
    rows.append(TrialRecord(cfg, n_size, "mean", status=status))
    return rows


def run_trial(cfg: TrialConfig, ctx=None) -> list[TrialRecord]:
    """bench.cpp:166-218: warm-up, `repeats` measured runs, then the mean row; never raises."""
    try:
        validate_trial_config(cfg)
        model = _model(cfg)
    except Exception as e:  # noqa: BLE001 - the reference catches std::exception
        return _failed_rows(cfg, 0, sanitize_status(str(e)))
    n_size = model.state_size
    t_max = cfg.t_max if cfg.t_max > 0.0 else DEFAULT_T_MAX[cfg.problem]
    grid = api.TimeGrid.uniform(cfg.n_time, cfg.n_batch, t_max)
    try:
        _run_once(model, cfg, grid, ctx)  # warm-up, unmeasured
    except Exception as e:  # noqa: BLE001
        return _failed_rows(cfg, n_size, sanitize_status(str(e)))
    rows, fs, bs, last = [], 0.0, 0.0, None
    for r in range(1, cfg.repeats + 1):
        try:
            last = _run_once(model, cfg, grid, ctx)
        except Exception as e:  # noqa: BLE001
            return _failed_rows(cfg, n_size, sanitize_status(str(e)))
        fwd, bwd, L, gn, w = last
        rows.append(TrialRecord(cfg, n_size, str(r), fwd, bwd, fwd + bwd, L, gn, w, "ok"))
        fs += fwd
        bs += bwd
    _, _, L, gn, w = last
    rows.append(TrialRecord(cfg, n_size, "mean", fs / cfg.repeats, bs / cfg.repeats,
                            fs / cfg.repeats + bs / cfg.repeats, L, gn, w, "ok"))
    return rows


def write_csv_header(os_) -> None:
    os_.write(CSV_HEADER + "\n")


def write_csv_row(os_, rec: TrialRecord) -> None:
    """bench.cpp:222-231."""
    c, w = rec.config, rec.work
    os_.write(",".join([c.problem, str(c.n_unit), str(rec.n_size), str(c.n_batch), str(c.n_time), str(c.n_chunk),
                        c.jacobian, c.gradient, c.solver, c.integration, rec.repeat_label, fmt17(rec.forward_s),
                        fmt17(rec.backward_s), fmt17(rec.total_s), fmt17(rec.loss), fmt17(rec.grad_norm),
                        str(w.newton_iterations), str(w.rate_evals), str(w.jacobian_evals), str(w.linear_solves),
                        sanitize_status(rec.status)]) + "\n")


# ---------------------------------------------------------------------------
# study grids (bench.cpp:235-416)
# ---------------------------------------------------------------------------
@dataclass
class StudyGrid:
    entries: list = field(default_factory=list)  # [(key, [values])] in canonical key order


def _int(s: str, key: str) -> int:
    try:
        return int(s)
    except ValueError:
        raise Error(f"grid: '{s}' is not an integer (key {key})") from None


def _apply(cfg: TrialConfig, key: str, value: str) -> TrialConfig:
    if key in ("problem", "jacobian", "gradient", "solver", "integration"):
        return replace(cfg, **{key: value})
    if key in ("n_unit", "n_batch", "n_time", "n_chunk", "n_switch", "repeats"):
        return replace(cfg, **{key: _int(value, key)})
    if key == "seed":
        try:
            v = int(value)
            if v < 0:
                raise ValueError
        except ValueError:
            raise Error(f"grid: '{value}' is not an unsigned integer (key {key})") from None
        return replace(cfg, seed=v)
    if key == "t_max":
        try:
            return replace(cfg, t_max=float(value))
        except ValueError:
            raise Error(f"grid: '{value}' is not a number (key {key})") from None
    raise Error(f"grid: unknown key '{key}'")


def parse_grid_file(src) -> StudyGrid:
    """`key = v1, v2` per line, '#' comments, canonical key order (bench.cpp:346-382). `src` is a path or
    an iterable of lines."""
    if isinstance(src, str):
        try:
            with open(src) as fh:
                lines = fh.read().splitlines()
        except OSError:
            raise Error(f"grid: cannot open '{src}'") from None
    else:
        lines = list(src)
    entries = []
    for no, line in enumerate(lines, 1):
        line = line.split("#", 1)[0].strip()
        if not line:
            continue
        if "=" not in line:
            raise Error(f"grid: line {no} has no '='")
        key, rest = line.split("=", 1)
        key = key.strip()
        if key not in GRID_KEYS:
            raise Error(f"grid: unknown key '{key}' on line {no}")
        if any(k == key for k, _ in entries):
            raise Error(f"grid: duplicate key '{key}'")
        values = [v.strip() for v in rest.split(",")]
        if any(not v for v in values):
            raise Error(f"grid: empty value for key '{key}' on line {no}")
        entries.append((key, values))
    entries.sort(key=lambda kv: GRID_KEYS.index(kv[0]))
    return StudyGrid(entries)


def expand_grid(grid: StudyGrid) -> list[TrialConfig]:
    """The Cartesian product, last key fastest; no `problem` key -> no trials (bench.cpp:313-342)."""
    if not any(k == "problem" for k, _ in grid.entries):
        return []
    out = [TrialConfig()]
    for key, values in grid.entries:
        out = [_apply(cfg, key, v) for cfg in out for v in values]
    return out


def run_study(grid: StudyGrid, csv, parallel: bool = False, ctx=None) -> int:
    """bench.cpp:390-416: header, then each trial's rows as it finishes; returns the failed trial count."""
    configs = expand_grid(grid)
    write_csv_header(csv)
    failed = 0

    def emit(rows):
        nonlocal failed
        for rec in rows:
            write_csv_row(csv, rec)
        if any(r.status != "ok" for r in rows):
            failed += 1
        csv.flush()

    if not parallel:
        for cfg in configs:
            emit(run_trial(cfg, ctx))
        return failed
    results: list = [None] * len(configs)

    def work(i, cfg):
        results[i] = run_trial(cfg, api.Context(ctx.device if ctx else 0))

    threads = [threading.Thread(target=work, args=(i, c)) for i, c in enumerate(configs)]
    for t in threads:
        t.start()
    for i, t in enumerate(threads):
        t.join()
        emit(results[i])
    return failed


def dump_trajectory(cfg: TrialConfig, os_, ctx=None) -> None:
    """bench.cpp:418-441: one integration, `time,batch,component,value` per (step, lane, component)."""
    validate_trial_config(cfg)
    model = _model(cfg)
    ns = model.state_size
    t_max = cfg.t_max if cfg.t_max > 0.0 else DEFAULT_T_MAX[cfg.problem]
    grid = api.TimeGrid.uniform(cfg.n_time, cfg.n_batch, t_max)
    y0 = np.zeros((cfg.n_batch, ns))
    traj = (api.integrate_backward_euler(model, y0, grid, cfg.n_chunk, api.NewtonSettings(), _solver(cfg), ctx,
                                         strategy=cfg.jacobian)
            if _scheme(cfg) == api.Scheme.backward_euler
            else api.integrate_forward_euler(model, y0, grid, cfg.n_chunk, ctx))
    os_.write("time,batch,component,value\n")
    t = grid.times
    buf = io.StringIO()
    for step in range(traj.n_time + 1):
        row = traj.states[step]
        for b in range(cfg.n_batch):
            tb = fmt17(float(t[step, b]))
            for i in range(ns):
                buf.write(f"{tb},{b},{i},{fmt17(float(row[b * ns + i]))}\n")
        if buf.tell() > 1 << 20:
            os_.write(buf.getvalue())
            buf = io.StringIO()
    os_.write(buf.getvalue())


def study_from_lines(lines: Iterable[str]) -> StudyGrid:
    return parse_grid_file(list(lines))
