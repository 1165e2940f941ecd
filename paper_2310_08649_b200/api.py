"""Python mirror of the reference chunkode API for the backward-Euler path.

Same names, argument meanings and error behaviour as
/root/reference/proj/core/include/chunkode/{time_grid,integrate,adjoint,linalg}.hpp;
every call runs on the GPU through the C ABI (include/chunkode_b200.h).
"""
from __future__ import annotations

import ctypes as C
import threading
from dataclasses import dataclass, field
from typing import Callable, Optional

import numpy as np

from . import abi
from ._native import lib
from .abi import dptr
from .errors import Error, InvalidTimeGrid, ShapeMismatch, raise_for
from .models import Model


# ---------------------------------------------------------------------------
# settings and counters (integrate.hpp:9-32, linalg.hpp:89-95)
# ---------------------------------------------------------------------------
class SolverKind:
    thomas = abi.CKO_SOLVER_THOMAS
    pcr = abi.CKO_SOLVER_PCR
    hybrid = abi.CKO_SOLVER_HYBRID


_KIND_BY_NAME = {"thomas": 0, "pcr": 1, "hybrid": 2}


@dataclass
class SolverChoice:
    kind: int = SolverKind.thomas
    n_switch: int = 1

    def c(self) -> abi.CkoSolverChoice:
        k = _KIND_BY_NAME[self.kind] if isinstance(self.kind, str) else int(self.kind)
        return abi.CkoSolverChoice(k, int(self.n_switch))


@dataclass
class NewtonSettings:
    tol_a: float = 1e-8
    tol_r: float = 1e-6
    max_iter: int = 100

    def c(self) -> abi.CkoNewtonSettings:
        return abi.CkoNewtonSettings(float(self.tol_a), float(self.tol_r), int(self.max_iter))


@dataclass
class WorkCounters:
    newton_iterations: int = 0
    rate_evals: int = 0
    jacobian_evals: int = 0
    linear_solves: int = 0
    reduction_sweeps: int = 0

    @classmethod
    def from_c(cls, w: abi.CkoWork) -> "WorkCounters":
        return cls(*(int(getattr(w, k)) for k, _ in abi.CkoWork._fields_))

    def as_dict(self) -> dict:
        return dict(self.__dict__)

    def __iadd__(self, o):
        for k in self.__dict__:
            setattr(self, k, getattr(self, k) + getattr(o, k))
        return self


# ---------------------------------------------------------------------------
# time grid (time_grid.hpp:10-28, time_grid.cpp:7-29)
# ---------------------------------------------------------------------------
class TimeGrid:
    def __init__(self, times):
        t = np.ascontiguousarray(times, dtype=np.float64)
        if t.ndim != 2 or t.shape[0] < 2 or t.shape[1] < 1:
            raise InvalidTimeGrid("time grid needs at least one step and one batch lane")
        bad = ~(t[1:] > t[:-1])
        if bad.any():
            i, b = np.argwhere(bad)[0]
            raise InvalidTimeGrid(f"time grid must be strictly increasing (step {i + 1}, batch {b})")
        self._t = t

    @staticmethod
    def uniform(n_time: int, n_batch: int, t_max: float) -> "TimeGrid":
        if n_time < 1 or n_batch < 1:
            raise InvalidTimeGrid("uniform grid needs n_time, n_batch >= 1")
        ti = np.array([t_max * float(i) / float(n_time) for i in range(n_time + 1)])
        return TimeGrid(np.repeat(ti[:, None], n_batch, axis=1))

    @property
    def n_time(self) -> int:
        return self._t.shape[0] - 1

    @property
    def n_batch(self) -> int:
        return self._t.shape[1]

    @property
    def times(self) -> np.ndarray:
        return self._t

    def time(self, step: int, b: int) -> float:
        return float(self._t[step, b])

    def dt(self, step: int, b: int) -> float:
        return float(self._t[step, b] - self._t[step - 1, b])


@dataclass
class Trajectory:
    """integrate.hpp:34-50: states (n_time + 1, n_batch * n_size)."""

    states: np.ndarray
    grid: TimeGrid
    n_batch: int
    n_size: int
    work: WorkCounters = field(default_factory=WorkCounters)

    @property
    def n_time(self) -> int:
        return self.states.shape[0] - 1

    def point(self, step: int, b: int) -> np.ndarray:
        return self.states[step, b * self.n_size:(b + 1) * self.n_size]


@dataclass
class LossSpec:
    """adjoint.hpp:14-20. value(traj) -> float, state_gradient(traj) -> array shaped like traj.states.
    frobenius=True selects the fused device Frobenius loss."""

    value: Optional[Callable] = None
    state_gradient: Optional[Callable] = None
    frobenius: bool = False


def loss_frobenius() -> LossSpec:
    """adjoint.cpp:196-221: sqrt of the sum of squares over steps 1..n_time."""
    def value(tr):
        return float(np.sqrt(np.sum(tr.states[1:] ** 2)))

    def grad(tr):
        L = value(tr)
        g = np.zeros_like(tr.states)
        if L > 0:
            g[1:] = tr.states[1:] / L
        return g

    return LossSpec(value, grad, frobenius=True)


@dataclass
class GradientResult:
    loss: float
    gradient: np.ndarray
    trajectory: Trajectory
    backward_work: WorkCounters


# ---------------------------------------------------------------------------
# device context + model cache
# ---------------------------------------------------------------------------
class Context:
    """cko_ctx: one CUDA device, one stream, a workspace pool."""

    def __init__(self, device: int = 0):
        self.device = device
        h = C.c_void_p()
        e = abi.CkoError()
        raise_for(lib().cko_ctx_create(device, C.byref(h), C.byref(e)), e)
        self.h = h
        self._models: dict = {}

    def close(self):
        for dm in self._models.values():
            lib().cko_model_destroy(dm)
        self._models.clear()
        if self.h:
            lib().cko_ctx_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def set_stream(self, stream_handle: int):
        lib().cko_ctx_set_stream(self.h, C.c_void_p(stream_handle))

    def set_kernel_generation(self, gen: int):
        """2 (default): warp-specialised Thomas kernels where instantiated; 1: generic kernels only."""
        if lib().cko_ctx_set_kernel_generation(self.h, int(gen)) != 0:
            raise ValueError(f"kernel generation must be 1 or 2, got {gen}")

    def set_jacobian_strategy(self, strategy) -> None:
        """JacobianStrategy of the following calls: 'analytic', 'forward_ad', 'finite_difference' (or 0/1/2)."""
        k = _STRATEGY[strategy] if isinstance(strategy, str) else int(strategy)
        if lib().cko_ctx_set_jacobian_strategy(self.h, k) != 0:
            raise ValueError(f"unknown Jacobian strategy {strategy!r}")

    def kernel_generation_used(self) -> int:
        """Kernel generation the last forward / adjoint call ran (1 or 2)."""
        return int(lib().cko_ctx_kernel_generation_used(self.h))

    # bits of structured_used() (include/chunkode_b200.h CKO_SP_*)
    SP_FWD, SP_ADJ, SP_FWD_FALLBACK, SP_ADJ_FALLBACK = 1, 2, 4, 8

    def set_structured(self, on: bool) -> None:
        """Structured-record Thomas kernels for arrow + tridiagonal blocks (the MDS chain); on by default."""
        if lib().cko_ctx_set_structured(self.h, 1 if on else 0) != 0:
            raise ValueError("set_structured failed")

    def structured_used(self) -> int:
        """CKO_SP_* bits of the last forward / adjoint call: which ran structured, which fell back."""
        return int(lib().cko_ctx_structured_used(self.h))

    def model(self, m: Model) -> C.c_void_p:
        key = (m.kind, m.n_unit, m.width, m.n_batch, m.lane_offset, m.params.tobytes())
        dm = self._models.get(key)
        if dm is None:
            dm = C.c_void_p()
            e = abi.CkoError()
            d = m.desc()
            raise_for(lib().cko_model_create(self.h, C.byref(d), C.byref(dm), C.byref(e)), e)
            if len(self._models) > 64:
                for v in self._models.values():
                    lib().cko_model_destroy(v)
                self._models.clear()
            self._models[key] = dm
        return dm


_STRATEGY = {"analytic": abi.CKO_JACOBIAN_ANALYTIC, "forward_ad": abi.CKO_JACOBIAN_FORWARD_AD,
             "finite_difference": abi.CKO_JACOBIAN_FINITE_DIFFERENCE}


class _Strategy:
    """Run one call under a JacobianStrategy (ode_model.hpp:14), restoring analytic afterwards."""

    def __init__(self, ctx: "Context", strategy):
        self.ctx, self.strategy = ctx, strategy

    def __enter__(self):
        if self.strategy not in ("analytic", 0):
            self.ctx.set_jacobian_strategy(self.strategy)
        return self.ctx

    def __exit__(self, *exc):
        if self.strategy not in ("analytic", 0):
            self.ctx.set_jacobian_strategy("analytic")


_tls = threading.local()


def default_context(device: int = 0) -> Context:
    ctxs = getattr(_tls, "ctxs", None)
    if ctxs is None:
        ctxs = _tls.ctxs = {}
    if device not in ctxs:
        ctxs[device] = Context(device)
    return ctxs[device]


def _f64(a) -> np.ndarray:
    return np.ascontiguousarray(a, dtype=np.float64)


# ---------------------------------------------------------------------------
# integrator / adjoint (integrate.hpp:86-89, adjoint.hpp:63-80)
# ---------------------------------------------------------------------------
def integrate_backward_euler(model: Model, y0, grid: TimeGrid, n_chunk: int,
                             settings: NewtonSettings | None = None, solver: SolverChoice | None = None,
                             ctx: Context | None = None, strategy: str = "analytic") -> Trajectory:
    settings = settings or NewtonSettings()
    solver = solver or SolverChoice()
    y0 = _f64(y0)
    if y0.ndim != 2 or y0.shape[1] != model.state_size:
        raise ShapeMismatch("integrate: y0 width != state size")
    if y0.shape[0] != grid.n_batch:
        raise ShapeMismatch("integrate: y0 rows != grid batch width")
    ctx = ctx or default_context()
    nb, nt, n = grid.n_batch, grid.n_time, model.state_size
    states = np.zeros((nt + 1, nb * n))
    w, e = abi.CkoWork(), abi.CkoError()
    st, sv = settings.c(), solver.c()
    with _Strategy(ctx, strategy):
        rc = lib().cko_be_forward(ctx.h, ctx.model(model), dptr(y0), dptr(grid.times), nb, nt, int(n_chunk),
                                  C.byref(st), C.byref(sv), dptr(states), None, C.byref(w), C.byref(e))
    raise_for(rc, e)
    return Trajectory(states, grid, nb, n, WorkCounters.from_c(w))


class Scheme:
    """adjoint.hpp:12: the discrete adjoint follows the scheme that produced the trajectory."""
    backward_euler = "backward_euler"
    forward_euler = "forward_euler"


def integrate_forward_euler(model: Model, y0, grid: TimeGrid, n_chunk: int = 1,
                            ctx: Context | None = None) -> Trajectory:
    """integrate.hpp:91-96: explicit, strictly step-sequential (results independent of n_chunk)."""
    y0 = _f64(y0)
    if y0.ndim != 2 or y0.shape[1] != model.state_size:
        raise ShapeMismatch("integrate: y0 width != state size")
    if y0.shape[0] != grid.n_batch:
        raise ShapeMismatch("integrate: y0 rows != grid batch width")
    if n_chunk < 1:
        raise ShapeMismatch("integrate: n_chunk must be >= 1")
    ctx = ctx or default_context()
    nb, nt, n = grid.n_batch, grid.n_time, model.state_size
    states = np.zeros((nt + 1, nb * n))
    w, e = abi.CkoWork(), abi.CkoError()
    raise_for(lib().cko_fe_forward(ctx.h, ctx.model(model), dptr(y0), dptr(grid.times), nb, nt, int(n_chunk),
                                   dptr(states), C.byref(w), C.byref(e)), e)
    return Trajectory(states, grid, nb, n, WorkCounters.from_c(w))


def adjoint_backward(model: Model, traj: Trajectory, n_chunk: int, loss: LossSpec | None = None,
                     solver: SolverChoice | None = None, work: WorkCounters | None = None,
                     ctx: Context | None = None, scheme: str = Scheme.backward_euler, strategy: str = "analytic"):
    """Returns (loss, gradient) like adjoint.hpp:63-66; `work` (if given) receives the backward counters."""
    loss = loss or loss_frobenius()
    solver = solver or SolverChoice()
    if traj.n_size != model.state_size:
        raise ShapeMismatch("adjoint: trajectory width != model size")
    if n_chunk < 1:
        raise ShapeMismatch("adjoint: n_chunk must be >= 1")
    if loss.value is None or loss.state_gradient is None:
        raise ShapeMismatch("loss: both callbacks must be set")
    ctx = ctx or default_context()
    grad = np.zeros(model.params.size)
    L = C.c_double(0.0)
    w, e = abi.CkoWork(), abi.CkoError()
    sv = solver.c()
    if loss.frobenius:
        kind, dL = abi.CKO_LOSS_FROBENIUS, None
    else:
        kind = abi.CKO_LOSS_USER
        dL = _f64(loss.state_gradient(traj))
        if dL.shape != traj.states.shape:
            raise ShapeMismatch("loss gradient: output must be shaped like the trajectory states")
    strat = _Strategy(ctx, strategy)
    strat.__enter__()
    if scheme == Scheme.forward_euler:
        rc = lib().cko_fe_adjoint_host(ctx.h, ctx.model(model), dptr(_f64(traj.states)), dptr(traj.grid.times),
                                       traj.n_batch, traj.n_time, int(n_chunk), kind, dptr(dL), C.byref(L),
                                       dptr(grad), C.byref(w), C.byref(e))
    else:
        rc = lib().cko_be_adjoint_host(ctx.h, ctx.model(model), dptr(_f64(traj.states)), dptr(traj.grid.times),
                                       traj.n_batch, traj.n_time, int(n_chunk), C.byref(sv), kind, dptr(dL),
                                       C.byref(L), dptr(grad), C.byref(w), C.byref(e))
    strat.__exit__()
    raise_for(rc, e)
    if work is not None:
        work += WorkCounters.from_c(w)
    Lv = L.value if loss.frobenius else float(loss.value(traj))
    return Lv, grad


def gradient_adjoint(model: Model, y0, grid: TimeGrid, n_chunk: int, loss: LossSpec | None = None,
                     solver: SolverChoice | None = None, settings: NewtonSettings | None = None,
                     ctx: Context | None = None, scheme: str = Scheme.backward_euler,
                     strategy: str = "analytic") -> GradientResult:
    """adjoint.cpp:299-313; the Frobenius loss runs fully on the device."""
    loss = loss or loss_frobenius()
    settings = settings or NewtonSettings()
    solver = solver or SolverChoice()
    if scheme == Scheme.forward_euler:
        tr = integrate_forward_euler(model, y0, grid, n_chunk, ctx)
        bw = WorkCounters()
        L, g = adjoint_backward(model, tr, n_chunk, loss, solver, bw, ctx, scheme=scheme, strategy=strategy)
        return GradientResult(L, g, tr, bw)
    if not loss.frobenius:
        tr = integrate_backward_euler(model, y0, grid, n_chunk, settings, solver, ctx, strategy)
        bw = WorkCounters()
        L, g = adjoint_backward(model, tr, n_chunk, loss, solver, bw, ctx, strategy=strategy)
        return GradientResult(L, g, tr, bw)
    y0 = _f64(y0)
    if y0.ndim != 2 or y0.shape[1] != model.state_size or y0.shape[0] != grid.n_batch:
        raise ShapeMismatch("integrate: y0 shape does not match the model / grid")
    ctx = ctx or default_context()
    nb, nt, n = grid.n_batch, grid.n_time, model.state_size
    states = np.zeros((nt + 1, nb * n))
    grad = np.zeros(model.params.size)
    L = C.c_double(0.0)
    wf, wb, e = abi.CkoWork(), abi.CkoWork(), abi.CkoError()
    st, sv = settings.c(), solver.c()
    with _Strategy(ctx, strategy):
        rc = lib().cko_gradient_adjoint(ctx.h, ctx.model(model), dptr(y0), dptr(grid.times), nb, nt, int(n_chunk),
                                        C.byref(st), C.byref(sv), dptr(states), C.byref(L), dptr(grad), C.byref(wf),
                                        C.byref(wb), C.byref(e))
    raise_for(rc, e)
    tr = Trajectory(states, grid, nb, n, WorkCounters.from_c(wf))
    return GradientResult(L.value, grad, tr, WorkCounters.from_c(wb))


def gradient_adjoint_device(model: Model, d_y0, d_times, n_chunk: int, solver: SolverChoice | None = None,
                            settings: NewtonSettings | None = None, ctx: Context | None = None, d_states=None):
    """gradient_adjoint (adjoint.cpp:299-313, Frobenius loss) over CUDA tensors: d_y0 (nb, n) and d_times
    (nt+1, nb) float64 on the context's device; the trajectory goes to d_states ((nt+1, nb*n), allocated when
    None). One C call: the loss rides on the forward's residual passes. Returns (loss, gradient, d_states,
    forward WorkCounters, backward WorkCounters)."""
    import torch
    settings = settings or NewtonSettings()
    solver = solver or SolverChoice()
    ctx = ctx or default_context()
    n = model.state_size
    if d_y0.dtype != torch.float64 or d_times.dtype != torch.float64 or not (d_y0.is_cuda and d_times.is_cuda):
        raise TypeError("gradient_adjoint_device: float64 CUDA tensors expected")
    if d_y0.dim() != 2 or d_y0.shape[1] != n or d_times.dim() != 2 or d_times.shape[1] != d_y0.shape[0]:
        raise ShapeMismatch("integrate: y0 shape does not match the model / grid")
    nb, nt = d_y0.shape[0], d_times.shape[0] - 1
    if d_states is None:
        d_states = torch.empty((nt + 1, nb * n), dtype=torch.float64, device=d_y0.device)
    d_y0, d_times = d_y0.contiguous(), d_times.contiguous()
    grad = np.zeros(model.params.size)
    L = C.c_double(0.0)
    wf, wb, e = abi.CkoWork(), abi.CkoWork(), abi.CkoError()
    st, sv = settings.c(), solver.c()
    rc = lib().cko_gradient_adjoint_device(ctx.h, ctx.model(model), C.c_void_p(d_y0.data_ptr()),
                                           C.c_void_p(d_times.data_ptr()), nb, nt, int(n_chunk), C.byref(st),
                                           C.byref(sv), C.c_void_p(d_states.data_ptr()), C.byref(L), dptr(grad),
                                           C.byref(wf), C.byref(wb), C.byref(e))
    raise_for(rc, e)
    return L.value, grad, d_states, WorkCounters.from_c(wf), WorkCounters.from_c(wb)


def newton_solve_chunk(model: Model, y_start, dy, t_chunk, dt_chunk, settings: NewtonSettings | None = None,
                       solver: SolverChoice | None = None, work: WorkCounters | None = None,
                       chunk_start_step: int = 1, ctx: Context | None = None):
    """integrate.hpp:63-67: dy (c, nb, n) updated in place; returns the iteration count."""
    settings = settings or NewtonSettings()
    solver = solver or SolverChoice()
    ctx = ctx or default_context()
    y_start = _f64(y_start)
    t_chunk, dt_chunk = _f64(t_chunk), _f64(dt_chunk)
    c, nb = t_chunk.shape
    buf = _f64(dy).copy()
    it = C.c_int(0)
    w, e = abi.CkoWork(), abi.CkoError()
    st, sv = settings.c(), solver.c()
    rc = lib().cko_newton_solve_chunk(ctx.h, ctx.model(model), dptr(y_start), dptr(buf), dptr(t_chunk),
                                      dptr(dt_chunk), c, nb, C.byref(st), C.byref(sv), int(chunk_start_step),
                                      C.byref(it), C.byref(w), C.byref(e))
    raise_for(rc, e)
    dy[...] = buf
    if work is not None:
        work += WorkCounters.from_c(w)
    return int(it.value)


def _chunk_args(model: Model, y_start, dy, t_chunk, dt_chunk):
    """check_chunk_args (integrate.cpp:12-21)."""
    y_start, dy = _f64(y_start), _f64(dy)
    t_chunk, dt_chunk = _f64(t_chunk), _f64(dt_chunk)
    n = model.state_size
    if y_start.ndim != 2 or y_start.shape[1] != n:
        raise ShapeMismatch("chunk op: y_start width != state size")
    if dy.ndim != 3 or dy.shape[2] != n:
        raise ShapeMismatch("chunk op: dy width != state size")
    if y_start.shape[0] != dy.shape[1]:
        raise ShapeMismatch("chunk op: y_start rows != batch width")
    if t_chunk.shape != dy.shape[:2]:
        raise ShapeMismatch("chunk op: t_chunk must be (chunk_len, n_batch)")
    if dt_chunk.shape != dy.shape[:2]:
        raise ShapeMismatch("chunk op: dt_chunk must be (chunk_len, n_batch)")
    return y_start, dy, t_chunk, dt_chunk


def chunk_residual(model: Model, y_start, dy, t_chunk, dt_chunk, ctx: Context | None = None) -> np.ndarray:
    """integrate.hpp:53-55: out(j) = dy(j) - dy(j-1) - h(y_start + dy(j), t(j)) dt(j), shape (c, nb, n)."""
    y_start, dy, t_chunk, dt_chunk = _chunk_args(model, y_start, dy, t_chunk, dt_chunk)
    ctx = ctx or default_context()
    c, nb, n = dy.shape
    out = np.empty_like(dy)
    e = abi.CkoError()
    raise_for(lib().cko_chunk_residual(ctx.h, ctx.model(model), dptr(y_start), dptr(dy), dptr(t_chunk),
                                       dptr(dt_chunk), c, nb, dptr(out), C.byref(e)), e)
    return out


def chunk_jacobian(model: Model, y_start, dy, t_chunk, dt_chunk, ctx: Context | None = None,
                   strategy: str = "analytic") -> "BlockBidiagonalSystem":
    """integrate.hpp:57-61: diag I - J dt, offdiag -I; J by the given JacobianStrategy."""
    y_start, dy, t_chunk, dt_chunk = _chunk_args(model, y_start, dy, t_chunk, dt_chunk)
    ctx = ctx or default_context()
    c, nb, n = dy.shape
    sys = BlockBidiagonalSystem.zeros(c, nb, n)
    e = abi.CkoError()
    with _Strategy(ctx, strategy):
        rc = lib().cko_chunk_jacobian(ctx.h, ctx.model(model), dptr(y_start), dptr(dy), dptr(t_chunk),
                                      dptr(dt_chunk), c, nb, dptr(sys.diag), dptr(sys.offdiag) if c > 1 else None,
                                      C.byref(e))
    raise_for(rc, e)
    return sys


@dataclass
class AdjointState:
    """adjoint.hpp:26-31: lambda (n_batch, n_size) and the gradient accumulator (n_params)."""

    lam: np.ndarray
    grad: np.ndarray

    @classmethod
    def zeros(cls, model: Model, n_batch: int) -> "AdjointState":
        return cls(np.zeros((n_batch, model.state_size)), np.zeros(model.params.size))


def _check_state(model: Model, state: AdjointState, nb: int):
    """check_adjoint_state (adjoint.cpp:129-134)."""
    if state.lam.shape != (nb, model.state_size):
        raise ShapeMismatch("adjoint: lambda must be (n_batch, n_size)")
    if state.grad.shape != (model.params.size,):
        raise ShapeMismatch("adjoint: gradient accumulator length != parameter count")


def adjoint_chunk_solve(model: Model, traj: Trajectory, step_hi: int, chunk_len: int, dL_dy, state: AdjointState,
                        solver: SolverChoice | None = None, work: WorkCounters | None = None,
                        ctx: Context | None = None) -> None:
    """adjoint.hpp:49-56: reverse steps step_hi - chunk_len + 1 .. step_hi in one coupled solve; updates
    state.lam and accumulates into state.grad."""
    solver = solver or SolverChoice()
    if traj.n_size != model.state_size:
        raise ShapeMismatch("adjoint chunk: trajectory width != model size")
    if not (chunk_len >= 1 and step_hi >= chunk_len and step_hi <= traj.n_time):
        raise ShapeMismatch("adjoint chunk: step range out of bounds")
    dL = _f64(dL_dy)
    if dL.shape != traj.states.shape:
        raise ShapeMismatch("adjoint chunk: dL_dy must be shaped like the trajectory states")
    _check_state(model, state, traj.n_batch)
    ctx = ctx or default_context()
    lam, grad = _f64(state.lam).copy(), _f64(state.grad).copy()
    w, e = abi.CkoWork(), abi.CkoError()
    sv = solver.c()
    raise_for(lib().cko_adjoint_chunk_solve(ctx.h, ctx.model(model), dptr(_f64(traj.states)), dptr(traj.grid.times),
                                            traj.n_batch, traj.n_time, int(step_hi), int(chunk_len), dptr(dL),
                                            C.byref(sv), dptr(lam), dptr(grad), C.byref(w), C.byref(e)), e)
    state.lam[...] = lam
    state.grad[...] = grad
    if work is not None:
        work += WorkCounters.from_c(w)


def adjoint_step_sequential(model: Model, y_i, y_prev, t_i, t_prev, dL_dy_i, state: AdjointState,
                            solver: SolverChoice | None = None, ctx: Context | None = None) -> None:
    """adjoint.hpp:36-47: one reverse backward-Euler step, state updated in place."""
    solver = solver or SolverChoice()
    y_i, y_prev, dl = _f64(y_i), _f64(y_prev), _f64(dL_dy_i)
    t_i, t_prev = _f64(t_i), _f64(t_prev)
    nb, n = y_i.shape
    if n != model.state_size:
        raise ShapeMismatch("adjoint step: state width != model size")
    if y_prev.shape != (nb, n):
        raise ShapeMismatch("adjoint step: y_prev shape")
    if t_i.shape != (nb,) or t_prev.shape != (nb,):
        raise ShapeMismatch("adjoint step: time spans")
    if dl.shape != (nb, n):
        raise ShapeMismatch("adjoint step: loss jump shape")
    _check_state(model, state, nb)
    ctx = ctx or default_context()
    lam, grad = _f64(state.lam).copy(), _f64(state.grad).copy()
    e = abi.CkoError()
    sv = solver.c()
    raise_for(lib().cko_adjoint_step_sequential(ctx.h, ctx.model(model), dptr(y_i), dptr(y_prev), dptr(t_i),
                                                dptr(t_prev), dptr(dl), nb, C.byref(sv), dptr(lam), dptr(grad),
                                                C.byref(e)), e)
    state.lam[...] = lam
    state.grad[...] = grad


# ---------------------------------------------------------------------------
# block-bidiagonal solvers (linalg.hpp:19-87)
# ---------------------------------------------------------------------------
@dataclass
class BlockBidiagonalSystem:
    diag: np.ndarray       # (nc, nb, n, n)
    offdiag: np.ndarray    # (nc - 1, nb, n, n)

    @classmethod
    def zeros(cls, n_chunk, n_batch, n_size):
        return cls(np.zeros((n_chunk, n_batch, n_size, n_size)),
                   np.zeros((max(n_chunk - 1, 0), n_batch, n_size, n_size)))


def _solve(sys_diag, sys_off, rhs, solver: SolverChoice, unit: bool, ctx: Context | None):
    ctx = ctx or default_context()
    diag = _f64(sys_diag)
    if diag.ndim != 4 or diag.shape[2] != diag.shape[3]:
        raise ShapeMismatch("block bidiagonal system must be non-empty")
    nc, nb, n, _ = diag.shape
    x = _f64(rhs).copy()
    if x.shape != (nc, nb, n):
        raise ShapeMismatch("right-hand side shape must match the system")
    off = None
    if not unit:
        off = _f64(sys_off)
        if nc > 1 and off.shape != (nc - 1, nb, n, n):
            raise ShapeMismatch("off-diagonal block array must be (n_chunk-1, n_batch, n_size, n_size)")
    sw = C.c_longlong(0)
    e = abi.CkoError()
    sv = solver.c()
    rc = lib().cko_block_bidiag_solve(ctx.h, C.byref(sv), nc, nb, n, dptr(diag),
                                      dptr(off) if off is not None else None, dptr(x), C.byref(sw), C.byref(e))
    raise_for(rc, e)
    return x, int(sw.value)


def solve_thomas(sys: BlockBidiagonalSystem, rhs, ctx=None) -> np.ndarray:
    return _solve(sys.diag, sys.offdiag, rhs, SolverChoice(SolverKind.thomas), False, ctx)[0]


def solve_pcr(sys: BlockBidiagonalSystem, rhs, ctx=None):
    """Returns (x, sweep_count) — sweep_count is the reference's out-parameter."""
    return _solve(sys.diag, sys.offdiag, rhs, SolverChoice(SolverKind.pcr), False, ctx)


def solve_hybrid(sys: BlockBidiagonalSystem, rhs, n_switch: int, ctx=None):
    if n_switch < 0:
        raise Error("solve_hybrid: n_switch must be >= 0")
    return _solve(sys.diag, sys.offdiag, rhs, SolverChoice(SolverKind.hybrid, n_switch), False, ctx)


def solve_unit_offdiag(diag, rhs, solver: SolverChoice, ctx=None):
    """detail::solve_unit_offdiag (linalg.cpp:288-303): couplings exactly -I."""
    return _solve(diag, None, rhs, solver, True, ctx)
