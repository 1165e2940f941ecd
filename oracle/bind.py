"""ctypes bindings of the two CPU checkers (TEST INFRASTRUCTURE ONLY)."""
from __future__ import annotations

import ctypes as C
import os
import subprocess
from dataclasses import dataclass

import numpy as np

from paper_2310_08649_b200 import abi
from paper_2310_08649_b200.abi import dptr
from paper_2310_08649_b200.errors import raise_for

HERE = os.path.dirname(os.path.abspath(__file__))
PORT_SO = os.path.join(HERE, "_build", "libcko_oracle.so")
REF_SO = os.path.join(HERE, "_ref", "libchunkode_ref.so")
REF_SRC = "/root/reference/proj/core"

_P = C.POINTER


def build(ref: bool | None = None) -> None:
    """Compile the restatement, and the reference too when its sources exist."""
    subprocess.run(["make", "-s", "-C", HERE, "all"], check=True)
    if ref is None:
        ref = os.path.isdir(REF_SRC)
    if ref:
        subprocess.run(["make", "-s", "-C", HERE, "ref"], check=True)


def ref_available() -> bool:
    return os.path.exists(REF_SO)


@dataclass
class Result:
    states: np.ndarray | None = None
    loss: float | None = None
    grad: np.ndarray | None = None
    fwd: dict | None = None
    bwd: dict | None = None
    seconds: tuple | None = None


def work_dict(w: abi.CkoWork) -> dict:
    return {k: int(getattr(w, k)) for k, _ in abi.CkoWork._fields_}


class Oracle:
    """One CPU checker. kind = 'port' (C restatement) or 'ref' (compiled reference)."""

    def __init__(self, kind: str):
        self.kind = kind
        path = PORT_SO if kind == "port" else REF_SO
        if not os.path.exists(path):
            build(ref=(kind == "ref"))
        self.lib = C.CDLL(path)
        L = self.lib
        if kind == "port":
            L.cko_oracle_forward.restype = C.c_int
            L.cko_oracle_adjoint.restype = C.c_int
            L.cko_oracle_solve.restype = C.c_int
            L.cko_oracle_sharded_timing.restype = C.c_double
            self._fwd = L.cko_oracle_forward
            self._adj = L.cko_oracle_adjoint
            self._solve = L.cko_oracle_solve
        else:
            L.ref_forward.restype = C.c_int
            L.ref_adjoint.restype = C.c_int
            L.ref_solve.restype = C.c_int
            L.ref_gradient_adjoint.restype = C.c_int
            L.ref_sharded_seconds.restype = C.c_double
            L.ref_default_params.restype = C.c_int
            self._fwd = L.ref_forward
            self._adj = L.ref_adjoint
            self._solve = L.ref_solve

    # -- integrator / adjoint -------------------------------------------------
    def forward(self, model, y0, times, n_chunk, settings=(1e-8, 1e-6, 100), solver=(0, 1)):
        y0 = np.ascontiguousarray(y0, np.float64)
        times = np.ascontiguousarray(times, np.float64)
        nt, nb = times.shape[0] - 1, times.shape[1]
        n = model.state_size
        states = np.zeros((nt + 1, nb * n))
        st = abi.CkoNewtonSettings(*settings)
        sv = abi.CkoSolverChoice(*solver)
        w, e = abi.CkoWork(), abi.CkoError()
        d = model.desc()
        rc = self._fwd(C.byref(d), dptr(y0), dptr(times), nb, nt, n_chunk, C.byref(st), C.byref(sv),
                       dptr(states), C.byref(w), C.byref(e))
        raise_for(rc, e)
        return Result(states=states, fwd=work_dict(w))

    def adjoint(self, model, states, times, n_chunk, solver=(0, 1), dL=None):
        states = np.ascontiguousarray(states, np.float64)
        times = np.ascontiguousarray(times, np.float64)
        nt, nb = times.shape[0] - 1, times.shape[1]
        grad = np.zeros(model.params.size)
        L = C.c_double(0.0)
        sv = abi.CkoSolverChoice(*solver)
        w, e = abi.CkoWork(), abi.CkoError()
        d = model.desc()
        kind = abi.CKO_LOSS_FROBENIUS if dL is None else abi.CKO_LOSS_USER
        dLa = None if dL is None else np.ascontiguousarray(dL, np.float64)
        rc = self._adj(C.byref(d), dptr(states), dptr(times), nb, nt, n_chunk, C.byref(sv), kind,
                       dptr(dLa), C.byref(L), dptr(grad), C.byref(w), C.byref(e))
        raise_for(rc, e)
        return Result(loss=L.value, grad=grad, bwd=work_dict(w))

    def gradient(self, model, y0, times, n_chunk, settings=(1e-8, 1e-6, 100), solver=(0, 1)):
        f = self.forward(model, y0, times, n_chunk, settings, solver)
        a = self.adjoint(model, f.states, times, n_chunk, solver)
        return Result(states=f.states, loss=a.loss, grad=a.grad, fwd=f.fwd, bwd=a.bwd)

    # -- solver ---------------------------------------------------------------
    def solve(self, diag, offdiag, rhs, solver=(0, 1)):
        diag = np.ascontiguousarray(diag, np.float64)
        nc, nb, n, _ = diag.shape
        x = np.ascontiguousarray(rhs, np.float64).copy()
        off = None if offdiag is None else np.ascontiguousarray(offdiag, np.float64)
        sw = C.c_longlong(0)
        sv = abi.CkoSolverChoice(*solver)
        e = abi.CkoError()
        rc = self._solve(C.byref(sv), nc, nb, n, dptr(diag), dptr(off), dptr(x), C.byref(sw), C.byref(e))
        raise_for(rc, e)
        return x, int(sw.value)

    # -- timing baselines -------------------------------------------------------
    def timed_gradient(self, model, y0, times, n_chunk, settings=(1e-8, 1e-6, 100), solver=(0, 1)):
        """Reference only: gradient_adjoint with steady_clock around both phases."""
        assert self.kind == "ref"
        y0 = np.ascontiguousarray(y0, np.float64)
        times = np.ascontiguousarray(times, np.float64)
        nt, nb = times.shape[0] - 1, times.shape[1]
        grad = np.zeros(model.params.size)
        L = C.c_double(0.0)
        secs = (C.c_double * 2)()
        st, sv = abi.CkoNewtonSettings(*settings), abi.CkoSolverChoice(*solver)
        wf, wb, e = abi.CkoWork(), abi.CkoWork(), abi.CkoError()
        d = model.desc()
        rc = self.lib.ref_gradient_adjoint(C.byref(d), dptr(y0), dptr(times), nb, nt, n_chunk, C.byref(st),
                                           C.byref(sv), None, C.byref(L), dptr(grad), C.byref(wf), C.byref(wb),
                                           secs, C.byref(e))
        raise_for(rc, e)
        return Result(loss=L.value, grad=grad, fwd=work_dict(wf), bwd=work_dict(wb), seconds=(secs[0], secs[1]))

    def sharded_seconds(self, model, y0, times, n_chunk, threads, settings=(1e-8, 1e-6, 100), solver=(0, 1)):
        y0 = np.ascontiguousarray(y0, np.float64)
        times = np.ascontiguousarray(times, np.float64)
        nt, nb = times.shape[0] - 1, times.shape[1]
        st, sv = abi.CkoNewtonSettings(*settings), abi.CkoSolverChoice(*solver)
        d = model.desc()
        fn = self.lib.ref_sharded_seconds if self.kind == "ref" else self.lib.cko_oracle_sharded_timing
        return float(fn(C.byref(d), dptr(y0), dptr(times), nb, nt, n_chunk, C.byref(st), C.byref(sv), threads))

    # -- reference-only helpers ------------------------------------------------
    def default_params(self, model, seed=7):
        assert self.kind == "ref"
        buf = np.zeros(max(model.params.size, 1) + 16)
        e = abi.CkoError()
        d = model.desc()
        k = self.lib.ref_default_params(C.byref(d), C.c_ulonglong(seed), dptr(buf), buf.size, C.byref(e))
        if k < 0:
            raise_for(-k, e)
        return buf[:k].copy()

    def random_system(self, nc, nb, n, seed):
        assert self.kind == "ref"
        diag = np.zeros((nc, nb, n, n))
        off = np.zeros((max(nc - 1, 0), nb, n, n))
        self.lib.ref_random_system(nc, nb, n, C.c_ulonglong(seed), dptr(diag), dptr(off))
        return diag, off

    def random_rhs(self, nc, nb, n, seed):
        assert self.kind == "ref"
        rhs = np.zeros((nc, nb, n))
        self.lib.ref_random_rhs(nc, nb, n, C.c_ulonglong(seed), dptr(rhs))
        return rhs

    def solve_dense(self, diag, offdiag, rhs):
        assert self.kind == "ref"
        diag = np.ascontiguousarray(diag, np.float64)
        nc, nb, n, _ = diag.shape
        x = np.ascontiguousarray(rhs, np.float64).copy()
        off = np.ascontiguousarray(offdiag, np.float64)
        e = abi.CkoError()
        rc = self.lib.ref_solve_dense(nc, nb, n, dptr(diag), dptr(off), dptr(x), C.byref(e))
        raise_for(rc, e)
        return x

    def set_jacobian_strategy(self, strategy: str) -> None:
        """JacobianStrategy of the following reference calls on this thread."""
        assert self.kind == "ref"
        self.lib.ref_set_jacobian_strategy({"analytic": 0, "forward_ad": 1, "finite_difference": 2}[strategy])

    # -- the reference's benchmark harness (reference only) -----------------------
    def _text(self, fn, *args):
        cap = 1 << 16
        while True:
            buf = C.create_string_buffer(cap)
            e = abi.CkoError()
            k = fn(*args, buf, cap, C.byref(e))
            if k == -1:
                raise_for(e.code or abi.CKO_ERROR, e)
            if k >= 0:
                return buf.value.decode()
            cap = -k + 16

    def study_csv(self, grid_text: str) -> str:
        assert self.kind == "ref"
        self.lib.ref_study_csv.restype = C.c_int
        return self._text(self.lib.ref_study_csv, grid_text.encode())

    def dump_trajectory(self, problem, n_unit, n_batch, n_time, n_chunk, solver="thomas", n_switch=1,
                        integration="backward", t_max=0.0) -> str:
        assert self.kind == "ref"
        self.lib.ref_dump_trajectory.restype = C.c_int
        return self._text(self.lib.ref_dump_trajectory, problem.encode(), n_unit, n_batch, n_time, n_chunk,
                          solver.encode(), n_switch, integration.encode(), C.c_double(t_max))

    # -- forward Euler scheme (reference only) ----------------------------------
    def fe_gradient(self, model, y0, times, n_chunk, dL=None):
        assert self.kind == "ref"
        y0 = np.ascontiguousarray(y0, np.float64)
        times = np.ascontiguousarray(times, np.float64)
        nt, nb = times.shape[0] - 1, times.shape[1]
        states = np.zeros((nt + 1, nb * model.state_size))
        wf, wb, e = abi.CkoWork(), abi.CkoWork(), abi.CkoError()
        d = model.desc()
        self.lib.ref_fe_forward.restype = C.c_int
        self.lib.ref_fe_adjoint.restype = C.c_int
        raise_for(self.lib.ref_fe_forward(C.byref(d), dptr(y0), dptr(times), nb, nt, n_chunk, dptr(states),
                                          C.byref(wf), C.byref(e)), e)
        grad = np.zeros(model.params.size)
        L = C.c_double(0.0)
        kind = abi.CKO_LOSS_FROBENIUS if dL is None else abi.CKO_LOSS_USER
        dLa = None if dL is None else np.ascontiguousarray(dL, np.float64)
        raise_for(self.lib.ref_fe_adjoint(C.byref(d), dptr(states), dptr(times), nb, nt, n_chunk, kind, dptr(dLa),
                                          C.byref(L), dptr(grad), C.byref(wb), C.byref(e)), e)
        return Result(states=states, loss=L.value, grad=grad, fwd=work_dict(wf), bwd=work_dict(wb))

    # -- public single-chunk ops (reference only) --------------------------------
    def chunk_op(self, model, op, y_start, dy, t_chunk, dt_chunk, settings=(1e-8, 1e-6, 100), solver=(0, 1)):
        """op 0 chunk_residual -> r; 1 chunk_jacobian -> (diag, offdiag); 2 newton_solve_chunk ->
        (dy, iterations, work)."""
        assert self.kind == "ref"
        y_start = np.ascontiguousarray(y_start, np.float64)
        dy = np.ascontiguousarray(dy, np.float64).copy()
        t_chunk = np.ascontiguousarray(t_chunk, np.float64)
        dt_chunk = np.ascontiguousarray(dt_chunk, np.float64)
        c, nb, n = dy.shape
        out = np.zeros((c, nb, n) if op == 0 else (c, nb, n, n))
        out2 = np.zeros((max(c - 1, 0), nb, n, n))
        st, sv = abi.CkoNewtonSettings(*settings), abi.CkoSolverChoice(*solver)
        it = C.c_int(0)
        w, e = abi.CkoWork(), abi.CkoError()
        d = model.desc()
        self.lib.ref_chunk_op.restype = C.c_int
        rc = self.lib.ref_chunk_op(C.byref(d), op, dptr(y_start), dptr(dy), dptr(t_chunk), dptr(dt_chunk), c, nb,
                                   C.byref(st), C.byref(sv), dptr(out), dptr(out2), C.byref(it), C.byref(w),
                                   C.byref(e))
        raise_for(rc, e)
        if op == 0:
            return out
        if op == 1:
            return out, out2
        return dy, int(it.value), work_dict(w)

    def adjoint_chunk(self, model, op, states, times, step_hi, chunk_len, dL, lam, grad, solver=(0, 1)):
        """op 0 adjoint_chunk_solve over (states, times, dL); op 1 adjoint_step_sequential with
        states/times/dL = 2-row [prev; i] arrays. Returns (lambda, grad, work)."""
        assert self.kind == "ref"
        states = np.ascontiguousarray(states, np.float64)
        times = np.ascontiguousarray(times, np.float64)
        dL = np.ascontiguousarray(dL, np.float64)
        lam = np.ascontiguousarray(lam, np.float64).copy()
        grad = np.ascontiguousarray(grad, np.float64).copy()
        nt, nb = times.shape[0] - 1, times.shape[1]
        sv = abi.CkoSolverChoice(*solver)
        w, e = abi.CkoWork(), abi.CkoError()
        d = model.desc()
        self.lib.ref_adjoint_chunk.restype = C.c_int
        rc = self.lib.ref_adjoint_chunk(C.byref(d), op, dptr(states), dptr(times), nb, nt, step_hi, chunk_len,
                                        dptr(dL), C.byref(sv), dptr(lam), dptr(grad), C.byref(w), C.byref(e))
        raise_for(rc, e)
        return lam, grad, work_dict(w)

    def model_eval(self, model, what, t, y, w=None):
        """what: 0 rate, 1 jacobian, 2 parameter_vjp (accumulated from zero)."""
        t = np.ascontiguousarray(t, np.float64)
        y = np.ascontiguousarray(y, np.float64)
        c, nb = t.shape
        n = model.state_size
        if what == 0:
            out = np.zeros((c, nb, n))
        elif what == 1:
            out = np.zeros((c, nb, n, n))
        else:
            out = np.zeros(model.params.size)
        d = model.desc()
        if self.kind == "ref":
            e = abi.CkoError()
            wa = None if w is None else np.ascontiguousarray(w, np.float64)
            rc = self.lib.ref_model_eval(C.byref(d), what, dptr(t), dptr(y), dptr(wa), c, nb, dptr(out), C.byref(e))
            raise_for(rc, e)
        else:
            fn = [self.lib.cko_oracle_rate, self.lib.cko_oracle_jacobian, self.lib.cko_oracle_param_vjp][what]
            if what == 2:
                wa = np.ascontiguousarray(w, np.float64)
                rc = fn(C.byref(d), dptr(t), dptr(y), dptr(wa), c, nb, dptr(out))
            else:
                rc = fn(C.byref(d), dptr(t), dptr(y), c, nb, dptr(out))
            assert rc == 0, rc
        return out


_cache: dict = {}


def load_port() -> Oracle:
    if "port" not in _cache:
        _cache["port"] = Oracle("port")
    return _cache["port"]


def load_ref() -> Oracle:
    if "ref" not in _cache:
        _cache["ref"] = Oracle("ref")
    return _cache["ref"]
