"""Model descriptors: the host-side image of the reference OdeModel identity.

Builders mirror /root/reference/proj/core/include/chunkode/models.hpp:14-41
and produce the exact default parameter vectors of the reference builders
(linspace rules of models_mds.cpp:85-94, models_chaboche.cpp:188-197, the
mt19937_64 draws of models_node.cpp:183-199). A Model carries no code: the
device twin is selected by `kind` inside the CUDA library.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, field, replace

import numpy as np

from . import abi
from .errors import ShapeMismatch


def linspace(lo: float, hi: float, n: int) -> np.ndarray:
    """chunkode::linspace (linalg.cpp:386-396): lo + (hi-lo)*i/(n-1), last = hi."""
    if n <= 0:
        return np.zeros(0)
    if n == 1:
        return np.array([lo], dtype=np.float64)
    v = np.array([lo + (hi - lo) * float(i) / float(n - 1) for i in range(n)], dtype=np.float64)
    v[-1] = hi
    return v


class MT19937_64:
    """std::mt19937_64 (the engine the reference NODE init uses)."""

    def __init__(self, seed: int):
        self.mt = [0] * 312
        self.mt[0] = seed & 0xFFFFFFFFFFFFFFFF
        for i in range(1, 312):
            self.mt[i] = (6364136223846793005 * (self.mt[i - 1] ^ (self.mt[i - 1] >> 62)) + i) & 0xFFFFFFFFFFFFFFFF
        self.idx = 312

    def __call__(self) -> int:
        if self.idx >= 312:
            mt = self.mt
            for i in range(312):
                x = (mt[i] & 0xFFFFFFFF80000000) | (mt[(i + 1) % 312] & 0x7FFFFFFF)
                xa = x >> 1
                if x & 1:
                    xa ^= 0xB5026F5AA96619E9
                mt[i] = mt[(i + 156) % 312] ^ xa
            self.idx = 0
        y = self.mt[self.idx]
        self.idx += 1
        y ^= (y >> 29) & 0x5555555555555555
        y ^= (y << 17) & 0x71D67FFFEDA60000
        y ^= (y << 37) & 0xFFF7EEE000000000
        y ^= y >> 43
        return y & 0xFFFFFFFFFFFFFFFF


_NAMES = {
    abi.CKO_MODEL_SCALAR_DECAY: "scalar_decay",
    abi.CKO_MODEL_CONSTANT_RATE: "constant_rate",
    abi.CKO_MODEL_LIN3: "lin3",
    abi.CKO_MODEL_MDS: "mds",
    abi.CKO_MODEL_CHABOCHE: "chaboche",
    abi.CKO_MODEL_NODE: "node",
    abi.CKO_MODEL_NEURON: "neuron",
}


@dataclass(frozen=True)
class Model:
    """Immutable model identity (ode_model.hpp:24-25): kind + dims + params."""

    kind: int
    params: np.ndarray
    n_unit: int = 0
    width: int = 0
    n_batch: int = 0  # parameterised batch width; 0 = any (OdeModel::n_batch)
    lane_offset: int = 0
    _keep: list = field(default_factory=list, repr=False, compare=False)

    @property
    def name(self) -> str:
        if self.kind == abi.CKO_MODEL_NODE and self.width != self.n_unit + 1:
            return "node_wide"
        return _NAMES[self.kind]

    @property
    def state_size(self) -> int:
        return {
            abi.CKO_MODEL_SCALAR_DECAY: 1,
            abi.CKO_MODEL_CONSTANT_RATE: 1,
            abi.CKO_MODEL_LIN3: 3,
            abi.CKO_MODEL_MDS: 2 * self.n_unit,
            abi.CKO_MODEL_CHABOCHE: 2 + self.n_unit,
            abi.CKO_MODEL_NODE: self.n_unit,
            abi.CKO_MODEL_NEURON: 4 * self.n_unit,
        }[self.kind]

    @property
    def default_t_max(self) -> float:
        return 10.0 if self.kind in (abi.CKO_MODEL_CHABOCHE, abi.CKO_MODEL_NEURON) else 1.0

    def with_params(self, p) -> "Model":
        """OdeModel::with_params (ode_model.hpp:112-117): count must not change."""
        p = np.ascontiguousarray(p, dtype=np.float64).copy()
        if p.size != self.params.size:
            raise ShapeMismatch("with_params: parameter count must not change")
        return replace(self, params=p, _keep=[])

    def shard(self, lane_offset: int) -> "Model":
        """Same parameters, local lane 0 mapped to global lane `lane_offset`."""
        return replace(self, lane_offset=lane_offset, _keep=[])

    def desc(self) -> abi.CkoModelDesc:
        p = np.ascontiguousarray(self.params, dtype=np.float64)
        self._keep.clear()
        self._keep.append(p)
        return abi.CkoModelDesc(self.kind, self.n_unit, self.width, self.n_batch, self.lane_offset,
                                int(p.size), p.ctypes.data_as(C.POINTER(C.c_double)))


def build_scalar_decay(p0: float) -> Model:
    """models_simple.cpp:9-27 / :62-64."""
    return Model(abi.CKO_MODEL_SCALAR_DECAY, np.array([p0], dtype=np.float64))


def build_constant_rate(c0: float) -> Model:
    """models_simple.cpp:29-45 / :66-68."""
    return Model(abi.CKO_MODEL_CONSTANT_RATE, np.array([c0], dtype=np.float64))


def build_mass_damper_spring(n_unit: int, n_batch: int) -> Model:
    """models_mds.cpp:85-104: [K linspace(1e-2,1), C linspace(1e-6,1e-4), M linspace(1e-7,1e-5), f_a=1, T linspace(1e-2,1,nb)]."""
    if n_unit < 1 or n_batch < 1:
        raise ShapeMismatch("build_mass_damper_spring: n_unit, n_batch >= 1")
    p = np.concatenate([linspace(1e-2, 1.0, n_unit), linspace(1e-6, 1e-4, n_unit),
                        linspace(1e-7, 1e-5, n_unit), [1.0], linspace(1e-2, 1.0, n_batch)])
    return Model(abi.CKO_MODEL_MDS, p, n_unit=n_unit, n_batch=n_batch)


def build_chaboche(n_unit: int, n_batch: int) -> Model:
    """models_chaboche.cpp:188-202: [E,n,eta,s0,Kinf,tau]=[10,5,2,1,10,1], C, gamma, eps_a, T=1."""
    if n_unit < 1 or n_batch < 1:
        raise ShapeMismatch("build_chaboche: n_unit, n_batch >= 1")
    p = np.concatenate([[10.0, 5.0, 2.0, 1.0, 10.0, 1.0], linspace(0.1, 1.0, n_unit),
                        linspace(0.1, 0.5, n_unit), linspace(0.1, 1.0, n_batch), [1.0]])
    return Model(abi.CKO_MODEL_CHABOCHE, p, n_unit=n_unit, n_batch=n_batch)


def _node_params(n: int, width: int, seed: int, fan_ins) -> np.ndarray:
    gen = MT19937_64(seed)
    out = []
    for rows, fan_in in fan_ins:
        half = float(np.sqrt(1.0 / float(fan_in)))
        for _ in range(rows * fan_in + rows):
            u = float(gen() >> 11) * 2.0 ** -53
            out.append(-half + 2.0 * half * u)
    return np.array(out, dtype=np.float64)


def build_neural_ode(n_unit: int, n_batch: int, seed: int = 7) -> Model:
    """models_node.cpp:13-212: widths (n+1 -> n+1 -> n+1 -> n), U(+-sqrt(1/(n+1)))."""
    if n_unit < 1 or n_batch < 1:
        raise ShapeMismatch("build_neural_ode: n_unit, n_batch >= 1")
    w = n_unit + 1
    # every layer of the reference draws from +-sqrt(1/(n+1)); draw order W1,b1,W2,b2,W3,b3
    p = _node_params(n_unit, w, seed, [(w, w), (w, w), (n_unit, w)])
    return Model(abi.CKO_MODEL_NODE, p, n_unit=n_unit, width=w, n_batch=n_batch)


def build_node_wide(n: int, width: int, n_batch: int, seed: int = 7) -> Model:
    """(n+1 -> W -> W -> n), U(+-sqrt(1/fan_in)) per layer."""
    p = _node_params(n, width, seed, [(width, n + 1), (width, width), (n, width)])
    return Model(abi.CKO_MODEL_NODE, p, n_unit=n, width=width, n_batch=n_batch)


def build_neuron(n_unit: int, n_batch: int, period: float | None = None) -> Model:
    """models_neuron.cpp:110-148: fourteen per-unit segments (linspace rules), I_a = linspace(0.1, 1, nb),
    then the per-unit drive periods T = linspace(0.5, 2, u) (or a constant override)."""
    if n_unit < 1 or n_batch < 1:
        raise ShapeMismatch("build_neuron: n_unit, n_batch >= 1")
    u = n_unit
    seg = [(0.1, 1.0)] * 8 + [(0.5, 5.0), (0.1, 1.0), (1.5, 15.0), (0.1, 1.0), (1.0, 10.0), (1e-3, 1e-2)]
    parts = [linspace(lo, hi, u) for lo, hi in seg] + [linspace(0.1, 1.0, n_batch)]
    parts.append(np.full(u, float(period)) if period is not None else linspace(0.5, 2.0, u))
    return Model(abi.CKO_MODEL_NEURON, np.concatenate(parts), n_unit=u, n_batch=n_batch)


def build_lin3(n_batch: int) -> Model:
    """A = [[-1,.5,0],[.5,-1e3,10],[0,10,-1e6]], f_a = 1, T_b = linspace(1e-2,1,nb)."""
    p = np.array([-1.0, 0.5, 0.0, 0.5, -1e3, 10.0, 0.0, 10.0, -1e6, 1.0], dtype=np.float64)
    return Model(abi.CKO_MODEL_LIN3, p, n_batch=n_batch)


def build_problem(key: str, n_unit: int, n_batch: int, seed: int = 7) -> Model:
    """models_simple.cpp:70-76 (plus lin3 / node_wide)."""
    if key == "mds":
        return build_mass_damper_spring(n_unit, n_batch)
    if key == "chaboche":
        return build_chaboche(n_unit, n_batch)
    if key == "node":
        return build_neural_ode(n_unit, n_batch, seed)
    if key == "lin3":
        return build_lin3(n_batch)
    if key == "neuron":
        return build_neuron(n_unit, n_batch)
    from .errors import Error
    raise Error(f"unknown problem '{key}' (expected mds, chaboche, node, or lin3)")


def param_count(kind: int, n_unit: int = 0, width: int = 0, n_batch: int = 0) -> int:
    u, W, nb = n_unit, width, n_batch
    return {
        abi.CKO_MODEL_SCALAR_DECAY: 1,
        abi.CKO_MODEL_CONSTANT_RATE: 1,
        abi.CKO_MODEL_LIN3: 10,
        abi.CKO_MODEL_MDS: 3 * u + 1 + nb,
        abi.CKO_MODEL_CHABOCHE: 6 + 2 * u + nb + 1,
        abi.CKO_MODEL_NODE: W * (u + 1) + W + W * W + W + u * W + u,
        abi.CKO_MODEL_NEURON: 15 * u + nb,
    }[kind]
