"""Batch sharding through the real device exchange, on one GPU.

Two contexts on device 0 form a world-2 group (each rank's exchange buffer is a
plain device allocation of this process, so no IPC is needed); two host threads
run the ranks' forward + adjoint concurrently, small enough that both
cooperative kernels are co-resident. The per-iteration Newton predicate
exchange, the loss sum and the gradient sum must reproduce the single-process
oracle on the full batch: states per shard, loss, gradient and WorkCounters
(strict-parity mode).
"""
import ctypes as C
import os
import threading

import numpy as np
import pytest

import paper_2310_08649_b200 as P
from paper_2310_08649_b200 import abi, api
from paper_2310_08649_b200._native import lib
from paper_2310_08649_b200.errors import raise_for
from tests.cases import chaboche_plastic
from tests.conftest import rel_max, uniform_times

pytestmark = pytest.mark.gpu
TOL = 1e-10


def _group(ctxs):
    L = lib()
    world = len(ctxs)
    bufs = []
    for c in ctxs:
        p = C.c_void_p()
        h = C.create_string_buffer(64)
        e = abi.CkoError()
        raise_for(L.cko_comm_alloc(c.h, C.byref(p), h, C.byref(e)), e)
        bufs.append(p.value)
    ptrs = (C.c_void_p * world)(*bufs)
    for r, c in enumerate(ctxs):
        e = abi.CkoError()
        raise_for(L.cko_ctx_set_group(c.h, r, world, ptrs, C.byref(e)), e)


def _run_group(full, nb_local, world, y0, t_local, nc, solver):
    # No retry: the one-GPU emulation used to stall when a rank's host thread launched a group-only kernel
    # for the first time (lazy module loading waits for the device while the peer kernel spins on the
    # exchange). cko_ctx_set_group now loads every kernel up front (cko::preload_kernels).
    return _run_group_once(full, nb_local, world, y0, t_local, nc, solver)


def _run_group_once(full, nb_local, world, y0, t_local, nc, solver):
    ctxs = [api.Context(0) for _ in range(world)]
    shards = [full.shard(r * nb_local) for r in range(world)]
    grids = [api.TimeGrid(t) for t in t_local] if isinstance(t_local, list) else [api.TimeGrid(t_local)] * world
    sv = api.SolverChoice(*solver)
    # allocate every buffer first (world 1), so the concurrent runs never free / grow device memory
    for r in range(world):
        api.gradient_adjoint(shards[r], y0[r * nb_local:(r + 1) * nb_local], grids[r], nc, solver=sv, ctx=ctxs[r])
    _group(ctxs)
    os.environ["CKO_PLAIN_LAUNCH"] = "1"  # two ranks' grids concurrently on one GPU (see cko_common.cuh)
    out, errs = [None] * world, [None] * world

    def rank(r):
        try:
            out[r] = api.gradient_adjoint(shards[r], y0[r * nb_local:(r + 1) * nb_local], grids[r], nc, solver=sv,
                                          ctx=ctxs[r])
            out[r].sp_bits = ctxs[r].structured_used()
        except Exception as ex:  # surfaced below
            errs[r] = ex

    th = [threading.Thread(target=rank, args=(r,)) for r in range(world)]
    for t in th:
        t.start()
    for t in th:
        t.join(timeout=120)
    del os.environ["CKO_PLAIN_LAUNCH"]
    for ex in errs:
        if ex is not None:
            raise ex
    return out


@pytest.mark.parametrize("solver", [(0, 1), (1, 1)])
def test_two_ranks_match_single_process(port, solver):
    world, nb_local, nt, nc = 2, 3, 48, 8
    full = chaboche_plastic(3, nb_local * world)
    y0 = np.zeros((nb_local * world, 5))
    t_full = uniform_times(nt, nb_local * world, 5.0)
    want = port.gradient(full, y0, t_full, nc, solver=solver)
    got = _run_group(full, nb_local, world, y0, uniform_times(nt, nb_local, 5.0), nc, solver)
    n = 5
    for r, g in enumerate(got):
        cols = slice(r * nb_local * n, (r + 1) * nb_local * n)
        assert g.trajectory.work.as_dict() == want.fwd, "forward WorkCounters differ (global predicate)"
        assert g.backward_work.as_dict() == want.bwd
        assert rel_max(g.trajectory.states, want.states[:, cols]) <= TOL
        assert abs(g.loss - want.loss) <= TOL * abs(want.loss)
        assert rel_max(g.gradient, want.grad) <= TOL
    assert np.array_equal(got[0].gradient, got[1].gradient), "ranks must hold bitwise-identical sums"


def test_two_ranks_mds_sequential_edge(port):
    """MDS at n_chunk = 1: early chunks converge at iteration 0 only because EVERY lane does; a shard-local
    predicate would give different Newton counts."""
    world, nb_local, nt, nc = 2, 4, 120, 1
    full = P.build_mass_damper_spring(10, nb_local * world)
    y0 = np.zeros((nb_local * world, 20))
    want = port.gradient(full, y0, uniform_times(nt, nb_local * world, nt * 1e-6), nc)
    got = _run_group(full, nb_local, world, y0, uniform_times(nt, nb_local, nt * 1e-6), nc, (0, 1))
    for r, g in enumerate(got):
        cols = slice(r * nb_local * 20, (r + 1) * nb_local * 20)
        assert g.trajectory.work.as_dict() == want.fwd
        assert rel_max(g.trajectory.states, want.states[:, cols]) <= TOL
        assert rel_max(g.gradient, want.grad) <= TOL


def test_two_ranks_structured_fallback_on_one_rank(port):
    """Structured MDS kernels in a group: one lane of rank 1 has steps at which the reference pivots. Its
    forward raises the fallback flag; the group exchange carries it, so BOTH ranks stop at the same iteration
    and re-run on the group-LU kernels (no rank waits on a peer that left). Results match the oracle on the
    full batch."""
    world, nb_local, nt, nc = 2, 4, 24, 6
    full = P.build_mass_damper_spring(10, nb_local * world)
    y0 = np.random.default_rng(5).uniform(-1e-3, 1e-3, (nb_local * world, 20))
    t_full = uniform_times(nt, nb_local * world, nt * 1e-6)
    t_full[:, nb_local + 2] = np.linspace(0.0, nt * 5e-4, nt + 1)  # global lane 6: rank 1's local lane 2
    want = port.gradient(full, y0, t_full, nc)
    t_ranks = [np.ascontiguousarray(t_full[:, r * nb_local:(r + 1) * nb_local]) for r in range(world)]
    got = _run_group(full, nb_local, world, y0, t_ranks, nc, (0, 1))
    for r, g in enumerate(got):
        assert g.sp_bits & api.Context.SP_FWD_FALLBACK, (r, g.sp_bits)
        cols = slice(r * nb_local * 20, (r + 1) * nb_local * 20)
        assert g.trajectory.work.as_dict() == want.fwd
        assert rel_max(g.trajectory.states, want.states[:, cols]) <= TOL
        assert abs(g.loss - want.loss) <= TOL * abs(want.loss)
        assert rel_max(g.gradient, want.grad) <= TOL
