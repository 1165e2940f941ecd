"""Batch sharding host logic, world_size 2 over gloo on CPU.

Checks the decomposition the multi-GPU path relies on: lane
shards addressed through lane_offset see the global per-lane parameters,
the Frobenius loss is the rank sum of squares, and the gradient is the rank
sum of shard gradients computed with the global loss. The per-shard compute
here is the CPU oracle; the group join protocol (IPC handle exchange) runs
against a stub library.
"""
import os
import socket

import numpy as np
import pytest
import torch.distributed as dist
import torch.multiprocessing as mp

import paper_2310_08649_b200 as P
from tests.conftest import rel_max, uniform_times


def free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def worker(rank, world, port, out):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import torch
    from oracle import load_port
    orc = load_port()
    nb_local, nt, nc = 3, 40, 8
    full = P.build_mass_damper_spring(3, nb_local * world)
    shard = full.shard(rank * nb_local)
    t = uniform_times(nt, nb_local, 2e-3)
    y0 = np.zeros((nb_local, shard.state_size))
    f = orc.forward(shard, y0, t, nc)
    ss = torch.tensor([float(np.sum(f.states[1:] ** 2))], dtype=torch.float64)
    dist.all_reduce(ss)
    L = float(np.sqrt(ss.item()))
    dL = np.zeros_like(f.states)
    dL[1:] = f.states[1:] / L
    a = orc.adjoint(shard, f.states, t, nc, dL=dL)
    g = torch.from_numpy(a.grad.copy())
    dist.all_reduce(g)
    # group join protocol against a stub library
    from paper_2310_08649_b200 import group

    class StubLib:
        def __init__(self):
            self.table = None

        def cko_comm_alloc(self, h, own, handle, e):
            own._obj.value = 0x1000 * (rank + 1)
            handle.raw = bytes([rank]) * 64
            return 0

        def cko_comm_open(self, h, handle, peer, e):
            peer._obj.value = 0x1000 * (handle.raw[0] + 1) + 0x10
            return 0

        def cko_ctx_set_group(self, h, r, w, ptrs, e):
            self.table = (r, w, [ptrs[i] for i in range(w)])
            return 0

    stub = StubLib()
    orig = group.lib
    group.lib = lambda: stub

    class Ctx:
        h = None
    try:
        group.join(Ctx(), rank, world)
    finally:
        group.lib = orig
    if rank == 0:
        out.put((L, g.numpy(), stub.table))
    else:
        out.put(("table", stub.table))
    dist.destroy_process_group()


def test_two_rank_shard_sum_matches_unsharded(port):
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    p = free_port()
    procs = [ctx.Process(target=worker, args=(r, world, p, q)) for r in range(world)]
    for pr in procs:
        pr.start()
    res = [q.get(timeout=120) for _ in range(world)]
    for pr in procs:
        pr.join(timeout=60)
        assert pr.exitcode == 0
    L, g, table0 = next(r for r in res if r[0] != "table")
    table1 = next(r for r in res if r[0] == "table")[1]
    # unsharded oracle on the full batch
    full = P.build_mass_damper_spring(3, 6)
    want = port.gradient(full, np.zeros((6, 6)), uniform_times(40, 6, 2e-3), 8)
    assert abs(L - want.loss) <= 1e-13 * want.loss
    assert rel_max(g, want.grad) <= 1e-12
    # each rank sees its own buffer at its index and the mapped peer elsewhere
    assert table0 == (0, 2, [0x1000, 0x2000 + 0x10])
    assert table1 == (1, 2, [0x1000 + 0x10, 0x2000])
