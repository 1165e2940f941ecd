"""Batch sharding across PROCESSES through CUDA IPC (the bench's multi-GPU plumbing), on one GPU.

Two spawned processes, one rank each: each allocates its exchange buffer, the
IPC handles travel through torch.distributed (gloo, 127.0.0.1), each maps its
peer's buffer (cko_comm_open) and runs forward + adjoint on its lane shard.
Without MPS the two contexts time-slice the GPU, so every exchange waits for
a context switch: small sizes only. The result must reproduce the
single-process oracle on the full batch (states per shard, loss, gradient,
WorkCounters), as on 2 GPUs.
"""
import os
import socket

import numpy as np
import pytest

from tests.conftest import ROOT, rel_max, uniform_times

pytestmark = pytest.mark.gpu
TOL = 1e-10


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _rank(rank, world, port, nb_local, nt, nc, out_dir):
    import sys
    sys.path.insert(0, ROOT)
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    import torch.distributed as dist

    from paper_2310_08649_b200 import api, group
    from tests.cases import chaboche_plastic
    dist.init_process_group("gloo", rank=rank, world_size=world)
    full = chaboche_plastic(3, nb_local * world)
    shard = full.shard(rank * nb_local)
    ctx = api.Context(0)
    group.join(ctx, rank, world)
    y0 = np.zeros((nb_local, 5))
    r = api.gradient_adjoint(shard, y0, api.TimeGrid(uniform_times(nt, nb_local, 5.0)), nc, ctx=ctx)
    np.savez(os.path.join(out_dir, f"rank{rank}.npz"), states=r.trajectory.states, loss=r.loss, grad=r.gradient,
             fwd=np.array(list(r.trajectory.work.as_dict().values())),
             bwd=np.array(list(r.backward_work.as_dict().values())))
    dist.barrier()
    dist.destroy_process_group()


def test_two_process_ipc_group(port, tmp_path):
    import torch.multiprocessing as mp

    from tests.cases import chaboche_plastic
    world, nb_local, nt, nc = 2, 3, 24, 8
    full = chaboche_plastic(3, nb_local * world)
    want = port.gradient(full, np.zeros((nb_local * world, 5)), uniform_times(nt, nb_local * world, 5.0), nc)
    mp.start_processes(_rank, args=(world, _free_port(), nb_local, nt, nc, str(tmp_path)), nprocs=world,
                       join=True, start_method="spawn")
    got = [np.load(tmp_path / f"rank{r}.npz") for r in range(world)]
    for r, g in enumerate(got):
        cols = slice(r * nb_local * 5, (r + 1) * nb_local * 5)
        assert list(g["fwd"]) == list(want.fwd.values()), "forward WorkCounters differ (global predicate)"
        assert list(g["bwd"]) == list(want.bwd.values())
        assert rel_max(g["states"], want.states[:, cols]) <= TOL
        assert abs(float(g["loss"]) - want.loss) <= TOL * abs(want.loss)
        assert rel_max(g["grad"], want.grad) <= TOL
    assert np.array_equal(got[0]["grad"], got[1]["grad"]), "ranks must hold bitwise-identical sums"
