"""Batch sharding across GPUs: one process per GPU.

join() gives every rank's context a view of every rank's exchange buffer:
each rank allocates a buffer and exports a CUDA IPC handle
(cko_comm_alloc), the handles travel once through torch.distributed
(all_gather_object, any backend), and each rank maps its peers' buffers
(cko_comm_open). From then on the kernels exchange data directly over
NVLink / NVSwitch with P2P stores: the Newton convergence flag every
iteration (the all-lanes predicate of integrate.cpp:176-182 spans every
shard), and the loss / gradient sums once per adjoint pass.
"""
from __future__ import annotations

import ctypes as C

from . import abi
from ._native import lib
from .errors import raise_for


def join(ctx, rank: int, world: int, gather=None):
    """Attach `ctx` to a group of `world` ranks. `gather(obj) -> list` defaults to
    torch.distributed.all_gather_object on the default process group."""
    L = lib()
    if world <= 1:
        return
    if gather is None:
        import torch.distributed as dist

        def gather(obj):
            out = [None] * world
            dist.all_gather_object(out, obj)
            return out
    own = C.c_void_p()
    handle = C.create_string_buffer(64)
    e = abi.CkoError()
    raise_for(L.cko_comm_alloc(ctx.h, C.byref(own), handle, C.byref(e)), e)
    handles = gather(bytes(handle.raw))
    ptrs = (C.c_void_p * world)()
    for r in range(world):
        if r == rank:
            ptrs[r] = own.value
            continue
        peer = C.c_void_p()
        raise_for(L.cko_comm_open(ctx.h, C.create_string_buffer(handles[r], 64), C.byref(peer), C.byref(e)), e)
        ptrs[r] = peer.value
    raise_for(L.cko_ctx_set_group(ctx.h, rank, world, ptrs, C.byref(e)), e)
    ctx._group = (own, ptrs)
    # every rank must have mapped its peers before any kernel writes into them
    gather(b"ready")
