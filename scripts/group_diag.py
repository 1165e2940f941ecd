"""Diagnostics for the single-GPU two-rank group run: call timing per thread."""
import ctypes as C
import os
import sys
import threading
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2310_08649_b200 import abi, api  # noqa: E402
from paper_2310_08649_b200._native import lib  # noqa: E402
from tests.cases import chaboche_plastic  # noqa: E402
from tests.conftest import uniform_times  # noqa: E402
from tests.test_gpu_group import _group  # noqa: E402

world, nbl, nt, nc = 2, 3, 48, 8
full = chaboche_plastic(3, nbl * world)
ctxs = [api.Context(0) for _ in range(world)]
shards = [full.shard(r * nbl) for r in range(world)]
grid = api.TimeGrid(uniform_times(nt, nbl, 5.0))
y0 = np.zeros((nbl, 5))
for r in range(world):
    api.gradient_adjoint(shards[r], y0, grid, nc, ctx=ctxs[r])
_group(ctxs)
os.environ["CKO_PLAIN_LAUNCH"] = os.environ.get("PLAIN", "1")
t0 = time.time()


MODE = os.environ.get("MODE", "grad")


def rank(r, it):
    try:
        if MODE == "fwd":
            tr = api.integrate_backward_euler(shards[r], y0, grid, nc, ctx=ctxs[r])
            msg = f"iters {tr.work.newton_iterations}"
        else:
            g = api.gradient_adjoint(shards[r], y0, grid, nc, ctx=ctxs[r])
            msg = f"loss {g.loss:.12g}"
        print(f"it {it} rank {r} done {time.time() - t0:.3f} {msg}", flush=True)
    except Exception as ex:
        print(f"it {it} rank {r} error {time.time() - t0:.3f} {ex}", flush=True)


for it in range(int(os.environ.get("REPS", "6"))):
    th = [threading.Thread(target=rank, args=(r, it)) for r in range(world)]
    for t in th:
        t.start()
    for t in th:
        t.join()
