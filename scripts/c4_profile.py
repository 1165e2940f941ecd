"""Kernel-time breakdown of one C4 training step (neural ODE, width 128)."""
import ctypes as C
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2310_08649_b200 as P  # noqa: E402
from paper_2310_08649_b200 import api  # noqa: E402
from paper_2310_08649_b200._native import lib  # noqa: E402

nb, nt, nc = 256, 2000, int(sys.argv[1]) if len(sys.argv) > 1 else 100
m = P.build_node_wide(8, 128, nb)
grid = api.TimeGrid.uniform(nt, nb, 1.0)
ctx = api.Context(0)
L = lib()
L.cko_ctx_enable_timing(ctx.h, 1)
kms = (C.c_double * 4)()
tr = api.integrate_backward_euler(m, np.zeros((nb, 8)), grid, nc, ctx=ctx)
t0 = time.perf_counter()
tr = api.integrate_backward_euler(m, np.zeros((nb, 8)), grid, nc, ctx=ctx)
L.cko_ctx_last_kernel_ms(ctx.h, kms)
fwd = kms[0]
t1 = time.perf_counter()
loss, g = api.adjoint_backward(m, tr, nc, ctx=ctx)
L.cko_ctx_last_kernel_ms(ctx.h, kms)
print(f"nc={nc} fwd kernel {fwd:.1f} ms (wall {1e3 * (t1 - t0):.1f}); adj kernel {kms[1]:.1f} ms, vjp {kms[2]:.1f} ms, "
      f"loss {kms[3]:.2f} ms; newton iters {tr.work.newton_iterations}")
