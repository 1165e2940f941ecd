"""e2e diagnostics: pinned H2D bandwidth of the grid-sized copy, and cko_gradient_adjoint from pinned host
buffers vs the device-resident call (C2 shape)."""
import ctypes as C
import time

import numpy as np
import torch

import paper_2310_08649_b200 as P
from paper_2310_08649_b200 import abi, api
from paper_2310_08649_b200._native import lib
from paper_2310_08649_b200.errors import raise_for
from tests.conftest import uniform_times

nb, nt, nc = 1000, 10000, 100
h = torch.from_numpy(uniform_times(nt, nb, 0.01)).pin_memory()
d = torch.empty_like(h, device="cuda")
for _ in range(3):
    torch.cuda.synchronize(); t0 = time.perf_counter(); d.copy_(h, non_blocking=True); torch.cuda.synchronize()
    print(f"H2D pinned {h.numel() * 8 / 1e6:.0f} MB: {h.numel() * 8 / (time.perf_counter() - t0) / 1e9:.1f} GB/s")
L = lib()
ctx = api.Context(0)
m = P.build_mass_damper_spring(10, nb)
dm = ctx.model(m)
h_y0 = torch.zeros((nb, 20), dtype=torch.float64).pin_memory()
st, sv = api.NewtonSettings().c(), api.SolverChoice(0, 1).c()
wf, wb, e = abi.CkoWork(), abi.CkoWork(), abi.CkoError()
loss = C.c_double()
grad = np.zeros(m.params.size)
kms = (C.c_double * 4)()
L.cko_ctx_enable_timing(ctx.h, 1)
for it in range(6):
    torch.cuda.synchronize(); t0 = time.perf_counter()
    hp = lambda t: C.cast(C.c_void_p(t.data_ptr()), C.POINTER(C.c_double))
    raise_for(L.cko_gradient_adjoint(ctx.h, dm, hp(h_y0), hp(h), nb, nt, nc, C.byref(st), C.byref(sv), None,
                                     C.byref(loss), abi.dptr(grad), C.byref(wf), C.byref(wb), C.byref(e)), e)
    t1 = time.perf_counter()
    L.cko_ctx_last_kernel_ms(ctx.h, kms)
    print(f"e2e call {1e3 * (t1 - t0):.2f} ms; kernels fwd {kms[0]:.2f} adj {kms[1]:.2f} vjp {kms[2]:.2f}")
