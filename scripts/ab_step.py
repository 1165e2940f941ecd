"""A/B of the C2 step's kernel times between library builds (CKO_LIB_PATH): forward / adjoint / VJP / loss
kernel milliseconds through cko_be_forward_device + cko_be_adjoint_device (symbols every build has)."""
import ctypes as C
import sys

import numpy as np
import torch

import paper_2310_08649_b200 as P
from paper_2310_08649_b200 import abi, api
from paper_2310_08649_b200._native import lib
from paper_2310_08649_b200.errors import raise_for
from tests.conftest import uniform_times

nb, nt, nc, reps = 1000, 10000, 100, int(sys.argv[1]) if len(sys.argv) > 1 else 5
fused = len(sys.argv) > 2 and sys.argv[2] == "fused"  # one cko_gradient_adjoint_device call per step
L = lib()
ctx = api.Context(0)
m = P.build_mass_damper_spring(10, nb)
dm = ctx.model(m)
d_t = torch.from_numpy(uniform_times(nt, nb, 0.01)).cuda()
d_y0 = torch.zeros((nb, 20), dtype=torch.float64, device="cuda")
d_s = torch.empty((nt + 1, nb * 20), dtype=torch.float64, device="cuda")
st, sv = api.NewtonSettings().c(), api.SolverChoice(0, 1).c()
wf, wb, e = abi.CkoWork(), abi.CkoWork(), abi.CkoError()
loss = C.c_double()
grad = np.zeros(m.params.size)
kms = (C.c_double * 4)()
L.cko_ctx_enable_timing(ctx.h, 1)
acc = np.zeros(4)
for it in range(reps + 2):
    if fused:
        raise_for(L.cko_gradient_adjoint_device(ctx.h, dm, C.c_void_p(d_y0.data_ptr()), C.c_void_p(d_t.data_ptr()), nb,
                                                nt, nc, C.byref(st), C.byref(sv), C.c_void_p(d_s.data_ptr()),
                                                C.byref(loss), abi.dptr(grad), C.byref(wf), C.byref(wb), C.byref(e)), e)
        L.cko_ctx_last_kernel_ms(ctx.h, kms)
        if it >= 2:
            acc += list(kms)
        continue
    raise_for(L.cko_be_forward_device(ctx.h, dm, C.c_void_p(d_y0.data_ptr()), C.c_void_p(d_t.data_ptr()), nb, nt, nc,
                                      C.byref(st), C.byref(sv), C.c_void_p(d_s.data_ptr()), C.byref(wf), C.byref(e)), e)
    L.cko_ctx_last_kernel_ms(ctx.h, kms)
    f = kms[0]
    raise_for(L.cko_be_adjoint_device(ctx.h, dm, C.c_void_p(d_s.data_ptr()), C.c_void_p(d_t.data_ptr()), nb, nt, nc,
                                      C.byref(sv), abi.CKO_LOSS_FROBENIUS, None, C.byref(loss), abi.dptr(grad),
                                      C.byref(wb), C.byref(e)), e)
    L.cko_ctx_last_kernel_ms(ctx.h, kms)
    if it >= 2:
        acc += [f, kms[1], kms[2], kms[3]]
acc /= reps
print(f"fwd {acc[0]:.3f} adj {acc[1]:.3f} vjp {acc[2]:.3f} loss {acc[3]:.3f} total {acc.sum():.3f} L={loss.value!r}")
