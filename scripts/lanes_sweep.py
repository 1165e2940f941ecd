"""C2 training-step time at several lane counts on one GPU (device-resident grid, fused call), structured
kernels on / off: python scripts/lanes_sweep.py 125,1000"""
import ctypes as C
import sys

import numpy as np
import torch

import paper_2310_08649_b200 as P
from paper_2310_08649_b200 import abi, api
from paper_2310_08649_b200._native import lib
from paper_2310_08649_b200.errors import raise_for
from tests.conftest import uniform_times

nt, nc = 10000, 100
L = lib()
for nb in [int(v) for v in sys.argv[1].split(",")]:
    for sp in (1, 0):
        ctx = api.Context(0)
        ctx.set_structured(bool(sp))
        m = P.build_mass_damper_spring(10, nb)
        dm = ctx.model(m)
        d_t = torch.from_numpy(uniform_times(nt, nb, 0.01)).cuda()
        d_y0 = torch.zeros((nb, 20), dtype=torch.float64, device="cuda")
        d_s = torch.empty((nt + 1, nb * 20), dtype=torch.float64, device="cuda")
        st, sv = api.NewtonSettings().c(), api.SolverChoice(0, 1).c()
        wf, wb, e = abi.CkoWork(), abi.CkoWork(), abi.CkoError()
        loss = C.c_double()
        grad = np.zeros(m.params.size)
        ms = []
        for it in range(5):
            t0, t1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            torch.cuda.synchronize()
            t0.record()
            raise_for(L.cko_gradient_adjoint_device(ctx.h, dm, C.c_void_p(d_y0.data_ptr()), C.c_void_p(d_t.data_ptr()),
                                                    nb, nt, nc, C.byref(st), C.byref(sv), C.c_void_p(d_s.data_ptr()),
                                                    C.byref(loss), abi.dptr(grad), C.byref(wf), C.byref(wb),
                                                    C.byref(e)), e)
            t1.record()
            torch.cuda.synchronize()
            if it >= 2:
                ms.append(t0.elapsed_time(t1))
        v = float(np.median(ms))
        print(f"nb={nb} structured={sp} sp_bits={ctx.structured_used()} {v:.2f} ms/step "
              f"{nb * nt / (v * 1e-3):.3e} series*steps/s loss={loss.value:.6e}", flush=True)
