"""C2 (MDS n=20, nt=10000, t_max=0.01) solver family on one GPU: device-resident forward + adjoint per
(solver, n_chunk, nb), kernel time from the library's CUDA events. One JSON line each."""
import ctypes as C
import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2310_08649_b200 as P  # noqa: E402
from paper_2310_08649_b200 import abi, api  # noqa: E402
from paper_2310_08649_b200._native import lib  # noqa: E402
from paper_2310_08649_b200.errors import raise_for  # noqa: E402
from tests.conftest import uniform_times  # noqa: E402

nt = int(os.environ.get("NT", 10000))
cfgs = [a.split(",") for a in sys.argv[1:]] or [["pcr", "100", "1000"], ["hybrid", "16", "1000"]]
L = lib()
ctx = api.Context(0)
L.cko_ctx_enable_timing(ctx.h, 1)
for name, nc, nb in cfgs:
    nc, nb = int(nc), int(nb)
    kind = {"thomas": 0, "pcr": 1, "hybrid": 2}[name]
    m = P.build_mass_damper_spring(10, nb)
    dm = ctx.model(m)
    d_times = torch.from_numpy(uniform_times(nt, nb, 0.01 * nt / 10000)).cuda()
    d_y0 = torch.zeros((nb, 20), dtype=torch.float64, device="cuda")
    d_states = torch.empty((nt + 1, nb * 20), dtype=torch.float64, device="cuda")
    grad = np.zeros(m.params.size)
    loss = C.c_double()
    st, sv = api.NewtonSettings().c(), api.SolverChoice(kind, int(os.environ.get("NSW", 1))).c()
    wf, wb, e = abi.CkoWork(), abi.CkoWork(), abi.CkoError()
    kms = (C.c_double * 4)()
    tot = []
    for it in range(2):
        raise_for(L.cko_be_forward_device(ctx.h, dm, C.c_void_p(d_y0.data_ptr()), C.c_void_p(d_times.data_ptr()), nb,
                                          nt, nc, C.byref(st), C.byref(sv), C.c_void_p(d_states.data_ptr()),
                                          C.byref(wf), C.byref(e)), e)
        L.cko_ctx_last_kernel_ms(ctx.h, kms)
        f_ms = kms[0]
        raise_for(L.cko_be_adjoint_device(ctx.h, dm, C.c_void_p(d_states.data_ptr()), C.c_void_p(d_times.data_ptr()),
                                          nb, nt, nc, C.byref(sv), abi.CKO_LOSS_FROBENIUS, None, C.byref(loss),
                                          abi.dptr(grad), C.byref(wb), C.byref(e)), e)
        L.cko_ctx_last_kernel_ms(ctx.h, kms)
        tot.append((f_ms, kms[1], kms[2] + kms[3]))
    f_ms, a_ms, o_ms = tot[-1]
    ms = f_ms + a_ms + o_ms
    print(json.dumps({"solver": name, "n_chunk": nc, "nb": nb, "nt": nt, "fwd_ms": f_ms, "adj_ms": a_ms,
                      "other_ms": o_ms, "series_steps_per_s": nb * nt / (ms * 1e-3),
                      "gen": ctx.kernel_generation_used(), "newton": wf.newton_iterations,
                      "sweeps": wf.reduction_sweeps, "loss": loss.value}), flush=True)
