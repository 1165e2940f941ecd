#!/usr/bin/env python
"""Benchmark: series*steps/s of backward-Euler forward + discrete adjoint (PCR).

Workload (BASELINE.json configs[1]): mass-damper-spring chain,
10 units (n = 20), nb = 1000 series per GPU, nt = 10000 steps, t_max = 0.01
(finite horizon), y0 = 0, Frobenius loss, analytic Jacobians,
PCR block-bidiagonal solves at n_chunk = --n-chunk. Synthetic inputs (the
reference's own deterministic model parameters and uniform time grid).

One step = integrate_backward_euler + adjoint_backward over the whole
workload, inputs resident in HBM (value) / through the C ABI from pinned host
buffers (e2e). Inputs (1.6 GB trajectory, 80 MB grid) exceed the 126 MB L2,
so no explicit flush is needed between steps.

  python bench.py [--gpus N --steps K --warmup W] [--impl reference]
Under torchrun each rank integrates its own nb lanes of a global
nb * world-lane problem (weak scaling, lane_offset sharding); the only
cross-rank traffic is the per-Newton-iteration convergence flag and the
loss / gradient sums.
"""
from __future__ import annotations

import argparse
import ctypes as C
import json
import math
import os
import statistics
import subprocess
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--nb", type=int, default=1000, help="series per GPU (--scaling weak)")
    ap.add_argument("--scaling", default="weak", choices=["weak", "strong"],
                    help="weak: nb series per GPU; strong: --nb-total series split over the GPUs (north-star target)")
    ap.add_argument("--nb-total", type=int, default=1000, help="series over all GPUs (--scaling strong)")
    ap.add_argument("--nt", type=int, default=10000)
    ap.add_argument("--n-unit", type=int, default=10)
    ap.add_argument("--t-max", type=float, default=0.01)
    ap.add_argument("--n-chunk", type=int, default=100)
    ap.add_argument("--solver", default="thomas", choices=["thomas", "pcr", "hybrid"])
    ap.add_argument("--n-switch", type=int, default=1)
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--cpu-sample-steps", type=int, default=0, help="CPU sample steps (0: one chunk, n_chunk)")
    ap.add_argument("--quiet-clocks", action="store_true", help="skip nvidia-smi sampling (profiler runs)")
    ap.add_argument("--no-c3", action="store_true", help="skip the C3 chunked-PCR vs sequential side measurement")
    return ap.parse_args()


SOLVER_ID = {"thomas": 0, "pcr": 1, "hybrid": 2}


def uniform_times(nt, nb, t_max):
    ti = np.array([t_max * float(i) / float(nt) for i in range(nt + 1)])
    return np.ascontiguousarray(np.repeat(ti[:, None], nb, axis=1))


def sweeps_per_solve(c, solver, n_switch):
    if solver == "thomas":
        return 0
    s = 0
    for bit in range(30, -1, -1):
        m = 1 << bit
        if c & m:
            e = m.bit_length() - 1
            s += e if solver == "pcr" else min(n_switch, e)
    return s


def flops_per_series_step(n, nc, solver, n_switch, k_avg, structured=False):
    """Algorithmic fp64 flops per series*step (MDS analytic model):
    forward: (k+1) residual passes (rate ~ 8u + 3n each) + k x [J assembly n^2,
    LU L(n), solve 2n^2 (+ PCR sweeps)], adjoint: one J^T lambda (2n^2), one LU,
    one solve (+ sweeps), quadrature + VJP (~12u). PCR adds (4n^3 + 2n^2) per
    row per sweep beyond the first-level right solve, averaged over the chunk.
    structured: the arrow + tridiagonal kernels (cko_sparse.cuh) do only the
    nonzero work of the same LU / substitution — assembly + factor ~19u,
    substitution ~15u per block."""
    L = sum(1 + m + 2 * m * m for m in range(n))
    u = n // 2
    F_h = 8 * u + 3 * n
    sw = sweeps_per_solve(nc, solver, n_switch) / max(nc, 1)  # sweeps per row
    pcr_row = sw * (4 * n ** 3 + 2 * n * n) if solver != "thomas" else 0.0
    if structured:
        fwd = (k_avg + 1) * F_h + k_avg * (19 * u + 15 * u)
        adj = 19 * u + 15 * u + 3 * n + 12 * u + 2 * n
        return fwd + adj
    fwd = (k_avg + 1) * F_h + k_avg * (n * n + L + 2 * n * n + pcr_row)
    adj = 2 * n * n + n * n + L + 2 * n * n + pcr_row + 12 * u + 2 * n
    return fwd + adj


class ClockSampler:
    """nvidia-smi clocks + throttle reasons during the timed region (B200_PROFILING.md)."""

    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, device, enabled=True):
        self.device, self.enabled, self.proc, self.lines = device, enabled, None, []

    def __enter__(self):
        if self.enabled:
            try:
                self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.device), f"--query-gpu={self.Q}",
                                              "--format=csv,noheader,nounits", "-lms", "200"],
                                             stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
                time.sleep(0.3)
            except OSError:
                self.proc = None
        return self

    def __exit__(self, *a):
        if self.proc:
            time.sleep(0.25)
            self.proc.terminate()
            out, _ = self.proc.communicate(timeout=5)
            self.lines = [ln for ln in out.splitlines() if ln.strip()]

    def summary(self):
        if not self.lines:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        sm, mx, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            f = [x.strip() for x in ln.split(",")]
            try:
                sm.append(float(f[1]))
                mx = float(f[2])
            except (ValueError, IndexError):
                continue
            for nm, v in zip(names, f[5:9]):
                if v.lower() == "active":
                    reasons.add(nm)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": mx, "reasons": sorted(reasons),
                "samples": len(sm)}


def load_traffic(kernel, args):
    """DRAM bytes per launch of `kernel` from the committed ncu capture of this configuration
    (profiles/traffic.json, written from `ncu --set full` by scripts/ncu_traffic.py), else None."""
    try:
        tab = json.load(open(os.path.join(ROOT, "profiles", "traffic.json")))
    except (OSError, ValueError):
        return None
    key = f"{kernel}:{args.solver}:{args.n_chunk}:{args.nb}:{args.nt}"
    return tab.get(key)


def dist_env():
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return rank, world, local


def lane_split(args, world, rank):
    """(lanes of this rank, global lane offset, lanes over all ranks): weak scaling gives every rank
    args.nb lanes; strong scaling splits args.nb_total contiguously (the first nb_total % world ranks get
    one more lane)."""
    if args.scaling == "weak":
        return args.nb, rank * args.nb, args.nb * world
    base, extra = divmod(args.nb_total, world)
    nb = base + (1 if rank < extra else 0)
    off = rank * base + min(rank, extra)
    return nb, off, args.nb_total


def mds_workload(args, world, rank):
    import paper_2310_08649_b200 as P
    nb, off, nb_total = lane_split(args, world, rank)
    model = P.build_mass_damper_spring(args.n_unit, nb_total)
    times = uniform_times(args.nt, nb, args.t_max)
    y0 = np.zeros((nb, model.state_size))
    return model.shard(off), y0, times


def golden_parity(args, nb_total, loss, grad, wf, wb):
    """The bench run's loss / gradient / WorkCounters against the compiled reference's own full-size run
    (tests/golden/full_c2.npz, oracle/make_golden_full.py) when the workload is that configuration."""
    path = os.path.join(ROOT, "tests", "golden", "full_c2.npz")
    if not os.path.exists(path):
        return {"checked": False, "why": "tests/golden/full_c2.npz missing"}
    g = np.load(path)
    same = (nb_total == int(g["nb"]) and args.nt == int(g["nt"]) and args.n_chunk == int(g["n_chunk"])
            and args.solver == "thomas" and args.n_unit == int(g["n_unit"]) and args.t_max == float(g["t_max"]))
    if not same:
        return {"checked": False, "why": "workload differs from the golden's (C2, nb=1000, nt=10000, thomas/100)"}
    keys = [k for k, _ in __import__("paper_2310_08649_b200.abi", fromlist=["x"]).CkoWork._fields_]
    gl = float(g["thomas_loss"])
    loss_rel = abs(loss - gl) / abs(gl)
    grad_rel = float(np.max(np.abs(grad - g["thomas_grad"])) / np.max(np.abs(g["thomas_grad"])))
    cnt = ([int(getattr(wf, k)) for k in keys] == [int(x) for x in g["thomas_fwd"]]
           and [int(getattr(wb, k)) for k in keys] == [int(x) for x in g["thomas_bwd"]])
    return {"checked": True, "against": "compiled reference, full C2 (tests/golden/full_c2.npz)",
            "loss_rel": loss_rel, "grad_rel_max": grad_rel, "counters_equal": cnt,
            "ok": bool(cnt and loss_rel <= 1e-10 and grad_rel <= 1e-10)}


def config_dict(args, world, extra=None):
    nb0, _, nb_total = lane_split(args, world, 0)
    per = f"nb={nb0}/GPU" if args.scaling == "weak" else f"nb={nb_total} over {world} GPU(s) ({nb0} on rank 0)"
    d = {"workload": (f"C2 mass-damper-spring chain (SURVEY §8d): {args.n_unit} units (n={2 * args.n_unit}), "
                      f"{per}, nt={args.nt}, t_max={args.t_max}, backward Euler + discrete adjoint, "
                      f"{args.solver} n_chunk={args.n_chunk}, Frobenius loss"),
         "model": "mds", "n_unit": args.n_unit, "n_size": 2 * args.n_unit, "n_batch_per_gpu": nb0,
         "n_batch_total": nb_total, "n_time": args.nt, "n_chunk": args.n_chunk, "solver": args.solver,
         "t_max": args.t_max, "parallelism": f"batch-sharded dp{world} ({args.scaling} scaling)",
         "l2": (f"inputs larger than L2 (trajectory {8 * (args.nt + 1) * nb0 * 2 * args.n_unit / 1e9:.2f} GB/GPU), "
                "no flush")}
    if extra:
        d.update(extra)
    return d


# ---------------------------------------------------------------------------
# reference arm: the compiled reference (oracle/_ref) on the host cores
# ---------------------------------------------------------------------------
def cpu_sample(args, world):
    """The reference arms' bounded sample of the bench workload: every lane of the arm's config, the first
    n_chunk steps of the full grid (same dt), solved with the same solver and n_chunk -- one full chunk of
    the real configuration, so nothing is extrapolated but the step count."""
    _, _, nb_total = lane_split(args, world, 0)
    import paper_2310_08649_b200 as P
    model = P.build_mass_damper_spring(args.n_unit, nb_total)
    nt_s = args.cpu_sample_steps or args.n_chunk
    times = uniform_times(nt_s, nb_total, args.t_max * nt_s / args.nt)
    y0 = np.zeros((nb_total, model.state_size))
    return model, y0, times, nt_s, min(args.n_chunk, nt_s)


def run_reference(args):
    rank, world, _ = dist_env()
    if rank != 0:
        return
    from oracle import load_port, load_ref, ref_available
    kind = "reference" if ref_available() else "port"
    orc = load_ref() if kind == "reference" else load_port()
    cores = os.cpu_count() or 1
    model, y0, times, nt_s, nc = cpu_sample(args, max(world, args.gpus))
    nb = y0.shape[0]
    sv = (SOLVER_ID[args.solver], args.n_switch)
    secs = []
    for i in range(args.warmup + args.steps):
        s = orc.sharded_seconds(model, y0, times, nc, cores, solver=sv)
        if s < 0:
            raise SystemExit("reference run failed")
        if i >= args.warmup:
            secs.append(s)
    sec = statistics.mean(secs)
    v = nb * nt_s / sec
    line = {"impl": "reference", "metric": "series*steps/s forward+adjoint (backward Euler, PCR)",
            "value": v, "unit": "series*steps/s", "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": sec * 1e3, "higher_is_better": True, "scaling": args.scaling, "vs_baseline": None,
            "dtype": "f64", "data": "synthetic",
            "config": config_dict(args, max(world, args.gpus),
                                  {"sample": f"all {nb} lanes x the first {nt_s} steps (dt as the full grid), "
                                             f"{args.solver} n_chunk={nc}"}),
            "cpu_baseline": {"value": v, "unit": "series*steps/s", "cores": cores, "kind": kind,
                             "sample": f"{nb} lanes x {nt_s} steps per step (n_chunk={nc}), {cores} threads over "
                                       f"contiguous lane shards (timing only: shard-local Newton predicate)"},
            "e2e": {"value": v, "unit": "series*steps/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


def cpu_baseline_single(args):
    """Single-thread compiled reference on a bounded sample (rank 0, N = 1)."""
    from oracle import load_port, load_ref, ref_available
    kind = "reference" if ref_available() else "port"
    orc = load_ref() if kind == "reference" else load_port()
    model, y0, times, nt_s, nc = cpu_sample(args, 1)
    nb = y0.shape[0]
    t0 = time.perf_counter()
    orc.gradient(model, y0, times, nc, solver=(SOLVER_ID[args.solver], args.n_switch))
    sec = time.perf_counter() - t0
    return {"value": nb * nt_s / sec, "unit": "series*steps/s", "cores": 1, "kind": kind,
            "sample": f"all {nb} lanes x the first {nt_s} steps (same dt, n_chunk={nc}: one full chunk of the "
                      f"workload), single thread, forward+adjoint, {sec:.1f} s"}


def c3_pcr_vs_sequential(ctx, reps=2):
    """North-star side target: stiff Chaboche (eps_a x10), sparse batch nb=50, nt=20000,
    forward + adjoint through the public API on this GPU: chunked PCR (n_chunk=256) against sequential
    stepping (n_chunk=1). Device-resident host calls, wall clock around synchronous calls."""
    import paper_2310_08649_b200 as P
    from paper_2310_08649_b200 import api
    nb, nt, nu = 50, 20000, 3
    m = P.build_chaboche(nu, nb)
    p = m.params.copy()
    p[6 + 2 * nu:6 + 2 * nu + nb] *= 10.0
    m = m.with_params(p)
    grid = api.TimeGrid.uniform(nt, nb, 10.0)
    y0 = np.zeros((nb, m.state_size))
    out = {}
    for name, kind, nc in (("sequential", 0, 1), ("pcr", 1, 256)):
        sv = api.SolverChoice(kind, 1)
        api.gradient_adjoint(m, y0, grid, nc, solver=sv, ctx=ctx)
        t0 = time.perf_counter()
        for _ in range(reps):
            r = api.gradient_adjoint(m, y0, grid, nc, solver=sv, ctx=ctx)
        out[name] = {"n_chunk": nc, "seconds": (time.perf_counter() - t0) / reps,
                     "newton_iterations": r.trajectory.work.newton_iterations,
                     "kernel_generation": ctx.kernel_generation_used()}
    out["speedup_pcr_over_sequential"] = out["sequential"]["seconds"] / out["pcr"]["seconds"]
    out["workload"] = "C3 Chaboche n_unit=3 (n=5), eps_a x10, nb=50, nt=20000, t_max=10, forward+adjoint"
    return out


def c4_training_step(ctx, reps=2, ncs=(10, 20, 100), cpu_steps=100):
    """North-star C4: neural ODE, state 8, hidden width 128 (18 824 parameters, MLP rate on DMMA),
    nb = 256, nt = 2000, one adjoint training step (forward + adjoint + parameter gradient) through the public
    API with host buffers; n_chunk sweep, wall clock around the synchronous calls. cpu_baseline: the compiled
    reference integrator + adjoint running the same NodeWide model (oracle/src/ref_models.hpp), single thread,
    on the first `cpu_steps` steps of the same grid."""
    import paper_2310_08649_b200 as P
    from paper_2310_08649_b200 import api
    nb, nt = 256, 2000
    m = P.build_node_wide(8, 128, nb)
    grid = api.TimeGrid.uniform(nt, nb, 1.0)
    y0 = np.zeros((nb, 8))
    out = {"workload": "C4 neural ODE n=8, W=128, nb=256, nt=2000, t_max=1, thomas, forward+adjoint+gradient"}
    best = None
    for nc in ncs:
        sv = api.SolverChoice(0, 1)
        api.gradient_adjoint(m, y0, grid, nc, solver=sv, ctx=ctx)
        t0 = time.perf_counter()
        for _ in range(reps):
            r = api.gradient_adjoint(m, y0, grid, nc, solver=sv, ctx=ctx)
        sec = (time.perf_counter() - t0) / reps
        v = nb * nt / sec
        out[f"n_chunk={nc}"] = {"seconds": sec, "series_steps_per_s": v,
                                "newton_iterations": r.trajectory.work.newton_iterations, "loss": r.loss,
                                "launches": ctx.last_launches() if hasattr(ctx, "last_launches") else None}
        if best is None or v > best[1]:
            best = (nc, v)
    out["best"] = {"n_chunk": best[0], "series_steps_per_s": best[1]}
    try:
        from oracle import load_ref, ref_available
        if ref_available():
            ts = grid.times[:cpu_steps + 1]
            t0 = time.perf_counter()
            load_ref().gradient(m, y0, ts, min(20, cpu_steps))
            sec = time.perf_counter() - t0
            out["cpu_baseline"] = {"value": nb * cpu_steps / sec, "unit": "series*steps/s", "cores": 1,
                                   "kind": "reference", "sample": f"all {nb} lanes x the first {cpu_steps} steps, "
                                   f"n_chunk={min(20, cpu_steps)}, single thread, {sec:.1f} s"}
    except Exception as ex:  # the checker build is missing on this box
        out["cpu_baseline"] = {"value": None, "error": str(ex)[:200]}
    return out


def c2_solver_family(args, local, nt_s=None, reps=1):
    """The headline workload's chunked solver family on this GPU at FULL size (nb lanes x nt steps, the bench
    grid), device-resident through the C ABI and timed with the kernels' own CUDA events: Thomas/n_chunk (the
    bench line's solver) next to PCR/100 and hybrid/16 on the generation-2 warp-cooperative PCR kernels
    (cko_pcrw.cuh), so the metric's PCR member is on record at the headline shape (PCR
    does ~40x the fp64 work of Thomas at n = 20 and pays only when the batch cannot fill the GPU)."""
    import ctypes as C

    import torch

    import paper_2310_08649_b200 as P
    from paper_2310_08649_b200 import abi, api
    from paper_2310_08649_b200._native import lib
    from paper_2310_08649_b200.errors import raise_for
    nt_s = nt_s or args.nt
    L = lib()
    ctx = api.Context(local)
    m = P.build_mass_damper_spring(args.n_unit, args.nb)
    nb, n = args.nb, m.state_size
    dm = ctx.model(m)
    d_times = torch.from_numpy(uniform_times(nt_s, nb, args.t_max * nt_s / args.nt)).cuda()
    d_y0 = torch.zeros((nb, n), dtype=torch.float64, device="cuda")
    d_states = torch.empty((nt_s + 1, nb * n), dtype=torch.float64, device="cuda")
    grad = np.zeros(m.params.size)
    loss = C.c_double()
    st = api.NewtonSettings().c()
    wf, wb, e = abi.CkoWork(), abi.CkoWork(), abi.CkoError()
    kms = (C.c_double * 4)()
    L.cko_ctx_enable_timing(ctx.h, 1)
    out = {}
    for name, kind, nc in (("thomas", 0, args.n_chunk), ("pcr", 1, 100), ("hybrid", 2, 16)):
        sv = api.SolverChoice(kind, 1).c()
        tot = 0.0
        for it in range(reps + 1):
            raise_for(L.cko_gradient_adjoint_device(ctx.h, dm, C.c_void_p(d_y0.data_ptr()),
                                                    C.c_void_p(d_times.data_ptr()), nb, nt_s, nc, C.byref(st),
                                                    C.byref(sv), C.c_void_p(d_states.data_ptr()), C.byref(loss),
                                                    abi.dptr(grad), C.byref(wf), C.byref(wb), C.byref(e)), e)
            L.cko_ctx_last_kernel_ms(ctx.h, kms)
            if it:  # the first pass warms up
                tot += kms[0] + kms[1] + kms[2] + kms[3]
        ms = tot / reps
        out[name] = {"n_chunk": nc, "series_steps_per_s": nb * nt_s / (ms * 1e-3), "kernel_ms": ms,
                     "kernel_generation": ctx.kernel_generation_used()}
    L.cko_ctx_enable_timing(ctx.h, 0)
    out["sample"] = f"nb={nb} x nt={nt_s} (the full grid), device-resident, kernel time, {reps} timed pass(es)"
    return out


def north_star_strong(args, ctx, world, rank, stream, hbm_peak, reps=3, warmup=2):
    """The north-star target (BASELINE.json): the 1000-series, 10k-step MDS case split over all ranks of this
    run (strong scaling, 1000/world lanes per GPU), forward + adjoint per step, device-resident, timed with
    CUDA events on the compute stream, max over ranks; HBM fraction from the compulsory bytes
    B_alg = 16 n + 16 per series*step; loss / gradient / counters checked against the
    compiled reference's full-size run."""
    import torch
    import torch.distributed as dist

    from paper_2310_08649_b200 import abi, api
    from paper_2310_08649_b200._native import lib
    from paper_2310_08649_b200.errors import raise_for
    sa = argparse.Namespace(**vars(args))
    sa.scaling, sa.nb_total = "strong", 1000
    model, y0, times = mds_workload(sa, world, rank)
    nb, nt, n = y0.shape[0], sa.nt, model.state_size
    L = lib()
    dm = ctx.model(model)
    d_y0 = torch.from_numpy(y0).cuda()
    d_times = torch.from_numpy(times).cuda()
    d_states = torch.empty((nt + 1, nb * n), dtype=torch.float64, device="cuda")
    st, sv = api.NewtonSettings().c(), api.SolverChoice(SOLVER_ID[sa.solver], sa.n_switch).c()
    grad = np.zeros(model.params.size)
    loss = C.c_double()
    wf, wb, e = abi.CkoWork(), abi.CkoWork(), abi.CkoError()

    def step():
        raise_for(L.cko_gradient_adjoint_device(ctx.h, dm, C.c_void_p(d_y0.data_ptr()),
                                                C.c_void_p(d_times.data_ptr()), nb, nt, sa.n_chunk, C.byref(st),
                                                C.byref(sv), C.c_void_p(d_states.data_ptr()), C.byref(loss),
                                                abi.dptr(grad), C.byref(wf), C.byref(wb), C.byref(e)), e)
    for _ in range(warmup):
        step()
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    ev0.record(stream)
    for _ in range(reps):
        step()
    ev1.record(stream)
    torch.cuda.synchronize()
    ms = ev0.elapsed_time(ev1) / reps
    if world > 1:
        t = torch.tensor([ms], dtype=torch.float64, device="cpu" if os.environ.get("CKO_BENCH_ONE_GPU") == "1"
                         else "cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())
    v = 1000 * nt / (ms * 1e-3)
    b_alg = 16 * n + 16
    return {"workload": f"C2 MDS n={n}, 1000 series over {world} GPU(s) ({nb} lanes on rank 0), nt={nt}, "
                        f"{sa.solver} n_chunk={sa.n_chunk}, forward+adjoint", "value": v, "unit": "series*steps/s",
            "ms_per_step": ms, "steps": reps, "warmup": warmup,
            "hbm": {"achieved_gbs": v * b_alg / 1e9, "peak_gbs": hbm_peak, "frac": v * b_alg / 1e9 / hbm_peak,
                    "alg_bytes_per_series_step": b_alg},
            "parity": golden_parity(sa, 1000, loss.value, grad, wf, wb)}


# ---------------------------------------------------------------------------
# B200 arm
# ---------------------------------------------------------------------------
def self_launch(args):
    """`python bench.py --gpus N` outside torchrun: re-run this script under torch.distributed.run with one
    rank per GPU (the driver's own launch line), rendezvous on 127.0.0.1."""
    import socket
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr", "127.0.0.1", "--master-port", str(port), os.path.abspath(__file__)] + sys.argv[1:]
    os.execv(sys.executable, cmd)


def main():
    args = parse()
    if args.impl == "reference":
        run_reference(args)
        return
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        self_launch(args)
    import torch
    import torch.distributed as dist

    from paper_2310_08649_b200 import abi, api
    from paper_2310_08649_b200._native import lib
    from paper_2310_08649_b200.errors import raise_for

    rank, world, local = dist_env()
    # CKO_BENCH_ONE_GPU=1: every rank on cuda:0 with a gloo process group -- exercises the multi-rank
    # plumbing (self-launch, IPC group, per-iteration exchange, max-over-ranks timing) on a one-GPU box;
    # the contexts time-slice the GPU, so its timings mean nothing.
    one_gpu = os.environ.get("CKO_BENCH_ONE_GPU") == "1"
    if one_gpu:
        local = 0
    torch.cuda.set_device(local)
    if world > 1:
        if one_gpu:
            dist.init_process_group("gloo")
        else:
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    model, y0, times = mds_workload(args, world, rank)
    nb, nt, n = y0.shape[0], args.nt, model.state_size
    _, _, nb_total = lane_split(args, world, rank)
    ctx = api.Context(local)
    stream = torch.cuda.current_stream()
    ctx.set_stream(stream.cuda_stream)
    if world > 1:
        from paper_2310_08649_b200 import group
        group.join(ctx, rank, world)
    print(json.dumps({"join": rank, "world": world, "device": local, "gpu": torch.cuda.get_device_name(local),
                      "lanes": [model.lane_offset, model.lane_offset + nb], "n_batch_total": nb_total}),
          file=sys.stderr, flush=True)
    L = lib()
    dm = ctx.model(model)
    d_y0 = torch.from_numpy(y0).cuda()
    d_times = torch.from_numpy(times).cuda()
    d_states = torch.empty((nt + 1, nb * n), dtype=torch.float64, device="cuda")
    st = api.NewtonSettings().c()
    sv = api.SolverChoice(SOLVER_ID[args.solver], args.n_switch).c()
    grad = np.zeros(model.params.size)
    loss = C.c_double()
    wf, wb, e = abi.CkoWork(), abi.CkoWork(), abi.CkoError()
    L.cko_ctx_enable_timing(ctx.h, 1)
    kms = (C.c_double * 4)()

    def step(record=None):
        # one training step through the device-buffer gradient_adjoint: forward, loss, adjoint, parameter VJP
        rc = L.cko_gradient_adjoint_device(ctx.h, dm, C.c_void_p(d_y0.data_ptr()), C.c_void_p(d_times.data_ptr()),
                                           nb, nt, args.n_chunk, C.byref(st), C.byref(sv),
                                           C.c_void_p(d_states.data_ptr()), C.byref(loss), abi.dptr(grad),
                                           C.byref(wf), C.byref(wb), C.byref(e))
        raise_for(rc, e)
        if record is not None:
            L.cko_ctx_last_kernel_ms(ctx.h, kms)
            record["fwd"] += kms[0]
            record["adj"] += kms[1]
            record["vjp"] += kms[2]
            record["loss"] += kms[3]
            record["launches"] += L.cko_ctx_last_launches(ctx.h)

    for _ in range(args.warmup):
        step()
    rec = {"fwd": 0.0, "adj": 0.0, "vjp": 0.0, "loss": 0.0, "launches": 0}
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    with ClockSampler(local, enabled=not args.quiet_clocks) as clk:
        ev0.record(stream)
        for _ in range(args.steps):
            step(rec)
        ev1.record(stream)
        torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    ms = ev0.elapsed_time(ev1) / args.steps
    if world > 1:
        t = torch.tensor([ms], device="cpu" if one_gpu else "cuda", dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())
    value = nb_total * nt / (ms * 1e-3)

    # ---- e2e: the public C ABI with pinned HOST buffers, H2D/D2H inside the timed region
    e2e = None
    if not args.no_e2e:
        h_y0 = torch.from_numpy(y0).pin_memory()
        h_times = torch.from_numpy(times).pin_memory()
        hp = lambda t: C.cast(C.c_void_p(t.data_ptr()), C.POINTER(C.c_double))  # noqa: E731
        L.cko_ctx_enable_timing(ctx.h, 0)

        def e2e_step():
            rc = L.cko_gradient_adjoint(ctx.h, dm, hp(h_y0), hp(h_times), nb, nt, args.n_chunk, C.byref(st),
                                        C.byref(sv), None, C.byref(loss), abi.dptr(grad), C.byref(wf), C.byref(wb),
                                        C.byref(e))
            raise_for(rc, e)
        for _ in range(2):
            e2e_step()
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        for _ in range(args.steps):
            e2e_step()
        torch.cuda.synchronize()
        e_ms = (time.perf_counter() - t0) * 1e3 / args.steps
        if world > 1:
            t = torch.tensor([e_ms], device="cpu" if one_gpu else "cuda", dtype=torch.float64)
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            e_ms = float(t.item())
        e2e = {"value": nb_total * nt / (e_ms * 1e-3), "unit": "series*steps/s",
               "h2d_bytes_per_step": int(h_y0.numel() * 8 + h_times.numel() * 8),
               "d2h_bytes_per_step": int(grad.size * 8 + 8), "ms_per_step": e_ms,
               "path": "cko_gradient_adjoint (C ABI, pinned host y0/times -> loss + gradient)"}

    hbm_peak = 6536.7
    try:
        hbm_peak = float(json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))["hbm_gbs"])
        peak_src = "measured (MEASURED_PEAKS.json hbm_gbs)"
    except Exception:
        peak_src = "fallback"
    # the north-star target: 1000 series over the ranks of this run (all ranks take part)
    if world > 1 or args.scaling == "strong" or nb_total != 1000:
        try:
            ns_line = north_star_strong(args, ctx, world, rank, stream, hbm_peak)
        except Exception as ex:  # side measurement only
            ns_line = {"error": str(ex)[:200]}
    else:
        ns_line = None  # this run IS the 1000-series configuration: filled from the main line below

    if rank != 0:
        if world > 1:
            dist.destroy_process_group()
        return

    # ---- roofline of the dominant kernel
    k = args.steps
    kern = {"fwd_kernel": rec["fwd"] / k, "adj_kernel": rec["adj"] / k, "vjp_kernels": rec["vjp"] / k,
            "loss_kernels": rec["loss"] / k}
    dom = max(kern, key=kern.get)
    units = nb * nt  # series*steps per launch on this rank
    bytes_per = {"fwd_kernel": 8 * n + 8, "adj_kernel": 8 * n + 8 + 8 * n, "vjp_kernels": 8 * n + 8 + 8 * n,
                 "loss_kernels": 8 * n}[dom]
    achieved = units * bytes_per / (kern[dom] * 1e-3) / 1e9
    k_avg = wf.newton_iterations / max(1, math.ceil(nt / args.n_chunk))
    sp_bits = L.cko_ctx_structured_used(ctx.h) if hasattr(L, "cko_ctx_structured_used") else 0
    structured = (sp_bits & 3) == 3  # both passes ran on the structured-record kernels
    fl = flops_per_series_step(n, args.n_chunk, args.solver, args.n_switch, k_avg, structured)
    tf = C.c_double(0.0)
    L.cko_probe_fp64_tflops(ctx.h, C.byref(tf), C.byref(e))
    step_tflops = units * fl / (ms * 1e-3) / 1e12
    line = {
        "metric": "series*steps/s forward+adjoint (backward Euler, PCR)",
        "value": value, "unit": "series*steps/s", "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": ms, "higher_is_better": True, "scaling": args.scaling, "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (reference model parameters, uniform grid, y0 = 0)",
        "config": config_dict(args, world),
        "roofline": {"bound": "hbm", "kernel": dom, "achieved": achieved, "peak": hbm_peak, "unit": "GB/s",
                     "frac": achieved / hbm_peak, "traffic": None, "peak_source": peak_src,
                     "alg_bytes_per_series_step": bytes_per, "kernel_ms": kern[dom]},
        "roofline_fp64": {"bound": "fp64", "achieved": step_tflops, "peak": tf.value, "unit": "TFLOP/s",
                          "frac": step_tflops / tf.value if tf.value else None,
                          "peak_source": "measured DFMA probe (cko_probe_fp64_tflops)",
                          "alg_flops_per_series_step": fl,
                          "note": "whole step (fwd+adj), all kernels" + (
                              "; structured-record kernels: nonzero work only (the step is bound by the "
                              "per-lane substitution chain's latency, not by FP64 or HBM throughput)"
                              if structured else "")},
        "kernel_ms_per_step": kern,
        "newton": {"fwd": {kk: int(getattr(wf, kk)) for kk, _ in abi.CkoWork._fields_},
                   "bwd": {kk: int(getattr(wb, kk)) for kk, _ in abi.CkoWork._fields_}},
        "loss": loss.value,
        "parity": golden_parity(args, nb_total, loss.value, grad, wf, wb),
        "gpu_launches": rec["launches"],
        "e2e": e2e,
    }
    line["kernel_generation"] = L.cko_ctx_kernel_generation_used(ctx.h)
    line["structured_kernels"] = {"bits": sp_bits, "forward": bool(sp_bits & 1), "adjoint": bool(sp_bits & 2),
                                  "fallback": bool(sp_bits & 12)}
    if ns_line is None:
        b_alg = 16 * n + 16
        ns_line = {"workload": "this run (1000 series on 1 GPU)", "value": value, "unit": "series*steps/s",
                   "ms_per_step": ms, "hbm": {"achieved_gbs": value * b_alg / 1e9, "peak_gbs": hbm_peak,
                                              "frac": value * b_alg / 1e9 / hbm_peak,
                                              "alg_bytes_per_series_step": b_alg},
                   "parity": line["parity"]}
    line["north_star_1000_series"] = ns_line
    traffic = load_traffic(dom, args)
    if traffic is not None:
        line["roofline"]["traffic"] = traffic["bytes_per_launch"]
        line["roofline"]["traffic_source"] = traffic["source"]
    if world == 1 and not args.no_c3:
        try:
            line["c2_solver_family"] = c2_solver_family(args, local)
        except Exception as ex:  # side measurement only
            line["c2_solver_family"] = {"error": str(ex)[:200]}
        try:
            line["c3_pcr_vs_sequential"] = c3_pcr_vs_sequential(api.Context(local))
        except Exception as ex:
            line["c3_pcr_vs_sequential"] = {"error": str(ex)[:200]}
        try:
            line["c4_training_step"] = c4_training_step(api.Context(local))
        except Exception as ex:
            line["c4_training_step"] = {"error": str(ex)[:200]}
    if world == 1 and not args.no_cpu_baseline:
        try:
            line["cpu_baseline"] = cpu_baseline_single(args)
        except Exception as ex:  # the checker build is missing on this box
            line["cpu_baseline"] = {"value": None, "error": str(ex)[:200]}
    line["clocks"] = clk.summary()
    print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
