// ref_capi.cpp — C entry points over the COMPILED REFERENCE (the unmodified
// /root/reference/proj/core sources, linked by oracle/Makefile into
// oracle/_ref/libchunkode_ref.so). Lets Python tests, the golden-vector
// generator and bench.py's reference arm drive the reference's own
// integrate_backward_euler / adjoint_backward / solvers with the same flat
// inputs as the product C ABI (include/chunkode_b200.h).
// TEST INFRASTRUCTURE ONLY.
#include <chrono>
#include <cstring>
#include <exception>
#include <memory>
#include <sstream>
#include <string>
#include <thread>
#include <vector>

#include "chunkode/adjoint.hpp"
#include "chunkode/bench.hpp"
#include "chunkode/integrate.hpp"
#include "chunkode/linalg.hpp"
#include "chunkode/models.hpp"
#include "chunkode/verify.hpp"
#include "chunkode_b200.h"
#include "ref_models.hpp"

using namespace chunkode;

namespace {

thread_local JacobianStrategy g_strategy = JacobianStrategy::analytic;  // ref_set_jacobian_strategy

void fill(cko_error* e, int code, const char* msg) {
  if (!e) return;
  std::memset(e, 0, sizeof(*e));
  e->code = code;
  std::snprintf(e->msg, sizeof e->msg, "%s", msg);
}

int map_exception(cko_error* e) {
  try {
    throw;
  } catch (const SingularBlock& x) {
    fill(e, CKO_SINGULAR_BLOCK, x.what());
    if (e) e->chunk_index = x.chunk_index, e->batch_index = x.batch_index;
    return CKO_SINGULAR_BLOCK;
  } catch (const NewtonDivergence& x) {
    fill(e, CKO_NEWTON_DIVERGENCE, x.what());
    if (e) {
      e->chunk_start_step = x.chunk_start_step;
      e->batch_index = x.batch_index;
      e->iterations = x.iterations;
      e->residual_norm = x.residual_norm;
      e->initial_norm = x.initial_norm;
    }
    return CKO_NEWTON_DIVERGENCE;
  } catch (const NonFiniteOutput& x) {
    fill(e, CKO_NON_FINITE, x.what());
    return CKO_NON_FINITE;
  } catch (const StrategyUnavailable& x) {
    fill(e, CKO_STRATEGY_UNAVAILABLE, x.what());
    return CKO_STRATEGY_UNAVAILABLE;
  } catch (const SizeGuardExceeded& x) {
    fill(e, CKO_SIZE_GUARD, x.what());
    return CKO_SIZE_GUARD;
  } catch (const InvalidTimeGrid& x) {
    fill(e, CKO_INVALID_TIME_GRID, x.what());
    return CKO_INVALID_TIME_GRID;
  } catch (const ShapeMismatch& x) {
    fill(e, CKO_SHAPE_MISMATCH, x.what());
    return CKO_SHAPE_MISMATCH;
  } catch (const Error& x) {
    fill(e, CKO_ERROR, x.what());
    return CKO_ERROR;
  } catch (const std::exception& x) {
    fill(e, CKO_ERROR, x.what());
    return CKO_ERROR;
  }
}

// Build the reference model for a descriptor, then adopt desc->params.
std::unique_ptr<OdeModel> build(const cko_model_desc* d) {
  std::unique_ptr<OdeModel> m;
  const int nb = d->n_batch_model;
  switch (d->kind) {
    case CKO_MODEL_SCALAR_DECAY: m = build_scalar_decay(1.0); break;
    case CKO_MODEL_CONSTANT_RATE: m = build_constant_rate(0.0); break;
    case CKO_MODEL_MDS: m = build_mass_damper_spring(d->n_unit, nb); break;
    case CKO_MODEL_CHABOCHE: m = build_chaboche(d->n_unit, nb); break;
    case CKO_MODEL_NEURON: m = build_neuron(d->n_unit, nb); break;
    case CKO_MODEL_LIN3: m = std::make_unique<cko_ref::Lin3>(cko_ref::Lin3::default_params(), nb); break;
    case CKO_MODEL_NODE:
      if (d->width == d->n_unit + 1)
        m = build_neural_ode(d->n_unit, nb, 7);
      else
        m = std::make_unique<cko_ref::NodeWide>(
            d->n_unit, d->width, nb, cko_ref::NodeWide::default_params(d->n_unit, d->width, 7));
      break;
    default: throw StrategyUnavailable("ref_capi: unknown model kind");
  }
  if (d->params && d->n_params > 0)
    m = m->with_params(std::span<const double>(d->params, size_t(d->n_params)));
  return m;
}

SolverChoice solver_of(const cko_solver_choice* s) {
  SolverChoice c;
  c.kind = s->kind == CKO_SOLVER_PCR ? SolverKind::pcr
           : s->kind == CKO_SOLVER_HYBRID ? SolverKind::hybrid
                                          : SolverKind::thomas;
  c.n_switch = s->n_switch;
  return c;
}

void put_work(cko_work* w, const WorkCounters& c) {
  if (!w) return;
  w->newton_iterations = c.newton_iterations;
  w->rate_evals = c.rate_evals;
  w->jacobian_evals = c.jacobian_evals;
  w->linear_solves = c.linear_solves;
  w->reduction_sweeps = c.reduction_sweeps;
}

TimeGrid grid_of(const double* times, int nb, int nt) {
  Array2d t(nt + 1, nb);
  std::memcpy(t.data(), times, sizeof(double) * size_t(nt + 1) * nb);
  return TimeGrid(std::move(t));
}

}  // namespace

extern "C" {

// JacobianStrategy of the following reference calls on this thread (0 analytic, 1 forward_ad,
// 2 finite_difference).
void ref_set_jacobian_strategy(int s) {
  g_strategy = s == 1 ? JacobianStrategy::forward_ad
               : s == 2 ? JacobianStrategy::finite_difference : JacobianStrategy::analytic;
}

// Default parameters of the reference builders (models.hpp:14-41); for NODE
// the `seed` drives mt19937_64 exactly as the reference does.
int ref_default_params(const cko_model_desc* d, unsigned long long seed, double* out, int cap,
                       cko_error* err) {
  try {
    std::vector<double> p;
    if (d->kind == CKO_MODEL_NODE && d->width != d->n_unit + 1)
      p = cko_ref::NodeWide::default_params(d->n_unit, d->width, seed);
    else if (d->kind == CKO_MODEL_NODE)
      p = build_neural_ode(d->n_unit, d->n_batch_model, seed)->params();
    else {
      cko_model_desc dd = *d;
      dd.params = nullptr;
      dd.n_params = 0;
      p = build(&dd)->params();
    }
    if (int(p.size()) > cap) throw Error("ref_default_params: buffer too small");
    std::memcpy(out, p.data(), sizeof(double) * p.size());
    fill(err, CKO_OK, "");
    return int(p.size());
  } catch (...) {
    return -map_exception(err);
  }
}

int ref_forward(const cko_model_desc* d, const double* y0, const double* times, int nb, int nt,
                int n_chunk, const cko_newton_settings* st, const cko_solver_choice* sv,
                double* states_out, cko_work* work, cko_error* err) {
  try {
    auto m = build(d);
    Array2d Y0(nb, m->state_size());
    std::memcpy(Y0.data(), y0, sizeof(double) * Y0.size());
    NewtonSettings ns{st->tol_a, st->tol_r, st->max_iter};
    Trajectory tr =
        integrate_backward_euler(*m, Y0, grid_of(times, nb, nt), n_chunk, ns, solver_of(sv), g_strategy);
    std::memcpy(states_out, tr.states.data(), sizeof(double) * tr.states.size());
    put_work(work, tr.work);
    fill(err, CKO_OK, "");
    return 0;
  } catch (...) {
    return map_exception(err);
  }
}

int ref_adjoint(const cko_model_desc* d, const double* states, const double* times, int nb, int nt,
                int n_chunk, const cko_solver_choice* sv, int loss_kind, const double* dL,
                double* loss_out, double* grad_out, cko_work* bwd, cko_error* err) {
  try {
    auto m = build(d);
    Trajectory tr;
    tr.grid = grid_of(times, nb, nt);
    tr.n_batch = nb;
    tr.n_size = m->state_size();
    tr.states = Array2d(nt + 1, nb * tr.n_size);
    std::memcpy(tr.states.data(), states, sizeof(double) * tr.states.size());
    LossSpec loss = loss_frobenius();
    if (loss_kind == CKO_LOSS_USER) {
      const double* g = dL;
      loss.value = [](const Trajectory&) { return std::nan(""); };
      loss.state_gradient = [g](const Trajectory&, Array2d& out) {
        std::memcpy(out.data(), g, sizeof(double) * out.size());
      };
    }
    WorkCounters w;
    auto [L, grad] = adjoint_backward(*m, tr, n_chunk, loss, Scheme::backward_euler, solver_of(sv),
                                      g_strategy, &w);
    if (loss_out) *loss_out = L;
    std::memcpy(grad_out, grad.data(), sizeof(double) * grad.size());
    put_work(bwd, w);
    fill(err, CKO_OK, "");
    return 0;
  } catch (...) {
    return map_exception(err);
  }
}

// integrate_forward_euler (integrate.cpp:371-407).
int ref_fe_forward(const cko_model_desc* d, const double* y0, const double* times, int nb, int nt, int n_chunk,
                   double* states_out, cko_work* work, cko_error* err) {
  try {
    auto m = build(d);
    Array2d Y0(nb, m->state_size());
    std::memcpy(Y0.data(), y0, sizeof(double) * Y0.size());
    Trajectory tr = integrate_forward_euler(*m, Y0, grid_of(times, nb, nt), n_chunk);
    std::memcpy(states_out, tr.states.data(), sizeof(double) * tr.states.size());
    put_work(work, tr.work);
    fill(err, CKO_OK, "");
    return 0;
  } catch (...) {
    return map_exception(err);
  }
}

// adjoint_backward(..., Scheme::forward_euler, ...) (adjoint.cpp:157-188, 263-297).
int ref_fe_adjoint(const cko_model_desc* d, const double* states, const double* times, int nb, int nt, int n_chunk,
                   int loss_kind, const double* dL, double* loss_out, double* grad_out, cko_work* bwd,
                   cko_error* err) {
  try {
    auto m = build(d);
    Trajectory tr;
    tr.grid = grid_of(times, nb, nt);
    tr.n_batch = nb;
    tr.n_size = m->state_size();
    tr.states = Array2d(nt + 1, nb * tr.n_size);
    std::memcpy(tr.states.data(), states, sizeof(double) * tr.states.size());
    LossSpec loss = loss_frobenius();
    if (loss_kind == CKO_LOSS_USER) {
      const double* g = dL;
      loss.value = [](const Trajectory&) { return std::nan(""); };
      loss.state_gradient = [g](const Trajectory&, Array2d& out) {
        std::memcpy(out.data(), g, sizeof(double) * out.size());
      };
    }
    WorkCounters w;
    auto [L, grad] = adjoint_backward(*m, tr, n_chunk, loss, Scheme::forward_euler, SolverChoice{},
                                      g_strategy, &w);
    if (loss_out) *loss_out = L;
    std::memcpy(grad_out, grad.data(), sizeof(double) * grad.size());
    put_work(bwd, w);
    fill(err, CKO_OK, "");
    return 0;
  } catch (...) {
    return map_exception(err);
  }
}

// gradient_adjoint (adjoint.cpp:299-313) with timings of both phases.
int ref_gradient_adjoint(const cko_model_desc* d, const double* y0, const double* times, int nb,
                         int nt, int n_chunk, const cko_newton_settings* st,
                         const cko_solver_choice* sv, double* states_out, double* loss_out,
                         double* grad_out, cko_work* fwd, cko_work* bwd, double* seconds,
                         cko_error* err) {
  try {
    auto m = build(d);
    Array2d Y0(nb, m->state_size());
    std::memcpy(Y0.data(), y0, sizeof(double) * Y0.size());
    NewtonSettings ns{st->tol_a, st->tol_r, st->max_iter};
    const auto grid = grid_of(times, nb, nt);
    const auto t0 = std::chrono::steady_clock::now();
    Trajectory tr = integrate_backward_euler(*m, Y0, grid, n_chunk, ns, solver_of(sv), g_strategy);
    const auto t1 = std::chrono::steady_clock::now();
    WorkCounters w;
    auto [L, grad] = adjoint_backward(*m, tr, n_chunk, loss_frobenius(), Scheme::backward_euler,
                                      solver_of(sv), g_strategy, &w);
    const auto t2 = std::chrono::steady_clock::now();
    if (seconds) {
      seconds[0] = std::chrono::duration<double>(t1 - t0).count();
      seconds[1] = std::chrono::duration<double>(t2 - t1).count();
    }
    if (states_out) std::memcpy(states_out, tr.states.data(), sizeof(double) * tr.states.size());
    if (loss_out) *loss_out = L;
    if (grad_out) std::memcpy(grad_out, grad.data(), sizeof(double) * grad.size());
    put_work(fwd, tr.work);
    put_work(bwd, w);
    fill(err, CKO_OK, "");
    return 0;
  } catch (...) {
    return map_exception(err);
  }
}

// Batch-sharded timing run: `threads` std::threads each run gradient_adjoint
// on a contiguous lane slice (per-lane parameters re-sliced through a model
// built for the slice width). Timing baseline only.
double ref_sharded_seconds(const cko_model_desc* d, const double* y0, const double* times, int nb,
                           int nt, int n_chunk, const cko_newton_settings* st,
                           const cko_solver_choice* sv, int threads) {
  if (threads < 1) threads = 1;
  if (threads > nb) threads = nb;
  std::vector<std::thread> pool;
  std::vector<int> rc(threads, 0);
  const int n = cko_model_state_size(d);
  // per-shard descriptors: slice per-lane parameter segments
  auto run = [&](int i) {
    const int lo = int((long long)nb * i / threads), hi = int((long long)nb * (i + 1) / threads);
    const int nbs = hi - lo;
    std::vector<double> p(d->params, d->params + d->n_params);
    cko_model_desc s = *d;
    s.n_batch_model = nbs;
    std::vector<double> ps;
    if (d->kind == CKO_MODEL_MDS) {
      ps.assign(p.begin(), p.begin() + 3 * d->n_unit + 1);
      ps.insert(ps.end(), p.begin() + 3 * d->n_unit + 1 + lo, p.begin() + 3 * d->n_unit + 1 + hi);
    } else if (d->kind == CKO_MODEL_CHABOCHE) {
      const int o = 6 + 2 * d->n_unit;
      ps.assign(p.begin(), p.begin() + o);
      ps.insert(ps.end(), p.begin() + o + lo, p.begin() + o + hi);
      ps.push_back(p.back());
    } else {
      ps = p;  // lin3 / node periods are re-derived for the slice width (timing only)
    }
    s.params = ps.data();
    s.n_params = int(ps.size());
    std::vector<double> ys(size_t(nbs) * n), ts(size_t(nt + 1) * nbs);
    std::memcpy(ys.data(), y0 + size_t(lo) * n, sizeof(double) * ys.size());
    for (int r = 0; r <= nt; ++r)
      std::memcpy(ts.data() + size_t(r) * nbs, times + size_t(r) * nb + lo, sizeof(double) * nbs);
    std::vector<double> g(ps.size());
    double L;
    cko_work wf, wb;
    cko_error e;
    rc[i] = ref_gradient_adjoint(&s, ys.data(), ts.data(), nbs, nt, n_chunk, st, sv, nullptr, &L,
                                 g.data(), &wf, &wb, nullptr, &e);
  };
  const auto t0 = std::chrono::steady_clock::now();
  for (int i = 0; i < threads; ++i) pool.emplace_back(run, i);
  for (auto& t : pool) t.join();
  const auto t1 = std::chrono::steady_clock::now();
  for (int r : rc)
    if (r) return -1.0;
  return std::chrono::duration<double>(t1 - t0).count();
}

int ref_solve(const cko_solver_choice* sv, int nc, int nb, int n, const double* diag,
              const double* offdiag, double* rhs, long long* sweeps, cko_error* err) {
  try {
    BlockBidiagonalSystem sys(nc, nb, n);
    std::memcpy(sys.diag.data(), diag, sizeof(double) * sys.diag.size());
    BatchedChunkVector x(nc, nb, n);
    std::memcpy(x.data(), rhs, sizeof(double) * x.size());
    long sw = 0;
    if (!offdiag) {
      // the stepper's -I couplings through detail::solve_unit_offdiag
      DiagonalFactorization f = factor_diagonal_blocks(sys);
      BatchedBlockArray scratch(nc > 1 ? nc - 1 : 0, nb, n);
      detail::solve_unit_offdiag(f, scratch, x, solver_of(sv), &sw);
    } else {
      if (nc > 1) std::memcpy(sys.offdiag.data(), offdiag, sizeof(double) * sys.offdiag.size());
      if (sv->kind == CKO_SOLVER_THOMAS)
        x = solve_thomas(sys, x);
      else if (sv->kind == CKO_SOLVER_PCR)
        x = solve_pcr(sys, x, &sw);
      else
        x = solve_hybrid(sys, x, sv->n_switch, &sw);
    }
    std::memcpy(rhs, x.data(), sizeof(double) * x.size());
    if (sweeps) *sweeps = sw;
    fill(err, CKO_OK, "");
    return 0;
  } catch (...) {
    return map_exception(err);
  }
}

int ref_solve_dense(int nc, int nb, int n, const double* diag, const double* offdiag, double* rhs,
                    cko_error* err) {
  try {
    BlockBidiagonalSystem sys(nc, nb, n);
    std::memcpy(sys.diag.data(), diag, sizeof(double) * sys.diag.size());
    if (nc > 1) std::memcpy(sys.offdiag.data(), offdiag, sizeof(double) * sys.offdiag.size());
    BatchedChunkVector x(nc, nb, n);
    std::memcpy(x.data(), rhs, sizeof(double) * x.size());
    x = solve_dense_oracle(sys, x);
    std::memcpy(rhs, x.data(), sizeof(double) * x.size());
    fill(err, CKO_OK, "");
    return 0;
  } catch (...) {
    return map_exception(err);
  }
}

// make_random_system / make_random_rhs (verify.cpp:413-433)
void ref_random_system(int nc, int nb, int n, unsigned long long seed, double* diag,
                       double* offdiag) {
  auto sys = make_random_system(nc, nb, n, seed);
  std::memcpy(diag, sys.diag.data(), sizeof(double) * sys.diag.size());
  if (nc > 1) std::memcpy(offdiag, sys.offdiag.data(), sizeof(double) * sys.offdiag.size());
}
void ref_random_rhs(int nc, int nb, int n, unsigned long long seed, double* rhs) {
  auto r = make_random_rhs(nc, nb, n, seed);
  std::memcpy(rhs, r.data(), sizeof(double) * r.size());
}

// OdeModel::rate / jacobian_state(analytic) / parameter_vjp on a (c, nb) grid.
int ref_model_eval(const cko_model_desc* d, int what, const double* t, const double* y,
                   const double* w, int c, int nb, double* out, cko_error* err) {
  try {
    auto m = build(d);
    const int n = m->state_size();
    Array2d T(c, nb);
    std::memcpy(T.data(), t, sizeof(double) * T.size());
    BatchedChunkVector Y(c, nb, n);
    std::memcpy(Y.data(), y, sizeof(double) * Y.size());
    if (what == 0) {
      BatchedChunkVector o(c, nb, n);
      m->rate(T, Y, o);
      std::memcpy(out, o.data(), sizeof(double) * o.size());
    } else if (what == 1) {
      BatchedBlockArray o(c, nb, n);
      jacobian_state(*m, T, Y, g_strategy, o);
      std::memcpy(out, o.data(), sizeof(double) * o.size());
    } else {
      BatchedChunkVector W(c, nb, n);
      std::memcpy(W.data(), w, sizeof(double) * W.size());
      std::span<double> g(out, m->params().size());
      parameter_vjp(*m, T, Y, W, g);
    }
    fill(err, CKO_OK, "");
    return 0;
  } catch (...) {
    return map_exception(err);
  }
}

// Public single-chunk ops of the reference (integrate.hpp:53-67, adjoint.hpp:36-56).
// op 0 chunk_residual -> out (c, nb, n); op 1 chunk_jacobian -> out diag (c, nb, n, n)
// and out2 offdiag (c-1, nb, n, n); op 2 newton_solve_chunk -> dy in/out, iters.
int ref_chunk_op(const cko_model_desc* d, int op, const double* y_start, double* dy,
                 const double* t_chunk, const double* dt_chunk, int c, int nb,
                 const cko_newton_settings* st, const cko_solver_choice* sv, double* out,
                 double* out2, int* iters, cko_work* work, cko_error* err) {
  try {
    auto m = build(d);
    const int n = m->state_size();
    Array2d ys(nb, n), T(c, nb), DT(c, nb);
    std::memcpy(ys.data(), y_start, sizeof(double) * ys.size());
    std::memcpy(T.data(), t_chunk, sizeof(double) * T.size());
    std::memcpy(DT.data(), dt_chunk, sizeof(double) * DT.size());
    BatchedChunkVector D(c, nb, n);
    std::memcpy(D.data(), dy, sizeof(double) * D.size());
    if (op == 0) {
      BatchedChunkVector o(c, nb, n);
      chunk_residual(*m, ys, D, T, DT, o);
      std::memcpy(out, o.data(), sizeof(double) * o.size());
    } else if (op == 1) {
      BlockBidiagonalSystem sys(c, nb, n);
      chunk_jacobian(*m, ys, D, T, DT, g_strategy, sys);
      std::memcpy(out, sys.diag.data(), sizeof(double) * sys.diag.size());
      if (out2 && c > 1) std::memcpy(out2, sys.offdiag.data(), sizeof(double) * sys.offdiag.size());
    } else {
      WorkCounters w;
      NewtonSettings ns{st->tol_a, st->tol_r, st->max_iter};
      const int it = newton_solve_chunk(*m, ys, D, T, DT, ns, solver_of(sv), g_strategy, &w, 1);
      std::memcpy(dy, D.data(), sizeof(double) * D.size());
      if (iters) *iters = it;
      put_work(work, w);
    }
    fill(err, CKO_OK, "");
    return 0;
  } catch (...) {
    return map_exception(err);
  }
}

// adjoint_chunk_solve over a host trajectory (op 0) or adjoint_step_sequential
// (op 1: states rows [y_prev; y_i], times rows [t_prev; t_i], dL row 1 = dL_i).
int ref_adjoint_chunk(const cko_model_desc* d, int op, const double* states, const double* times,
                      int nb, int nt, int step_hi, int chunk_len, const double* dL,
                      const cko_solver_choice* sv, double* lambda, double* grad, cko_work* work,
                      cko_error* err) {
  try {
    auto m = build(d);
    const int n = m->state_size();
    AdjointState state;
    state.lambda = Array2d(nb, n);
    std::memcpy(state.lambda.data(), lambda, sizeof(double) * state.lambda.size());
    state.grad.assign(grad, grad + m->params().size());
    if (op == 0) {
      Trajectory tr;
      tr.grid = grid_of(times, nb, nt);
      tr.n_batch = nb;
      tr.n_size = n;
      tr.states = Array2d(nt + 1, nb * n);
      std::memcpy(tr.states.data(), states, sizeof(double) * tr.states.size());
      Array2d G(nt + 1, nb * n);
      std::memcpy(G.data(), dL, sizeof(double) * G.size());
      WorkCounters w;
      adjoint_chunk_solve(*m, tr, step_hi, chunk_len, G, state, solver_of(sv), g_strategy, &w);
      put_work(work, w);
    } else {
      Array2d yi(nb, n), yp(nb, n), g(nb, n);
      std::memcpy(yp.data(), states, sizeof(double) * yp.size());
      std::memcpy(yi.data(), states + size_t(nb) * n, sizeof(double) * yi.size());
      std::memcpy(g.data(), dL + size_t(nb) * n, sizeof(double) * g.size());
      adjoint_step_sequential(*m, yi, yp, std::span<const double>(times + nb, nb),
                              std::span<const double>(times, nb), g, state, solver_of(sv),
                              g_strategy);
    }
    std::memcpy(lambda, state.lambda.data(), sizeof(double) * state.lambda.size());
    std::memcpy(grad, state.grad.data(), sizeof(double) * state.grad.size());
    fill(err, CKO_OK, "");
    return 0;
  } catch (...) {
    return map_exception(err);
  }
}

// The reference's benchmark harness: run_study over a grid given as text
// (bench.cpp:346-416) and dump_trajectory (bench.cpp:418-441), CSV into `out`.
// Returns the CSV length, or -(needed length) when `cap` is too small, or -1
// on an exception (message in err).
static int put_text(const std::string& s, char* out, int cap) {
  if (int(s.size()) + 1 > cap) return -int(s.size() + 1);
  std::memcpy(out, s.data(), s.size());
  out[s.size()] = 0;
  return int(s.size());
}

int ref_study_csv(const char* grid_text, char* out, int cap, cko_error* err) {
  try {
    std::istringstream in(grid_text);
    std::ostringstream os;
    run_study(parse_grid_file(in), os, false);
    fill(err, CKO_OK, "");
    return put_text(os.str(), out, cap);
  } catch (...) {
    map_exception(err);
    return -1;
  }
}

int ref_dump_trajectory(const char* problem, int n_unit, int n_batch, int n_time, int n_chunk, const char* solver,
                        int n_switch, const char* integration, double t_max, char* out, int cap, cko_error* err) {
  try {
    TrialConfig cfg;
    cfg.problem = problem;
    cfg.n_unit = n_unit;
    cfg.n_batch = n_batch;
    cfg.n_time = n_time;
    cfg.n_chunk = n_chunk;
    cfg.solver = solver;
    cfg.n_switch = n_switch;
    cfg.integration = integration;
    cfg.t_max = t_max;
    std::ostringstream os;
    dump_trajectory(cfg, os);
    fill(err, CKO_OK, "");
    return put_text(os.str(), out, cap);
  } catch (...) {
    map_exception(err);
    return -1;
  }
}

int cko_model_state_size(const cko_model_desc* d) {
  switch (d->kind) {
    case CKO_MODEL_SCALAR_DECAY:
    case CKO_MODEL_CONSTANT_RATE: return 1;
    case CKO_MODEL_LIN3: return 3;
    case CKO_MODEL_MDS: return 2 * d->n_unit;
    case CKO_MODEL_CHABOCHE: return 2 + d->n_unit;
    case CKO_MODEL_NODE: return d->n_unit;
  }
  return -1;
}

}  // extern "C"
