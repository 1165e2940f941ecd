// chunkode_dropin.cpp — the reference's C++ integrator / adjoint / solver API
// with its EXACT signatures, implemented on the B200 C ABI
// (include/chunkode_b200.h). Compiled against the reference's own headers
// (/root/reference/proj/core/include, never copied) it replaces
// src/integrate.cpp and src/adjoint.cpp and the public solver wrappers of
// src/linalg.cpp; the reference's model layer (ode_model.cpp, models_*.cpp),
// time grid, bench harness and verify suites link unchanged on top of it
// (shim/Makefile builds that library: libchunkode_b200_dropin.so).
//
// Boundary rules:
//  * a model crosses the ABI as cko_model_desc: its kind from name(), its sizes
//    from state_size() / params().size() / n_batch() (no extra arguments);
//    models without a device twin throw StrategyUnavailable — no CPU fallback;
//  * JacobianStrategy: analytic, forward_ad (device dual numbers) and
//    finite_difference are all honoured on the device;
//  * Scheme: backward_euler and forward_euler both run on the device;
//  * LossSpec: loss_frobenius() (defined here) runs fused on the device; any
//    other LossSpec is evaluated through its callbacks and its state gradient
//    is shipped as the adjoint's jumps;
//  * cko_status codes come back as the reference exception types
//    (errors.hpp:9-69) with their location fields.
// One device context per host thread (CUDA device CKO_DEVICE, default 0).
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <memory>
#include <string>
#include <typeinfo>
#include <vector>

#include "chunkode/adjoint.hpp"
#include "chunkode/integrate.hpp"
#include "chunkode/linalg.hpp"
#include "chunkode/ode_model.hpp"
#include "chunkode_b200.h"

namespace chunkode {

namespace {

[[noreturn]] void rethrow(int status, const cko_error& e) {
  const std::string msg = e.msg;
  switch (status) {
    case CKO_SHAPE_MISMATCH: throw ShapeMismatch(msg);
    case CKO_SINGULAR_BLOCK: throw SingularBlock(e.chunk_index, e.batch_index);
    case CKO_NEWTON_DIVERGENCE:
      throw NewtonDivergence(e.chunk_start_step, e.batch_index, e.iterations, e.residual_norm, e.initial_norm);
    case CKO_NON_FINITE: throw NonFiniteOutput(msg);
    case CKO_STRATEGY_UNAVAILABLE: throw StrategyUnavailable(msg);
    case CKO_SIZE_GUARD: throw SizeGuardExceeded(msg);
    case CKO_INVALID_TIME_GRID: throw InvalidTimeGrid(msg);
    default: throw Error("chunkode_b200: " + msg);
  }
}

void check(int status, const cko_error& e) {
  if (status != CKO_OK) rethrow(status, e);
}

struct ThreadCtx {
  cko_ctx* c = nullptr;
  ~ThreadCtx() {
    if (c) cko_ctx_destroy(c);
  }
};

cko_ctx* ctx() {
  thread_local ThreadCtx t;
  if (!t.c) {
    const char* dev = std::getenv("CKO_DEVICE");
    cko_error e{};
    check(cko_ctx_create(dev ? std::atoi(dev) : 0, &t.c, &e), e);
  }
  return t.c;
}

// The device image of one OdeModel (uploaded parameters), released on scope exit.
struct DeviceModel {
  cko_model* m = nullptr;
  std::vector<double> params;
  explicit DeviceModel(const OdeModel& model) {
    const std::string name = model.name();
    const int n = model.state_size();
    const int np = int(model.params().size());
    params = model.params();
    cko_model_desc d{};
    d.n_params = np;
    d.params = params.data();
    d.n_batch_model = model.n_batch();
    if (name == "scalar_decay") {
      d.kind = CKO_MODEL_SCALAR_DECAY;
    } else if (name == "constant_rate") {
      d.kind = CKO_MODEL_CONSTANT_RATE;
    } else if (name == "lin3") {
      d.kind = CKO_MODEL_LIN3;
    } else if (name == "mds") {  // [K(u), C(u), M(u), f_a, T(nb)]
      d.kind = CKO_MODEL_MDS;
      d.n_unit = n / 2;
      d.n_batch_model = np - 3 * d.n_unit - 1;
    } else if (name == "chaboche") {  // [E, n, eta, s0, Kinf, tau, C(u), gamma(u), eps_a(nb), T]
      d.kind = CKO_MODEL_CHABOCHE;
      d.n_unit = n - 2;
      d.n_batch_model = np - 6 - 2 * d.n_unit - 1;
    } else if (name == "neuron") {  // [14 per-unit segments, I_a(nb), T(u)]
      d.kind = CKO_MODEL_NEURON;
      d.n_unit = n / 4;
      d.n_batch_model = np - 15 * d.n_unit;
    } else if (name == "node" || name == "node_wide") {
      // np = W (n+1) + W + W^2 + W + n W + n  ->  W^2 + (2n + 3) W + n - np = 0
      d.kind = CKO_MODEL_NODE;
      d.n_unit = n;
      const double bq = 2.0 * n + 3.0, disc = bq * bq - 4.0 * (double(n) - np);
      d.width = int(std::lround((-bq + std::sqrt(disc)) / 2.0));
    } else {
      throw StrategyUnavailable("model '" + name + "' has no device twin in the B200 path");
    }
    if (cko_model_param_count(&d) != np)
      throw ShapeMismatch("model '" + name + "': parameter count does not match its device twin");
    cko_error e{};
    check(cko_model_create(ctx(), &d, &m, &e), e);
  }
  ~DeviceModel() { cko_model_destroy(m); }
  DeviceModel(const DeviceModel&) = delete;
  DeviceModel& operator=(const DeviceModel&) = delete;
};

// The call's JacobianStrategy on the device context (analytic, forward-mode duals or central differences,
// ode_model.hpp:14); every entry point sets it, so one context serves calls with different strategies.
void use_strategy(JacobianStrategy s) {
  const int k = s == JacobianStrategy::forward_ad          ? CKO_JACOBIAN_FORWARD_AD
                : s == JacobianStrategy::finite_difference ? CKO_JACOBIAN_FINITE_DIFFERENCE
                                                           : CKO_JACOBIAN_ANALYTIC;
  cko_ctx_set_jacobian_strategy(ctx(), k);
}

cko_solver_choice solver_c(const SolverChoice& s) {
  cko_solver_choice c{};
  c.kind = s.kind == SolverKind::pcr ? CKO_SOLVER_PCR : s.kind == SolverKind::hybrid ? CKO_SOLVER_HYBRID
                                                                                      : CKO_SOLVER_THOMAS;
  c.n_switch = s.n_switch;
  return c;
}

void add_work(WorkCounters* w, const cko_work& c) {
  if (!w) return;
  WorkCounters d;
  d.newton_iterations = long(c.newton_iterations);
  d.rate_evals = long(c.rate_evals);
  d.jacobian_evals = long(c.jacobian_evals);
  d.linear_solves = long(c.linear_solves);
  d.reduction_sweeps = long(c.reduction_sweeps);
  *w += d;
}

// check_integrate_args (integrate.cpp:257-265)
void check_integrate(const OdeModel& model, const Array2d& y0, const TimeGrid& grid, int n_chunk) {
  require(y0.cols() == model.state_size(), "integrate: y0 width != state size");
  require(y0.rows() == grid.n_batch(), "integrate: y0 rows != grid batch width");
  require(model.n_batch() == 0 || model.n_batch() == y0.rows(), "integrate: model batch width != y0 rows");
  require(grid.n_time() >= 1, "integrate: need at least one step");
  require(n_chunk >= 1, "integrate: n_chunk must be >= 1");
}

Trajectory make_traj(const TimeGrid& grid, int nb, int ns) {
  Trajectory tr;
  tr.states = Array2d(grid.n_time() + 1, nb * ns);
  tr.grid = grid;
  tr.n_batch = nb;
  tr.n_size = ns;
  return tr;
}

// loss_frobenius() callbacks: their types identify the fused device loss.
struct FrobeniusValue {
  double operator()(const Trajectory& traj) const {
    double s = 0.0;
    for (int step = 1; step <= traj.n_time(); ++step)
      for (double x : traj.states.row(step)) s += x * x;
    return std::sqrt(s);
  }
};
struct FrobeniusGradient {
  void operator()(const Trajectory& traj, Array2d& g) const {
    require(g.rows() == traj.states.rows() && g.cols() == traj.states.cols(),
            "loss gradient: output must be shaped like the trajectory states");
    const double norm = FrobeniusValue{}(traj);
    for (auto& x : g.row(0)) x = 0.0;
    for (int step = 1; step <= traj.n_time(); ++step) {
      const auto y = traj.states.row(step);
      auto out = g.row(step);
      for (size_t i = 0; i < y.size(); ++i) out[i] = norm > 0.0 ? y[i] / norm : 0.0;
    }
  }
};

bool is_frobenius(const LossSpec& loss) {
  return loss.value.target_type() == typeid(FrobeniusValue) &&
         loss.state_gradient.target_type() == typeid(FrobeniusGradient);
}

void check_loss(const LossSpec& loss) {
  require(bool(loss.value) && bool(loss.state_gradient), "loss: both callbacks must be set");
}

}  // namespace

LossSpec loss_frobenius() {
  LossSpec spec;
  spec.value = FrobeniusValue{};
  spec.state_gradient = FrobeniusGradient{};
  return spec;
}

// ---- integrator (integrate.hpp:53-96) --------------------------------------------------------------
Trajectory integrate_backward_euler(const OdeModel& model, const Array2d& y0, const TimeGrid& grid, int n_chunk,
                                    const NewtonSettings& settings, const SolverChoice& solver,
                                    JacobianStrategy strategy) {
  check_integrate(model, y0, grid, n_chunk);
  use_strategy(strategy);
  DeviceModel dm(model);
  const int nb = y0.rows(), ns = y0.cols();
  Trajectory tr = make_traj(grid, nb, ns);
  cko_newton_settings st{settings.tol_a, settings.tol_r, settings.max_iter};
  cko_solver_choice sv = solver_c(solver);
  cko_work w{};
  cko_error e{};
  check(cko_be_forward(ctx(), dm.m, y0.data(), grid.times().data(), nb, grid.n_time(), n_chunk, &st, &sv,
                       tr.states.data(), nullptr, &w, &e),
        e);
  add_work(&tr.work, w);
  return tr;
}

Trajectory integrate_forward_euler(const OdeModel& model, const Array2d& y0, const TimeGrid& grid, int n_chunk) {
  check_integrate(model, y0, grid, n_chunk);
  DeviceModel dm(model);
  const int nb = y0.rows(), ns = y0.cols();
  Trajectory tr = make_traj(grid, nb, ns);
  cko_work w{};
  cko_error e{};
  check(cko_fe_forward(ctx(), dm.m, y0.data(), grid.times().data(), nb, grid.n_time(), n_chunk, tr.states.data(), &w,
                       &e),
        e);
  add_work(&tr.work, w);
  return tr;
}

namespace {
void check_chunk(const OdeModel& model, const Array2d& y_start, const BatchedChunkVector& dy, const Array2d& t_chunk,
                 const Array2d& dt_chunk) {  // check_chunk_args (integrate.cpp:12-21)
  require(y_start.cols() == model.state_size(), "chunk op: y_start width != state size");
  require(dy.n_size() == model.state_size(), "chunk op: dy width != state size");
  require(y_start.rows() == dy.n_batch(), "chunk op: y_start rows != batch width");
  require(t_chunk.rows() == dy.n_chunk() && t_chunk.cols() == dy.n_batch(),
          "chunk op: t_chunk must be (chunk_len, n_batch)");
  require(dt_chunk.rows() == dy.n_chunk() && dt_chunk.cols() == dy.n_batch(),
          "chunk op: dt_chunk must be (chunk_len, n_batch)");
}
}  // namespace

void chunk_residual(const OdeModel& model, const Array2d& y_start, const BatchedChunkVector& dy,
                    const Array2d& t_chunk, const Array2d& dt_chunk, BatchedChunkVector& out) {
  check_chunk(model, y_start, dy, t_chunk, dt_chunk);
  require(out.n_chunk() == dy.n_chunk() && out.n_batch() == dy.n_batch() && out.n_size() == dy.n_size(),
          "chunk_residual: out must match dy");
  DeviceModel dm(model);
  cko_error e{};
  check(cko_chunk_residual(ctx(), dm.m, y_start.data(), dy.data(), t_chunk.data(), dt_chunk.data(), dy.n_chunk(),
                           dy.n_batch(), out.data(), &e),
        e);
}

void chunk_jacobian(const OdeModel& model, const Array2d& y_start, const BatchedChunkVector& dy,
                    const Array2d& t_chunk, const Array2d& dt_chunk, JacobianStrategy strategy,
                    BlockBidiagonalSystem& out) {
  check_chunk(model, y_start, dy, t_chunk, dt_chunk);
  require(out.n_chunk() == dy.n_chunk() && out.n_batch() == dy.n_batch() && out.n_size() == dy.n_size(),
          "chunk_jacobian: out system shape must match dy");
  use_strategy(strategy);
  DeviceModel dm(model);
  cko_error e{};
  check(cko_chunk_jacobian(ctx(), dm.m, y_start.data(), dy.data(), t_chunk.data(), dt_chunk.data(), dy.n_chunk(),
                           dy.n_batch(), out.diag.data(), dy.n_chunk() > 1 ? out.offdiag.data() : nullptr, &e),
        e);
}

int newton_solve_chunk(const OdeModel& model, const Array2d& y_start, BatchedChunkVector& dy,
                       const Array2d& t_chunk, const Array2d& dt_chunk, const NewtonSettings& settings,
                       const SolverChoice& solver, JacobianStrategy strategy, WorkCounters* work,
                       int chunk_start_step) {
  check_chunk(model, y_start, dy, t_chunk, dt_chunk);
  use_strategy(strategy);
  DeviceModel dm(model);
  cko_newton_settings st{settings.tol_a, settings.tol_r, settings.max_iter};
  cko_solver_choice sv = solver_c(solver);
  cko_work w{};
  cko_error e{};
  int it = 0;
  check(cko_newton_solve_chunk(ctx(), dm.m, y_start.data(), dy.data(), t_chunk.data(), dt_chunk.data(),
                               dy.n_chunk(), dy.n_batch(), &st, &sv, chunk_start_step, &it, &w, &e),
        e);
  add_work(work, w);
  return it;
}

// ---- adjoint (adjoint.hpp:24-89) -------------------------------------------------------------------
std::pair<double, std::vector<double>> adjoint_backward(const OdeModel& model, const Trajectory& traj, int n_chunk,
                                                        const LossSpec& loss, Scheme scheme,
                                                        const SolverChoice& solver, JacobianStrategy strategy,
                                                        WorkCounters* work) {
  check_loss(loss);
  require(traj.n_size == model.state_size(), "adjoint: trajectory width != model size");
  require(n_chunk >= 1, "adjoint: n_chunk must be >= 1");
  use_strategy(strategy);
  DeviceModel dm(model);
  const bool fused = is_frobenius(loss);
  double L = 0.0;
  Array2d dL;
  if (!fused) {
    L = loss.value(traj);
    dL = Array2d(traj.states.rows(), traj.states.cols());
    loss.state_gradient(traj, dL);
  }
  std::vector<double> grad(model.params().size(), 0.0);
  const int kind = fused ? CKO_LOSS_FROBENIUS : CKO_LOSS_USER;
  double Ldev = 0.0;
  cko_work w{};
  cko_error e{};
  if (scheme == Scheme::backward_euler) {
    cko_solver_choice sv = solver_c(solver);
    check(cko_be_adjoint_host(ctx(), dm.m, traj.states.data(), traj.grid.times().data(), traj.n_batch,
                              traj.n_time(), n_chunk, &sv, kind, fused ? nullptr : dL.data(), &Ldev, grad.data(), &w,
                              &e),
          e);
  } else {
    check(cko_fe_adjoint_host(ctx(), dm.m, traj.states.data(), traj.grid.times().data(), traj.n_batch,
                              traj.n_time(), n_chunk, kind, fused ? nullptr : dL.data(), &Ldev, grad.data(), &w, &e),
          e);
  }
  add_work(work, w);
  return {fused ? Ldev : L, std::move(grad)};
}

GradientResult gradient_adjoint(const OdeModel& model, const Array2d& y0, const TimeGrid& grid, int n_chunk,
                                const LossSpec& loss, Scheme scheme, const SolverChoice& solver,
                                JacobianStrategy strategy, const NewtonSettings& settings) {
  GradientResult res;
  if (scheme == Scheme::backward_euler && is_frobenius(loss)) {  // one upload, the trajectory stays resident
    check_integrate(model, y0, grid, n_chunk);
    use_strategy(strategy);
    DeviceModel dm(model);
    const int nb = y0.rows(), ns = y0.cols();
    res.trajectory = make_traj(grid, nb, ns);
    res.gradient.assign(model.params().size(), 0.0);
    cko_newton_settings st{settings.tol_a, settings.tol_r, settings.max_iter};
    cko_solver_choice sv = solver_c(solver);
    cko_work wf{}, wb{};
    cko_error e{};
    check(cko_gradient_adjoint(ctx(), dm.m, y0.data(), grid.times().data(), nb, grid.n_time(), n_chunk, &st, &sv,
                               res.trajectory.states.data(), &res.loss, res.gradient.data(), &wf, &wb, &e),
          e);
    add_work(&res.trajectory.work, wf);
    add_work(&res.backward_work, wb);
    return res;
  }
  res.trajectory = scheme == Scheme::backward_euler
                       ? integrate_backward_euler(model, y0, grid, n_chunk, settings, solver, strategy)
                       : integrate_forward_euler(model, y0, grid, n_chunk);
  auto [L, g] = adjoint_backward(model, res.trajectory, n_chunk, loss, scheme, solver, strategy, &res.backward_work);
  res.loss = L;
  res.gradient = std::move(g);
  return res;
}

namespace {
void check_state(const OdeModel& model, const AdjointState& state, int nb) {  // adjoint.cpp:129-134
  require(state.lambda.rows() == nb && state.lambda.cols() == model.state_size(),
          "adjoint: lambda must be (n_batch, n_size)");
  require(state.grad.size() == model.params().size(), "adjoint: gradient accumulator length != parameter count");
}
}  // namespace

void adjoint_step_sequential(const OdeModel& model, const Array2d& y_i, const Array2d& y_prev,
                             std::span<const double> t_i, std::span<const double> t_prev, const Array2d& dL_dy_i,
                             AdjointState& state, const SolverChoice& solver, JacobianStrategy strategy) {
  const int nb = y_i.rows(), ns = y_i.cols();
  require(ns == model.state_size(), "adjoint step: state width != model size");
  require(y_prev.rows() == nb && y_prev.cols() == ns, "adjoint step: y_prev shape");
  require(int(t_i.size()) == nb && int(t_prev.size()) == nb, "adjoint step: time spans");
  require(dL_dy_i.rows() == nb && dL_dy_i.cols() == ns, "adjoint step: loss jump shape");
  check_state(model, state, nb);
  use_strategy(strategy);
  DeviceModel dm(model);
  cko_solver_choice sv = solver_c(solver);
  cko_error e{};
  check(cko_adjoint_step_sequential(ctx(), dm.m, y_i.data(), y_prev.data(), t_i.data(), t_prev.data(),
                                    dL_dy_i.data(), nb, &sv, state.lambda.data(), state.grad.data(), &e),
        e);
}

void adjoint_chunk_solve(const OdeModel& model, const Trajectory& traj, int step_hi, int chunk_len,
                         const Array2d& dL_dy, AdjointState& state, const SolverChoice& solver,
                         JacobianStrategy strategy, WorkCounters* work) {
  require(traj.n_size == model.state_size(), "adjoint chunk: trajectory width != model size");
  require(chunk_len >= 1 && step_hi >= chunk_len && step_hi <= traj.n_time(),
          "adjoint chunk: step range out of bounds");
  require(dL_dy.rows() == traj.states.rows() && dL_dy.cols() == traj.states.cols(),
          "adjoint chunk: dL_dy must be shaped like the trajectory states");
  check_state(model, state, traj.n_batch);
  use_strategy(strategy);
  DeviceModel dm(model);
  cko_solver_choice sv = solver_c(solver);
  cko_work w{};
  cko_error e{};
  check(cko_adjoint_chunk_solve(ctx(), dm.m, traj.states.data(), traj.grid.times().data(), traj.n_batch,
                                traj.n_time(), step_hi, chunk_len, dL_dy.data(), &sv, state.lambda.data(),
                                state.grad.data(), &w, &e),
        e);
  add_work(work, w);
}

// Central-difference reference gradient (adjoint.cpp:315-342) on the device integrator.
std::vector<double> gradient_fd_oracle(const OdeModel& model, const Array2d& y0, const TimeGrid& grid,
                                       const LossSpec& loss, Scheme scheme, const NewtonSettings& settings) {
  check_loss(loss);
  const std::vector<double>& p0 = model.params();
  if (p0.size() > 500)
    throw SizeGuardExceeded("finite-difference gradient guarded to 500 parameters, got " + std::to_string(p0.size()));
  const JacobianStrategy strategy = preferred_jacobian_strategy(model);
  std::vector<double> g(p0.size(), 0.0), p(p0);
  for (size_t j = 0; j < p0.size(); ++j) {
    const double delta = 1e-6 * (1.0 + std::fabs(p0[j]));
    double L[2];
    for (int side = 0; side < 2; ++side) {
      p[j] = p0[j] + (side == 0 ? delta : -delta);
      auto m = model.with_params(p);
      const Trajectory traj = scheme == Scheme::backward_euler
                                  ? integrate_backward_euler(*m, y0, grid, 1, settings, SolverChoice{}, strategy)
                                  : integrate_forward_euler(*m, y0, grid, 1);
      L[side] = loss.value(traj);
    }
    p[j] = p0[j];
    g[j] = (L[0] - L[1]) / (2.0 * delta);
  }
  return g;
}

// ---- public block-bidiagonal solvers (linalg.hpp:55-81) ---------------------------------------------
namespace {
BatchedChunkVector solve_on_device(const BlockBidiagonalSystem& sys, const BatchedChunkVector& rhs,
                                   const cko_solver_choice& sv, long* sweep_count) {
  require(sys.n_chunk() >= 1 && sys.n_batch() >= 1 && sys.n_size() >= 1, "block bidiagonal system must be non-empty");
  if (sys.n_chunk() > 1)
    require(sys.offdiag.n_chunk() == sys.n_chunk() - 1 && sys.offdiag.n_batch() == sys.n_batch() &&
                sys.offdiag.n_size() == sys.n_size(),
            "off-diagonal block array must be (n_chunk-1, n_batch, n_size, n_size)");
  require(rhs.n_chunk() == sys.n_chunk() && rhs.n_batch() == sys.n_batch() && rhs.n_size() == sys.n_size(),
          "right-hand side shape must match the system");
  BatchedChunkVector x = rhs;
  long long sw = 0;
  cko_error e{};
  check(cko_block_bidiag_solve(ctx(), &sv, sys.n_chunk(), sys.n_batch(), sys.n_size(), sys.diag.data(),
                               sys.offdiag.data(), x.data(), &sw, &e),
        e);
  if (sweep_count) *sweep_count = long(sw);
  return x;
}
}  // namespace

BatchedChunkVector solve_thomas(const BlockBidiagonalSystem& sys, const BatchedChunkVector& rhs) {
  return solve_on_device(sys, rhs, cko_solver_choice{CKO_SOLVER_THOMAS, 1}, nullptr);
}

BatchedChunkVector solve_pcr(const BlockBidiagonalSystem& sys, const BatchedChunkVector& rhs, long* sweep_count) {
  return solve_on_device(sys, rhs, cko_solver_choice{CKO_SOLVER_PCR, 1}, sweep_count);
}

BatchedChunkVector solve_hybrid(const BlockBidiagonalSystem& sys, const BatchedChunkVector& rhs, int n_switch,
                                long* sweep_count) {
  if (n_switch < 0) throw Error("solve_hybrid: n_switch must be >= 0");
  return solve_on_device(sys, rhs, cko_solver_choice{CKO_SOLVER_HYBRID, n_switch}, sweep_count);
}

}  // namespace chunkode
