// acceptance_b200.cpp — the reference's release gate (SPEC.md:512-521,
// /root/reference/proj/tests/acceptance.cpp) replayed against the DROP-IN
// library: this program is written against the reference's own C++ API
// (chunkode/*.hpp, unchanged signatures) and links libchunkode_b200_dropin.so,
// so every integrate / adjoint / solve call below runs on the B200.
//
// Criteria replayed (numbering of acceptance.cpp): 1 solver equivalence with the
// dense oracle, 2 implicit-stepping correctness, 3 chunk invariance, 4 adjoint
// vs central differences (both schemes), 5 derivative strategies of the model
// layer, 7 reduction sweep accounting, 8 study determinism with the CSV schema.
// Criterion 6 is a CPU wall-clock trend and does not apply. All four benchmark
// models run on their device twins (mds, neuron, chaboche, node).
// One PASS/FAIL line per criterion; exit status = number of failures.
#include <chrono>
#include <cmath>
#include <cstdio>
#include <functional>
#include <random>
#include <sstream>
#include <string>
#include <vector>

#include "chunkode/adjoint.hpp"
#include "chunkode/bench.hpp"
#include "chunkode/integrate.hpp"
#include "chunkode/linalg.hpp"
#include "chunkode/models.hpp"
#include "chunkode/verify.hpp"

using namespace chunkode;

namespace {

double inf_norm(const double* a, size_t n) {
  double m = 0.0;
  for (size_t i = 0; i < n; ++i) m = std::max(m, std::fabs(a[i]));
  return m;
}
double inf_gap(const double* a, const double* b, size_t n) {
  double m = 0.0;
  for (size_t i = 0; i < n; ++i) m = std::max(m, std::fabs(a[i] - b[i]));
  return m;
}
// the gate's relative measure: gap / max(1, |ref|_inf)
double gate_rel(const double* a, const double* ref, size_t n) {
  return inf_gap(a, ref, n) / std::max(1.0, inf_norm(ref, n));
}
Array2d zeros(int r, int c) { return Array2d(r, c); }

std::string say(const char* f, double a = 0, double b = 0, double c = 0) {
  char buf[300];
  std::snprintf(buf, sizeof buf, f, a, b, c);
  return buf;
}

// 1 -----------------------------------------------------------------------------------------------
std::string solvers_match_dense() {
  unsigned long long seed = 2000;
  const int chunk_counts[] = {1, 2, 3, 4, 5, 6, 7, 9, 12, 16, 17, 24, 31, 32, 33};
  for (int nc : chunk_counts)
    for (int ns = 1; ns <= 5; ++ns)
      for (int nb = 1; nb <= 3; ++nb) {
        const BlockBidiagonalSystem sys = make_random_system(nc, nb, ns, seed);
        const BatchedChunkVector rhs = make_random_rhs(nc, nb, ns, seed + 1);
        seed += 2;
        const BatchedChunkVector dense = solve_dense_oracle(sys, rhs);
        const std::pair<const char*, BatchedChunkVector> got[] = {
            {"thomas", solve_thomas(sys, rhs)},       {"pcr", solve_pcr(sys, rhs)},
            {"hybrid0", solve_hybrid(sys, rhs, 0)},   {"hybrid2", solve_hybrid(sys, rhs, 2)},
            {"hybrid30", solve_hybrid(sys, rhs, 30)}};
        for (const auto& [name, x] : got) {
          const double e = gate_rel(x.data(), dense.data(), x.size());
          if (e > 1e-9) {
            std::ostringstream m;
            m << name << " differs by " << e << " (nc=" << nc << " ns=" << ns << " nb=" << nb << ")";
            return m.str();
          }
        }
      }
  return "";
}

// 2 -----------------------------------------------------------------------------------------------
std::string implicit_stepping() {
  {  // one step of dy/dt = -p y is y / (1 + p dt)
    auto m = build_scalar_decay(2.5);
    Array2d y0 = zeros(1, 1);
    y0(0, 0) = 1.3;
    const Trajectory tr = integrate_backward_euler(*m, y0, TimeGrid::uniform(1, 1, 0.1), 1);
    const double want = 1.3 / (1.0 + 2.5 * 0.1);
    if (std::fabs(tr.point(1, 0)[0] - want) > 1e-14 * std::fabs(want)) return "closed-form step off";
  }
  {  // first order: halving dt halves the error
    auto m = build_scalar_decay(1.0);
    Array2d y0 = zeros(1, 1);
    y0(0, 0) = 1.0;
    double last = 0.0;
    for (int n = 16; n <= 128; n *= 2) {
      const Trajectory tr =
          integrate_backward_euler(*m, y0, TimeGrid::uniform(n, 1, 1.0), 4, NewtonSettings{1e-13, 1e-12, 100});
      const double err = std::fabs(tr.point(n, 0)[0] - std::exp(-1.0));
      if (n > 16 && (last / err < 1.8 || last / err > 2.2)) return say("error ratio %.3f at n=%g", last / err, n);
      last = err;
    }
  }
  {  // stiff p = 1e6: implicit stays bounded, explicit overflows
    auto m = build_scalar_decay(1e6);
    Array2d y0 = zeros(1, 1);
    y0(0, 0) = 1.0;
    const TimeGrid g = TimeGrid::uniform(60, 1, 60.0);
    const Trajectory tr = integrate_backward_euler(*m, y0, g, 10);
    for (int s = 1; s <= 60; ++s)
      if (!(std::fabs(tr.point(s, 0)[0]) <= 1.0)) return say("implicit left [-1, 1] at step %g", s);
    try {
      integrate_forward_euler(*m, y0, g);
      return "explicit scheme stayed finite";
    } catch (const NonFiniteOutput&) {
    }
  }
  return "";
}

// 3 -----------------------------------------------------------------------------------------------
std::string chunk_invariance() {
  const int nt = 64, nb = 3;
  const NewtonSettings tight{1e-12, 1e-10, 100};
  const std::pair<const char*, int> models[] = {{"mds", 3}, {"neuron", 2}, {"chaboche", 3}, {"node", 3}};
  for (const auto& [key, nu] : models) {
    auto m = build_problem(key, nu, nb);
    const Array2d y0 = zeros(nb, m->state_size());
    const TimeGrid g = TimeGrid::uniform(nt, nb, m->default_t_max());
    std::vector<GradientResult> runs;
    const int chunks[] = {1, 2, 4, 8, 16, 64};
    for (int nc : chunks)
      runs.push_back(gradient_adjoint(*m, y0, g, nc, loss_frobenius(), Scheme::backward_euler, SolverChoice{},
                                      preferred_jacobian_strategy(*m), tight));
    for (size_t i = 0; i < runs.size(); ++i)
      for (size_t j = i + 1; j < runs.size(); ++j) {
        const auto& a = runs[i].trajectory.states;
        const auto& b = runs[j].trajectory.states;
        if (inf_gap(a.data(), b.data(), a.size()) > 1e-6)
          return std::string(key) + say(": trajectories differ (n_chunk %g vs %g)", chunks[i], chunks[j]);
        if (gate_rel(runs[i].gradient.data(), runs[j].gradient.data(), runs[i].gradient.size()) > 1e-8)
          return std::string(key) + say(": gradients differ (n_chunk %g vs %g)", chunks[i], chunks[j]);
      }
  }
  return "";
}

// 4 -----------------------------------------------------------------------------------------------
std::string adjoint_vs_differences() {
  const NewtonSettings tight{1e-12, 1e-10, 100};
  struct C {
    const char* key;
    double t_implicit, t_explicit;  // 0: the model's default horizon
  };
  for (const C c : {C{"mds", 2e-4, 2e-4}, C{"neuron", 0.0, 0.5}, C{"chaboche", 0.0, 0.3}, C{"node", 0.0, 1.0}}) {
    auto m = build_problem(c.key, 2, 2);
    const Array2d y0 = zeros(2, m->state_size());
    for (const Scheme sc : {Scheme::backward_euler, Scheme::forward_euler}) {
      const bool be = sc == Scheme::backward_euler;
      const double T = be ? (c.t_implicit > 0 ? c.t_implicit : m->default_t_max()) : c.t_explicit;
      const TimeGrid g = TimeGrid::uniform(32, 2, T);
      const GradientResult r =
          gradient_adjoint(*m, y0, g, 4, loss_frobenius(), sc, SolverChoice{}, preferred_jacobian_strategy(*m), tight);
      const std::vector<double> fd = gradient_fd_oracle(*m, y0, g, loss_frobenius(), sc);
      for (size_t j = 0; j < fd.size(); ++j)
        if (std::fabs(r.gradient[j] - fd[j]) > 1e-4 * (1.0 + std::fabs(fd[j]))) {
          std::ostringstream o;
          o << c.key << (be ? " backward" : " forward") << " parameter " << j << ": " << r.gradient[j] << " vs "
            << fd[j];
          return o.str();
        }
    }
  }
  return "";
}

// 5 -----------------------------------------------------------------------------------------------
std::string derivative_strategies() {
  std::mt19937_64 rng(2024);
  std::uniform_real_distribution<double> u(-1.0, 1.0), c01(0.0, 1.0);
  const std::pair<const char*, int> models[] = {{"mds", 2}, {"neuron", 2}, {"chaboche", 2}, {"node", 2}};
  for (const auto& [key, nu] : models) {
    auto m = build_problem(key, nu, 2);
    const int ns = m->state_size();
    for (int trial = 0; trial < 20; ++trial) {
      Array2d t(1, 2);
      BatchedChunkVector y(1, 2, ns);
      for (int b = 0; b < 2; ++b) {
        t(0, b) = c01(rng) * m->default_t_max();
        auto p = y.point(0, b);
        if (std::string(key) == "chaboche") {  // away from the yield kink
          const bool plastic = c01(rng) < 0.5;
          p[0] = plastic ? 2.0 + 2.0 * c01(rng) : -0.3 + 0.6 * c01(rng);
          p[1] = plastic ? 0.1 + 0.4 * c01(rng) : 1.0 + c01(rng);
          for (int i = 2; i < ns; ++i) p[i] = 0.1 * u(rng);
        } else {
          for (int i = 0; i < ns; ++i) p[i] = u(rng);
        }
      }
      BatchedBlockArray an(1, 2, ns), ad(1, 2, ns), fdj(1, 2, ns);
      jacobian_state(*m, t, y, JacobianStrategy::analytic, an);
      jacobian_state(*m, t, y, JacobianStrategy::forward_ad, ad);
      jacobian_state(*m, t, y, JacobianStrategy::finite_difference, fdj);
      if (inf_gap(ad.data(), an.data(), an.size()) > 1e-12 * std::max(1.0, inf_norm(an.data(), an.size())))
        return std::string(key) + ": forward mode vs analytic";
      if (inf_gap(ad.data(), fdj.data(), ad.size()) > 1e-5 * std::max(1.0, inf_norm(ad.data(), ad.size())))
        return std::string(key) + ": forward mode vs differences";
    }
  }
  return "";
}

// 5b (device): the same agreement through the drop-in's chunk_jacobian, whose blocks I - J dt the B200
// path builds with each strategy (dual numbers and central differences on the device).
std::string device_strategies() {
  const std::pair<const char*, int> models[] = {{"mds", 2}, {"neuron", 2}, {"chaboche", 2}, {"node", 2}};
  std::mt19937_64 rng(77);
  std::uniform_real_distribution<double> u(-0.5, 0.5);
  for (const auto& [key, nu] : models) {
    auto m = build_problem(key, nu, 2);
    const int ns = m->state_size(), c = 3;
    Array2d ys(2, ns), t(c, 2), dt(c, 2);
    for (int b = 0; b < 2; ++b)
      for (int i = 0; i < ns; ++i) ys(b, i) = u(rng);
    for (int k = 0; k < c; ++k)
      for (int b = 0; b < 2; ++b) t(k, b) = 0.01 * (k + 1), dt(k, b) = 0.01;
    BatchedChunkVector dy(c, 2, ns);
    BlockBidiagonalSystem an(c, 2, ns), ad(c, 2, ns), fdj(c, 2, ns);
    chunk_jacobian(*m, ys, dy, t, dt, JacobianStrategy::analytic, an);
    chunk_jacobian(*m, ys, dy, t, dt, JacobianStrategy::forward_ad, ad);
    chunk_jacobian(*m, ys, dy, t, dt, JacobianStrategy::finite_difference, fdj);
    const size_t sz = an.diag.size();
    if (inf_gap(ad.diag.data(), an.diag.data(), sz) > 1e-12 * std::max(1.0, inf_norm(an.diag.data(), sz)))
      return std::string(key) + ": device forward mode vs analytic";
    if (inf_gap(ad.diag.data(), fdj.diag.data(), sz) > 1e-5 * std::max(1.0, inf_norm(ad.diag.data(), sz)))
      return std::string(key) + ": device forward mode vs differences";
  }
  return "";
}

// 7 -----------------------------------------------------------------------------------------------
std::string sweep_accounting() {
  for (int nc = 1; nc <= 33; ++nc) {
    long want = 0;
    for (int e = 0; (1 << e) <= nc; ++e)
      if (nc & (1 << e)) want += e;
    long got = -1;
    solve_pcr(make_random_system(nc, 1, 2, 4000 + nc), make_random_rhs(nc, 1, 2, 4100 + nc), &got);
    if (got != want) return say("n_chunk=%g: %g sweeps, expected %g", nc, double(got), double(want));
  }
  return "";
}

// 8 -----------------------------------------------------------------------------------------------
std::vector<std::vector<std::string>> csv_rows(const std::string& text) {
  std::vector<std::vector<std::string>> rows;
  std::istringstream in(text);
  std::string line;
  while (std::getline(in, line)) {
    std::vector<std::string> f(1);
    for (char ch : line) {
      if (ch == ',')
        f.emplace_back();
      else
        f.back() += ch;
    }
    rows.push_back(f);
  }
  return rows;
}

std::string study_determinism() {
  const char* text =
      "problem = mds, chaboche\nn_unit = 1, 2\nn_batch = 2\nn_time = 16\nn_chunk = 1, 4\nrepeats = 2\n";
  std::ostringstream a, b;
  {
    std::istringstream g(text);
    if (run_study(parse_grid_file(g), a) != 0) return "first study had failed trials";
  }
  {
    std::istringstream g(text);
    if (run_study(parse_grid_file(g), b) != 0) return "second study had failed trials";
  }
  const auto ra = csv_rows(a.str()), rb = csv_rows(b.str());
  std::ostringstream hdr;
  write_csv_header(hdr);
  if (ra.empty() || a.str().substr(0, hdr.str().size()) != hdr.str()) return "header is not the documented schema";
  if (ra.size() != 1 + 8 * 3 || rb.size() != ra.size()) return say("row count %g", double(ra.size()));
  const auto& h = ra[0];
  for (size_t r = 1; r < ra.size(); ++r) {
    if (ra[r].size() != h.size() || rb[r].size() != h.size()) return say("row %g: column count", double(r));
    for (size_t c = 0; c < h.size(); ++c) {
      if (h[c] == "forward_s" || h[c] == "backward_s" || h[c] == "total_s") continue;
      if (ra[r][c] != rb[r][c]) return "row " + std::to_string(r) + " column " + h[c] + " differs";
    }
    if (ra[r].back() != "ok") return "row " + std::to_string(r) + " status " + ra[r].back();
  }
  return "";
}

}  // namespace

int main() {
  const std::pair<const char*, std::function<std::string()>> gate[] = {
      {"1. linear solvers agree with the dense reference (<= 1e-9)", solvers_match_dense},
      {"2. implicit stepping: closed form, first order, stiff-stable", implicit_stepping},
      {"3. chunk-size invariance of trajectories (1e-6) and gradients (1e-8)", chunk_invariance},
      {"4. adjoint gradients match central differences (1e-4), both schemes", adjoint_vs_differences},
      {"5. derivative strategies agree (analytic 1e-12, differences 1e-5)", derivative_strategies},
      {"5b. the same strategies through the device chunk_jacobian", device_strategies},
      {"7. reduction sweep counts follow the power-of-two partitioning", sweep_accounting},
      {"8. study sweeps are deterministic with the documented CSV schema", study_determinism},
  };
  int failed = 0;
  for (const auto& [label, run] : gate) {
    const auto t0 = std::chrono::steady_clock::now();
    std::string why;
    try {
      why = run();
    } catch (const std::exception& e) {
      why = std::string("unexpected exception: ") + e.what();
    }
    const double s = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
    failed += !why.empty();
    std::printf("%s  %-70s [%7.2fs]%s%s\n", why.empty() ? "PASS" : "FAIL", label, s, why.empty() ? "" : "  -- ",
                why.c_str());
    std::fflush(stdout);
  }
  std::printf(failed ? "%d criteria failed\n" : "all criteria satisfied%.0d\n", failed);
  return failed;
}
