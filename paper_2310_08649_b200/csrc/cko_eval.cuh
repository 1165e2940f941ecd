// cko_eval.cuh — templated point evaluations of every device model, the device
// counterpart of ModelBase<Derived>::eval_point<T> (ode_model.hpp:103-188):
// one body serves plain doubles and forward-mode duals, with the parameters
// read through a view (ParamPlain / ParamAsDual / ParamSeeded, cko_dual.cuh).
// On top of them: the JacobianStrategy dispatch of the generic kernels —
// analytic (the hand-written twins), forward_ad (eight Jacobian columns per
// dual pass, jacobian_forward_ad ode_model.hpp:132-151) and finite_difference
// (central differences, jacobian_finite_difference ode_model.cpp:44-66).
// Expression orders follow the reference model sources cited per model.
#pragma once

#include "cko_dual.cuh"

namespace cko {

enum : int { JAC_ANALYTIC = 0, JAC_FORWARD_AD = 1, JAC_FINITE_DIFFERENCE = 2 };
constexpr int CKO_KIND_NEURON = 6;

// models_mds.cpp:27-51
template <class T, class PA>
__device__ void eval_mds(const DevModel& m, const T& t, const PA& p, const T* y, T* out, int b) {
  const int n = m.nu;
  for (int u = 0; u < n; ++u) out[u] = y[n + u];
  for (int u = 0; u < n; ++u) {
    T acc(0.0);
    if (u > 0) acc += (p(u) / p(2 * n + u)) * (y[u] - y[u - 1]) + (p(n + u) / p(2 * n + u)) * (y[n + u] - y[n + u - 1]);
    if (u + 1 < n)
      acc -= (p(u + 1) / p(2 * n + u + 1)) * (y[u + 1] - y[u]) +
             (p(n + u + 1) / p(2 * n + u + 1)) * (y[n + u + 1] - y[n + u]);
    if (u == 0) acc += p(3 * n) * sin(CKO_TWO_PI * t / p(3 * n + 1 + m.off + b));
    out[n + u] = acc;
  }
}

// models_chaboche.cpp:30-62
template <class T, class PA>
__device__ void eval_chaboche(const DevModel& m, const T& t, const PA& p, const T* y, T* out, int b) {
  const int n = m.nu;
  const T E = p(0), nn = p(1), eta = p(2), s0 = p(3), Kinf = p(4), tau = p(5);
  const T ea = p(6 + 2 * n + m.off + b), Tp = p(6 + 2 * n + m.nbm);
  const T& sig = y[0];
  const T& K = y[1];
  T s = sig;
  for (int i = 0; i < n; ++i) s -= y[2 + i];
  const double sg = sign_of(s);
  const T over = (fabs(s) - K - s0) / eta;
  const T ramp = pow(positive_part(over), nn);
  const T ep = ramp * sg;
  const T ep_abs = ramp * (sg * sg);
  out[0] = E * (ea * sin(CKO_TWO_PI * t / Tp) - ep);
  out[1] = tau * (Kinf - K);
  for (int i = 0; i < n; ++i) out[2 + i] = (2.0 / 3.0) * p(6 + i) * ep - p(6 + n + i) * y[2 + i] * ep_abs;
}

// models_node.cpp:37-67 (any hidden width W: the C4 model is W = 128)
template <class T, class PA>
__device__ void eval_node(const DevModel& m, const T& t, const PA& p, const T* y, T* out, int b) {
  const int n = m.n, W = m.W, w0 = n + 1;
  const int oW1 = 0, ob1 = W * w0, oW2 = ob1 + W, ob2 = oW2 + W * W, oW3 = ob2 + W, ob3 = oW3 + n * W;
  T z0[NODE_MAX_N + 1], z1[NODE_MAX_W], z2[NODE_MAX_W];
  for (int i = 0; i < n; ++i) z0[i] = y[i];
  z0[n] = 1.0 * sin(CKO_TWO_PI * t / m.periods[m.off + b]);
  for (int i = 0; i < W; ++i) {
    T acc = p(ob1 + i);
    for (int j = 0; j < w0; ++j) acc += p(oW1 + i * w0 + j) * z0[j];
    z1[i] = tanh(acc);
  }
  for (int i = 0; i < W; ++i) {
    T acc = p(ob2 + i);
    for (int j = 0; j < W; ++j) acc += p(oW2 + i * W + j) * z1[j];
    z2[i] = tanh(acc);
  }
  for (int i = 0; i < n; ++i) {
    T acc = p(ob3 + i);
    for (int j = 0; j < W; ++j) acc += p(oW3 + i * W + j) * z2[j];
    out[i] = tanh(acc);
  }
}

// 3-state linear stiff ODE (oracle/src/ref_models.hpp Lin3): h = A y + [f_a sin(2 pi t / T_b), 0, 0]
template <class T, class PA>
__device__ void eval_lin3(const DevModel& m, const T& t, const PA& p, const T* y, T* out, int b) {
  for (int i = 0; i < 3; ++i) {
    T acc = p(3 * i) * y[0];
    acc += p(3 * i + 1) * y[1];
    acc += p(3 * i + 2) * y[2];
    if (i == 0) acc += p(9) * sin(CKO_TWO_PI * t / m.periods[m.off + b]);
    out[i] = acc;
  }
}

// models_neuron.cpp:28-64: per-unit [C, g_Na, E_Na, g_K, E_K, g_L, E_L, m_inf, tau_m, h_inf, tau_h, n_inf,
// tau_n, g_C] segments, I_a per lane, the per-unit drive periods T.
template <class T, class PA>
__device__ void eval_neuron(const DevModel& m, const T& t, const PA& p, const T* y, T* out, int b) {
  const int n = m.nu;
  T vsum(0.0);
  for (int u = 0; u < n; ++u) vsum += y[4 * u];
  const T Ia = p(14 * n + m.off + b);
  for (int u = 0; u < n; ++u) {
    const T& V = y[4 * u];
    const T& mg = y[4 * u + 1];
    const T& h = y[4 * u + 2];
    const T& ng = y[4 * u + 3];
    const T m3 = mg * mg * mg;
    const T n2 = ng * ng;
    const T n4 = n2 * n2;
    T acc = -p(n + u) * m3 * h * (V - p(2 * n + u)) - p(3 * n + u) * n4 * (V - p(4 * n + u)) -
            p(5 * n + u) * (V - p(6 * n + u));
    acc += Ia * sin(CKO_TWO_PI * t / p(14 * n + m.nbm + u));
    acc += p(13 * n + u) * (double(n) * V - vsum);
    out[4 * u] = acc / p(u);
    out[4 * u + 1] = (p(7 * n + u) - mg) / p(8 * n + u);
    out[4 * u + 2] = (p(9 * n + u) - h) / p(10 * n + u);
    out[4 * u + 3] = (p(11 * n + u) - ng) / p(12 * n + u);
  }
}

// models_simple.cpp:9-45
template <class T, class PA>
__device__ void eval_model(const DevModel& m, const T& t, const PA& p, const T* y, T* out, int b) {
  switch (m.kind) {
    case 0: out[0] = -p(0) * y[0]; break;  // scalar decay
    case 1: out[0] = T(0.0) + p(0); break;  // constant rate
    case 2: eval_lin3(m, t, p, y, out, b); break;
    case 3: eval_mds(m, t, p, y, out, b); break;
    case 4: eval_chaboche(m, t, p, y, out, b); break;
    case 5: eval_node(m, t, p, y, out, b); break;
    case CKO_KIND_NEURON: eval_neuron(m, t, p, y, out, b); break;
  }
}

// jacobian_forward_ad (ode_model.hpp:132-151): eight columns per dual pass, state tangents seeded.
template <class Y, class J>
__device__ void jacobian_fad(const DevModel& m, double t, const Y& y, J& jac, int b) {
  const int n = m.n;
  Dual8 yd[kFadMaxN], od[kFadMaxN];
  for (int j0 = 0; j0 < n; j0 += 8) {
    const int lanes = n - j0 < 8 ? n - j0 : 8;
    for (int i = 0; i < n; ++i) yd[i] = Dual8(y[i]);
    for (int l = 0; l < lanes; ++l) yd[j0 + l].d[l] = 1.0;
    eval_model(m, Dual8(t), ParamAsDual<8>{m.p}, yd, od, b);
    for (int i = 0; i < n; ++i)
      for (int l = 0; l < lanes; ++l) jac(i, j0 + l) = od[i].d[l];
  }
}

// jacobian_finite_difference (ode_model.cpp:44-66): central differences, delta = 1e-6 (1 + |y_j|).
template <class Y, class J>
__device__ void jacobian_fd(const DevModel& m, double t, const Y& y, J& jac, int b) {
  const int n = m.n;
  Exact yp[kFadMaxN], ym[kFadMaxN], rp[kFadMaxN], rm[kFadMaxN];
  for (int i = 0; i < n; ++i) yp[i] = ym[i] = Exact(y[i]);
  for (int j = 0; j < n; ++j) {
    const double yj = yp[j].v;
    const double d = 1e-6 * (1.0 + ::fabs(yj));
    yp[j] = Exact(yj + d);
    ym[j] = Exact(yj - d);
    eval_model(m, Exact(t), ParamExact{m.p}, yp, rp, b);
    eval_model(m, Exact(t), ParamExact{m.p}, ym, rm, b);
    const double inv = 1.0 / (2.0 * d);
    for (int i = 0; i < n; ++i) jac(i, j) = xmul(xsub(rp[i].v, rm[i].v), inv);
    yp[j] = ym[j] = Exact(yj);
  }
}

// The Jacobian the strategy selects (jacobian_state_unscanned, ode_model.cpp:98-123).
template <class MD, class Y, class J>
__device__ inline void model_jacobian(const DevModel& m, double t, const Y& y, J& jac, int b) {
  if (m.jstrat == JAC_FORWARD_AD)
    jacobian_fad(m, t, y, jac, b);
  else if (m.jstrat == JAC_FINITE_DIFFERENCE)
    jacobian_fd(m, t, y, jac, b);
  else
    MD::jacobian(m, t, y, jac, b);
}

// Neuron twin (models_neuron.cpp): rate and analytic Jacobian as in the reference; the parameter product
// is the reference's forward-mode one (the model has no analytic VJP): windows of eight parameters seeded
// per dual pass, the lane's own I_a among them, other lanes' I_a skipped (their tangent is zero).
struct MNeuron {
  template <class Y, class O>
  __device__ static void rate(const DevModel& m, double t, const Y& y, O& out, int b) {
    Exact yl[kFadMaxN], o[kFadMaxN];
    for (int i = 0; i < m.n; ++i) yl[i] = Exact(y[i]);
    eval_neuron(m, Exact(t), ParamExact{m.p}, yl, o, b);
    for (int i = 0; i < m.n; ++i) out[i] = o[i].v;
  }
  // models_neuron.cpp:66-108
  template <class Y, class J>
  __device__ static void jacobian(const DevModel& m, double, const Y& y, J& jac, int) {
    const int n = m.nu, ns = 4 * n;
    const double* p = m.p;
    for (int i = 0; i < ns; ++i)
      for (int j = 0; j < ns; ++j) jac(i, j) = 0.0;
    for (int u = 0; u < n; ++u) {
      const int q = 4 * u;
      const double V = y[q], mg = y[q + 1], h = y[q + 2], ng = y[q + 3];
      const double m3 = mg * mg * mg, n3 = ng * ng * ng;
      const double invC = 1.0 / p[u];
      const double gNa = p[n + u], ENa = p[2 * n + u], gK = p[3 * n + u], EK = p[4 * n + u], gL = p[5 * n + u];
      const double gC = p[13 * n + u];
      for (int j = 0; j < n; ++j) jac(q, 4 * j) = -gC * invC;
      jac(q, q) = xmul(xadd(xsub(xsub(xmul(xmul(-gNa, m3), h), xmul(xmul(gK, n3), ng)), gL), xmul(gC, double(n - 1))),
                       invC);
      jac(q, q + 1) = xmul(xmul(xmul(xmul(xmul(-3.0, gNa), mg), mg), h), V - ENa) * invC;
      jac(q, q + 2) = xmul(xmul(xmul(-gNa, m3), V - ENa), invC);
      jac(q, q + 3) = xmul(xmul(xmul(xmul(-4.0, gK), n3), V - EK), invC);
      jac(q + 1, q + 1) = -1.0 / p[8 * n + u];
      jac(q + 2, q + 2) = -1.0 / p[10 * n + u];
      jac(q + 3, q + 3) = -1.0 / p[12 * n + u];
    }
  }
  template <class Y, class Wt, class G>
  __device__ static void vjp(const DevModel& m, double t, const Y& y, const Wt& w, G& g, int b) {
    const int n = m.n, nu = m.nu, np = m.np;
    const int lo = 14 * nu, hi = lo + m.nbm, own = lo + m.off + b;
    Dual8 yd[kFadMaxN], od[kFadMaxN];
    for (int j0 = 0; j0 < np; j0 += 8) {
      const int lanes = np - j0 < 8 ? np - j0 : 8;
      if (j0 >= lo && j0 + lanes <= hi && !(own >= j0 && own < j0 + lanes)) continue;  // other lanes' I_a only
      for (int i = 0; i < n; ++i) yd[i] = Dual8(y[i]);
      eval_neuron(m, Dual8(t), ParamSeeded<8>{m.p, j0, lanes}, yd, od, b);
      for (int l = 0; l < lanes; ++l) {
        const int j = j0 + l;
        double s = 0.0;
        for (int i = 0; i < n; ++i) s = xadd(s, xmul(w[i], od[i].d[l]));
        if (j >= lo && j < hi) {
          if (j == own) g.lane_add(j, s);
        } else {
          g.add(j, s);
        }
      }
    }
  }
};

}  // namespace cko
