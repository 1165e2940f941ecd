// cko_models.cuh — device twins of the reference ODE models.
//
// Each model exposes, per point (t, y, lane):
//   rate(t, y, out)          h(y, t)            (OdeModel::rate, ode_model.hpp:39-40)
//   jacobian(t, y, J)        dh/dy, every entry (jacobian_analytic)
//   vjp(t, y, w, G)          G += w . dh/dp     (param_vjp_analytic / the Dual8 sweep)
// over generic accessors (Y[i], J(i, j), G.add(j, v)), so the same code runs
// on workspace slabs and on register arrays. Expression orders follow the
// reference sources cited on each model.
#pragma once

#include "cko_common.cuh"

namespace cko {

#define CKO_TWO_PI (2.0 * 3.14159265358979323846)

struct DevModel {
  int kind;
  int n;    // state size
  int nu;   // n_unit
  int W;    // NODE hidden width
  int nbm;  // parameterised batch width
  int off;  // lane offset (global lane of local lane 0)
  int np;   // parameter count
  const double* p;        // device parameters
  const double* periods;  // device per-lane periods (LIN3 / NODE), length nbm
  int jstrat;             // JacobianStrategy of the call: 0 analytic, 1 forward_ad, 2 finite_difference
};

__device__ __forceinline__ double sign_of(double x) { return x > 0.0 ? 1.0 : (x < 0.0 ? -1.0 : 0.0); }

// pow_value (dual.hpp:141-157): integer exponents 0..32 by squaring.
__device__ inline double pow_value(double x, double n) {
  const int ni = (int)n;
  if ((double)ni == n && ni >= 0 && ni <= 32) {
    double r = 1.0, base = x;
    int e = ni;
    while (e > 0) {
      if (e & 1) r = xmul(r, base);
      base = xmul(base, base);
      e >>= 1;
    }
    return r;
  }
  return pow(x, n);
}

// ---------------------------------------------------------------------------
// dy/dt = -p y (models_simple.cpp:9-27); VJP from the Dual8 rule: -y.
struct MScalarDecay {
  template <class Y, class O>
  __device__ static void rate(const DevModel& m, double, const Y& y, O& out, int) {
    out[0] = -m.p[0] * y[0];
  }
  template <class Y, class J>
  __device__ static void jacobian(const DevModel& m, double, const Y&, J& jac, int) {
    jac(0, 0) = -m.p[0];
  }
  template <class Y, class Wt, class G>
  __device__ static void vjp(const DevModel&, double, const Y& y, const Wt& w, G& g, int) {
    g.add(0, w[0] * (-y[0]));
  }
};

// dy/dt = p (models_simple.cpp:29-45).
struct MConstantRate {
  template <class Y, class O>
  __device__ static void rate(const DevModel& m, double, const Y&, O& out, int) {
    out[0] = m.p[0];
  }
  template <class Y, class J>
  __device__ static void jacobian(const DevModel&, double, const Y&, J& jac, int) {
    jac(0, 0) = 0.0;
  }
  template <class Y, class Wt, class G>
  __device__ static void vjp(const DevModel&, double, const Y&, const Wt& w, G& g, int) {
    g.add(0, w[0]);
  }
};

// 3-state linear stiff ODE, config C1 (oracle/src/ref_models.hpp Lin3).
struct MLin3 {
  template <class Y, class O>
  __device__ static void rate(const DevModel& m, double t, const Y& y, O& out, int b) {
    const double* p = m.p;
    const double y0 = y[0], y1 = y[1], y2 = y[2];
#pragma unroll
    for (int i = 0; i < 3; ++i) {
      double acc = xmul(p[3 * i], y0);
      acc = xadd(acc, xmul(p[3 * i + 1], y1));
      acc = xadd(acc, xmul(p[3 * i + 2], y2));
      if (i == 0) acc = xadd(acc, xmul(p[9], sin(CKO_TWO_PI * t / m.periods[m.off + b])));
      out[i] = acc;
    }
  }
  template <class Y, class J>
  __device__ static void jacobian(const DevModel& m, double, const Y&, J& jac, int) {
#pragma unroll
    for (int i = 0; i < 3; ++i)
#pragma unroll
      for (int j = 0; j < 3; ++j) jac(i, j) = m.p[3 * i + j];
  }
  template <class Y, class Wt, class G>
  __device__ static void vjp(const DevModel& m, double t, const Y& y, const Wt& w, G& g, int b) {
#pragma unroll
    for (int i = 0; i < 3; ++i)
#pragma unroll
      for (int j = 0; j < 3; ++j) g.add(3 * i + j, w[i] * y[j]);
    g.add(9, w[0] * sin(CKO_TWO_PI * t / m.periods[m.off + b]));
  }
};

// Mass-damper-spring chain (models_mds.cpp:16-97). The VJP is the closed
// form of SURVEY Appendix A (the reference uses a Dual8 sweep over all
// 3u+1+nb parameters).
struct MMds {
  template <class Y, class O>
  __device__ static void rate(const DevModel& m, double t, const Y& y, O& out, int b) {
    const int n = m.nu;
    const double *K = m.p, *C = m.p + n, *M = m.p + 2 * n;
    const double fa = m.p[3 * n], Tb = m.p[3 * n + 1 + m.off + b];
    for (int u = 0; u < n; ++u) out[u] = y[n + u];
    for (int u = 0; u < n; ++u) {
      double acc = 0.0;
      // no contraction: the reference's separately rounded products and sums
      if (u > 0)
        acc = xadd(acc, xadd(xmul(K[u] / M[u], y[u] - y[u - 1]), xmul(C[u] / M[u], y[n + u] - y[n + u - 1])));
      if (u + 1 < n)
        acc = xsub(acc, xadd(xmul(K[u + 1] / M[u + 1], y[u + 1] - y[u]),
                             xmul(C[u + 1] / M[u + 1], y[n + u + 1] - y[n + u])));
      if (u == 0) acc = xadd(acc, xmul(fa, sin(CKO_TWO_PI * t / Tb)));
      out[n + u] = acc;
    }
  }
  template <class Y, class J>
  __device__ static void jacobian(const DevModel& m, double, const Y&, J& jac, int) {
    const int n = m.nu, ns = 2 * n;
    const double *K = m.p, *C = m.p + n, *M = m.p + 2 * n;
    for (int i = 0; i < ns; ++i)
      for (int j = 0; j < ns; ++j) jac(i, j) = 0.0;
    for (int u = 0; u < n; ++u) {
      jac(u, n + u) = 1.0;
      double a0 = 0.0, c0 = 0.0, am = 0.0, cm = 0.0, ap = 0.0, cp = 0.0;
      if (u > 0) {
        const double a = K[u] / M[u], c = C[u] / M[u];
        a0 += a;
        am -= a;
        c0 += c;
        cm -= c;
      }
      if (u + 1 < n) {
        const double a = K[u + 1] / M[u + 1], c = C[u + 1] / M[u + 1];
        a0 += a;
        ap -= a;
        c0 += c;
        cp -= c;
      }
      jac(n + u, u) = a0;
      jac(n + u, n + u) = c0;
      if (u > 0) jac(n + u, u - 1) = am, jac(n + u, n + u - 1) = cm;
      if (u + 1 < n) jac(n + u, u + 1) = ap, jac(n + u, n + u + 1) = cp;
    }
  }
  template <class Y, class Wt, class G>
  __device__ static void vjp(const DevModel& m, double t, const Y& y, const Wt& w, G& g, int b) {
    const int n = m.nu;
    const double *K = m.p, *C = m.p + n, *M = m.p + 2 * n;
    const double fa = m.p[3 * n], Tb = m.p[3 * n + 1 + m.off + b];
    for (int j = 1; j < n; ++j) {
      const double om = w[n + j] - w[n + j - 1];
      const double dd = y[j] - y[j - 1], dv = y[n + j] - y[n + j - 1];
      g.add(j, om * dd / M[j]);
      g.add(n + j, om * dv / M[j]);
      g.add(2 * n + j, -(om * (K[j] * dd + C[j] * dv) / (M[j] * M[j])));
    }
    const double ph = CKO_TWO_PI * t / Tb;
    double s, c;
    sincos(ph, &s, &c);
    g.add(3 * n, w[n] * s);
    g.lane_add(3 * n + 1 + m.off + b, w[n] * fa * c * (-ph / Tb));
  }
};

// Chaboche viscoplasticity (models_chaboche.cpp:19-194).
struct MChaboche {
  template <class Y, class O>
  __device__ static void rate(const DevModel& m, double t, const Y& y, O& out, int b) {
    const int n = m.nu;
    const double* p = m.p;
    const double E = p[0], nn = p[1], eta = p[2], s0 = p[3], Kinf = p[4], tau = p[5];
    const double *C = p + 6, *gam = p + 6 + n;
    const double ea = p[6 + 2 * n + m.off + b], Tp = p[6 + 2 * n + m.nbm];
    const double sig = y[0], K = y[1];
    double s = sig;
    for (int i = 0; i < n; ++i) s -= y[2 + i];
    const double sg = sign_of(s);
    const double over = (fabs(s) - K - s0) / eta;
    const double ramp = pow_value(over > 0.0 ? over : 0.0, nn);
    const double ep = ramp * sg;
    const double ep_abs = ramp * (sg * sg);
    out[0] = xmul(E, xsub(xmul(ea, sin(CKO_TWO_PI * t / Tp)), ep));
    out[1] = tau * (Kinf - K);
    for (int i = 0; i < n; ++i)
      out[2 + i] = xsub(xmul(xmul(2.0 / 3.0, C[i]), ep), xmul(xmul(gam[i], y[2 + i]), ep_abs));
  }
  template <class Y, class J>
  __device__ static void jacobian(const DevModel& m, double, const Y& y, J& jac, int) {
    const int n = m.nu;
    const double* p = m.p;
    const double E = p[0], nn = p[1], eta = p[2], s0 = p[3], tau = p[5];
    const double *C = p + 6, *gam = p + 6 + n;
    const double sig = y[0], K = y[1];
    double s = sig;
    for (int i = 0; i < n; ++i) s -= y[2 + i];
    const double sg = sign_of(s), sg2 = sg * sg;
    const double over = (fabs(s) - K - s0) / eta;
    const double D = over > 0.0 ? nn * pow_value(over, nn - 1.0) / eta : 0.0;
    const double ramp = over > 0.0 ? pow_value(over, nn) : 0.0;
    jac(0, 0) = -E * D * sg2;
    jac(0, 1) = E * D * sg;
    for (int j = 0; j < n; ++j) jac(0, 2 + j) = E * D * sg2;
    jac(1, 0) = 0.0;
    jac(1, 1) = -tau;
    for (int j = 0; j < n; ++j) jac(1, 2 + j) = 0.0;
    for (int i = 0; i < n; ++i) {
      const double Xi = y[2 + i];
      const double ci = (2.0 / 3.0) * C[i];
      const double gX = xmul(gam[i], Xi);
      jac(2 + i, 0) = xsub(xmul(xmul(ci, D), sg2), xmul(xmul(gX, D), sg));
      jac(2 + i, 1) = xadd(xmul(xmul(-ci, D), sg), xmul(xmul(gX, D), sg2));
      const double v = xadd(xmul(xmul(-ci, D), sg2), xmul(xmul(gX, D), sg));
      for (int j = 0; j < n; ++j) jac(2 + i, 2 + j) = v;
      jac(2 + i, 2 + i) = xsub(v, xmul(xmul(gam[i], ramp), sg2));
    }
  }
  template <class Y, class Wt, class G>
  __device__ static void vjp(const DevModel& m, double t, const Y& y, const Wt& w, G& g, int b) {
    const int n = m.nu;
    const double* p = m.p;
    const double E = p[0], nn = p[1], eta = p[2], s0 = p[3], Kinf = p[4], tau = p[5];
    const double *C = p + 6, *gam = p + 6 + n;
    const int gb = m.off + b;
    const double eab = p[6 + 2 * n + gb];
    const double Tp = p[6 + 2 * n + m.nbm];
    const double two_pi_over_T = CKO_TWO_PI / Tp;
    const double sig = y[0], K = y[1];
    const double w_sig = w[0], w_K = w[1];
    double s = sig;
    for (int i = 0; i < n; ++i) s -= y[2 + i];
    const double sg = sign_of(s), sg2 = sg * sg;
    const double over = (fabs(s) - K - s0) / eta;
    const double phase = two_pi_over_T * t;
    double sinp, cosp;
    sincos(phase, &sinp, &cosp);
    g.add(4, w_K * tau);
    g.add(5, w_K * (Kinf - K));
    g.lane_add(6 + 2 * n + gb, w_sig * E * sinp);
    g.add(6 + 2 * n + m.nbm, w_sig * E * eab * cosp * (-phase / Tp));
    if (over > 0.0) {
      const double ramp = pow_value(over, nn);
      const double dramp = nn * pow_value(over, nn - 1.0);
      const double ep = ramp * sg, ep_abs = ramp * sg2;
      double S = -E * w_sig * sg;
      for (int i = 0; i < n; ++i) {
        const double Xi = y[2 + i], wx = w[2 + i];
        S += wx * ((2.0 / 3.0) * C[i] * sg - gam[i] * Xi * sg2);
        g.add(6 + i, wx * (2.0 / 3.0) * ep);
        g.add(6 + n + i, -(wx * Xi * ep_abs));
      }
      g.add(0, w_sig * (eab * sinp - ep));
      g.add(1, S * ramp * log(over));
      g.add(2, S * dramp * (-over / eta));
      g.add(3, S * dramp * (-1.0 / eta));
    } else {
      g.add(0, w_sig * eab * sinp);
    }
  }
};

// Neural ODE, hidden width W (models_node.cpp:13-205 is the W = n+1 case):
// params [W1 (W x (n+1)), b1, W2 (W x W), b2, W3 (n x W), b3]. The point-wise
// version here keeps its activations in a per-thread scratch of
// NODE_SCRATCH doubles (small widths); the wide case runs the batched-GEMM
// kernels in cko_node_wide.cuh.
constexpr int NODE_MAX_W = 128;
constexpr int NODE_MAX_N = 16;

struct MNode {
  __device__ static void forward(const DevModel& m, double t, const double* y, int b, double* z0,
                                 double* z1, double* z2, double* o) {
    const int n = m.n, W = m.W, w0 = n + 1;
    const double* W1 = m.p;
    const double* b1 = W1 + W * w0;
    const double* W2 = b1 + W;
    const double* b2 = W2 + W * W;
    const double* W3 = b2 + W;
    const double* b3 = W3 + n * W;
    for (int i = 0; i < n; ++i) z0[i] = y[i];
    z0[n] = sin(CKO_TWO_PI * t / m.periods[m.off + b]);
    for (int i = 0; i < W; ++i) {
      double acc = b1[i];
      for (int j = 0; j < w0; ++j) acc = xadd(acc, xmul(W1[i * w0 + j], z0[j]));
      z1[i] = tanh(acc);
    }
    for (int i = 0; i < W; ++i) {
      double acc = b2[i];
      for (int j = 0; j < W; ++j) acc = xadd(acc, xmul(W2[i * W + j], z1[j]));
      z2[i] = tanh(acc);
    }
    for (int i = 0; i < n; ++i) {
      double acc = b3[i];
      for (int j = 0; j < W; ++j) acc = xadd(acc, xmul(W3[i * W + j], z2[j]));
      o[i] = tanh(acc);
    }
  }
  template <class Y, class O>
  __device__ static void rate(const DevModel& m, double t, const Y& y, O& out, int b) {
    double yl[NODE_MAX_N], z0[NODE_MAX_N + 1], z1[NODE_MAX_W], z2[NODE_MAX_W], o[NODE_MAX_N];
    for (int i = 0; i < m.n; ++i) yl[i] = y[i];
    forward(m, t, yl, b, z0, z1, z2, o);
    for (int i = 0; i < m.n; ++i) out[i] = o[i];
  }
  // J = diag(1 - o^2) W3 diag(1 - z2^2) W2 diag(1 - z1^2) W1[:, :n], one
  // column at a time so only two width-W vectors are live (models_node.cpp:69-107).
  template <class Y, class J>
  __device__ static void jacobian(const DevModel& m, double t, const Y& y, J& jac, int b) {
    const int n = m.n, W = m.W, w0 = n + 1;
    double yl[NODE_MAX_N], z0[NODE_MAX_N + 1], z1[NODE_MAX_W], z2[NODE_MAX_W], o[NODE_MAX_N];
    for (int i = 0; i < n; ++i) yl[i] = y[i];
    forward(m, t, yl, b, z0, z1, z2, o);
    const double* W1 = m.p;
    const double* W2 = W1 + W * w0 + W;
    const double* W3 = W2 + W * W + W;
    for (int j = 0; j < n; ++j) {
      double m1[NODE_MAX_W], m2[NODE_MAX_W];
      for (int i = 0; i < W; ++i) m1[i] = (1.0 - z1[i] * z1[i]) * W1[i * w0 + j];
      for (int i = 0; i < W; ++i) {
        double acc = 0.0;
        for (int l = 0; l < W; ++l) acc += W2[i * W + l] * m1[l];
        m2[i] = (1.0 - z2[i] * z2[i]) * acc;
      }
      for (int i = 0; i < n; ++i) {
        double acc = 0.0;
        for (int l = 0; l < W; ++l) acc += W3[i * W + l] * m2[l];
        jac(i, j) = (1.0 - o[i] * o[i]) * acc;
      }
    }
  }
  template <class Y, class Wt, class G>
  __device__ static void vjp(const DevModel& m, double t, const Y& y, const Wt& w, G& g, int b) {
    const int n = m.n, W = m.W, w0 = n + 1;
    double yl[NODE_MAX_N], z0[NODE_MAX_N + 1], z1[NODE_MAX_W], z2[NODE_MAX_W], o[NODE_MAX_N];
    double d3[NODE_MAX_N], d2[NODE_MAX_W];
    for (int i = 0; i < n; ++i) yl[i] = y[i];
    forward(m, t, yl, b, z0, z1, z2, o);
    const double* W2 = m.p + W * w0 + W;
    const double* W3 = W2 + W * W + W;
    const int ob1 = W * w0, oW2 = ob1 + W, ob2 = oW2 + W * W, oW3 = ob2 + W, ob3 = oW3 + n * W;
    for (int i = 0; i < n; ++i) d3[i] = w[i] * (1.0 - o[i] * o[i]);
    for (int i = 0; i < W; ++i) {
      double acc = 0.0;
      for (int l = 0; l < n; ++l) acc += W3[l * W + i] * d3[l];
      d2[i] = acc * (1.0 - z2[i] * z2[i]);
    }
    for (int i = 0; i < n; ++i) {
      for (int j = 0; j < W; ++j) g.add(oW3 + i * W + j, d3[i] * z2[j]);
      g.add(ob3 + i, d3[i]);
    }
    for (int i = 0; i < W; ++i) {
      for (int j = 0; j < W; ++j) g.add(oW2 + i * W + j, d2[i] * z1[j]);
      g.add(ob2 + i, d2[i]);
    }
    for (int i = 0; i < W; ++i) {
      double acc = 0.0;
      for (int l = 0; l < W; ++l) acc += W2[l * W + i] * d2[l];
      const double d1 = acc * (1.0 - z1[i] * z1[i]);
      for (int j = 0; j < w0; ++j) g.add(i * w0 + j, d1 * z0[j]);
      g.add(ob1 + i, d1);
    }
  }
};

}  // namespace cko
