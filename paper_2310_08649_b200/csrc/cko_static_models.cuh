// cko_static_models.cuh — compile-time-sized device twins of the reference
// models for the v2 (warp-specialised) kernels.
//
// The v1 twins in cko_models.cuh loop over runtime sizes, which forces
// per-thread arrays into local memory. These versions fix the state size N at
// compile time so every state vector and Jacobian row lives in registers:
//   load_consts(m, cs)          per-CTA constants into shared memory once
//                               (e.g. the MDS ratios K_u / M_u, bit-identical
//                               to the reference's per-call division)
//   rate(m, cs, t, y, h, b)     h(y, t)           (OdeModel::rate)
//   jac_row(m, cs, t, y, i, r, b)  row i of dh/dy  (jacobian_analytic)
// Expression order follows the reference sources cited per model.
#pragma once

#include "cko_models.cuh"

namespace cko {
namespace v2 {

// Mass-damper-spring chain, n_unit = NU (models_mds.cpp:27-82).
// Parameter layout [K(NU), C(NU), M(NU), f_a, T(nb)] (models_mds.cpp:14-15).
template <int NU>
struct MdsS {
  static constexpr int N = 2 * NU;
  // The Jacobian depends on neither the state, the time nor the lane
  // (models_mds.cpp:54-82: entries are parameter ratios), so the kernels keep
  // it in shared memory: J (row-major), J^T, and two shifted copies of a unit
  // vector whose slices are the rows of I written as 1 / -0.0 (adding -0.0
  // leaves every off-diagonal product bit-identical).
  static constexpr bool kConstJac = true;
  // M = I - dt J in 2 x 2 blocks: identity, one / three diagonals, tridiagonal (cko_sparse.cuh)
  static constexpr bool kArrowTri = true;
  static constexpr int JOFF = ((2 * NU + 1) + 1) / 2 * 2;
  static constexpr int JTOFF = JOFF + N * N;
  static constexpr int ZOFF = JTOFF + N * N;
  static constexpr int NCONST = ZOFF + 4 * N;
  // cs[u] = K_u / M_u, cs[NU + u] = C_u / M_u, cs[2 NU] = f_a, then J, J^T, Z
  __device__ static void load_consts(const DevModel& m, double* cs) {
    for (int u = threadIdx.x; u < NU; u += blockDim.x) {
      cs[u] = m.p[u] / m.p[2 * NU + u];
      cs[NU + u] = m.p[NU + u] / m.p[2 * NU + u];
    }
    if (threadIdx.x == 0) cs[2 * NU] = m.p[3 * NU];
    __syncthreads();
    for (int e = threadIdx.x; e < N * N; e += blockDim.x) {
      const int i = e / N, j = e % N;
      double row[N], y[N] = {};
      jac_row(m, cs, 0.0, y, i, row, 0);
      double v = 0.0;
#pragma unroll
      for (int q = 0; q < N; ++q) v = q == j ? row[q] : v;
      cs[JOFF + e] = v;
      cs[JTOFF + j * N + i] = v;
    }
    for (int e = threadIdx.x; e < 4 * N; e += blockDim.x)
      cs[ZOFF + e] = (e == N - 1 || e == 2 * N + N) ? 1.0 : -0.0;
  }
  // (J^T lambda)_i over the structural nonzeros of column i of J (jac_row's entries), ascending j: the
  // dense j-ascending multiply-add over all N entries adds only exact zeros besides these.
  __device__ static double jt_lambda(const double* cs, int i, const double* lm) {
    // branch-free (the lanes of a group hold different columns): absent neighbours add exact zeros
    const bool vel = i >= NU;
    const int k = vel ? i - NU : i;
    const double* c = cs + (vel ? NU : 0);
    const double lo = k > 0 ? -c[k] : 0.0, hi = k + 1 < NU ? -c[k + 1] : 0.0;
    const double mid = (0.0 + (k > 0 ? c[k] : 0.0)) + (k + 1 < NU ? c[k + 1] : 0.0);
    double tmp = 0.0;
    if (vel) tmp += 1.0 * lm[k];
    tmp += lo * lm[NU + (k > 0 ? k - 1 : 0)];
    tmp += mid * lm[NU + k];
    tmp += hi * lm[NU + (k + 1 < NU ? k + 1 : k)];
    return tmp;
  }
  // row i of I (1 on the diagonal, -0.0 elsewhere), 16-byte aligned
  __device__ static const double* unit_row(const double* cs, int i) {
    const int s = N - 1 - i;
    return cs + ZOFF + ((s & 1) ? 2 * N + s + 1 : s);
  }
  __device__ static void rate(const DevModel& m, const double* cs, double t, const double (&y)[N], double (&h)[N],
                              int b) {
    const double Tb = m.p[3 * NU + 1 + m.off + b];
#pragma unroll
    for (int u = 0; u < NU; ++u) h[u] = y[NU + u];
#pragma unroll
    for (int u = 0; u < NU; ++u) {
      // no contraction: the reference's separately rounded products and sums
      double acc = 0.0;
      if (u > 0)
        acc = xadd(acc, xadd(xmul(cs[u], y[u] - y[u - 1]), xmul(cs[NU + u], y[NU + u] - y[NU + u - 1])));
      if (u + 1 < NU)
        acc = xsub(acc, xadd(xmul(cs[u + 1], y[u + 1] - y[u]), xmul(cs[NU + u + 1], y[NU + u + 1] - y[NU + u])));
      if (u == 0) acc = xadd(acc, xmul(cs[2 * NU], sin(CKO_TWO_PI * t / Tb)));
      h[NU + u] = acc;
    }
  }
  // Rows of M = I - dt J (ndt = -dt) when the row kind is known: slot 0 is the
  // position row u (J row = e_{NU+u}), slot 1 the velocity row NU + u — the
  // v2 group layout with 10-lane groups holds exactly these. Same roundings
  // as xadd(xmul(ndt, J_ij), [i == j]) on jac_row's entries.
  static constexpr bool kSlotRows = true;
  __device__ static void m_row_slot(const double* cs, int slot, int u, double ndt, double (&m)[N]) {
    const double z = xmul(ndt, 0.0);
    if (slot == 0) {
#pragma unroll
      for (int j = 0; j < NU; ++j) {
        m[j] = j == u ? xadd(z, 1.0) : z;
        m[NU + j] = j == u ? xmul(ndt, 1.0) : z;
      }
    } else {
      const double am = u > 0 ? cs[u] : 0.0, cm = u > 0 ? cs[NU + u] : 0.0;
      const double ap = u + 1 < NU ? cs[u + 1] : 0.0, cp = u + 1 < NU ? cs[NU + u + 1] : 0.0;
      const double a0 = (0.0 + am) + ap, c0 = (0.0 + cm) + cp;
      const double ka = xmul(ndt, a0), km = xmul(ndt, -am), kp = xmul(ndt, -ap);
      const double ca = xadd(xmul(ndt, c0), 1.0), cmv = xmul(ndt, -cm), cpv = xmul(ndt, -cp);
#pragma unroll
      for (int j = 0; j < NU; ++j) {
        m[j] = j == u ? ka : (j + 1 == u ? km : (j == u + 1 ? kp : z));
        m[NU + j] = j == u ? ca : (j + 1 == u ? cmv : (j == u + 1 ? cpv : z));
      }
    }
  }
  // Row i of the analytic Jacobian (models_mds.cpp:54-82); the state does not
  // enter. Written as per-entry selects so the row stays in registers.
  __device__ static void jac_row(const DevModel&, const double* cs, double, const double (&)[N], int i,
                                 double (&row)[N], int) {
    const bool vel = i >= NU;
    const int u = vel ? i - NU : -8;
    const double am = (vel && u > 0) ? cs[u] : 0.0, cm = (vel && u > 0) ? cs[NU + u] : 0.0;
    const double ap = (vel && u + 1 < NU) ? cs[u + 1] : 0.0, cp = (vel && u + 1 < NU) ? cs[NU + u + 1] : 0.0;
    // out += a (u > 0 term first, then the u + 1 term), as the reference accumulates
    const double a0 = (0.0 + am) + ap, c0 = (0.0 + cm) + cp;
#pragma unroll
    for (int j = 0; j < NU; ++j) {
      row[j] = j == u ? a0 : (j + 1 == u ? -am : (j == u + 1 ? -ap : 0.0));
      row[NU + j] = !vel ? (j == i ? 1.0 : 0.0) : (j == u ? c0 : (j + 1 == u ? -cm : (j == u + 1 ? -cp : 0.0)));
    }
  }
};

// 3-state linear stiff ODE, config C1 (oracle/src/ref_models.hpp Lin3).
struct Lin3S {
  static constexpr int N = 3;
  static constexpr int NCONST = 10;
  __device__ static void load_consts(const DevModel& m, double* cs) {
    for (int i = threadIdx.x; i < 10; i += blockDim.x) cs[i] = m.p[i];
  }
  __device__ static void rate(const DevModel& m, const double* cs, double t, const double (&y)[N], double (&h)[N],
                              int b) {
#pragma unroll
    for (int i = 0; i < 3; ++i) {
      double acc = xmul(cs[3 * i], y[0]);
      acc = xadd(acc, xmul(cs[3 * i + 1], y[1]));
      acc = xadd(acc, xmul(cs[3 * i + 2], y[2]));
      if (i == 0) acc = xadd(acc, xmul(cs[9], sin(CKO_TWO_PI * t / m.periods[m.off + b])));
      h[i] = acc;
    }
  }
  __device__ static void jac_row(const DevModel&, const double* cs, double, const double (&)[N], int i,
                                 double (&row)[N], int) {
#pragma unroll
    for (int j = 0; j < 3; ++j) row[j] = cs[3 * i + j];
  }
};

// Chaboche viscoplasticity with NU backstresses (models_chaboche.cpp:30-62,
// 137-181). Constants: [E, n, eta, s0, Kinf, tau, C(NU), gamma(NU), T].
template <int NU>
struct ChabS {
  static constexpr int N = 2 + NU;
  static constexpr int NCONST = 7 + 2 * NU;
  __device__ static void load_consts(const DevModel& m, double* cs) {
    for (int i = threadIdx.x; i < 6 + 2 * NU; i += blockDim.x) cs[i] = m.p[i];
    if (threadIdx.x == 0) cs[6 + 2 * NU] = m.p[6 + 2 * NU + m.nbm];
  }
  __device__ static void rate(const DevModel& m, const double* cs, double t, const double (&y)[N], double (&h)[N],
                              int b) {
    const double E = cs[0], nn = cs[1], eta = cs[2], s0 = cs[3], Kinf = cs[4], tau = cs[5];
    const double* C = cs + 6;
    const double* gam = cs + 6 + NU;
    const double ea = m.p[6 + 2 * NU + m.off + b], Tp = cs[6 + 2 * NU];
    const double sig = y[0], K = y[1];
    double s = sig;
#pragma unroll
    for (int i = 0; i < NU; ++i) s -= y[2 + i];
    const double sg = sign_of(s);
    const double over = (fabs(s) - K - s0) / eta;
    const double ramp = pow_value(over > 0.0 ? over : 0.0, nn);
    const double ep = ramp * sg;
    const double ep_abs = ramp * (sg * sg);
    h[0] = xmul(E, xsub(xmul(ea, sin(CKO_TWO_PI * t / Tp)), ep));
    h[1] = tau * (Kinf - K);
#pragma unroll
    for (int i = 0; i < NU; ++i) h[2 + i] = xsub(xmul(xmul(2.0 / 3.0, C[i]), ep), xmul(xmul(gam[i], y[2 + i]), ep_abs));
  }
  __device__ static void jac_row(const DevModel&, const double* cs, double, const double (&y)[N], int i,
                                 double (&row)[N], int) {
    const double E = cs[0], nn = cs[1], eta = cs[2], s0 = cs[3], tau = cs[5];
    const double* C = cs + 6;
    const double* gam = cs + 6 + NU;
    const double sig = y[0], K = y[1];
    double s = sig;
#pragma unroll
    for (int q = 0; q < NU; ++q) s -= y[2 + q];
    const double sg = sign_of(s), sg2 = sg * sg;
    const double over = (fabs(s) - K - s0) / eta;
    const double D = over > 0.0 ? nn * pow_value(over, nn - 1.0) / eta : 0.0;
    const double ramp = over > 0.0 ? pow_value(over, nn) : 0.0;
    if (i == 0) {
      row[0] = -E * D * sg2;
      row[1] = E * D * sg;
#pragma unroll
      for (int j = 0; j < NU; ++j) row[2 + j] = E * D * sg2;
    } else if (i == 1) {
#pragma unroll
      for (int j = 0; j < N; ++j) row[j] = 0.0;
      row[1] = -tau;
    } else {
      // row 2 + q: runtime q, static register destinations
      double ci = 0.0, gi = 0.0, Xi = 0.0;
#pragma unroll
      for (int q = 0; q < NU; ++q)
        if (i == 2 + q) ci = (2.0 / 3.0) * C[q], gi = gam[q], Xi = y[2 + q];
      const double gX = xmul(gi, Xi);
      row[0] = xsub(xmul(xmul(ci, D), sg2), xmul(xmul(gX, D), sg));
      row[1] = xadd(xmul(xmul(-ci, D), sg), xmul(xmul(gX, D), sg2));
      const double v = xadd(xmul(xmul(-ci, D), sg2), xmul(xmul(gX, D), sg));
#pragma unroll
      for (int j = 0; j < NU; ++j) row[2 + j] = (i == 2 + j) ? xsub(v, xmul(xmul(gi, ramp), sg2)) : v;
    }
  }
};

struct ScalarDecayS {
  static constexpr int N = 1;
  static constexpr int NCONST = 1;
  __device__ static void load_consts(const DevModel& m, double* cs) {
    if (threadIdx.x == 0) cs[0] = m.p[0];
  }
  __device__ static void rate(const DevModel&, const double* cs, double, const double (&y)[1], double (&h)[1], int) {
    h[0] = -cs[0] * y[0];
  }
  __device__ static void jac_row(const DevModel&, const double* cs, double, const double (&)[1], int, double (&row)[1],
                                 int) {
    row[0] = -cs[0];
  }
};

struct ConstantRateS {
  static constexpr int N = 1;
  static constexpr int NCONST = 1;
  __device__ static void load_consts(const DevModel& m, double* cs) {
    if (threadIdx.x == 0) cs[0] = m.p[0];
  }
  __device__ static void rate(const DevModel&, const double* cs, double, const double (&)[1], double (&h)[1], int) {
    h[0] = cs[0];
  }
  __device__ static void jac_row(const DevModel&, const double*, double, const double (&)[1], int, double (&row)[1],
                                 int) {
    row[0] = 0.0;
  }
};

}  // namespace v2
}  // namespace cko
