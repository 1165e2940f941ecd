/*
 * cko_oracle.c — CPU restatement (plain C11) of the reference chunked
 * backward-Euler path: models, block LU, Thomas / PCR / hybrid block-
 * bidiagonal solves, the Newton chunk loop and the discrete adjoint.
 *
 * TEST INFRASTRUCTURE ONLY (see cko_oracle.h). Every function cites the
 * reference file:line it restates; paths are relative to
 * /root/reference/proj/core. Loop orders and rounding-relevant expression
 * orders follow the reference so results agree to roundoff; the one
 * deliberate difference is the mass-damper-spring parameter product, which
 * the reference forms by Dual8 forward sweeps (ode_model.hpp:154-182) and
 * this file forms analytically; the golden fixtures
 * pin the two to <= 1e-12.
 */
#define _POSIX_C_SOURCE 200809L
#include "cko_oracle.h"

#include <math.h>
#include <pthread.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>
#include <time.h>

#define TWO_PI (2.0 * 3.14159265358979323846)

/* ------------------------------------------------------------------------ */
/* errors                                                                    */
/* ------------------------------------------------------------------------ */

static int set_err(cko_error* e, int code, const char* msg) {
  if (e) {
    memset(e, 0, sizeof(*e));
    e->code = code;
    snprintf(e->msg, sizeof e->msg, "%s", msg);
  }
  return code;
}

static int err_singular(cko_error* e, int k, int b) {
  if (e) {
    memset(e, 0, sizeof(*e));
    e->code = CKO_SINGULAR_BLOCK;
    e->chunk_index = k;
    e->batch_index = b;
    snprintf(e->msg, sizeof e->msg, "singular diagonal block at chunk row %d, batch %d", k, b);
  }
  return CKO_SINGULAR_BLOCK;
}

static int err_divergence(cko_error* e, int start, int b, int it, double rn, double r0) {
  if (e) {
    memset(e, 0, sizeof(*e));
    e->code = CKO_NEWTON_DIVERGENCE;
    e->chunk_start_step = start;
    e->batch_index = b;
    e->iterations = it;
    e->residual_norm = rn;
    e->initial_norm = r0;
    snprintf(e->msg, sizeof e->msg,
             "Newton did not converge for chunk starting at step %d (batch %d): |r| = %g after "
             "%d iterations, |r0| = %g",
             start, b, rn, it, r0);
  }
  return CKO_NEWTON_DIVERGENCE;
}

/* ------------------------------------------------------------------------ */
/* models (models_*.cpp); local lane b maps to global lane lane_offset + b   */
/* ------------------------------------------------------------------------ */

typedef struct {
  int kind, n, nu, W, nbm, off;
  const double* p;
  int np;
} model_t;

/* linspace (linalg.cpp:386-396) */
static double linspace_at(double lo, double hi, int n, int i) {
  if (n <= 1) return lo;
  if (i == n - 1) return hi;
  return lo + (hi - lo) * (double)i / (double)(n - 1);
}

static int state_size_of(const cko_model_desc* d) {
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

static int param_count_of(const cko_model_desc* d) {
  const int u = d->n_unit, W = d->width, nb = d->n_batch_model;
  switch (d->kind) {
    case CKO_MODEL_SCALAR_DECAY:
    case CKO_MODEL_CONSTANT_RATE: return 1;
    case CKO_MODEL_LIN3: return 10;
    case CKO_MODEL_MDS: return 3 * u + 1 + nb;
    case CKO_MODEL_CHABOCHE: return 6 + 2 * u + nb + 1;
    case CKO_MODEL_NODE: return W * (u + 1) + W + W * W + W + u * W + u;
  }
  return -1;
}

static int model_init(model_t* m, const cko_model_desc* d, cko_error* e) {
  memset(m, 0, sizeof *m);
  m->kind = d->kind;
  m->n = state_size_of(d);
  m->nu = d->n_unit;
  m->W = d->width;
  m->nbm = d->n_batch_model;
  m->off = d->lane_offset;
  m->p = d->params;
  m->np = d->n_params;
  if (m->n < 1) return set_err(e, CKO_STRATEGY_UNAVAILABLE, "oracle: unknown model kind");
  if (param_count_of(d) != d->n_params)
    return set_err(e, CKO_SHAPE_MISMATCH, "oracle: parameter count does not match the model");
  return 0;
}

static double sign_of(double x) { return x > 0.0 ? 1.0 : (x < 0.0 ? -1.0 : 0.0); }

/* pow_value (dual.hpp:141-157) */
static double pow_value(double x, double n) {
  const int ni = (int)n;
  if ((double)ni == n && ni >= 0 && ni <= 32) {
    double r = 1.0, base = x;
    int e = ni;
    while (e > 0) {
      if (e & 1) r *= base;
      base *= base;
      e >>= 1;
    }
    return r;
  }
  return pow(x, n);
}

/* NODE forward pass (models_node.cpp:153-181, generalised to hidden width W
 * with input width n+1; the reference is the W = n+1 case). */
static void node_forward(const model_t* m, double t, const double* y, int gb, double* z0, double* z1,
                         double* z2, double* o) {
  const int n = m->n, W = m->W, w0 = n + 1;
  const double* W1 = m->p;
  const double* b1 = W1 + (size_t)W * w0;
  const double* W2 = b1 + W;
  const double* b2 = W2 + (size_t)W * W;
  const double* W3 = b2 + W;
  const double* b3 = W3 + (size_t)n * W;
  for (int i = 0; i < n; ++i) z0[i] = y[i];
  z0[n] = 1.0 * sin(TWO_PI * t / linspace_at(1e-2, 1.0, m->nbm, gb));
  for (int i = 0; i < W; ++i) {
    double acc = b1[i];
    for (int j = 0; j < w0; ++j) acc += W1[(size_t)i * w0 + j] * z0[j];
    z1[i] = tanh(acc);
  }
  for (int i = 0; i < W; ++i) {
    double acc = b2[i];
    for (int j = 0; j < W; ++j) acc += W2[(size_t)i * W + j] * z1[j];
    z2[i] = tanh(acc);
  }
  for (int i = 0; i < n; ++i) {
    double acc = b3[i];
    for (int j = 0; j < W; ++j) acc += W3[(size_t)i * W + j] * z2[j];
    o[i] = tanh(acc);
  }
}

/* h(y, t) at one point (ModelBase::rate -> Derived::eval_point,
 * ode_model.hpp:119-128). */
static void point_rate(const model_t* m, double t, const double* y, double* out, int b,
                       double* scratch) {
  const int gb = m->off + b;
  const double* p = m->p;
  switch (m->kind) {
    case CKO_MODEL_SCALAR_DECAY: out[0] = -p[0] * y[0]; break;  /* models_simple.cpp:18-21 */
    case CKO_MODEL_CONSTANT_RATE: out[0] = p[0]; break;         /* models_simple.cpp:37-40 */
    case CKO_MODEL_LIN3: {                                       /* oracle/src/ref_models.hpp */
      for (int i = 0; i < 3; ++i) {
        double acc = p[3 * i] * y[0];
        acc += p[3 * i + 1] * y[1];
        acc += p[3 * i + 2] * y[2];
        if (i == 0) acc += p[9] * sin(TWO_PI * t / linspace_at(1e-2, 1.0, m->nbm, gb));
        out[i] = acc;
      }
      break;
    }
    case CKO_MODEL_MDS: { /* models_mds.cpp:27-51 */
      const int n = m->nu;
      const double *K = p, *C = p + n, *M = p + 2 * n;
      const double fa = p[3 * n], Tb = p[3 * n + 1 + gb];
      const double *d = y, *v = y + n;
      for (int u = 0; u < n; ++u) out[u] = v[u];
      for (int u = 0; u < n; ++u) {
        double acc = 0.0;
        if (u > 0) acc += (K[u] / M[u]) * (d[u] - d[u - 1]) + (C[u] / M[u]) * (v[u] - v[u - 1]);
        if (u + 1 < n)
          acc -= (K[u + 1] / M[u + 1]) * (d[u + 1] - d[u]) + (C[u + 1] / M[u + 1]) * (v[u + 1] - v[u]);
        if (u == 0) acc += fa * sin(TWO_PI * t / Tb);
        out[n + u] = acc;
      }
      break;
    }
    case CKO_MODEL_CHABOCHE: { /* models_chaboche.cpp:30-62 */
      const int n = m->nu;
      const double E = p[0], nn = p[1], eta = p[2], s0 = p[3], Kinf = p[4], tau = p[5];
      const double *C = p + 6, *gam = p + 6 + n;
      const double ea = p[6 + 2 * n + gb], Tp = p[6 + 2 * n + m->nbm];
      const double sig = y[0], K = y[1];
      const double* X = y + 2;
      double s = sig;
      for (int i = 0; i < n; ++i) s -= X[i];
      const double sg = sign_of(s);
      const double over = (fabs(s) - K - s0) / eta;
      const double ramp = pow_value(over > 0.0 ? over : 0.0, nn);
      const double ep = ramp * sg;
      const double ep_abs = ramp * (sg * sg);
      out[0] = E * (ea * sin(TWO_PI * t / Tp) - ep);
      out[1] = tau * (Kinf - K);
      for (int i = 0; i < n; ++i) out[2 + i] = (2.0 / 3.0) * C[i] * ep - gam[i] * X[i] * ep_abs;
      break;
    }
    case CKO_MODEL_NODE: {
      const int n = m->n, W = m->W;
      double *z0 = scratch, *z1 = z0 + n + 1, *z2 = z1 + W;
      node_forward(m, t, y, gb, z0, z1, z2, out);
      break;
    }
  }
}

/* J = dh/dy at one point, row-major n x n, every entry written
 * (jacobian_analytic of each model). */
static void point_jacobian(const model_t* m, double t, const double* y, double* J, int b,
                           double* scratch) {
  const int nsz = m->n, gb = m->off + b;
  const double* p = m->p;
  switch (m->kind) {
    case CKO_MODEL_SCALAR_DECAY: J[0] = -p[0]; break; /* models_simple.cpp:23-27 */
    case CKO_MODEL_CONSTANT_RATE: J[0] = 0.0; break;  /* models_simple.cpp:42-45 */
    case CKO_MODEL_LIN3:
      for (int i = 0; i < 9; ++i) J[i] = p[i];
      break;
    case CKO_MODEL_MDS: { /* models_mds.cpp:53-82 */
      const int n = m->nu;
      const double *K = p, *C = p + n, *M = p + 2 * n;
      for (int i = 0; i < nsz * nsz; ++i) J[i] = 0.0;
      for (int u = 0; u < n; ++u) {
        J[(size_t)u * nsz + n + u] = 1.0;
        if (u > 0) {
          const double a = K[u] / M[u], c = C[u] / M[u];
          J[(size_t)(n + u) * nsz + u] += a;
          J[(size_t)(n + u) * nsz + u - 1] -= a;
          J[(size_t)(n + u) * nsz + n + u] += c;
          J[(size_t)(n + u) * nsz + n + u - 1] -= c;
        }
        if (u + 1 < n) {
          const double a = K[u + 1] / M[u + 1], c = C[u + 1] / M[u + 1];
          J[(size_t)(n + u) * nsz + u] += a;
          J[(size_t)(n + u) * nsz + u + 1] -= a;
          J[(size_t)(n + u) * nsz + n + u] += c;
          J[(size_t)(n + u) * nsz + n + u + 1] -= c;
        }
      }
      break;
    }
    case CKO_MODEL_CHABOCHE: { /* models_chaboche.cpp:137-181 */
      const int n = m->nu;
      const double E = p[0], nn = p[1], eta = p[2], s0 = p[3], tau = p[5];
      const double *C = p + 6, *gam = p + 6 + n;
      for (int i = 0; i < nsz * nsz; ++i) J[i] = 0.0;
      const double sig = y[0], K = y[1];
      double s = sig;
      for (int i = 0; i < n; ++i) s -= y[2 + i];
      const double sg = sign_of(s), sg2 = sg * sg;
      const double over = (fabs(s) - K - s0) / eta;
      const double D = over > 0.0 ? nn * pow_value(over, nn - 1.0) / eta : 0.0;
      const double ramp = over > 0.0 ? pow_value(over, nn) : 0.0;
      J[0] = -E * D * sg2;
      J[1] = E * D * sg;
      for (int j = 0; j < n; ++j) J[2 + j] = E * D * sg2;
      J[(size_t)1 * nsz + 1] = -tau;
      for (int i = 0; i < n; ++i) {
        const double Xi = y[2 + i];
        const double ci = (2.0 / 3.0) * C[i];
        double* row = J + (size_t)(2 + i) * nsz;
        row[0] = ci * D * sg2 - gam[i] * Xi * D * sg;
        row[1] = -ci * D * sg + gam[i] * Xi * D * sg2;
        for (int j = 0; j < n; ++j) row[2 + j] = -ci * D * sg2 + gam[i] * Xi * D * sg;
        row[2 + i] -= gam[i] * ramp * sg2;
      }
      break;
    }
    case CKO_MODEL_NODE: { /* models_node.cpp:69-107 */
      const int n = m->n, W = m->W, w0 = n + 1;
      double *z0 = scratch, *z1 = z0 + w0, *z2 = z1 + W, *o = z2 + W, *M1 = o + n, *M2 = M1 + (size_t)W * n;
      const double* W1 = p;
      const double* W2 = p + (size_t)W * w0 + W;
      const double* W3 = W2 + (size_t)W * W + W;
      node_forward(m, t, y, gb, z0, z1, z2, o);
      for (int i = 0; i < W; ++i) {
        const double g = 1.0 - z1[i] * z1[i];
        for (int j = 0; j < n; ++j) M1[(size_t)i * n + j] = g * W1[(size_t)i * w0 + j];
      }
      for (int i = 0; i < W; ++i) {
        const double g = 1.0 - z2[i] * z2[i];
        for (int j = 0; j < n; ++j) {
          double acc = 0.0;
          for (int l = 0; l < W; ++l) acc += W2[(size_t)i * W + l] * M1[(size_t)l * n + j];
          M2[(size_t)i * n + j] = g * acc;
        }
      }
      for (int i = 0; i < n; ++i) {
        const double g = 1.0 - o[i] * o[i];
        for (int j = 0; j < n; ++j) {
          double acc = 0.0;
          for (int l = 0; l < W; ++l) acc += W3[(size_t)i * W + l] * M2[(size_t)l * n + j];
          J[(size_t)i * n + j] = g * acc;
        }
      }
      break;
    }
  }
}

/* grad += w . dh/dp at one point (param_vjp_analytic; MDS by the closed
 * form of SURVEY Appendix A in place of the Dual8 sweep). */
static void point_vjp(const model_t* m, double t, const double* y, const double* w, double* grad,
                      int b, double* scratch) {
  const int gb = m->off + b;
  const double* p = m->p;
  switch (m->kind) {
    case CKO_MODEL_SCALAR_DECAY: grad[0] += w[0] * (-y[0]); break;
    case CKO_MODEL_CONSTANT_RATE: grad[0] += w[0]; break;
    case CKO_MODEL_LIN3: {
      for (int i = 0; i < 3; ++i)
        for (int j = 0; j < 3; ++j) grad[3 * i + j] += w[i] * y[j];
      grad[9] += w[0] * sin(TWO_PI * t / linspace_at(1e-2, 1.0, m->nbm, gb));
      break;
    }
    case CKO_MODEL_MDS: {
      const int n = m->nu;
      const double *K = p, *C = p + n, *M = p + 2 * n;
      const double fa = p[3 * n], Tb = p[3 * n + 1 + gb];
      const double *d = y, *v = y + n;
      for (int j = 1; j < n; ++j) {
        const double om = w[n + j] - w[n + j - 1];
        const double dd = d[j] - d[j - 1], dv = v[j] - v[j - 1];
        grad[j] += om * dd / M[j];
        grad[n + j] += om * dv / M[j];
        grad[2 * n + j] -= om * (K[j] * dd + C[j] * dv) / (M[j] * M[j]);
      }
      const double ph = TWO_PI * t / Tb;
      grad[3 * n] += w[n] * sin(ph);
      grad[3 * n + 1 + gb] += w[n] * fa * cos(ph) * (-ph / Tb);
      break;
    }
    case CKO_MODEL_CHABOCHE: { /* models_chaboche.cpp:72-135 */
      const int n = m->nu;
      const double E = p[0], nn = p[1], eta = p[2], s0 = p[3], Kinf = p[4], tau = p[5];
      const double *C = p + 6, *gam = p + 6 + n, *ea = p + 6 + 2 * n;
      const double Tp = p[6 + 2 * n + m->nbm];
      const double two_pi_over_T = TWO_PI / Tp;
      const double sig = y[0], K = y[1];
      const double* X = y + 2;
      const double w_sig = w[0], w_K = w[1];
      const double* w_X = w + 2;
      double s = sig;
      for (int i = 0; i < n; ++i) s -= X[i];
      const double sg = sign_of(s), sg2 = sg * sg;
      const double over = (fabs(s) - K - s0) / eta;
      const double phase = two_pi_over_T * t;
      const double sinp = sin(phase);
      grad[4] += w_K * tau;
      grad[5] += w_K * (Kinf - K);
      grad[6 + 2 * n + gb] += w_sig * E * sinp;
      grad[6 + 2 * n + m->nbm] += w_sig * E * ea[gb] * cos(phase) * (-phase / Tp);
      if (over > 0.0) {
        const double ramp = pow_value(over, nn);
        const double dramp = nn * pow_value(over, nn - 1.0);
        const double ep = ramp * sg, ep_abs = ramp * sg2;
        double S = -E * w_sig * sg;
        for (int i = 0; i < n; ++i) {
          S += w_X[i] * ((2.0 / 3.0) * C[i] * sg - gam[i] * X[i] * sg2);
          grad[6 + i] += w_X[i] * (2.0 / 3.0) * ep;
          grad[6 + n + i] -= w_X[i] * X[i] * ep_abs;
        }
        grad[0] += w_sig * (ea[gb] * sinp - ep);
        grad[1] += S * ramp * log(over);
        grad[2] += S * dramp * (-over / eta);
        grad[3] += S * dramp * (-1.0 / eta);
      } else {
        grad[0] += w_sig * ea[gb] * sinp;
      }
      break;
    }
    case CKO_MODEL_NODE: { /* models_node.cpp:109-151 */
      const int n = m->n, W = m->W, w0 = n + 1;
      double *z0 = scratch, *z1 = z0 + w0, *z2 = z1 + W, *o = z2 + W, *d3 = o + n, *d2 = d3 + n, *d1 = d2 + W;
      const double* W2 = p + (size_t)W * w0 + W;
      const double* W3 = W2 + (size_t)W * W + W;
      const size_t ob1 = (size_t)W * w0, oW2 = ob1 + W, ob2 = oW2 + (size_t)W * W;
      const size_t oW3 = ob2 + W, ob3 = oW3 + (size_t)n * W;
      node_forward(m, t, y, gb, z0, z1, z2, o);
      for (int i = 0; i < n; ++i) d3[i] = w[i] * (1.0 - o[i] * o[i]);
      for (int i = 0; i < W; ++i) {
        double acc = 0.0;
        for (int l = 0; l < n; ++l) acc += W3[(size_t)l * W + i] * d3[l];
        d2[i] = acc * (1.0 - z2[i] * z2[i]);
      }
      for (int i = 0; i < W; ++i) {
        double acc = 0.0;
        for (int l = 0; l < W; ++l) acc += W2[(size_t)l * W + i] * d2[l];
        d1[i] = acc * (1.0 - z1[i] * z1[i]);
      }
      for (int i = 0; i < n; ++i) {
        for (int j = 0; j < W; ++j) grad[oW3 + (size_t)i * W + j] += d3[i] * z2[j];
        grad[ob3 + i] += d3[i];
      }
      for (int i = 0; i < W; ++i) {
        for (int j = 0; j < W; ++j) grad[oW2 + (size_t)i * W + j] += d2[i] * z1[j];
        grad[ob2 + i] += d2[i];
      }
      for (int i = 0; i < W; ++i) {
        for (int j = 0; j < w0; ++j) grad[(size_t)i * w0 + j] += d1[i] * z0[j];
        grad[ob1 + i] += d1[i];
      }
      break;
    }
  }
}

static size_t scratch_len(const model_t* m) {
  return (size_t)4 * (m->n + 1) + (size_t)4 * m->W + (size_t)2 * m->W * m->n + 16;
}

/* ------------------------------------------------------------------------ */
/* block linear algebra (linalg.cpp)                                         */
/* ------------------------------------------------------------------------ */

/* lu_factor_block (linalg.cpp:13-44) */
static int lu_factor_block(double* a, int* piv, int n) {
  double scale = 0.0;
  for (int i = 0; i < n * n; ++i) {
    const double v = fabs(a[i]);
    scale = (scale < v) ? v : scale; /* std::max(scale, v) */
  }
  const double tiny = 1e-14 * scale;
  for (int c = 0; c < n; ++c) {
    int p = c;
    double best = fabs(a[(size_t)c * n + c]);
    for (int r = c + 1; r < n; ++r) {
      const double v = fabs(a[(size_t)r * n + c]);
      if (v > best) {
        best = v;
        p = r;
      }
    }
    piv[c] = p;
    if (best < tiny || best == 0.0) return 0;
    if (p != c)
      for (int j = 0; j < n; ++j) {
        const double t = a[(size_t)c * n + j];
        a[(size_t)c * n + j] = a[(size_t)p * n + j];
        a[(size_t)p * n + j] = t;
      }
    const double inv = 1.0 / a[(size_t)c * n + c];
    for (int r = c + 1; r < n; ++r) {
      const double l = a[(size_t)r * n + c] * inv;
      a[(size_t)r * n + c] = l;
      if (l != 0.0)
        for (int j = c + 1; j < n; ++j) a[(size_t)r * n + j] -= l * a[(size_t)c * n + j];
    }
  }
  return 1;
}

/* lu_solve_vec (linalg.cpp:46-60) */
static void lu_solve_vec(const double* lu, const int* piv, int n, double* y) {
  for (int i = 0; i < n; ++i)
    if (piv[i] != i) {
      const double t = y[i];
      y[i] = y[piv[i]];
      y[piv[i]] = t;
    }
  for (int i = 1; i < n; ++i) {
    double s = y[i];
    for (int j = 0; j < i; ++j) s -= lu[(size_t)i * n + j] * y[j];
    y[i] = s;
  }
  for (int i = n - 1; i >= 0; --i) {
    double s = y[i];
    for (int j = i + 1; j < n; ++j) s -= lu[(size_t)i * n + j] * y[j];
    y[i] = s / lu[(size_t)i * n + i];
  }
}

/* lu_right_solve_mat (linalg.cpp:62-82): X A = Y in place, Y m x n */
static void lu_right_solve_mat(const double* lu, const int* piv, int n, double* y, int m) {
  for (int r = 0; r < m; ++r) {
    double* w = y + (size_t)r * n;
    for (int i = 0; i < n; ++i) {
      double s = w[i];
      for (int j = 0; j < i; ++j) s -= lu[(size_t)j * n + i] * w[j];
      w[i] = s / lu[(size_t)i * n + i];
    }
    for (int i = n - 2; i >= 0; --i) {
      double s = w[i];
      for (int j = i + 1; j < n; ++j) s -= lu[(size_t)j * n + i] * w[j];
      w[i] = s;
    }
    for (int i = n - 1; i >= 0; --i)
      if (piv[i] != i) {
        const double t = w[i];
        w[i] = w[piv[i]];
        w[piv[i]] = t;
      }
  }
}

/* gemv_sub (linalg.cpp:101-108): y -= M x */
static void gemv_sub(const double* M, const double* x, double* y, int n) {
  for (int i = 0; i < n; ++i) {
    double s = 0.0;
    const double* row = M + (size_t)i * n;
    for (int j = 0; j < n; ++j) s += row[j] * x[j];
    y[i] -= s;
  }
}

/* gemm_neg (linalg.cpp:110-123): C = -(A B) */
static void gemm_neg(const double* A, const double* B, double* C, int n) {
  for (int i = 0; i < n; ++i) {
    double* crow = C + (size_t)i * n;
    for (int j = 0; j < n; ++j) crow[j] = 0.0;
    const double* arow = A + (size_t)i * n;
    for (int k = 0; k < n; ++k) {
      const double a = arow[k];
      if (a == 0.0) continue;
      const double* brow = B + (size_t)k * n;
      for (int j = 0; j < n; ++j) crow[j] -= a * brow[j];
    }
  }
}

typedef struct {
  int nc, nb, n;
  double* lu; /* (nc, nb, n, n) */
  int* piv;   /* (nc, nb, n) */
} fac_t;

static double* fblk(const fac_t* f, int k, int b) { return f->lu + ((size_t)k * f->nb + b) * f->n * f->n; }
static int* fpiv(const fac_t* f, int k, int b) { return f->piv + ((size_t)k * f->nb + b) * f->n; }

/* thomas_into (linalg.cpp:152-162); offd NULL = thomas_unit_into (:164-175) */
static void thomas_solve(const fac_t* f, const double* offd, double* x) {
  const int nc = f->nc, nb = f->nb, n = f->n;
  for (int b = 0; b < nb; ++b) lu_solve_vec(fblk(f, 0, b), fpiv(f, 0, b), n, x + (size_t)b * n);
  for (int k = 1; k < nc; ++k)
    for (int b = 0; b < nb; ++b) {
      double* cur = x + ((size_t)k * nb + b) * n;
      const double* prev = x + ((size_t)(k - 1) * nb + b) * n;
      if (offd)
        gemv_sub(offd + ((size_t)(k - 1) * nb + b) * n * n, prev, cur, n);
      else
        for (int i = 0; i < n; ++i) cur[i] += prev[i];
      lu_solve_vec(fblk(f, k, b), fpiv(f, k, b), n, cur);
    }
}

/* strided_solve_into (linalg.cpp:197-255) with partition_sizes (:126-133).
 * offd is scratch holding the couplings on entry (destroyed). */
static void strided_solve(const fac_t* f, double* offd, double* x, int n_switch, long long* sweeps) {
  const int nc = f->nc, nb = f->nb, n = f->n;
  double* pbuf = (double*)malloc(sizeof(double) * (size_t)n * n);
  int base = 0;
  for (int bit = 30; bit >= 0; --bit) {
    const int m = 1 << bit;
    if (!(nc & m)) continue;
    if (base > 0)
      for (int b = 0; b < nb; ++b)
        gemv_sub(offd + ((size_t)(base - 1) * nb + b) * n * n, x + ((size_t)(base - 1) * nb + b) * n,
                 x + ((size_t)base * nb + b) * n, n);
    int e = 0;
    while ((1 << e) < m) ++e;
    const int nsw = (n_switch < 0) ? e : (n_switch < e ? n_switch : e);
    for (int sidx = 0; sidx < nsw; ++sidx) {
      const int s = 1 << sidx;
      for (int r = base + m - 1; r >= base + s; --r) {
        const int q = r - s;
        for (int b = 0; b < nb; ++b) {
          double* Br = offd + ((size_t)(r - 1) * nb + b) * n * n;
          memcpy(pbuf, Br, sizeof(double) * (size_t)n * n);
          lu_right_solve_mat(fblk(f, q, b), fpiv(f, q, b), n, pbuf, n);
          gemv_sub(pbuf, x + ((size_t)q * nb + b) * n, x + ((size_t)r * nb + b) * n, n);
          if (q - base >= s) gemm_neg(pbuf, offd + ((size_t)(q - 1) * nb + b) * n * n, Br, n);
        }
      }
    }
    if (sweeps) *sweeps += nsw;
    const int stride = 1 << nsw;
    for (int c = 0; c < (stride < m ? stride : m); ++c)
      for (int b = 0; b < nb; ++b) {
        const int r0 = base + c;
        lu_solve_vec(fblk(f, r0, b), fpiv(f, r0, b), n, x + ((size_t)r0 * nb + b) * n);
        for (int r = r0 + stride; r < base + m; r += stride) {
          gemv_sub(offd + ((size_t)(r - 1) * nb + b) * n * n, x + ((size_t)(r - stride) * nb + b) * n,
                   x + ((size_t)r * nb + b) * n, n);
          lu_solve_vec(fblk(f, r, b), fpiv(f, r, b), n, x + ((size_t)r * nb + b) * n);
        }
      }
    base += m;
  }
  free(pbuf);
}

/* fill_minus_identity (linalg.cpp:261-266) */
static void fill_minus_identity(double* offd, int rows, int nb, int n) {
  memset(offd, 0, sizeof(double) * (size_t)rows * nb * n * n);
  for (size_t q = 0; q < (size_t)rows * nb; ++q)
    for (int i = 0; i < n; ++i) offd[q * n * n + (size_t)i * n + i] = -1.0;
}

/* detail::solve_unit_offdiag (linalg.cpp:288-303) */
static void solve_unit(const fac_t* f, double* scratch, double* x, const cko_solver_choice* s,
                       long long* sweeps) {
  if (s->kind == CKO_SOLVER_THOMAS) {
    thomas_solve(f, NULL, x);
    return;
  }
  if (f->nc > 1) fill_minus_identity(scratch, f->nc - 1, f->nb, f->n);
  strided_solve(f, scratch, x, s->kind == CKO_SOLVER_PCR ? -1 : s->n_switch, sweeps);
}

int cko_oracle_solve(const cko_solver_choice* solver, int nc, int nb, int n, const double* diag,
                     const double* offdiag, double* rhs, long long* sweeps, cko_error* err) {
  if (nc < 1 || nb < 1 || n < 1)
    return set_err(err, CKO_SHAPE_MISMATCH, "block bidiagonal system must be non-empty");
  if (solver->kind == CKO_SOLVER_HYBRID && solver->n_switch < 0)
    return set_err(err, CKO_ERROR, "solve_hybrid: n_switch must be >= 0");
  fac_t f = {nc, nb, n, NULL, NULL};
  f.lu = (double*)malloc(sizeof(double) * (size_t)nc * nb * n * n);
  f.piv = (int*)malloc(sizeof(int) * (size_t)nc * nb * n);
  memcpy(f.lu, diag, sizeof(double) * (size_t)nc * nb * n * n);
  int rc = 0;
  for (int k = 0; k < nc && !rc; ++k)
    for (int b = 0; b < nb; ++b)
      if (!lu_factor_block(fblk(&f, k, b), fpiv(&f, k, b), n)) {
        rc = err_singular(err, k, b);
        break;
      }
  if (!rc) {
    if (sweeps) *sweeps = 0;
    const size_t ob = (size_t)(nc > 1 ? nc - 1 : 0) * nb * n * n;
    double* scratch = (double*)malloc(sizeof(double) * (ob ? ob : 1));
    if (offdiag && ob) memcpy(scratch, offdiag, sizeof(double) * ob);
    if (!offdiag)
      solve_unit(&f, scratch, rhs, solver, sweeps);
    else if (solver->kind == CKO_SOLVER_THOMAS)
      thomas_solve(&f, offdiag, rhs);
    else
      strided_solve(&f, scratch, rhs, solver->kind == CKO_SOLVER_PCR ? -1 : solver->n_switch, sweeps);
    free(scratch);
  }
  free(f.lu);
  free(f.piv);
  if (!rc && err) set_err(err, CKO_OK, "");
  return rc;
}

/* ------------------------------------------------------------------------ */
/* forward integrator (integrate.cpp)                                        */
/* ------------------------------------------------------------------------ */

typedef struct {
  int c, nb, n;
  double *yy, *hr, *t, *dt, *ys, *r0, *rn, *offd, *scr;
  fac_t fac;
} nws_t;

/* rate_residual_norms (integrate.cpp:64-95) */
static void rate_residual_norms(const model_t* m, nws_t* w, double* norms) {
  const int c = w->c, nb = w->nb, n = w->n;
  for (int k = 0; k < c; ++k)
    for (int b = 0; b < nb; ++b)
      point_rate(m, w->t[(size_t)k * nb + b], w->yy + ((size_t)k * nb + b) * n,
                 w->hr + ((size_t)k * nb + b) * n, b, w->scr);
  for (int b = 0; b < nb; ++b) norms[b] = 0.0;
  for (int k = 0; k < c; ++k)
    for (int b = 0; b < nb; ++b) {
      const double dt = w->dt[(size_t)k * nb + b];
      const double* yk = w->yy + ((size_t)k * nb + b) * n;
      const double* ym = k == 0 ? w->ys + (size_t)b * n : w->yy + ((size_t)(k - 1) * nb + b) * n;
      double* out = w->hr + ((size_t)k * nb + b) * n;
      double s = 0.0;
      for (int i = 0; i < n; ++i) {
        const double v = yk[i] - ym[i] - out[i] * dt;
        out[i] = v;
        s += v * v;
      }
      norms[b] += s;
    }
  for (int b = 0; b < nb; ++b) norms[b] = sqrt(norms[b]);
}

/* worst_lane (integrate.cpp:167-174) */
static int worst_lane(const double* rn, int nb) {
  int w = 0;
  for (int b = 0; b < nb; ++b) {
    if (!isfinite(rn[b])) return b;
    if (rn[b] > rn[w]) w = b;
  }
  return w;
}

static int lanes_converged(const double* rn, const double* r0, int nb, const cko_newton_settings* st) {
  for (int b = 0; b < nb; ++b)
    if (!(rn[b] <= st->tol_a || rn[b] <= st->tol_r * r0[b])) return 0;
  return 1;
}

static int lanes_finite(const double* rn, int nb) {
  for (int b = 0; b < nb; ++b)
    if (!isfinite(rn[b])) return 0;
  return 1;
}

/* assemble I - J dt and LU one block (integrate.cpp:118-135, :213-221) */
static int assemble_factor_point(const model_t* m, nws_t* w, int k, int b) {
  const int n = w->n, nb = w->nb;
  double* blk = fblk(&w->fac, k, b);
  point_jacobian(m, w->t[(size_t)k * nb + b], w->yy + ((size_t)k * nb + b) * n, blk, b, w->scr);
  const double dt = w->dt[(size_t)k * nb + b];
  for (int i = 0; i < n * n; ++i) blk[i] = -dt * blk[i];
  for (int i = 0; i < n; ++i) blk[i * n + i] += 1.0;
  return lu_factor_block(blk, fpiv(&w->fac, k, b), n);
}

/* newton_chunk (integrate.cpp:192-255). Returns 0 or an error code;
 * *iters receives the iteration count. */
static int newton_chunk(const model_t* m, nws_t* w, const cko_newton_settings* st,
                        const cko_solver_choice* solver, cko_work* work, int start_step,
                        int* iters, cko_error* err) {
  const int c = w->c, nb = w->nb, n = w->n;
  rate_residual_norms(m, w, w->r0);
  if (work) ++work->rate_evals;
  memcpy(w->rn, w->r0, sizeof(double) * nb);
  if (!lanes_finite(w->rn, nb)) {
    const int b = worst_lane(w->rn, nb);
    return err_divergence(err, start_step, b + m->off, 0, w->rn[b], w->r0[b]);
  }
  *iters = 0;
  if (lanes_converged(w->rn, w->r0, nb, st)) return 0;
  for (int it = 1; it <= st->max_iter; ++it) {
    long long sweeps = 0;
    if (solver->kind == CKO_SOLVER_THOMAS) {
      /* fused Thomas loop (integrate.cpp:208-231) */
      for (int k = 0; k < c; ++k)
        for (int b = 0; b < nb; ++b) {
          if (!assemble_factor_point(m, w, k, b)) return err_singular(err, k, b + m->off);
          double* x = w->hr + ((size_t)k * nb + b) * n;
          if (k > 0) {
            const double* prev = w->hr + ((size_t)(k - 1) * nb + b) * n;
            for (int i = 0; i < n; ++i) x[i] += prev[i];
          }
          lu_solve_vec(fblk(&w->fac, k, b), fpiv(&w->fac, k, b), n, x);
          double* yyp = w->yy + ((size_t)k * nb + b) * n;
          for (int i = 0; i < n; ++i) yyp[i] -= x[i];
        }
    } else {
      for (int k = 0; k < c; ++k)
        for (int b = 0; b < nb; ++b)
          if (!assemble_factor_point(m, w, k, b)) return err_singular(err, k, b + m->off);
      solve_unit(&w->fac, w->offd, w->hr, solver, &sweeps);
      for (size_t i = 0; i < (size_t)c * nb * n; ++i) w->yy[i] -= w->hr[i];
    }
    if (work) {
      ++work->jacobian_evals;
      ++work->linear_solves;
      ++work->newton_iterations;
      work->reduction_sweeps += sweeps;
    }
    rate_residual_norms(m, w, w->rn);
    if (work) ++work->rate_evals;
    if (!lanes_finite(w->rn, nb)) {
      const int b = worst_lane(w->rn, nb);
      return err_divergence(err, start_step, b + m->off, it, w->rn[b], w->r0[b]);
    }
    if (lanes_converged(w->rn, w->r0, nb, st)) {
      *iters = it;
      return 0;
    }
  }
  const int b = worst_lane(w->rn, nb);
  return err_divergence(err, start_step, b + m->off, st->max_iter, w->rn[b], w->r0[b]);
}

static void nws_alloc(nws_t* w, const model_t* m, int c, int nb) {
  const int n = m->n;
  w->c = c;
  w->nb = nb;
  w->n = n;
  w->yy = (double*)calloc((size_t)c * nb * n, sizeof(double));
  w->hr = (double*)calloc((size_t)c * nb * n, sizeof(double));
  w->t = (double*)calloc((size_t)c * nb, sizeof(double));
  w->dt = (double*)calloc((size_t)c * nb, sizeof(double));
  w->ys = (double*)calloc((size_t)nb * n, sizeof(double));
  w->r0 = (double*)calloc((size_t)nb, sizeof(double));
  w->rn = (double*)calloc((size_t)nb, sizeof(double));
  w->offd = (double*)calloc((size_t)(c > 1 ? c - 1 : 1) * nb * n * n, sizeof(double));
  w->scr = (double*)calloc(scratch_len(m), sizeof(double));
  w->fac.nc = c;
  w->fac.nb = nb;
  w->fac.n = n;
  w->fac.lu = (double*)calloc((size_t)c * nb * n * n, sizeof(double));
  w->fac.piv = (int*)calloc((size_t)c * nb * n, sizeof(int));
}

static void nws_free(nws_t* w) {
  free(w->yy); free(w->hr); free(w->t); free(w->dt); free(w->ys); free(w->r0); free(w->rn);
  free(w->offd); free(w->scr); free(w->fac.lu); free(w->fac.piv);
  memset(w, 0, sizeof *w);
}

static int check_grid(const double* times, int nt, int nb, cko_error* err) {
  if (nt < 1 || nb < 1)
    return set_err(err, CKO_INVALID_TIME_GRID, "time grid needs at least one step and one batch lane");
  for (int i = 1; i <= nt; ++i)
    for (int b = 0; b < nb; ++b)
      if (!(times[(size_t)i * nb + b] > times[(size_t)(i - 1) * nb + b])) {
        char msg[128];
        snprintf(msg, sizeof msg, "time grid must be strictly increasing (step %d, batch %d)", i, b);
        return set_err(err, CKO_INVALID_TIME_GRID, msg);
      }
  return 0;
}

int cko_oracle_forward(const cko_model_desc* desc, const double* y0, const double* times, int nb,
                       int nt, int n_chunk, const cko_newton_settings* st,
                       const cko_solver_choice* solver, double* states, cko_work* work,
                       cko_error* err) {
  model_t m;
  int rc = model_init(&m, desc, err);
  if (rc) return rc;
  if ((rc = check_grid(times, nt, nb, err))) return rc;
  if (m.nbm > 0 && m.kind != CKO_MODEL_SCALAR_DECAY && m.kind != CKO_MODEL_CONSTANT_RATE &&
      m.off + nb > m.nbm)
    return set_err(err, CKO_SHAPE_MISMATCH, "integrate: model batch width != y0 rows");
  if (n_chunk < 1) return set_err(err, CKO_SHAPE_MISMATCH, "integrate: n_chunk must be >= 1");
  const int n = m.n;
  if (work) memset(work, 0, sizeof *work);
  memcpy(states, y0, sizeof(double) * (size_t)nb * n);
  nws_t w;
  memset(&w, 0, sizeof w);
  int cur = -1, step = 0;
  while (step < nt) {
    const int c = n_chunk < nt - step ? n_chunk : nt - step;
    if (c != cur) {
      if (cur > 0) nws_free(&w);
      nws_alloc(&w, &m, c, nb);
      cur = c;
    }
    memcpy(w.ys, states + (size_t)step * nb * n, sizeof(double) * (size_t)nb * n);
    for (int j = 0; j < c; ++j)
      for (int b = 0; b < nb; ++b) {
        w.t[(size_t)j * nb + b] = times[(size_t)(step + 1 + j) * nb + b];
        w.dt[(size_t)j * nb + b] =
            times[(size_t)(step + 1 + j) * nb + b] - times[(size_t)(step + j) * nb + b];
      }
    for (int j = 0; j < c; ++j) memcpy(w.yy + (size_t)j * nb * n, w.ys, sizeof(double) * (size_t)nb * n);
    int iters = 0;
    rc = newton_chunk(&m, &w, st, solver, work, step + 1, &iters, err);
    if (rc) break;
    memcpy(states + (size_t)(step + 1) * nb * n, w.yy, sizeof(double) * (size_t)c * nb * n);
    step += c;
  }
  if (cur > 0) nws_free(&w);
  if (!rc && err) set_err(err, CKO_OK, "");
  return rc;
}

/* ------------------------------------------------------------------------ */
/* adjoint (adjoint.cpp)                                                     */
/* ------------------------------------------------------------------------ */

/* be_chunk_core (adjoint.cpp:49-127) on rows r <-> steps step_hi - r. */
static int be_chunk(const model_t* m, nws_t* w, double* lambda, double* grad, double* wq,
                    const cko_solver_choice* solver, cko_work* work, cko_error* err) {
  const int c = w->c, nb = w->nb, n = w->n;
  double* jtl = (double*)malloc(sizeof(double) * (size_t)n);
  if (work) ++work->jacobian_evals;
  for (int r = 0; r < c; ++r)
    for (int b = 0; b < nb; ++b) {
      double* d = fblk(&w->fac, r, b);
      point_jacobian(m, w->t[(size_t)r * nb + b], w->yy + ((size_t)r * nb + b) * n, d, b, w->scr);
    }
  for (int r = 0; r < c; ++r)
    for (int b = 0; b < nb; ++b) {
      double* d = fblk(&w->fac, r, b);
      const double dt = w->dt[(size_t)r * nb + b];
      /* gemv_transpose (adjoint.cpp:36-43) */
      const double* lam = lambda + (size_t)b * n;
      for (int i = 0; i < n; ++i) jtl[i] = 0.0;
      for (int j = 0; j < n; ++j) {
        const double vj = lam[j];
        const double* row = d + (size_t)j * n;
        for (int i = 0; i < n; ++i) jtl[i] += row[i] * vj;
      }
      double* out = w->hr + ((size_t)r * nb + b) * n;
      for (int i = 0; i < n; ++i) out[i] += dt * jtl[i];
      for (int i = 0; i < n; ++i) {
        for (int q = i + 1; q < n; ++q) {
          const double a = d[(size_t)i * n + q];
          d[(size_t)i * n + q] = -dt * d[(size_t)q * n + i];
          d[(size_t)q * n + i] = -dt * a;
        }
        d[(size_t)i * n + i] = 1.0 - dt * d[(size_t)i * n + i];
      }
      if (!lu_factor_block(d, fpiv(&w->fac, r, b), n)) {
        free(jtl);
        return err_singular(err, r, b + m->off);
      }
    }
  free(jtl);
  long long sweeps = 0;
  solve_unit(&w->fac, w->offd, w->hr, solver, &sweeps);
  for (int r = 0; r < c; ++r)
    for (int b = 0; b < nb; ++b) {
      const double* carry = lambda + (size_t)b * n;
      const double* delta = w->hr + ((size_t)r * nb + b) * n;
      double* wr = wq + ((size_t)r * nb + b) * n;
      const double dt = w->dt[(size_t)r * nb + b];
      for (int i = 0; i < n; ++i) wr[i] = (carry[i] + delta[i]) * dt;
    }
  if (work) {
    ++work->linear_solves;
    work->reduction_sweeps += sweeps;
  }
  /* parameter_vjp (ode_model.cpp:135-153) */
  for (int r = 0; r < c; ++r)
    for (int b = 0; b < nb; ++b)
      point_vjp(m, w->t[(size_t)r * nb + b], w->yy + ((size_t)r * nb + b) * n,
                wq + ((size_t)r * nb + b) * n, grad, b, w->scr);
  for (int j = 0; j < m->np; ++j)
    if (!isfinite(grad[j]))
      return set_err(err, CKO_NON_FINITE, "parameter product of the model is not finite");
  for (int b = 0; b < nb; ++b)
    for (int i = 0; i < n; ++i) lambda[(size_t)b * n + i] += w->hr[((size_t)(c - 1) * nb + b) * n + i];
  return 0;
}

int cko_oracle_adjoint(const cko_model_desc* desc, const double* states, const double* times,
                       int nb, int nt, int n_chunk, const cko_solver_choice* solver,
                       int loss_kind, const double* dLu, double* loss_out, double* grad_out,
                       cko_work* bwd, cko_error* err) {
  model_t m;
  int rc = model_init(&m, desc, err);
  if (rc) return rc;
  if (n_chunk < 1) return set_err(err, CKO_SHAPE_MISMATCH, "adjoint: n_chunk must be >= 1");
  const int n = m.n;
  const size_t row = (size_t)nb * n;
  if (bwd) memset(bwd, 0, sizeof *bwd);
  /* loss_frobenius (adjoint.cpp:196-221) */
  double s = 0.0;
  for (int step = 1; step <= nt; ++step)
    for (size_t i = 0; i < row; ++i) s += states[step * row + i] * states[step * row + i];
  const double L = sqrt(s);
  double* dL = (double*)calloc((nt + 1) * row, sizeof(double));
  if (loss_kind == CKO_LOSS_USER) {
    memcpy(dL, dLu, sizeof(double) * (nt + 1) * row);
    if (loss_out) *loss_out = NAN;
  } else {
    for (int step = 1; step <= nt; ++step)
      for (size_t i = 0; i < row; ++i) dL[step * row + i] = L > 0.0 ? states[step * row + i] / L : 0.0;
    if (loss_out) *loss_out = L;
  }
  double* lambda = (double*)calloc(row, sizeof(double));
  for (int j = 0; j < m.np; ++j) grad_out[j] = 0.0;
  nws_t w;
  memset(&w, 0, sizeof w);
  double* wq = NULL;
  int cur = -1, step_hi = nt;
  while (step_hi >= 1) {
    const int c = n_chunk < step_hi ? n_chunk : step_hi;
    if (c != cur) {
      if (cur > 0) {
        nws_free(&w);
        free(wq);
      }
      nws_alloc(&w, &m, c, nb);
      wq = (double*)calloc((size_t)c * row, sizeof(double));
      cur = c;
    }
    /* gather_be_chunk (adjoint.cpp:136-149) */
    for (int r = 0; r < c; ++r) {
      const int mstep = step_hi - r;
      memcpy(w.yy + (size_t)r * row, states + (size_t)mstep * row, sizeof(double) * row);
      memcpy(w.hr + (size_t)r * row, dL + (size_t)mstep * row, sizeof(double) * row);
      for (int b = 0; b < nb; ++b) {
        w.t[(size_t)r * nb + b] = times[(size_t)mstep * nb + b];
        w.dt[(size_t)r * nb + b] = times[(size_t)mstep * nb + b] - times[(size_t)(mstep - 1) * nb + b];
      }
    }
    rc = be_chunk(&m, &w, lambda, grad_out, wq, solver, bwd, err);
    if (rc) break;
    step_hi -= c;
  }
  if (cur > 0) {
    nws_free(&w);
    free(wq);
  }
  free(lambda);
  free(dL);
  if (!rc && err) set_err(err, CKO_OK, "");
  return rc;
}

/* ------------------------------------------------------------------------ */
/* model-level entry points                                                  */
/* ------------------------------------------------------------------------ */

int cko_oracle_rate(const cko_model_desc* desc, const double* t, const double* y, int c, int nb,
                    double* out) {
  model_t m;
  int rc = model_init(&m, desc, NULL);
  if (rc) return rc;
  double* scr = (double*)calloc(scratch_len(&m), sizeof(double));
  for (int k = 0; k < c; ++k)
    for (int b = 0; b < nb; ++b)
      point_rate(&m, t[(size_t)k * nb + b], y + ((size_t)k * nb + b) * m.n,
                 out + ((size_t)k * nb + b) * m.n, b, scr);
  free(scr);
  return 0;
}

int cko_oracle_jacobian(const cko_model_desc* desc, const double* t, const double* y, int c,
                        int nb, double* out) {
  model_t m;
  int rc = model_init(&m, desc, NULL);
  if (rc) return rc;
  double* scr = (double*)calloc(scratch_len(&m), sizeof(double));
  for (int k = 0; k < c; ++k)
    for (int b = 0; b < nb; ++b)
      point_jacobian(&m, t[(size_t)k * nb + b], y + ((size_t)k * nb + b) * m.n,
                     out + ((size_t)k * nb + b) * m.n * m.n, b, scr);
  free(scr);
  return 0;
}

int cko_oracle_param_vjp(const cko_model_desc* desc, const double* t, const double* y,
                         const double* w, int c, int nb, double* grad) {
  model_t m;
  int rc = model_init(&m, desc, NULL);
  if (rc) return rc;
  double* scr = (double*)calloc(scratch_len(&m), sizeof(double));
  for (int k = 0; k < c; ++k)
    for (int b = 0; b < nb; ++b)
      point_vjp(&m, t[(size_t)k * nb + b], y + ((size_t)k * nb + b) * m.n,
                w + ((size_t)k * nb + b) * m.n, grad, b, scr);
  free(scr);
  return 0;
}

/* ------------------------------------------------------------------------ */
/* batch-sharded CPU timing run                                              */
/* ------------------------------------------------------------------------ */

typedef struct {
  cko_model_desc d;
  const double *y0, *times;
  int nb, nb_s, lo, nt, nc;
  cko_newton_settings st;
  cko_solver_choice sv;
  int rc;
} shard_job;

static void* shard_run(void* arg) {
  shard_job* j = (shard_job*)arg;
  const int n = state_size_of(&j->d);
  double* y0 = (double*)malloc(sizeof(double) * (size_t)j->nb_s * n);
  double* tt = (double*)malloc(sizeof(double) * (size_t)(j->nt + 1) * j->nb_s);
  double* st = (double*)malloc(sizeof(double) * (size_t)(j->nt + 1) * j->nb_s * n);
  double* g = (double*)malloc(sizeof(double) * (size_t)j->d.n_params);
  memcpy(y0, j->y0 + (size_t)j->lo * n, sizeof(double) * (size_t)j->nb_s * n);
  for (int i = 0; i <= j->nt; ++i)
    memcpy(tt + (size_t)i * j->nb_s, j->times + (size_t)i * j->nb + j->lo, sizeof(double) * j->nb_s);
  cko_work wf, wb;
  cko_error e;
  double L;
  j->rc = cko_oracle_forward(&j->d, y0, tt, j->nb_s, j->nt, j->nc, &j->st, &j->sv, st, &wf, &e);
  if (!j->rc)
    j->rc = cko_oracle_adjoint(&j->d, st, tt, j->nb_s, j->nt, j->nc, &j->sv, CKO_LOSS_FROBENIUS, NULL,
                               &L, g, &wb, &e);
  free(y0); free(tt); free(st); free(g);
  return NULL;
}

double cko_oracle_sharded_timing(const cko_model_desc* desc, const double* y0, const double* times,
                                 int nb, int nt, int n_chunk, const cko_newton_settings* settings,
                                 const cko_solver_choice* solver, int threads) {
  if (threads < 1) threads = 1;
  if (threads > nb) threads = nb;
  shard_job* jobs = (shard_job*)calloc((size_t)threads, sizeof(shard_job));
  pthread_t* th = (pthread_t*)calloc((size_t)threads, sizeof(pthread_t));
  struct timespec a, b;
  clock_gettime(CLOCK_MONOTONIC, &a);
  for (int i = 0; i < threads; ++i) {
    const int lo = (int)((long long)nb * i / threads), hi = (int)((long long)nb * (i + 1) / threads);
    jobs[i].d = *desc;
    jobs[i].d.lane_offset = desc->lane_offset + lo;
    jobs[i].y0 = y0;
    jobs[i].times = times;
    jobs[i].nb = nb;
    jobs[i].nb_s = hi - lo;
    jobs[i].lo = lo;
    jobs[i].nt = nt;
    jobs[i].nc = n_chunk;
    jobs[i].st = *settings;
    jobs[i].sv = *solver;
    pthread_create(&th[i], NULL, shard_run, &jobs[i]);
  }
  int rc = 0;
  for (int i = 0; i < threads; ++i) {
    pthread_join(th[i], NULL);
    if (jobs[i].rc) rc = jobs[i].rc;
  }
  clock_gettime(CLOCK_MONOTONIC, &b);
  free(jobs);
  free(th);
  if (rc) return -1.0;
  return (double)(b.tv_sec - a.tv_sec) + 1e-9 * (double)(b.tv_nsec - a.tv_nsec);
}
