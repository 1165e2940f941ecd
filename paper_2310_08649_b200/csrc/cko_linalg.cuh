// cko_linalg.cuh — per-point dense block kernels on generic accessors:
// LU with partial pivoting, vector solve, right solve X A = Y, y -= M x and
// C = -(A B). Semantics (pivot rule, singular threshold, multiply by the
// reciprocal in elimination, divide in back substitution) follow
// /root/reference/proj/core/src/linalg.cpp:13-123.
#pragma once

#include "cko_common.cuh"

namespace cko {

// lu_factor_block (linalg.cpp:13-44). Returns false on a negligible pivot.
template <class B, class P>
__device__ inline bool lu_factor(const B& a, const P& piv, int n) {
  double scale = 0.0;
  for (int i = 0; i < n; ++i)
    for (int j = 0; j < n; ++j) {
      const double v = fabs(a(i, j));
      scale = (scale < v) ? v : scale;
    }
  const double tiny = 1e-14 * scale;
  for (int c = 0; c < n; ++c) {
    int p = c;
    double best = fabs(a(c, c));
    for (int r = c + 1; r < n; ++r) {
      const double v = fabs(a(r, c));
      if (v > best) {
        best = v;
        p = r;
      }
    }
    piv[c] = p;
    if (best < tiny || best == 0.0) return false;
    if (p != c)
      for (int j = 0; j < n; ++j) {
        const double t = a(c, j);
        a(c, j) = a(p, j);
        a(p, j) = t;
      }
    const double inv = 1.0 / a(c, c);
    for (int r = c + 1; r < n; ++r) {
      const double l = a(r, c) * inv;
      a(r, c) = l;
      if (l != 0.0)
        for (int j = c + 1; j < n; ++j) a(r, j) -= l * a(c, j);
    }
  }
  return true;
}

// lu_solve_vec (linalg.cpp:46-60), in place on y.
template <class B, class P, class V>
__device__ inline void lu_solve(const B& lu, const P& piv, int n, const V& y) {
  for (int i = 0; i < n; ++i) {
    const int p = piv[i];
    if (p != i) {
      const double t = y[i];
      y[i] = y[p];
      y[p] = t;
    }
  }
  for (int i = 1; i < n; ++i) {
    double s = y[i];
    for (int j = 0; j < i; ++j) s -= lu(i, j) * y[j];
    y[i] = s;
  }
  for (int i = n - 1; i >= 0; --i) {
    double s = y[i];
    for (int j = i + 1; j < n; ++j) s -= lu(i, j) * y[j];
    y[i] = s / lu(i, i);
  }
}

// lu_right_solve_mat (linalg.cpp:62-82): rows of Y (n x n) become X with X A = Y.
template <class B, class P, class M>
__device__ inline void lu_right_solve(const B& lu, const P& piv, int n, const M& y) {
  for (int r = 0; r < n; ++r) {
    for (int i = 0; i < n; ++i) {
      double s = y(r, i);
      for (int j = 0; j < i; ++j) s -= lu(j, i) * y(r, j);
      y(r, i) = s / lu(i, i);
    }
    for (int i = n - 2; i >= 0; --i) {
      double s = y(r, i);
      for (int j = i + 1; j < n; ++j) s -= lu(j, i) * y(r, j);
      y(r, i) = s;
    }
    for (int i = n - 1; i >= 0; --i) {
      const int p = piv[i];
      if (p != i) {
        const double t = y(r, i);
        y(r, i) = y(r, p);
        y(r, p) = t;
      }
    }
  }
}

// out = y - M x (gemv_sub, linalg.cpp:101-108); out may alias y.
template <class M, class V1, class V2, class V3>
__device__ inline void gemv_sub_into(const M& mat, const V1& x, const V2& y, const V3& out, int n) {
  for (int i = 0; i < n; ++i) {
    double s = 0.0;
    for (int j = 0; j < n; ++j) s += mat(i, j) * x[j];
    out[i] = y[i] - s;
  }
}

// C = -(A B) (gemm_neg, linalg.cpp:110-123); C must not alias A or B.
template <class MA, class MB, class MC>
__device__ inline void gemm_neg(const MA& A, const MB& Bm, const MC& Cm, int n) {
  for (int i = 0; i < n; ++i) {
    for (int j = 0; j < n; ++j) Cm(i, j) = 0.0;
    for (int k = 0; k < n; ++k) {
      const double a = A(i, k);
      if (a == 0.0) continue;
      for (int j = 0; j < n; ++j) Cm(i, j) -= a * Bm(k, j);
    }
  }
}

}  // namespace cko
