// cko_lu_thread.cuh — one thread factors one N x N block held in its own
// shared-memory record (row-major, 16-byte aligned rows when N is even).
//
// lu_thread_nopiv: right-looking LU in panels of 4 columns (LAPACK getrf
// order) for blocks where the reference's partial-pivoting scan keeps every
// diagonal (|a(r,c)| <= |a(c,c)| for r > c, checked on the fly and reported in
// `viol`). The panel and the U12 strip live in registers, the trailing matrix
// streams through shared memory once per panel (4 B of traffic per
// multiply-add). Every entry accumulates its updates in the same order as the
// unblocked lu_factor_block (linalg.cpp:13-44): results are bit-identical.
//
// lu_thread_pivot: the unblocked reference algorithm with partial pivoting
// and physical row swaps, for the rare blocks that need an exchange.
#pragma once

#include <cuda_runtime.h>

namespace cko {
namespace lt {

constexpr int NB = 4;

// One panel step of lu_thread_nopiv (P0 = first column of the panel); the
// panels are unrolled through template recursion so every register array
// index is a compile-time constant.
template <int N, int P0>
__device__ __forceinline__ void lu_panel(double* __restrict__ A, double* __restrict__ rd, double tiny, bool& ok,
                                         bool& viol) {
  if constexpr (P0 < N) {
    constexpr int W = (N - P0) < NB ? (N - P0) : NB;
    double L11[NB][NB];
    {
      // ---- panel: rows P0..N-1, columns P0..P0+W-1, in registers
      double P[N - P0][W];
#pragma unroll
      for (int r = 0; r < N - P0; ++r)
#pragma unroll
        for (int q = 0; q < W; ++q) P[r][q] = A[(P0 + r) * N + P0 + q];
#pragma unroll
      for (int q = 0; q < W; ++q) {
        const double piv = P[q][q];
        const double apiv = fabs(piv);
        if (apiv < tiny || piv == 0.0) ok = false;
        const double inv = __drcp_rn(piv);
        rd[P0 + q] = inv;
#pragma unroll
        for (int r = q + 1; r < N - P0; ++r) {
          const double v = P[r][q];
          viol |= fabs(v) > apiv;
          const double l = v * inv;
          P[r][q] = l;
#pragma unroll
          for (int q2 = q + 1; q2 < W; ++q2) P[r][q2] -= l * P[q][q2];
        }
      }
#pragma unroll
      for (int r = 0; r < N - P0; ++r)
#pragma unroll
        for (int q = 0; q < W; ++q) A[(P0 + r) * N + P0 + q] = P[r][q];
#pragma unroll
      for (int q = 0; q < W; ++q)
#pragma unroll
        for (int m = 0; m < W; ++m) L11[q][m] = P[q][m];
    }
    if constexpr (P0 + NB < N) {
      constexpr int J0 = P0 + NB, NJ = N - J0;
      // ---- U12 = L11^{-1} A12 (columns J0..N-1), kept in registers
      double U[NB][NJ];
#pragma unroll
      for (int j = 0; j < NJ; ++j) {
#pragma unroll
        for (int q = 0; q < NB; ++q) {
          double u = A[(P0 + q) * N + J0 + j];
#pragma unroll
          for (int m = 0; m < q; ++m) u -= L11[q][m] * U[m][j];
          U[q][j] = u;
          A[(P0 + q) * N + J0 + j] = u;
        }
      }
      // ---- trailing update A22 -= L21 U12, one row at a time (rolled)
#pragma unroll 1
      for (int r = J0; r < N; ++r) {
        double* ar = A + r * N;
        double l[NB];
#pragma unroll
        for (int q = 0; q < NB; ++q) l[q] = ar[P0 + q];
#pragma unroll
        for (int j = 0; j < NJ; ++j) {
          double v = ar[J0 + j];
#pragma unroll
          for (int q = 0; q < NB; ++q) v -= l[q] * U[q][j];
          ar[J0 + j] = v;
        }
      }
    }
    lu_panel<N, P0 + NB>(A, rd, tiny, ok, viol);
  }
}

// Factor A in place; rd[c] = 1 / U_cc. `tiny` = 1e-14 max|A| (the caller
// tracks max|A| while assembling). Returns false on a negligible pivot.
template <int N>
__device__ inline bool lu_thread_nopiv(double* __restrict__ A_, double* __restrict__ rd, double tiny, bool& viol) {
  double* A = static_cast<double*>(__builtin_assume_aligned(A_, 16));
  bool ok = true;
  viol = false;
  lu_panel<N, 0>(A, rd, tiny, ok, viol);
  return ok;
}

// Unblocked LU with partial pivoting and physical row swaps (linalg.cpp:13-44),
// the reference's exact algorithm; perm[i] = original row now at position i.
template <int N>
__device__ inline bool lu_thread_pivot(double* __restrict__ A, double* __restrict__ rd, int* __restrict__ perm,
                                       double tiny) {
  for (int i = 0; i < N; ++i) perm[i] = i;
  for (int c = 0; c < N; ++c) {
    int p = c;
    double best = fabs(A[c * N + c]);
    for (int r = c + 1; r < N; ++r) {
      const double v = fabs(A[r * N + c]);
      if (v > best) best = v, p = r;
    }
    if (best < tiny || best == 0.0) return false;
    if (p != c) {
      for (int j = 0; j < N; ++j) {
        const double t = A[c * N + j];
        A[c * N + j] = A[p * N + j];
        A[p * N + j] = t;
      }
      const int t = perm[c];
      perm[c] = perm[p];
      perm[p] = t;
    }
    const double inv = __drcp_rn(A[c * N + c]);
    rd[c] = inv;
    for (int r = c + 1; r < N; ++r) {
      const double l = A[r * N + c] * inv;
      A[r * N + c] = l;
      for (int j = c + 1; j < N; ++j) A[r * N + j] -= l * A[c * N + j];
    }
  }
  return true;
}

}  // namespace lt
}  // namespace cko
