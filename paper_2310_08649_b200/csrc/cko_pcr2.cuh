// cko_pcr2.cuh — generation-2 kernels for the parallel-cyclic-reduction and
// hybrid solvers (strided_solve_into, linalg.cpp:197-255) on small blocks
// (N <= 8), one thread per (row, lane) point.
//
// PCR's point is parallelism in time: when the batch is too small to fill the
// GPU (C3: 50 lanes), every row of a chunk is factored at once and the
// block-bidiagonal system is reduced in log2(c) sweeps. A CTA owns whole lanes,
// so the sweeps only need __syncthreads; the forward's all-lanes Newton
// predicate is the only grid-wide step (grid_reduce_or, as in fwd2_kernel).
// Per-point records (LU, B, x, ...) live in shared memory when the chunk fits
// (c * L * STRIDE * 8 bytes <= ~200 KB), otherwise in a per-CTA global slab.
// Arithmetic follows the reference operation by operation: lu_right_solve_mat,
// gemv_sub and gemm_neg (linalg.cpp:62-123) with the couplings initialised to
// -I (fill_minus_identity, linalg.cpp:261-266).
#pragma once

#include "cko_lu_thread.cuh"
#include "cko_v2.cuh"

namespace cko {
namespace v2 {

template <int N>
struct PRec {
  static constexpr int LU = 0;
  static constexpr int RD = N * N;
  static constexpr int PERM = RD + N;  // N ints + identity flag
  static constexpr int B = PERM + (N + 2) / 2;
  static constexpr int BN = B + N * N;
  static constexpr int X = BN + N * N;
  static constexpr int XT = X + N;
  static constexpr int VS = XT + N;
  static constexpr int RAW = VS + N;
  static constexpr int STRIDE = RAW + ((2 - RAW % 16) + 16) % 16;  // 16-byte aligned records
};

// v <- M^{-1} v from a PRec record (lu_solve_vec, linalg.cpp:46-60)
template <int N>
__device__ inline void prec_solve(const double* rec, double (&v)[N]) {
  const int* perm = reinterpret_cast<const int*>(rec + PRec<N>::PERM);
  double y[N];
  if (perm[N]) {
#pragma unroll
    for (int i = 0; i < N; ++i) y[i] = v[i];
  } else {
    double* vs = const_cast<double*>(rec) + PRec<N>::VS;
#pragma unroll
    for (int i = 0; i < N; ++i) vs[i] = v[i];
#pragma unroll
    for (int i = 0; i < N; ++i) y[i] = vs[perm[i]];
  }
#pragma unroll
  for (int i = 1; i < N; ++i) {
    double s = y[i];
#pragma unroll
    for (int j = 0; j < i; ++j) s -= rec[i * N + j] * y[j];
    y[i] = s;
  }
#pragma unroll
  for (int i = N - 1; i >= 0; --i) {
    double s = y[i];
#pragma unroll
    for (int j = i + 1; j < N; ++j) s -= rec[i * N + j] * y[j];
    y[i] = s * rec[PRec<N>::RD + i];
  }
#pragma unroll
  for (int i = 0; i < N; ++i) v[i] = y[i];
}

// Rows of P (N x N) become X with X M = P (lu_right_solve_mat, linalg.cpp:62-82).
template <int N>
__device__ inline void prec_right_solve(const double* rec, double (&P)[N][N]) {
  const int* perm = reinterpret_cast<const int*>(rec + PRec<N>::PERM);
  const bool ident = perm[N] != 0;
#pragma unroll
  for (int r = 0; r < N; ++r) {
#pragma unroll
    for (int i = 0; i < N; ++i) {
      double s = P[r][i];
#pragma unroll
      for (int j = 0; j < i; ++j) s -= rec[j * N + i] * P[r][j];
      P[r][i] = s * rec[PRec<N>::RD + i];
    }
#pragma unroll
    for (int i = N - 2; i >= 0; --i) {
      double s = P[r][i];
#pragma unroll
      for (int j = i + 1; j < N; ++j) s -= rec[j * N + i] * P[r][j];
      P[r][i] = s;
    }
  }
  if (!ident) {  // X = Z P: column perm[i] of X is column i of Z
    double* vs = const_cast<double*>(rec) + PRec<N>::VS;
#pragma unroll
    for (int r = 0; r < N; ++r) {
#pragma unroll
      for (int i = 0; i < N; ++i) vs[perm[i]] = P[r][i];
#pragma unroll
      for (int i = 0; i < N; ++i) P[r][i] = vs[i];
    }
  }
}

// Factor the block assembled in rec[LU] (no-exchange fast path, reference
// pivoting fallback). `rebuild` re-assembles the block for the fallback.
template <int N, class Rebuild>
__device__ inline bool prec_factor(double* rec, double tiny, const Rebuild& rebuild) {
  bool viol;
  bool ok = lt::lu_thread_nopiv<N>(rec, rec + PRec<N>::RD, tiny, viol);
  int* perm = reinterpret_cast<int*>(rec + PRec<N>::PERM);
  if (viol) {
    rebuild();
    ok = lt::lu_thread_pivot<N>(rec, rec + PRec<N>::RD, perm, tiny);
    perm[N] = 0;
  } else {
#pragma unroll
    for (int i = 0; i < N; ++i) perm[i] = i;
    perm[N] = 1;
  }
  return ok;
}

struct PcrCtx {
  double* ws;   // records of this CTA (shared or global)
  int L, c;     // lanes of this CTA, rows of the chunk
  int nsw_arg;  // -1 (PCR) or n_switch (hybrid)
};

// Block-bidiagonal solve with -I couplings over every lane of the CTA
// (solve_unit_offdiag -> strided_solve_into); x in rec[X] in, solution out.
template <int N>
__device__ void pcr_solve_cta(const PcrCtx& pc) {
  const int T = blockDim.x, tid = threadIdx.x, L = pc.L, c = pc.c;
  auto rec = [&](int k, int lb) { return pc.ws + (size_t)(k * L + lb) * PRec<N>::STRIDE; };
  // couplings start as -I (fill_minus_identity)
  for (int p = tid; p < c * L; p += T) {
    double* B = pc.ws + (size_t)p * PRec<N>::STRIDE + PRec<N>::B;
#pragma unroll
    for (int i = 0; i < N; ++i)
#pragma unroll
      for (int j = 0; j < N; ++j) B[i * N + j] = (i == j) ? -1.0 : 0.0;
  }
  __syncthreads();
  int base = 0;
  for (int bit = 30; bit >= 0; --bit) {
    const int m = 1 << bit;
    if (!(c & m)) continue;
    if (base > 0) {  // fold the solved previous partition through the original coupling
      for (int lb = tid; lb < L; lb += T) {
        double* xr = rec(base, lb) + PRec<N>::X;
        const double* xp = rec(base - 1, lb) + PRec<N>::X;
        const double* Br = rec(base, lb) + PRec<N>::B;
#pragma unroll
        for (int i = 0; i < N; ++i) {
          double s = 0.0;
#pragma unroll
          for (int j = 0; j < N; ++j) s += Br[i * N + j] * xp[j];
          xr[i] -= s;
        }
      }
      __syncthreads();
    }
    int e = 0;
    while ((1 << e) < m) ++e;
    const int nsw = (pc.nsw_arg < 0) ? e : (pc.nsw_arg < e ? pc.nsw_arg : e);
    for (int sidx = 0; sidx < nsw; ++sidx) {
      const int s = 1 << sidx;
      const int cnt = (m - s) * L;
      for (int idx = tid; idx < cnt; idx += T) {
        const int r = base + s + idx / L, lb = idx % L, q = r - s;
        double* rr = rec(r, lb);
        const double* rq = rec(q, lb);
        double P[N][N];
#pragma unroll
        for (int i = 0; i < N; ++i)
#pragma unroll
          for (int j = 0; j < N; ++j) P[i][j] = rr[PRec<N>::B + i * N + j];
        prec_right_solve<N>(rq, P);
#pragma unroll
        for (int i = 0; i < N; ++i) {  // gemv_sub: x_r - P x_q
          double acc = 0.0;
#pragma unroll
          for (int j = 0; j < N; ++j) acc += P[i][j] * rq[PRec<N>::X + j];
          rr[PRec<N>::XT + i] = rr[PRec<N>::X + i] - acc;
        }
        if (q - base >= s) {  // gemm_neg: B_r <- -(P B_q)
#pragma unroll
          for (int i = 0; i < N; ++i) {
            double cr[N];
#pragma unroll
            for (int j = 0; j < N; ++j) cr[j] = 0.0;
#pragma unroll
            for (int kk = 0; kk < N; ++kk) {
              const double av = P[i][kk];
              if (av == 0.0) continue;
#pragma unroll
              for (int j = 0; j < N; ++j) cr[j] -= av * rq[PRec<N>::B + kk * N + j];
            }
#pragma unroll
            for (int j = 0; j < N; ++j) rr[PRec<N>::BN + i * N + j] = cr[j];
          }
        }
      }
      __syncthreads();
      for (int idx = tid; idx < cnt; idx += T) {
        const int r = base + s + idx / L, lb = idx % L, q = r - s;
        double* rr = rec(r, lb);
#pragma unroll
        for (int i = 0; i < N; ++i) rr[PRec<N>::X + i] = rr[PRec<N>::XT + i];
        if (q - base >= s) {
#pragma unroll
          for (int i = 0; i < N * N; ++i) rr[PRec<N>::B + i] = rr[PRec<N>::BN + i];
        }
      }
      __syncthreads();
    }
    // finish the independent strided chains
    const int stride = 1 << nsw;
    const int nch = stride < m ? stride : m;
    for (int idx = tid; idx < nch * L; idx += T) {
      const int ch = idx / L, lb = idx % L, r0 = base + ch;
      double xp[N];
      {
        double* rr = rec(r0, lb);
#pragma unroll
        for (int i = 0; i < N; ++i) xp[i] = rr[PRec<N>::X + i];
        prec_solve<N>(rr, xp);
#pragma unroll
        for (int i = 0; i < N; ++i) rr[PRec<N>::X + i] = xp[i];
      }
      for (int r = r0 + stride; r < base + m; r += stride) {
        double* rr = rec(r, lb);
        double v[N];
#pragma unroll
        for (int i = 0; i < N; ++i) {
          double acc = 0.0;
#pragma unroll
          for (int j = 0; j < N; ++j) acc += rr[PRec<N>::B + i * N + j] * xp[j];
          v[i] = rr[PRec<N>::X + i] - acc;
        }
        prec_solve<N>(rr, v);
#pragma unroll
        for (int i = 0; i < N; ++i) rr[PRec<N>::X + i] = v[i], xp[i] = v[i];
      }
    }
    __syncthreads();
    base += m;
  }
}

template <class MS>
__device__ inline double* pcr_workspace(const Slab& slab, double* smem_ws, bool in_smem, int c, int L) {
  if (in_smem) return smem_ws;
  // after this CTA's residual rows and norms in the forward slab layout
  return slab.base + (size_t)blockIdx.x * slab.doubles + (size_t)slab.Pmax * (MS::N + 1);
}

// ---------------------------------------------------------------------------
// forward
// ---------------------------------------------------------------------------
template <class MS>
__global__ void __launch_bounds__(512, 1) fwd_pcr2_kernel(FwdLaunch a, int in_smem) {
  constexpr int N = MS::N;
  extern __shared__ __align__(16) double smem[];
  __shared__ unsigned s_bcast, s_flags, s_sing;
  double* cs = smem;
  constexpr int OCS = ((MS::NCONST + 1) / 2) * 2;
  MS::load_consts(a.m, cs);
  if (threadIdx.x == 0) s_sing = 0;
  FwdCtx x;
  lane_range(a.nb, x.lb0, x.L);
  x.row = (size_t)a.nb * N;
  double* hr = a.slab.base + (size_t)blockIdx.x * a.slab.doubles;
  double* nrm = hr + (size_t)a.slab.Pmax * N;
  const bool leader = blockIdx.x == 0 && threadIdx.x == 0;
  const int T = blockDim.x, tid = threadIdx.x, nb = a.nb;
  __syncthreads();
  int step = 0, chunk = 0;
  if (a.loss_part) *loss_slot(a) = 0.0;  // Frobenius loss partial: sum y^2 of converged rows (this thread's)
  while (step < a.nt) {
    const int c = min(a.nc, a.nt - step);
    if (a.times_ready && !wait_times_rows(a, step + c + 1)) {  // this chunk's rows of the streamed grid
      if (leader) a.info[0] = 4, a.info[1] = step + 1, a.info[2] = 0;
      return;
    }
    x.step = step;
    x.c = c;
    PcrCtx pc{pcr_workspace<MS>(a.slab, smem + OCS, in_smem != 0, c, x.L), x.L, c, a.solver == 1 ? -1 : a.n_switch};
    for (int p = tid; p < c * x.L; p += T) {  // initial iterate: every row at y_start
      const int k = p / x.L, b = x.lb0 + p % x.L;
      double v[N];
      load_vec<N>(a.states + (size_t)step * x.row + (size_t)b * N, v);  // all loads before any store
      if (a.dy_init) {
        double d[N];
        load_vec<N>(a.dy_init + ((size_t)k * nb + b) * N, d);
#pragma unroll
        for (int i = 0; i < N; ++i) v[i] += d[i];
      }
      double* dst = a.states + (size_t)(step + 1 + k) * x.row + (size_t)b * N;
#pragma unroll
      for (int i = 0; i < N; ++i) dst[i] = v[i];
    }
    __syncthreads();
    int it = 0;
    // residual staging in the (idle) shared-memory PCR workspace, if it lives there
    const int stage_cap = in_smem ? (int)(dyn_smem_bytes() / 8) - OCS : 0;
    unsigned f = residual2<MS>(a, x, cs, hr, nrm, smem + OCS, stage_cap, true, &s_flags, a.loss_part ? loss_slot(a) + 1 : nullptr);
    f = grid_reduce_or(a.gs, a.grp, f, a.budget_ns, &s_bcast);
    if (f & (FLAG_TIMEOUT | FLAG_NON_FINITE)) {
      if (leader) a.info[0] = (f & FLAG_TIMEOUT) ? 4 : 2, a.info[1] = step + 1, a.info[2] = 0;
      return;
    }
    while (f & FLAG_NOT_CONVERGED) {
      if (it == a.max_iter) {
        if (leader) a.info[0] = 2, a.info[1] = step + 1, a.info[2] = a.max_iter;
        return;
      }
      ++it;
      // assemble M = I - J dt, factor, x = r (assemble_factor, integrate.cpp:118-135)
      for (int p = tid; p < c * x.L; p += T) {
        const int k = p / x.L, lb = p % x.L, b = x.lb0 + lb;
        double* rec = pc.ws + (size_t)p * PRec<N>::STRIDE;
        const double t = a.times[(size_t)(step + 1 + k) * nb + b];
        const double dt = t - a.times[(size_t)(step + k) * nb + b];
        double y[N];
        load_vec<N>(a.states + (size_t)(step + 1 + k) * x.row + (size_t)b * N, y);
        const double ndt = -dt;
        double mx = 0.0;
        auto build = [&]() {
#pragma unroll
          for (int i = 0; i < N; ++i) {
            double row[N];
            MS::jac_row(a.m, cs, t, y, i, row, b);
#pragma unroll
            for (int j = 0; j < N; ++j) {
              double v = xmul(ndt, row[j]);
              if (j == i) v = xadd(v, 1.0);
              rec[i * N + j] = v;
              mx = fmax(mx, fabs(v));
            }
          }
        };
        build();
        const double* r = hr + (size_t)p * N;
#pragma unroll
        for (int i = 0; i < N; ++i) rec[PRec<N>::X + i] = r[i];
        if (!prec_factor<N>(rec, 1e-14 * mx, build)) {
          atomicMin(a.sing_key, (unsigned long long)k * nb + b);
          atomicOr(&s_sing, 1u);
        }
      }
      __syncthreads();
      pcr_solve_cta<N>(pc);
      for (int p = tid; p < c * x.L; p += T) {  // yy -= x
        const int k = p / x.L, b = x.lb0 + p % x.L;
        double* yy = a.states + (size_t)(step + 1 + k) * x.row + (size_t)b * N;
        const double* xv = pc.ws + (size_t)p * PRec<N>::STRIDE + PRec<N>::X;
#pragma unroll
        for (int i = 0; i < N; ++i) yy[i] -= xv[i];
      }
      __syncthreads();
      const unsigned fl = s_sing ? FLAG_SINGULAR : 0u;
      f = residual2<MS>(a, x, cs, hr, nrm, smem + OCS, stage_cap, false, &s_flags, a.loss_part ? loss_slot(a) + 1 : nullptr) | fl;
      f = grid_reduce_or(a.gs, a.grp, f, a.budget_ns, &s_bcast);
      if (f & (FLAG_TIMEOUT | FLAG_SINGULAR | FLAG_NON_FINITE)) {
        if (leader) {
          a.info[0] = (f & FLAG_TIMEOUT) ? 4 : (f & FLAG_SINGULAR) ? 1 : 2;
          a.info[1] = step + 1;
          a.info[2] = it;
        }
        return;
      }
    }
    if (a.loss_part) loss_slot(a)[0] += loss_slot(a)[1];  // the last residual pass saw the converged iterate
    if (leader) a.iters[chunk] = it;
    step += c;
    ++chunk;
    __syncthreads();
  }
  if (leader) a.info[3] = chunk;
  if (a.loss_part) fwd_loss_store(a.loss_part, *loss_slot(a));
}

// ---------------------------------------------------------------------------
// adjoint
// ---------------------------------------------------------------------------
template <class MS>
__global__ void __launch_bounds__(512, 1) adj_pcr2_kernel(AdjLaunch a, int in_smem) {
  constexpr int N = MS::N;
  extern __shared__ __align__(16) double smem[];
  double* cs = smem;
  constexpr int OCS = ((MS::NCONST + 1) / 2) * 2;
  MS::load_consts(a.m, cs);
  int lb0, L;
  lane_range(a.nb, lb0, L);
  const int T = blockDim.x, tid = threadIdx.x, nb = a.nb;
  const size_t row = (size_t)nb * N;
  const double Lval = adj_loss_value(a);
  double* lam = smem + OCS;  // (L, N) carry
  const int olam = OCS + ((L * N + 1) / 2) * 2;
  for (int i = tid; i < L * N; i += T) lam[i] = 0.0;
  __syncthreads();
  int step_hi = a.nt;
  unsigned long long ord = 0;
  while (step_hi >= 1) {
    const int c = min(a.nc, step_hi);
    double* ws = in_smem ? smem + olam : a.slab.base + (size_t)blockIdx.x * a.slab.doubles;
    PcrCtx pc{ws, L, c, a.solver == 1 ? -1 : a.n_switch};
    // gather + J + rhs_r = dL + dt J^T lambda + transposed LU (adjoint.cpp:53-81)
    for (int p = tid; p < c * L; p += T) {
      const int r = p / L, lb = p % L, b = lb0 + lb, m = step_hi - r;
      double* rec = ws + (size_t)p * PRec<N>::STRIDE;
      const double t = a.times[(size_t)m * nb + b];
      const double dt = t - a.times[(size_t)(m - 1) * nb + b];
      double y[N];
      load_vec<N>(a.states + (size_t)m * row + (size_t)b * N, y);
      const double* lc = lam + (size_t)lb * N;
      double tmp[N];
#pragma unroll
      for (int i = 0; i < N; ++i) tmp[i] = 0.0;
      double mx = 0.0;
      auto build = [&]() {
#pragma unroll
        for (int i = 0; i < N; ++i) {  // J row i -> column i of M^T
          double jr[N];
          MS::jac_row(a.m, cs, t, y, i, jr, b);
#pragma unroll
          for (int j = 0; j < N; ++j) {
            const double v = (j == i) ? 1.0 - dt * jr[j] : -dt * jr[j];
            rec[j * N + i] = v;
            mx = fmax(mx, fabs(v));
          }
        }
      };
#pragma unroll
      for (int i = 0; i < N; ++i) {  // (J^T lambda): out[i] += row_j[i] * lambda_j, j outer
        double jr[N];
        MS::jac_row(a.m, cs, t, y, i, jr, b);
#pragma unroll
        for (int j = 0; j < N; ++j) tmp[j] += jr[j] * lc[i];
      }
      build();
#pragma unroll
      for (int i = 0; i < N; ++i) {
        const double dl = a.dL ? a.dL[(size_t)m * row + (size_t)b * N + i] : (Lval > 0.0 ? y[i] / Lval : 0.0);
        rec[PRec<N>::X + i] = dl + dt * tmp[i];
      }
      if (!prec_factor<N>(rec, 1e-14 * mx, build))
        atomicMin(a.sing_key, ord * (unsigned long long)a.nc * nb + (unsigned long long)r * nb + b);
    }
    __syncthreads();
    pcr_solve_cta<N>(pc);
    // quadrature weights w_r = (carry + delta_r) dt_r (adjoint.cpp:103-113)
    for (int p = tid; p < c * L; p += T) {
      const int r = p / L, lb = p % L, b = lb0 + lb, m = step_hi - r;
      const double dt = a.times[(size_t)m * nb + b] - a.times[(size_t)(m - 1) * nb + b];
      const double* d = ws + (size_t)p * PRec<N>::STRIDE + PRec<N>::X;
      const double* lc = lam + (size_t)lb * N;
      double* w = a.wq + (size_t)m * row + (size_t)b * N;
#pragma unroll
      for (int i = 0; i < N; ++i) w[i] = (lc[i] + d[i]) * dt;
    }
    __syncthreads();
    for (int idx = tid; idx < L * N; idx += T)  // new carry (adjoint.cpp:121-126)
      lam[idx] += ws[(size_t)((c - 1) * L + idx / N) * PRec<N>::STRIDE + PRec<N>::X + idx % N];
    __syncthreads();
    step_hi -= c;
    ++ord;
  }
  for (int i = tid; i < L * N; i += T) a.lambda[(size_t)lb0 * N + i] = lam[i];
}

// Launch plumbing. The global fallback workspace the host allocates per CTA is
// Pmax (n + 1) (forward residual rows + norms) + Pmax * pcr2_stride_bound(n).
__host__ __device__ constexpr int pcr2_stride_bound(int n) { return 3 * n * n + 5 * n + 20; }
static_assert(PRec<8>::STRIDE <= pcr2_stride_bound(8), "pcr2 record bound");
static_assert(PRec<5>::STRIDE <= pcr2_stride_bound(5), "pcr2 record bound");

// Workspace doubles per CTA for a chunk of c rows and Lmax lanes.
template <class MS>
inline size_t pcr2_ws_doubles(int c, int Lmax) {
  return (size_t)c * Lmax * PRec<MS::N>::STRIDE;
}

template <class MS>
inline int pcr2_threads(int c, int Lmax) {
  int t = c * Lmax;
  t = ((t + 31) / 32) * 32;
  return t < 64 ? 64 : (t > 512 ? 512 : t);
}

constexpr size_t kPcr2SmemBudget = 200 * 1024;

template <class MS>
cudaError_t fwd_pcr2_launch(const FwdLaunch* a, cudaStream_t st) {
  if (!a) return preload((const void*)fwd_pcr2_kernel<MS>);
  const int Lmax = (a->nb + a->grid - 1) / a->grid;
  const int c = a->nc < a->nt ? a->nc : a->nt;
  const size_t ws = pcr2_ws_doubles<MS>(c, Lmax);
  const size_t ocs = ((MS::NCONST + 1) / 2) * 2;
  const bool in_smem = (ocs + ws) * 8 <= kPcr2SmemBudget;
  const int smem = (int)((ocs + (in_smem ? ws : 0)) * 8);
  CKO_ALLOW_FULL_SMEM(fwd_pcr2_kernel<MS>);
  FwdLaunch copy = *a;
  int flag = in_smem ? 1 : 0;
  void* args[] = {&copy, &flag};
  return launch_persistent((const void*)fwd_pcr2_kernel<MS>, dim3(a->grid),
                                     dim3(pcr2_threads<MS>(c, Lmax)), args, smem, st);
}

template <class MS>
cudaError_t adj_pcr2_launch(const AdjLaunch* a, cudaStream_t st) {
  if (!a) return preload((const void*)adj_pcr2_kernel<MS>);
  const int Lmax = (a->nb + a->grid - 1) / a->grid;
  const int c = a->nc < a->nt ? a->nc : a->nt;
  const size_t ws = pcr2_ws_doubles<MS>(c, Lmax);
  const size_t ocs = ((MS::NCONST + 1) / 2) * 2;
  const size_t olam = ocs + ((Lmax * MS::N + 1) / 2) * 2;
  const bool in_smem = (olam + ws) * 8 <= kPcr2SmemBudget;
  const int smem = (int)((olam + (in_smem ? ws : 0)) * 8);
  CKO_ALLOW_FULL_SMEM(adj_pcr2_kernel<MS>);
  adj_pcr2_kernel<MS><<<a->grid, pcr2_threads<MS>(c, Lmax), smem, st>>>(*a, in_smem ? 1 : 0);
  return cudaGetLastError();
}

}  // namespace v2
}  // namespace cko
