// cko_pcrw.cuh — generation-2 parallel-cyclic-reduction / hybrid kernels for
// blocks too large for a thread (8 < N <= 24; the north-star MDS chain has
// N = 20), warp-cooperative (strided_solve_into, linalg.cpp:197-255).
//
// One persistent CTA per SM owns a lane range; a chunk's c x L points are
// records in a per-CTA global slab (L2-resident for the shapes used):
//  * factor: the diagonal blocks M = I - dt J (or (I - dt J)^T) are built and
//    LU-factored three per warp by the producer group LU of cko_v2.cuh
//    (rows over 10-lane groups, register resident, the reference's pivot
//    sequence), straight into the records;
//  * sweeps: one warp per (row r, lane) task. The partner row q = r - s (its
//    LU factors, coupling B_q and x_q) is staged in the warp's shared-memory
//    slot; lane i holds row i of B_r in registers and runs the reference's
//    operations on it: the right solve P = B_r M_q^{-1} through U^T, L^T and
//    the permutation (lu_right_solve_mat, linalg.cpp:62-82), x_r -= P x_q
//    (gemv_sub) and B_r <- -(P B_q) (gemm_neg, skipping zero multipliers as
//    the reference does); updated rows go to temporaries and are committed
//    after the sweep, which is the all-at-once update the reduction is defined
//    by (the reference gets it from its descending row order);
//  * finisher: the independent strided chains (one row each after a full
//    reduction) by forward substitution, one thread per chain.
// The couplings start as -I (fill_minus_identity, linalg.cpp:261-266); the
// residual, Newton predicate and adjoint quadrature are those of cko_v2.cuh.
#pragma once

#include "cko_v2.cuh"

namespace cko {
namespace v2 {

// Record: the v2 factor record (LU, 1/U_ii, x in RHS, PERM), then the coupling
// B, its sweep temporary BT and the x temporary XT.
template <int N>
struct WRec {
  static constexpr int B = ((Rec<N>::STRIDE + 1) / 2) * 2;
  static constexpr int BT = B + N * N;
  static constexpr int XT = BT + N * N;
  static constexpr int STRIDE = XT + N + (N & 1);
};

#ifndef CKO_PCRW_ROWS
#define CKO_PCRW_ROWS 64  // knob: records per lane tile (c x lanes; the tile stays in L2, the warps stay busy)
#endif
constexpr int kPcrwRows = CKO_PCRW_ROWS;
__device__ __forceinline__ int pcrw_tile_lanes(int c) { return c >= kPcrwRows ? 1 : kPcrwRows / c; }
constexpr int kPcrwWarps = 12;  // 168 registers per thread (the producer group LU and the sweep rows)

// Per-warp staging slot of the sweep: partner LU, 1/U_ii, perm, B_q, x_q.
template <int N>
struct WSlot {
  static constexpr int LU = 0;
  static constexpr int RD = N * N;
  static constexpr int BQ = RD + N;
  static constexpr int XQ = BQ + N * N;
  static constexpr int PERM = XQ + N;  // N ints + identity flag
  static constexpr int STRIDE = PERM + (N + 2) / 2 + ((N + 2) / 2 & 1);
};


static_assert(Rec<20>::PERM + 11 <= WSlot<20>::STRIDE, "a sweep slot holds a dummy factor record");

template <int N>
__host__ __device__ constexpr int pcrw_smem_doubles(int nconst) {
  return ((nconst + 1) / 2) * 2 + kPcrwWarps * WSlot<N>::STRIDE + kPcrwWarps * Geo<N>::GPW * kPb<N> + 8;
}

// One sweep task: row r reduces against its partner q (records rr, rq).
template <int N>
__device__ inline void pcrw_task(double* __restrict__ rr, const double* __restrict__ rq, double* slot, bool upd_b,
                                 int lane) {
  // stage the partner (coalesced), its B and x
  for (int e = lane; e < N * N; e += 32) {
    slot[WSlot<N>::LU + e] = rq[e];
    slot[WSlot<N>::BQ + e] = rq[WRec<N>::B + e];
  }
  for (int e = lane; e < N; e += 32) {
    slot[WSlot<N>::RD + e] = rq[Rec<N>::RD + e];
    slot[WSlot<N>::XQ + e] = rq[Rec<N>::RHS + e];
  }
  const int* gperm = reinterpret_cast<const int*>(rq + Rec<N>::PERM);
  int* sperm = reinterpret_cast<int*>(slot + WSlot<N>::PERM);
  for (int e = lane; e <= N; e += 32) sperm[e] = gperm[e];
  __syncwarp();
  const double* lu = slot + WSlot<N>::LU;
  const double* rd = slot + WSlot<N>::RD;
  if (lane < N) {
    const int i = lane;
    double w[N];
#pragma unroll
    for (int j = 0; j < N; ++j) w[j] = rr[WRec<N>::B + i * N + j];
    // U^T (lower, non-unit) then L^T (upper, unit)
#pragma unroll
    for (int k = 0; k < N; ++k) {
      double s = w[k];
#pragma unroll
      for (int j = 0; j < k; ++j) s -= lu[j * N + k] * w[j];
      w[k] = s * rd[k];
    }
#pragma unroll
    for (int k = N - 2; k >= 0; --k) {
      double s = w[k];
#pragma unroll
      for (int j = k + 1; j < N; ++j) s -= lu[j * N + k] * w[j];
      w[k] = s;
    }
    if (!sperm[N]) {  // X = Z P: column perm[k] of X is column k of Z (registers indexed statically)
      double z[N];
#pragma unroll
      for (int k = 0; k < N; ++k) z[k] = w[k];
#pragma unroll
      for (int k = 0; k < N; ++k) {
        const int pk = sperm[k];
#pragma unroll
        for (int j = 0; j < N; ++j)
          if (j == pk) w[j] = z[k];
      }
    }
    // gemv_sub: x_r - P x_q (row i)
    double acc = 0.0;
#pragma unroll
    for (int j = 0; j < N; ++j) acc += w[j] * slot[WSlot<N>::XQ + j];
    rr[WRec<N>::XT + i] = rr[Rec<N>::RHS + i] - acc;
    if (upd_b) {  // gemm_neg: B_r <- -(P B_q), row i
      double cr[N];
#pragma unroll
      for (int j = 0; j < N; ++j) cr[j] = 0.0;
#pragma unroll
      for (int k = 0; k < N; ++k) {
        const double av = w[k];
        if (av == 0.0) continue;
        const double* bq = slot + WSlot<N>::BQ + k * N;
#pragma unroll
        for (int j = 0; j < N; ++j) cr[j] -= av * bq[j];
      }
#pragma unroll
      for (int j = 0; j < N; ++j) rr[WRec<N>::BT + i * N + j] = cr[j];
    }
  }
  __syncwarp();
}

// solve_unit_offdiag -> strided_solve_into over the CTA's c x L records (x in RHS).
template <int N>
__device__ void pcrw_solve_cta(double* ws, int c, int L, int nsw_arg, double* slots) {
  const int T = blockDim.x, tid = threadIdx.x, warp = tid >> 5, lane = tid & 31, nw = T >> 5;
  auto rec = [&](int k, int lb) { return ws + (size_t)(k * L + lb) * WRec<N>::STRIDE; };
  double* slot = slots + (size_t)warp * WSlot<N>::STRIDE;
  for (size_t e = tid; e < (size_t)c * L * N * N; e += T) {  // couplings start as -I
    const size_t p = e / (N * N);
    const int ij = (int)(e % (N * N));
    ws[p * WRec<N>::STRIDE + WRec<N>::B + ij] = (ij / N == ij % N) ? -1.0 : 0.0;
  }
  __syncthreads();
  int base = 0;
  for (int bit = 30; bit >= 0; --bit) {
    const int m = 1 << bit;
    if (!(c & m)) continue;
    if (base > 0) {  // fold the solved previous partition through the original coupling
      for (int lb = tid; lb < L; lb += T) {
        double* xr = rec(base, lb) + Rec<N>::RHS;
        const double* xp = rec(base - 1, lb) + Rec<N>::RHS;
        const double* Br = rec(base, lb) + WRec<N>::B;
#pragma unroll 4
        for (int i = 0; i < N; ++i) {
          double s = 0.0;
          for (int j = 0; j < N; ++j) s += Br[i * N + j] * xp[j];
          xr[i] -= s;
        }
      }
      __syncthreads();
    }
    int e = 0;
    while ((1 << e) < m) ++e;
    const int nsw = (nsw_arg < 0) ? e : (nsw_arg < e ? nsw_arg : e);
    for (int sidx = 0; sidx < nsw; ++sidx) {
      const int s = 1 << sidx;
      const int cnt = (m - s) * L;
      for (int idx = warp; idx < cnt; idx += nw) {
        const int r = base + s + idx / L, lb = idx % L, q = r - s;
        pcrw_task<N>(rec(r, lb), rec(q, lb), slot, q - base >= s, lane);
      }
      __syncthreads();
      for (size_t e2 = tid; e2 < (size_t)cnt * (N * N + N); e2 += T) {  // commit the sweep
        const int idx = (int)(e2 / (N * N + N)), o = (int)(e2 % (N * N + N));
        const int r = base + s + idx / L, lb = idx % L, q = r - s;
        double* rr = rec(r, lb);
        if (o < N)
          rr[Rec<N>::RHS + o] = rr[WRec<N>::XT + o];
        else if (q - base >= s)
          rr[WRec<N>::B + o - N] = rr[WRec<N>::BT + o - N];
      }
      __syncthreads();
    }
    // finish the independent strided chains by forward substitution
    const int stride = 1 << nsw;
    const int nch = stride < m ? stride : m;
    for (int idx = tid; idx < nch * L; idx += T) {
      const int ch = idx / L, lb = idx % L, r0 = base + ch;
      double xp[N];
      double* vs = rec(r0, lb) + WRec<N>::XT;  // per-record scratch for the permuted gather
      {
        double* rr = rec(r0, lb);
        load_vec<N>(rr + Rec<N>::RHS, xp);
        lu_solve_rec<N>(rr, vs, xp);
#pragma unroll
        for (int i = 0; i < N; ++i) rr[Rec<N>::RHS + i] = xp[i];
      }
      for (int r = r0 + stride; r < base + m; r += stride) {
        double* rr = rec(r, lb);
        double v[N];
#pragma unroll
        for (int i = 0; i < N; ++i) {
          double acc = 0.0;
#pragma unroll
          for (int j = 0; j < N; ++j) acc += rr[WRec<N>::B + i * N + j] * xp[j];
          v[i] = rr[Rec<N>::RHS + i] - acc;
        }
        lu_solve_rec<N>(rr, rr + WRec<N>::XT, v);
#pragma unroll
        for (int i = 0; i < N; ++i) rr[Rec<N>::RHS + i] = v[i], xp[i] = v[i];
      }
    }
    __syncthreads();
    base += m;
  }
}

// Records start 16-byte aligned (the v2 record code moves rows as double2): the host sizes the slab with
// pcr2_ws_bound(n) doubles per point, which leaves room for the alignment step.
__device__ inline double* align16(double* p) {
  return reinterpret_cast<double*>((reinterpret_cast<uintptr_t>(p) + 15) & ~uintptr_t(15));
}
template <class MS>
__device__ inline double* pcrw_workspace(const Slab& slab) {
  // after this CTA's residual rows and norms in the forward slab layout
  return align16(slab.base + (size_t)blockIdx.x * slab.doubles + (size_t)slab.Pmax * (MS::N + 1));
}

// ---------------------------------------------------------------------------
// forward (integrate_backward_euler with the PCR / hybrid solver)
// ---------------------------------------------------------------------------
template <class MS>
__global__ void __launch_bounds__(32 * kPcrwWarps, 1) fwd_pcrw_kernel(FwdLaunch a) {
  constexpr int N = MS::N;
  using Gm = Geo<N>;
  extern __shared__ __align__(16) double smem[];
  __shared__ unsigned s_bcast, s_flags, s_sing;
  double* cs = smem;
  constexpr int OCS = ((MS::NCONST + 1) / 2) * 2;
  double* slots = smem + OCS;
  double* pbs = slots + kPcrwWarps * WSlot<N>::STRIDE;
  MS::load_consts(a.m, cs);
  if (threadIdx.x == 0) s_sing = 0;
  FwdCtx x;
  lane_range(a.nb, x.lb0, x.L);
  x.row = (size_t)a.nb * N;
  double* hr = a.slab.base + (size_t)blockIdx.x * a.slab.doubles;
  double* nrm = hr + (size_t)a.slab.Pmax * N;
  double* ws = pcrw_workspace<MS>(a.slab);
  const bool leader = blockIdx.x == 0 && threadIdx.x == 0;
  const int T = blockDim.x, tid = threadIdx.x, nb = a.nb, warp = tid >> 5, lane = tid & 31;
  const int stage_cap = kPcrwWarps * WSlot<N>::STRIDE;  // residual staging in the idle sweep slots
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
    for (int p = tid; p < c * x.L; p += T) {  // initial iterate: every row at y_start
      const int k = p / x.L, b = x.lb0 + p % x.L;
      double v[N];
      load_vec<N>(a.states + (size_t)step * x.row + (size_t)b * N, v);
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
    unsigned f = residual2<MS>(a, x, cs, hr, nrm, slots, stage_cap, true, &s_flags, a.loss_part ? loss_slot(a) + 1 : nullptr);
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
      // lanes in tiles of ~kPcrwRows records: a tile stays L2-resident through the sweeps
      const int LTW = pcrw_tile_lanes(c);
      for (int l0 = 0; l0 < x.L; l0 += LTW) {
      const int Lt = min(LTW, x.L - l0);
      // assemble M = I - J dt and factor (assemble_factor, integrate.cpp:118-135), x = r: three points per warp
      {
        const GroupLane<N> gr(lane);
        const int P = c * Lt;
        for (int p0 = warp * Gm::GPW; p0 < P; p0 += kPcrwWarps * Gm::GPW) {
          const bool active = p0 + gr.g < P;
          const int p = active ? p0 + gr.g : P - 1;  // inactive groups factor a duplicate, no side effects
          const int k = p / Lt, lb = l0 + p % Lt, b = x.lb0 + lb;
          // inactive groups factor a duplicate point into the warp's idle sweep slot (never the live record)
          double* rec = active ? ws + (size_t)p * WRec<N>::STRIDE : slots + (size_t)warp * WSlot<N>::STRIDE;
          double* pb = pbs + (size_t)(warp * Gm::GPW + gr.g) * kPb<N>;
          const double t = a.times[(size_t)(step + 1 + k) * nb + b];
          const double dt = t - a.times[(size_t)(step + k) * nb + b];
          double y[N];
          load_vec<N>(a.states + (size_t)(step + 1 + k) * x.row + (size_t)b * N, y);
          const double ndt = -dt;
          auto build = [&](double (&mm)[Gm::R][N]) {
#pragma unroll
            for (int q = 0; q < Gm::R; ++q) {
              const int i = gr.gl + q * Gm::G;
              if (i < N) {
                MS::jac_row(a.m, cs, t, y, i, mm[q], b);
#pragma unroll
                for (int j = 0; j < N; ++j) {
                  mm[q][j] = xmul(ndt, mm[q][j]);
                  if (j == i) mm[q][j] = xadd(mm[q][j], 1.0);
                }
              } else {
#pragma unroll
                for (int j = 0; j < N; ++j) mm[q][j] = 0.0;
              }
            }
          };
          const bool ok = factor_block<N, false>(build, build, gr.gl, gr.base, pb, rec);
          if (active) {
            const double* r = hr + (size_t)(k * x.L + lb) * N;
#pragma unroll
            for (int q = 0; q < Gm::R; ++q) {
              const int i = gr.gl + q * Gm::G;
              if (i < N) rec[Rec<N>::RHS + i] = r[i];
            }
            if (!ok && gr.gl == 0) {
              atomicMin(a.sing_key, (unsigned long long)k * nb + b);
              atomicOr(&s_sing, 1u);
            }
          }
        }
      }
      __syncthreads();
      pcrw_solve_cta<N>(ws, c, Lt, a.solver == 1 ? -1 : a.n_switch, slots);
      for (int p = tid; p < c * Lt; p += T) {  // yy -= x
        const int k = p / Lt, b = x.lb0 + l0 + p % Lt;
        double* yy = a.states + (size_t)(step + 1 + k) * x.row + (size_t)b * N;
        const double* xv = ws + (size_t)p * WRec<N>::STRIDE + Rec<N>::RHS;
#pragma unroll
        for (int i = 0; i < N; ++i) yy[i] -= xv[i];
      }
      __syncthreads();
      }  // lane tiles
      const unsigned fl = s_sing ? FLAG_SINGULAR : 0u;
      f = residual2<MS>(a, x, cs, hr, nrm, slots, stage_cap, false, &s_flags, a.loss_part ? loss_slot(a) + 1 : nullptr) | fl;
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
// adjoint (be_chunk_core with the PCR / hybrid solver, adjoint.cpp:49-127)
// ---------------------------------------------------------------------------
template <class MS>
__global__ void __launch_bounds__(32 * kPcrwWarps, 1) adj_pcrw_kernel(AdjLaunch a) {
  constexpr int N = MS::N;
  using Gm = Geo<N>;
  extern __shared__ __align__(16) double smem[];
  double* cs = smem;
  constexpr int OCS = ((MS::NCONST + 1) / 2) * 2;
  double* slots = smem + OCS;
  double* pbs = slots + kPcrwWarps * WSlot<N>::STRIDE;
  MS::load_consts(a.m, cs);
  int lb0, L;
  lane_range(a.nb, lb0, L);
  const int T = blockDim.x, tid = threadIdx.x, nb = a.nb, warp = tid >> 5, lane = tid & 31;
  const size_t row = (size_t)nb * N;
  const double Lval = adj_loss_value(a);
  double* ws = align16(a.slab.base + (size_t)blockIdx.x * a.slab.doubles);
  double* lam = a.lambda + (size_t)lb0 * N;  // the carry (global, this CTA's lanes)
  for (int i = tid; i < L * N; i += T) lam[i] = 0.0;
  __syncthreads();
  int step_hi = a.nt;
  unsigned long long ord = 0;
  while (step_hi >= 1) {
    const int c = min(a.nc, step_hi);
    const int LTW = pcrw_tile_lanes(c);
    for (int l0 = 0; l0 < L; l0 += LTW) {  // lanes in tiles: the tile's records stay L2-resident
    const int Lt = min(LTW, L - l0);
    // gather + J + rhs_r = dL + dt J^T lambda + transposed LU (adjoint.cpp:53-81), three points per warp
    {
      const GroupLane<N> gr(lane);
      const int P = c * Lt;
      for (int p0 = warp * Gm::GPW; p0 < P; p0 += kPcrwWarps * Gm::GPW) {
        const bool active = p0 + gr.g < P;
        const int p = active ? p0 + gr.g : P - 1;
        const int r = p / Lt, lb = l0 + p % Lt, b = lb0 + lb, m = step_hi - r;
        double* rec = active ? ws + (size_t)p * WRec<N>::STRIDE : slots + (size_t)warp * WSlot<N>::STRIDE;
        double* pb = pbs + (size_t)(warp * Gm::GPW + gr.g) * kPb<N>;
        const double t = a.times[(size_t)m * nb + b];
        const double dt = t - a.times[(size_t)(m - 1) * nb + b];
        double y[N];
        load_vec<N>(a.states + (size_t)m * row + (size_t)b * N, y);
        const double* lc = lam + (size_t)lb * N;
        // the rows of M^T this lane holds are the columns i of I - dt J; the rhs entries come with them
        auto build = [&](double (&mt)[Gm::R][N]) {
          double jr[N];
#pragma unroll
          for (int q = 0; q < Gm::R; ++q)
#pragma unroll
            for (int j = 0; j < N; ++j) mt[q][j] = 0.0;
          double tmp[Gm::R];
#pragma unroll
          for (int q = 0; q < Gm::R; ++q) tmp[q] = 0.0;
#pragma unroll
          for (int jrow = 0; jrow < N; ++jrow) {  // J row jrow gives M^T(i, jrow) for every held i
            MS::jac_row(a.m, cs, t, y, jrow, jr, b);
            const double lj = lc[jrow];
#pragma unroll
            for (int q = 0; q < Gm::R; ++q) {
              const int i = gr.gl + q * Gm::G;
              double v = 0.0;
#pragma unroll
              for (int j = 0; j < N; ++j) v = j == i ? jr[j] : v;
              if (i < N) {
                tmp[q] += v * lj;  // (J^T lambda)_i, j ascending (gemv_transpose)
                mt[q][jrow] = (jrow == i) ? 1.0 - dt * v : -dt * v;
              }
            }
          }
          if (active) {
#pragma unroll
            for (int q = 0; q < Gm::R; ++q) {
              const int i = gr.gl + q * Gm::G;
              if (i < N) {
                const double dl = a.dL ? a.dL[(size_t)m * row + (size_t)b * N + i] : (Lval > 0.0 ? y[i] / Lval : 0.0);
                rec[Rec<N>::RHS + i] = dl + dt * tmp[q];
              }
            }
          }
        };
        auto rows = [&](double (&mt)[Gm::R][N]) {  // entries of M^T as rows of I - dt J (exact singular test)
#pragma unroll
          for (int q = 0; q < Gm::R; ++q) {
            const int i = gr.gl + q * Gm::G;
            if (i < N) {
              MS::jac_row(a.m, cs, t, y, i, mt[q], b);
#pragma unroll
              for (int j = 0; j < N; ++j) mt[q][j] = (j == i) ? 1.0 - dt * mt[q][j] : -dt * mt[q][j];
            } else {
#pragma unroll
              for (int j = 0; j < N; ++j) mt[q][j] = 0.0;
            }
          }
        };
        const bool ok = factor_block<N, true>(build, rows, gr.gl, gr.base, pb, rec);
        if (!ok && active && gr.gl == 0)
          atomicMin(a.sing_key, ord * (unsigned long long)a.nc * nb + (unsigned long long)r * nb + b);
      }
    }
    __syncthreads();
    pcrw_solve_cta<N>(ws, c, Lt, a.solver == 1 ? -1 : a.n_switch, slots);
    // quadrature weights w_r = (carry + delta_r) dt_r (adjoint.cpp:103-113)
    for (int p = tid; p < c * Lt; p += T) {
      const int r = p / Lt, lb = l0 + p % Lt, b = lb0 + lb, m = step_hi - r;
      const double dt = a.times[(size_t)m * nb + b] - a.times[(size_t)(m - 1) * nb + b];
      const double* d = ws + (size_t)p * WRec<N>::STRIDE + Rec<N>::RHS;
      const double* lc = lam + (size_t)lb * N;
      double* w = a.wq + (size_t)m * row + (size_t)b * N;
#pragma unroll
      for (int i = 0; i < N; ++i) w[i] = (lc[i] + d[i]) * dt;
    }
    __syncthreads();
    for (int idx = tid; idx < Lt * N; idx += T)  // new carry (adjoint.cpp:121-126)
      lam[(size_t)l0 * N + idx] += ws[(size_t)((c - 1) * Lt + idx / N) * WRec<N>::STRIDE + Rec<N>::RHS + idx % N];
    __syncthreads();
    }  // lane tiles
    step_hi -= c;
    ++ord;
  }
}

template <class MS>
cudaError_t fwd_pcrw_launch(const FwdLaunch* a, cudaStream_t st) {
  if (!a) return preload((const void*)fwd_pcrw_kernel<MS>);
  const int smem = pcrw_smem_doubles<MS::N>(MS::NCONST) * 8;
  CKO_ALLOW_FULL_SMEM(fwd_pcrw_kernel<MS>);
  FwdLaunch copy = *a;
  void* args[] = {&copy};
  return launch_persistent((const void*)fwd_pcrw_kernel<MS>, dim3(a->grid), dim3(32 * kPcrwWarps), args, smem, st);
}

template <class MS>
cudaError_t adj_pcrw_launch(const AdjLaunch* a, cudaStream_t st) {
  if (!a) return preload((const void*)adj_pcrw_kernel<MS>);
  const int smem = pcrw_smem_doubles<MS::N>(MS::NCONST) * 8;
  CKO_ALLOW_FULL_SMEM(adj_pcrw_kernel<MS>);
  adj_pcrw_kernel<MS><<<a->grid, 32 * kPcrwWarps, smem, st>>>(*a);
  return cudaGetLastError();
}

}  // namespace v2
}  // namespace cko
