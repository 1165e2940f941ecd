// cko_impl.cuh — sm_100a kernels (templates; instantiated per model in cko_inst_*.cu) of the chunked backward-Euler path.
//
//  fwd_kernel  : the whole forward integration (integrate.cpp:321-369) in one
//                cooperative persistent launch. CTAs own disjoint lane ranges;
//                per chunk they run the Newton loop (integrate.cpp:192-255):
//                fused residual + lane norms, Jacobian -> I - J dt -> LU, then
//                Thomas (integrate.cpp:208-231) or PCR/hybrid
//                (linalg.cpp:197-255) on the -I coupled block-bidiagonal
//                system. The all-lanes convergence predicate
//                (integrate.cpp:176-182) is the only cross-CTA (and, sharded,
//                cross-GPU) coupling: one flag OR-reduction per iteration.
//  adj_kernel  : the discrete adjoint (adjoint.cpp:49-127, 263-297), lane
//                parallel with no grid barrier at all; it emits the
//                quadrature weights w_m = lambda_m dt_m.
//  vjp_kernel  : the parameter product sum w . dh/dp (ode_model.cpp:135-153)
//                over every (step, lane) point, reduced deterministically.
//  loss / solve kernels: Frobenius loss (adjoint.cpp:196-221) and the
//                standalone block-bidiagonal solvers (linalg.cpp:307-344).
#pragma once
#include <cfloat>
#include <climits>

#include "cko_kernels.cuh"
#include "cko_linalg.cuh"
#include "cko_eval.cuh"

namespace cko {

constexpr int kMaxThreads = 256;

// Views of one CTA's slab.
struct CtaWs {
  int n, S;
  double *yy, *hr, *lu, *nrm, *B, *Bn, *Pb, *xt;
  int* piv;
  __device__ SVec v(double* a, int p) const { return {a + p, S}; }
  __device__ SBlk b(double* a, int p) const { return {a + p, S, n}; }
  __device__ SPiv pv(int p) const { return {piv + p, S}; }
};

__device__ inline CtaWs make_ws(const Slab& s, int n, bool pcr) {
  CtaWs w;
  w.n = n;
  w.S = s.Pmax;
  const size_t S = (size_t)s.Pmax;
  double* base = s.base + (size_t)blockIdx.x * s.doubles;
  w.yy = base;
  w.hr = base + (size_t)n * S;
  w.lu = base + 2 * (size_t)n * S;
  w.nrm = w.lu + (size_t)n * n * S;
  w.B = w.Bn = w.Pb = w.xt = nullptr;
  if (pcr) {
    w.B = w.nrm + S;
    w.Bn = w.B + (size_t)n * n * S;
    w.Pb = w.Bn + (size_t)n * n * S;
    w.xt = w.Pb + (size_t)n * n * S;
  }
  w.piv = s.pbase + (size_t)blockIdx.x * s.ints;
  return w;
}

// -I, the implicit coupling block of the stepper system.
struct NegI {
  __device__ double operator()(int i, int j) const { return i == j ? -1.0 : 0.0; }
};
struct CVec {  // contiguous read-only vector
  const double* p;
  __device__ double operator[](int i) const { return p[i]; }
};
struct MVec {  // contiguous mutable vector
  double* p;
  __device__ double& operator[](int i) const { return p[i]; }
};

__device__ inline void lane_range(int nb, int& lb0, int& L) {
  const int G = gridDim.x, c = blockIdx.x;
  lb0 = (int)((long long)nb * c / G);
  L = (int)((long long)nb * (c + 1) / G) - lb0;
}

// ---------------------------------------------------------------------------
// PCR / hybrid on one CTA's lanes (strided_solve_into, linalg.cpp:197-255),
// rows of each power-of-two partition processed in parallel. B[r] holds the
// coupling of row r to row r-1; `unit` means every coupling is -I and B is
// only materialised once a sweep writes it. x lives in w.hr.
// ---------------------------------------------------------------------------
template <class BR, class BQ>
__device__ inline void pcr_point(const CtaWs& w, int pr, int pq, const BR& Br, const BQ& Bq, bool updB) {
  const int n = w.n;
  SBlk P = w.b(w.Pb, pr);
  for (int i = 0; i < n; ++i)
    for (int j = 0; j < n; ++j) P(i, j) = Br(i, j);
  lu_right_solve(w.b(w.lu, pq), w.pv(pq), n, P);
  gemv_sub_into(P, w.v(w.hr, pq), w.v(w.hr, pr), w.v(w.xt, pr), n);
  if (updB) gemm_neg(P, Bq, w.b(w.Bn, pr), n);
}

__device__ inline void cta_pcr(const CtaWs& w, int c, int L, int n_switch, bool unit) {
  const int T = blockDim.x, tid = threadIdx.x, n = w.n;
  int base = 0;
  for (int bit = 30; bit >= 0; --bit) {
    const int m = 1 << bit;
    if (!(c & m)) continue;
    if (base > 0) {
      for (int lb = tid; lb < L; lb += T) {
        const int pr = base * L + lb, pp = (base - 1) * L + lb;
        if (unit)
          gemv_sub_into(NegI{}, w.v(w.hr, pp), w.v(w.hr, pr), w.v(w.hr, pr), n);
        else
          gemv_sub_into(w.b(w.B, pr), w.v(w.hr, pp), w.v(w.hr, pr), w.v(w.hr, pr), n);
      }
      __syncthreads();
    }
    int e = 0;
    while ((1 << e) < m) ++e;
    const int nsw = (n_switch < 0) ? e : (n_switch < e ? n_switch : e);
    for (int sidx = 0; sidx < nsw; ++sidx) {
      const int s = 1 << sidx;
      const int cnt = (m - s) * L;
      for (int idx = tid; idx < cnt; idx += T) {
        const int r = base + s + idx / L, lb = idx % L, q = r - s;
        const int pr = r * L + lb, pq = q * L + lb;
        const bool updB = (q - base >= s);
        if (unit && sidx == 0)
          pcr_point(w, pr, pq, NegI{}, NegI{}, updB);
        else
          pcr_point(w, pr, pq, w.b(w.B, pr), w.b(w.B, pq), updB);
      }
      __syncthreads();
      for (int idx = tid; idx < cnt; idx += T) {
        const int r = base + s + idx / L, lb = idx % L, q = r - s;
        const int pr = r * L + lb;
        SVec x = w.v(w.hr, pr), xt = w.v(w.xt, pr);
        for (int i = 0; i < n; ++i) x[i] = xt[i];
        if (q - base >= s) {
          SBlk Bd = w.b(w.B, pr), Bs = w.b(w.Bn, pr);
          for (int i = 0; i < n; ++i)
            for (int j = 0; j < n; ++j) Bd(i, j) = Bs(i, j);
        }
      }
      __syncthreads();
    }
    const int stride = 1 << nsw;
    const int nch = stride < m ? stride : m;
    for (int idx = tid; idx < nch * L; idx += T) {
      const int ch = idx / L, lb = idx % L, r0 = base + ch;
      lu_solve(w.b(w.lu, r0 * L + lb), w.pv(r0 * L + lb), n, w.v(w.hr, r0 * L + lb));
      for (int r = r0 + stride; r < base + m; r += stride) {
        const int pr = r * L + lb, pp = (r - stride) * L + lb;
        if (unit && nsw == 0)
          gemv_sub_into(NegI{}, w.v(w.hr, pp), w.v(w.hr, pr), w.v(w.hr, pr), n);
        else
          gemv_sub_into(w.b(w.B, pr), w.v(w.hr, pp), w.v(w.hr, pr), w.v(w.hr, pr), n);
        lu_solve(w.b(w.lu, pr), w.pv(pr), n, w.v(w.hr, pr));
      }
    }
    __syncthreads();
    base += m;
  }
}

// Thomas with -I couplings (thomas_unit_into, linalg.cpp:164-175), one
// thread per lane; `sub` additionally applies yy -= x (integrate.cpp:222-230).
__device__ inline void cta_thomas_unit(const CtaWs& w, int c, int L, bool sub) {
  const int n = w.n;
  for (int lb = threadIdx.x; lb < L; lb += blockDim.x) {
    for (int k = 0; k < c; ++k) {
      const int p = k * L + lb;
      SVec x = w.v(w.hr, p);
      if (k > 0) {
        SVec prev = w.v(w.hr, p - L);
        for (int i = 0; i < n; ++i) x[i] += prev[i];
      }
      lu_solve(w.b(w.lu, p), w.pv(p), n, x);
      if (sub) {
        SVec y = w.v(w.yy, p);
        for (int i = 0; i < n; ++i) y[i] -= x[i];
      }
    }
  }
}

// ---------------------------------------------------------------------------
// forward
// ---------------------------------------------------------------------------

// Fused rate + residual + lane norms (rate_residual_norms, integrate.cpp:64-95).
template <class MD>
__device__ unsigned residual_phase(const FwdLaunch& a, const CtaWs& w, int step, int c, int L, int lb0,
                                   bool first, unsigned* s_flags) {
  const int nb = a.nb, n = w.n, T = blockDim.x, tid = threadIdx.x;
  const size_t row = (size_t)nb * n;
  for (int p = tid; p < c * L; p += T) {
    const int k = p / L, lb = p % L, b = lb0 + lb;
    const double t = a.times[(size_t)(step + 1 + k) * nb + b];
    const double dt = a.dts ? a.dts[(size_t)(step + k) * nb + b] : t - a.times[(size_t)(step + k) * nb + b];
    SVec y = w.v(w.yy, p), h = w.v(w.hr, p);
    MD::rate(a.m, t, y, h, b);
    double s = 0.0;
    if (k == 0) {
      const double* ym = a.states + (size_t)step * row + (size_t)b * n;
      for (int i = 0; i < n; ++i) {
        const double v = xsub(xsub(y[i], ym[i]), xmul(h[i], dt));
        h[i] = v;
        s = xadd(s, xmul(v, v));
      }
    } else {
      SVec ym = w.v(w.yy, p - L);
      for (int i = 0; i < n; ++i) {
        const double v = xsub(xsub(y[i], ym[i]), xmul(h[i], dt));
        h[i] = v;
        s = xadd(s, xmul(v, v));
      }
    }
    w.nrm[p] = s;
  }
  if (tid == 0) *s_flags = 0;
  __syncthreads();
  unsigned f = 0;
  for (int lb = tid; lb < L; lb += T) {
    const int b = lb0 + lb;
    double acc = 0.0;
    for (int k = 0; k < c; ++k) acc = xadd(acc, w.nrm[k * L + lb]);
    const double rn = sqrt(acc);
    double r0v;
    if (first) {
      a.r0[b] = rn;
      r0v = rn;
    } else {
      r0v = a.r0[b];
    }
    a.rn[b] = rn;
    if (!isfinite(rn)) f |= FLAG_NON_FINITE;
    if (!(rn <= a.tol_a || rn <= xmul(a.tol_r, r0v))) f |= FLAG_NOT_CONVERGED;
  }
  if (f) atomicOr(s_flags, f);
  __syncthreads();
  return *s_flags;
}

// Jacobian -> M = I - J dt -> LU (integrate.cpp:118-135, :213-221).
template <class MD>
__device__ unsigned jac_lu_phase(const FwdLaunch& a, const CtaWs& w, int step, int c, int L, int lb0) {
  const int nb = a.nb, n = w.n, T = blockDim.x;
  unsigned f = 0;
  for (int p = threadIdx.x; p < c * L; p += T) {
    const int k = p / L, lb = p % L, b = lb0 + lb;
    const double t = a.times[(size_t)(step + 1 + k) * nb + b];
    const double dt = a.dts ? a.dts[(size_t)(step + k) * nb + b] : t - a.times[(size_t)(step + k) * nb + b];
    SBlk J = w.b(w.lu, p);
    SVec y = w.v(w.yy, p);
    model_jacobian<MD>(a.m, t, y, J, b);
    const double ndt = -dt;
    for (int i = 0; i < n; ++i)
      for (int j = 0; j < n; ++j) J(i, j) = xmul(ndt, J(i, j));
    for (int i = 0; i < n; ++i) J(i, i) = xadd(J(i, i), 1.0);
    if (!lu_factor(J, w.pv(p), n)) {
      atomicMin(a.sing_key, (unsigned long long)k * nb + b);
      f |= FLAG_SINGULAR;
    }
  }
  return f;
}

enum : int { INFO_OK = 0, INFO_SINGULAR = 1, INFO_DIVERGED = 2, INFO_NONFINITE0 = 3, INFO_TIMEOUT = 4 };

template <class MD>
__global__ void __launch_bounds__(kMaxThreads) fwd_kernel(FwdLaunch a) {
  __shared__ unsigned s_bcast, s_flags;
  const int nb = a.nb, n = a.m.n, T = blockDim.x, tid = threadIdx.x;
  int lb0, L;
  lane_range(nb, lb0, L);
  const bool pcr = a.solver != 0;
  const int nsw_arg = a.solver == 1 ? -1 : a.n_switch;
  CtaWs w = make_ws(a.slab, n, pcr);
  const size_t row = (size_t)nb * n;
  const bool leader = blockIdx.x == 0 && tid == 0;
  int step = 0, chunk = 0;
  while (step < a.nt) {
    const int c = min(a.nc, a.nt - step);
    const int P = c * L;
    for (int p = tid; p < P; p += T) {  // initial iterate: every row at y_start
      const int k = p / L, b = lb0 + p % L;
      const double* src = a.states + (size_t)step * row + (size_t)b * n;
      SVec y = w.v(w.yy, p);
      if (a.dy_init) {
        const double* d = a.dy_init + ((size_t)k * nb + b) * n;
        for (int i = 0; i < n; ++i) y[i] = src[i] + d[i];
      } else {
        for (int i = 0; i < n; ++i) y[i] = src[i];
      }
    }
    __syncthreads();
    int it = 0;
    unsigned f = residual_phase<MD>(a, w, step, c, L, lb0, true, &s_flags);
    f = grid_reduce_or(a.gs, a.grp, f, a.budget_ns, &s_bcast);
    if (f & (FLAG_TIMEOUT | FLAG_NON_FINITE)) {
      if (leader) a.info[0] = (f & FLAG_TIMEOUT) ? INFO_TIMEOUT : INFO_DIVERGED, a.info[1] = step + 1, a.info[2] = 0;
      return;
    }
    while (f & FLAG_NOT_CONVERGED) {
      if (it == a.max_iter) {
        if (leader) a.info[0] = INFO_DIVERGED, a.info[1] = step + 1, a.info[2] = a.max_iter;
        return;
      }
      ++it;
      unsigned fl = jac_lu_phase<MD>(a, w, step, c, L, lb0);
      __syncthreads();
      if (!pcr) {
        cta_thomas_unit(w, c, L, true);
      } else {
        cta_pcr(w, c, L, nsw_arg, true);
        for (int p = tid; p < P; p += T) {
          SVec y = w.v(w.yy, p), x = w.v(w.hr, p);
          for (int i = 0; i < n; ++i) y[i] -= x[i];
        }
      }
      __syncthreads();
      fl |= residual_phase<MD>(a, w, step, c, L, lb0, false, &s_flags);
      f = grid_reduce_or(a.gs, a.grp, fl, a.budget_ns, &s_bcast);
      if (f & (FLAG_TIMEOUT | FLAG_SINGULAR | FLAG_NON_FINITE)) {
        if (leader) {
          a.info[0] = (f & FLAG_TIMEOUT) ? INFO_TIMEOUT : (f & FLAG_SINGULAR) ? INFO_SINGULAR : INFO_DIVERGED;
          a.info[1] = step + 1;
          a.info[2] = it;
        }
        return;
      }
    }
    for (int p = tid; p < P; p += T) {
      const int k = p / L, b = lb0 + p % L;
      double* dst = a.states + (size_t)(step + 1 + k) * row + (size_t)b * n;
      SVec y = w.v(w.yy, p);
      for (int i = 0; i < n; ++i) dst[i] = y[i];
    }
    if (leader) a.iters[chunk] = it;
    step += c;
    ++chunk;
    __syncthreads();
  }
  if (leader) a.info[3] = chunk;
}

// ---------------------------------------------------------------------------
// adjoint
// ---------------------------------------------------------------------------
template <class MD>
__global__ void __launch_bounds__(kMaxThreads) adj_kernel(AdjLaunch a) {
  const int nb = a.nb, n = a.m.n, T = blockDim.x, tid = threadIdx.x;
  int lb0, L;
  lane_range(nb, lb0, L);
  const bool pcr = a.solver != 0;
  const int nsw_arg = a.solver == 1 ? -1 : a.n_switch;
  CtaWs w = make_ws(a.slab, n, pcr);
  const size_t row = (size_t)nb * n;
  const double Lval = a.loss ? *a.loss : 0.0;
  if (!a.keep_lambda)
    for (int idx = tid; idx < L * n; idx += T) a.lambda[(size_t)lb0 * n + idx] = 0.0;
  __syncthreads();
  int step_hi = a.nt;
  unsigned long long ord = 0;
  while (step_hi >= 1) {
    const int c = min(a.nc, step_hi);
    const int P = c * L;
    // gather + J + rhs_r = jump + dt J^T lambda + transposed LU (adjoint.cpp:136-149, 53-81)
    for (int p = tid; p < P; p += T) {
      const int r = p / L, lb = p % L, b = lb0 + lb, m = step_hi - r;
      const double* ym = a.states + (size_t)m * row + (size_t)b * n;
      CVec y{ym};
      const double t = a.times[(size_t)m * nb + b];
      const double dt = t - a.times[(size_t)(m - 1) * nb + b];
      SBlk J = w.b(w.lu, p);
      model_jacobian<MD>(a.m, t, y, J, b);
      SVec rhs = w.v(w.hr, p);
      if (a.dL) {
        const double* g = a.dL + (size_t)m * row + (size_t)b * n;
        for (int i = 0; i < n; ++i) rhs[i] = g[i];
      } else {
        for (int i = 0; i < n; ++i) rhs[i] = Lval > 0.0 ? ym[i] / Lval : 0.0;
      }
      const double* lam = a.lambda + (size_t)b * n;
      for (int i = 0; i < n; ++i) {
        double tmp = 0.0;
        for (int j = 0; j < n; ++j) tmp += J(j, i) * lam[j];
        rhs[i] += dt * tmp;
      }
      for (int i = 0; i < n; ++i) {
        for (int q = i + 1; q < n; ++q) {
          const double v = J(i, q);
          J(i, q) = -dt * J(q, i);
          J(q, i) = -dt * v;
        }
        J(i, i) = 1.0 - dt * J(i, i);
      }
      if (!lu_factor(J, w.pv(p), n))
        atomicMin(a.sing_key, ord * (unsigned long long)a.nc * nb + (unsigned long long)r * nb + b);
    }
    __syncthreads();
    if (!pcr)
      cta_thomas_unit(w, c, L, false);
    else
      cta_pcr(w, c, L, nsw_arg, true);
    __syncthreads();
    // quadrature weights w_r = (carry + delta_r) dt_r (adjoint.cpp:90-113)
    for (int p = tid; p < P; p += T) {
      const int r = p / L, lb = p % L, b = lb0 + lb, m = step_hi - r;
      const double dt = a.times[(size_t)m * nb + b] - a.times[(size_t)(m - 1) * nb + b];
      const double* lam = a.lambda + (size_t)b * n;
      SVec d = w.v(w.hr, p);
      double* out = a.wq + (size_t)m * row + (size_t)b * n;
      for (int i = 0; i < n; ++i) out[i] = (lam[i] + d[i]) * dt;
    }
    __syncthreads();
    for (int idx = tid; idx < L * n; idx += T) {  // new carry (adjoint.cpp:121-126)
      const int lb = idx / n, i = idx % n;
      a.lambda[(size_t)(lb0 + lb) * n + i] += w.hr[(size_t)i * w.S + (c - 1) * L + lb];
    }
    __syncthreads();
    step_hi -= c;
    ++ord;
  }
}

// ---------------------------------------------------------------------------
// parameter VJP: grad = sum over (m >= 1, b) of w_m . dh/dp(y_m, t_m)
// ---------------------------------------------------------------------------
constexpr int kVjpBlocks = 296;

__host__ __device__ inline void lane_segment(const DevModel& m, int& lo, int& hi) {
  if (m.kind == 3) {  // MDS: T_b
    lo = 3 * m.nu + 1;
    hi = lo + m.nbm;
  } else if (m.kind == 4) {  // Chaboche: eps_a_b
    lo = 6 + 2 * m.nu;
    hi = lo + m.nbm;
  } else if (m.kind == 6) {  // Neuron: I_a per lane
    lo = 14 * m.nu;
    hi = lo + m.nbm;
  } else {
    lo = hi = m.np;
  }
}

template <int NPS>
struct LocalAcc {
  double sh[NPS];
  int lo, hi;
  double* lane_row;
  __device__ void add(int j, double v) { sh[j < lo ? j : j - (hi - lo)] += v; }
  __device__ void lane_add(int j, double v) { lane_row[j] += v; }
};

template <class MD, int NPS>
__global__ void __launch_bounds__(256) vjp_kernel(DevModel m, const double* states, const double* times,
                                                  const double* wq, int nb, int nt, double* part) {
  __shared__ double red[8][NPS > 64 ? 64 : NPS];
  const int n = m.n, T = blockDim.x, tid = threadIdx.x;
  const size_t row = (size_t)nb * n;
  double* prow = part + (size_t)blockIdx.x * m.np;
  for (int j = tid; j < m.np; j += T) prow[j] = 0.0;
  __syncthreads();
  LocalAcc<NPS> acc;
  lane_segment(m, acc.lo, acc.hi);
  acc.lane_row = prow;
  const int nps = m.np - (acc.hi - acc.lo);
  for (int j = 0; j < NPS; ++j) acc.sh[j] = 0.0;
  for (int mm = 1 + blockIdx.x; mm <= nt; mm += gridDim.x)
    for (int b = tid; b < nb; b += T) {
      CVec y{states + (size_t)mm * row + (size_t)b * n};
      CVec wv{wq + (size_t)mm * row + (size_t)b * n};
      MD::vjp(m, times[(size_t)mm * nb + b], y, wv, acc, b);
    }
  // deterministic block reduction of the shared-parameter accumulators
  const int warp = tid / 32, lane = tid % 32, nw = T / 32;
  constexpr int CH = NPS > 64 ? 64 : NPS;
  for (int j0 = 0; j0 < nps; j0 += CH) {
    for (int jj = 0; jj < CH && j0 + jj < nps; ++jj) {
      double v = acc.sh[j0 + jj];
      for (int o = 16; o > 0; o >>= 1) v += __shfl_down_sync(0xffffffffu, v, o);
      if (lane == 0) red[warp][jj] = v;
    }
    __syncthreads();
    for (int jj = tid; jj < CH && j0 + jj < nps; jj += T) {
      double s = 0.0;
      for (int q = 0; q < nw; ++q) s += red[q][jj];
      const int jc = j0 + jj;
      const int j = jc < acc.lo ? jc : jc + (acc.hi - acc.lo);
      prow[j] += s;
    }
    __syncthreads();
  }
}

// ---------------------------------------------------------------------------
// public single-chunk ops (integrate.cpp:269-297): thread per point (k, b)
// ---------------------------------------------------------------------------
struct PBlk {
  double* p;
  int n;
  __device__ __forceinline__ double& operator()(int i, int j) const { return p[i * n + j]; }
};

// op 0 chunk_residual: out(k) = dy(k) - dy(k-1) - h(y_start + dy(k), t(k)) dt(k) (residual_into,
// integrate.cpp:37-56), flags |= 1 when h is not finite. op 1 chunk_jacobian: out(k) = I - J dt
// (jacobian_into, integrate.cpp:100-113), flags |= 1 when J is not finite (jacobian_state,
// ode_model.cpp:126-133). yyb: (c, nb, n) scratch for y_start + dy.
template <class MD>
__global__ void chunk_op_kernel(DevModel m, int op, const double* __restrict__ ys, const double* __restrict__ dy,
                                const double* __restrict__ t, const double* __restrict__ dt, int c, int nb,
                                double* yyb, double* out, unsigned* flags) {
  const int n = m.n;
  for (int p = blockIdx.x * blockDim.x + threadIdx.x; p < c * nb; p += gridDim.x * blockDim.x) {
    const int k = p / nb, b = p % nb;
    double* yy = yyb + (size_t)p * n;
    const double* d = dy + (size_t)p * n;
    for (int i = 0; i < n; ++i) yy[i] = xadd(ys[(size_t)b * n + i], d[i]);
    const double dtv = dt[p];
    bool fin = true;
    if (op == 0) {
      double* h = out + (size_t)p * n;
      MD::rate(m, t[p], yy, h, b);
      for (int i = 0; i < n; ++i) fin &= isfinite(h[i]);
      for (int i = 0; i < n; ++i)
        h[i] = k == 0 ? xsub(d[i], xmul(h[i], dtv)) : xsub(xsub(d[i], d[i - (ptrdiff_t)nb * n]), xmul(h[i], dtv));
    } else {
      PBlk J{out + (size_t)p * n * n, n};
      model_jacobian<MD>(m, t[p], yy, J, b);
      for (int e = 0; e < n * n; ++e) fin &= isfinite(J.p[e]);
      for (int e = 0; e < n * n; ++e) J.p[e] = xmul(-dtv, J.p[e]);
      for (int i = 0; i < n; ++i) J(i, i) = xadd(J(i, i), 1.0);
    }
    if (!fin) atomicOr(flags, 1u);
  }
}

// ---------------------------------------------------------------------------
// forward Euler scheme: thread per lane, steps in order
// ---------------------------------------------------------------------------
// integrate_forward_euler (integrate.cpp:371-407): y_s = y_{s-1} + h(y_{s-1}, t_{s-1}) dt_s with the
// reference's roundings; *bad = the first step whose state is not finite (min over lanes).
template <class MD>
__global__ void fe_forward_kernel(DevModel m, double* states, const double* times, int nb, int nt, double* hbuf,
                                  int* bad) {
  const int n = m.n;
  const size_t row = (size_t)nb * n;
  for (int b = blockIdx.x * blockDim.x + threadIdx.x; b < nb; b += gridDim.x * blockDim.x) {
    MVec h{hbuf + (size_t)b * n};
    int first_bad = INT_MAX;
    for (int s = 1; s <= nt; ++s) {
      const double* yp = states + (size_t)(s - 1) * row + (size_t)b * n;
      double* y = states + (size_t)s * row + (size_t)b * n;
      const double tp = times[(size_t)(s - 1) * nb + b];
      const double dt = times[(size_t)s * nb + b] - tp;
      MD::rate(m, tp, CVec{yp}, h, b);
      bool fin = true;
      for (int i = 0; i < n; ++i) {
        const double v = xadd(yp[i], xmul(h[i], dt));
        y[i] = v;
        fin &= isfinite(v);
      }
      if (!fin && s < first_bad) first_bad = s;
    }
    if (first_bad != INT_MAX) atomicMin(bad, first_bad);
  }
}

// The forward-Euler discrete adjoint (fe_chunk_core, adjoint.cpp:157-188), per lane from the top:
// lambda += jump_m; w_m = lambda dt_m; lambda += dt_m J(y_{m-1}, t_{m-1})^T lambda (gemv_transpose's
// order, adjoint.cpp:38-45). No solve. w_m goes to wq row m; the parameter product is evaluated at
// (y_{m-1}, t_{m-1}) by the VJP kernels on row-shifted views. *bad |= 1 for a non-finite Jacobian
// (jacobian_state, ode_model.cpp:126-133). Jb (nb, n, n) and tmp (nb, n) are scratch.
template <class MD>
__global__ void fe_adjoint_kernel(DevModel m, const double* states, const double* times, const double* dL,
                                  const double* loss, int nb, int nt, double* lambda, double* Jbuf, double* tmp,
                                  double* wq, unsigned* bad) {
  const int n = m.n;
  const size_t row = (size_t)nb * n;
  const double Lval = loss ? *loss : 0.0;
  for (int b = blockIdx.x * blockDim.x + threadIdx.x; b < nb; b += gridDim.x * blockDim.x) {
    double* lam = lambda + (size_t)b * n;
    double* Jb = Jbuf + (size_t)b * n * n;
    double* tp = tmp + (size_t)b * n;
    for (int i = 0; i < n; ++i) lam[i] = 0.0;
    bool fin = true;
    for (int ms = nt; ms >= 1; --ms) {
      const double* ym = states + (size_t)ms * row + (size_t)b * n;
      for (int i = 0; i < n; ++i)
        lam[i] = xadd(lam[i], dL ? dL[(size_t)ms * row + (size_t)b * n + i] : (Lval > 0.0 ? ym[i] / Lval : 0.0));
      const double t0 = times[(size_t)(ms - 1) * nb + b];
      const double dt = times[(size_t)ms * nb + b] - t0;
      double* w = wq + (size_t)ms * row + (size_t)b * n;
      for (int i = 0; i < n; ++i) w[i] = xmul(lam[i], dt);
      PBlk J{Jb, n};
      model_jacobian<MD>(m, t0, CVec{states + (size_t)(ms - 1) * row + (size_t)b * n}, J, b);
      for (int e = 0; e < n * n; ++e) fin &= isfinite(Jb[e]);
      for (int i = 0; i < n; ++i) tp[i] = 0.0;
      for (int j = 0; j < n; ++j) {
        const double vj = lam[j];
        for (int i = 0; i < n; ++i) tp[i] = xadd(tp[i], xmul(Jb[j * n + i], vj));
      }
      for (int i = 0; i < n; ++i) lam[i] = xadd(lam[i], xmul(dt, tp[i]));
    }
    if (!fin) atomicOr(bad, 1u);
  }
}

// Per-model launchers, defined by CKO_INSTANTIATE in cko_inst_*.cu.
#define CKO_DECLARE(NAME)                                                                       \
  cudaError_t fwd_run_##NAME(const FwdLaunch& a, cudaStream_t st);                                 \
  cudaError_t fwd_occ_##NAME(int threads, int* blocks);                                            \
  cudaError_t preload_##NAME();                                                                    \
  cudaError_t fe_forward_run_##NAME(const DevModel& m, double* states, const double* times, int nb,   \
                                    int nt, double* hbuf, int* bad, cudaStream_t st);                  \
  cudaError_t fe_adjoint_run_##NAME(const DevModel& m, const double* states, const double* times,     \
                                    const double* dL, const double* loss, int nb, int nt,              \
                                    double* lambda, double* Jb, double* tmp, double* wq,               \
                                    unsigned* bad, cudaStream_t st);                                   \
  cudaError_t chunk_op_run_##NAME(const DevModel& m, int op, const double* ys, const double* dy,       \
                                  const double* t, const double* dt, int c, int nb, double* yyb,       \
                                  double* out, unsigned* flags, cudaStream_t st);                      \
  cudaError_t adj_run_##NAME(const AdjLaunch& a, cudaStream_t st);                                 \
  cudaError_t vjp_run_##NAME(const DevModel& m, const double* states, const double* times,          \
                             const double* wq, int nb, int nt, double* scratch, cudaStream_t st);

}  // namespace cko
