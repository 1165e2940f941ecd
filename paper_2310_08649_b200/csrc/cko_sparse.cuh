// cko_sparse.cuh — structured Thomas epochs for the mass-damper-spring chain
// (included by cko_v2.cuh; the kernels fwd2_kernel / adj2_kernel select them
// with their SP template flag).
//
// The block of a chunk row is M = I - dt J (forward) or its transpose
// (adjoint). The MDS Jacobian (models_mds.cpp:54-82) has a fixed pattern:
// position row u holds J[u][NU+u] = 1, velocity row NU+u holds columns
// u-1..u+1 and NU+u-1..NU+u+1. So, in 2x2 blocks of NU x NU,
//     M = [ I   B ]      B, C: one or three diagonals, D: tridiagonal,
//         [ C   D ]
// and every other entry is an exact zero. lu_factor_block (linalg.cpp:13-44)
// on such a block, whenever it does not exchange rows, does exactly this:
//   * columns 0..NU-1: the pivot is M[c][c] = 1 exactly, so inv = 1 and the
//     multipliers are C's entries unchanged; each row NU+v is updated only on
//     the (tridiagonal) entries that row c of B reaches: D' = D - C B, one
//     update per entry, in the same column order as the dense loop;
//   * columns NU..N-1: LU of the tridiagonal D' (one multiplier per column).
// Every update the dense loop applies beyond these is `x -= l * 0` or skipped
// by its own `if (l != 0.0)`: exact no-ops for finite entries. The factors
// (and the substitution of lu_solve_vec, linalg.cpp:46-60, over the nonzero
// terms in the same order) are therefore the dense ones, at ~14 NU doubles
// per record instead of N^2 and a few hundred flops instead of ~N^3 / 3.
//
// Eligibility is checked per block, exactly as the reference's scan decides:
// a row exchange (some |a(r, c)| > |pivot| below the diagonal), a pivot under
// the singularity threshold 1e-14 max|M|, or a non-finite entry makes the
// block ineligible. The kernels then raise FLAG_FALLBACK (forward: through the
// grid barrier, so every CTA and rank stops at the same iteration; adjoint: a
// device word) and the host re-runs the call on the dense group-LU kernels,
// which reproduce the reference's pivoting and singular-block reports.
#pragma once

#ifndef CKO_SP_DIAG
#define CKO_SP_DIAG 0  // diagnostics only (wrong results): 1 adjoint consumer skips its stores, 2 skips the solve
#endif

namespace cko {
namespace v2 {

template <class MS, class = void>
struct HasArrowTri {
  static constexpr bool value = false;
};
template <class MS>
struct HasArrowTri<MS, std::void_t<decltype(MS::kArrowTri)>> {
  static constexpr bool value = MS::kArrowTri;
};

// Structured record (doubles, 16-byte aligned pairs). C3: the entries of the
// three-diagonal off-block (forward: C, row NU+v at columns v-1..v+1;
// adjoint: B^T's rows) — 3 per row, chain-end slots never read; C1: the
// one-diagonal off-block (forward: B[u][NU+u] = -dt, adjoint: C[v][v]);
// TL: the tridiagonal multipliers (row NU+v, column NU+v-1); TR: 1 / U_ii of
// the velocity rows; TE: their superdiagonal already scaled by 1 / U_ii.
// The stride is 2 mod 16 doubles so the consumer threads' same-offset 16-byte
// loads of consecutive records fall in different bank groups.
template <int NU>
struct SpRec {
  static constexpr int N = 2 * NU;
  static constexpr int RHS = 0;
  static constexpr int Y = N;
  static constexpr int C3 = 2 * N;
  static constexpr int C1 = C3 + 3 * NU;
  static constexpr int TL = C1 + NU;
  static constexpr int TR = TL + NU;
  static constexpr int TE = TR + NU;
  static constexpr int DT = TE + NU;
  static constexpr int RAW = ((DT + 1) + 1) / 2 * 2;
  static constexpr int STRIDE = RAW + ((2 - RAW % 16) + 16) % 16;
  static_assert(C3 % 2 == 0 && C1 % 2 == 0 && TL % 2 == 0 && TR % 2 == 0 && TE % 2 == 0, "pairs stay aligned");
};

// Which of the three B / C diagonals are structural: forward M has C on three
// (velocity row NU+v couples to positions v-1..v+1) and B on one (J[u][NU+u]);
// the adjoint's M^T the other way round.
template <bool TR>
struct ArrowMask {
  static constexpr bool c(int o) { return TR ? o == 1 : true; }
  static constexpr bool b(int o) { return TR ? true : o == 1; }
};

template <int NU>
__device__ __forceinline__ constexpr bool in_chain(int v, int o) {
  return v + o - 1 >= 0 && v + o - 1 < NU;
}

// Schur update D' = D - C B (columns 0..NU-1 of the elimination) and the
// tridiagonal LU of D'. Lc, Ub: the entries of C and B; D: on entry D, on exit
// [multiplier, U diagonal, U superdiagonal] per velocity row; rinv: 1 / U_ii.
// mx: max |M| over the block. Returns false when lu_factor_block would pivot,
// call the block singular, or see a non-finite value.
template <int NU, bool TR>
__device__ __forceinline__ bool arrow_factor(const double (&Lc)[NU][3], const double (&Ub)[NU][3], double (&D)[NU][3],
                                             double mx, double (&rinv)[NU]) {
  using Mk = ArrowMask<TR>;
  const double tiny = 1e-14 * mx;
  bool ok = mx < INFINITY && !(1.0 < tiny);  // columns 0..NU-1: the pivot is 1
  // rows NU+v whose column c entry could beat the unit pivot (the scan's strict '>')
#pragma unroll
  for (int v = 0; v < NU; ++v)
#pragma unroll
    for (int o = 0; o < 3; ++o)
      if (Mk::c(o) && in_chain<NU>(v, o)) ok &= !(fabs(Lc[v][o]) > 1.0);
  // D' = D - C B: row NU+v, column c = v + oc - 1 (ascending), pivot-row entries at NU + c + ou - 1
#pragma unroll
  for (int v = 0; v < NU; ++v)
#pragma unroll
    for (int oc = 0; oc < 3; ++oc) {
      if (!Mk::c(oc) || !in_chain<NU>(v, oc)) continue;
      const int c = v + oc - 1;
      const double l = Lc[v][oc];  // a(NU+v, c) * (1 / 1)
#pragma unroll
      for (int ou = 0; ou < 3; ++ou) {
        if (!Mk::b(ou) || !in_chain<NU>(c, ou)) continue;
        const int od = c + ou - 1 - v + 1;  // column NU + c + ou - 1 relative to row NU + v
        if (od >= 0 && od < 3) D[v][od] -= l * Ub[c][ou];
      }
    }
  // tridiagonal LU of D' (columns NU..N-1)
#pragma unroll
  for (int u = 0; u < NU; ++u) {
    const double p = D[u][1];
    const double ap = fabs(p);
    ok &= ap >= tiny && ap != 0.0 && ap < INFINITY;
    const double inv = 1.0 / p;
    rinv[u] = inv;
    if (u + 1 < NU) {
      ok &= !(fabs(D[u + 1][0]) > ap);
      const double l = D[u + 1][0] * inv;
      D[u + 1][0] = l;
      D[u + 1][1] -= l * D[u][2];
    }
  }
  return ok;
}

template <int N>
__device__ __forceinline__ void lds_pairs(const double* __restrict__ p, double (&v)[N]) {
  static_assert(N % 2 == 0, "pairs");
#pragma unroll
  for (int i = 0; i < N; i += 2) {
    const double2 t = *reinterpret_cast<const double2*>(p + i);
    v[i] = t.x, v[i + 1] = t.y;
  }
}

// x <- M^{-1} x from a structured record: lu_solve_vec (linalg.cpp:46-60) over
// the nonzero terms. Forward sweep as the reference (j ascending); backward
// sweep with the row scaled by 1 / U_ii (x_i = y_i / U_ii - (U_ij / U_ii) x_j:
// one multiply-add on the substitution chain instead of a subtract and a
// division; rounding-level reordering of the reference's (y_i - U_ij x_j) / U_ii).
template <int NU, bool TR>
__device__ __forceinline__ void arrow_solve(const double* __restrict__ rec, double (&x)[2 * NU]) {
  using R = SpRec<NU>;
  using Mk = ArrowMask<TR>;
  double c3[3 * NU + (3 * NU) % 2], c1[NU + NU % 2], tl[NU + NU % 2], tr[NU + NU % 2], te[NU + NU % 2];
  lds_pairs(rec + R::C3, c3);
  lds_pairs(rec + R::C1, c1);
  lds_pairs(rec + R::TL, tl);
  lds_pairs(rec + R::TR, tr);
  lds_pairs(rec + R::TE, te);
  // forward, unit lower: rows 0..NU-1 have no multipliers; row NU+v: the position columns, then NU+v-1
#pragma unroll
  for (int v = 0; v < NU; ++v) {
    double s = x[NU + v];
    if constexpr (TR) {
      s -= c1[v] * x[v];
    } else {
#pragma unroll
      for (int o = 0; o < 3; ++o)
        if (in_chain<NU>(v, o)) s -= c3[3 * v + o] * x[v + o - 1];
    }
    if (v > 0) s -= tl[v] * x[NU + v - 1];
    x[NU + v] = s;
  }
  // backward: velocity rows, then position rows (U_ii = 1: B's columns only)
#pragma unroll
  for (int v = NU - 1; v >= 0; --v) {
    const double yv = x[NU + v] * tr[v];
    x[NU + v] = v + 1 < NU ? fma(-te[v], x[NU + v + 1], yv) : yv;
  }
#pragma unroll
  for (int u = 0; u < NU; ++u) {
    double s = x[u];
    if constexpr (TR) {
#pragma unroll
      for (int o = 0; o < 3; ++o)
        if (in_chain<NU>(u, o)) s -= c3[3 * u + o] * x[NU + u + o - 1];
    } else {
      s -= c1[u] * x[NU + u];
    }
    x[u] = s;
  }
  (void)Mk::c(0);
}

// Factor and store: Lc / Ub / D hold the block's entries; the factors go to `rec`.
template <int NU, bool TR>
__device__ __forceinline__ bool arrow_factor_store(const double (&Lc)[NU][3], const double (&Ub)[NU][3],
                                                   double (&D)[NU][3], double* rec) {
  using R = SpRec<NU>;
  using Mk = ArrowMask<TR>;
  double mx = 1.0;  // the position rows' unit diagonal
  bool finite = true;  // fmax drops NaN: any NaN entry must still make the block ineligible
#pragma unroll
  for (int v = 0; v < NU; ++v)
#pragma unroll
    for (int o = 0; o < 3; ++o) {
      if (Mk::c(o) && in_chain<NU>(v, o)) mx = fmax(mx, fabs(Lc[v][o])), finite &= Lc[v][o] == Lc[v][o];
      if (Mk::b(o) && in_chain<NU>(v, o)) mx = fmax(mx, fabs(Ub[v][o])), finite &= Ub[v][o] == Ub[v][o];
      if (in_chain<NU>(v, o)) mx = fmax(mx, fabs(D[v][o])), finite &= D[v][o] == D[v][o];
    }
  double rinv[NU];
  const bool ok = arrow_factor<NU, TR>(Lc, Ub, D, finite ? mx : INFINITY, rinv);
  // 16-byte stores of value pairs (half the shared-memory instructions of 8-byte stores)
  double c3[3 * NU + 1], c1[NU + 1], tl[NU + 1], tr[NU + 1], te[NU + 1];
#pragma unroll
  for (int v = 0; v < NU; ++v) {
#pragma unroll
    for (int o = 0; o < 3; ++o) c3[3 * v + o] = in_chain<NU>(v, o) ? (TR ? Ub[v][o] : Lc[v][o]) : 0.0;
    c1[v] = TR ? Lc[v][1] : Ub[v][1];
    tl[v] = v > 0 ? D[v][0] : 0.0;
    tr[v] = rinv[v];
    te[v] = v + 1 < NU ? D[v][2] * rinv[v] : 0.0;
  }
  c3[3 * NU] = c1[NU] = tl[NU] = tr[NU] = te[NU] = 0.0;
  auto put = [&](int off, const double* v, int n) {
#pragma unroll
    for (int i = 0; i < n; i += 2) *reinterpret_cast<double2*>(rec + off + i) = make_double2(v[i], v[i + 1]);
  };
  put(R::C3, c3, 3 * NU);
  put(R::C1, c1, NU);
  put(R::TL, tl, NU);
  put(R::TR, tr, NU);
  put(R::TE, te, NU);
  return ok;
}

// Consumer side of the ring with the structured shape's compile-time geometry (32 records per slot,
// kSpSlots slots): RingConsumer's bookkeeping without runtime divisions.
#ifndef CKO_SP_SLOTS
#define CKO_SP_SLOTS 3  // knob: producer sets = slots (one warp, one 32-record slot each), barriers 1 .. 2 slots;
                        // measured C2 adjoint ms: 7 sets 6.90, 6: 5.68, 5: 5.47, 4: 5.29, 3: 5.18 (fewer producers
                        // contend less with the consumer; 3 still keep up)
#endif
constexpr int kSpSlots = CKO_SP_SLOTS;
#ifndef CKO_SP_WARPS
#define CKO_SP_WARPS 8  // knob: warps of the structured kernels (up to 255 registers per thread at 8: no spills)
#endif
constexpr int kSpWarps = CKO_SP_WARPS;
static_assert(kSpWarps >= 4 && kSpWarps <= kMaxWarps, "consumer + producer warps");
static_assert(kSpSlots <= 7, "named barriers 1 .. 14");
struct RingSp {
  int LTc, J, synced, released;
  __device__ RingSp(int ltc, int c) : LTc(ltc), J((c * ltc + 31) >> 5), synced(0), released(0) {}
  __device__ __forceinline__ void acquire(int k) {
    const int need = ((k + 1) * LTc - 1) >> 5;
    while (synced <= need) {
      bar_sync(1 + synced % kSpSlots, 64);
      ++synced;
    }
  }
  __device__ __forceinline__ void release(int k) {
    const int done = ((k + 1) * LTc) >> 5;
    while (released < done) {
      if (released + kSpSlots < J) bar_arrive(1 + kSpSlots + released % kSpSlots, 64);
      ++released;
    }
  }
  __device__ __forceinline__ int record(int k, int lane) const {
    const int i = k * LTc + lane;
    return ((i >> 5) % kSpSlots) * 32 + (i & 31);
  }
};

// ---- forward epoch (one Newton iteration of one lane tile), structured records -----------------
// Ring as in fwd_epoch (RingConsumer), with one thread per record: producer set s (one warp) fills
// slots s, s + S, ... of RS = 32 items; the consumer warp runs one lane per thread.
template <class MS>
__device__ void fwd_epoch_sp(const FwdLaunch& a, const FwdCtx& x, const Shape& sh, const double* cs, double* recs,
                             const double* hr, int t0, int LTc, unsigned* s_fb) {
  constexpr int N = MS::N, NU = N / 2;
  using R = SpRec<NU>;
  constexpr int kS = R::STRIDE;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  constexpr int S = kSpSlots, Q = kSpSlots, RS = 32;
  constexpr int nthr = 64;
  const int nb = a.nb;
  const int pw = producer_of(warp);
  (void)sh;
  if (pw >= 0 && pw < S) {
    const int I = x.c * LTc, J = (I + RS - 1) / RS;
    const double* Jm = cs + MS::JOFF;
    // CKO_TRACE: slot js of the traced chunk in CTA 0: [0] wait start, [1] acquired, [2] factor start, [3] done
    unsigned long long* tr0 = (a.trace && blockIdx.x == 0 && x.step == trace_step(a) && lane == 0) ? a.trace + 64 : nullptr;
    for (int js = pw; js < J; js += S) {
      unsigned long long* tr = (tr0 && js < x.c) ? tr0 + js * 8 : nullptr;
      if (tr) tr[0] = globaltimer_ns();
      const int q = js % Q;
      const bool active = js * RS + lane < I;
      const int item = active ? js * RS + lane : I - 1;
      const int k = item / LTc, lb = t0 + item % LTc, b = x.lb0 + lb;
      double* rec = recs + (size_t)(q * RS + lane) * kS;
      // the point's iterate, residual and times are requested before the slot wait
      const double2* yrow = reinterpret_cast<const double2*>(a.states + (size_t)(x.step + 1 + k) * x.row + (size_t)b * N);
      const double2* rrow = reinterpret_cast<const double2*>(hr + (size_t)(k * x.L + lb) * N);  // slabs: even
      double2 ye[NU], re[NU];
#pragma unroll
      for (int i = 0; i < NU; ++i) ye[i] = yrow[i], re[i] = rrow[i];
      const double t = a.times[(size_t)(x.step + 1 + k) * nb + b];
      const double dt = t - a.times[(size_t)(x.step + k) * nb + b];
      if (js >= Q) bar_sync(1 + Q + q, nthr);
      if (tr) tr[1] = globaltimer_ns();
      if (active) {
#pragma unroll
        for (int i = 0; i < N; i += 2) {
          *reinterpret_cast<double2*>(rec + R::RHS + i) = re[i / 2];
          *reinterpret_cast<double2*>(rec + R::Y + i) = ye[i / 2];
        }
        // M = I - dt J (the dense build's roundings: xmul(-dt, J_ij), + 1 on the diagonal)
        const double ndt = -dt;
        double Lc[NU][3], Ub[NU][3], D[NU][3];
#pragma unroll
        for (int v = 0; v < NU; ++v)
#pragma unroll
          for (int o = 0; o < 3; ++o) {
            const bool in = in_chain<NU>(v, o);
            const int cix = in ? v + o - 1 : v;
            Lc[v][o] = in ? xmul(ndt, Jm[(NU + v) * N + cix]) : 0.0;
            D[v][o] = in ? xmul(ndt, Jm[(NU + v) * N + NU + cix]) : 0.0;
            Ub[v][o] = o == 1 ? xmul(ndt, Jm[v * N + NU + v]) : 0.0;
          }
#pragma unroll
        for (int v = 0; v < NU; ++v) D[v][1] = xadd(D[v][1], 1.0);
        if (tr) tr[2] = globaltimer_ns();
        if (!arrow_factor_store<NU, false>(Lc, Ub, D, rec)) atomicOr(s_fb, 1u);
      }
      if (tr) tr[3] = globaltimer_ns();
      bar_arrive(1 + q, nthr);
    }
  } else if (warp == 0) {
    // consumer: x_k = M_k^{-1}(r_k + x_{k-1}), yy_k -= x_k, one thread per lane
    const int lt = lane;
    const bool active = lt < LTc;
    const int b = x.lb0 + t0 + lt;
    double xv[N];
#pragma unroll
    for (int i = 0; i < N; ++i) xv[i] = 0.0;
    unsigned long long* tr = (a.trace && blockIdx.x == 0 && x.step == trace_step(a) && lane == 0) ? a.trace + 64 : nullptr;
    RingSp ring(LTc, x.c);
    for (int k = 0; k < x.c; ++k) {
      if (tr) tr[k * 8 + 4] = globaltimer_ns();
      ring.acquire(k);
      if (tr) tr[k * 8 + 5] = globaltimer_ns();
      if (active) {
        const double* rec = recs + (size_t)ring.record(k, lt) * kS;
        double rh[N];
        lds_pairs(rec + R::RHS, rh);
#pragma unroll
        for (int i = 0; i < N; ++i) xv[i] = rh[i] + xv[i];
        arrow_solve<NU, false>(rec, xv);
        double yv[N];
        lds_pairs(rec + R::Y, yv);
        double2* yy = reinterpret_cast<double2*>(a.states + (size_t)(x.step + 1 + k) * x.row + (size_t)b * N);
#pragma unroll
        for (int i = 0; i < NU; ++i) yy[i] = make_double2(yv[2 * i] - xv[2 * i], yv[2 * i + 1] - xv[2 * i + 1]);
      }
      if (tr) tr[k * 8 + 6] = globaltimer_ns();
      ring.release(k);
    }
  }
}

// ---- adjoint epoch (one reversed chunk of one lane tile), structured records --------------------
template <class MS>
__device__ void adj_epoch_sp(const AdjLaunch& a, const Shape& sh, const double* cs, double* recs, const double* lam,
                             const double* jtl, int lb0, int t0, int LTc, int step_hi, int c, double Lval,
                             double (&dcar)[MS::N]) {
  static_assert(HasJtLambda<MS>::value, "the structured adjoint forms J^T lambda once per chunk");
  constexpr int N = MS::N, NU = N / 2;
  using R = SpRec<NU>;
  constexpr int kS = R::STRIDE;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  constexpr int S = kSpSlots, Q = kSpSlots, RS = 32;
  constexpr int nthr = 64;
  const int nb = a.nb;
  const size_t row = (size_t)nb * N;
  const double rL = Lval > 0.0 ? 1.0 / Lval : 0.0;
  const int pw = producer_of(warp);
  (void)sh;
  if (pw >= 0 && pw < S) {
    const int I = c * LTc, J = (I + RS - 1) / RS;
    const double* Jm = cs + MS::JOFF;
    for (int js = pw; js < J; js += S) {
      const int q = js % Q;
      const bool active = js * RS + lane < I;
      const int item = active ? js * RS + lane : I - 1;
      const int r = item / LTc, ltc = item % LTc;
      const int b = lb0 + t0 + ltc;
      const int m = step_hi - r;
      double* rec = recs + (size_t)(q * RS + lane) * kS;
      const double* yrow = (a.dL ? a.dL : a.states) + (size_t)m * row + (size_t)b * N;
      double yq[N];
      if ((reinterpret_cast<uintptr_t>(a.dL) & 15) == 0) {  // the trajectory (or an aligned user dL): pairs
#pragma unroll
        for (int i = 0; i < N; i += 2) {
          const double2 v = *reinterpret_cast<const double2*>(yrow + i);
          yq[i] = v.x, yq[i + 1] = v.y;
        }
      } else {
#pragma unroll
        for (int i = 0; i < N; ++i) yq[i] = yrow[i];
      }
      const double t = a.times[(size_t)m * nb + b];
      const double dt = t - a.times[(size_t)(m - 1) * nb + b];
      if (js >= Q) bar_sync(1 + Q + q, nthr);
      if (active) {
        // rhs = dL_m + dt J^T lambda_c (adjoint.cpp:88-100); J^T lambda_c is the same for every row of the
        // reversed chunk (J is constant, lambda_c is the chunk's carry): jtl, formed once per chunk
        const double* g = jtl + (size_t)ltc * N;
#pragma unroll
        for (int i = 0; i < N; i += 2) {
          // y / L from the correctly rounded 1 / L and one remainder correction (div_rn: the quotient)
          const double d0 = a.dL ? yq[i] : (Lval > 0.0 ? div_rn(yq[i], Lval, rL) : 0.0);
          const double d1 = a.dL ? yq[i + 1] : (Lval > 0.0 ? div_rn(yq[i + 1], Lval, rL) : 0.0);
          *reinterpret_cast<double2*>(rec + R::RHS + i) = make_double2(d0 + dt * g[i], d1 + dt * g[i + 1]);
        }
        rec[R::DT] = dt;
        // M^T: B^T-side entries M[NU+u+o-1][u], C^T-side M[v][NU+v], D^T entries M[NU+v+o-1][NU+v]
        const double ndt = -dt;
        double Lc[NU][3], Ub[NU][3], D[NU][3];
#pragma unroll
        for (int v = 0; v < NU; ++v)
#pragma unroll
          for (int o = 0; o < 3; ++o) {
            const bool in = in_chain<NU>(v, o);
            const int rix = in ? v + o - 1 : v;
            Ub[v][o] = in ? xmul(ndt, Jm[(NU + rix) * N + v]) : 0.0;
            D[v][o] = in ? xmul(ndt, Jm[(NU + rix) * N + NU + v]) : 0.0;
            Lc[v][o] = o == 1 ? xmul(ndt, Jm[v * N + NU + v]) : 0.0;
          }
#pragma unroll
        for (int v = 0; v < NU; ++v) D[v][1] = xadd(D[v][1], 1.0);
        if (!arrow_factor_store<NU, true>(Lc, Ub, D, rec)) atomicOr(a.sp_fallback, 1u);
      }
      bar_arrive(1 + q, nthr);
    }
  } else if (warp == 0) {
    const int lt = lane;
    const bool active = lt < LTc;
    double d[N];  // delta_{r-1}, then delta_r
#pragma unroll
    for (int i = 0; i < N; ++i) d[i] = 0.0;
    const int b = lb0 + t0 + lt;
    const double* lc = lam + (size_t)lt * N;
    RingSp ring(LTc, c);
    for (int r = 0; r < c; ++r) {
      ring.acquire(r);
      if (active) {
        const int m = step_hi - r;
        const double* rec = recs + (size_t)ring.record(r, lt) * kS;
        double rh[N];
        lds_pairs(rec + R::RHS, rh);
#pragma unroll
        for (int i = 0; i < N; ++i) d[i] = rh[i] + d[i];
        const double dt = rec[R::DT];
        if (CKO_SP_DIAG != 2) arrow_solve<NU, true>(rec, d);
        double* w = a.wq + (size_t)m * row + (size_t)b * N;
#pragma unroll
        for (int i = 0; i < N; i += 2)
          if (CKO_SP_DIAG != 1)
            __stcs(reinterpret_cast<double2*>(w + i), make_double2((lc[i] + d[i]) * dt, (lc[i + 1] + d[i + 1]) * dt));
      }
      ring.release(r);
    }
#pragma unroll
    for (int i = 0; i < N; ++i) dcar[i] = d[i];
  }
}

// Launch shape of the structured kernels: S one-warp producer sets, one 32-record slot each.
template <class MS>
inline Shape make_shape_sp(int L, bool stage_residuals) {
  constexpr int N = MS::N;
  Shape sh;
  sh.Ws = 1;
  sh.RS = 32;
  sh.S = kSpSlots;
  sh.Q = kSpSlots;
  sh.inv = 0;
  sh.stride = SpRec<N / 2>::STRIDE;
  sh.threads = 32 * kSpWarps;
  sh.LT = L < 32 ? L : 32;
  int o_cs, o_rec, o_pb, o_vs, o_lam, tot;
  // the record region takes the rest of shared memory: the forward's residual passes stage through it
  // (more trajectory rows per staged block, fewer blocks per pass)
  sh.ring = sh.Q * sh.RS * sh.stride;
  smem_layout<MS>(sh.S, sh.Q, sh.Ws, sh.RS, sh.LT, sh.stride, o_cs, o_rec, o_pb, o_vs, o_lam, tot, true, sh.ring);
  const int spare = kSmemCap / 8 - tot - 8;
  if (stage_residuals && spare > 0) sh.ring += spare & ~1;
  smem_layout<MS>(sh.S, sh.Q, sh.Ws, sh.RS, sh.LT, sh.stride, o_cs, o_rec, o_pb, o_vs, o_lam, tot, true, sh.ring);
  sh.smem_bytes = tot * 8;
  return sh;
}

}  // namespace v2
}  // namespace cko
