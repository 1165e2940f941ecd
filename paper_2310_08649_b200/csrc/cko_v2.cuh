// cko_v2.cuh — warp-specialised sm_100a kernels for the chunked backward-Euler
// path with Thomas (block-substitution) solves.
//
// Mapping:
//  * one persistent CTA per SM owns a contiguous lane range; lanes are
//    processed in tiles of <= LT lanes;
//  * a Newton iteration of a chunk (integrate.cpp:208-231) or one reversed
//    chunk of the adjoint (adjoint.cpp:64-101) is an "epoch" over its rows
//    k = 0..c-1: PRODUCER warps build M_k = I - dt J_k (or its transpose) and
//    LU-factor it with the rows spread over a group of G lanes (register
//    resident, logical partial pivoting that reproduces the reference's pivot
//    sequence, linalg.cpp:13-44); a CONSUMER warp runs the sequential
//    substitution x_k = M_k^{-1}(r_k + x_{k-1}) one thread per lane. The two
//    meet in an S-slot shared-memory ring guarded by named barriers, so the
//    factorisation of rows k+1..k+S overlaps the substitution of row k;
//  * the forward's all-lanes convergence predicate (integrate.cpp:176-182)
//    stays the only cross-CTA coupling (grid_reduce_or, cko_common.cuh).
#pragma once

#include <type_traits>
#include <cfloat>
#include <climits>

#include "cko_impl.cuh"
#include "cko_static_models.cuh"

namespace cko {
namespace v2 {

// Rows of an N x N block are spread over G lanes, R rows per lane
// (row i -> lane i % G, slot i / G); GPW groups per warp. Lanes past GPW * G
// (G = 10: lanes 30, 31) shadow the last group's first lanes: they compute the
// same values and write the same addresses, which keeps the warp converged.
template <int N>
struct Geo {
#ifndef CKO_G20
#define CKO_G20 10  // lanes per group for 17 <= n <= 20 (knob; 7 spills)
#endif
  static constexpr int G = N <= 8 ? 1 : (N <= 16 ? 8 : (N <= 20 ? CKO_G20 : 16));
  static constexpr int R = (N + G - 1) / G;
  static constexpr int GPW = 32 / G;
};

// Lane roles inside a warp of producer groups.
template <int N>
struct GroupLane {
  int g, gl, base;
  __device__ explicit GroupLane(int lane) {
    constexpr int G = Geo<N>::G, GPW = Geo<N>::GPW;
    g = lane / G;
    gl = lane % G;
    if (g >= GPW) g = GPW - 1;
    base = g * G;
  }
};

constexpr int kMaxWarps = 12;  // 3 warps per SMSP: up to 168 registers per thread
constexpr int kMaxProducers = 9;  // warp 0 consumes alone on SMSP 0 (warps 4, 8 idle)

// producer index of a warp, -1 for the consumer (0) and the idle warps (4, 8)
__device__ __forceinline__ int producer_of(int warp) {
  if ((warp & 3) == 0) return -1;
  return warp - 1 - (warp >> 2);
}
constexpr int kMaxSlots = 7;  // record slots: named barriers 1..2Q must stay below 16
constexpr int kSmemCap = 224 * 1024;
constexpr int kRoundBarrier = 15;  // producers only; ring barriers use 1 .. 2Q <= 14
constexpr bool kFwdRounds = true;   // producer sets advance in rounds (instruction-cache locality)

// Tuning knobs: compile-time, A/B-tested with scripts/build_variant.sh and
// scripts/gpu_variants.sh / gpu_cmp_dt.sh; the defaults are the measured best
// (DESIGN.md section 7 lists what each alternative cost).
#ifndef CKO_ROUND_PER_SMSP
#define CKO_ROUND_PER_SMSP 1  // round barrier among the 3 producer warps of each SMSP (0: all 9)
#endif
#ifndef CKO_ROUND_EVERY
#define CKO_ROUND_EVERY 1  // rounds between producer barriers
#endif
#ifndef CKO_XCHG2
#define CKO_XCHG2 2  // row exchange: 0 all rows through the record; 1 shuffle argmax + owner lanes; 2 scan + owner lanes
#endif
#ifndef CKO_LOOKAHEAD
#define CKO_LOOKAHEAD 0  // group LU publishes row c + 1 during column c
#endif
#ifndef CKO_FWD_SHARED_JAC
#define CKO_FWD_SHARED_JAC 0  // forward builds M from the shared-memory J rows instead of per-entry selects
#endif
#ifndef CKO_FWD_SLOT_ROWS
#define CKO_FWD_SLOT_ROWS 0  // forward builds MDS rows by kind (position / velocity slot)
#endif
#ifndef CKO_LU_SKIP
#define CKO_LU_SKIP 0  // knob: skip a slot's trailing update when every multiplier in it is zero (measured: slower)
#endif
#ifndef CKO_FWD_PRED
#define CKO_FWD_PRED 0  // predicated (not branched) trailing update in the forward LU
#endif
constexpr int kRoundEvery = CKO_ROUND_EVERY;
constexpr bool kLookahead = CKO_LOOKAHEAD;
constexpr bool kFwdSharedJac = CKO_FWD_SHARED_JAC;
constexpr bool kFwdSlotRows = CKO_FWD_SLOT_ROWS;
constexpr bool kFwdPred = CKO_FWD_PRED;
constexpr int kMaxWs = 3;     // producer warps per slot
#ifndef CKO_INV_MAX_LANES
#define CKO_INV_MAX_LANES 2  // knob: explicit-inverse records up to this many lanes per CTA (0: never)
#endif
constexpr int kInvMaxLanes = CKO_INV_MAX_LANES;
#ifndef CKO_ADJ_VEC_W
#define CKO_ADJ_VEC_W 1  // adjoint consumer: weights as 16-byte streaming stores (measured: adjoint 24.6 -> 24.1 ms)
#endif
constexpr bool kAdjVecW = CKO_ADJ_VEC_W;
#ifndef CKO_FWD_EARLY_LOADS
#define CKO_FWD_EARLY_LOADS 2  // forward producers request the point's iterate / residual (1), and times (2),
#endif                         // before the slot wait
constexpr int kFwdEarlyLoads = CKO_FWD_EARLY_LOADS;
#ifndef CKO_ADJ_LEAN_RHS
#define CKO_ADJ_LEAN_RHS 12  // adjoint producers, bit mask: 1 sparse J^T lambda, 2 y / L by reciprocal, 4 y loads first,
                             // 8 times before the slot wait, 16 y before the slot wait
                             // (measured adjoint ms: none 24.07, 1: 24.39, 2: 24.38, 4: 23.28, 7: 23.71, 8: 25.2, 12: 22.75)
#endif
constexpr int kAdjLeanRhs = CKO_ADJ_LEAN_RHS;

// Shared-memory record of one factored point (doubles): the LU factors in
// the reference's row order (row-major), 1/U_ii, rhs (residual / adjoint
// rhs), the iterate (forward), dt, and the row permutation (ints; PERM[N] = 1
// when it is the identity).
// The stride is padded to 2 mod 16 doubles so the consumer threads' same-offset
// 16-byte loads of different records fall in different bank groups.
template <int N>
struct Rec {
  static constexpr int LU = 0;
  static constexpr int RD = N * N;
  static constexpr int RHS = RD + N;
  static constexpr int Y = RHS + N;
  static constexpr int DT = Y + N;
  static constexpr int PERM = DT + 1;                       // ints start here (as double offset)
  static constexpr int RAW = PERM + (N + 2) / 2;
  static constexpr int STRIDE = RAW + ((2 - RAW % 16) + 16) % 16;
  // explicit-inverse records (small lane counts, see lu_inverse_group): M^{-1} row-major after the rest
  static constexpr int INV = ((RAW + 1) / 2) * 2;
  static constexpr int RAW_INV = INV + N * N;
  static constexpr int STRIDE_INV = RAW_INV + ((2 - RAW_INV % 16) + 16) % 16;
};

// Models whose Jacobian is a per-CTA constant in shared memory (MdsS).
template <class MS, class = void>
struct HasConstJac {
  static constexpr bool value = false;
};
template <class MS>
struct HasConstJac<MS, std::void_t<decltype(MS::kConstJac)>> {
  static constexpr bool value = MS::kConstJac;
};

// Models with a structural-nonzero J^T lambda (MdsS::jt_lambda).
template <class MS, class = void>
struct HasJtLambda {
  static constexpr bool value = false;
};
template <class MS>
struct HasJtLambda<MS, std::void_t<decltype(&MS::jt_lambda)>> {
  static constexpr bool value = true;
};

// y / x from r = RN(1 / x): q = y r and one remainder correction (Markstein), the correctly rounded
// quotient for finite operands away from the overflow / underflow ranges — y / x without the divide
// sequence.
__device__ __forceinline__ double div_rn(double y, double x, double r) {
  const double q = y * r;
  return fma(fma(-x, q, y), r, q);
}

// Models that build M row by row kind in the 10-lane group layout (MdsS).
template <class MS, class = void>
struct HasSlotRows {
  static constexpr bool value = false;
};
template <class MS>
struct HasSlotRows<MS, std::void_t<decltype(MS::kSlotRows)>> {
  static constexpr bool value = MS::kSlotRows;
};

// Per-group pivot-row buffer: two rows of N + 2 doubles (16-byte aligned halves).
template <int N>
constexpr int kPbRow = ((N + 3) / 2) * 2;  // even: both halves stay 16-byte aligned for the pair stores
template <int N>
constexpr int kPb = 2 * kPbRow<N>;

struct Shape {
  int S, Ws, LT;       // producer sets, producer warps per set, lanes per tile
  int Q;               // record slots in the ring (a multiple of S: each set fills every S-th slot)
  int RS;              // records per slot (= groups per set)
  int threads;
  int smem_bytes;
  int inv;             // records carry M^{-1} and the consumer multiplies (few lanes per CTA)
  int stride;          // record stride in doubles (Rec<N>::STRIDE or STRIDE_INV)
  int ring;            // doubles of the record region (>= Q RS stride; the residual passes stage through it)
};

template <class MS>
__host__ __device__ inline void smem_layout(int S, int Q, int Ws, int RS, int LT, int stride, int& o_cs, int& o_rec,
                                            int& o_pb, int& o_vs, int& o_lam, int& total_doubles, bool sp = false,
                                            int ring = -1) {
  constexpr int N = MS::N;
  o_cs = 0;
  o_rec = ((MS::NCONST + 1) / 2) * 2;
  o_pb = o_rec + (ring >= 0 ? ring : Q * RS * stride);
  const int groups = sp ? 0 : S * RS;  // structured records (cko_sparse.cuh) need no pivot-row buffers
  o_vs = o_pb + groups * kPb<N>;
  o_lam = o_vs + LT * N + (N & 1);
  total_doubles = o_lam + LT * N + 8;
}

__device__ __forceinline__ void bar_sync(int id, int n) { asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(n) : "memory"); }
__device__ __forceinline__ void bar_arrive(int id, int n) {
  asm volatile("bar.arrive %0, %1;" ::"r"(id), "r"(n) : "memory");
}

// round barrier: all producer warps (15), or per SMSP (13 .. 15, three producer warps each)
__device__ __forceinline__ void producer_round_sync(int warp, int nprod) {
  if (CKO_ROUND_PER_SMSP && nprod == 9)
    bar_sync(12 + (warp & 3), 96);
  else
    bar_sync(15, 32 * nprod);
}


// 1 / x to within an ulp: the hardware seed refined by two Newton steps (no
// special-case path; pivots here are finite and nonzero or the block is
// flagged singular anyway). The reference divides; the factors differ from it
// at rounding level only.
__device__ __forceinline__ double rcp_nr(double x) {
  double r;
  asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(x));
  double e = fma(-x, r, 1.0);
  r = fma(r, e, r);
  e = fma(-x, r, 1.0);
  return fma(r, e, r);
}

// Rotation reduction inside a group of G lanes starting at lane `base`:
// after steps 1, 2, 4, ... every lane has combined a window of >= G lanes
// (idempotent ops only: max / argmax). Works for any G, not just powers of 2.
template <int G>
__device__ __forceinline__ int rot_src(int base, int gl, int off) {
  return base + (gl + off) % G;
}

template <int G>
__device__ __forceinline__ double group_max_nonneg(double v, int base, int gl) {
#pragma unroll
  for (int off = 1; off < G; off <<= 1) v = fmax(v, __shfl_sync(0xffffffffu, v, rot_src<G>(base, gl, off)));
  return v;
}

enum { kLuOk = 0, kLuSingular = 1, kLuCheckExact = 2 };

__device__ __forceinline__ float fmax_nan(float a, float b) {
  float r;
  asm("max.NaN.f32 %0, %1, %2;" : "=f"(r) : "f"(a), "f"(b));
  return r;
}

template <int G>
__device__ __forceinline__ double group_min(double v, int base, int gl) {
#pragma unroll
  for (int off = 1; off < G; off <<= 1) v = fmin(v, __shfl_sync(0xffffffffu, v, rot_src<G>(base, gl, off)));
  return v;
}

template <int G>
__device__ __forceinline__ float group_max_f(float v, int base, int gl) {
#pragma unroll
  for (int off = 1; off < G; off <<= 1) v = fmax_nan(v, __shfl_sync(0xffffffffu, v, rot_src<G>(base, gl, off)));
  return v;
}

// Owner lane publishes row c of the block (columns c .. N-1) to the group
// buffer; pairs go as 16-byte stores (buf is 16-byte aligned).
template <int N>
__device__ __forceinline__ void publish_row(double* buf, const double (&v)[N], int c) {
  if (c & 1) buf[c] = v[c];
#pragma unroll
  for (int j = (c + 1) & ~1; j < N; j += 2) {
    if (j + 1 < N)
      *reinterpret_cast<double2*>(buf + j) = make_double2(v[j], v[j + 1]);
    else
      buf[j] = v[j];
  }
}

// Row moves through shared memory, 16-byte accesses when rows stay aligned.
template <int N>
__device__ __forceinline__ void store_row(double* dst, const double (&v)[N]) {
  if constexpr (N % 2 == 0) {
#pragma unroll
    for (int j = 0; j < N; j += 2) *reinterpret_cast<double2*>(dst + j) = make_double2(v[j], v[j + 1]);
  } else {
#pragma unroll
    for (int j = 0; j < N; ++j) dst[j] = v[j];
  }
}
template <int N>
__device__ __forceinline__ void load_row(const double* src, double (&v)[N]) {
  if constexpr (N % 2 == 0) {
#pragma unroll
    for (int j = 0; j < N; j += 2) {
      const double2 t = *reinterpret_cast<const double2*>(src + j);
      v[j] = t.x;
      v[j + 1] = t.y;
    }
  } else {
#pragma unroll
    for (int j = 0; j < N; ++j) v[j] = src[j];
  }
}

// LU with partial pivoting (lu_factor_block, linalg.cpp:13-44) of the block
// whose rows lane gl of a G-lane group holds in a[s] (row gl + s G), factors
// to `rec` in the reference's row order. Rows sit at static lanes/slots, so
// the common column (the diagonal already wins the reference's strict '>'
// scan) is a plain elimination step: the owner of row c publishes it to the
// group buffer, every lane reads the pivot, and a warp vote checks that no row
// below beats it. Only when one does (warp-uniform branch) is the argmax taken
// — the largest |a(r, c)|, ties to the smallest r, exactly the reference's scan
// — and rows c and p are exchanged physically through `rec` (scratch until
// the factors are stored: each row is written to its swapped position and
// read back), so the static layout holds again; `orig` tracks
// each row's source row for the permutation. Arithmetic per column is then
// identical to the reference's (multiplier by the pivot reciprocal). The whole
// warp must call this; pb is a kPb<N>-double group buffer.
template <int N, bool kPred = false>
__device__ inline int lu_group(double (&a)[Geo<N>::R][N], int gl, int base, double* pb, double* rec) {
  constexpr int G = Geo<N>::G, R = Geo<N>::R;
  // max |a| for the singularity threshold on the high words only (one float
  // max per element; exact order for |a| < 2^1017, NaN-propagating so any
  // inf/NaN/huge entry defers to the exact test)
  float lmf = 0.0f;
#pragma unroll
  for (int s = 0; s < R; ++s)
    if (gl + s * G < N)
#pragma unroll
      for (int j = 0; j < N; ++j) lmf = fmax_nan(lmf, fabsf(__int_as_float(__double2hiint(a[s][j]))));
  int orig[R];
#pragma unroll
  for (int s = 0; s < R; ++s) orig[s] = gl + s * G;
  bool swapped = false;  // group-uniform
  int* iscr = reinterpret_cast<int*>(rec + Rec<N>::PERM);  // row-source scratch until perm is stored
#pragma unroll
  for (int c = 0; c < N; ++c) {
    double* buf = pb + (c & 1) * kPbRow<N>;
    const int sc = c / G, lc = c % G;  // slot / lane of row c
    if ((!kLookahead || c == 0) && gl == lc) publish_row<N>(buf, a[sc], c);
    __syncwarp();
    double piv = buf[c];
    bool beat = false;
#pragma unroll
    for (int s = 0; s < R; ++s)
      if (s * G + G - 1 > c && gl + s * G > c && gl + s * G < N) beat |= fabs(a[s][c]) > fabs(piv);
    if (__any_sync(0xffffffffu, beat)) {
#if CKO_XCHG2
#if CKO_XCHG2 == 2
      // the reference's scan (strict '>' from row c down) over |a(r, c)| staged in the idle half of pb
      double* cand = pb + ((c + 1) & 1) * kPbRow<N>;
#pragma unroll
      for (int s = 0; s < R; ++s) {
        const int r = gl + s * G;
        if (s * G + G - 1 >= c && r >= c && r < N) cand[r] = fabs(a[s][c]);
      }
      __syncwarp();
      int p = c;
      double bv = cand[c];
#pragma unroll 4
      for (int r = c + 1; r < N; ++r) {
        const double v = cand[r];
        if (v > bv) bv = v, p = r;
      }
#else
      // argmax over the group's rows r >= c by rotation shuffles (larger |a| wins, ties to the smaller
      // r): the first maximum of the reference's strict '>' scan; a NaN pivot keeps row c like the scan
      double bv = -1.0;
      int br = INT_MAX;
#pragma unroll
      for (int s = 0; s < R; ++s) {
        const int r = gl + s * G;
        if (s * G + G - 1 >= c && r >= c && r < N) {
          const double v = fabs(a[s][c]);
          if (v > bv) bv = v, br = r;  // slots ascend in r: '>' keeps the smaller r on ties
        }
      }
#pragma unroll
      for (int off = 1; off < G; off <<= 1) {
        const int src = rot_src<G>(base, gl, off);
        const double ov = __shfl_sync(0xffffffffu, bv, src);
        const int orr = __shfl_sync(0xffffffffu, br, src);
        if (ov > bv || (ov == bv && orr < br)) bv = ov, br = orr;
      }
      const int p = (br == INT_MAX || !(fabs(piv) < bv)) ? c : br;
#endif
      // exchange rows c and p through two scratch rows at the front of the record (the factors are
      // stored at the end); the owner(s) write both rows, then read them back swapped
      const int sp = p / G, lp = p % G;
      const bool cross = p != c;
      if (cross && gl == lc) {
        store_row<N>(rec, a[sc]);
        iscr[0] = orig[sc];
      }
      if (cross && gl == lp) {
#pragma unroll
        for (int s = 0; s < R; ++s)
          if (s == sp) {
            store_row<N>(rec + N, a[s]);
            iscr[1] = orig[s];
          }
      }
      __syncwarp();
      if (cross && gl == lc) {
        load_row<N>(rec + N, a[sc]);
        orig[sc] = iscr[1];
      }
      if (cross && gl == lp) {
#pragma unroll
        for (int s = 0; s < R; ++s)
          if (s == sp) {
            load_row<N>(rec, a[s]);
            orig[s] = iscr[0];
          }
      }
#else
      // the reference's scan (strict '>' from row c down) over |a(r, c)| staged in the idle half of pb
      double* cand = pb + ((c + 1) & 1) * kPbRow<N>;
#pragma unroll
      for (int s = 0; s < R; ++s) {
        const int r = gl + s * G;
        if (s * G + G - 1 >= c && r >= c && r < N) cand[r] = fabs(a[s][c]);
      }
      __syncwarp();
      int p = c;
      double bv = cand[c];
#pragma unroll 4
      for (int r = c + 1; r < N; ++r) {
        const double v = cand[r];
        if (v > bv) bv = v, p = r;
      }
      // exchange rows c and p: every row goes to its swapped position in the record, then reads back
#pragma unroll
      for (int s = 0; s < R; ++s) {
        const int r = gl + s * G;
        if (r < N) {
          const int d = r == c ? p : (r == p ? c : r);
          store_row<N>(rec + d * N, a[s]);
          iscr[d] = orig[s];
        }
      }
      __syncwarp();
#pragma unroll
      for (int s = 0; s < R; ++s) {
        const int r = gl + s * G;
        if (r < N) {
          load_row<N>(rec + r * N, a[s]);
          orig[s] = iscr[r];
        }
      }
#endif
      swapped |= p != c;
      if (gl == lc) publish_row<N>(buf, a[sc], c);
      __syncwarp();
      piv = buf[c];
    }
    const double inv = rcp_nr(piv);
    if (gl == 0) rec[Rec<N>::RD + c] = inv;
    // slot s holds rows s G .. s G + G - 1: nothing below the pivot once c >= s G + G - 1.
    // kPred: predicated, not branched — rows on or above the pivot run the update with l = 0,
    // which leaves them unchanged (up to the sign of a zero entry). Measured per kernel.
    // The reference skips a row whose multiplier is exactly zero (lu_factor_block's `if (l != 0.0)`,
    // linalg.cpp:36-40): x - 0 y is x, so skipping is exact. Here the whole slot's update is skipped when no
    // lane of the warp has a nonzero multiplier in it (the warp's blocks share a sparsity pattern, e.g. the
    // MDS chain's I - dt J), which removes most of the chain matrices' trailing updates.
    auto update = [&](int s) {
      if constexpr (kPred) {
        if (s * G + G - 1 > c) {
          const bool below = gl + s * G > c && gl + s * G < N;
          const double l = below ? a[s][c] * inv : 0.0;
          if (below) a[s][c] = l;
          if (!CKO_LU_SKIP || __any_sync(0xffffffffu, l != 0.0)) {
#pragma unroll
            for (int j = c + 1; j < N; ++j) a[s][j] -= l * buf[j];
          }
        }
      } else if (CKO_LU_SKIP) {
        if (s * G + G - 1 > c) {
          const bool below = gl + s * G > c && gl + s * G < N;
          const double l = below ? a[s][c] * inv : 0.0;
          if (below) a[s][c] = l;
          if (__any_sync(0xffffffffu, l != 0.0) && below) {
#pragma unroll
            for (int j = c + 1; j < N; ++j) a[s][j] -= l * buf[j];
          }
        }
      } else if (s * G + G - 1 > c && gl + s * G > c && gl + s * G < N) {
        const double l = a[s][c] * inv;
        a[s][c] = l;
#pragma unroll
        for (int j = c + 1; j < N; ++j) a[s][j] -= l * buf[j];
      }
    };
    if (kLookahead && c + 1 < N) {
      // look-ahead: the slot holding row c + 1 first, its owner publishes it for the next
      // column while the other slot updates
      const int sn = (c + 1) / G;
      update(sn);
      if (gl == (c + 1) % G) publish_row<N>(pb + ((c + 1) & 1) * kPbRow<N>, a[sn], c + 1);
#pragma unroll
      for (int s = 0; s < R; ++s)
        if (s != sn) update(s);
    } else {
#pragma unroll
      for (int s = 0; s < R; ++s) update(s);
    }
  }
  __syncwarp();  // rec scratch reads done before the factors overwrite it
  int* perm = reinterpret_cast<int*>(rec + Rec<N>::PERM);
#pragma unroll
  for (int s = 0; s < R; ++s) {
    const int i = gl + s * G;
    if (i < N) {
      store_row<N>(rec + i * N, a[s]);
      perm[i] = orig[s];
    }
  }
  if (gl == 0) perm[N] = swapped ? 0 : 1;
  __syncwarp();
  // singularity (|pivot| < 1e-14 max|a| or a zero pivot) from the stored U diagonal
  double pmin = INFINITY;
#pragma unroll
  for (int s = 0; s < R; ++s) {
    const int i = gl + s * G;
    if (i < N) pmin = fmin(pmin, fabs(rec[i * N + i]));
  }
  pmin = group_min<G>(pmin, base, gl);
  lmf = group_max_f<G>(lmf, base, gl);
  if (pmin == 0.0) return kLuSingular;
  if (lmf != lmf) return kLuCheckExact;
  const double mhi = __hiloint2double(__float_as_int(lmf), 0);  // <= max|a| < mhi (1 + 2^-20)
  const double lo = 1e-14 * mhi;
  if (pmin < lo) return kLuSingular;
  if (pmin >= lo * (1.0 + 0x1p-18)) return kLuOk;
  return kLuCheckExact;  // within 2^-18 of the threshold: the caller decides on the exact max
}

// Exact form of the singularity test (rare: huge/non-finite entries or a
// pivot within 2^-18 of the threshold): `rows(m)` rebuilds the block's
// entries (in any row/column order — the adjoint passes the untransposed
// rows) for the exact max |a|; the pivots are read from the stored factors.
template <int N, class Rows>
__device__ inline bool lu_exact_check(const Rows& rows, const double* rec, int gl, int base) {
  constexpr int G = Geo<N>::G, R = Geo<N>::R;
  double m[R][N];
  rows(m);
  double lm = 0.0, pmin = INFINITY;
#pragma unroll
  for (int s = 0; s < R; ++s) {
    const int i = gl + s * G;
    if (i < N) {
#pragma unroll
      for (int j = 0; j < N; ++j) lm = fmax(lm, fabs(m[s][j]));
      pmin = fmin(pmin, fabs(rec[i * N + i]));
    }
  }
  const double tiny = 1e-14 * group_max_nonneg<G>(lm, base, gl);
  pmin = group_min<G>(pmin, base, gl);
  return !(pmin < tiny || pmin == 0.0);
}

// Build the block with `build(m)` (rows this lane holds) and factor it;
// `rows` rebuilds the entries for the rare exact singularity test.
template <int N, bool kPred = false, class Build, class Rows>
__device__ inline bool factor_block(const Build& build, const Rows& rows, int gl, int base, double* pb, double* rec) {
  int st;
  {
    double m[Geo<N>::R][N];
    build(m);
    st = lu_group<N, kPred>(m, gl, base, pb, rec);
  }
  if (__any_sync(0xffffffffu, st == kLuCheckExact)) {
    const bool ok = lu_exact_check<N>(rows, rec, gl, base);
    if (st == kLuCheckExact) return ok;
  }
  return st == kLuOk;
}

// lu_solve_vec (linalg.cpp:46-60) from a record, one thread: v <- M^{-1} v.
// Rows go in blocks of B whose multiply-add chains advance together (B
// independent chains keep the FP64 pipe busy). The forward sweep accumulates
// each row in the reference's order (j ascending, bit-identical); the backward
// sweep accumulates j descending so a row's chain can start before the row
// just below it is final (a rounding-level reordering of the reference's
// j-ascending sum). vs: this thread's N-double scratch for the permuted gather.
template <int N>
__device__ inline void lu_solve_rec(const double* __restrict__ rec_in, double* vs, double (&v)[N]) {
#ifndef CKO_SOLVE_B
#define CKO_SOLVE_B 4  // substitution rows per block (knob; 2 / 5 / 8 measured equal or slower)
#endif
  constexpr int B = CKO_SOLVE_B;
  const double* rec = static_cast<const double*>(__builtin_assume_aligned(rec_in, 16));
  const int* perm = reinterpret_cast<const int*>(rec + Rec<N>::PERM);
  double y[N];
  if (perm[N]) {
#pragma unroll
    for (int i = 0; i < N; ++i) y[i] = v[i];
  } else {
#pragma unroll
    for (int i = 0; i < N; ++i) vs[i] = v[i];
#pragma unroll
    for (int i = 0; i < N; ++i) y[i] = vs[perm[i]];
  }
  // forward (unit lower): y_i -= L_ij y_j, j ascending
#pragma unroll
  for (int lo = 1; lo < N; lo += B) {
    const int hi = lo + B - 1 < N - 1 ? lo + B - 1 : N - 1;  // block rows lo..hi
#pragma unroll
    for (int j = 0; j < hi; ++j)
#pragma unroll
      for (int i = lo; i <= hi; ++i)
        if (j < i) y[i] -= rec[i * N + j] * y[j];
  }
  // backward: y_i = (y_i - U_ij y_j (j descending)) / U_ii
#pragma unroll
  for (int hi = N - 1; hi >= 0; hi -= B) {
    const int lo = hi - B + 1 > 0 ? hi - B + 1 : 0;
#pragma unroll
    for (int j = N - 1; j >= lo; --j) {
      if (j <= hi) y[j] *= rec[Rec<N>::RD + j];
#pragma unroll
      for (int i = lo; i <= hi; ++i)
        if (i < j) y[i] -= rec[i * N + j] * y[j];
    }
  }
#pragma unroll
  for (int i = 0; i < N; ++i) v[i] = y[i];
}

// The consumer's lane split over a group of TPL threads: thread gt of the group
// holds rows gt, gt + TPL, ... (R of them), so one lane's substitution chain
// advances TPL rows per step instead of one.
#ifndef CKO_COOP_CONSUMER
#define CKO_COOP_CONSUMER 0  // knob: 1 = each lane on a thread group (measured: no gain, adjoint slower)
#endif
template <int N, int TPL>
struct Coop {
  static constexpr int R = (N + TPL - 1) / TPL;
};

// v <- M^{-1} v (lu_solve_vec, linalg.cpp:46-60) on a TPL-thread group: the
// permuted gather goes through the lane's shared scratch `vs`; every finished
// entry is broadcast to the group by a shuffle. The forward sweep subtracts
// in the reference's order (j ascending); the backward sweep finishes y_j and
// then removes it from the rows above (the same rounding-level reordering as
// lu_solve_rec).
template <int N, int TPL>
__device__ __forceinline__ void lu_solve_coop(const double* __restrict__ rec, double* vs,
                                              double (&y)[Coop<N, TPL>::R], int gt, int gbase, bool writer) {
  constexpr int R = Coop<N, TPL>::R;
  const int* perm = reinterpret_cast<const int*>(rec + Rec<N>::PERM);
  if (!perm[N]) {
    __syncwarp();
#pragma unroll
    for (int s = 0; s < R; ++s) {
      const int i = gt + s * TPL;
      if (writer && i < N) vs[i] = y[s];
    }
    __syncwarp();
#pragma unroll
    for (int s = 0; s < R; ++s) {
      const int i = gt + s * TPL;
      if (i < N) y[s] = vs[perm[i]];
    }
  }
#pragma unroll
  for (int j = 0; j < N - 1; ++j) {
    const double yj = __shfl_sync(0xffffffffu, y[j / TPL], gbase + j % TPL);
#pragma unroll
    for (int s = 0; s < R; ++s) {
      const int i = gt + s * TPL;
      if (s * TPL + TPL - 1 > j && i > j && i < N) y[s] -= rec[i * N + j] * yj;
    }
  }
#pragma unroll
  for (int j = N - 1; j >= 0; --j) {
    if (gt == j % TPL) y[j / TPL] *= rec[Rec<N>::RD + j];
    const double yj = __shfl_sync(0xffffffffu, y[j / TPL], gbase + j % TPL);
#pragma unroll
    for (int s = 0; s < R; ++s) {
      const int i = gt + s * TPL;
      if (s * TPL < j && i < j) y[s] -= rec[i * N + j] * yj;
    }
  }
}

// M^{-1} from the factors in `rec` (P M = L U): lane gl of the block's group
// solves M x = e_j for its columns j = gl, gl + G, ... (L y = P e_j, U x = y,
// the reference's substitution order) and writes them to rec[INV]. The
// consumer then applies M^{-1} as one matrix-vector product whose rows are
// independent, instead of a 2N-long dependent substitution chain.
#ifndef CKO_INV_FENCE
#define CKO_INV_FENCE 0  // knob: compiler fence between the factor rows of the inverse (measured: slower)
#endif
template <int N>
__device__ inline void lu_inverse_group(double* rec, int gl) {
  constexpr int G = Geo<N>::G;
  constexpr int NC = (N + G - 1) / G;  // columns per lane
  const int* perm = reinterpret_cast<const int*>(rec + Rec<N>::PERM);
  const bool ident = perm[N] != 0;
  double* inv = rec + Rec<N>::INV;
  // the lane's columns side by side in registers (independent chains); each factor row is loaded once per
  // step behind a compiler fence, so the loads are not all hoisted (the producer's registers are tight)
  double y[NC][N];
  int col[NC];
#pragma unroll
  for (int c = 0; c < NC; ++c) {
    col[c] = gl + c * G;
#pragma unroll
    for (int i = 0; i < N; ++i) y[c][i] = (col[c] < N && (ident ? i == col[c] : perm[i] == col[c])) ? 1.0 : 0.0;
  }
#pragma unroll
  for (int i = 1; i < N; ++i) {  // L y = P e_j (unit lower)
    if (CKO_INV_FENCE) asm volatile("" ::: "memory");
    double li[N];
#pragma unroll
    for (int k = 0; k < i; ++k) li[k] = rec[i * N + k];
#pragma unroll
    for (int c = 0; c < NC; ++c) {
      double t0 = y[c][i], t1 = 0.0;
#pragma unroll
      for (int k = 0; k < i; ++k) {
        if (k & 1)
          t1 -= li[k] * y[c][k];
        else
          t0 -= li[k] * y[c][k];
      }
      y[c][i] = t0 + t1;
    }
  }
#pragma unroll
  for (int i = N - 1; i >= 0; --i) {  // U x = y
    if (CKO_INV_FENCE) asm volatile("" ::: "memory");
    double ui[N];
#pragma unroll
    for (int k = i + 1; k < N; ++k) ui[k] = rec[i * N + k];
    const double rd = rec[Rec<N>::RD + i];
#pragma unroll
    for (int c = 0; c < NC; ++c) {
      double t0 = y[c][i], t1 = 0.0;
#pragma unroll
      for (int k = i + 1; k < N; ++k) {
        if (k & 1)
          t1 -= ui[k] * y[c][k];
        else
          t0 -= ui[k] * y[c][k];
      }
      y[c][i] = (t0 + t1) * rd;
    }
  }
#pragma unroll
  for (int c = 0; c < NC; ++c)
    if (col[c] < N)
#pragma unroll
      for (int i = 0; i < N; ++i) inv[i * N + col[c]] = y[c][i];
}

// x <- M^{-1} v with the lane's rows on a TPL-thread group: every v_j is
// broadcast once, each thread forms its rows' dot products (j ascending).
template <int N, int TPL>
__device__ __forceinline__ void inv_apply_coop(const double* __restrict__ rec, double (&v)[Coop<N, TPL>::R], int gt,
                                               int gbase) {
  constexpr int R = Coop<N, TPL>::R;
  const double* inv = rec + Rec<N>::INV;
  double acc[R];
#pragma unroll
  for (int q = 0; q < R; ++q) acc[q] = 0.0;
#pragma unroll
  for (int j = 0; j < N; ++j) {
    const double vj = __shfl_sync(0xffffffffu, v[j / TPL], gbase + j % TPL);
#pragma unroll
    for (int q = 0; q < R; ++q) {
      const int i = gt + q * TPL;
      if (i < N) acc[q] += inv[i * N + j] * vj;
    }
  }
#pragma unroll
  for (int q = 0; q < R; ++q) v[q] = acc[q];
}

// Threads per lane for a tile of LTc lanes (the largest power of two that fits the warp).
__device__ __forceinline__ int coop_tpl(int LTc) {
  return LTc <= 1 ? 32 : LTc <= 2 ? 16 : LTc <= 4 ? 8 : LTc <= 8 ? 4 : LTc <= 16 ? 2 : 1;
}

template <int N>
__device__ __forceinline__ void load_vec(const double* __restrict__ p, double (&v)[N]) {
#pragma unroll
  for (int i = 0; i < N; ++i) v[i] = p[i];
}

// ---------------------------------------------------------------------------
// forward
// ---------------------------------------------------------------------------
// The producer/consumer ring of one epoch is flattened over work items
// i = k * LTc + lane (row k of lane `lane` of the tile): slot j holds the RS
// records of items j RS .. j RS + RS - 1, so no producer group idles when the
// tile has fewer lanes than a set has groups. Set s fills slots s, s + S, ...
// into ring position j % Q; full(q) = barrier 1 + q, empty(q) = 1 + Q + q.
// The consumer syncs each slot once, in order, and releases a slot when the
// rows it serves are solved (only if a later slot reuses the position).
struct RingConsumer {
  int RS, Q, LTc, J, nthr, synced, released;
  __device__ RingConsumer(int rs, int q, int ltc, int c, int n)
      : RS(rs), Q(q), LTc(ltc), J((c * ltc + rs - 1) / rs), nthr(n), synced(0), released(0) {}
  __device__ __forceinline__ void acquire(int k) {  // every slot holding an item of row k
    const int need = ((k + 1) * LTc - 1) / RS;
    while (synced <= need) {
      bar_sync(1 + synced % Q, nthr);
      ++synced;
    }
  }
  __device__ __forceinline__ void release(int k) {  // slots whose items all belong to rows <= k
    const int done = ((k + 1) * LTc) / RS;
    while (released < done) {
      if (released + Q < J) bar_arrive(1 + Q + released % Q, nthr);
      ++released;
    }
  }
  __device__ __forceinline__ int record(int k, int lane) const {
    const int i = k * LTc + lane;
    return (i / RS % Q) * RS + i % RS;
  }
};

// CKO_TRACE diagnostics record the second chunk (the first one runs cold).
__device__ __forceinline__ int trace_step(const FwdLaunch& a) { return a.nt > a.nc ? a.nc : 0; }

struct FwdCtx {
  int lb0, L, step, c;
  size_t row;  // nb * N
};

__device__ __forceinline__ void cp_async8(double* smem_dst, const double* gsrc) {
  const unsigned s = (unsigned)__cvta_generic_to_shared(smem_dst);
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(s), "l"(gsrc) : "memory");
}
__device__ __forceinline__ void cp_async16(double* smem_dst, const double* gsrc) {
  const unsigned s = (unsigned)__cvta_generic_to_shared(smem_dst);
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(s), "l"(gsrc) : "memory");
}
__device__ __forceinline__ void cp_async_wait_all() { asm volatile("cp.async.wait_all;" ::: "memory"); }

__device__ __forceinline__ unsigned dyn_smem_bytes() {
  unsigned r;
  asm("mov.u32 %0, %%dynamic_smem_size;" : "=r"(r));
  return r;
}

// Residual + lane norms for all c x L points of this CTA (rate_residual_norms,
// integrate.cpp:64-95). The chunk's iterate yy_k lives in its final place,
// trajectory row step + 1 + k, so yy_{-1} = y_start is row `step`.
// *ssq (if given): this thread's sum of y_i^2 over the points it evaluated (its
// share of the Frobenius loss of the chunk's rows once the chunk converges).
template <class MS>
__device__ unsigned residual2(const FwdLaunch& a, const FwdCtx& x, const double* cs, double* hr, double* nrm,
                              double* stage, int cap, bool first, unsigned* s_flags, double* ssq,
                              unsigned long long* rtr = nullptr) {
  double sq = 0.0;
  constexpr int N = MS::N;
  const int nb = a.nb, L = x.L, LN = L * N, P = x.c * L;
  // Staged in shared memory (the idle record ring): the CTA's lanes of one
  // trajectory row are L N contiguous doubles, so rows come in and residuals
  // go out (hr is point-major, contiguous over the chunk) fully coalesced.
  if (P <= cap / 4) {  // point norms in shared memory too when they fit
    nrm = stage + cap - P;
    cap -= P;
  }
  // lanes per staged tile: all of them when at least 4 rows fit, else fewer (wide CTAs)
  int Lt = L;
  if (cap < 9 * LN + 9 * L) Lt = max(1, min(L, cap / (9 * (N + 1))));
  const int LtN = Lt * N;
#ifndef CKO_RES_DIRECT
#define CKO_RES_DIRECT 0  // knob: 1 = every point straight from L2 (no shared-memory staging)
#endif
  const int KB = CKO_RES_DIRECT ? 0 : (cap > LtN + Lt ? (cap - LtN - Lt) / (2 * LtN + Lt) : 0);  // rows per staged block
  if (KB < 1) {  // no room to stage: one point per thread straight from L2
    for (int p = threadIdx.x; p < P; p += blockDim.x) {
      const int k = p / L, lb = p % L, b = x.lb0 + lb;
      const double t = a.times[(size_t)(x.step + 1 + k) * nb + b];
      const double dt = t - a.times[(size_t)(x.step + k) * nb + b];
      double y[N], ym[N], h[N];
      load_vec<N>(a.states + (size_t)(x.step + 1 + k) * x.row + (size_t)b * N, y);
      load_vec<N>(a.states + (size_t)(x.step + k) * x.row + (size_t)b * N, ym);
      MS::rate(a.m, cs, t, y, h, b);
      double s = 0.0;
      double* o = hr + (size_t)p * N;
#pragma unroll
      for (int i = 0; i < N; ++i) {
        const double v = xsub(xsub(y[i], ym[i]), xmul(h[i], dt));
        o[i] = v;
        s = xadd(s, xmul(v, v));
        sq += y[i] * y[i];
      }
      nrm[p] = s;
    }
  }
  for (int l0 = 0; KB >= 1 && l0 < L; l0 += Lt) {
    const int Lc = min(Lt, L - l0), LcN = Lc * N;
    for (int k0 = 0; k0 < x.c; k0 += KB) {
      const int kb = min(KB, x.c - k0);
      double* Y = stage;               // trajectory rows step + k0 .. step + k0 + kb, lanes l0 .. l0 + Lc
      double* T = Y + (kb + 1) * LcN;  // their times
      double* O = T + (kb + 1) * Lc;   // residuals of rows k0 .. k0 + kb - 1
      const double* src = a.states + (size_t)(x.step + k0) * x.row + (size_t)(x.lb0 + l0) * N;
      // asynchronous copies: every element in flight at once instead of one L2 round trip per element
      {
        // thread -> (row, 16-byte unit): several rows per pass, no divisions in the loop
        constexpr int U = N % 2 == 0 ? 2 : 1;  // doubles per copy unit (rows stay 16-byte aligned for even N)
        const int W = LcN / U, rpp = blockDim.x >= W ? blockDim.x / W : 1;
        const int r0 = threadIdx.x / W, e0 = threadIdx.x - r0 * W;
        if (r0 < rpp)
          for (int rr = r0; rr <= kb; rr += rpp)
            for (int e = e0; e < W; e += blockDim.x) {
              if constexpr (U == 2)
                cp_async16(Y + rr * LcN + 2 * e, src + (size_t)rr * x.row + 2 * e);
              else
                cp_async8(Y + rr * LcN + e, src + (size_t)rr * x.row + e);
            }
      }
      const double* ts = a.times + (size_t)(x.step + k0) * nb + x.lb0 + l0;
      for (int e = threadIdx.x; e < (kb + 1) * Lc; e += blockDim.x) {
        const int rr = e / Lc;
        cp_async8(T + e, ts + (size_t)rr * nb + (e - rr * Lc));
      }
      cp_async_wait_all();
      __syncthreads();
      if (rtr && k0 == 0 && l0 == 0) rtr[3] = globaltimer_ns();
      for (int p = threadIdx.x; p < kb * Lc; p += blockDim.x) {
        const int kk = p / Lc, lt = p - kk * Lc, lb = l0 + lt, b = x.lb0 + lb;
        const double t = T[(kk + 1) * Lc + lt];
        const double dt = t - T[kk * Lc + lt];
        double y[N], ym[N], h[N];
        load_vec<N>(Y + (kk + 1) * LcN + lt * N, y);
        load_vec<N>(Y + kk * LcN + lt * N, ym);
        MS::rate(a.m, cs, t, y, h, b);
        double s = 0.0;
        double* o = O + p * N;
#pragma unroll
        for (int i = 0; i < N; ++i) {
          const double v = xsub(xsub(y[i], ym[i]), xmul(h[i], dt));
          o[i] = v;
          s = xadd(s, xmul(v, v));
          sq += y[i] * y[i];
        }
        nrm[(k0 + kk) * L + lb] = s;
      }
      __syncthreads();
      if (rtr && k0 == 0 && l0 == 0) rtr[4] = globaltimer_ns();
      if (Lc == L) {  // the block's residuals are one contiguous run of hr
        double* dst = hr + (size_t)k0 * LN;
        for (int e = threadIdx.x; e < kb * LN; e += blockDim.x) dst[e] = O[e];
      } else {
        for (int e = threadIdx.x; e < kb * LcN; e += blockDim.x) {
          const int kk = e / LcN;
          hr[((size_t)(k0 + kk) * L + l0) * N + (e - kk * LcN)] = O[e];
        }
      }
      __syncthreads();
    }
  }
  if (ssq) *ssq = sq;
  if (threadIdx.x == 0) *s_flags = 0;
  if (rtr) rtr[0] = globaltimer_ns();
  __syncthreads();
  if (rtr) rtr[1] = globaltimer_ns();
  unsigned f = 0;
  for (int lb = threadIdx.x; lb < x.L; lb += blockDim.x) {
    const int b = x.lb0 + lb;
    double acc = 0.0;
    for (int k = 0; k < x.c; ++k) acc = xadd(acc, nrm[k * x.L + lb]);
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
  if (rtr) rtr[2] = globaltimer_ns();
  __syncthreads();
  return *s_flags;
}

// Streamed time grid: block until rows [0, rows) of a.times have landed (the
// host uploads the grid in pieces on a copy stream while the forward runs; the
// piece boundaries are 128-byte aligned, so no cache line straddles a piece).
// The whole CTA calls it; false on timeout.
__device__ inline bool wait_times_rows(const FwdLaunch& a, int rows) {
  __shared__ int s_ok;
  if (threadIdx.x == 0) {
    const unsigned long long want = a.times_tag + (unsigned long long)rows;
    const uint64_t t0 = globaltimer_ns();
    int ok = 1;
    for (;;) {
      unsigned long long v;
      asm volatile("ld.acquire.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(a.times_ready) : "memory");
      if (v >= want) break;
      if (globaltimer_ns() - t0 > a.budget_ns) {
        ok = 0;
        break;
      }
      __nanosleep(256);
    }
    s_ok = ok;
  }
  __syncthreads();
  return s_ok != 0;
}

// This thread's [committed, pending] sums of y^2 (global, after the per-CTA
// partials: nothing stays live in registers through the factorisations).
__device__ __forceinline__ double* loss_slot(const FwdLaunch& a) {
  return a.loss_part + a.grid + 2 * ((size_t)blockIdx.x * blockDim.x + threadIdx.x);
}

// The CTA's Frobenius-loss partial (sum of y^2 over its converged rows) in a
// fixed order: warp sums, then warp 0 over the warps. The whole CTA calls it.
__device__ inline void fwd_loss_store(double* loss_part, double v) {
  __shared__ double red[32];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = (blockDim.x + 31) >> 5;
  for (int o = 16; o > 0; o >>= 1) v += __shfl_down_sync(0xffffffffu, v, o);
  __syncthreads();
  if (lane == 0) red[warp] = v;
  __syncthreads();
  if (threadIdx.x == 0) {
    double s = 0.0;
    for (int w = 0; w < nw; ++w) s += red[w];
    loss_part[blockIdx.x] = s;
  }
}

// The Frobenius loss L for the adjoint's dL/dy = y / L: the device scalar, or —
// straight after the forward that left per-CTA sums of y^2 — their sum (warp 0,
// fixed order; every CTA forms the same value) and CTA 0 publishes it. The whole
// CTA calls it.
__device__ inline double adj_loss_value(const AdjLaunch& a) {
  if (!a.loss_part) return a.loss ? *a.loss : 0.0;
  __shared__ double s_L;
  if (threadIdx.x < 32) {
    double v = 0.0;
    for (int i = threadIdx.x; i < a.loss_nparts; i += 32) v += a.loss_part[i];
    for (int o = 16; o > 0; o >>= 1) v += __shfl_down_sync(0xffffffffu, v, o);
    if (threadIdx.x == 0) {
      s_L = sqrt(v);
      if (blockIdx.x == 0) *a.loss_out = s_L;
    }
  }
  __syncthreads();
  return s_L;
}

// One Newton iteration over the rows of one lane tile (integrate.cpp:208-231).
template <class MS, bool INV>
__device__ void fwd_epoch(const FwdLaunch& a, const FwdCtx& x, const Shape& sh, const double* cs, double* recs,
                          double* pbs, double* vss, const double* hr, int t0, int LTc, unsigned* s_sing) {
  constexpr int N = MS::N;
  constexpr int kStride = INV ? Rec<N>::STRIDE_INV : Rec<N>::STRIDE;
  using Gm = Geo<N>;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int S = sh.S, Q = sh.Q, Ws = sh.Ws;
  const int nthr = 32 * (Ws + 1);
  const int nb = a.nb;
  const int pw = producer_of(warp);
  if (pw >= 0 && pw < S * Ws) {
    // ---- producer: J -> M = I - J dt -> LU for rows k = s, s + S, ...; it
    // also stages r_k and yy_k in the record so the consumer never waits on L2.
    const int s = pw / Ws, sw = pw % Ws;
    const GroupLane<N> gr(lane);
    const int g = gr.g, gl = gr.gl;
    const int gi = sw * Gm::GPW + g;  // record within the slot
    const int RS = sh.RS, I = x.c * LTc, J = (I + RS - 1) / RS;
    double* pb = pbs + (size_t)(s * RS + gi) * kPb<N>;
    unsigned long long* tr0 = (a.trace && blockIdx.x == 0 && x.step == trace_step(a) && lane == 0) ? a.trace + 64 : nullptr;
    for (int js0 = 0; js0 < J; js0 += S) {
      // the sets advance in rounds: producer warps stay at nearby code (instruction-cache locality)
      if (kFwdRounds && js0 > 0 && (js0 / S) % kRoundEvery == 0) producer_round_sync(warp, S * Ws);
      const int js = js0 + s;
      if (js >= J) continue;
      const int q = js % Q;
      const bool active = js * RS + gi < I;  // inactive groups factor a duplicate item, no side effects
      const int item = active ? js * RS + gi : I - 1;
      const int k = item / LTc, lb = t0 + item % LTc, b = x.lb0 + lb;
      double* rec = recs + (size_t)(q * RS + gi) * kStride;
      unsigned long long* tr = (tr0 && js < x.c) ? tr0 + js * 8 : nullptr;  // slot js: tr[js * 8 + 0..3]
      if (tr) tr[0] = globaltimer_ns();
      // the point's iterate and residual entries (global) are requested before the slot wait: their
      // latency overlaps it and the row build
      [[maybe_unused]] double ye[Gm::R], re[Gm::R];
      if constexpr (kFwdEarlyLoads >= 1) {
        const double* yrow = a.states + (size_t)(x.step + 1 + k) * x.row + (size_t)b * N;
        const double* rrow = hr + (size_t)(k * x.L + lb) * N;
#pragma unroll
        for (int q2 = 0; q2 < Gm::R; ++q2) {
          const int i = gl + q2 * Gm::G;
          ye[q2] = i < N ? yrow[i] : 0.0;
          re[q2] = i < N ? rrow[i] : 0.0;
        }
      }
      double t, dt;
      if constexpr (kFwdEarlyLoads >= 2) {  // the step size before the slot wait too
        t = a.times[(size_t)(x.step + 1 + k) * nb + b];
        dt = t - a.times[(size_t)(x.step + k) * nb + b];
      }
      if (js >= Q) bar_sync(1 + Q + q, nthr);
      if (tr) tr[1] = globaltimer_ns();
      if constexpr (kFwdEarlyLoads < 2) {
        t = a.times[(size_t)(x.step + 1 + k) * nb + b];
        dt = t - a.times[(size_t)(x.step + k) * nb + b];
      }
      double y[N];
      load_vec<N>(a.states + (size_t)(x.step + 1 + k) * x.row + (size_t)b * N, y);
      [[maybe_unused]] const double* r = hr + (size_t)(k * x.L + lb) * N;
      const double ndt = -dt;
      auto build = [&](double (&m)[Gm::R][N]) {
#pragma unroll
        for (int q = 0; q < Gm::R; ++q) {
          const int i = gl + q * Gm::G;
          if (i < N) {
            if constexpr (kFwdSlotRows && HasSlotRows<MS>::value && Gm::G == MS::N / 2) {
              MS::m_row_slot(cs, q, gl, ndt, m[q]);  // lane gl: position row gl, velocity row N/2 + gl
            } else if constexpr (kFwdSharedJac && HasConstJac<MS>::value) {  // M = -dt J + I from shared memory
              const double* Jr = cs + MS::JOFF + i * N;
              const double* Er = MS::unit_row(cs, i);
#pragma unroll
              for (int j = 0; j < N; ++j) m[q][j] = xadd(xmul(ndt, Jr[j]), Er[j]);
            } else {
              MS::jac_row(a.m, cs, t, y, i, m[q], b);
#pragma unroll
              for (int j = 0; j < N; ++j) {
                m[q][j] = xmul(ndt, m[q][j]);
                if (j == i) m[q][j] = xadd(m[q][j], 1.0);
              }
            }
            if constexpr (kFwdEarlyLoads >= 1) {
              rec[Rec<N>::Y + i] = ye[q];
              rec[Rec<N>::RHS + i] = re[q];
            } else {
              rec[Rec<N>::Y + i] = a.states[(size_t)(x.step + 1 + k) * x.row + (size_t)b * N + i];
              rec[Rec<N>::RHS + i] = r[i];
            }
          } else {
#pragma unroll
            for (int j = 0; j < N; ++j) m[q][j] = 0.0;
          }
        }
      };
      if (tr) tr[2] = globaltimer_ns();
      if (!factor_block<N, kFwdPred>(build, build, gl, gr.base, pb, rec) && active && gl == 0) {
        atomicMin(a.sing_key, (unsigned long long)k * nb + b);
        atomicOr(s_sing, 1u);
      }
      if constexpr (INV) {
        __syncwarp();
        lu_inverse_group<N>(rec, gl);
      }
      if (tr) tr[3] = globaltimer_ns();
      bar_arrive(1 + q, nthr);
    }
  } else if (INV && warp == 0) {
    // ---- consumer with explicit inverses: x_k = M_k^{-1}(r_k + x_{k-1}) as one product, each lane on a group
    const int tpl = coop_tpl(LTc);
    auto run = [&](auto tag) {
      constexpr int TPL = decltype(tag)::value;
      constexpr int R = Coop<N, TPL>::R;
      const int lt = lane / TPL, gt = lane % TPL, gbase = lt * TPL;
      const bool active = lt < LTc;
      const int ltc = active ? lt : LTc - 1;
      const int b = x.lb0 + t0 + ltc;
      double xv[R];
#pragma unroll
      for (int q = 0; q < R; ++q) xv[q] = 0.0;
      unsigned long long* tr =
          (a.trace && blockIdx.x == 0 && x.step == trace_step(a) && lane == 0) ? a.trace + 64 : nullptr;
      RingConsumer ring(sh.RS, Q, LTc, x.c, nthr);
      for (int k = 0; k < x.c; ++k) {
        if (tr) tr[k * 8 + 4] = globaltimer_ns();
        ring.acquire(k);
        if (tr) tr[k * 8 + 5] = globaltimer_ns();
        const double* rec = recs + (size_t)ring.record(k, ltc) * kStride;
#pragma unroll
        for (int q = 0; q < R; ++q) {
          const int i = gt + q * TPL;
          if (i < N) xv[q] = rec[Rec<N>::RHS + i] + xv[q];
        }
        inv_apply_coop<N, TPL>(rec, xv, gt, gbase);
        double* yy = a.states + (size_t)(x.step + 1 + k) * x.row + (size_t)b * N;
#pragma unroll
        for (int q = 0; q < R; ++q) {
          const int i = gt + q * TPL;
          if (active && i < N) yy[i] = rec[Rec<N>::Y + i] - xv[q];
        }
        if (tr) tr[k * 8 + 6] = globaltimer_ns();
        ring.release(k);
      }
    };
    static_assert(kInvMaxLanes <= 2, "explicit-inverse consumers are instantiated for 1 or 2 lanes per tile");
    if (tpl == 32)
      run(std::integral_constant<int, 32>{});
    else
      run(std::integral_constant<int, 16>{});
  } else if (warp == 0 && CKO_COOP_CONSUMER) {
    // ---- consumer: x_k = M_k^{-1}(r_k + x_{k-1}), yy_k -= x_k, each lane on a group of threads
    const int tpl = coop_tpl(LTc);
    auto run = [&](auto tag) {
      constexpr int TPL = decltype(tag)::value;
      constexpr int R = Coop<N, TPL>::R;
      const int lt = lane / TPL, gt = lane % TPL, gbase = lt * TPL;
      const bool active = lt < LTc;
      const int ltc = active ? lt : LTc - 1;  // idle groups shadow the last lane (no stores)
      const int b = x.lb0 + t0 + ltc;
      double* vs = vss + (size_t)ltc * N;
      double xv[R];
#pragma unroll
      for (int q = 0; q < R; ++q) xv[q] = 0.0;
      RingConsumer ring(sh.RS, Q, LTc, x.c, nthr);
      for (int k = 0; k < x.c; ++k) {
        ring.acquire(k);
        const double* rec = recs + (size_t)ring.record(k, ltc) * kStride;
#pragma unroll
        for (int q = 0; q < R; ++q) {
          const int i = gt + q * TPL;
          if (i < N) xv[q] = rec[Rec<N>::RHS + i] + xv[q];
        }
        lu_solve_coop<N, TPL>(rec, vs, xv, gt, gbase, active);
        double* yy = a.states + (size_t)(x.step + 1 + k) * x.row + (size_t)b * N;
#pragma unroll
        for (int q = 0; q < R; ++q) {
          const int i = gt + q * TPL;
          if (active && i < N) yy[i] = rec[Rec<N>::Y + i] - xv[q];
        }
        ring.release(k);
      }
    };
    switch (tpl) {
      case 32: run(std::integral_constant<int, 32>{}); break;
      case 16: run(std::integral_constant<int, 16>{}); break;
      case 8: run(std::integral_constant<int, 8>{}); break;
      case 4: run(std::integral_constant<int, 4>{}); break;
      case 2: run(std::integral_constant<int, 2>{}); break;
      default: run(std::integral_constant<int, 1>{}); break;
    }
  } else if (warp == 0) {
    // ---- consumer: x_k = M_k^{-1}(r_k + x_{k-1}), yy_k -= x_k, one thread per lane
    const int lt = lane;
    const bool active = lt < LTc;
    const int lb = t0 + lt, b = x.lb0 + lb;
    double xv[N];
#pragma unroll
    for (int i = 0; i < N; ++i) xv[i] = 0.0;
    double* vs = vss + (size_t)lt * N;
    unsigned long long* tr = (a.trace && blockIdx.x == 0 && x.step == trace_step(a) && lane == 0) ? a.trace + 64 : nullptr;
    RingConsumer ring(sh.RS, Q, LTc, x.c, nthr);
    for (int k = 0; k < x.c; ++k) {
      if (tr) tr[k * 8 + 4] = globaltimer_ns();
      ring.acquire(k);
      if (tr) tr[k * 8 + 5] = globaltimer_ns();
      if (active) {
        const double* rec = recs + (size_t)ring.record(k, lt) * kStride;
#pragma unroll
        for (int i = 0; i < N; ++i) xv[i] = rec[Rec<N>::RHS + i] + xv[i];
        lu_solve_rec<N>(rec, vs, xv);
        double* yy = a.states + (size_t)(x.step + 1 + k) * x.row + (size_t)b * N;
#pragma unroll
        for (int i = 0; i < N; ++i) yy[i] = rec[Rec<N>::Y + i] - xv[i];
      }
      if (tr) tr[k * 8 + 6] = globaltimer_ns();
      ring.release(k);
    }
  }
}

}  // namespace v2
}  // namespace cko
#include "cko_sparse.cuh"
namespace cko {
namespace v2 {

// SP: the structured (arrow + tridiagonal) records of cko_sparse.cuh instead of the group LU.
template <class MS, bool INV, bool SP = false>
__global__ void __launch_bounds__(SP ? 32 * kSpWarps : 32 * kMaxWarps, 1) fwd2_kernel(FwdLaunch a, Shape sh) {
  constexpr int N = MS::N;
  const int kStride = sh.stride;
  extern __shared__ __align__(16) double smem[];
  __shared__ unsigned s_bcast, s_flags, s_sing, s_fb;
  int o_cs, o_rec, o_pb, o_vs, o_lam, tot;
  smem_layout<MS>(sh.S, sh.Q, sh.Ws, sh.RS, sh.LT, sh.stride, o_cs, o_rec, o_pb, o_vs, o_lam, tot, SP, sh.ring);
  double* cs = smem + o_cs;
  double* recs = smem + o_rec;
  double* pbs = smem + o_pb;
  double* vss = smem + o_vs;
  MS::load_consts(a.m, cs);
  if (threadIdx.x == 0) s_sing = 0, s_fb = 0;
  FwdCtx x;
  lane_range(a.nb, x.lb0, x.L);
  x.row = (size_t)a.nb * N;
  double* hr = a.slab.base + (size_t)blockIdx.x * a.slab.doubles;
  // residual staging: the record ring (idle between epochs)
  const int ring_doubles = sh.ring;
  (void)kStride;
  double* nrm = hr + (size_t)a.slab.Pmax * N;
  const bool leader = blockIdx.x == 0 && threadIdx.x == 0;
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
    for (int p = threadIdx.x; p < c * x.L; p += blockDim.x) {  // initial iterate: every row at y_start
      const int k = p / x.L, b = x.lb0 + p % x.L;
      double v[N];
      load_vec<N>(a.states + (size_t)step * x.row + (size_t)b * N, v);  // all loads before any store
      if (a.dy_init) {
        double d[N];
        load_vec<N>(a.dy_init + ((size_t)k * a.nb + b) * N, d);
#pragma unroll
        for (int i = 0; i < N; ++i) v[i] += d[i];
      }
      double* dst = a.states + (size_t)(step + 1 + k) * x.row + (size_t)b * N;
#pragma unroll
      for (int i = 0; i < N; ++i) dst[i] = v[i];
    }
    __syncthreads();
    int it = 0;
    unsigned long long* ktr = (a.trace && blockIdx.x == 0 && threadIdx.x == 0 && chunk < 4) ? a.trace + chunk * 16 : nullptr;
    // per-CTA timeline of the traced chunk: start, res0, barrier, epoch end, res, barrier
    unsigned long long* ctr = (a.trace && threadIdx.x == 0 && step == trace_step(a))
                                  ? a.trace + 64 + 8 * (size_t)min(a.nc, a.nt) + 8 * blockIdx.x : nullptr;
    if (ctr) ctr[0] = globaltimer_ns();
    if (ktr) ktr[0] = globaltimer_ns();
    unsigned f = residual2<MS>(a, x, cs, hr, nrm, recs, ring_doubles, true, &s_flags, a.loss_part ? loss_slot(a) + 1 : nullptr, ktr ? ktr + 11 : nullptr);
    if (ktr) ktr[1] = globaltimer_ns();
    if (ctr) ctr[1] = globaltimer_ns();
    f = grid_reduce_or(a.gs, a.grp, f, a.budget_ns, &s_bcast);
    if (ctr) ctr[2] = globaltimer_ns();
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
      if (ktr && it < 4) ktr[2 + 3 * (it - 1)] = globaltimer_ns();
      for (int t0 = 0; t0 < x.L; t0 += sh.LT) {
        if constexpr (SP)
          fwd_epoch_sp<MS>(a, x, sh, cs, recs, hr, t0, min(sh.LT, x.L - t0), &s_fb);
        else
          fwd_epoch<MS, INV>(a, x, sh, cs, recs, pbs, vss, hr, t0, min(sh.LT, x.L - t0), &s_sing);
        __syncthreads();
      }
      const unsigned fl = (s_sing ? FLAG_SINGULAR : 0u) | (s_fb ? FLAG_FALLBACK : 0u);
      if (ktr && it < 4) ktr[3 + 3 * (it - 1)] = globaltimer_ns();
      if (ctr && it == 1) ctr[3] = globaltimer_ns();
      f = residual2<MS>(a, x, cs, hr, nrm, recs, ring_doubles, false, &s_flags, a.loss_part ? loss_slot(a) + 1 : nullptr) | fl;
      if (ctr && it == 1) ctr[4] = globaltimer_ns();
      f = grid_reduce_or(a.gs, a.grp, f, a.budget_ns, &s_bcast);
      if (ctr && it == 1) ctr[5] = globaltimer_ns();
      if (ktr && it < 4) ktr[4 + 3 * (it - 1)] = globaltimer_ns();
      if (f & (FLAG_TIMEOUT | FLAG_SINGULAR | FLAG_NON_FINITE | FLAG_FALLBACK)) {
        if (leader) {
          // a structured block the reference would pivot on (or call singular): the host re-runs the call
          // on the group-LU kernels, whatever else this iteration saw
          a.info[0] = (f & FLAG_TIMEOUT) ? 4 : (f & FLAG_FALLBACK) ? 5 : (f & FLAG_SINGULAR) ? 1 : 2;
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
// One reversed chunk of one lane tile (be_chunk_core, adjoint.cpp:49-127):
// rows r <-> steps m = step_hi - r. Producers: J(y_m) -> rhs_r = dL_m +
// dt J^T lambda_c, M_r = (I - J dt)^T, LU. Consumer: delta_r = M_r^{-1}(rhs_r +
// delta_{r-1}), quadrature weight w_m = (lambda_c + delta_r) dt, and the new
// carry lambda_c += delta_{c-1}.
template <class MS, bool INV>
__device__ void adj_epoch(const AdjLaunch& a, const Shape& sh, const double* cs, double* recs, double* pbs,
                          double* vss, double* lam, int lb0, int t0, int LTc, int step_hi, int c, double Lval,
                          unsigned long long ord, double (&dcar)[MS::N]) {
  constexpr int N = MS::N;
  constexpr int kStride = INV ? Rec<N>::STRIDE_INV : Rec<N>::STRIDE;
  using Gm = Geo<N>;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int S = sh.S, Q = sh.Q, Ws = sh.Ws;
  const int nthr = 32 * (Ws + 1);
  const int nb = a.nb;
  const size_t row = (size_t)nb * N;
  const double rL = Lval > 0.0 ? 1.0 / Lval : 0.0;  // y / L by div_rn
  (void)rL;
  const int pw = producer_of(warp);
  if (pw >= 0 && pw < S * Ws) {
    const int s = pw / Ws, sw = pw % Ws;
    const GroupLane<N> gr(lane);
    const int g = gr.g, gl = gr.gl;
    const int gi = sw * Gm::GPW + g;  // record within the slot
    const int RS = sh.RS, I = c * LTc, J = (I + RS - 1) / RS;
    double* pb = pbs + (size_t)(s * RS + gi) * kPb<N>;
    for (int js0 = 0; js0 < J; js0 += S) {
      // the sets advance in rounds: producer warps stay at nearby code (instruction-cache locality)
      if (js0 > 0 && (js0 / S) % kRoundEvery == 0) producer_round_sync(warp, S * Ws);
      const int js = js0 + s;
      if (js >= J) continue;
      const int q = js % Q;
      const bool active = js * RS + gi < I;  // inactive groups factor a duplicate item, no side effects
      const int item = active ? js * RS + gi : I - 1;
      const int r = item / LTc, ltc = item % LTc;
      const int b = lb0 + t0 + ltc;
      const double* lm = lam + (size_t)ltc * N;
      double* rec = recs + (size_t)(q * RS + gi) * kStride;
      const int m = step_hi - r;
      // (8) the point's times, (16) its y (or dL) entries, requested before the slot wait
      [[maybe_unused]] double yq8[Gm::R];
      double t, dt;
      if constexpr ((kAdjLeanRhs & 16) != 0) {  // (16) the y entries too
#pragma unroll
        for (int q2 = 0; q2 < Gm::R; ++q2) {
          const int i = gl + q2 * Gm::G;
          yq8[q2] = i < N ? (a.dL ? a.dL : a.states)[(size_t)m * row + (size_t)b * N + i] : 0.0;
        }
      }
      if constexpr ((kAdjLeanRhs & 8) != 0) {
        t = a.times[(size_t)m * nb + b];
        dt = t - a.times[(size_t)(m - 1) * nb + b];
      }
      if (js >= Q) bar_sync(1 + Q + q, nthr);
      if constexpr ((kAdjLeanRhs & 8) == 0) {
        t = a.times[(size_t)m * nb + b];
        dt = t - a.times[(size_t)(m - 1) * nb + b];
      }
      double y[N];
      load_vec<N>(a.states + (size_t)m * row + (size_t)b * N, y);
      // J rows into the record (scratch), then read back transposed
      auto build = [&](double (&mt)[Gm::R][N]) {
        if constexpr (HasConstJac<MS>::value) {  // J^T rows straight from shared memory
          const double ndt = -dt;
          if constexpr (kAdjLeanRhs != 0 && HasJtLambda<MS>::value) {
            double yq[Gm::R];  // (4) the point's y (or user dL) entries first: latency under the row build
            if constexpr ((kAdjLeanRhs & 16) != 0) {
#pragma unroll
              for (int q = 0; q < Gm::R; ++q) yq[q] = yq8[q];
            } else if constexpr ((kAdjLeanRhs & 4) != 0) {
#pragma unroll
              for (int q = 0; q < Gm::R; ++q) {
                const int i = gl + q * Gm::G;
                yq[q] = i < N ? (a.dL ? a.dL : a.states)[(size_t)m * row + (size_t)b * N + i] : 0.0;
              }
            }
#pragma unroll
            for (int q = 0; q < Gm::R; ++q) {
              const int i = gl + q * Gm::G;
              if (i < N) {
                const double* JTr = cs + MS::JTOFF + i * N;  // J[j][i], j = 0 .. N-1
                const double* Er = MS::unit_row(cs, i);
                double tmp = 0.0;  // (J^T lambda)_i (gemv_transpose)
                if constexpr ((kAdjLeanRhs & 1) != 0) {
#pragma unroll
                  for (int j = 0; j < N; ++j) mt[q][j] = xadd(xmul(ndt, JTr[j]), Er[j]);
                  tmp = MS::jt_lambda(cs, i, lm);  // (1) structural nonzeros only: the dense sum's value
                } else {
#pragma unroll
                  for (int j = 0; j < N; ++j) {
                    const double x = JTr[j];
                    tmp += x * lm[j];
                    mt[q][j] = xadd(xmul(ndt, x), Er[j]);
                  }
                }
                if constexpr ((kAdjLeanRhs & 20) == 0)
                  yq[q] = (a.dL ? a.dL : a.states)[(size_t)m * row + (size_t)b * N + i];
                double dl;
                if constexpr ((kAdjLeanRhs & 2) != 0)  // (2) y / L from the reciprocal, one correction
                  dl = a.dL ? yq[q] : (Lval > 0.0 ? div_rn(yq[q], Lval, rL) : 0.0);
                else
                  dl = a.dL ? yq[q] : (Lval > 0.0 ? yq[q] / Lval : 0.0);
                rec[Rec<N>::RHS + i] = dl + dt * tmp;
              } else {
#pragma unroll
                for (int j = 0; j < N; ++j) mt[q][j] = 0.0;
              }
            }
          } else {
#pragma unroll
          for (int q = 0; q < Gm::R; ++q) {
            const int i = gl + q * Gm::G;
            if (i < N) {
              const double* JTr = cs + MS::JTOFF + i * N;  // J[j][i], j = 0 .. N-1
              const double* Er = MS::unit_row(cs, i);
              double tmp = 0.0;  // (J^T lambda)_i (gemv_transpose)
#pragma unroll
              for (int j = 0; j < N; ++j) {
                const double x = JTr[j];
                tmp += x * lm[j];
                mt[q][j] = xadd(xmul(ndt, x), Er[j]);
              }
              const double yi = a.states[(size_t)m * row + (size_t)b * N + i];
              const double dl = a.dL ? a.dL[(size_t)m * row + (size_t)b * N + i] : (Lval > 0.0 ? yi / Lval : 0.0);
              rec[Rec<N>::RHS + i] = dl + dt * tmp;
            } else {
#pragma unroll
              for (int j = 0; j < N; ++j) mt[q][j] = 0.0;
            }
          }
          }
          if (gl == 0) rec[Rec<N>::DT] = dt;
        } else {
#pragma unroll
          for (int q = 0; q < Gm::R; ++q) {
            const int i = gl + q * Gm::G;
            if (i < N) {
              double jr[N];
              MS::jac_row(a.m, cs, t, y, i, jr, b);
#pragma unroll
              for (int j = 0; j < N; ++j) rec[i * N + j] = jr[j];
            }
          }
          __syncwarp();
#pragma unroll
          for (int q = 0; q < Gm::R; ++q) {
            const int i = gl + q * Gm::G;
            if (i < N) {
#pragma unroll
              for (int j = 0; j < N; ++j) mt[q][j] = rec[j * N + i];  // J[j][i]
              double tmp = 0.0;                                      // (J^T lambda)_i (gemv_transpose)
#pragma unroll
              for (int j = 0; j < N; ++j) tmp += mt[q][j] * lm[j];
              const double yi = a.states[(size_t)m * row + (size_t)b * N + i];
              const double dl = a.dL ? a.dL[(size_t)m * row + (size_t)b * N + i] : (Lval > 0.0 ? yi / Lval : 0.0);
              rec[Rec<N>::RHS + i] = dl + dt * tmp;
#pragma unroll
              for (int j = 0; j < N; ++j) mt[q][j] = (j == i) ? 1.0 - dt * mt[q][j] : -dt * mt[q][j];
            } else {
#pragma unroll
              for (int j = 0; j < N; ++j) mt[q][j] = 0.0;
            }
          }
          if (gl == 0) rec[Rec<N>::DT] = dt;
          __syncwarp();
        }
      };
      // the entries of M^T without the transpose scratch (same values, rows of I - dt J)
      auto rows = [&](double (&mt)[Gm::R][N]) {
#pragma unroll
        for (int q = 0; q < Gm::R; ++q) {
          const int i = gl + q * Gm::G;
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
      bool fok;
      if constexpr (HasConstJac<MS>::value)
        fok = factor_block<N, true>(build, build, gl, gr.base, pb, rec);  // build leaves the factors alone
      else
        fok = factor_block<N, true>(build, rows, gl, gr.base, pb, rec);
      if (!fok && active && gl == 0)
        atomicMin(a.sing_key, ord * (unsigned long long)a.nc * nb + (unsigned long long)r * nb + b);
      if constexpr (INV) {
        __syncwarp();
        lu_inverse_group<N>(rec, gl);
      }
      bar_arrive(1 + q, nthr);
    }
  } else if ((INV || CKO_COOP_CONSUMER) && warp == 0) {
    const int tpl = coop_tpl(LTc);
    constexpr bool use_inv = INV;
    auto run = [&](auto tag) {
      constexpr int TPL = decltype(tag)::value;
      constexpr int R = Coop<N, TPL>::R;
      const int lt = lane / TPL, gt = lane % TPL, gbase = lt * TPL;
      const bool active = lt < LTc;
      const int ltc = active ? lt : LTc - 1;
      const int b = lb0 + t0 + ltc;
      double* vs = vss + (size_t)ltc * N;
      const double* lc = lam + (size_t)ltc * N;
      double d[R];  // delta_{r-1}, then delta_r
#pragma unroll
      for (int q = 0; q < R; ++q) d[q] = 0.0;
      RingConsumer ring(sh.RS, Q, LTc, c, nthr);
      for (int r = 0; r < c; ++r) {
        ring.acquire(r);
        const double* rec = recs + (size_t)ring.record(r, ltc) * kStride;
        const int m = step_hi - r;
#pragma unroll
        for (int q = 0; q < R; ++q) {
          const int i = gt + q * TPL;
          if (i < N) d[q] = rec[Rec<N>::RHS + i] + d[q];
        }
        const double dt = rec[Rec<N>::DT];
        if constexpr (use_inv)
          inv_apply_coop<N, TPL>(rec, d, gt, gbase);
        else
          lu_solve_coop<N, TPL>(rec, vs, d, gt, gbase, active);
        double* w = a.wq + (size_t)m * row + (size_t)b * N;
#pragma unroll
        for (int q = 0; q < R; ++q) {
          const int i = gt + q * TPL;
          if (active && i < N) w[i] = (lc[i] + d[q]) * dt;
        }
        ring.release(r);
      }
      __syncwarp();
#pragma unroll
      for (int q = 0; q < R; ++q) {  // the new carry's increment, for the caller (adjoint.cpp:121-126)
        const int i = gt + q * TPL;
        if (active && i < N) vs[i] = d[q];
      }
    };
    if constexpr (INV) {  // 1 or 2 lanes per tile (kInvMaxLanes)
      if (tpl == 32)
        run(std::integral_constant<int, 32>{});
      else
        run(std::integral_constant<int, 16>{});
    } else {
      switch (tpl) {
        case 32: run(std::integral_constant<int, 32>{}); break;
        case 16: run(std::integral_constant<int, 16>{}); break;
        case 8: run(std::integral_constant<int, 8>{}); break;
        case 4: run(std::integral_constant<int, 4>{}); break;
        case 2: run(std::integral_constant<int, 2>{}); break;
        default: run(std::integral_constant<int, 1>{}); break;
      }
    }
  } else if (warp == 0) {
    const int lt = lane;
    const bool active = lt < LTc;
    const int b = lb0 + t0 + lt;
    double* vs = vss + (size_t)lt * N;
    const double* lc = lam + (size_t)lt * N;
    double d[N];  // delta_{r-1}, then delta_r
#pragma unroll
    for (int i = 0; i < N; ++i) d[i] = 0.0;
    RingConsumer ring(sh.RS, Q, LTc, c, nthr);
    for (int r = 0; r < c; ++r) {
      ring.acquire(r);
      if (active) {
        const double* rec = recs + (size_t)ring.record(r, lt) * kStride;
        const int m = step_hi - r;
#pragma unroll
        for (int i = 0; i < N; ++i) d[i] = rec[Rec<N>::RHS + i] + d[i];
        const double dt = rec[Rec<N>::DT];
        lu_solve_rec<N>(rec, vs, d);
        double* w = a.wq + (size_t)m * row + (size_t)b * N;
        if constexpr (kAdjVecW && N % 2 == 0) {  // 16-byte streaming stores (rows of an even N stay aligned)
#pragma unroll
          for (int i = 0; i < N; i += 2) {
            const double2 l2 = *reinterpret_cast<const double2*>(lc + i);
            __stcs(reinterpret_cast<double2*>(w + i), make_double2((l2.x + d[i]) * dt, (l2.y + d[i + 1]) * dt));
          }
        } else {
#pragma unroll
          for (int i = 0; i < N; ++i) w[i] = (lc[i] + d[i]) * dt;
        }
      }
      ring.release(r);
    }
#pragma unroll
    for (int i = 0; i < N; ++i) dcar[i] = d[i];
  }
}

template <class MS, bool INV, bool SP = false>
__global__ void __launch_bounds__(SP ? 32 * kSpWarps : 32 * kMaxWarps, 1) adj2_kernel(AdjLaunch a, Shape sh) {
  constexpr int N = MS::N;
  extern __shared__ __align__(16) double smem[];
  int o_cs, o_rec, o_pb, o_vs, o_lam, tot;
  smem_layout<MS>(sh.S, sh.Q, sh.Ws, sh.RS, sh.LT, sh.stride, o_cs, o_rec, o_pb, o_vs, o_lam, tot, SP, sh.ring);
  double* cs = smem + o_cs;
  double* recs = smem + o_rec;
  double* pbs = smem + o_pb;
  double* vss = smem + o_vs;
  double* lam = smem + o_lam;
  MS::load_consts(a.m, cs);
  int lb0, L;
  lane_range(a.nb, lb0, L);
  const double Lval = adj_loss_value(a);
  const int consumer = threadIdx.x >> 5 == 0;
  const int lane = threadIdx.x & 31;
  for (int t0 = 0; t0 < L; t0 += sh.LT) {
    const int LTc = min(sh.LT, L - t0);
    for (int i = threadIdx.x; i < LTc * N; i += blockDim.x) lam[i] = 0.0;
    __syncthreads();
    int step_hi = a.nt;
    unsigned long long ord = 0;
    while (step_hi >= 1) {
      const int c = min(a.nc, step_hi);
      double dcar[N];
      if constexpr (SP) {
        if constexpr (HasJtLambda<MS>::value) {
          // (J^T lambda_c)_i per lane of the tile (gemv_transpose over J's structural nonzeros, the dense sum's
          // value), once per reversed chunk instead of per row
          for (int e = threadIdx.x; e < LTc * N; e += blockDim.x) vss[e] = MS::jt_lambda(cs, e % N, lam + (e / N) * N);
          __syncthreads();
        }
        adj_epoch_sp<MS>(a, sh, cs, recs, lam, vss, lb0, t0, LTc, step_hi, c, Lval, dcar);
      } else {
        adj_epoch<MS, INV>(a, sh, cs, recs, pbs, vss, lam, lb0, t0, LTc, step_hi, c, Lval, ord, dcar);
      }
      __syncthreads();
      if (!SP && (INV || CKO_COOP_CONSUMER)) {  // new carry (adjoint.cpp:121-126): the increments left in vss
        for (int i = threadIdx.x; i < LTc * N; i += blockDim.x) lam[i] += vss[i];
      } else if (consumer && lane < LTc) {
#pragma unroll
        for (int i = 0; i < N; ++i) lam[(size_t)lane * N + i] += dcar[i];
      }
      __syncthreads();
      step_hi -= c;
      ++ord;
    }
    for (int i = threadIdx.x; i < LTc * N; i += blockDim.x)
      a.lambda[(size_t)(lb0 + t0) * N + i] = lam[i];
    __syncthreads();
  }
}

// Launch shape: producer warps per slot cover one step of a lane tile.
template <class MS>
inline Shape make_shape(int L) {
  constexpr int N = MS::N;
  Shape sh;
  const int gpw = Geo<N>::GPW;
  int Ws = (L + gpw - 1) / gpw;
  if (Ws > kMaxWs) Ws = kMaxWs;
  if (Ws < 1) Ws = 1;
  sh.Ws = Ws;
  sh.S = kMaxProducers / Ws;  // producer sets: as many as the producer warps allow
  if (sh.S > kMaxSlots) sh.S = kMaxSlots;
  sh.RS = Ws * gpw;
  sh.threads = 32 * kMaxWarps;
  // Two record slots per set when they fit: a set factors slot j + S while the
  // consumer still reads slot j, so the producers never wait on the solve.
  int o_cs, o_rec, o_pb, o_vs, o_lam, tot;
  // Few lanes per CTA (the strong-scaled shapes): the substitution chain, one 20x20 solve per row on a
  // single thread, is the critical path while the producers idle, so the records carry M^{-1} and the
  // consumer multiplies (lu_inverse_group); otherwise the plain LU records.
  for (sh.inv = L <= kInvMaxLanes ? 1 : 0; sh.inv >= 0; --sh.inv) {
    sh.stride = sh.inv ? Rec<N>::STRIDE_INV : Rec<N>::STRIDE;
    for (sh.Q = 2 * sh.S;; sh.Q = sh.S) {
      // a tile row must never need a slot more than Q - 1 slots past the oldest unreleased one
      sh.LT = min(min(32, L), (sh.Q - 1) * sh.RS);  // no wider than the CTA's lanes (shared memory)
      smem_layout<MS>(sh.S, sh.Q, sh.Ws, sh.RS, sh.LT, sh.stride, o_cs, o_rec, o_pb, o_vs, o_lam, tot);
      if (sh.Q == sh.S || (sh.Q <= kMaxSlots && tot * 8 <= kSmemCap)) break;
    }
    if (tot * 8 <= kSmemCap || sh.inv == 0) break;
  }
  sh.ring = sh.Q * sh.RS * sh.stride;
  sh.smem_bytes = tot * 8;
  return sh;
}

template <class MS>
cudaError_t fwd2_launch(const FwdLaunch* a, cudaStream_t st) {
  if (!a) {  // probe: also loads the kernels (lazy module loading)
    cudaError_t e = preload((const void*)fwd2_kernel<MS, false>);
    if (e == cudaSuccess) e = preload((const void*)fwd2_kernel<MS, true>);
    if constexpr (HasArrowTri<MS>::value)
      if (e == cudaSuccess) e = preload((const void*)fwd2_kernel<MS, false, true>);
    return e;
  }
  const int Lmax = (a->nb + a->grid - 1) / a->grid;
  if constexpr (HasArrowTri<MS>::value) {
    if (a->structured) {
      Shape sh = make_shape_sp<MS>(Lmax, true);
      const void* k = (const void*)fwd2_kernel<MS, false, true>;
      CKO_ALLOW_FULL_SMEM(k);
      FwdLaunch copy = *a;
      void* args[] = {&copy, &sh};
      return launch_persistent(k, dim3(a->grid), dim3(sh.threads), args, sh.smem_bytes, st);
    }
  }
  Shape sh = make_shape<MS>(Lmax);
  const void* k = sh.inv ? (const void*)fwd2_kernel<MS, true> : (const void*)fwd2_kernel<MS, false>;
  CKO_ALLOW_FULL_SMEM(k);
  FwdLaunch copy = *a;
  void* args[] = {&copy, &sh};
  return launch_persistent(k, dim3(a->grid), dim3(sh.threads), args, sh.smem_bytes, st);
}

template <class MS>
cudaError_t adj2_launch(const AdjLaunch* a, cudaStream_t st) {
  if (!a) {
    cudaError_t e = preload((const void*)adj2_kernel<MS, false>);
    if (e == cudaSuccess) e = preload((const void*)adj2_kernel<MS, true>);
    if constexpr (HasArrowTri<MS>::value)
      if (e == cudaSuccess) e = preload((const void*)adj2_kernel<MS, false, true>);
    return e;
  }
  const int Lmax = (a->nb + a->grid - 1) / a->grid;
  if constexpr (HasArrowTri<MS>::value) {
    if (a->structured) {
      const Shape sh = make_shape_sp<MS>(Lmax, false);
      CKO_ALLOW_FULL_SMEM((adj2_kernel<MS, false, true>));
      adj2_kernel<MS, false, true><<<a->grid, sh.threads, sh.smem_bytes, st>>>(*a, sh);
      return cudaGetLastError();
    }
  }
  Shape sh = make_shape<MS>(Lmax);
  if (sh.inv) {
    CKO_ALLOW_FULL_SMEM((adj2_kernel<MS, true>));
    adj2_kernel<MS, true><<<a->grid, sh.threads, sh.smem_bytes, st>>>(*a, sh);
  } else {
    CKO_ALLOW_FULL_SMEM((adj2_kernel<MS, false>));
    adj2_kernel<MS, false><<<a->grid, sh.threads, sh.smem_bytes, st>>>(*a, sh);
  }
  return cudaGetLastError();
}

}  // namespace v2

// Per-model v2 launchers (cko_inst_*.cu), dispatching on the state size n;
// a == nullptr probes support. cudaErrorNotSupported when n has no
// instantiation (the v1 kernels then run).
#define CKO_V2_DECLARE(NAME)                                                    \
  cudaError_t fwd2_run_##NAME(int n, const FwdLaunch* a, cudaStream_t st);      \
  cudaError_t adj2_run_##NAME(int n, const AdjLaunch* a, cudaStream_t st);      \
  cudaError_t fwdp_run_##NAME(int n, const FwdLaunch* a, cudaStream_t st);      \
  cudaError_t adjp_run_##NAME(int n, const AdjLaunch* a, cudaStream_t st);

}  // namespace cko
