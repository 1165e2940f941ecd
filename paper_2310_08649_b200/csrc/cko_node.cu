// cko_node.cu — the wide neural ODE (state 8, hidden width
// 128) on fp64 tensor cores.
//
// Every rate and Jacobian evaluation of the MLP right-hand side
//   h = tanh(W3 tanh(W2 tanh(W1 [y; s] + b1) + b2) + b3),
//   J = diag(1 - o^2) W3 diag(1 - z2^2) W2 diag(1 - z1^2) W1[:, :8]
// (models_node.cpp:37-107) is dominated by W2 (128 x 128) times per-point
// operands. node_eval_kernel batches 8 points per tile and runs those products
// as DMMA m8n8k4 (mma.sync f64, SASS DMMA.8x8x4) against one operand matrix
// [M1 of 8 points (64 columns) | z1 of 8 points (8 columns)]: 72 columns,
// 9 tile columns, 32 k-steps.
//
// The Newton loop around it runs from the host (one launch per phase, the
// all-lanes predicate read back through pinned memory): node_residual_kernel
// (integrate.cpp:64-95), node_factor_kernel (thread per point: M = I - J dt,
// LU with the reference's pivot rule) and node_thomas_kernel (thread per lane:
// substitution, iterate update). The adjoint uses the same pieces on
// (I - J dt)^T (adjoint.cpp:49-127). Arithmetic outside the DMMA products
// follows the reference; the products accumulate in tensor-core order.
#include <cmath>
#include <cstring>
#include <utility>
#include <vector>

#include "cko_kernels.cuh"
#include "cko_lu_thread.cuh"

namespace cko {
namespace node {

constexpr int N = 8, W = 128, W0 = N + 1;
constexpr int TP = 8;                 // points per tile
constexpr int BC = TP * N + TP;       // operand columns: M1 (64) | z1 (8)
constexpr int kEvalThreads = 256;

struct Views {
  const double *W1, *b1, *W2, *b2, *W3, *b3;
  __device__ explicit Views(const double* p) {
    W1 = p;
    b1 = W1 + W * W0;
    W2 = b1 + W;
    b2 = W2 + W * W;
    W3 = b2 + W;
    b3 = W3 + N * W;
  }
};

__device__ __forceinline__ void dmma(double& c0, double& c1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0, %1}, {%2}, {%3}, {%0, %1};"
               : "+d"(c0), "+d"(c1)
               : "d"(a), "d"(b));
}

// Points are (k, b) pairs of a chunk, p = k * nb + b, state rows at
// states[(row0 + k) * nb * N + b * N], times t[(row0 + k) * nb + b]. H (P, N)
// receives h, J (P, N, N) the Jacobian (when want_j).
// the products overwrite the operand once every warp has read it: ~75 KB, two CTAs per SM (registers)
constexpr int kEvalSmem = (W * BC + TP * W0 + TP * N) * 8;  // operand / products, z0, 1 - o^2

// Point p = k * nb + b sits on trajectory row row0 + dir * k (dir = -1: the
// descending rows of a reversed adjoint chunk).
__global__ void __launch_bounds__(kEvalThreads) node_eval_kernel(DevModel m, const double* states,
                                                                 const double* times, int row0, int dir, int nb,
                                                                 int P, double* H, double* J, int want_j,
                                                                 const int* dyn) {
  if (dyn) {  // device-driven Newton loop: the chunk comes from the control block
    if (dyn[2]) return;
    row0 = dyn[0] + 1;
    P = dyn[1] * nb;
  }
  extern __shared__ __align__(16) double smem[];
  double* sB = smem;               // operand  (W x 72) = 72 KB
  double* sX = sB;                 // products overwrite it after the tensor-core pass
  double (*sz0)[W0] = reinterpret_cast<double (*)[W0]>(sB + W * BC);
  double (*sg3)[N] = reinterpret_cast<double (*)[N]>(sB + W * BC + TP * W0);
  const Views v(m.p);
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int ntiles = (P + TP - 1) / TP;
  const size_t row = (size_t)nb * N;
  for (int tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
    const int p0 = tile * TP;
    // z0 = [y; sin(2 pi t / T_b)]
    for (int e = tid; e < TP * W0; e += blockDim.x) {
      const int q = e / W0, i = e % W0, p = min(p0 + q, P - 1);
      const int k = p / nb, b = p % nb, rw = row0 + dir * k;
      if (i < N)
        sz0[q][i] = states[(size_t)rw * row + (size_t)b * N + i];
      else
        sz0[q][i] = sin(CKO_TWO_PI * times[(size_t)rw * nb + b] / m.periods[m.off + b]);
    }
    __syncthreads();
    // z1 = tanh(W1 z0 + b1); operand columns: M1 = (1 - z1^2) W1[:, :8] per point, then z1
    for (int e = tid; e < TP * W; e += blockDim.x) {
      const int q = e / W, i = e % W;
      double acc = v.b1[i];
      for (int j = 0; j < W0; ++j) acc += v.W1[i * W0 + j] * sz0[q][j];
      const double z1 = tanh(acc), g1 = 1.0 - z1 * z1;
      double* brow = sB + i * BC;
      for (int j = 0; j < N; ++j) brow[q * N + j] = g1 * v.W1[i * W0 + j];
      brow[TP * N + q] = z1;
    }
    __syncthreads();
    // X = W2 [M1 | z1] on the tensor cores: warp w owns rows 16w..16w+15 (two 8-row tiles)
    {
      double acc[2][BC / 8][2];
#pragma unroll
      for (int i = 0; i < 2; ++i)
#pragma unroll
        for (int j = 0; j < BC / 8; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;
      const int r0 = warp * 16;
      for (int k = 0; k < W; k += 4) {
        const double a0 = __ldg(v.W2 + (r0 + lane / 4) * W + k + lane % 4);
        const double a1 = __ldg(v.W2 + (r0 + 8 + lane / 4) * W + k + lane % 4);
#pragma unroll
        for (int j = 0; j < BC / 8; ++j) {
          const double bv = sB[(k + lane % 4) * BC + 8 * j + lane / 4];
          dmma(acc[0][j][0], acc[0][j][1], a0, bv);
          dmma(acc[1][j][0], acc[1][j][1], a1, bv);
        }
      }
      __syncthreads();  // every warp is done with the operand
#pragma unroll
      for (int i = 0; i < 2; ++i)
#pragma unroll
        for (int j = 0; j < BC / 8; ++j) {
          double* out = sX + (r0 + 8 * i + lane / 4) * BC + 8 * j + 2 * (lane % 4);
          out[0] = acc[i][j][0];
          out[1] = acc[i][j][1];
        }
    }
    __syncthreads();
    // z2 = tanh(a2 + b2); M2 = (1 - z2^2) X in place; z2 kept in the z1 columns
    for (int e = tid; e < TP * W; e += blockDim.x) {
      const int q = e / W, i = e % W;
      double* xrow = sX + i * BC;
      const double z2 = tanh(xrow[TP * N + q] + v.b2[i]), g2 = 1.0 - z2 * z2;
      xrow[TP * N + q] = z2;
      for (int j = 0; j < N; ++j) xrow[q * N + j] *= g2;
    }
    __syncthreads();
    // o = tanh(W3 z2 + b3), h = o
    for (int e = tid; e < TP * N; e += blockDim.x) {
      const int q = e / N, i = e % N, p = p0 + q;
      double acc = v.b3[i];
      for (int l = 0; l < W; ++l) acc += v.W3[i * W + l] * sX[l * BC + TP * N + q];
      const double o = tanh(acc);
      sg3[q][i] = 1.0 - o * o;
      if (p < P) H[(size_t)p * N + i] = o;
    }
    if (want_j) {
      __syncthreads();
      // J = diag(g3) W3 M2
      for (int e = tid; e < TP * N * N; e += blockDim.x) {
        const int q = e / (N * N), i = (e / N) % N, j = e % N, p = p0 + q;
        double acc = 0.0;
        for (int l = 0; l < W; ++l) acc += v.W3[i * W + l] * sX[l * BC + q * N + j];
        if (p < P) J[(size_t)p * N * N + i * N + j] = sg3[q][i] * acc;
      }
    }
    __syncthreads();
  }
}

// Residual of the chunk's points + lane norms + predicate flags (integrate.cpp:64-95, 176-188).
__global__ void node_residual_kernel(const double* states, const double* times, const double* H, int step, int c,
                                     int nb, double* R, double* r0, double* rn, int first, double tol_a,
                                     double tol_r, unsigned* flags, const int* dyn) {
  if (dyn) {
    if (dyn[2]) return;
    step = dyn[0], c = dyn[1];
  }
  const size_t row = (size_t)nb * N;
  for (int b = blockIdx.x * blockDim.x + threadIdx.x; b < nb; b += gridDim.x * blockDim.x) {
    double acc = 0.0;
    for (int k = 0; k < c; ++k) {
      const int p = k * nb + b;
      const double t = times[(size_t)(step + 1 + k) * nb + b];
      const double dt = t - times[(size_t)(step + k) * nb + b];
      const double* y = states + (size_t)(step + 1 + k) * row + (size_t)b * N;
      const double* ym = states + (size_t)(step + k) * row + (size_t)b * N;
      double s = 0.0;
      for (int i = 0; i < N; ++i) {
        const double vv = xsub(xsub(y[i], ym[i]), xmul(H[(size_t)p * N + i], dt));
        R[(size_t)p * N + i] = vv;
        s = xadd(s, xmul(vv, vv));
      }
      acc = xadd(acc, s);
    }
    const double nrm = sqrt(acc);
    double base = nrm;
    if (first)
      r0[b] = nrm;
    else
      base = r0[b];
    rn[b] = nrm;
    unsigned f = 0;
    if (!isfinite(nrm)) f |= FLAG_NON_FINITE;
    if (!(nrm <= tol_a || nrm <= xmul(tol_r, base))) f |= FLAG_NOT_CONVERGED;
    if (f) atomicOr(flags, f);
  }
}

// Point-parallel form for chunks of at most 128 rows: a block holds 128 / c
// lanes x c rows, one thread per point, then one thread per lane sums the
// rows' squared norms in order (same arithmetic as node_residual_kernel).
__global__ void __launch_bounds__(128) node_residual_pp_kernel(const double* states, const double* times,
                                                               const double* H, int step, int c, int nb, double* R,
                                                               double* r0, double* rn, int first, double tol_a,
                                                               double tol_r, unsigned* flags, const int* dyn) {
  if (dyn) {
    if (dyn[2]) return;
    step = dyn[0], c = dyn[1];
  }
  __shared__ double ps[128];
  const size_t row = (size_t)nb * N;
  const int Lb = 128 / c, b0 = blockIdx.x * Lb;
  const int k = threadIdx.x / Lb, lb = threadIdx.x % Lb, b = b0 + lb;
  if (k < c && b < nb) {
    const int p = k * nb + b;
    const double t = times[(size_t)(step + 1 + k) * nb + b];
    const double dt = t - times[(size_t)(step + k) * nb + b];
    const double* y = states + (size_t)(step + 1 + k) * row + (size_t)b * N;
    const double* ym = states + (size_t)(step + k) * row + (size_t)b * N;
    double yv[N], ymv[N], hv[N];
    for (int i = 0; i < N; ++i) yv[i] = y[i], ymv[i] = ym[i], hv[i] = H[(size_t)p * N + i];
    double sq = 0.0;
    for (int i = 0; i < N; ++i) {
      const double vv = xsub(xsub(yv[i], ymv[i]), xmul(hv[i], dt));
      R[(size_t)p * N + i] = vv;
      sq = xadd(sq, xmul(vv, vv));
    }
    ps[k * Lb + lb] = sq;
  }
  __syncthreads();
  if (threadIdx.x < Lb && b0 + (int)threadIdx.x < nb) {
    const int bl = b0 + threadIdx.x;
    double acc = 0.0;
    for (int kk = 0; kk < c; ++kk) acc = xadd(acc, ps[kk * Lb + threadIdx.x]);
    const double nrm = sqrt(acc);
    double base = nrm;
    if (first)
      r0[bl] = nrm;
    else
      base = r0[bl];
    rn[bl] = nrm;
    unsigned f = 0;
    if (!isfinite(nrm)) f |= FLAG_NON_FINITE;
    if (!(nrm <= tol_a || nrm <= xmul(tol_r, base))) f |= FLAG_NOT_CONVERGED;
    if (f) atomicOr(flags, f);
  }
}

constexpr int kRec = N * N + N + 6;  // LU | 1/U_ii | perm (N + 1 ints) — 16-byte aligned stride

// Thread per point: assemble M (forward: I - J dt; adjoint: (I - J dt)^T and the rhs
// dL + dt J^T lambda) and factor it (lu_factor_block rule).
__global__ void node_factor_kernel(const double* J, const double* times, int step_or_hi, int c, int nb,
                                   int adjoint, double* recs, unsigned long long* sing_key, unsigned long long ord,
                                   int nc, unsigned* flags, const int* dyn) {
  if (dyn) {
    if (dyn[2]) return;
    step_or_hi = dyn[0], c = dyn[1];
  }
  for (int p = blockIdx.x * blockDim.x + threadIdx.x; p < c * nb; p += gridDim.x * blockDim.x) {
    const int k = p / nb, b = p % nb;
    const int m = adjoint ? step_or_hi - k : step_or_hi + 1 + k;
    const double dt = times[(size_t)m * nb + b] - times[(size_t)(m - 1) * nb + b];
    const double* Jp = J + (size_t)p * N * N;
    double* rec = recs + (size_t)p * kRec;
    // factor in a thread-local copy (L1-resident local memory), then store the record once
    __align__(16) double loc[N * N + N];
    double mx = 0.0;
    auto build = [&]() {
      double jv[N * N];
#pragma unroll
      for (int e = 0; e < N * N; ++e) jv[e] = Jp[e];  // every load in flight at once
#pragma unroll
      for (int i = 0; i < N; ++i)
#pragma unroll
        for (int j = 0; j < N; ++j) {
          double vv;
          if (adjoint)
            vv = (i == j) ? 1.0 - dt * jv[j * N + i] : -dt * jv[j * N + i];
          else
            vv = (i == j) ? xadd(xmul(-dt, jv[i * N + j]), 1.0) : xmul(-dt, jv[i * N + j]);
          loc[i * N + j] = vv;
          mx = fmax(mx, fabs(vv));
        }
    };
    build();
    bool viol;
    bool ok = lt::lu_thread_nopiv<N>(loc, loc + N * N, 1e-14 * mx, viol);
    int* perm = reinterpret_cast<int*>(rec + N * N + N);
    if (viol) {
      build();
      ok = lt::lu_thread_pivot<N>(loc, loc + N * N, perm, 1e-14 * mx);
      perm[N] = 0;
    } else {
      for (int i = 0; i < N; ++i) perm[i] = i;
      perm[N] = 1;
    }
#pragma unroll
    for (int e = 0; e < N * N + N; e += 2)
      *reinterpret_cast<double2*>(rec + e) = make_double2(loc[e], loc[e + 1]);
    if (!ok) {
      atomicMin(sing_key, adjoint ? ord * (unsigned long long)nc * nb + (unsigned long long)k * nb + b
                                  : (unsigned long long)k * nb + b);
      if (flags) atomicOr(flags, FLAG_SINGULAR);  // reaches the peers through the group flag exchange
    }
  }
}

__device__ inline void rec_solve(const double* rec, double (&v)[N]) {
  const int* perm = reinterpret_cast<const int*>(rec + N * N + N);
  double y[N];
  if (perm[N]) {
    for (int i = 0; i < N; ++i) y[i] = v[i];
  } else {
    for (int i = 0; i < N; ++i) y[i] = v[perm[i]];
  }
  for (int i = 1; i < N; ++i) {
    double s = y[i];
    for (int j = 0; j < i; ++j) s -= rec[i * N + j] * y[j];
    y[i] = s;
  }
  for (int i = N - 1; i >= 0; --i) {
    double s = y[i];
    for (int j = i + 1; j < N; ++j) s -= rec[i * N + j] * y[j];
    y[i] = s * rec[N * N + i];
  }
  for (int i = 0; i < N; ++i) v[i] = y[i];
}

// The substitution kernels run one thread per lane (a few warps on the whole
// GPU): each thread streams its rows' records and right-hand sides into its
// own shared-memory ring with cp.async, kSubD rows ahead of the solve, so the
// L2 latency leaves the dependency chain.
constexpr int kSubD = 4;                 // rows in flight per thread
constexpr int kSubS = kRec + N;          // staged doubles per row: record | rhs (16-byte multiple)
constexpr int kSubThreads = 64;
constexpr int kSubSmem = kSubThreads * kSubD * kSubS * 8;
static_assert(kRec % 2 == 0 && kSubS % 2 == 0, "16-byte staging");

__device__ __forceinline__ void sub_stage(double* dst, const double* rec, const double* rhs) {
  for (int e = 0; e < kRec; e += 2) {
    const unsigned s = (unsigned)__cvta_generic_to_shared(dst + e);
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(s), "l"(rec + e) : "memory");
  }
  for (int e = 0; e < N; e += 2) {
    const unsigned s = (unsigned)__cvta_generic_to_shared(dst + kRec + e);
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(s), "l"(rhs + e) : "memory");
  }
}
// rec_solve on a staged record: the permuted gather goes through the staged
// rhs slot (already consumed) instead of a dynamically indexed register array.
__device__ inline void rec_solve_staged(double* st, double (&v)[N]) {
  const int* perm = reinterpret_cast<const int*>(st + N * N + N);
  double y[N];
  if (perm[N]) {
#pragma unroll
    for (int i = 0; i < N; ++i) y[i] = v[i];
  } else {
    double* sc = st + kRec;
#pragma unroll
    for (int i = 0; i < N; ++i) sc[i] = v[i];
#pragma unroll
    for (int i = 0; i < N; ++i) y[i] = sc[perm[i]];
  }
#pragma unroll
  for (int i = 1; i < N; ++i) {
    double s = y[i];
#pragma unroll
    for (int j = 0; j < i; ++j) s -= st[i * N + j] * y[j];
    y[i] = s;
  }
#pragma unroll
  for (int i = N - 1; i >= 0; --i) {
    double s = y[i];
#pragma unroll
    for (int j = i + 1; j < N; ++j) s -= st[i * N + j] * y[j];
    y[i] = s * st[N * N + i];
  }
#pragma unroll
  for (int i = 0; i < N; ++i) v[i] = y[i];
}
__device__ __forceinline__ void sub_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
__device__ __forceinline__ void sub_wait() { asm volatile("cp.async.wait_group %0;" ::"n"(kSubD - 1) : "memory"); }

// Thread per lane: forward substitution x_k = M_k^{-1}(r_k + x_{k-1}), yy_k -= x_k.
__global__ void __launch_bounds__(kSubThreads) node_thomas_fwd_kernel(double* states, const double* R,
                                                                      const double* recs, int step, int c, int nb,
                                                                      const int* dyn) {
  if (dyn) {
    if (dyn[2]) return;
    step = dyn[0], c = dyn[1];
  }
  extern __shared__ __align__(16) double sub_smem[];
  double* my = sub_smem + (size_t)threadIdx.x * kSubD * kSubS;
  const size_t row = (size_t)nb * N;
  for (int b = blockIdx.x * blockDim.x + threadIdx.x; b < nb; b += gridDim.x * blockDim.x) {
    for (int k = 0; k < kSubD - 1; ++k) {
      if (k < c) sub_stage(my + k * kSubS, recs + ((size_t)k * nb + b) * kRec, R + ((size_t)k * nb + b) * N);
      sub_commit();
    }
    double x[N];
    for (int i = 0; i < N; ++i) x[i] = 0.0;
    for (int k = 0; k < c; ++k) {
      const int kn = k + kSubD - 1;
      if (kn < c)
        sub_stage(my + (kn % kSubD) * kSubS, recs + ((size_t)kn * nb + b) * kRec, R + ((size_t)kn * nb + b) * N);
      sub_commit();
      sub_wait();
      double* st = my + (k % kSubD) * kSubS;
      double v[N];
      for (int i = 0; i < N; ++i) v[i] = st[kRec + i] + x[i];
      rec_solve_staged(st, v);
      double* yy = states + (size_t)(step + 1 + k) * row + (size_t)b * N;
      for (int i = 0; i < N; ++i) {
        x[i] = v[i];
        yy[i] -= v[i];
      }
    }
  }
}

// Adjoint rhs of a reversed chunk: rhs_r = dL_m + dt J_m^T lambda (adjoint.cpp:64-72).
__global__ void node_adj_rhs_kernel(const double* states, const double* times, const double* J, const double* dL,
                                    const double* loss, const double* lam, int step_hi, int c, int nb, double* R) {
  const size_t row = (size_t)nb * N;
  const double Lval = loss ? *loss : 0.0;
  for (int p = blockIdx.x * blockDim.x + threadIdx.x; p < c * nb; p += gridDim.x * blockDim.x) {
    const int r = p / nb, b = p % nb, m = step_hi - r;
    const double dt = times[(size_t)m * nb + b] - times[(size_t)(m - 1) * nb + b];
    const double* Jp = J + (size_t)p * N * N;
    const double* lb = lam + (size_t)b * N;
    const double* y = states + (size_t)m * row + (size_t)b * N;
    double tmp[N];
    for (int i = 0; i < N; ++i) tmp[i] = 0.0;
    for (int j = 0; j < N; ++j)
      for (int i = 0; i < N; ++i) tmp[i] += Jp[j * N + i] * lb[j];
    for (int i = 0; i < N; ++i) {
      const double dl = dL ? dL[(size_t)m * row + (size_t)b * N + i] : (Lval > 0.0 ? y[i] / Lval : 0.0);
      R[(size_t)p * N + i] = dl + dt * tmp[i];
    }
  }
}

// Thread per lane: delta_r = M_r^{-1}(rhs_r + delta_{r-1}), w_m = (lambda + delta_r) dt, lambda += delta_{c-1}.
__global__ void __launch_bounds__(kSubThreads) node_thomas_adj_kernel(const double* R, const double* recs,
                                                                      const double* times, int step_hi, int c,
                                                                      int nb, double* lam, double* wq) {
  extern __shared__ __align__(16) double sub_smem[];
  double* my = sub_smem + (size_t)threadIdx.x * kSubD * kSubS;
  const size_t row = (size_t)nb * N;
  for (int b = blockIdx.x * blockDim.x + threadIdx.x; b < nb; b += gridDim.x * blockDim.x) {
    for (int r = 0; r < kSubD - 1; ++r) {
      if (r < c) sub_stage(my + r * kSubS, recs + ((size_t)r * nb + b) * kRec, R + ((size_t)r * nb + b) * N);
      sub_commit();
    }
    double d[N], lc[N];
    for (int i = 0; i < N; ++i) d[i] = 0.0, lc[i] = lam[(size_t)b * N + i];
    for (int r = 0; r < c; ++r) {
      const int m = step_hi - r;
      const int rn = r + kSubD - 1;
      if (rn < c)
        sub_stage(my + (rn % kSubD) * kSubS, recs + ((size_t)rn * nb + b) * kRec, R + ((size_t)rn * nb + b) * N);
      sub_commit();
      sub_wait();
      double* st = my + (r % kSubD) * kSubS;
      const double dt = times[(size_t)m * nb + b] - times[(size_t)(m - 1) * nb + b];
      for (int i = 0; i < N; ++i) d[i] = st[kRec + i] + d[i];
      rec_solve_staged(st, d);
      double* w = wq + (size_t)m * row + (size_t)b * N;
      for (int i = 0; i < N; ++i) w[i] = (lc[i] + d[i]) * dt;
    }
    for (int i = 0; i < N; ++i) lam[(size_t)b * N + i] = lc[i] + d[i];
  }
}

__global__ void node_init_chunk_kernel(double* states, const double* dy, int step, int c, int nb, const int* dyn) {
  if (dyn) {
    if (dyn[2]) return;
    step = dyn[0], c = dyn[1];
  }
  const size_t row = (size_t)nb * N;
  for (size_t e = blockIdx.x * (size_t)blockDim.x + threadIdx.x; e < (size_t)c * row;
       e += (size_t)gridDim.x * blockDim.x) {
    const int k = (int)(e / row);
    const size_t off = e % row;
    states[(size_t)(step + 1 + k) * row + off] =
        states[(size_t)step * row + off] + (dy ? dy[(size_t)k * row + off] : 0.0);
  }
}

// One-thread exchange of the predicate flags with the group (same generation
// counter as the grid barriers).
__global__ void node_group_flags_kernel(GroupView g, GridSync* gs, unsigned* flags, uint64_t budget_ns,
                                        const int* dyn) {
  if (dyn && dyn[2]) return;
  if (threadIdx.x == 0 && g.world > 1) {
    gs->ext_gen += 1;
    *flags = group_exchange(g, gs->ext_gen, *flags, globaltimer_ns() + budget_ns);
  }
}

inline int blocks_for(size_t work, int threads) {
  size_t b = (work + threads - 1) / threads;
  if (b < 1) b = 1;
  if (b > 148 * 8) b = 148 * 8;
  return (int)b;
}

}  // namespace node

namespace node {

// Per-point vectors of the parameter VJP (cko_node_vjp.cu, models_node.cpp:109-151)
// for the C4 shape, 32 points per tile: z0, z1 = tanh(W1 z0 + b1),
// z2 = tanh(W2 z1 + b2), o = tanh(W3 z2 + b3), d3 = w (1 - o^2),
// d2 = (W3^T d3)(1 - z2^2), d1 = (W2^T d2)(1 - z1^2). The two 128 x 128 products
// (W2 z1, W2^T d2) run as DMMA m8n8k4 (warp w: rows 16w .. 16w+15, 4 tile
// columns, 32 k-steps); outputs feature-major x[f * P + p] like node_vectors_kernel.
constexpr int TV = 32;                     // points per tile
constexpr int kVecThreads = 256;
constexpr int kVecSmem = (3 * W * TV + TV * W0 + N * TV) * 8;  // z1, X, d2 | z0 | d3

__global__ void __launch_bounds__(kVecThreads) node_vectors_dmma_kernel(DevModel m, const double* states,
                                                                        const double* times, const double* wq,
                                                                        int nb, size_t P, double* vec) {
  extern __shared__ __align__(16) double smem[];
  double* sZ1 = smem;            // (W x TV)
  double* sX = sZ1 + W * TV;     // (W x TV): W2 z1 + b2 -> z2
  double* sD2 = sX + W * TV;     // (W x TV)
  double* sZ0 = sD2 + W * TV;    // (TV x W0)
  double* sD3 = sZ0 + TV * W0;   // (N x TV)
  const Views v(m.p);
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const size_t row = (size_t)nb * N;
  double* Z0 = vec;
  double* Z1 = Z0 + (size_t)W0 * P;
  double* Z2 = Z1 + (size_t)W * P;
  double* D1 = Z2 + (size_t)W * P;
  double* D2 = D1 + (size_t)W * P;
  double* D3 = D2 + (size_t)W * P;
  const size_t ntiles = (P + TV - 1) / TV;
  for (size_t tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
    const size_t p0 = tile * TV;
    // z0 = [y; sin(2 pi t / T_b)] of trajectory row mm = 1 + p / nb
    for (int e = tid; e < TV * W0; e += blockDim.x) {
      const int q = e / W0, i = e % W0;
      const size_t p = min(p0 + q, P - 1);
      const int mm = 1 + (int)(p / nb), b = (int)(p % nb);
      const double z = i < N ? states[(size_t)mm * row + (size_t)b * N + i]
                             : sin(CKO_TWO_PI * times[(size_t)mm * nb + b] / m.periods[m.off + b]);
      sZ0[q * W0 + i] = z;
      if (p0 + q < P) Z0[(size_t)i * P + p0 + q] = z;
    }
    __syncthreads();
    for (int e = tid; e < W * TV; e += blockDim.x) {  // z1 (thread: feature i, point q; q fastest)
      const int i = e / TV, q = e % TV;
      double acc = v.b1[i];
      for (int j = 0; j < W0; ++j) acc += v.W1[i * W0 + j] * sZ0[q * W0 + j];
      const double z1 = tanh(acc);
      sZ1[i * TV + q] = z1;
      if (p0 + q < P) Z1[(size_t)i * P + p0 + q] = z1;
    }
    __syncthreads();
    const int r0 = warp * 16;
    {  // X = W2 z1 on the tensor cores
      double acc[2][TV / 8][2] = {};
      for (int k = 0; k < W; k += 4) {
        const double a0 = __ldg(v.W2 + (r0 + lane / 4) * W + k + lane % 4);
        const double a1 = __ldg(v.W2 + (r0 + 8 + lane / 4) * W + k + lane % 4);
#pragma unroll
        for (int j = 0; j < TV / 8; ++j) {
          const double bv = sZ1[(k + lane % 4) * TV + 8 * j + lane / 4];
          dmma(acc[0][j][0], acc[0][j][1], a0, bv);
          dmma(acc[1][j][0], acc[1][j][1], a1, bv);
        }
      }
#pragma unroll
      for (int i = 0; i < 2; ++i)
#pragma unroll
        for (int j = 0; j < TV / 8; ++j) {
          const int r = r0 + 8 * i + lane / 4, q = 8 * j + 2 * (lane % 4);
          sX[r * TV + q] = tanh(acc[i][j][0] + v.b2[r]);
          sX[r * TV + q + 1] = tanh(acc[i][j][1] + v.b2[r]);
        }
    }
    __syncthreads();
    for (int e = tid; e < W * TV; e += blockDim.x) {
      const int i = e / TV, q = e % TV;
      if (p0 + q < P) Z2[(size_t)i * P + p0 + q] = sX[i * TV + q];
    }
    for (int e = tid; e < N * TV; e += blockDim.x) {  // o, d3 = w (1 - o^2)
      const int i = e / TV, q = e % TV;
      const size_t p = min(p0 + q, P - 1);
      double acc = v.b3[i];
      for (int l = 0; l < W; ++l) acc += v.W3[i * W + l] * sX[l * TV + q];
      const double o = tanh(acc);
      const int mm = 1 + (int)(p / nb), b = (int)(p % nb);
      const double d3 = wq[(size_t)mm * row + (size_t)b * N + i] * (1.0 - o * o);
      sD3[i * TV + q] = d3;
      if (p0 + q < P) D3[(size_t)i * P + p0 + q] = d3;
    }
    __syncthreads();
    for (int e = tid; e < W * TV; e += blockDim.x) {  // d2 = (W3^T d3)(1 - z2^2)
      const int i = e / TV, q = e % TV;
      double acc = 0.0;
      for (int l = 0; l < N; ++l) acc += v.W3[l * W + i] * sD3[l * TV + q];
      const double z2 = sX[i * TV + q];
      const double d2 = acc * (1.0 - z2 * z2);
      sD2[i * TV + q] = d2;
      if (p0 + q < P) D2[(size_t)i * P + p0 + q] = d2;
    }
    __syncthreads();
    {  // d1 = (W2^T d2)(1 - z1^2) on the tensor cores: A(i, k) = W2[k][i]
      double acc[2][TV / 8][2] = {};
      for (int k = 0; k < W; k += 4) {
        const double a0 = __ldg(v.W2 + (k + lane % 4) * W + r0 + lane / 4);
        const double a1 = __ldg(v.W2 + (k + lane % 4) * W + r0 + 8 + lane / 4);
#pragma unroll
        for (int j = 0; j < TV / 8; ++j) {
          const double bv = sD2[(k + lane % 4) * TV + 8 * j + lane / 4];
          dmma(acc[0][j][0], acc[0][j][1], a0, bv);
          dmma(acc[1][j][0], acc[1][j][1], a1, bv);
        }
      }
#pragma unroll
      for (int i = 0; i < 2; ++i)
#pragma unroll
        for (int j = 0; j < TV / 8; ++j) {
          const int r = r0 + 8 * i + lane / 4, q = 8 * j + 2 * (lane % 4);
#pragma unroll
          for (int h = 0; h < 2; ++h) {
            const double z1 = sZ1[r * TV + q + h];
            if (p0 + q + h < P) D1[(size_t)r * P + p0 + q + h] = acc[i][j][h] * (1.0 - z1 * z1);
          }
        }
    }
    __syncthreads();
  }
}

}  // namespace node

cudaError_t launch_node_vectors_dmma(const DevModel& m, const double* states, const double* times, const double* wq,
                                     int nb, size_t P, double* vec, cudaStream_t st) {
  const cudaError_t attr = allow_smem((const void*)node::node_vectors_dmma_kernel, node::kVecSmem);
  if (attr != cudaSuccess) return attr;
  node::node_vectors_dmma_kernel<<<2 * 148, node::kVecThreads, node::kVecSmem, st>>>(m, states, times, wq, nb, P,
                                                                                      vec);
  return cudaGetLastError();
}


bool node_fast_path(const DevModel& m) { return m.kind == 5 && m.n == node::N && m.W == node::W; }

size_t node_scratch_doubles(int nb, int c) {
  const size_t P = (size_t)nb * c;
  return P * (node::N + node::N * node::N + node::N + node::kRec) + 8;
}

cudaError_t node_eval(const DevModel& m, const double* states, const double* times, int row0, int dir, int nb,
                      int P, double* H, double* J, bool want_j, cudaStream_t st) {
  const cudaError_t attr = allow_smem((const void*)node::node_eval_kernel, node::kEvalSmem);
  if (attr != cudaSuccess) return attr;
  const int tiles = (P + node::TP - 1) / node::TP;
  node::node_eval_kernel<<<tiles < 2 * 148 ? tiles : 2 * 148, node::kEvalThreads, node::kEvalSmem, st>>>(
      m, states, times, row0, dir, nb, P, H, J, want_j ? 1 : 0, nullptr);
  return cudaGetLastError();
}

static void launch_node_residual(const double* states, const double* times, const double* H, int step, int c, int nb,
                                 double* R, double* r0, double* rn, int first, double tol_a, double tol_r,
                                 unsigned* flags, cudaStream_t st) {
  using namespace node;
  if (c <= 128) {
    const int Lb = 128 / c;
    node_residual_pp_kernel<<<(nb + Lb - 1) / Lb, 128, 0, st>>>(states, times, H, step, c, nb, R, r0, rn, first,
                                                                tol_a, tol_r, flags, nullptr);
  } else {
    node_residual_kernel<<<blocks_for(nb, 128), 128, 0, st>>>(states, times, H, step, c, nb, R, r0, rn, first, tol_a,
                                                             tol_r, flags, nullptr);
  }
}

// Host-driven Newton integration for the wide neural ODE (Thomas solver).
// Returns 0 ok, 1 singular (key), 2 divergence (info), 4 group timeout.
cudaError_t node_forward(const DevModel& m, double* states, const double* times, const double* dy, int nb, int nt,
                         int nc, double tol_a, double tol_r, int max_iter, double* scratch, double* r0, double* rn,
                         unsigned* d_flags, unsigned* h_flags, unsigned long long* sing_key, const GroupView& grp,
                         GridSync* gs, int* iters, int* info, cudaStream_t st) {
  using namespace node;
  const int cmax = nc < nt ? nc : nt;
  const size_t Pmax = (size_t)cmax * nb;
  double* H = scratch;
  double* Jb = H + Pmax * N;
  double* R = Jb + Pmax * N * N;
  double* recs = R + Pmax * N;
  cudaError_t e;
  int step = 0, chunk = 0;
  info[0] = 0;
  auto flags = [&](unsigned& f) -> cudaError_t {
    if (grp.world > 1) node_group_flags_kernel<<<1, 32, 0, st>>>(grp, gs, d_flags, 60ull * 1000 * 1000 * 1000, nullptr);
    cudaError_t ee = cudaMemcpyAsync(h_flags, d_flags, sizeof(unsigned), cudaMemcpyDeviceToHost, st);
    if (ee == cudaSuccess) ee = cudaStreamSynchronize(st);
    f = *h_flags;
    return ee;
  };
  while (step < nt) {
    const int c = min(nc, nt - step);
    const int P = c * nb;
    node_init_chunk_kernel<<<blocks_for((size_t)P * N, 256), 256, 0, st>>>(states, dy, step, c, nb, nullptr);
    if ((e = node_eval(m, states, times, step + 1, 1, nb, P, H, Jb, false, st)) != cudaSuccess) return e;
    if ((e = cudaMemsetAsync(d_flags, 0, sizeof(unsigned), st)) != cudaSuccess) return e;
    launch_node_residual(states, times, H, step, c, nb, R, r0, rn, 1, tol_a, tol_r, d_flags, st);
    unsigned f = 0;
    if ((e = flags(f)) != cudaSuccess) return e;
    int it = 0;
    if (f & FLAG_TIMEOUT) return info[0] = 4, cudaSuccess;
    if (f & FLAG_NON_FINITE) return info[0] = 2, info[1] = step + 1, info[2] = 0, cudaSuccess;
    while (f & FLAG_NOT_CONVERGED) {
      if (it == max_iter) return info[0] = 2, info[1] = step + 1, info[2] = max_iter, cudaSuccess;
      ++it;
      if ((e = node_eval(m, states, times, step + 1, 1, nb, P, H, Jb, true, st)) != cudaSuccess) return e;
      if ((e = cudaMemsetAsync(d_flags, 0, sizeof(unsigned), st)) != cudaSuccess) return e;
      node_factor_kernel<<<blocks_for(P, 128), 128, 0, st>>>(Jb, times, step, c, nb, 0, recs, sing_key, 0, nc,
                                                               d_flags, nullptr);
      const cudaError_t fattr = allow_smem((const void*)node_thomas_fwd_kernel, kSubSmem);
      if (fattr != cudaSuccess) return fattr;
      node_thomas_fwd_kernel<<<blocks_for(nb, kSubThreads), kSubThreads, kSubSmem, st>>>(states, R, recs, step, c, nb,
                                                                                          nullptr);
      if ((e = node_eval(m, states, times, step + 1, 1, nb, P, H, Jb, false, st)) != cudaSuccess) return e;
      launch_node_residual(states, times, H, step, c, nb, R, r0, rn, 0, tol_a, tol_r, d_flags, st);
      if ((e = flags(f)) != cudaSuccess) return e;
      unsigned long long key = ~0ull;
      if ((e = cudaMemcpyAsync(h_flags + 2, sing_key, sizeof key, cudaMemcpyDeviceToHost, st)) != cudaSuccess)
        return e;
      if ((e = cudaStreamSynchronize(st)) != cudaSuccess) return e;
      std::memcpy(&key, h_flags + 2, sizeof key);
      if (f & FLAG_TIMEOUT) return info[0] = 4, cudaSuccess;
      // FLAG_SINGULAR with no local key: the singular block sits on a peer rank
      if (key != ~0ull || (f & FLAG_SINGULAR)) return info[0] = 1, info[1] = step + 1, info[2] = it, cudaSuccess;
      if (f & FLAG_NON_FINITE) return info[0] = 2, info[1] = step + 1, info[2] = it, cudaSuccess;
    }
    iters[chunk] = it;
    step += c;
    ++chunk;
  }
  info[3] = chunk;
  return cudaSuccess;
}

// ---------------------------------------------------------------------------
// Device-driven Newton loop (one CUDA graph per integration): an outer WHILE
// node walks the chunks, an inner WHILE node runs the Newton iterations; the
// predicate (integrate.cpp:176-188) and the divergence / singular-block
// outcomes are decided by one-thread control kernels that set the
// conditionals on the device, so no iteration waits on a host round trip.
// The kernels read the chunk (step, c) from the control block and return at
// once after a failure was recorded (dyn[2] != 0).
//   dyn: [0] step [1] c [2] status (0 ok, 1 singular, 2 divergence, 4 timeout)
//        [3] iteration [4] chunk [5] failing chunk's first step [6] its iteration
//        [7] nt [8] nc [9] max_iter;   iters[chunk] = Newton iterations.
// ---------------------------------------------------------------------------
namespace node {

__global__ void ctl_newton_start(int* dyn, const unsigned* flags, cudaGraphConditionalHandle outer,
                                 cudaGraphConditionalHandle inner) {
  const unsigned f = *flags;
  int st = 0;
  if (f & FLAG_TIMEOUT)
    st = 4;
  else if (f & FLAG_NON_FINITE)
    st = 2, dyn[5] = dyn[0] + 1, dyn[6] = 0;
  dyn[3] = 0;
  if (st) {
    dyn[2] = st;
    cudaGraphSetConditional(outer, 0);
  }
  cudaGraphSetConditional(inner, (!st && (f & FLAG_NOT_CONVERGED)) ? 1u : 0u);
}

__global__ void ctl_newton_iter(int* dyn, unsigned* flags, cudaGraphConditionalHandle outer,
                                cudaGraphConditionalHandle inner) {
  if (dyn[3] == dyn[9]) {  // the iteration cap: NewtonDivergence (integrate.cpp:247-254)
    dyn[2] = 2, dyn[5] = dyn[0] + 1, dyn[6] = dyn[9];
    cudaGraphSetConditional(inner, 0);
    cudaGraphSetConditional(outer, 0);
    return;
  }
  dyn[3] += 1;
  *flags = 0;
}

__global__ void ctl_newton_end(int* dyn, const unsigned* flags, const unsigned long long* key,
                               cudaGraphConditionalHandle outer, cudaGraphConditionalHandle inner) {
  if (dyn[2]) {
    cudaGraphSetConditional(inner, 0);
    cudaGraphSetConditional(outer, 0);
    return;
  }
  const unsigned f = *flags;
  int st = 0;
  if (f & FLAG_TIMEOUT)
    st = 4;
  else if (*key != ~0ull || (f & FLAG_SINGULAR))  // a singular block here or on a peer rank
    st = 1;
  else if (f & FLAG_NON_FINITE)
    st = 2;
  if (st) {
    dyn[2] = st, dyn[5] = dyn[0] + 1, dyn[6] = dyn[3];
    cudaGraphSetConditional(inner, 0);
    cudaGraphSetConditional(outer, 0);
    return;
  }
  cudaGraphSetConditional(inner, (f & FLAG_NOT_CONVERGED) ? 1u : 0u);
}

__global__ void ctl_chunk_end(int* dyn, int* iters, unsigned* flags, cudaGraphConditionalHandle outer) {
  if (dyn[2]) {
    cudaGraphSetConditional(outer, 0);
    return;
  }
  iters[dyn[4]] = dyn[3];
  dyn[0] += dyn[1];
  dyn[4] += 1;
  const int rem = dyn[7] - dyn[0];
  dyn[1] = rem < dyn[8] ? rem : dyn[8];
  *flags = 0;
  cudaGraphSetConditional(outer, dyn[0] < dyn[7] ? 1u : 0u);
}

// The last node of a captured chain (the one nothing depends on).
cudaError_t graph_leaf(cudaGraph_t g, cudaGraphNode_t* leaf) {
  size_t n = 0;
  cudaError_t e = cudaGraphGetNodes(g, nullptr, &n);
  if (e != cudaSuccess) return e;
  std::vector<cudaGraphNode_t> nodes(n);
  if ((e = cudaGraphGetNodes(g, nodes.data(), &n)) != cudaSuccess) return e;
  for (cudaGraphNode_t v : nodes) {
    size_t k = 0;
    if ((e = cudaGraphNodeGetDependentNodes(v, nullptr, &k)) != cudaSuccess) return e;
    if (k == 0) {
      *leaf = v;
      return cudaSuccess;
    }
  }
  return cudaErrorInvalidValue;
}

}  // namespace node

cudaError_t node_forward_graph(const DevModel& m, double* states, const double* times, const double* dy, int nb,
                               int nt, int nc, double tol_a, double tol_r, int max_iter, double* scratch, double* r0,
                               double* rn, unsigned* d_flags, unsigned long long* sing_key, const GroupView& grp,
                               GridSync* gs, int* d_ctl, cudaStream_t st) {
  using namespace node;
  const int cmax = nc < nt ? nc : nt;
  const size_t Pmax = (size_t)cmax * nb;
  double* H = scratch;
  double* Jb = H + Pmax * N;
  double* R = Jb + Pmax * N * N;
  double* recs = R + Pmax * N;
  int* dyn = d_ctl;
  int* iters = d_ctl + 16;
  cudaError_t e;
  const int host_ctl[10] = {0, cmax, 0, 0, 0, 0, 0, nt, nc, max_iter};
  if ((e = cudaMemcpyAsync(dyn, host_ctl, sizeof host_ctl, cudaMemcpyHostToDevice, st)) != cudaSuccess) return e;
  if ((e = cudaMemsetAsync(d_flags, 0, sizeof(unsigned), st)) != cudaSuccess) return e;
  for (const auto& [f, b] : {std::pair<const void*, int>{(const void*)node_eval_kernel, kEvalSmem},
                             {(const void*)node_thomas_fwd_kernel, kSubSmem}})
    if ((e = allow_smem(f, b)) != cudaSuccess) return e;
  const int eval_grid = (int)((Pmax + TP - 1) / TP) < 2 * 148 ? (int)((Pmax + TP - 1) / TP) : 2 * 148;
  const int Lb = cmax <= 128 ? 128 / cmax : 0;
  cudaStream_t cs;
  if ((e = cudaStreamCreateWithFlags(&cs, cudaStreamNonBlocking)) != cudaSuccess) return e;
  cudaGraph_t g = nullptr, outer_body = nullptr, inner_body = nullptr;
  cudaGraphExec_t ge = nullptr;
  auto eval = [&](int want_j) {
    node_eval_kernel<<<eval_grid, kEvalThreads, kEvalSmem, cs>>>(m, states, times, 0, 1, nb, (int)Pmax, H, Jb, want_j,
                                                               dyn);
  };
  auto residual = [&](int first) {
    if (Lb)
      node_residual_pp_kernel<<<(nb + Lb - 1) / Lb, 128, 0, cs>>>(states, times, H, 0, cmax, nb, R, r0, rn, first, tol_a,
                                                                 tol_r, d_flags, dyn);
    else
      node_residual_kernel<<<blocks_for(nb, 128), 128, 0, cs>>>(states, times, H, 0, cmax, nb, R, r0, rn, first, tol_a,
                                                               tol_r, d_flags, dyn);
    if (grp.world > 1) node_group_flags_kernel<<<1, 32, 0, cs>>>(grp, gs, d_flags, 60ull * 1000 * 1000 * 1000, dyn);
  };
  auto build = [&]() -> cudaError_t {
    cudaError_t r;
    if ((r = cudaGraphCreate(&g, 0)) != cudaSuccess) return r;
    cudaGraphConditionalHandle h_outer, h_inner;
    if ((r = cudaGraphConditionalHandleCreate(&h_outer, g, 1, cudaGraphCondAssignDefault)) != cudaSuccess) return r;
    cudaGraphNodeParams op = {};
    op.type = cudaGraphNodeTypeConditional;
    op.conditional.handle = h_outer;
    op.conditional.type = cudaGraphCondTypeWhile;
    op.conditional.size = 1;
    cudaGraphNode_t outer_node;
    if ((r = cudaGraphAddNode(&outer_node, g, nullptr, 0, &op)) != cudaSuccess) return r;
    outer_body = op.conditional.phGraph_out[0];
    if ((r = cudaGraphConditionalHandleCreate(&h_inner, outer_body, 0, 0)) != cudaSuccess) return r;
    // chunk prologue: initial iterate, rate, first residual and the predicate
    if ((r = cudaStreamBeginCaptureToGraph(cs, outer_body, nullptr, nullptr, 0, cudaStreamCaptureModeRelaxed)) !=
        cudaSuccess)
      return r;
    node_init_chunk_kernel<<<blocks_for(Pmax * N, 256), 256, 0, cs>>>(states, dy, 0, cmax, nb, dyn);
    eval(0);
    residual(1);
    ctl_newton_start<<<1, 1, 0, cs>>>(dyn, d_flags, h_outer, h_inner);
    if ((r = cudaStreamEndCapture(cs, &outer_body)) != cudaSuccess) return r;
    cudaGraphNode_t pro_leaf;
    if ((r = graph_leaf(outer_body, &pro_leaf)) != cudaSuccess) return r;
    // Newton iterations
    cudaGraphNodeParams ip = {};
    ip.type = cudaGraphNodeTypeConditional;
    ip.conditional.handle = h_inner;
    ip.conditional.type = cudaGraphCondTypeWhile;
    ip.conditional.size = 1;
    cudaGraphNode_t inner_node;
    if ((r = cudaGraphAddNode(&inner_node, outer_body, &pro_leaf, 1, &ip)) != cudaSuccess) return r;
    inner_body = ip.conditional.phGraph_out[0];
    if ((r = cudaStreamBeginCaptureToGraph(cs, inner_body, nullptr, nullptr, 0, cudaStreamCaptureModeRelaxed)) !=
        cudaSuccess)
      return r;
    ctl_newton_iter<<<1, 1, 0, cs>>>(dyn, d_flags, h_outer, h_inner);
    eval(1);
    node_factor_kernel<<<blocks_for(Pmax, 128), 128, 0, cs>>>(Jb, times, 0, cmax, nb, 0, recs, sing_key, 0, nc, d_flags,
                                                             dyn);
    node_thomas_fwd_kernel<<<blocks_for(nb, kSubThreads), kSubThreads, kSubSmem, cs>>>(states, R, recs, 0, cmax, nb,
                                                                                        dyn);
    eval(0);
    residual(0);
    ctl_newton_end<<<1, 1, 0, cs>>>(dyn, d_flags, sing_key, h_outer, h_inner);
    if ((r = cudaStreamEndCapture(cs, &inner_body)) != cudaSuccess) return r;
    // chunk epilogue
    if ((r = cudaStreamBeginCaptureToGraph(cs, outer_body, &inner_node, nullptr, 1, cudaStreamCaptureModeRelaxed)) !=
        cudaSuccess)
      return r;
    ctl_chunk_end<<<1, 1, 0, cs>>>(dyn, iters, d_flags, h_outer);
    if ((r = cudaStreamEndCapture(cs, &outer_body)) != cudaSuccess) return r;
    return cudaGraphInstantiate(&ge, g, 0);
  };
  e = build();
  if (e == cudaSuccess) e = cudaGraphLaunch(ge, st);
  if (ge) cudaGraphExecDestroy(ge);
  if (g) cudaGraphDestroy(g);
  cudaStreamDestroy(cs);
  return e;
}

// Adjoint over a trajectory for the wide neural ODE (Thomas solver); writes the
// quadrature weights wq and the final lambda.
cudaError_t node_adjoint(const DevModel& m, const double* states, const double* times, const double* dL,
                         const double* loss, int nb, int nt, int nc, double* scratch, double* lam, double* wq,
                         unsigned long long* sing_key, cudaStream_t st) {
  using namespace node;
  const int cmax = nc < nt ? nc : nt;
  const size_t Pmax = (size_t)cmax * nb;
  double* H = scratch;
  double* Jb = H + Pmax * N;
  double* R = Jb + Pmax * N * N;
  double* recs = R + Pmax * N;
  cudaError_t e;
  if ((e = cudaMemsetAsync(lam, 0, sizeof(double) * (size_t)nb * N, st)) != cudaSuccess) return e;
  int step_hi = nt;
  unsigned long long ord = 0;
  while (step_hi >= 1) {
    const int c = min(nc, step_hi);
    const int P = c * nb;
    // row r of the chunk is trajectory step step_hi - r
    if ((e = node_eval(m, states, times, step_hi, -1, nb, P, H, Jb, true, st)) != cudaSuccess) return e;
    node_adj_rhs_kernel<<<blocks_for(P, 128), 128, 0, st>>>(states, times, Jb, dL, loss, lam, step_hi, c, nb, R);
    node_factor_kernel<<<blocks_for(P, 128), 128, 0, st>>>(Jb, times, step_hi, c, nb, 1, recs, sing_key, ord, nc,
                                                             nullptr, nullptr);
    const cudaError_t aattr = allow_smem((const void*)node_thomas_adj_kernel, kSubSmem);
    if (aattr != cudaSuccess) return aattr;
    node_thomas_adj_kernel<<<blocks_for(nb, kSubThreads), kSubThreads, kSubSmem, st>>>(R, recs, times, step_hi, c,
                                                                                        nb, lam, wq);
    step_hi -= c;
    ++ord;
  }
  return cudaGetLastError();
}

cudaError_t preload_node_kernels() {
  using namespace node;
  for (const void* f : {(const void*)ctl_newton_start, (const void*)ctl_newton_iter, (const void*)ctl_newton_end,
                        (const void*)ctl_chunk_end, (const void*)node_eval_kernel, (const void*)node_residual_kernel,
                        (const void*)node_residual_pp_kernel, (const void*)node_factor_kernel,
                        (const void*)node_thomas_fwd_kernel, (const void*)node_adj_rhs_kernel,
                        (const void*)node_thomas_adj_kernel, (const void*)node_init_chunk_kernel,
                        (const void*)node_group_flags_kernel, (const void*)node_vectors_dmma_kernel})
    if (cudaError_t e = preload(f)) return e;
  return cudaSuccess;
}

}  // namespace cko
