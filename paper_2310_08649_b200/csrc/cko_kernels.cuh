// cko_kernels.cuh — launch interface between the C ABI (cko_api.cu) and the
// sm_100a kernels (cko_kernels.cu).
#pragma once

#include <cstddef>
#include <cstdint>
#include <cuda_runtime.h>

#include "cko_common.cuh"
#include "cko_models.cuh"

namespace cko {

// Per-CTA workspace slab. Arrays are [elements][Pmax] with Pmax = nc * Lmax
// points (point p = row * L + local lane).
struct Slab {
  double* base;    // G slabs of `doubles` each
  int* pbase;      // G pivot slabs of `ints` each
  size_t doubles;  // per CTA
  size_t ints;     // per CTA
  int Pmax;
  int Lmax;
};

size_t slab_doubles_per_point(int n, bool pcr);

struct FwdLaunch {
  DevModel m;
  double* states;        // (nt+1, nb, n), row 0 = y0 on entry
  const double* times;   // (nt+1, nb)
  const double* dy_init; // optional (nc, nb, n): initial increments (newton_solve_chunk)
  const double* dts;     // optional (nt, nb): explicit step sizes dt(s, b) = dts[(s-1) nb + b] instead of
                         // t(s) - t(s-1) (newton_solve_chunk's independent dt_chunk; generic kernels only)
  int nb, nt, nc;
  double tol_a, tol_r;
  int max_iter;
  int solver, n_switch;
  Slab slab;
  double* rn;             // (nb) last residual norms
  double* r0;             // (nb) initial residual norms of the current chunk
  int* iters;             // (n_chunks) Newton iterations per chunk
  GridSync* gs;
  GroupView grp;
  unsigned long long* sing_key;  // min over k * nb + b of singular blocks
  int* info;             // [0] status, [1] chunk_start_step, [2] iterations, [3] n_chunks done
  uint64_t budget_ns;
  unsigned long long* trace;  // optional diagnostics (CKO_TRACE): per-row timestamps of CTA 0
  double* loss_part;      // optional (grid): per-CTA sum of y^2 over rows 1..nt (generation-2 kernels)
  // optional streamed time grid (generation-2 kernels): rows [0, R) of `times` are resident once
  // *times_ready >= times_tag + R (written by the copy stream after each piece)
  const unsigned long long* times_ready;
  unsigned long long times_tag;
  int grid;               // CTAs
  int threads;
  int structured;         // 1: structured-record kernels where the model has them (cko_sparse.cuh);
                          // info[0] = 5 asks the caller to re-run with 0
};

struct AdjLaunch {
  DevModel m;
  const double* states;  // (nt+1, nb, n)
  const double* times;   // (nt+1, nb)
  const double* dL;      // optional user dL (nt+1, nb, n); null = Frobenius y / L
  const double* loss;    // device scalar L (Frobenius)
  const double* loss_part;  // optional: the forward's per-CTA sums of y^2 (loss_nparts of them); the v2 kernel
  int loss_nparts;          // then forms L itself and CTA 0 stores it to loss_out
  double* loss_out;
  int nb, nt, nc;
  int solver, n_switch;
  Slab slab;
  double* lambda;        // (nb, n): the carry; zeroed on entry unless keep_lambda (adjoint_chunk_solve)
  int keep_lambda;       // generic kernels only
  double* wq;            // (nt+1, nb, n) quadrature weights lambda_m dt_m (row 0 unused)
  unsigned long long* sing_key;  // min over (chunk ordinal, r, b)
  int grid;
  int threads;
  int structured;          // as FwdLaunch::structured; an ineligible block sets *sp_fallback
  unsigned* sp_fallback;
};

struct SolveLaunch {
  const double* diag;     // (nc, nb, n, n)
  const double* offdiag;  // (nc-1, nb, n, n) or null (-I)
  double* x;              // (nc, nb, n) rhs in, solution out
  int nc, nb, n;
  int solver, n_switch;
  Slab slab;
  unsigned long long* sing_key;
  int grid;
  int threads;
};

cudaError_t launch_forward(const FwdLaunch& a, cudaStream_t st);
int forward_max_grid(int kind, int threads, int device);
cudaError_t launch_adjoint(const AdjLaunch& a, cudaStream_t st);
cudaError_t launch_solve(const SolveLaunch& a, cudaStream_t st);
// v2 warp-specialised Thomas kernels (cko_v2.cuh), one CTA per SM with
// a.grid CTAs; a == nullptr probes support for (kind, n). Forward needs a
// slab of Pmax * (n + 1) doubles per CTA (residual rows + point norms).
cudaError_t launch_forward_v2(int kind, int n, const FwdLaunch* a, cudaStream_t st);
cudaError_t launch_adjoint_v2(int kind, int n, const AdjLaunch* a, cudaStream_t st);
// Wide neural ODE (state 8, width 128) on DMMA tensor cores, host-driven
// Newton loop (cko_node.cu). Scratch: node_scratch_doubles(nb, min(nc, nt)).
bool node_fast_path(const DevModel& m);
size_t node_scratch_doubles(int nb, int c);
// The same integration with the Newton loop on the device (nested CUDA-graph WHILE nodes); d_ctl holds
// 16 control ints then the per-chunk iteration counts.
cudaError_t node_forward_graph(const DevModel& m, double* states, const double* times, const double* dy, int nb,
                               int nt, int nc, double tol_a, double tol_r, int max_iter, double* scratch, double* r0,
                               double* rn, unsigned* d_flags, unsigned long long* sing_key, const GroupView& grp,
                               GridSync* gs, int* d_ctl, cudaStream_t st);
cudaError_t node_forward(const DevModel& m, double* states, const double* times, const double* dy, int nb, int nt,
                         int nc, double tol_a, double tol_r, int max_iter, double* scratch, double* r0, double* rn,
                         unsigned* d_flags, unsigned* h_flags, unsigned long long* sing_key, const GroupView& grp,
                         GridSync* gs, int* iters, int* info, cudaStream_t st);
cudaError_t node_adjoint(const DevModel& m, const double* states, const double* times, const double* dL,
                         const double* loss, int nb, int nt, int nc, double* scratch, double* lam, double* wq,
                         unsigned long long* sing_key, cudaStream_t st);
// v2 PCR / hybrid kernels for small blocks (cko_pcr2.cuh), one CTA per SM.
// Slab per CTA: Pmax (n + 1) + Pmax * pcr2_ws_bound(n) doubles.
cudaError_t launch_forward_pcr2(int kind, int n, const FwdLaunch* a, cudaStream_t st);
cudaError_t launch_adjoint_pcr2(int kind, int n, const AdjLaunch* a, cudaStream_t st);
inline int pcr2_ws_bound(int n) { return 3 * n * n + 5 * n + 20; }
// L = sqrt(sum_{m>=1} y^2) into *loss (device); scratch >= 1025 doubles. With a
// group (world > 1) the sum of squares is summed over ranks first.
cudaError_t launch_loss(const double* states, int nt, int row, double* scratch, double* loss,
                        const GroupView& g, GridSync* gs, unsigned* status, cudaStream_t st);
// The same from nparts per-CTA partial sums of y^2 (FwdLaunch::loss_part); scratch >= 1 double.
cudaError_t launch_loss_final(const double* part, int nparts, double* scratch, double* loss, const GroupView& g,
                              GridSync* gs, unsigned* status, cudaStream_t st);
// In-place deterministic sum of v[0..cnt) over the ranks of the group.
cudaError_t launch_chunk_op(const DevModel& m, int op, const double* ys, const double* dy, const double* t,
                            const double* dt, int c, int nb, double* yyb, double* out, unsigned* flags,
                            cudaStream_t st);
cudaError_t launch_fe_forward(const DevModel& m, double* states, const double* times, int nb, int nt, double* hbuf,
                              int* bad, cudaStream_t st);
cudaError_t launch_fe_adjoint(const DevModel& m, const double* states, const double* times, const double* dL,
                              const double* loss, int nb, int nt, double* lambda, double* Jb, double* tmp,
                              double* wq, unsigned* bad, cudaStream_t st);
cudaError_t preload_kernels();
cudaError_t preload_node_kernels();
cudaError_t launch_key_flag(const unsigned long long* key, double* v, cudaStream_t st);
cudaError_t launch_group_sum(const GroupView& g, GridSync* gs, double* v, int cnt, unsigned* status,
                             cudaStream_t st);
// grad (device, np) = sum over (m >= 1, b) of w . dh/dp; scratch sized by vjp_scratch_doubles.
size_t vjp_scratch_doubles(const DevModel& m, int nb, int nt);
// Wide neural ODE (parameter count beyond the per-thread accumulators): the
// VJP as split-K outer products (cko_node_vjp.cu).
bool vjp_needs_outer(const DevModel& m);
size_t node_vjp_scratch_doubles(const DevModel& m, int nb, int nt);
cudaError_t launch_node_vectors_dmma(const DevModel& m, const double* states, const double* times, const double* wq,
                                     int nb, size_t P, double* vec, cudaStream_t st);
cudaError_t launch_node_vjp(const DevModel& m, const double* states, const double* times, const double* wq, int nb,
                            int nt, double* scratch, double* grad, cudaStream_t st);
cudaError_t launch_vjp(const DevModel& m, const double* states, const double* times,
                       const double* wq, int nb, int nt, double* scratch, double* grad,
                       cudaStream_t st);

// 8 * iters DFMA per thread of `blocks` x 256 threads.
cudaError_t launch_fp64_probe(double* scratch, int blocks, int iters, cudaStream_t st);

}  // namespace cko
