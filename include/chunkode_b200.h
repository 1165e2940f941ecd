/*
 * chunkode_b200.h — C ABI of the B200-native chunked backward-Euler path.
 *
 * This is the drop-in boundary for the reference library `chunkode`
 * (/root/reference/proj/core). The reference exposes the path as C++ free
 * functions over an `OdeModel` virtual interface; a C++ shim keeps those
 * signatures and forwards here. Every entry point below
 * names the reference interface it replaces.
 *
 * Conventions:
 *  - no exceptions cross this ABI; every call returns a cko_status and fills
 *    a cko_error whose fields mirror the reference exception types
 *    (/root/reference/proj/core/include/chunkode/errors.hpp:9-69);
 *  - calls are synchronous on return;
 *  - host arrays use the reference layouts: y0 (nb, n) row-major
 *    (arrays.hpp:46-64), times (nt+1, nb) (time_grid.hpp:7-9), states
 *    (nt+1, nb*n) (integrate.hpp:34-50), blocks (nc, nb, n, n) row-major
 *    (arrays.hpp:103-131), chunk vectors (nc, nb, n) (arrays.hpp:66-101);
 *  - `*_device` variants take device pointers in the same layouts (inputs
 *    already resident in HBM) and run on the context's stream;
 *  - one context per host thread; a context is bound to one CUDA device.
 */
#ifndef CHUNKODE_B200_H
#define CHUNKODE_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define CKO_ABI_VERSION 1

/* Status codes: one per reference exception type (errors.hpp:9-69), plus
 * device/communication failures the CPU library cannot have. */
typedef enum {
  CKO_OK = 0,
  CKO_SHAPE_MISMATCH = 1,        /* ShapeMismatch        errors.hpp:14-16 */
  CKO_SINGULAR_BLOCK = 2,        /* SingularBlock        errors.hpp:20-28 */
  CKO_NEWTON_DIVERGENCE = 3,     /* NewtonDivergence     errors.hpp:48-64 */
  CKO_NON_FINITE = 4,            /* NonFiniteOutput      errors.hpp:41-44 */
  CKO_STRATEGY_UNAVAILABLE = 5,  /* StrategyUnavailable  errors.hpp:36-39 */
  CKO_SIZE_GUARD = 6,            /* SizeGuardExceeded    errors.hpp:31-34 */
  CKO_INVALID_TIME_GRID = 7,     /* InvalidTimeGrid      errors.hpp:67-69 */
  CKO_ERROR = 8,                 /* plain chunkode::Error errors.hpp:9-11 */
  CKO_CUDA = 9,                  /* CUDA runtime / launch failure */
  CKO_COMM = 10                  /* multi-GPU exchange failure */
} cko_status;

/* Error payload. Field meanings follow the reference exceptions:
 *  SingularBlock{chunk_index = row within the chunk, batch_index}
 *  NewtonDivergence{chunk_start_step, batch_index (worst lane, integrate.cpp:167-174),
 *                   iterations, residual_norm, initial_norm}
 * batch_index is always a GLOBAL lane index (lane_offset applied). */
typedef struct {
  int code;
  int chunk_index;
  int batch_index;
  int chunk_start_step;
  int iterations;
  double residual_norm;
  double initial_norm;
  char msg[256];
} cko_error;

/* WorkCounters (integrate.hpp:17-32): batched-call tallies. */
typedef struct {
  long long newton_iterations;
  long long rate_evals;
  long long jacobian_evals;
  long long linear_solves;
  long long reduction_sweeps;
} cko_work;

/* NewtonSettings (integrate.hpp:9-13). */
typedef struct {
  double tol_a; /* 1e-8 */
  double tol_r; /* 1e-6 */
  int max_iter; /* 100 */
} cko_newton_settings;

/* SolverChoice (linalg.hpp:89-95). */
typedef enum { CKO_SOLVER_THOMAS = 0, CKO_SOLVER_PCR = 1, CKO_SOLVER_HYBRID = 2 } cko_solver_kind;
typedef struct {
  int kind;     /* cko_solver_kind */
  int n_switch; /* hybrid reduction depth (default 1) */
} cko_solver_choice;

/* Device model kinds: device twins of the bundled reference models
 * (models.hpp:14-41) plus the two models the benchmark configs add. */
typedef enum {
  CKO_MODEL_SCALAR_DECAY = 0,  /* models_simple.cpp:9-27   n=1, p=[p]                    */
  CKO_MODEL_CONSTANT_RATE = 1, /* models_simple.cpp:29-45  n=1, p=[c]                    */
  CKO_MODEL_LIN3 = 2,          /* SURVEY §8d C1            n=3, p=[A(3x3), f_a]          */
  CKO_MODEL_MDS = 3,           /* models_mds.cpp:16-97     n=2u, p=[K(u),C(u),M(u),f_a,T(nb)] */
  CKO_MODEL_CHABOCHE = 4,      /* models_chaboche.cpp:19-194 n=2+u,
                                  p=[E,n,eta,s0,Kinf,tau,C(u),gamma(u),eps_a(nb),T]  */
  CKO_MODEL_NODE = 5,          /* models_node.cpp:13-205 (width = u+1) and the wide
                                  variant: n=u, p=[W1(Wx(u+1)),b1(W),
                                  W2(WxW),b2(W),W3(uxW),b3(u)]                        */
  CKO_MODEL_NEURON = 6         /* models_neuron.cpp:16-156 n=4u, p=[14 per-unit
                                  segments (C,g_Na,E_Na,g_K,E_K,g_L,E_L,m_inf,tau_m,
                                  h_inf,tau_h,n_inf,tau_n,g_C), I_a(nb), T(u)]; u <= 8 */
} cko_model_kind;

/* JacobianStrategy (ode_model.hpp:14): analytic = the device twins' hand-written
 * Jacobians; forward_ad = device dual numbers, eight columns per pass
 * (ode_model.hpp:132-151); finite_difference = central differences
 * (ode_model.cpp:44-66). Non-analytic strategies run the generic kernels. */
typedef enum {
  CKO_JACOBIAN_ANALYTIC = 0,
  CKO_JACOBIAN_FORWARD_AD = 1,
  CKO_JACOBIAN_FINITE_DIFFERENCE = 2
} cko_jacobian_strategy;

/* Flat model description, the C image of an OdeModel's identity:
 * kind + dims + params() (ode_model.hpp:35). n_batch_model is the batch width
 * the parameterisation was built for (OdeModel::n_batch, 0 = any);
 * lane_offset maps local lane 0 to a global lane (batch sharding), so
 * per-lane parameters (MDS T_b, Chaboche eps_a_b, NODE/LIN3 periods) are
 * indexed by lane_offset + local lane. `params` is a host pointer. */
typedef struct {
  int kind;          /* cko_model_kind */
  int n_unit;        /* MDS/Chaboche/NODE unit count; ignored otherwise */
  int width;         /* NODE hidden width W (reference node: n_unit+1) */
  int n_batch_model; /* parameterised batch width */
  int lane_offset;   /* global lane index of local lane 0 */
  int n_params;      /* length of params */
  const double* params;
} cko_model_desc;

typedef struct cko_ctx cko_ctx;
typedef struct cko_model cko_model;
typedef struct cko_traj cko_traj;

/* ---- context ------------------------------------------------------------ */
int cko_abi_version(void);
int cko_model_state_size(const cko_model_desc* desc);
/* Parameter count the kind implies for (n_unit, width, n_batch_model). */
int cko_model_param_count(const cko_model_desc* desc);

/* Bind a context to CUDA device `device` with its own non-blocking stream. */
cko_status cko_ctx_create(int device, cko_ctx** out, cko_error* err);
cko_status cko_ctx_destroy(cko_ctx* ctx);
/* Use an external stream (cudaStream_t) instead of the context's own. */
cko_status cko_ctx_set_stream(cko_ctx* ctx, void* cuda_stream);
/* Batch sharding: join a group of `world` ranks, one per GPU.
 * `peer_buffers` are this rank's view of every rank's exchange buffer (device
 * pointers made accessible through CUDA IPC/P2P, world entries, each
 * cko_comm_buffer_bytes() long, own buffer at index rank). The forward kernel
 * then ORs its Newton predicate flags across ranks every iteration, and the
 * adjoint sums the loss and the gradient across ranks, all through P2P stores
 * over NVLink. With world == 1 sharding is off. */
size_t cko_comm_buffer_bytes(void);
cko_status cko_ctx_set_group(cko_ctx* ctx, int rank, int world, void* const* peer_buffers,
                             cko_error* err);
/* Allocate this rank's zeroed exchange buffer and export its CUDA IPC handle
 * (64 bytes) for the peers; open a peer's handle into this process. The
 * caller moves handles between ranks (e.g. torch.distributed all_gather). */
cko_status cko_comm_alloc(cko_ctx* ctx, void** dev_buf, void* ipc_handle_out, cko_error* err);
cko_status cko_comm_open(cko_ctx* ctx, const void* ipc_handle, void** peer_buf, cko_error* err);

/* ---- models ------------------------------------------------------------- */
/* Validate `desc` and upload its parameters to the device once.
 * Replaces the per-call parameter walk of OdeModel::params()/eval_point
 * (ode_model.hpp:103-128). Unknown kinds -> CKO_STRATEGY_UNAVAILABLE. */
cko_status cko_model_create(cko_ctx* ctx, const cko_model_desc* desc, cko_model** out,
                            cko_error* err);
cko_status cko_model_destroy(cko_model* model);

/* ---- integrator --------------------------------------------------------- */
/* integrate_backward_euler (integrate.hpp:86-89, integrate.cpp:321-369).
 * y0 (nb, n), times (nt+1, nb) are HOST arrays; the trajectory stays on the
 * device (traj_out, may be NULL) and/or is copied to states_out (nt+1, nb*n)
 * (may be NULL). `work` receives the forward WorkCounters. */
cko_status cko_be_forward(cko_ctx* ctx, const cko_model* model, const double* y0,
                          const double* times, int nb, int nt, int n_chunk,
                          const cko_newton_settings* settings, const cko_solver_choice* solver,
                          double* states_out, cko_traj** traj_out, cko_work* work,
                          cko_error* err);

/* Same, device pointers in and out (d_states: (nt+1, nb*n)). */
cko_status cko_be_forward_device(cko_ctx* ctx, const cko_model* model, const double* d_y0,
                                 const double* d_times, int nb, int nt, int n_chunk,
                                 const cko_newton_settings* settings,
                                 const cko_solver_choice* solver, double* d_states,
                                 cko_work* work, cko_error* err);

/* ---- adjoint ------------------------------------------------------------ */
typedef enum { CKO_LOSS_FROBENIUS = 0, CKO_LOSS_USER = 1 } cko_loss_kind;

/* adjoint_backward(..., Scheme::backward_euler, ...) (adjoint.hpp:63-66,
 * adjoint.cpp:263-297) over a device trajectory. loss_kind FROBENIUS computes
 * L = sqrt(sum_{step>=1} y^2) and dL/dy = y / L (adjoint.cpp:196-221);
 * USER takes dL (nt+1, nb*n) from the host array dL_host (loss_out then
 * receives NaN: the loss value belongs to the caller). grad_out (np) is a
 * host array. */
cko_status cko_be_adjoint(cko_ctx* ctx, const cko_model* model, const cko_traj* traj, int n_chunk,
                          const cko_solver_choice* solver, int loss_kind, const double* dL_host,
                          double* loss_out, double* grad_out, cko_work* bwd, cko_error* err);

/* Same over a host trajectory: states (nt+1, nb*n), times (nt+1, nb). */
cko_status cko_be_adjoint_host(cko_ctx* ctx, const cko_model* model, const double* states,
                               const double* times, int nb, int nt, int n_chunk,
                               const cko_solver_choice* solver, int loss_kind,
                               const double* dL_host, double* loss_out, double* grad_out,
                               cko_work* bwd, cko_error* err);

/* Same, device pointers (d_dL may be NULL for FROBENIUS); grad_out is host. */
cko_status cko_be_adjoint_device(cko_ctx* ctx, const cko_model* model, const double* d_states,
                                 const double* d_times, int nb, int nt, int n_chunk,
                                 const cko_solver_choice* solver, int loss_kind,
                                 const double* d_dL, double* loss_out, double* grad_out,
                                 cko_work* bwd, cko_error* err);

/* gradient_adjoint (adjoint.hpp:76-80, adjoint.cpp:299-313) for the
 * Frobenius loss: forward then adjoint, host buffers in and out. states_out
 * may be NULL. */
cko_status cko_gradient_adjoint(cko_ctx* ctx, const cko_model* model, const double* y0,
                                const double* times, int nb, int nt, int n_chunk,
                                const cko_newton_settings* settings,
                                const cko_solver_choice* solver, double* states_out,
                                double* loss_out, double* grad_out, cko_work* fwd, cko_work* bwd,
                                cko_error* err);

/* Same over device buffers: d_y0 (nb, n) and d_times (nt+1, nb) in, the trajectory
 * into d_states (nt+1, nb*n; d_states may alias d_y0 as its row 0); loss_out and
 * grad_out (np) are host. One call is one training step: the Frobenius loss rides
 * on the forward's residual passes instead of a separate pass over the trajectory. */
cko_status cko_gradient_adjoint_device(cko_ctx* ctx, const cko_model* model, const double* d_y0,
                                       const double* d_times, int nb, int nt, int n_chunk,
                                       const cko_newton_settings* settings,
                                       const cko_solver_choice* solver, double* d_states,
                                       double* loss_out, double* grad_out, cko_work* fwd,
                                       cko_work* bwd, cko_error* err);

cko_status cko_traj_states(const cko_traj* traj, const double** d_states, int* nb, int* nt,
                           int* n);
cko_status cko_traj_destroy(cko_traj* traj);

/* ---- forward Euler scheme ----------------------------- */
/* integrate_forward_euler (integrate.hpp:91-96, integrate.cpp:371-407): host y0 (nb, n),
 * times (nt+1, nb) -> states_out (nt+1, nb*n); strictly step-sequential, so the result
 * does not depend on n_chunk (>= 1). A non-finite state -> CKO_NON_FINITE naming the step.
 * `work` receives rate_evals = nt. */
cko_status cko_fe_forward(cko_ctx* ctx, const cko_model* model, const double* y0, const double* times, int nb,
                          int nt, int n_chunk, double* states_out, cko_work* work, cko_error* err);

/* adjoint_backward(..., Scheme::forward_euler, ...) (adjoint.hpp:63-66, adjoint.cpp:157-188)
 * over a HOST trajectory; arguments as cko_be_adjoint_host. No linear solves: the backward
 * counters carry one Jacobian evaluation per chunk. */
cko_status cko_fe_adjoint_host(cko_ctx* ctx, const cko_model* model, const double* states, const double* times,
                               int nb, int nt, int n_chunk, int loss_kind, const double* dL_host,
                               double* loss_out, double* grad_out, cko_work* bwd, cko_error* err);

/* ---- block-bidiagonal solver -------------------------------------------- */
/* solve_thomas / solve_pcr / solve_hybrid (linalg.hpp:55-81,
 * linalg.cpp:307-344): diag (nc, nb, n, n), offdiag (nc-1, nb, n, n) or NULL
 * for the -I couplings of the stepper (detail::solve_unit_offdiag,
 * linalg.cpp:288-303); rhs (nc, nb, n) is overwritten by x. Host arrays.
 * *sweeps receives the reduction sweep count (sum of e_i over partitions). */
cko_status cko_block_bidiag_solve(cko_ctx* ctx, const cko_solver_choice* solver, int nc, int nb,
                                  int n, const double* diag, const double* offdiag,
                                  double* rhs_inout, long long* sweeps, cko_error* err);

/* ---- single-chunk ops (integrate.hpp:53-77, adjoint.hpp:36-56) ------------ */
/* Kernel-level parity points; they run the generic (generation 1) kernels.
 *
 * newton_solve_chunk (integrate.hpp:63-67, integrate.cpp:299-319): dy (c, nb, n)
 * in/out, y_start (nb, n), t_chunk and dt_chunk (c, nb) used as given (dt_chunk
 * need not be the differences of t_chunk); returns the iteration count in
 * *iterations; `work` receives this call's counters. */
cko_status cko_newton_solve_chunk(cko_ctx* ctx, const cko_model* model, const double* y_start,
                                  double* dy, const double* t_chunk, const double* dt_chunk,
                                  int c, int nb, const cko_newton_settings* settings,
                                  const cko_solver_choice* solver, int chunk_start_step,
                                  int* iterations, cko_work* work, cko_error* err);

/* chunk_residual (integrate.hpp:53-55, integrate.cpp:269-278):
 * out(j) = dy(j) - dy(j-1) - h(y_start + dy(j), t_chunk(j)) dt_chunk(j), out (c, nb, n).
 * A non-finite rate -> CKO_NON_FINITE (NonFiniteOutput). */
cko_status cko_chunk_residual(cko_ctx* ctx, const cko_model* model, const double* y_start, const double* dy,
                              const double* t_chunk, const double* dt_chunk, int c, int nb, double* out,
                              cko_error* err);

/* chunk_jacobian (integrate.hpp:57-61, integrate.cpp:280-297), analytic Jacobian:
 * diag_out (c, nb, n, n) = I - J(y_start + dy(j), t_chunk(j)) dt_chunk(j); offdiag_out
 * (c-1, nb, n, n) = -I (may be NULL). A non-finite J -> CKO_NON_FINITE. */
cko_status cko_chunk_jacobian(cko_ctx* ctx, const cko_model* model, const double* y_start, const double* dy,
                              const double* t_chunk, const double* dt_chunk, int c, int nb, double* diag_out,
                              double* offdiag_out, cko_error* err);

/* adjoint_chunk_solve (adjoint.hpp:49-56, adjoint.cpp:246-261) over a HOST trajectory
 * states (nt+1, nb*n), times (nt+1, nb) and loss gradient dL (nt+1, nb*n): reverses
 * steps step_hi - chunk_len + 1 .. step_hi in one coupled solve. lambda (nb, n) is the
 * AdjointState carry (in/out); grad (np) accumulates the chunk's quadrature. `work`
 * receives this call's counters (one Jacobian evaluation, one solve, its sweeps). */
cko_status cko_adjoint_chunk_solve(cko_ctx* ctx, const cko_model* model, const double* states,
                                   const double* times, int nb, int nt, int step_hi, int chunk_len,
                                   const double* dL, const cko_solver_choice* solver, double* lambda,
                                   double* grad, cko_work* work, cko_error* err);

/* adjoint_step_sequential (adjoint.hpp:36-47, adjoint.cpp:223-244): one reverse step
 * with y_i, y_prev, dL_i (nb, n) and t_i, t_prev (nb); t_i > t_prev per lane, else
 * CKO_SHAPE_MISMATCH. lambda (nb, n) in/out, grad (np) accumulates. */
cko_status cko_adjoint_step_sequential(cko_ctx* ctx, const cko_model* model, const double* y_i,
                                       const double* y_prev, const double* t_i, const double* t_prev,
                                       const double* dL_i, int nb, const cko_solver_choice* solver,
                                       double* lambda, double* grad, cko_error* err);

/* ---- measurement ----------------------------------------------------------- */
/* Record CUDA events around every kernel launch on the context stream;
 * cko_ctx_last_kernel_ms returns the durations of the last call's kernels:
 * out[0] forward kernel, out[1] adjoint kernel, out[2] parameter-VJP
 * kernels, out[3] loss kernels (0 when not launched). */
cko_status cko_ctx_enable_timing(cko_ctx* ctx, int on);
cko_status cko_ctx_last_kernel_ms(cko_ctx* ctx, double* out4);
/* Kernel launches made by the last forward / adjoint call (for accounting). */
int cko_ctx_last_launches(cko_ctx* ctx);
/* Kernel generation: 2 (default) runs the warp-specialised producer/consumer
 * Thomas kernels for the state sizes they are instantiated for, 1 forces the
 * generic per-point kernels everywhere (A/B measurement and cross-checks).
 * cko_ctx_kernel_generation_used reports what the last forward / adjoint ran. */
cko_status cko_ctx_set_kernel_generation(cko_ctx* ctx, int gen);
int cko_ctx_kernel_generation_used(cko_ctx* ctx);
/* Structured-record Thomas kernels (generation 2, models whose block
 * M = I - dt J is [I B; C D] with B, C diagonal bands and D tridiagonal: the
 * mass-damper-spring chain). On by default; they reproduce lu_factor_block /
 * lu_solve_vec (linalg.cpp:13-60) whenever the reference would not exchange
 * rows, and hand any other block (pivoting, singular, non-finite) back to the
 * group-LU kernels by re-running the call. cko_ctx_structured_used returns
 * the CKO_SP_* bits of the last forward / adjoint call. */
#define CKO_SP_FWD 1           /* the forward ran on the structured kernels */
#define CKO_SP_ADJ 2           /* the adjoint ran on the structured kernels */
#define CKO_SP_FWD_FALLBACK 4  /* the forward was re-run on the group-LU kernels */
#define CKO_SP_ADJ_FALLBACK 8  /* the adjoint was re-run on the group-LU kernels */
cko_status cko_ctx_set_structured(cko_ctx* ctx, int on);
int cko_ctx_structured_used(cko_ctx* ctx);
/* JacobianStrategy of the context's following calls (default analytic). */
cko_status cko_ctx_set_jacobian_strategy(cko_ctx* ctx, int strategy);
/* FP64 FMA-pipe throughput probe (dependent-chain-free DFMA stream over all
 * SMs); writes TFLOP/s (2 flops per DFMA). The FP64 roof for the roofline. */
cko_status cko_probe_fp64_tflops(cko_ctx* ctx, double* tflops, cko_error* err);

#ifdef __cplusplus
}
#endif

#endif /* CHUNKODE_B200_H */
