// cko_api.cu — host implementation of the C ABI in include/chunkode_b200.h.
//
// Owns CUDA resources (stream, grow-only workspace pool, model parameter
// uploads, device trajectories), validates arguments like the reference
// (ShapeMismatch / InvalidTimeGrid checks of integrate.cpp:12-21, 257-265,
// time_grid.cpp:7-19, linalg.cpp:86-98), launches the kernels of
// cko_kernels.cu and maps device status words back to the reference error
// types (errors.hpp:9-69). No CPU fallback exists: without a usable CUDA
// device every entry point returns CKO_CUDA.
#include <algorithm>
#include <atomic>
#include <cmath>
#include <cstdarg>
#include <cstdio>
#include <cstdlib>
#include <cstdint>
#include <cstring>
#include <cuda.h>
#include <new>
#include <numeric>
#include <thread>
#include <vector>

#include "../../include/chunkode_b200.h"
#include "cko_kernels.cuh"
#include "cko_eval.cuh"

using namespace cko;

namespace {

cko_status fail(cko_error* e, cko_status code, const char* fmt, ...) {
  if (e) {
    std::memset(e, 0, sizeof(*e));
    e->code = code;
    va_list ap;
    va_start(ap, fmt);
    std::vsnprintf(e->msg, sizeof e->msg, fmt, ap);
    va_end(ap);
  }
  return code;
}

cko_status ok(cko_error* e) {
  if (e) std::memset(e, 0, sizeof(*e));
  return CKO_OK;
}

#define CUDA_TRY(expr)                                                                    \
  do {                                                                                    \
    cudaError_t _e = (expr);                                                              \
    if (_e != cudaSuccess)                                                                \
      return fail(err, CKO_CUDA, "%s failed: %s", #expr, cudaGetErrorString(_e));        \
  } while (0)
#define CUDA_TRY_RAW(expr)           \
  do {                               \
    const cudaError_t _e = (expr);   \
    if (_e != cudaSuccess) return _e; \
  } while (0)

struct Buf {
  void* p = nullptr;
  size_t bytes = 0;
  void release() {
    if (p) cudaFree(p);
    p = nullptr;
    bytes = 0;
  }
  cudaError_t ensure(size_t b) {
    if (b <= bytes) return cudaSuccess;
    release();
    cudaError_t e = cudaMalloc(&p, b < 256 ? 256 : b);
    if (e == cudaSuccess) bytes = b;
    return e;
  }
  template <class T>
  T* as() const {
    return static_cast<T*>(p);
  }
};

int state_size(const cko_model_desc* d) {
  switch (d->kind) {
    case CKO_MODEL_SCALAR_DECAY:
    case CKO_MODEL_CONSTANT_RATE: return 1;
    case CKO_MODEL_LIN3: return 3;
    case CKO_MODEL_MDS: return d->n_unit >= 1 ? 2 * d->n_unit : -1;
    case CKO_MODEL_CHABOCHE: return d->n_unit >= 1 ? 2 + d->n_unit : -1;
    case CKO_MODEL_NODE: return d->n_unit >= 1 ? d->n_unit : -1;
    case CKO_MODEL_NEURON: return d->n_unit >= 1 ? 4 * d->n_unit : -1;
  }
  return -1;
}

int param_count(const cko_model_desc* d) {
  const int u = d->n_unit, W = d->width, nb = d->n_batch_model;
  switch (d->kind) {
    case CKO_MODEL_SCALAR_DECAY:
    case CKO_MODEL_CONSTANT_RATE: return 1;
    case CKO_MODEL_LIN3: return 10;
    case CKO_MODEL_MDS: return 3 * u + 1 + nb;
    case CKO_MODEL_CHABOCHE: return 6 + 2 * u + nb + 1;
    case CKO_MODEL_NODE: return W * (u + 1) + W + W * W + W + u * W + u;
    case CKO_MODEL_NEURON: return 15 * u + nb;
  }
  return -1;
}

// chunkode::linspace (linalg.cpp:386-396), bit-exact.
std::vector<double> linspace(double lo, double hi, int n) {
  std::vector<double> v(n > 0 ? n : 0);
  if (n <= 0) return v;
  if (n == 1) {
    v[0] = lo;
    return v;
  }
  for (int i = 0; i < n; ++i) v[i] = lo + (hi - lo) * double(i) / double(n - 1);
  v[n - 1] = hi;
  return v;
}

// Reduction sweeps of one solve of a c-row chunk (linalg.cpp:203-254).
long long sweeps_of(int c, int kind, int n_switch) {
  if (kind == CKO_SOLVER_THOMAS) return 0;
  long long s = 0;
  for (int bit = 30; bit >= 0; --bit) {
    const int m = 1 << bit;
    if (!(c & m)) continue;
    int e = 0;
    while ((1 << e) < m) ++e;
    s += kind == CKO_SOLVER_PCR ? e : (n_switch < e ? n_switch : e);
  }
  return s;
}

}  // namespace

// Grow-only pinned host staging for the small device-to-host results of every
// call (status words, chunk iteration counts, loss, gradient): pinned copies
// stay asynchronous on the context stream and never wait on other streams.
struct PinBuf {
  void* p = nullptr;
  size_t bytes = 0;
  void release() {
    if (p) cudaFreeHost(p);
    p = nullptr;
    bytes = 0;
  }
  cudaError_t ensure(size_t b) {
    if (b <= bytes) return cudaSuccess;
    release();
    const size_t want = b < (256u << 10) ? (256u << 10) : 2 * b;
    cudaError_t e = cudaHostAlloc(&p, want, cudaHostAllocDefault);
    if (e == cudaSuccess) bytes = want;
    return e;
  }
  template <class T>
  T* as(size_t byte_offset = 0) const {
    return reinterpret_cast<T*>(static_cast<char*>(p) + byte_offset);
  }
};

struct cko_ctx {
  int device = 0;
  cudaStream_t stream = nullptr;
  bool own_stream = false;
  cudaStream_t copy_stream = nullptr;  // trajectory downloads overlapping the adjoint
  cudaEvent_t fwd_done = nullptr;
  int sms = 0;
  // workspace pool
  Buf slab, piv, rn, r0, iters, gs, key, info, loss, scratch, lambda, wq, vjp, grad, status, spfb;
  Buf lpart;       // the last forward's per-CTA sums of y^2 (the fused Frobenius loss)
  Buf feed;        // streamed time grid: rows resident (tag + rows, written by the copy stream)
  const unsigned long long* feed_ready = nullptr;  // set for the next forward_core only
  unsigned long long feed_tag = 0;
  cudaEvent_t times_done = nullptr;
  int lpart_n = 0;  // how many (0: the last forward left none)
  Buf h_y0, h_times, h_states, h_dL, h_rhs, h_diag, h_off;  // staging for host-buffer calls
  std::vector<int> iters_host;
  PinBuf pin;
  // batch sharding
  GroupView grp{};
  // kernel timing (cko_ctx_enable_timing)
  int kernel_gen = 2;  // 2: warp-specialised Thomas kernels where instantiated; 1: generic kernels only
  int jstrat = 0;      // JacobianStrategy of the next calls (cko_ctx_set_jacobian_strategy)
  bool timing = false;
  cudaEvent_t ev[8] = {};
  double last_ms[4] = {0, 0, 0, 0};
  int last_launches = 0;
  int last_gen = 0;  // kernel generation the last forward/adjoint call ran
  // structured-record kernels (cko_sparse.cuh) for models with the arrow + tridiagonal block pattern:
  // on by default (CKO_STRUCTURED=0 or cko_ctx_set_structured(ctx, 0) turns them off)
  int structured = [] {
    const char* v = std::getenv("CKO_STRUCTURED");
    return (v && v[0] == '0') ? 0 : 1;
  }();
  int last_sp = 0;  // CKO_SP_* bits of the last forward / adjoint call
  void mark(int i) {
    if (timing) cudaEventRecord(ev[i], stream);
  }
  void collect(int first_pair, int npairs) {
    if (!timing) return;
    for (int k = first_pair; k < first_pair + npairs; ++k) {
      float ms = 0.f;
      if (cudaEventElapsedTime(&ms, ev[2 * k], ev[2 * k + 1]) == cudaSuccess) last_ms[k] = ms;
    }
  }
};

struct cko_model {
  cko_ctx* ctx = nullptr;
  cko_model_desc desc{};
  DevModel dm{};
  double* d_params = nullptr;
  double* d_periods = nullptr;
};

struct cko_traj {
  cko_ctx* ctx = nullptr;
  double* d_states = nullptr;
  double* d_times = nullptr;
  int nb = 0, nt = 0, n = 0;
};

extern "C" {

int cko_abi_version(void) { return CKO_ABI_VERSION; }
int cko_model_state_size(const cko_model_desc* d) { return d ? state_size(d) : -1; }
int cko_model_param_count(const cko_model_desc* d) { return d ? param_count(d) : -1; }
constexpr int kRedCap = 32768;  // doubles per rank row of the peer reduce buffer
constexpr size_t kSlotBytes = 256;
size_t cko_comm_buffer_bytes(void) { return kSlotBytes + sizeof(double) * 2 * 8 * (size_t)kRedCap; }

cko_status cko_ctx_create(int device, cko_ctx** out, cko_error* err) {
  if (!out) return fail(err, CKO_ERROR, "cko_ctx_create: null output");
  *out = nullptr;
  int count = 0;
  cudaError_t e = cudaGetDeviceCount(&count);
  if (e != cudaSuccess || count == 0)
    return fail(err, CKO_CUDA, "no CUDA device available (%s): the B200 path has no CPU fallback",
                e == cudaSuccess ? "0 devices" : cudaGetErrorString(e));
  if (device < 0 || device >= count) return fail(err, CKO_CUDA, "CUDA device %d out of range", device);
  CUDA_TRY(cudaSetDevice(device));
  cko_ctx* c = new (std::nothrow) cko_ctx();
  if (!c) return fail(err, CKO_ERROR, "out of host memory");
  c->device = device;
  cudaDeviceGetAttribute(&c->sms, cudaDevAttrMultiProcessorCount, device);
  e = cudaStreamCreateWithFlags(&c->stream, cudaStreamNonBlocking);
  if (e != cudaSuccess) {
    delete c;
    return fail(err, CKO_CUDA, "cudaStreamCreate: %s", cudaGetErrorString(e));
  }
  c->own_stream = true;
  c->grp.rank = 0;
  c->grp.world = 1;
  e = c->gs.ensure(sizeof(GridSync));
  if (e == cudaSuccess) e = cudaMemset(c->gs.p, 0, sizeof(GridSync));
  if (e != cudaSuccess) {
    delete c;
    return fail(err, CKO_CUDA, "workspace: %s", cudaGetErrorString(e));
  }
  *out = c;
  return ok(err);
}

cko_status cko_ctx_destroy(cko_ctx* c) {
  if (!c) return CKO_OK;
  cudaSetDevice(c->device);
  cudaStreamSynchronize(c->stream);
  for (Buf* b : {&c->slab, &c->piv, &c->rn, &c->r0, &c->iters, &c->gs, &c->key, &c->info, &c->loss, &c->status,
                 &c->scratch, &c->lambda, &c->wq, &c->vjp, &c->grad, &c->h_y0, &c->h_times,
                 &c->h_states, &c->h_dL, &c->h_rhs, &c->h_diag, &c->h_off})
    b->release();
  c->pin.release();
  for (cudaEvent_t& e : c->ev)
    if (e) cudaEventDestroy(e);
  if (c->own_stream) cudaStreamDestroy(c->stream);
  if (c->copy_stream) cudaStreamDestroy(c->copy_stream);
  if (c->fwd_done) cudaEventDestroy(c->fwd_done);
  delete c;
  return CKO_OK;
}

cko_status cko_ctx_enable_timing(cko_ctx* c, int on) {
  if (!c) return CKO_ERROR;
  cudaSetDevice(c->device);
  if (on && !c->ev[0])
    for (cudaEvent_t& e : c->ev)
      if (cudaEventCreate(&e) != cudaSuccess) return CKO_CUDA;
  c->timing = on != 0;
  return CKO_OK;
}

cko_status cko_ctx_last_kernel_ms(cko_ctx* c, double* out4) {
  if (!c || !out4) return CKO_ERROR;
  for (int i = 0; i < 4; ++i) out4[i] = c->last_ms[i];
  return CKO_OK;
}

int cko_ctx_last_launches(cko_ctx* c) { return c ? c->last_launches : 0; }

cko_status cko_ctx_set_kernel_generation(cko_ctx* c, int gen) {
  if (!c || (gen != 1 && gen != 2)) return CKO_ERROR;
  c->kernel_gen = gen;
  return CKO_OK;
}

int cko_ctx_kernel_generation_used(cko_ctx* c) { return c ? c->last_gen : 0; }

cko_status cko_ctx_set_structured(cko_ctx* c, int on) {
  if (!c || (on != 0 && on != 1)) return CKO_ERROR;
  c->structured = on;
  return CKO_OK;
}

int cko_ctx_structured_used(cko_ctx* c) { return c ? c->last_sp : 0; }

cko_status cko_ctx_set_jacobian_strategy(cko_ctx* c, int strategy) {
  if (!c || strategy < CKO_JACOBIAN_ANALYTIC || strategy > CKO_JACOBIAN_FINITE_DIFFERENCE) return CKO_ERROR;
  c->jstrat = strategy;
  return CKO_OK;
}

cko_status cko_probe_fp64_tflops(cko_ctx* c, double* tflops, cko_error* err) {
  if (!c || !tflops) return fail(err, CKO_ERROR, "null argument");
  CUDA_TRY(cudaSetDevice(c->device));
  CUDA_TRY(c->scratch.ensure(sizeof(double) * 1024));
  cudaEvent_t a, b;
  CUDA_TRY(cudaEventCreate(&a));
  CUDA_TRY(cudaEventCreate(&b));
  const int blocks = c->sms * 8, iters = 1 << 14;
  double best = 0.0;
  for (int rep = 0; rep < 4; ++rep) {
    CUDA_TRY(cudaEventRecord(a, c->stream));
    CUDA_TRY(launch_fp64_probe(c->scratch.as<double>(), blocks, iters, c->stream));
    CUDA_TRY(cudaEventRecord(b, c->stream));
    CUDA_TRY(cudaEventSynchronize(b));
    float ms = 0.f;
    CUDA_TRY(cudaEventElapsedTime(&ms, a, b));
    const double flops = 2.0 * 8.0 * iters * 256.0 * blocks;
    if (rep > 0 && ms > 0.f) best = std::max(best, flops / (ms * 1e-3) / 1e12);
  }
  cudaEventDestroy(a);
  cudaEventDestroy(b);
  *tflops = best;
  return ok(err);
}

cko_status cko_ctx_set_stream(cko_ctx* c, void* s) {
  if (!c) return CKO_ERROR;
  if (c->own_stream) cudaStreamDestroy(c->stream);
  c->stream = static_cast<cudaStream_t>(s);
  c->own_stream = false;
  return CKO_OK;
}

cko_status cko_ctx_set_group(cko_ctx* c, int rank, int world, void* const* peers, cko_error* err) {
  if (!c) return fail(err, CKO_ERROR, "null context");
  if (world < 1 || world > 8 || rank < 0 || rank >= world)
    return fail(err, CKO_ERROR, "cko_ctx_set_group: need 1 <= world <= 8, 0 <= rank < world");
  if (world > 1) {  // no lazy module load may stall a rank while its peers spin on the exchange
    CUDA_TRY(cudaSetDevice(c->device));
    CUDA_TRY(preload_kernels());
  }
  c->grp.rank = rank;
  c->grp.world = world;
  c->grp.red_cap = kRedCap;
  for (int r = 0; r < 8; ++r) {
    char* base = (world > 1 && r < world) ? static_cast<char*>(peers[r]) : nullptr;
    c->grp.peer_slots[r] = reinterpret_cast<unsigned long long*>(base);
    c->grp.peer_red[r] = base ? reinterpret_cast<double*>(base + kSlotBytes) : nullptr;
  }
  return ok(err);
}

cko_status cko_comm_alloc(cko_ctx* c, void** dev_buf, void* ipc_handle_out, cko_error* err) {
  if (!c || !dev_buf || !ipc_handle_out) return fail(err, CKO_ERROR, "null argument");
  CUDA_TRY(cudaSetDevice(c->device));
  const size_t bytes = cko_comm_buffer_bytes();
  void* p = nullptr;
  CUDA_TRY(cudaMalloc(&p, bytes));
  CUDA_TRY(cudaMemset(p, 0, bytes));
  cudaIpcMemHandle_t h;
  CUDA_TRY(cudaIpcGetMemHandle(&h, p));
  std::memcpy(ipc_handle_out, &h, sizeof h);
  *dev_buf = p;
  return ok(err);
}

cko_status cko_comm_open(cko_ctx* c, const void* ipc_handle, void** peer_buf, cko_error* err) {
  if (!c || !ipc_handle || !peer_buf) return fail(err, CKO_ERROR, "null argument");
  CUDA_TRY(cudaSetDevice(c->device));
  cudaIpcMemHandle_t h;
  std::memcpy(&h, ipc_handle, sizeof h);
  CUDA_TRY(cudaIpcOpenMemHandle(peer_buf, h, cudaIpcMemLazyEnablePeerAccess));
  return ok(err);
}

cko_status cko_model_create(cko_ctx* c, const cko_model_desc* d, cko_model** out, cko_error* err) {
  if (!c || !d || !out) return fail(err, CKO_ERROR, "cko_model_create: null argument");
  *out = nullptr;
  const int n = state_size(d);
  if (n < 1 || d->kind < 0 || d->kind > CKO_MODEL_NEURON)
    return fail(err, CKO_STRATEGY_UNAVAILABLE, "model kind %d has no device twin", d->kind);
  if (d->kind == CKO_MODEL_NEURON && n > kFadMaxN)
    return fail(err, CKO_STRATEGY_UNAVAILABLE, "neuron model with %d states exceeds the device twin (<= %d)", n,
                kFadMaxN);
  const bool lane_model = d->kind != CKO_MODEL_SCALAR_DECAY && d->kind != CKO_MODEL_CONSTANT_RATE;
  if (lane_model && d->n_batch_model < 1)
    return fail(err, CKO_SHAPE_MISMATCH, "model needs n_batch_model >= 1");
  if (d->kind == CKO_MODEL_NODE && (d->width < 1 || d->width > NODE_MAX_W || n > NODE_MAX_N))
    return fail(err, CKO_STRATEGY_UNAVAILABLE,
                "neural ODE width %d / state %d exceeds the point-wise device kernels (W <= %d, n <= %d)",
                d->width, n, NODE_MAX_W, NODE_MAX_N);
  const int np = param_count(d);
  if (np != d->n_params || !d->params)
    return fail(err, CKO_SHAPE_MISMATCH, "parameter count %d does not match the model (%d)", d->n_params, np);
  CUDA_TRY(cudaSetDevice(c->device));
  cko_model* m = new (std::nothrow) cko_model();
  if (!m) return fail(err, CKO_ERROR, "out of host memory");
  m->ctx = c;
  m->desc = *d;
  m->desc.params = nullptr;
  cudaError_t e = cudaMalloc(&m->d_params, sizeof(double) * np);
  if (e == cudaSuccess) e = cudaMemcpy(m->d_params, d->params, sizeof(double) * np, cudaMemcpyHostToDevice);
  if (e == cudaSuccess && lane_model) {
    const auto per = linspace(1e-2, 1.0, d->n_batch_model);
    e = cudaMalloc(&m->d_periods, sizeof(double) * per.size());
    if (e == cudaSuccess)
      e = cudaMemcpy(m->d_periods, per.data(), sizeof(double) * per.size(), cudaMemcpyHostToDevice);
  }
  if (e != cudaSuccess) {
    cudaFree(m->d_params);
    cudaFree(m->d_periods);
    delete m;
    return fail(err, CKO_CUDA, "model upload: %s", cudaGetErrorString(e));
  }
  DevModel& dm = m->dm;
  dm.kind = d->kind;
  dm.n = n;
  dm.nu = d->n_unit;
  dm.W = d->width;
  dm.nbm = d->n_batch_model;
  dm.off = d->lane_offset;
  dm.np = np;
  dm.p = m->d_params;
  dm.periods = m->d_periods;
  *out = m;
  return ok(err);
}

cko_status cko_model_destroy(cko_model* m) {
  if (!m) return CKO_OK;
  cudaSetDevice(m->ctx->device);
  cudaFree(m->d_params);
  cudaFree(m->d_periods);
  delete m;
  return CKO_OK;
}

}  // extern "C"

namespace {

cko_status check_lanes(const cko_model* m, int nb, cko_error* err) {
  const bool lane_model = m->desc.kind != CKO_MODEL_SCALAR_DECAY && m->desc.kind != CKO_MODEL_CONSTANT_RATE;
  if (lane_model && m->desc.lane_offset + nb > m->desc.n_batch_model)
    return fail(err, CKO_SHAPE_MISMATCH, "integrate: model batch width != y0 rows");
  return CKO_OK;
}

cko_status check_grid_shape(int nt, int nb, cko_error* err) {
  if (nt < 1 || nb < 1)
    return fail(err, CKO_INVALID_TIME_GRID, "time grid needs at least one step and one batch lane");
  return CKO_OK;
}

// TimeGrid validation (time_grid.cpp:7-19) on the device copy: the first
// non-increasing entry in the reference's scan order (step, then lane).
__global__ void grid_check_kernel(const double* __restrict__ t, long long total, int nb,
                                  unsigned long long* __restrict__ key) {
  for (long long e = nb + (long long)blockIdx.x * blockDim.x + threadIdx.x; e < total;
       e += (long long)gridDim.x * blockDim.x)
    if (!(t[e] > t[e - nb])) atomicMin(key, (unsigned long long)e);
}

cko_status check_grid_device(cko_ctx* c, const double* d_times, int nt, int nb, cko_error* err) {
  CUDA_TRY(c->key.ensure(sizeof(unsigned long long)));
  CUDA_TRY(c->pin.ensure(64));
  CUDA_TRY(cudaMemsetAsync(c->key.p, 0xff, sizeof(unsigned long long), c->stream));
  const long long total = (long long)nb * (nt + 1);
  grid_check_kernel<<<4 * c->sms, 256, 0, c->stream>>>(d_times, total, nb, c->key.as<unsigned long long>());
  CUDA_TRY(cudaGetLastError());
  unsigned long long* h = c->pin.as<unsigned long long>(48);
  CUDA_TRY(cudaMemcpyAsync(h, c->key.p, sizeof(unsigned long long), cudaMemcpyDeviceToHost, c->stream));
  CUDA_TRY(cudaStreamSynchronize(c->stream));
  if (*h != ~0ull) {
    const int i = (int)(*h / (unsigned long long)nb), b = (int)(*h % (unsigned long long)nb);
    return fail(err, CKO_INVALID_TIME_GRID, "time grid must be strictly increasing (step %d, batch %d)", i, b);
  }
  return CKO_OK;
}

cko_status prepare_slab(cko_ctx* c, int G, int nb, int nc, int n, bool pcr, Slab& s, cko_error* err) {
  const int Lmax = (nb + G - 1) / G;
  s.Lmax = Lmax;
  s.Pmax = nc * Lmax;
  s.doubles = (size_t)s.Pmax * slab_doubles_per_point(n, pcr);
  s.ints = (size_t)s.Pmax * n;
  CUDA_TRY(c->slab.ensure(sizeof(double) * s.doubles * G));
  CUDA_TRY(c->piv.ensure(sizeof(int) * s.ints * G));
  s.base = c->slab.as<double>();
  s.pbase = c->piv.as<int>();
  return CKO_OK;
}

constexpr int kThreads = 256;
constexpr int kThreadsMax = 1024;  // largest block of any forward kernel (the loss slots)

// Core forward on device buffers (states row 0 must hold y0).
// Whether forward_core runs a generation-2 forward (the kernels that can wait on a streamed grid):
// the same decision forward_core makes for a call without explicit step sizes.
bool fwd_streams_times(cko_ctx* c, const cko_model* m, const cko_solver_choice* sv) {
  if (c->jstrat != 0 || c->kernel_gen < 2 || sv->kind < 0 || sv->kind > 2) return false;
  const int n = m->dm.n;
  if (sv->kind != CKO_SOLVER_THOMAS) return launch_forward_pcr2(m->dm.kind, n, nullptr, c->stream) == cudaSuccess;
  return !node_fast_path(m->dm) && launch_forward_v2(m->dm.kind, n, nullptr, c->stream) == cudaSuccess;
}

// First flat index e >= nb of a host grid (nt+1, nb) with !(t[e] > t[e - nb]), or -1 (grid_check_kernel).
long long first_bad_time(const double* t, int nt, int nb) {
  const long long total = (long long)nb * (nt + 1);
  for (long long e = nb; e < total; ++e)
    if (!(t[e] > t[e - nb])) return e;
  return -1;
}

// cuStreamWriteValue64 (driver API, through the runtime's entry-point query), or null when the driver or
// the device lacks 64-bit stream memory operations.
using WriteValue64Fn = CUresult (*)(CUstream, CUdeviceptr, cuuint64_t, unsigned int);
WriteValue64Fn write_value64(int device) {
  static WriteValue64Fn fn = [] {
    void* f = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuStreamWriteValue64", &f, cudaEnableDefault, &q) != cudaSuccess ||
        q != cudaDriverEntryPointSuccess)
      f = nullptr;
    return reinterpret_cast<WriteValue64Fn>(f);
  }();
  using AttrFn = CUresult (*)(int*, CUdevice_attribute, CUdevice);
  static AttrFn attr = [] {
    void* f = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuDeviceGetAttribute", &f, cudaEnableDefault, &q) != cudaSuccess ||
        q != cudaDriverEntryPointSuccess)
      f = nullptr;
    return reinterpret_cast<AttrFn>(f);
  }();
  int ok = 0;
  if (!fn || !attr || attr(&ok, CU_DEVICE_ATTRIBUTE_CAN_USE_64_BIT_STREAM_MEM_OPS, device) != CUDA_SUCCESS) ok = 0;
  return ok ? fn : nullptr;
}

cko_status forward_core(cko_ctx* c, const cko_model* m, double* d_states, const double* d_times, int nb, int nt,
                        int nc, const cko_newton_settings* st, const cko_solver_choice* sv, const double* d_dy,
                        cko_work* work, int* iters_out, cko_error* err, const double* d_dts = nullptr,
                        bool want_loss_part = false) {
  if (m) const_cast<cko_model*>(m)->dm.jstrat = c->jstrat;  // the call's JacobianStrategy
  if (nc < 1) return fail(err, CKO_SHAPE_MISMATCH, "integrate: n_chunk must be >= 1");
  if (nt < 1) return fail(err, CKO_SHAPE_MISMATCH, "integrate: need at least one step");
  if (sv->kind < 0 || sv->kind > 2) return fail(err, CKO_ERROR, "unknown solver kind %d", sv->kind);
  if (sv->kind == CKO_SOLVER_HYBRID && sv->n_switch < 0)
    return fail(err, CKO_ERROR, "solve_hybrid: n_switch must be >= 0");
  if (cko_status s = check_lanes(m, nb, err)) return s;
  const int n = m->dm.n;
  const int nc_eff = nc < nt ? nc : nt;
  const bool pcr = sv->kind != CKO_SOLVER_THOMAS;
  // explicit step sizes (single-chunk op) or a non-analytic Jacobian strategy: generic kernels
  const int gen = (d_dts || c->jstrat != 0) ? 1 : c->kernel_gen;
  const bool nodep = !pcr && gen >= 2 && node_fast_path(m->dm);
  const bool v2 = !nodep && !pcr && gen >= 2 && launch_forward_v2(m->dm.kind, n, nullptr, c->stream) == cudaSuccess;
  const bool p2 = pcr && gen >= 2 && launch_forward_pcr2(m->dm.kind, n, nullptr, c->stream) == cudaSuccess;
  int G;
  Slab slab;
  if (v2 || p2) {
    G = nb < c->sms ? nb : c->sms;
    slab.Lmax = (nb + G - 1) / G;
    slab.Pmax = nc_eff * slab.Lmax;
    slab.doubles = (size_t)slab.Pmax * (n + 1) + (p2 ? (size_t)slab.Pmax * pcr2_ws_bound(n) : 0);
    slab.doubles = (slab.doubles + 1) & ~(size_t)1;  // every CTA's slab 16-byte aligned (pair loads)
    slab.ints = 0;
    CUDA_TRY(c->slab.ensure(sizeof(double) * slab.doubles * G));
    slab.base = c->slab.as<double>();
    slab.pbase = nullptr;
  } else {
    int maxg = forward_max_grid(m->dm.kind, kThreads, c->device);
    if (maxg < 1) return fail(err, CKO_CUDA, "forward kernel cannot be made resident");
    G = nb < maxg ? nb : maxg;
    if (cko_status s = prepare_slab(c, G, nb, nc_eff, n, pcr, slab, err)) return s;
  }
  const int n_chunks = (nt + nc - 1) / nc;
  CUDA_TRY(c->rn.ensure(sizeof(double) * nb));
  CUDA_TRY(c->r0.ensure(sizeof(double) * nb));
  CUDA_TRY(c->iters.ensure(sizeof(int) * n_chunks));
  CUDA_TRY(c->key.ensure(sizeof(unsigned long long)));
  CUDA_TRY(c->info.ensure(sizeof(int) * 4));
  CUDA_TRY(cudaMemsetAsync(c->gs.p, 0, offsetof(GridSync, ext_gen), c->stream));
  CUDA_TRY(cudaMemsetAsync(c->key.p, 0xff, sizeof(unsigned long long), c->stream));
  CUDA_TRY(cudaMemsetAsync(c->info.p, 0, sizeof(int) * 4, c->stream));
  FwdLaunch a{};
  a.m = m->dm;
  a.states = d_states;
  a.times = d_times;
  a.dy_init = d_dy;
  a.dts = d_dts;
  a.nb = nb;
  a.nt = nt;
  a.nc = nc;
  a.tol_a = st->tol_a;
  a.tol_r = st->tol_r;
  a.max_iter = st->max_iter;
  a.solver = sv->kind;
  a.n_switch = sv->n_switch;
  a.slab = slab;
  a.rn = c->rn.as<double>();
  a.r0 = c->r0.as<double>();
  a.iters = c->iters.as<int>();
  a.gs = c->gs.as<GridSync>();
  a.grp = c->grp;
  a.sing_key = c->key.as<unsigned long long>();
  a.info = c->info.as<int>();
  a.budget_ns = 60ull * 1000 * 1000 * 1000;
  a.grid = G;
  a.threads = kThreads;
  if (c->feed_ready) {  // the caller streams the grid only to the generation-2 kernels (fwd_streams_times)
    a.times_ready = c->feed_ready;
    a.times_tag = c->feed_tag;
    c->feed_ready = nullptr;
    if (!(v2 || p2)) return fail(err, CKO_ERROR, "internal: streamed time grid for a kernel that cannot wait on it");
  }
  c->lpart_n = 0;
  if (want_loss_part && (v2 || p2)) {  // the loss rides on the residual passes (one partial per CTA)
    CUDA_TRY(c->lpart.ensure(sizeof(double) * G * (1 + 2 * (size_t)kThreadsMax)));  // + per-thread slots
    a.loss_part = c->lpart.as<double>();
  }
  static const char* trace_path = std::getenv("CKO_TRACE");
  Buf tbuf;
  if (trace_path && v2) {
    CUDA_TRY(tbuf.ensure(sizeof(unsigned long long) * (64 + 8 * (size_t)nc_eff + 8 * (size_t)G)));
    CUDA_TRY(cudaMemsetAsync(tbuf.p, 0, tbuf.bytes, c->stream));
    a.trace = tbuf.as<unsigned long long>();
  }
  int info[4];
  unsigned long long key;
  if (nodep) {  // wide neural ODE: DMMA model evaluation, host-driven Newton loop (cko_node.cu)
    CUDA_TRY(c->scratch.ensure(sizeof(double) * node_scratch_doubles(nb, nc_eff)));
    CUDA_TRY(c->status.ensure(sizeof(unsigned)));
    CUDA_TRY(c->pin.ensure(64));
    std::memset(info, 0, sizeof info);
    c->iters_host.assign(n_chunks, 0);
    static const bool host_loop = [] {
      const char* v = std::getenv("CKO_NODE_HOST_LOOP");  // A/B: the host-driven Newton loop
      return v && v[0] == '1';
    }();
    if (host_loop) {
      c->mark(0);
      CUDA_TRY(node_forward(m->dm, d_states, d_times, d_dy, nb, nt, nc, st->tol_a, st->tol_r, st->max_iter,
                            c->scratch.as<double>(), c->r0.as<double>(), c->rn.as<double>(), c->status.as<unsigned>(),
                            c->pin.as<unsigned>(0), c->key.as<unsigned long long>(), c->grp, c->gs.as<GridSync>(),
                            c->iters_host.data(), info, c->stream));
      c->mark(1);
      CUDA_TRY(cudaMemcpyAsync(c->pin.as<unsigned long long>(16), c->key.p, sizeof key, cudaMemcpyDeviceToHost,
                               c->stream));
      CUDA_TRY(cudaStreamSynchronize(c->stream));
      key = *c->pin.as<unsigned long long>(16);
    } else {  // the Newton loop on the device: one graph launch for the whole integration
      CUDA_TRY(c->iters.ensure(sizeof(int) * (16 + (size_t)n_chunks)));
      CUDA_TRY(c->pin.ensure(64 + sizeof(int) * (16 + (size_t)n_chunks)));
      c->mark(0);
      CUDA_TRY(node_forward_graph(m->dm, d_states, d_times, d_dy, nb, nt, nc, st->tol_a, st->tol_r, st->max_iter,
                                  c->scratch.as<double>(), c->r0.as<double>(), c->rn.as<double>(),
                                  c->status.as<unsigned>(), c->key.as<unsigned long long>(), c->grp,
                                  c->gs.as<GridSync>(), c->iters.as<int>(), c->stream));
      c->mark(1);
      CUDA_TRY(cudaMemcpyAsync(c->pin.as<unsigned long long>(16), c->key.p, sizeof key, cudaMemcpyDeviceToHost,
                               c->stream));
      CUDA_TRY(cudaMemcpyAsync(c->pin.as<int>(64), c->iters.p, sizeof(int) * (16 + (size_t)n_chunks),
                               cudaMemcpyDeviceToHost, c->stream));
      CUDA_TRY(cudaStreamSynchronize(c->stream));
      key = *c->pin.as<unsigned long long>(16);
      const int* ctl = c->pin.as<int>(64);
      info[0] = ctl[2];
      info[1] = ctl[5];
      info[2] = ctl[6];
      info[3] = ctl[4];
      c->iters_host.assign(ctl + 16, ctl + 16 + n_chunks);
    }
    c->last_launches = 1 + 6 * (int)n_chunks;
    c->last_gen = 2;
  } else {
  c->last_sp = 0;
  a.structured = v2 && c->structured;
  for (int attempt = 0;; ++attempt) {
    if (attempt > 0) {  // the structured kernels met a block they cannot factor: the group-LU kernels re-run it
      CUDA_TRY(cudaMemsetAsync(c->gs.p, 0, offsetof(GridSync, ext_gen), c->stream));
      CUDA_TRY(cudaMemsetAsync(c->key.p, 0xff, sizeof(unsigned long long), c->stream));
      CUDA_TRY(cudaMemsetAsync(c->info.p, 0, sizeof(int) * 4, c->stream));
      a.structured = 0;
      c->last_sp |= CKO_SP_FWD_FALLBACK;
    }
    c->mark(0);
    if (v2)
      CUDA_TRY(launch_forward_v2(m->dm.kind, n, &a, c->stream));
    else if (p2)
      CUDA_TRY(launch_forward_pcr2(m->dm.kind, n, &a, c->stream));
    else
      CUDA_TRY(launch_forward(a, c->stream));
    c->mark(1);
    c->last_launches = attempt + 1;
    c->last_gen = (v2 || p2) ? 2 : 1;
    CUDA_TRY(c->pin.ensure(32 + sizeof(int) * (size_t)n_chunks));
    CUDA_TRY(cudaMemcpyAsync(c->pin.as<int>(0), c->info.p, sizeof info, cudaMemcpyDeviceToHost, c->stream));
    CUDA_TRY(cudaMemcpyAsync(c->pin.as<unsigned long long>(16), c->key.p, sizeof key, cudaMemcpyDeviceToHost,
                             c->stream));
    CUDA_TRY(cudaMemcpyAsync(c->pin.as<int>(32), c->iters.p, sizeof(int) * n_chunks, cudaMemcpyDeviceToHost,
                             c->stream));
    CUDA_TRY(cudaStreamSynchronize(c->stream));
    std::memcpy(info, c->pin.as<int>(0), sizeof info);
    key = *c->pin.as<unsigned long long>(16);
    c->iters_host.assign(c->pin.as<int>(32), c->pin.as<int>(32) + n_chunks);
    if (!(info[0] == 5 && a.structured)) break;
  }
  if (a.structured) c->last_sp |= CKO_SP_FWD;
  }
  if (a.trace) {
    std::vector<unsigned long long> h(tbuf.bytes / sizeof(unsigned long long));
    CUDA_TRY(cudaMemcpy(h.data(), tbuf.p, tbuf.bytes, cudaMemcpyDeviceToHost));
    if (FILE* fp = std::fopen(trace_path, "wb")) {
      std::fwrite(h.data(), sizeof(unsigned long long), h.size(), fp);
      std::fclose(fp);
    }
    tbuf.release();
  }
  c->last_ms[1] = c->last_ms[2] = c->last_ms[3] = 0.0;
  c->collect(0, 1);
  const int off = m->desc.lane_offset;
  if (info[0] == 4) return fail(err, CKO_COMM, "grid barrier timed out (device or peer stalled)");
  if (info[0] == 1 && key == ~0ull) {  // FLAG_SINGULAR came from a peer rank through the group exchange
    cko_status s = fail(err, CKO_SINGULAR_BLOCK, "singular diagonal block on a peer rank of the batch group");
    if (err) err->chunk_index = -1, err->batch_index = -1;
    return s;
  }
  if (info[0] == 1) {
    const int k = (int)(key / (unsigned long long)nb), b = (int)(key % (unsigned long long)nb);
    cko_status s = fail(err, CKO_SINGULAR_BLOCK, "singular diagonal block at chunk row %d, batch %d", k, b + off);
    if (err) err->chunk_index = k, err->batch_index = b + off;
    return s;
  }
  if (info[0] == 2) {
    std::vector<double> rn(nb), r0(nb);
    CUDA_TRY(cudaMemcpy(rn.data(), c->rn.p, sizeof(double) * nb, cudaMemcpyDeviceToHost));
    CUDA_TRY(cudaMemcpy(r0.data(), c->r0.p, sizeof(double) * nb, cudaMemcpyDeviceToHost));
    int w = 0;  // worst_lane (integrate.cpp:167-174)
    for (int b = 0; b < nb; ++b) {
      if (!std::isfinite(rn[b])) {
        w = b;
        break;
      }
      if (rn[b] > rn[w]) w = b;
    }
    cko_status s = fail(err, CKO_NEWTON_DIVERGENCE,
                        "Newton did not converge for chunk starting at step %d (batch %d): |r| = %g after %d "
                        "iterations, |r0| = %g",
                        info[1], w + off, rn[w], info[2], r0[w]);
    if (err) {
      err->chunk_start_step = info[1];
      err->batch_index = w + off;
      err->iterations = info[2];
      err->residual_norm = rn[w];
      err->initial_norm = r0[w];
    }
    return s;
  }
  if (info[3] != n_chunks) return fail(err, CKO_CUDA, "forward kernel stopped after %d of %d chunks", info[3], n_chunks);
  if (a.loss_part) c->lpart_n = G;
  if (work) {
    std::memset(work, 0, sizeof(*work));
    for (int j = 0; j < n_chunks; ++j) {
      const int cj = (j == n_chunks - 1) ? nt - j * nc : nc;
      const int it = c->iters_host[j];
      work->newton_iterations += it;
      work->rate_evals += it + 1;
      work->jacobian_evals += it;
      work->linear_solves += it;
      work->reduction_sweeps += (long long)it * sweeps_of(cj, sv->kind, sv->n_switch);
    }
  }
  if (iters_out) *iters_out = c->iters_host.empty() ? 0 : c->iters_host[0];
  return ok(err);
}

// Core adjoint on device buffers.
cko_status adjoint_core(cko_ctx* c, const cko_model* m, const double* d_states, const double* d_times, int nb,
                        int nt, int nc, const cko_solver_choice* sv, int loss_kind, const double* d_dL,
                        double* loss_out, double* grad_out, cko_work* bwd, cko_error* err,
                        bool keep_lambda = false, bool fwd_loss = false) {
  if (m) const_cast<cko_model*>(m)->dm.jstrat = c->jstrat;  // the call's JacobianStrategy
  if (nc < 1) return fail(err, CKO_SHAPE_MISMATCH, "adjoint: n_chunk must be >= 1");
  if (sv->kind < 0 || sv->kind > 2) return fail(err, CKO_ERROR, "unknown solver kind %d", sv->kind);
  if (sv->kind == CKO_SOLVER_HYBRID && sv->n_switch < 0)
    return fail(err, CKO_ERROR, "solve_hybrid: n_switch must be >= 0");
  if (loss_kind == CKO_LOSS_USER && !d_dL) return fail(err, CKO_ERROR, "user loss needs dL");
  if (cko_status s = check_lanes(m, nb, err)) return s;
  const int n = m->dm.n, np = m->dm.np;
  const int nc_eff = nc < nt ? nc : nt;
  const bool pcr = sv->kind != CKO_SOLVER_THOMAS;
  // a carried-in lambda (single-chunk op) or a non-analytic Jacobian strategy: generic kernels
  const int gen = (keep_lambda || c->jstrat != 0) ? 1 : c->kernel_gen;
  const bool nodep = !pcr && gen >= 2 && node_fast_path(m->dm);
  const bool v2 = !nodep && !pcr && gen >= 2 && launch_adjoint_v2(m->dm.kind, n, nullptr, c->stream) == cudaSuccess;
  const bool p2 = pcr && gen >= 2 && launch_adjoint_pcr2(m->dm.kind, n, nullptr, c->stream) == cudaSuccess;
  const int G = (v2 || p2) ? (nb < c->sms ? nb : c->sms) : (nb < 2 * c->sms ? nb : 2 * c->sms);
  Slab slab{};
  if (nodep) {
    CUDA_TRY(c->slab.ensure(sizeof(double) * node_scratch_doubles(nb, nc_eff)));
  } else if (p2) {
    slab.Lmax = (nb + G - 1) / G;
    slab.Pmax = nc_eff * slab.Lmax;
    slab.doubles = (size_t)slab.Pmax * pcr2_ws_bound(n);
    CUDA_TRY(c->slab.ensure(sizeof(double) * slab.doubles * G));
    slab.base = c->slab.as<double>();
  } else if (!v2) {
    if (cko_status s = prepare_slab(c, G, nb, nc_eff, n, pcr, slab, err)) return s;
  }
  const size_t row = (size_t)nb * n;
  CUDA_TRY(c->lambda.ensure(sizeof(double) * row));
  CUDA_TRY(c->wq.ensure(sizeof(double) * row * (nt + 1)));
  CUDA_TRY(c->key.ensure(sizeof(unsigned long long)));
  CUDA_TRY(c->loss.ensure(sizeof(double)));
  CUDA_TRY(c->scratch.ensure(sizeof(double) * 1040));
  CUDA_TRY(c->status.ensure(sizeof(unsigned)));
  CUDA_TRY(cudaMemsetAsync(c->status.p, 0, sizeof(unsigned), c->stream));
  if (c->grp.world > 1 && np > c->grp.red_cap)
    return fail(err, CKO_COMM, "parameter count %d exceeds the group reduce buffer (%d)", np, c->grp.red_cap);
  CUDA_TRY(c->vjp.ensure(sizeof(double) * vjp_scratch_doubles(m->dm, nb, nt)));
  CUDA_TRY(c->grad.ensure(sizeof(double) * (np + 1)));  // + the group's singular-block flag
  CUDA_TRY(cudaMemsetAsync(c->key.p, 0xff, sizeof(unsigned long long), c->stream));
  c->last_launches = 3;
  c->last_gen = (nodep || v2 || p2) ? 2 : 1;
  c->mark(6);
  // Frobenius loss: straight after this call's own forward, from the per-CTA partials the forward left
  // (formed inside the generation-2 adjoint on one rank, else one small kernel that also sums the group);
  // otherwise a pass over the trajectory
  const int lpart_n = c->lpart_n;
  const bool lpart = fwd_loss && lpart_n > 0 && loss_kind == CKO_LOSS_FROBENIUS;
  const bool lpart_in_adj = lpart && (v2 || p2) && c->grp.world <= 1;
  if (lpart && !lpart_in_adj) {
    CUDA_TRY(launch_loss_final(c->lpart.as<double>(), lpart_n, c->scratch.as<double>(), c->loss.as<double>(),
                               c->grp, c->gs.as<GridSync>(), c->status.as<unsigned>(), c->stream));
    c->last_launches += 1;
  } else if (!lpart && loss_kind == CKO_LOSS_FROBENIUS) {
    CUDA_TRY(launch_loss(d_states, nt, (int)row, c->scratch.as<double>(), c->loss.as<double>(), c->grp,
                         c->gs.as<GridSync>(), c->status.as<unsigned>(), c->stream));
    c->last_launches += 2;
  }
  c->lpart_n = 0;
  c->mark(7);
  AdjLaunch a{};
  a.m = m->dm;
  a.states = d_states;
  a.times = d_times;
  a.dL = loss_kind == CKO_LOSS_USER ? d_dL : nullptr;
  a.loss = loss_kind == CKO_LOSS_USER ? nullptr : c->loss.as<double>();
  if (lpart_in_adj) {
    a.loss_part = c->lpart.as<double>();
    a.loss_nparts = lpart_n;
    a.loss_out = c->loss.as<double>();
  }
  a.nb = nb;
  a.nt = nt;
  a.nc = nc;
  a.solver = sv->kind;
  a.n_switch = sv->n_switch;
  a.slab = slab;
  a.lambda = c->lambda.as<double>();
  a.keep_lambda = keep_lambda ? 1 : 0;
  a.wq = c->wq.as<double>();
  a.sing_key = c->key.as<unsigned long long>();
  a.grid = G;
  a.threads = kThreads;
  c->last_sp &= CKO_SP_FWD | CKO_SP_FWD_FALLBACK;  // keep the forward's bits of a gradient_adjoint call
  if (v2 && c->structured) {
    CUDA_TRY(c->spfb.ensure(sizeof(unsigned)));
    CUDA_TRY(cudaMemsetAsync(c->spfb.p, 0, sizeof(unsigned), c->stream));
    a.structured = 1;
    a.sp_fallback = c->spfb.as<unsigned>();
  }
  c->mark(2);
  if (nodep)
    CUDA_TRY(node_adjoint(m->dm, d_states, d_times, a.dL, a.loss, nb, nt, nc, c->slab.as<double>(),
                          c->lambda.as<double>(), c->wq.as<double>(), c->key.as<unsigned long long>(), c->stream));
  else if (v2)
    CUDA_TRY(launch_adjoint_v2(m->dm.kind, n, &a, c->stream));
  else if (p2)
    CUDA_TRY(launch_adjoint_pcr2(m->dm.kind, n, &a, c->stream));
  else
    CUDA_TRY(launch_adjoint(a, c->stream));
  c->mark(3);
  c->mark(4);
  CUDA_TRY(launch_vjp(m->dm, d_states, d_times, c->wq.as<double>(), nb, nt, c->vjp.as<double>(),
                      c->grad.as<double>(), c->stream));
  // structured adjoint: a block it cannot factor makes this rank re-run the adjoint and the VJP on the
  // group-LU kernels before anything is exchanged or read
  auto adjoint_fallback = [&]() -> cudaError_t {
    unsigned fb = 0;
    cudaError_t e = cudaMemcpyAsync(c->pin.as<unsigned>(0), c->spfb.p, sizeof fb, cudaMemcpyDeviceToHost, c->stream);
    if (e == cudaSuccess) e = cudaStreamSynchronize(c->stream);
    if (e != cudaSuccess) return e;
    fb = *c->pin.as<unsigned>(0);
    if (!fb) return cudaSuccess;
    a.structured = 0;
    c->last_sp |= CKO_SP_ADJ_FALLBACK;
    CUDA_TRY_RAW(cudaMemsetAsync(c->key.p, 0xff, sizeof(unsigned long long), c->stream));
    CUDA_TRY_RAW(launch_adjoint_v2(m->dm.kind, n, &a, c->stream));
    CUDA_TRY_RAW(launch_vjp(m->dm, d_states, d_times, c->wq.as<double>(), nb, nt, c->vjp.as<double>(),
                            c->grad.as<double>(), c->stream));
    c->last_launches += 2;
    return cudaSuccess;
  };
  if (a.structured) {
    CUDA_TRY(c->pin.ensure(32 + sizeof(double) * (size_t)(np + 1)));
    CUDA_TRY(adjoint_fallback());
    if (a.structured) c->last_sp |= CKO_SP_ADJ;
  }
  if (c->grp.world > 1) {
    CUDA_TRY(launch_key_flag(c->key.as<unsigned long long>(), c->grad.as<double>() + np, c->stream));
    CUDA_TRY(launch_group_sum(c->grp, c->gs.as<GridSync>(), c->grad.as<double>(), np + 1, c->status.as<unsigned>(),
                              c->stream));
    c->last_launches += 2;
  }
  c->mark(5);
  unsigned long long key;
  unsigned gstatus = 0;
  double L = NAN;
  CUDA_TRY(c->pin.ensure(32 + sizeof(double) * (size_t)(np + 1)));
  CUDA_TRY(cudaMemcpyAsync(c->pin.as<unsigned>(0), c->status.p, sizeof gstatus, cudaMemcpyDeviceToHost, c->stream));
  CUDA_TRY(cudaMemcpyAsync(c->pin.as<unsigned long long>(8), c->key.p, sizeof key, cudaMemcpyDeviceToHost,
                           c->stream));
  if (loss_kind == CKO_LOSS_FROBENIUS)
    CUDA_TRY(cudaMemcpyAsync(c->pin.as<double>(16), c->loss.p, sizeof L, cudaMemcpyDeviceToHost, c->stream));
  CUDA_TRY(cudaMemcpyAsync(c->pin.as<double>(32), c->grad.p, sizeof(double) * (np + 1), cudaMemcpyDeviceToHost,
                           c->stream));
  CUDA_TRY(cudaStreamSynchronize(c->stream));
  gstatus = *c->pin.as<unsigned>(0);
  key = *c->pin.as<unsigned long long>(8);
  if (loss_kind == CKO_LOSS_FROBENIUS) L = *c->pin.as<double>(16);
  std::memcpy(grad_out, c->pin.as<double>(32), sizeof(double) * np);
  const bool group_singular = c->grp.world > 1 && c->pin.as<double>(32)[np] > 0.0;
  c->last_ms[0] = 0.0;
  c->collect(1, 3);
  if (gstatus) return fail(err, CKO_COMM, "group reduction timed out (peer stalled)");
  const int off = m->desc.lane_offset;
  if (key != ~0ull) {
    const int b = (int)(key % (unsigned long long)nb);
    const int r = (int)((key / (unsigned long long)nb) % (unsigned long long)nc);
    cko_status s = fail(err, CKO_SINGULAR_BLOCK, "singular diagonal block at chunk row %d, batch %d", r, b + off);
    if (err) err->chunk_index = r, err->batch_index = b + off;
    return s;
  }
  if (group_singular) {
    cko_status s = fail(err, CKO_SINGULAR_BLOCK, "singular adjoint block on a peer rank of the batch group");
    if (err) err->chunk_index = -1, err->batch_index = -1;
    return s;
  }
  for (int j = 0; j < np; ++j)
    if (!std::isfinite(grad_out[j]))
      return fail(err, CKO_NON_FINITE, "parameter product of the model is not finite");
  if (loss_out) *loss_out = L;
  if (bwd) {
    std::memset(bwd, 0, sizeof(*bwd));
    for (int step_hi = nt; step_hi >= 1;) {
      const int cc = nc < step_hi ? nc : step_hi;
      bwd->jacobian_evals += 1;
      bwd->linear_solves += 1;
      bwd->reduction_sweeps += sweeps_of(cc, sv->kind, sv->n_switch);
      step_hi -= cc;
    }
  }
  return ok(err);
}

// ---- forward Euler scheme (integrate.cpp:371-407, adjoint.cpp:157-188) ----------------------------
cko_status fe_forward_core(cko_ctx* c, const cko_model* m, double* d_states, const double* d_times, int nb, int nt,
                           int nc, cko_work* work, cko_error* err) {
  if (m) const_cast<cko_model*>(m)->dm.jstrat = c->jstrat;  // the call's JacobianStrategy
  if (nc < 1) return fail(err, CKO_SHAPE_MISMATCH, "integrate: n_chunk must be >= 1");
  if (nt < 1) return fail(err, CKO_SHAPE_MISMATCH, "integrate: need at least one step");
  if (cko_status s = check_lanes(m, nb, err)) return s;
  CUDA_TRY(c->scratch.ensure(sizeof(double) * (size_t)nb * m->dm.n));
  CUDA_TRY(c->info.ensure(sizeof(int) * 4));
  CUDA_TRY(c->pin.ensure(64));
  CUDA_TRY(cudaMemsetAsync(c->info.p, 0x7f, sizeof(int), c->stream));
  c->mark(0);
  CUDA_TRY(launch_fe_forward(m->dm, d_states, d_times, nb, nt, c->scratch.as<double>(), c->info.as<int>(), c->stream));
  c->mark(1);
  CUDA_TRY(cudaMemcpyAsync(c->pin.p, c->info.p, sizeof(int), cudaMemcpyDeviceToHost, c->stream));
  CUDA_TRY(cudaStreamSynchronize(c->stream));
  c->last_launches = 1;
  c->last_gen = 1;
  c->last_ms[1] = c->last_ms[2] = c->last_ms[3] = 0.0;
  c->collect(0, 1);
  const int bad = *c->pin.as<int>(0);
  if (bad != 0x7f7f7f7f)
    return fail(err, CKO_NON_FINITE, "forward Euler produced a non-finite state at step %d", bad);
  if (work) {
    std::memset(work, 0, sizeof(*work));
    work->rate_evals = nt;  // one batched rate call per step
  }
  return ok(err);
}

cko_status fe_adjoint_core(cko_ctx* c, const cko_model* m, const double* d_states, const double* d_times, int nb,
                           int nt, int nc, int loss_kind, const double* d_dL, double* loss_out, double* grad_out,
                           cko_work* bwd, cko_error* err) {
  if (m) const_cast<cko_model*>(m)->dm.jstrat = c->jstrat;  // the call's JacobianStrategy
  if (nc < 1) return fail(err, CKO_SHAPE_MISMATCH, "adjoint: n_chunk must be >= 1");
  if (loss_kind == CKO_LOSS_USER && !d_dL) return fail(err, CKO_ERROR, "user loss needs dL");
  if (cko_status s = check_lanes(m, nb, err)) return s;
  const int n = m->dm.n, np = m->dm.np;
  const size_t row = (size_t)nb * n;
  CUDA_TRY(c->lambda.ensure(sizeof(double) * row));
  CUDA_TRY(c->wq.ensure(sizeof(double) * row * (nt + 1)));
  CUDA_TRY(c->slab.ensure(sizeof(double) * (row * n + row)));
  CUDA_TRY(c->key.ensure(sizeof(unsigned long long)));
  CUDA_TRY(c->loss.ensure(sizeof(double)));
  CUDA_TRY(c->scratch.ensure(sizeof(double) * 1040));
  CUDA_TRY(c->status.ensure(2 * sizeof(unsigned)));
  CUDA_TRY(c->vjp.ensure(sizeof(double) * vjp_scratch_doubles(m->dm, nb, nt)));
  CUDA_TRY(c->grad.ensure(sizeof(double) * (np + 1)));
  if (c->grp.world > 1 && np + 1 > c->grp.red_cap)
    return fail(err, CKO_COMM, "parameter count %d exceeds the group reduce buffer (%d)", np, c->grp.red_cap);
  CUDA_TRY(cudaMemsetAsync(c->status.p, 0, 2 * sizeof(unsigned), c->stream));
  CUDA_TRY(cudaMemsetAsync(c->key.p, 0xff, sizeof(unsigned long long), c->stream));
  c->last_launches = 3;
  c->last_gen = 1;
  c->mark(6);
  if (loss_kind == CKO_LOSS_FROBENIUS) {
    CUDA_TRY(launch_loss(d_states, nt, (int)row, c->scratch.as<double>(), c->loss.as<double>(), c->grp,
                         c->gs.as<GridSync>(), c->status.as<unsigned>(), c->stream));
    c->last_launches += 2;
  }
  c->mark(7);
  c->mark(2);
  double* Jb = c->slab.as<double>();
  CUDA_TRY(launch_fe_adjoint(m->dm, d_states, d_times, loss_kind == CKO_LOSS_USER ? d_dL : nullptr,
                             loss_kind == CKO_LOSS_USER ? nullptr : c->loss.as<double>(), nb, nt, c->lambda.as<double>(),
                             Jb, Jb + row * n, c->wq.as<double>(), c->status.as<unsigned>() + 1, c->stream));
  c->mark(3);
  c->mark(4);
  // the quadrature of step m sits at the step START (y_{m-1}, t_{m-1}): the VJP kernels read row-shifted views
  const double* st_prev = reinterpret_cast<const double*>(reinterpret_cast<uintptr_t>(d_states) - sizeof(double) * row);
  const double* t_prev = reinterpret_cast<const double*>(reinterpret_cast<uintptr_t>(d_times) - sizeof(double) * nb);
  CUDA_TRY(launch_vjp(m->dm, st_prev, t_prev, c->wq.as<double>(), nb, nt, c->vjp.as<double>(), c->grad.as<double>(),
                      c->stream));
  if (c->grp.world > 1) {
    CUDA_TRY(launch_group_sum(c->grp, c->gs.as<GridSync>(), c->grad.as<double>(), np, c->status.as<unsigned>(),
                              c->stream));
    c->last_launches += 1;
  }
  c->mark(5);
  CUDA_TRY(c->pin.ensure(32 + sizeof(double) * (size_t)(np + 1)));
  CUDA_TRY(cudaMemcpyAsync(c->pin.as<unsigned>(0), c->status.p, 2 * sizeof(unsigned), cudaMemcpyDeviceToHost,
                           c->stream));
  if (loss_kind == CKO_LOSS_FROBENIUS)
    CUDA_TRY(cudaMemcpyAsync(c->pin.as<double>(16), c->loss.p, sizeof(double), cudaMemcpyDeviceToHost, c->stream));
  CUDA_TRY(cudaMemcpyAsync(c->pin.as<double>(32), c->grad.p, sizeof(double) * np, cudaMemcpyDeviceToHost, c->stream));
  CUDA_TRY(cudaStreamSynchronize(c->stream));
  const unsigned gstatus = c->pin.as<unsigned>(0)[0], jbad = c->pin.as<unsigned>(0)[1];
  const double L = loss_kind == CKO_LOSS_FROBENIUS ? *c->pin.as<double>(16) : NAN;
  std::memcpy(grad_out, c->pin.as<double>(32), sizeof(double) * np);
  c->last_ms[0] = 0.0;
  c->collect(1, 3);
  if (gstatus) return fail(err, CKO_COMM, "group reduction timed out (peer stalled)");
  if (jbad) return fail(err, CKO_NON_FINITE, "Jacobian of the model is not finite");
  for (int j = 0; j < np; ++j)
    if (!std::isfinite(grad_out[j])) return fail(err, CKO_NON_FINITE, "parameter product of the model is not finite");
  if (loss_out) *loss_out = L;
  if (bwd) {
    std::memset(bwd, 0, sizeof(*bwd));
    for (int step_hi = nt; step_hi >= 1; step_hi -= (nc < step_hi ? nc : step_hi)) bwd->jacobian_evals += 1;
  }
  return ok(err);
}

}  // namespace

extern "C" {

cko_status cko_fe_forward(cko_ctx* c, const cko_model* m, const double* y0, const double* times, int nb, int nt,
                          int nc, double* states_out, cko_work* work, cko_error* err) {
  if (!c || !m || !y0 || !times || !states_out) return fail(err, CKO_ERROR, "null argument");
  if (cko_status s = check_grid_shape(nt, nb, err)) return s;
  CUDA_TRY(cudaSetDevice(c->device));
  const size_t row = (size_t)nb * m->dm.n;
  CUDA_TRY(c->h_states.ensure(sizeof(double) * row * (nt + 1)));
  CUDA_TRY(c->h_times.ensure(sizeof(double) * (size_t)nb * (nt + 1)));
  double* d_states = c->h_states.as<double>();
  double* d_times = c->h_times.as<double>();
  CUDA_TRY(cudaMemcpyAsync(d_times, times, sizeof(double) * (size_t)nb * (nt + 1), cudaMemcpyHostToDevice, c->stream));
  CUDA_TRY(cudaMemcpyAsync(d_states, y0, sizeof(double) * row, cudaMemcpyHostToDevice, c->stream));
  if (cko_status s = check_grid_device(c, d_times, nt, nb, err)) return s;
  if (cko_status s = fe_forward_core(c, m, d_states, d_times, nb, nt, nc, work, err)) return s;
  CUDA_TRY(cudaMemcpyAsync(states_out, d_states, sizeof(double) * row * (nt + 1), cudaMemcpyDeviceToHost, c->stream));
  CUDA_TRY(cudaStreamSynchronize(c->stream));
  return ok(err);
}

cko_status cko_fe_adjoint_host(cko_ctx* c, const cko_model* m, const double* states, const double* times, int nb,
                               int nt, int nc, int loss_kind, const double* dL_host, double* loss_out,
                               double* grad_out, cko_work* bwd, cko_error* err) {
  if (!c || !m || !states || !times || !grad_out) return fail(err, CKO_ERROR, "null argument");
  if (cko_status s = check_grid_shape(nt, nb, err)) return s;
  CUDA_TRY(cudaSetDevice(c->device));
  const size_t row = (size_t)nb * m->dm.n;
  CUDA_TRY(c->h_states.ensure(sizeof(double) * row * (nt + 1)));
  CUDA_TRY(c->h_times.ensure(sizeof(double) * (size_t)nb * (nt + 1)));
  CUDA_TRY(cudaMemcpyAsync(c->h_states.p, states, sizeof(double) * row * (nt + 1), cudaMemcpyHostToDevice, c->stream));
  CUDA_TRY(cudaMemcpyAsync(c->h_times.p, times, sizeof(double) * (size_t)nb * (nt + 1), cudaMemcpyHostToDevice,
                           c->stream));
  const double* d_dL = nullptr;
  if (loss_kind == CKO_LOSS_USER) {
    if (!dL_host) return fail(err, CKO_ERROR, "user loss needs dL");
    CUDA_TRY(c->h_dL.ensure(sizeof(double) * row * (nt + 1)));
    CUDA_TRY(cudaMemcpyAsync(c->h_dL.p, dL_host, sizeof(double) * row * (nt + 1), cudaMemcpyHostToDevice, c->stream));
    d_dL = c->h_dL.as<double>();
  }
  return fe_adjoint_core(c, m, c->h_states.as<double>(), c->h_times.as<double>(), nb, nt, nc, loss_kind, d_dL,
                         loss_out, grad_out, bwd, err);
}

cko_status cko_be_forward_device(cko_ctx* c, const cko_model* m, const double* d_y0, const double* d_times, int nb,
                                 int nt, int nc, const cko_newton_settings* st, const cko_solver_choice* sv,
                                 double* d_states, cko_work* work, cko_error* err) {
  if (!c || !m || !d_y0 || !d_times || !d_states || !st || !sv) return fail(err, CKO_ERROR, "null argument");
  if (nb < 1) return fail(err, CKO_SHAPE_MISMATCH, "integrate: y0 rows != grid batch width");
  CUDA_TRY(cudaSetDevice(c->device));
  const size_t row = (size_t)nb * m->dm.n;
  if (d_states != d_y0)
    CUDA_TRY(cudaMemcpyAsync(d_states, d_y0, sizeof(double) * row, cudaMemcpyDeviceToDevice, c->stream));
  return forward_core(c, m, d_states, d_times, nb, nt, nc, st, sv, nullptr, work, nullptr, err);
}

cko_status cko_gradient_adjoint_device(cko_ctx* c, const cko_model* m, const double* d_y0, const double* d_times,
                                       int nb, int nt, int nc, const cko_newton_settings* st,
                                       const cko_solver_choice* sv, double* d_states, double* loss_out,
                                       double* grad_out, cko_work* fwd, cko_work* bwd, cko_error* err) {
  if (!c || !m || !d_y0 || !d_times || !d_states || !st || !sv || !grad_out) return fail(err, CKO_ERROR, "null argument");
  if (nb < 1) return fail(err, CKO_SHAPE_MISMATCH, "integrate: y0 rows != grid batch width");
  CUDA_TRY(cudaSetDevice(c->device));
  const size_t row = (size_t)nb * m->dm.n;
  if (d_states != d_y0)
    CUDA_TRY(cudaMemcpyAsync(d_states, d_y0, sizeof(double) * row, cudaMemcpyDeviceToDevice, c->stream));
  if (cko_status s = forward_core(c, m, d_states, d_times, nb, nt, nc, st, sv, nullptr, fwd, nullptr, err, nullptr,
                                  true))
    return s;
  const int fwd_launches = c->last_launches;
  const double fwd_ms = c->last_ms[0];
  cko_status s = adjoint_core(c, m, d_states, d_times, nb, nt, nc, sv, CKO_LOSS_FROBENIUS, nullptr, loss_out,
                              grad_out, bwd, err, false, true);
  c->last_launches += fwd_launches;  // the step's launches and kernel times, forward included
  c->last_ms[0] = fwd_ms;
  return s;
}

cko_status cko_be_forward(cko_ctx* c, const cko_model* m, const double* y0, const double* times, int nb, int nt,
                          int nc, const cko_newton_settings* st, const cko_solver_choice* sv, double* states_out,
                          cko_traj** traj_out, cko_work* work, cko_error* err) {
  if (!c || !m || !y0 || !times || !st || !sv) return fail(err, CKO_ERROR, "null argument");
  if (traj_out) *traj_out = nullptr;
  if (cko_status s = check_grid_shape(nt, nb, err)) return s;
  CUDA_TRY(cudaSetDevice(c->device));
  const int n = m->dm.n;
  const size_t row = (size_t)nb * n;
  cko_traj* t = nullptr;
  double *d_states, *d_times;
  if (traj_out) {
    t = new (std::nothrow) cko_traj();
    if (!t) return fail(err, CKO_ERROR, "out of host memory");
    t->ctx = c;
    t->nb = nb;
    t->nt = nt;
    t->n = n;
    cudaError_t e = cudaMalloc(&t->d_states, sizeof(double) * row * (nt + 1));
    if (e == cudaSuccess) e = cudaMalloc(&t->d_times, sizeof(double) * (size_t)nb * (nt + 1));
    if (e != cudaSuccess) {
      cudaFree(t->d_states);
      cudaFree(t->d_times);
      delete t;
      return fail(err, CKO_CUDA, "trajectory allocation: %s", cudaGetErrorString(e));
    }
    d_states = t->d_states;
    d_times = t->d_times;
  } else {
    CUDA_TRY(c->h_states.ensure(sizeof(double) * row * (nt + 1)));
    CUDA_TRY(c->h_times.ensure(sizeof(double) * (size_t)nb * (nt + 1)));
    d_states = c->h_states.as<double>();
    d_times = c->h_times.as<double>();
  }
  auto cleanup = [&](cko_status s) {
    if (s != CKO_OK && t) {
      cudaFree(t->d_states);
      cudaFree(t->d_times);
      delete t;
      t = nullptr;
    }
    return s;
  };
  cudaError_t e = cudaMemcpyAsync(d_times, times, sizeof(double) * (size_t)nb * (nt + 1), cudaMemcpyHostToDevice,
                                  c->stream);
  if (e == cudaSuccess) e = cudaMemcpyAsync(d_states, y0, sizeof(double) * row, cudaMemcpyHostToDevice, c->stream);
  if (e != cudaSuccess) return cleanup(fail(err, CKO_CUDA, "H2D: %s", cudaGetErrorString(e)));
  if (cko_status s = check_grid_device(c, d_times, nt, nb, err)) return cleanup(s);
  cko_status s = forward_core(c, m, d_states, d_times, nb, nt, nc, st, sv, nullptr, work, nullptr, err);
  if (s != CKO_OK) return cleanup(s);
  if (states_out) {
    e = cudaMemcpyAsync(states_out, d_states, sizeof(double) * row * (nt + 1), cudaMemcpyDeviceToHost, c->stream);
    if (e == cudaSuccess) e = cudaStreamSynchronize(c->stream);
    if (e != cudaSuccess) return cleanup(fail(err, CKO_CUDA, "D2H: %s", cudaGetErrorString(e)));
  }
  if (traj_out) *traj_out = t;
  return ok(err);
}

cko_status cko_be_adjoint_device(cko_ctx* c, const cko_model* m, const double* d_states, const double* d_times,
                                 int nb, int nt, int nc, const cko_solver_choice* sv, int loss_kind,
                                 const double* d_dL, double* loss_out, double* grad_out, cko_work* bwd,
                                 cko_error* err) {
  if (!c || !m || !d_states || !d_times || !sv || !grad_out) return fail(err, CKO_ERROR, "null argument");
  if (nt < 1 || nb < 1) return fail(err, CKO_SHAPE_MISMATCH, "adjoint: empty trajectory");
  CUDA_TRY(cudaSetDevice(c->device));
  return adjoint_core(c, m, d_states, d_times, nb, nt, nc, sv, loss_kind, d_dL, loss_out, grad_out, bwd, err);
}

cko_status cko_be_adjoint(cko_ctx* c, const cko_model* m, const cko_traj* t, int nc, const cko_solver_choice* sv,
                          int loss_kind, const double* dL_host, double* loss_out, double* grad_out, cko_work* bwd,
                          cko_error* err) {
  if (!c || !m || !t || !sv || !grad_out) return fail(err, CKO_ERROR, "null argument");
  if (t->n != m->dm.n) return fail(err, CKO_SHAPE_MISMATCH, "adjoint: trajectory width != model size");
  CUDA_TRY(cudaSetDevice(c->device));
  const double* d_dL = nullptr;
  if (loss_kind == CKO_LOSS_USER) {
    if (!dL_host) return fail(err, CKO_ERROR, "user loss needs dL");
    const size_t bytes = sizeof(double) * (size_t)t->nb * t->n * (t->nt + 1);
    CUDA_TRY(c->h_dL.ensure(bytes));
    CUDA_TRY(cudaMemcpyAsync(c->h_dL.p, dL_host, bytes, cudaMemcpyHostToDevice, c->stream));
    d_dL = c->h_dL.as<double>();
  }
  return adjoint_core(c, m, t->d_states, t->d_times, t->nb, t->nt, nc, sv, loss_kind, d_dL, loss_out, grad_out,
                      bwd, err);
}

cko_status cko_be_adjoint_host(cko_ctx* c, const cko_model* m, const double* states, const double* times, int nb,
                               int nt, int nc, const cko_solver_choice* sv, int loss_kind, const double* dL_host,
                               double* loss_out, double* grad_out, cko_work* bwd, cko_error* err) {
  if (!c || !m || !states || !times || !sv || !grad_out) return fail(err, CKO_ERROR, "null argument");
  if (cko_status s = check_grid_shape(nt, nb, err)) return s;
  CUDA_TRY(cudaSetDevice(c->device));
  const size_t row = (size_t)nb * m->dm.n;
  CUDA_TRY(c->h_states.ensure(sizeof(double) * row * (nt + 1)));
  CUDA_TRY(c->h_times.ensure(sizeof(double) * (size_t)nb * (nt + 1)));
  CUDA_TRY(cudaMemcpyAsync(c->h_states.p, states, sizeof(double) * row * (nt + 1), cudaMemcpyHostToDevice, c->stream));
  CUDA_TRY(cudaMemcpyAsync(c->h_times.p, times, sizeof(double) * (size_t)nb * (nt + 1), cudaMemcpyHostToDevice,
                           c->stream));
  if (cko_status s = check_grid_device(c, c->h_times.as<double>(), nt, nb, err)) return s;
  const double* d_dL = nullptr;
  if (loss_kind == CKO_LOSS_USER) {
    if (!dL_host) return fail(err, CKO_ERROR, "user loss needs dL");
    CUDA_TRY(c->h_dL.ensure(sizeof(double) * row * (nt + 1)));
    CUDA_TRY(cudaMemcpyAsync(c->h_dL.p, dL_host, sizeof(double) * row * (nt + 1), cudaMemcpyHostToDevice, c->stream));
    d_dL = c->h_dL.as<double>();
  }
  return adjoint_core(c, m, c->h_states.as<double>(), c->h_times.as<double>(), nb, nt, nc, sv, loss_kind, d_dL,
                      loss_out, grad_out, bwd, err);
}

cko_status cko_gradient_adjoint(cko_ctx* c, const cko_model* m, const double* y0, const double* times, int nb,
                                int nt, int nc, const cko_newton_settings* st, const cko_solver_choice* sv,
                                double* states_out, double* loss_out, double* grad_out, cko_work* fwd, cko_work* bwd,
                                cko_error* err) {
  if (!c || !m || !y0 || !times || !st || !sv || !grad_out) return fail(err, CKO_ERROR, "null argument");
  if (cko_status s = check_grid_shape(nt, nb, err)) return s;
  CUDA_TRY(cudaSetDevice(c->device));
  const size_t row = (size_t)nb * m->dm.n;
  CUDA_TRY(c->h_states.ensure(sizeof(double) * row * (nt + 1)));
  CUDA_TRY(c->h_times.ensure(sizeof(double) * (size_t)nb * (nt + 1)));
  double* d_states = c->h_states.as<double>();
  double* d_times = c->h_times.as<double>();
  CUDA_TRY(cudaMemcpyAsync(d_states, y0, sizeof(double) * row, cudaMemcpyHostToDevice, c->stream));
  static const bool no_stream = [] {
    const char* v = std::getenv("CKO_NO_TIME_STREAM");  // A/B: upload the whole grid before the forward
    return v && v[0] == '1';
  }();
  const int nc_eff = nc < nt ? nc : nt;
  if (no_stream || nc < 1 || nt < 4 * nc_eff || !write_value64(c->device) || !fwd_streams_times(c, m, sv)) {
    CUDA_TRY(cudaMemcpyAsync(d_times, times, sizeof(double) * (size_t)nb * (nt + 1), cudaMemcpyHostToDevice,
                             c->stream));
    if (cko_status s = check_grid_device(c, d_times, nt, nb, err)) return s;
    if (cko_status s = forward_core(c, m, d_states, d_times, nb, nt, nc, st, sv, nullptr, fwd, nullptr, err,
                                    nullptr, true))
      return s;
  } else {
    // The grid streams in while the forward runs: the first chunk's rows, then pieces of several chunks, on
    // the copy stream, each followed by a stream write of the rows now resident
    // (the kernels wait per chunk, wait_times_rows). The grid check runs on the host meanwhile; a bad grid
    // discards the forward and reports the same first index as grid_check_kernel.
    if (!c->copy_stream) CUDA_TRY(cudaStreamCreateWithFlags(&c->copy_stream, cudaStreamNonBlocking));
    if (!c->times_done) CUDA_TRY(cudaEventCreateWithFlags(&c->times_done, cudaEventDisableTiming));
    if (!c->feed.p) {  // a recycled allocation may hold another context's count: start from zero
      CUDA_TRY(c->feed.ensure(sizeof(unsigned long long)));
      CUDA_TRY(cudaMemset(c->feed.p, 0, sizeof(unsigned long long)));
      CUDA_TRY(cudaDeviceSynchronize());
    }
    // tags grow process-wide, so a stale count from any earlier call can never satisfy this call's waits
    static std::atomic<unsigned long long> feed_calls{0};
    const unsigned long long tag = (++feed_calls) << 32;
    const int ra = 16 / std::gcd(nb, 16);  // rows per 128 bytes: piece boundaries on cache-line boundaries
    auto up = [&](long long r) { return std::min<long long>(nt + 1, (r + ra - 1) / ra * ra); };
    const long long r0 = up(nc_eff + 1);
    const long long piece = std::max<long long>(up(4LL * nc_eff), (4LL << 20) / (8LL * nb) / ra * ra);
    const CUdeviceptr flag = reinterpret_cast<CUdeviceptr>(c->feed.p);
    const WriteValue64Fn wv = write_value64(c->device);
    long long bad = -1;
    std::thread checker([&] { bad = first_bad_time(times, nt, nb); });
    cudaError_t feed_err = cudaSuccess;
    std::thread feeder([&] {  // a pageable grid blocks the issuing thread, not the forward's launch
      feed_err = cudaSetDevice(c->device);
      // one stream carries every piece and its write: the resident-row count only grows
      for (long long r = 0; feed_err == cudaSuccess && r < nt + 1; r = r == 0 ? r0 : r + piece) {
        const long long e = r == 0 ? r0 : std::min<long long>(nt + 1, r + piece);
        feed_err = cudaMemcpyAsync(d_times + (size_t)r * nb, times + (size_t)r * nb, sizeof(double) * nb * (e - r),
                                   cudaMemcpyHostToDevice, c->copy_stream);
        if (feed_err == cudaSuccess &&
            wv(reinterpret_cast<CUstream>(c->copy_stream), flag, tag + e, 0) != CUDA_SUCCESS)
          feed_err = cudaErrorUnknown;
      }
      if (feed_err == cudaSuccess) feed_err = cudaEventRecord(c->times_done, c->copy_stream);
    });
    c->feed_ready = reinterpret_cast<const unsigned long long*>(c->feed.p);
    c->feed_tag = tag;
    const cko_status fs = forward_core(c, m, d_states, d_times, nb, nt, nc, st, sv, nullptr, fwd, nullptr, err,
                                       nullptr, true);
    c->feed_ready = nullptr;
    feeder.join();
    checker.join();
    if (feed_err == cudaSuccess) feed_err = cudaStreamWaitEvent(c->stream, c->times_done, 0);
    if (feed_err == cudaSuccess) feed_err = cudaStreamSynchronize(c->copy_stream);
    if (bad >= 0) {
      const int i = (int)(bad / nb), b = (int)(bad % nb);
      return fail(err, CKO_INVALID_TIME_GRID, "time grid must be strictly increasing (step %d, batch %d)", i, b);
    }
    if (feed_err != cudaSuccess) return fail(err, CKO_CUDA, "time grid upload: %s", cudaGetErrorString(feed_err));
    if (fs != CKO_OK) return fs;
  }
  if (!states_out)
    return adjoint_core(c, m, d_states, d_times, nb, nt, nc, sv, CKO_LOSS_FROBENIUS, nullptr, loss_out, grad_out,
                        bwd, err, false, true);
  // The trajectory download overlaps the adjoint (both only read d_states): a helper thread copies it on
  // the context's copy stream (a pageable destination blocks the issuing thread, not the adjoint's
  // launches), while this thread runs the adjoint on the compute stream.
  if (!c->copy_stream) CUDA_TRY(cudaStreamCreateWithFlags(&c->copy_stream, cudaStreamNonBlocking));
  if (!c->fwd_done) CUDA_TRY(cudaEventCreateWithFlags(&c->fwd_done, cudaEventDisableTiming));
  CUDA_TRY(cudaEventRecord(c->fwd_done, c->stream));
  cudaError_t copy_err = cudaSuccess;
  std::thread copier([&] {
    copy_err = cudaSetDevice(c->device);
    if (copy_err == cudaSuccess) copy_err = cudaStreamWaitEvent(c->copy_stream, c->fwd_done, 0);
    if (copy_err == cudaSuccess)
      copy_err = cudaMemcpyAsync(states_out, d_states, sizeof(double) * row * (nt + 1), cudaMemcpyDeviceToHost,
                                 c->copy_stream);
    if (copy_err == cudaSuccess) copy_err = cudaStreamSynchronize(c->copy_stream);
  });
  cko_status s = adjoint_core(c, m, d_states, d_times, nb, nt, nc, sv, CKO_LOSS_FROBENIUS, nullptr, loss_out,
                              grad_out, bwd, err, false, true);
  copier.join();
  if (s != CKO_OK) return s;
  if (copy_err != cudaSuccess) return fail(err, CKO_CUDA, "trajectory D2H: %s", cudaGetErrorString(copy_err));
  return CKO_OK;
}

cko_status cko_traj_states(const cko_traj* t, const double** d_states, int* nb, int* nt, int* n) {
  if (!t) return CKO_ERROR;
  if (d_states) *d_states = t->d_states;
  if (nb) *nb = t->nb;
  if (nt) *nt = t->nt;
  if (n) *n = t->n;
  return CKO_OK;
}

cko_status cko_traj_destroy(cko_traj* t) {
  if (!t) return CKO_OK;
  cudaSetDevice(t->ctx->device);
  cudaFree(t->d_states);
  cudaFree(t->d_times);
  delete t;
  return CKO_OK;
}

cko_status cko_block_bidiag_solve(cko_ctx* c, const cko_solver_choice* sv, int nc, int nb, int n,
                                  const double* diag, const double* offdiag, double* rhs, long long* sweeps,
                                  cko_error* err) {
  if (!c || !sv || !diag || !rhs) return fail(err, CKO_ERROR, "null argument");
  if (nc < 1 || nb < 1 || n < 1) return fail(err, CKO_SHAPE_MISMATCH, "block bidiagonal system must be non-empty");
  if (sv->kind < 0 || sv->kind > 2) return fail(err, CKO_ERROR, "unknown solver kind %d", sv->kind);
  if (sv->kind == CKO_SOLVER_HYBRID && sv->n_switch < 0)
    return fail(err, CKO_ERROR, "solve_hybrid: n_switch must be >= 0");
  CUDA_TRY(cudaSetDevice(c->device));
  const size_t nd = (size_t)nc * nb * n * n, no = (size_t)(nc > 1 ? nc - 1 : 0) * nb * n * n,
               nr = (size_t)nc * nb * n;
  CUDA_TRY(c->h_diag.ensure(sizeof(double) * nd));
  CUDA_TRY(c->h_rhs.ensure(sizeof(double) * nr));
  CUDA_TRY(cudaMemcpyAsync(c->h_diag.p, diag, sizeof(double) * nd, cudaMemcpyHostToDevice, c->stream));
  CUDA_TRY(cudaMemcpyAsync(c->h_rhs.p, rhs, sizeof(double) * nr, cudaMemcpyHostToDevice, c->stream));
  const double* d_off = nullptr;
  if (offdiag) {
    CUDA_TRY(c->h_off.ensure(sizeof(double) * (no ? no : 1)));
    if (no) CUDA_TRY(cudaMemcpyAsync(c->h_off.p, offdiag, sizeof(double) * no, cudaMemcpyHostToDevice, c->stream));
    d_off = c->h_off.as<double>();
  }
  const int G = nb < 2 * c->sms ? nb : 2 * c->sms;
  Slab slab;
  if (cko_status s = prepare_slab(c, G, nb, nc, n, sv->kind != CKO_SOLVER_THOMAS || offdiag, slab, err)) return s;
  CUDA_TRY(c->key.ensure(sizeof(unsigned long long)));
  CUDA_TRY(cudaMemsetAsync(c->key.p, 0xff, sizeof(unsigned long long), c->stream));
  SolveLaunch a{};
  a.diag = c->h_diag.as<double>();
  a.offdiag = d_off;
  a.x = c->h_rhs.as<double>();
  a.nc = nc;
  a.nb = nb;
  a.n = n;
  a.solver = sv->kind;
  a.n_switch = sv->n_switch;
  a.slab = slab;
  a.sing_key = c->key.as<unsigned long long>();
  a.grid = G;
  a.threads = kThreads;
  CUDA_TRY(launch_solve(a, c->stream));
  unsigned long long key;
  CUDA_TRY(cudaMemcpyAsync(&key, c->key.p, sizeof key, cudaMemcpyDeviceToHost, c->stream));
  CUDA_TRY(cudaMemcpyAsync(rhs, c->h_rhs.p, sizeof(double) * nr, cudaMemcpyDeviceToHost, c->stream));
  CUDA_TRY(cudaStreamSynchronize(c->stream));
  if (key != ~0ull) {
    const int k = (int)(key / (unsigned long long)nb), b = (int)(key % (unsigned long long)nb);
    cko_status s = fail(err, CKO_SINGULAR_BLOCK, "singular diagonal block at chunk row %d, batch %d", k, b);
    if (err) err->chunk_index = k, err->batch_index = b;
    return s;
  }
  if (sweeps) *sweeps = sweeps_of(nc, sv->kind, sv->n_switch);
  return ok(err);
}

cko_status cko_newton_solve_chunk(cko_ctx* c, const cko_model* m, const double* y_start, double* dy,
                                  const double* t_chunk, const double* dt_chunk, int cc, int nb,
                                  const cko_newton_settings* st, const cko_solver_choice* sv, int chunk_start_step,
                                  int* iterations, cko_work* work, cko_error* err) {
  if (!c || !m || !y_start || !dy || !t_chunk || !dt_chunk || !st || !sv) return fail(err, CKO_ERROR, "null argument");
  if (cc < 1 || nb < 1) return fail(err, CKO_SHAPE_MISMATCH, "chunk op: empty chunk");
  CUDA_TRY(cudaSetDevice(c->device));
  // One chunk through the generic forward kernel with explicit step sizes: rate times are t_chunk (rows
  // 1..c of a (c+1)-row grid, row 0 unused), dt(k) = dt_chunk(k) exactly as newton_chunk reads them
  // (integrate.cpp:64-95, 118-135) — dt_chunk need not equal the differences of t_chunk.
  const int n = m->dm.n;
  const size_t row = (size_t)nb * n, trow = (size_t)nb;
  CUDA_TRY(c->h_states.ensure(sizeof(double) * row * (cc + 1)));
  CUDA_TRY(c->h_times.ensure(sizeof(double) * trow * (cc + 1 + cc)));
  CUDA_TRY(c->h_dL.ensure(sizeof(double) * row * cc));
  double* d_states = c->h_states.as<double>();
  double* d_times = c->h_times.as<double>();
  double* d_dts = d_times + trow * (cc + 1);
  CUDA_TRY(cudaMemcpyAsync(d_times + trow, t_chunk, sizeof(double) * trow * cc, cudaMemcpyHostToDevice, c->stream));
  CUDA_TRY(cudaMemcpyAsync(d_times, t_chunk, sizeof(double) * trow, cudaMemcpyHostToDevice, c->stream));
  CUDA_TRY(cudaMemcpyAsync(d_dts, dt_chunk, sizeof(double) * trow * cc, cudaMemcpyHostToDevice, c->stream));
  CUDA_TRY(cudaMemcpyAsync(d_states, y_start, sizeof(double) * row, cudaMemcpyHostToDevice, c->stream));
  CUDA_TRY(cudaMemcpyAsync(c->h_dL.p, dy, sizeof(double) * row * cc, cudaMemcpyHostToDevice, c->stream));
  cko_status s = forward_core(c, m, d_states, d_times, nb, cc, cc, st, sv, c->h_dL.as<double>(), work, iterations,
                              err, d_dts);
  if (s != CKO_OK) {
    if (s == CKO_NEWTON_DIVERGENCE && err) err->chunk_start_step = chunk_start_step;
    return s;
  }
  std::vector<double> out(row * (cc + 1));
  CUDA_TRY(cudaMemcpyAsync(out.data(), d_states, sizeof(double) * out.size(), cudaMemcpyDeviceToHost, c->stream));
  CUDA_TRY(cudaStreamSynchronize(c->stream));
  for (int k = 0; k < cc; ++k)
    for (size_t i = 0; i < row; ++i) dy[(size_t)k * row + i] = out[(size_t)(k + 1) * row + i] - y_start[i];
  return ok(err);
}

// chunk_residual / chunk_jacobian (integrate.cpp:269-297) on the device.
static cko_status chunk_op(cko_ctx* c, const cko_model* m, int op, const double* y_start, const double* dy,
                           const double* t_chunk, const double* dt_chunk, int cc, int nb, double* out,
                           double* offdiag_out, cko_error* err) {
  if (m) const_cast<cko_model*>(m)->dm.jstrat = c->jstrat;  // the call's JacobianStrategy
  if (!c || !m || !y_start || !dy || !t_chunk || !dt_chunk || !out) return fail(err, CKO_ERROR, "null argument");
  if (cc < 1 || nb < 1) return fail(err, CKO_SHAPE_MISMATCH, "chunk op: empty chunk");
  if (cko_status s = check_lanes(m, nb, err)) return s;
  CUDA_TRY(cudaSetDevice(c->device));
  const int n = m->dm.n;
  const size_t P = (size_t)cc * nb, nout = op == 0 ? P * n : P * n * n;
  CUDA_TRY(c->h_states.ensure(sizeof(double) * (2 * P * n + (size_t)nb * n)));
  CUDA_TRY(c->h_times.ensure(sizeof(double) * 2 * P));
  CUDA_TRY(c->h_diag.ensure(sizeof(double) * nout));
  CUDA_TRY(c->status.ensure(sizeof(unsigned)));
  double* d_ys = c->h_states.as<double>();
  double* d_dy = d_ys + (size_t)nb * n;
  double* d_yy = d_dy + P * n;
  double* d_t = c->h_times.as<double>();
  double* d_dt = d_t + P;
  CUDA_TRY(cudaMemcpyAsync(d_ys, y_start, sizeof(double) * nb * n, cudaMemcpyHostToDevice, c->stream));
  CUDA_TRY(cudaMemcpyAsync(d_dy, dy, sizeof(double) * P * n, cudaMemcpyHostToDevice, c->stream));
  CUDA_TRY(cudaMemcpyAsync(d_t, t_chunk, sizeof(double) * P, cudaMemcpyHostToDevice, c->stream));
  CUDA_TRY(cudaMemcpyAsync(d_dt, dt_chunk, sizeof(double) * P, cudaMemcpyHostToDevice, c->stream));
  CUDA_TRY(cudaMemsetAsync(c->status.p, 0, sizeof(unsigned), c->stream));
  CUDA_TRY(launch_chunk_op(m->dm, op, d_ys, d_dy, d_t, d_dt, cc, nb, d_yy, c->h_diag.as<double>(),
                           c->status.as<unsigned>(), c->stream));
  unsigned flag = 0;
  CUDA_TRY(cudaMemcpyAsync(out, c->h_diag.p, sizeof(double) * nout, cudaMemcpyDeviceToHost, c->stream));
  CUDA_TRY(cudaMemcpyAsync(&flag, c->status.p, sizeof flag, cudaMemcpyDeviceToHost, c->stream));
  CUDA_TRY(cudaStreamSynchronize(c->stream));
  c->last_launches = 1;
  c->last_gen = 1;
  if (flag)
    return fail(err, CKO_NON_FINITE, op == 0 ? "chunk_residual: model rate returned a non-finite value"
                                             : "Jacobian of the model is not finite");
  if (op == 1 && offdiag_out && cc > 1) {  // the -I couplings (fill_unit_offdiag, integrate.cpp:140-147)
    const size_t no = (size_t)(cc - 1) * nb * n * n;
    std::memset(offdiag_out, 0, sizeof(double) * no);
    for (size_t blk = 0; blk < (size_t)(cc - 1) * nb; ++blk)
      for (int i = 0; i < n; ++i) offdiag_out[blk * n * n + (size_t)i * n + i] = -1.0;
  }
  return ok(err);
}

cko_status cko_chunk_residual(cko_ctx* c, const cko_model* m, const double* y_start, const double* dy,
                              const double* t_chunk, const double* dt_chunk, int cc, int nb, double* out,
                              cko_error* err) {
  return chunk_op(c, m, 0, y_start, dy, t_chunk, dt_chunk, cc, nb, out, nullptr, err);
}

cko_status cko_chunk_jacobian(cko_ctx* c, const cko_model* m, const double* y_start, const double* dy,
                              const double* t_chunk, const double* dt_chunk, int cc, int nb, double* diag_out,
                              double* offdiag_out, cko_error* err) {
  return chunk_op(c, m, 1, y_start, dy, t_chunk, dt_chunk, cc, nb, diag_out, offdiag_out, err);
}

// One reversed chunk over host rows lo = step_hi - chunk_len .. step_hi of a trajectory: the rows are
// staged as a (chunk_len + 1)-row mini trajectory and reversed as its only chunk, lambda carried in and
// out, the chunk's parameter product added to grad (be_chunk_core, adjoint.cpp:49-127).
static cko_status chunk_reverse(cko_ctx* c, const cko_model* m, const double* states_rows, const double* times_rows,
                                const double* dL_rows, int nb, int chunk_len, const cko_solver_choice* sv,
                                double* lambda, double* grad, cko_work* work, cko_error* err) {
  const int n = m->dm.n, np = m->dm.np;
  const size_t row = (size_t)nb * n, rows = (size_t)chunk_len + 1;
  CUDA_TRY(c->h_states.ensure(sizeof(double) * row * rows));
  CUDA_TRY(c->h_times.ensure(sizeof(double) * (size_t)nb * rows));
  CUDA_TRY(c->h_dL.ensure(sizeof(double) * row * rows));
  CUDA_TRY(c->lambda.ensure(sizeof(double) * row));
  CUDA_TRY(cudaMemcpyAsync(c->h_states.p, states_rows, sizeof(double) * row * rows, cudaMemcpyHostToDevice,
                           c->stream));
  CUDA_TRY(cudaMemcpyAsync(c->h_times.p, times_rows, sizeof(double) * nb * rows, cudaMemcpyHostToDevice, c->stream));
  CUDA_TRY(cudaMemcpyAsync(c->h_dL.p, dL_rows, sizeof(double) * row * rows, cudaMemcpyHostToDevice, c->stream));
  CUDA_TRY(cudaMemcpyAsync(c->lambda.p, lambda, sizeof(double) * row, cudaMemcpyHostToDevice, c->stream));
  std::vector<double> g(np);
  cko_status s = adjoint_core(c, m, c->h_states.as<double>(), c->h_times.as<double>(), nb, chunk_len, chunk_len, sv,
                              CKO_LOSS_USER, c->h_dL.as<double>(), nullptr, g.data(), work, err, true);
  if (s != CKO_OK) return s;
  CUDA_TRY(cudaMemcpyAsync(lambda, c->lambda.p, sizeof(double) * row, cudaMemcpyDeviceToHost, c->stream));
  CUDA_TRY(cudaStreamSynchronize(c->stream));
  for (int j = 0; j < np; ++j) grad[j] += g[j];
  for (int j = 0; j < np; ++j)
    if (!std::isfinite(grad[j])) return fail(err, CKO_NON_FINITE, "parameter product of the model is not finite");
  return ok(err);
}

cko_status cko_adjoint_chunk_solve(cko_ctx* c, const cko_model* m, const double* states, const double* times, int nb,
                                   int nt, int step_hi, int chunk_len, const double* dL,
                                   const cko_solver_choice* sv, double* lambda, double* grad, cko_work* work,
                                   cko_error* err) {
  if (!c || !m || !states || !times || !dL || !sv || !lambda || !grad) return fail(err, CKO_ERROR, "null argument");
  if (!(chunk_len >= 1 && step_hi >= chunk_len && step_hi <= nt))
    return fail(err, CKO_SHAPE_MISMATCH, "adjoint chunk: step range out of bounds");
  CUDA_TRY(cudaSetDevice(c->device));
  const size_t row = (size_t)nb * m->dm.n, lo = (size_t)(step_hi - chunk_len);
  return chunk_reverse(c, m, states + lo * row, times + lo * nb, dL + lo * row, nb, chunk_len, sv, lambda, grad,
                       work, err);
}

cko_status cko_adjoint_step_sequential(cko_ctx* c, const cko_model* m, const double* y_i, const double* y_prev,
                                       const double* t_i, const double* t_prev, const double* dL_i, int nb,
                                       const cko_solver_choice* sv, double* lambda, double* grad, cko_error* err) {
  if (!c || !m || !y_i || !y_prev || !t_i || !t_prev || !dL_i || !sv || !lambda || !grad)
    return fail(err, CKO_ERROR, "null argument");
  if (nb < 1) return fail(err, CKO_SHAPE_MISMATCH, "adjoint step: empty batch");
  for (int b = 0; b < nb; ++b)
    if (!(t_i[b] > t_prev[b])) return fail(err, CKO_SHAPE_MISMATCH, "adjoint step: dt must be positive");
  CUDA_TRY(cudaSetDevice(c->device));
  const size_t row = (size_t)nb * m->dm.n;
  std::vector<double> st(2 * row), tt(2 * (size_t)nb), dl(2 * row, 0.0);
  std::memcpy(st.data(), y_prev, sizeof(double) * row);
  std::memcpy(st.data() + row, y_i, sizeof(double) * row);
  std::memcpy(tt.data(), t_prev, sizeof(double) * nb);
  std::memcpy(tt.data() + nb, t_i, sizeof(double) * nb);
  std::memcpy(dl.data() + row, dL_i, sizeof(double) * row);
  return chunk_reverse(c, m, st.data(), tt.data(), dl.data(), nb, 1, sv, lambda, grad, nullptr, err);
}

}  // extern "C"
