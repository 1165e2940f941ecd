// cko_common.cuh — shared device utilities for the sm_100a chunked
// backward-Euler kernels: strided slab views, IEEE-exact helpers for the
// parity-critical residual arithmetic, and a grid-wide barrier that carries
// the Newton convergence predicate.
#pragma once

#include <cstdint>
#include <cstdlib>
#include <map>
#include <mutex>
#include <utility>
#include <cuda_runtime.h>

namespace cko {

// Raise a kernel's dynamic shared-memory limit. Function attributes live in
// each device's context, so the setting is cached per (device, kernel): a
// second context on another device sets it again. Setting it on every launch
// would serialise concurrent launches of the same kernel from other streams
// (the attribute write waits for running instances).
inline cudaError_t allow_smem(const void* func, int bytes) {
  static std::mutex mu;
  static std::map<std::pair<int, const void*>, int> done;
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return e;
  std::lock_guard<std::mutex> lock(mu);
  auto it = done.find({dev, func});
  if (it != done.end() && it->second >= bytes) return cudaSuccess;
  e = cudaFuncSetAttribute(func, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes);
  if (e == cudaSuccess) done[{dev, func}] = bytes;
  return e;
}
// Force a kernel's module to load now. With lazy module loading (the CUDA 12
// default) the first launch of a kernel may wait for the device to go idle;
// in a batch group a rank whose host thread blocks there while its peer's
// kernel spins on the group exchange would stall both. cko_ctx_set_group
// therefore loads every kernel up front.
inline cudaError_t preload(const void* func) {
  cudaFuncAttributes fa;
  return cudaFuncGetAttributes(&fa, func);
}
#define CKO_ALLOW_FULL_SMEM(KERNEL)                                                   \
  do {                                                                               \
    const cudaError_t _cko_attr_err = ::cko::allow_smem((const void*)(KERNEL), 226 * 1024); \
    if (_cko_attr_err != cudaSuccess) return _cko_attr_err;                          \
  } while (0)

// Persistent grid-barrier kernels launch cooperatively (every CTA resident).
// CKO_PLAIN_LAUNCH=1 switches to an ordinary launch: used only by the
// single-GPU group test, where two ranks' small grids must run concurrently
// and CUDA does not overlap two cooperative launches (the grids there are a
// few CTAs, resident either way).
inline cudaError_t launch_persistent(const void* func, dim3 grid, dim3 block, void** args, size_t smem,
                                     cudaStream_t st) {
  const char* plain = std::getenv("CKO_PLAIN_LAUNCH");
  if (plain && plain[0] == '1') return cudaLaunchKernel(func, grid, block, args, smem, st);
  return cudaLaunchCooperativeKernel(func, grid, block, args, smem, st);
}

// Per-CTA workspace slabs are stored component-major / point-minor:
// element e of point p lives at base[e * stride + p], so consecutive threads
// (consecutive points) touch consecutive addresses.
struct SVec {
  double* p;
  int s;
  __device__ __forceinline__ double& operator[](int i) const { return p[(size_t)i * s]; }
};
struct SBlk {
  double* p;
  int s;
  int n;
  __device__ __forceinline__ double& operator()(int i, int j) const {
    return p[(size_t)(i * n + j) * s];
  }
};
struct SPiv {
  int* p;
  int s;
  __device__ __forceinline__ int& operator[](int i) const { return p[(size_t)i * s]; }
};

// Exact-rounding arithmetic, no FMA contraction: the residual and its norm
// decide the Newton predicate (integrate.cpp:64-95, :176-182), so they follow
// the reference's operation order to the bit.
__device__ __forceinline__ double xmul(double a, double b) { return __dmul_rn(a, b); }
__device__ __forceinline__ double xadd(double a, double b) { return __dadd_rn(a, b); }
__device__ __forceinline__ double xsub(double a, double b) { return __dsub_rn(a, b); }

__device__ __forceinline__ uint64_t globaltimer_ns() {
  uint64_t t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}

// Flags carried through the grid barrier (OR-reduced over all CTAs).
enum : unsigned {
  FLAG_NOT_CONVERGED = 1u,  // some lane fails |r| <= tol_a || |r| <= tol_r |r0|
  FLAG_NON_FINITE = 2u,     // some lane's residual norm is not finite
  FLAG_SINGULAR = 4u,       // a diagonal block failed the pivot check
  FLAG_TIMEOUT = 8u,        // barrier wait exceeded its budget (abort)
  FLAG_FALLBACK = 16u,      // a structured-record block is not eligible: re-run on the group-LU kernels
};

// Grid barrier state (device memory, zero-initialised by the host).
// `flags` is a 3-slot ring so the slot of barrier g+1 can be cleared by the
// releaser of barrier g without racing readers of slot g.
struct GridSync {
  unsigned count;
  unsigned gen;
  unsigned flags[3];
  unsigned pad;
  // multi-GPU exchange (see cko_comm): this rank's generation counter that
  // peers poll, and where peers deposit their flags.
  unsigned long long ext_gen;
};

// Multi-GPU group view passed to kernels: peer GridComm buffers mapped into
// this process. world == 1 disables the exchange.
struct GroupView {
  int rank;
  int world;
  unsigned long long* peer_slots[8];  // peer_slots[r] -> rank r's slot array [2][world]
  double* peer_red[8];                // peer_red[r]   -> rank r's reduce buffer [2][world][red_cap]
  int red_cap;
};

// Publish this rank's OR-reduced flags for generation `gen` to every peer and
// wait until every peer has published generation `gen`; return the OR over
// ranks. Slot word: (gen << 8) | flags, in the parity-(gen & 1) half of each
// rank's [2][world] slot array: a peer can run at most one generation ahead,
// so it never overwrites a word of the generation still being read.
// Called by exactly one thread per rank.
__device__ inline unsigned group_exchange(const GroupView& g, unsigned long long gen, unsigned flags,
                                          uint64_t deadline) {
  if (g.world <= 1) return flags;
  const unsigned long long word = (gen << 8) | (unsigned long long)(flags & 0xffu);
  const int half = (int)(gen & 1ull) * g.world;
  for (int r = 0; r < g.world; ++r) {
    volatile unsigned long long* slot = g.peer_slots[r] + half + g.rank;
    __threadfence_system();
    *slot = word;
  }
  __threadfence_system();
  unsigned acc = flags;
  volatile unsigned long long* mine = g.peer_slots[g.rank] + half;
  for (int r = 0; r < g.world; ++r) {
    unsigned long long v;
    while (((v = mine[r]) >> 8) < gen) {
      if (globaltimer_ns() > deadline) return acc | FLAG_TIMEOUT;
      __nanosleep(64);
    }
    acc |= (unsigned)(v & 0xffu);
  }
  return acc;
}

// Grid-wide barrier with an OR-reduction of per-CTA flags (and, for a
// sharded batch, of per-rank flags). Requires a cooperative launch so every
// CTA is resident. Spins are bounded by `budget_ns`; on expiry the barrier
// returns FLAG_TIMEOUT instead of hanging the device.
__device__ inline unsigned grid_reduce_or(GridSync* gs, const GroupView& grp, unsigned local,
                                          uint64_t budget_ns, unsigned* s_bcast) {
  __syncthreads();
  if (threadIdx.x == 0) {
    volatile unsigned* vgen = &gs->gen;
    const unsigned gen = *vgen;
    const unsigned slot = gen % 3u;
    if (local) atomicOr(&gs->flags[slot], local);
    __threadfence();
    const unsigned arrived = atomicAdd(&gs->count, 1u);
    const uint64_t deadline = globaltimer_ns() + budget_ns;
    unsigned result;
    if (arrived == gridDim.x - 1) {
      gs->count = 0;
      gs->flags[(gen + 1u) % 3u] = 0;
      __threadfence();
      unsigned f = *(volatile unsigned*)&gs->flags[slot];
      if (grp.world > 1) {
        gs->ext_gen += 1;
        f = group_exchange(grp, gs->ext_gen, f, deadline);
        *(volatile unsigned*)&gs->flags[slot] = f;
        __threadfence();
      }
      atomicExch(&gs->gen, gen + 1u);
      result = f;
    } else {
      while (*vgen == gen) {
        if (globaltimer_ns() > deadline) {
          result = FLAG_TIMEOUT;
          goto done;
        }
        __nanosleep(32);
      }
      __threadfence();
      result = *(volatile unsigned*)&gs->flags[slot];
    }
  done:
    *s_bcast = result;
  }
  __syncthreads();
  return *s_bcast;
}

// Deterministic sum over ranks of a small device vector (loss sum of squares,
// parameter gradient): every rank stores its vector into row `rank` of every
// peer's reduce buffer over NVLink (P2P stores), publishes a generation flag,
// waits for all peers, then sums rows 0..world-1 in rank order, so all ranks
// hold bitwise-identical results. Single block; `gs` carries the generation.
__device__ inline void group_sum_block(const GroupView& g, GridSync* gs, const double* local, int cnt, double* out,
                                       uint64_t budget_ns, unsigned* status) {
  __shared__ unsigned long long s_gen;
  __shared__ unsigned s_ok;
  if (threadIdx.x == 0) s_gen = gs->ext_gen + 1;
  __syncthreads();
  const unsigned long long gen = s_gen;
  const size_t half = (size_t)(gen & 1ull) * g.world * g.red_cap;
  for (int r = 0; r < g.world; ++r) {
    double* dst = g.peer_red[r] + half + (size_t)g.rank * g.red_cap;
    for (int i = threadIdx.x; i < cnt; i += blockDim.x) dst[i] = local[i];
  }
  __threadfence_system();
  __syncthreads();
  if (threadIdx.x == 0) {
    gs->ext_gen = gen;
    const unsigned f = group_exchange(g, gen, 0u, globaltimer_ns() + budget_ns);
    s_ok = (f & FLAG_TIMEOUT) ? 0u : 1u;
    __threadfence_system();
  }
  __syncthreads();
  if (!s_ok) {
    if (threadIdx.x == 0) *status = FLAG_TIMEOUT;
    return;
  }
  const double* mine = g.peer_red[g.rank] + half;
  for (int i = threadIdx.x; i < cnt; i += blockDim.x) {
    double s = 0.0;
    for (int r = 0; r < g.world; ++r) s += ((volatile const double*)mine)[(size_t)r * g.red_cap + i];
    out[i] = s;
  }
}

}  // namespace cko
