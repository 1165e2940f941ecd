// cko_inst.cuh — one translation unit per device model (parallel builds).
#pragma once
#include "cko_impl.cuh"
#include "cko_v2.cuh"
#include "cko_pcr2.cuh"

#define CKO_INSTANTIATE(NAME, MD)                                                                      \
  namespace cko {                                                                                     \
  cudaError_t fwd_run_##NAME(const FwdLaunch& a, cudaStream_t st) {                                   \
    FwdLaunch copy = a;                                                                               \
    void* args[] = {&copy};                                                                           \
    return launch_persistent((const void*)fwd_kernel<MD>, dim3(a.grid), dim3(a.threads),    \
                                       args, 0, st);                                                  \
  }                                                                                                   \
  cudaError_t fwd_occ_##NAME(int threads, int* blocks) {                                              \
    return cudaOccupancyMaxActiveBlocksPerMultiprocessor(blocks, fwd_kernel<MD>, threads, 0);         \
  }                                                                                                   \
  cudaError_t preload_##NAME() {                                                                      \
    for (const void* f : {(const void*)fwd_kernel<MD>, (const void*)adj_kernel<MD>,                   \
                          (const void*)vjp_kernel<MD, 16>, (const void*)vjp_kernel<MD, 64>,           \
                          (const void*)vjp_kernel<MD, 1024>})                                         \
      if (cudaError_t e = preload(f)) return e;                                                       \
    return cudaSuccess;                                                                               \
  }                                                                                                   \
  cudaError_t adj_run_##NAME(const AdjLaunch& a, cudaStream_t st) {                                   \
    adj_kernel<MD><<<a.grid, a.threads, 0, st>>>(a);                                                  \
    return cudaGetLastError();                                                                        \
  }                                                                                                   \
  cudaError_t vjp_run_##NAME(const DevModel& m, const double* states, const double* times,            \
                             const double* wq, int nb, int nt, double* scratch, cudaStream_t st) {    \
    int lo, hi;                                                                                       \
    lane_segment(m, lo, hi);                                                                          \
    const int nps = m.np - (hi - lo);                                                                 \
    if (nps <= 16)                                                                                    \
      vjp_kernel<MD, 16><<<kVjpBlocks, 256, 0, st>>>(m, states, times, wq, nb, nt, scratch);          \
    else if (nps <= 64)                                                                               \
      vjp_kernel<MD, 64><<<kVjpBlocks, 256, 0, st>>>(m, states, times, wq, nb, nt, scratch);          \
    else if (nps <= 1024)                                                                             \
      vjp_kernel<MD, 1024><<<kVjpBlocks, 64, 0, st>>>(m, states, times, wq, nb, nt, scratch);         \
    else                                                                                              \
      return cudaErrorNotSupported;                                                                   \
    return cudaGetLastError();                                                                        \
  }                                                                                                   \
  }
