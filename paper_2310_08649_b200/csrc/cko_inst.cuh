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
                          (const void*)vjp_kernel<MD, 1024>, (const void*)chunk_op_kernel<MD>,      \
                          (const void*)fe_forward_kernel<MD>, (const void*)fe_adjoint_kernel<MD>})    \
      if (cudaError_t e = preload(f)) return e;                                                       \
    return cudaSuccess;                                                                               \
  }                                                                                                   \
  cudaError_t chunk_op_run_##NAME(const DevModel& m, int op, const double* ys, const double* dy,       \
                                  const double* t, const double* dt, int c, int nb, double* yyb,       \
                                  double* out, unsigned* flags, cudaStream_t st) {                     \
    const int blocks = (c * nb + 127) / 128 < 1184 ? (c * nb + 127) / 128 : 1184;                     \
    chunk_op_kernel<MD><<<blocks, 128, 0, st>>>(m, op, ys, dy, t, dt, c, nb, yyb, out, flags);        \
    return cudaGetLastError();                                                                        \
  }                                                                                                   \
  cudaError_t fe_forward_run_##NAME(const DevModel& m, double* states, const double* times, int nb,   \
                                    int nt, double* hbuf, int* bad, cudaStream_t st) {                 \
    fe_forward_kernel<MD><<<(nb + 127) / 128, 128, 0, st>>>(m, states, times, nb, nt, hbuf, bad);     \
    return cudaGetLastError();                                                                        \
  }                                                                                                   \
  cudaError_t fe_adjoint_run_##NAME(const DevModel& m, const double* states, const double* times,     \
                                    const double* dL, const double* loss, int nb, int nt,              \
                                    double* lambda, double* Jb, double* tmp, double* wq,               \
                                    unsigned* bad, cudaStream_t st) {                                  \
    fe_adjoint_kernel<MD><<<(nb + 127) / 128, 128, 0, st>>>(m, states, times, dL, loss, nb, nt, lambda, \
                                                            Jb, tmp, wq, bad);                        \
    return cudaGetLastError();                                                                        \
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
