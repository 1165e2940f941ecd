// Micro-benchmark: latency of one consumer step (lu_solve_rec<20>) on one warp,
// alone and next to DFMA-busy warps. Diagnostics only.
#include <cstdio>
#include "../../paper_2310_08649_b200/csrc/cko_v2.cuh"
using namespace cko::v2;
constexpr int N = 20;

__global__ void k_solve(int iters, int busy_warps, long long* out, double* sink) {
  extern __shared__ __align__(16) double sm[];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  double* recs = sm;
  double* vs = sm + 8 * Rec<N>::STRIDE;
  for (int i = threadIdx.x; i < 8 * Rec<N>::STRIDE; i += blockDim.x) recs[i] = 0.001 * (i % 17);
  __syncthreads();
  if (threadIdx.x < 8)
    for (int i = 0; i < N; ++i) {
      recs[threadIdx.x * Rec<N>::STRIDE + i * N + i] = 1.0;
      recs[threadIdx.x * Rec<N>::STRIDE + Rec<N>::RD + i] = 1.0;
      reinterpret_cast<int*>(recs + threadIdx.x * Rec<N>::STRIDE + Rec<N>::PERM)[i] = i;
      reinterpret_cast<int*>(recs + threadIdx.x * Rec<N>::STRIDE + Rec<N>::PERM)[N] = 1;
    }
  __syncthreads();
  if (warp == 0) {
    double v[N];
    for (int i = 0; i < N; ++i) v[i] = lane + i;
    long long t0 = clock64();
    for (int it = 0; it < iters; ++it) {
      if (lane < 7) lu_solve_rec<N>(recs + lane * Rec<N>::STRIDE, vs + lane * N, v);
      __syncwarp();
    }
    long long t1 = clock64();
    if (lane == 0) out[0] = (t1 - t0) / iters;
    double s = 0;
    for (int i = 0; i < N; ++i) s += v[i];
    if (s == 1234.5) sink[0] = s;
  } else if (warp <= busy_warps) {
    double a[8];
    for (int k = 0; k < 8; ++k) a[k] = 1.0 + lane * 1e-3 + k;
    for (int it = 0; it < iters * 40; ++it)
      for (int k = 0; k < 8; ++k) a[k] = fma(a[k], 0.999999, 1e-9);
    double s = 0;
    for (int k = 0; k < 8; ++k) s += a[k];
    if (s == 1234.5) sink[0] = s;
  }
}

int main() {
  long long* d_out;
  double* d_sink;
  cudaMalloc(&d_out, 8);
  cudaMalloc(&d_sink, 8);
  const int smem = (8 * Rec<N>::STRIDE + 8 * N) * 8;
  cudaFuncSetAttribute(k_solve, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  for (int busy : {0, 3, 9}) {
    k_solve<<<1, 32 * (busy + 1), smem>>>(200, busy, d_out, d_sink);
    long long c = 0;
    cudaMemcpy(&c, d_out, 8, cudaMemcpyDeviceToHost);
    printf("busy warps %d: %lld cycles per consumer step\n", busy, c);
  }
  return 0;
}
