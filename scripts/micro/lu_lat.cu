// Micro-benchmark: latency of the producer's group LU (fast path) for N = 20
// on one warp (3 groups of 10 lanes), alone and with 8 more warps doing the same.
#include <cstdio>
#include "../../paper_2310_08649_b200/csrc/cko_v2.cuh"
using namespace cko::v2;
constexpr int N = 20;
using Gm = Geo<N>;

__global__ void k_lu(int iters, long long* out, double* sink) {
  extern __shared__ __align__(16) double sm[];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const GroupLane<N> gr(lane);
  __shared__ double init[N * N];
  for (int e = threadIdx.x; e < N * N; e += blockDim.x) {
    const int i = e / N, j = e % N;
    init[e] = (i == j) ? 1.0 : 0.01 * ((i * 7 + j * 3) % 11) - 0.05;
  }
  __syncthreads();
  double* pb = sm + (warp * Gm::GPW + gr.g) * 2 * (N + 2);
  double* rec = sm + 27 * 2 * (N + 2) + (warp * Gm::GPW + gr.g) * Rec<N>::STRIDE;
  bool okall = true;
  long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
    double m[Gm::R][N];
#pragma unroll
    for (int q = 0; q < Gm::R; ++q) {
      const int i = gr.gl + q * Gm::G;
#pragma unroll
      for (int j = 0; j < N; ++j) m[q][j] = init[(i < N ? i : 0) * N + j];
    }
    bool viol;
    okall &= lu_group_nopiv<N>(m, gr.gl, gr.base, pb, rec, viol);
    okall &= !viol;
  }
  long long t1 = clock64();
  if (threadIdx.x == 0) out[0] = (t1 - t0) / iters;
  if (!okall) sink[0] = 1.0;
}

int main() {
  long long* d_out;
  double* d_sink;
  cudaMalloc(&d_out, 8);
  cudaMalloc(&d_sink, 8);
  const int smem = (27 * 2 * (N + 2) + 27 * Rec<N>::STRIDE) * 8;
  cudaFuncSetAttribute(k_lu, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  for (int warps : {1, 3, 9}) {
    k_lu<<<1, 32 * warps, smem>>>(200, d_out, d_sink);
    printf("%s ", cudaGetErrorString(cudaGetLastError()));
    long long c = 0;
    cudaMemcpy(&c, d_out, 8, cudaMemcpyDeviceToHost);
    printf("warps %d: %lld cycles per group LU (3 LUs per warp)\n", warps, c);
  }
  double s = 0;
  cudaMemcpy(&s, d_sink, 8, cudaMemcpyDeviceToHost);
  printf("sink %g\n", s);
  return 0;
}
