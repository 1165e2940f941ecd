// Micro-benchmark: thread-per-block LU (cko_lu_thread.cuh) for N = 20, records
// in shared memory, 28 active threads per warp; 1 or 2 warps.
#include <cstdio>
#include "../../paper_2310_08649_b200/csrc/cko_lu_thread.cuh"
constexpr int N = 20;
constexpr int STRIDE = N * N + 2 * N + 2 + 14;  // 2 mod 16 doubles

__global__ void k_lut(int iters, long long* out, double* sink) {
  extern __shared__ __align__(16) double sm[];
  __shared__ double init[N * N];
  for (int e = threadIdx.x; e < N * N; e += blockDim.x) {
    const int i = e / N, j = e % N;
    init[e] = (i == j) ? 1.0 : 0.01 * ((i * 7 + j * 3) % 11) - 0.05;
  }
  __syncthreads();
  const int t = threadIdx.x, lane = t & 31;
  double* A = sm + t * STRIDE;
  double* rd = A + N * N;
  bool okall = true;
  long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
    if (lane < 28) {
      for (int e = 0; e < N * N; e += 2) *reinterpret_cast<double2*>(A + e) = *reinterpret_cast<const double2*>(init + e);
      bool viol;
      okall &= cko::lt::lu_thread_nopiv<N>(A, rd, 1e-14, viol);
      okall &= !viol;
    }
    __syncwarp();
  }
  long long t1 = clock64();
  if (t == 0) out[0] = (t1 - t0) / iters;
  if (!okall) sink[0] = 1.0;
}

int main() {
  long long* d_out;
  double* d_sink;
  cudaMalloc(&d_out, 8);
  cudaMalloc(&d_sink, 8);
  cudaMemset(d_sink, 0, 8);
  const int smem = 56 * STRIDE * 8;
  printf("smem %d\n", smem);
  cudaFuncSetAttribute(k_lut, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  for (int warps : {1, 2}) {
    k_lut<<<1, 32 * warps, smem>>>(50, d_out, d_sink);
    printf("%s ", cudaGetErrorString(cudaGetLastError()));
    long long c = 0;
    cudaMemcpy(&c, d_out, 8, cudaMemcpyDeviceToHost);
    printf("warps %d: %lld cycles per batch (28 LUs per warp) -> %.1f SM-cycles per LU\n", warps, c,
           (double)c / (28.0 * warps));
  }
  double s = 0;
  cudaMemcpy(&s, d_sink, 8, cudaMemcpyDeviceToHost);
  printf("sink %g (0 = all fast-path and nonsingular)\n", s);
  return 0;
}
