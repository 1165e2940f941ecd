// Micro-benchmarks: SHFL latency / throughput per SM, drcp latency, syncwarp+smem round trip.
#include <cstdio>
__global__ void k(int iters, long long* out, double* sink) {
  __shared__ double sm[64];
  const int lane = threadIdx.x & 31;
  double v = lane * 1.5;
  long long t0 = clock64();
  for (int i = 0; i < iters; ++i) v = __shfl_sync(0xffffffffu, v, (lane + 1) & 31) + 1.0;
  long long t1 = clock64();
  double w[8];
  for (int q = 0; q < 8; ++q) w[q] = v + q;
  long long t2 = clock64();
  for (int i = 0; i < iters; ++i)
#pragma unroll
    for (int q = 0; q < 8; ++q) w[q] = __shfl_sync(0xffffffffu, w[q], (lane + q) & 31);
  long long t3 = clock64();
  double r = 1.5 + lane;
  long long t4 = clock64();
  for (int i = 0; i < iters; ++i) r = __drcp_rn(r) + 1.0;
  long long t5 = clock64();
  double x = lane;
  long long t6 = clock64();
  for (int i = 0; i < iters; ++i) {
    if (lane == (i & 31)) sm[i & 31] = x;
    __syncwarp();
    x = sm[i & 31] + 1.0;
  }
  long long t7 = clock64();
  if (threadIdx.x == 0) { out[0] = t1 - t0; out[1] = t3 - t2; out[2] = t5 - t4; out[3] = t7 - t6; }
  double s = v + r + x;
  for (int q = 0; q < 8; ++q) s += w[q];
  if (s == 1.2345) sink[0] = s;
}
int main() {
  long long* d; double* s; cudaMalloc(&d, 64); cudaMalloc(&s, 8);
  int iters = 1000;
  for (int warps : {1, 4, 8, 16}) {
    k<<<1, 32 * warps>>>(iters, d, s);
    long long h[4]; cudaMemcpy(h, d, 32, cudaMemcpyDeviceToHost);
    printf("warps %2d: shfl(double) dep latency %.1f | shfl indep %.2f cyc per double-shfl per warp | drcp+add dep %.1f | sts-syncwarp-lds %.1f\n",
           warps, h[0] / (double)iters, h[1] / (8.0 * iters), h[2] / (double)iters, h[3] / (double)iters);
  }
  return 0;
}
