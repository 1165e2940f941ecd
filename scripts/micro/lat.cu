// Micro-benchmarks: DFMA dependent latency, DFMA issue rate of one warp, LDS latency.
#include <cstdio>
__global__ void k(int iters, long long* out, double* sink) {
  __shared__ double sm[1024];
  for (int i = threadIdx.x; i < 1024; i += blockDim.x) sm[i] = (i * 7) % 1024;
  __syncthreads();
  double a = threadIdx.x * 1e-3, b = 1.000001, c = 1e-9;
  long long t0 = clock64();
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int u = 0; u < 16; ++u) a = fma(a, b, c);
  }
  long long t1 = clock64();
  double x[8];
  for (int q = 0; q < 8; ++q) x[q] = a + q;
  long long t2 = clock64();
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int u = 0; u < 4; ++u)
#pragma unroll
      for (int q = 0; q < 8; ++q) x[q] = fma(x[q], b, c);
  }
  long long t3 = clock64();
  int idx = threadIdx.x;
  long long t4 = clock64();
  for (int i = 0; i < iters * 16; ++i) idx = (int)sm[idx & 1023];
  long long t5 = clock64();
  if (threadIdx.x == 0) {
    out[0] = t1 - t0; out[1] = t3 - t2; out[2] = t5 - t4;
  }
  double s = a + idx;
  for (int q = 0; q < 8; ++q) s += x[q];
  if (s == 1.2345) sink[0] = s;
}
int main() {
  long long* d; double* s; cudaMalloc(&d, 64); cudaMalloc(&s, 8);
  int iters = 1000;
  k<<<1, 32>>>(iters, d, s);
  long long h[3]; cudaMemcpy(h, d, 24, cudaMemcpyDeviceToHost);
  printf("DFMA dependent latency: %.2f cycles\n", h[0] / (16.0 * iters));
  printf("DFMA one-warp independent (8 chains): %.2f cycles per DFMA instr\n", h[1] / (32.0 * iters));
  printf("LDS dependent latency (incl cvt): %.2f cycles\n", h[2] / (16.0 * iters));
  k<<<1, 7>>>(iters, d, s);
  cudaMemcpy(h, d, 24, cudaMemcpyDeviceToHost);
  printf("[7 threads] DFMA dep %.2f, indep %.2f per instr\n", h[0] / (16.0 * iters), h[1] / (32.0 * iters));
  return 0;
}
