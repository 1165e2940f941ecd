// Dependent-chain latency of DFMA / DMUL / DADD and of an LDS round trip on one warp (clock64).
#include <cstdio>
__global__ void lat(double* out, long long* cyc, double a, double b, int n) {
  __shared__ double sm[64];
  sm[threadIdx.x] = a;
  __syncwarp();
  double x = a, y = b;
  long long t0 = clock64();
  for (int i = 0; i < n; ++i) x = fma(x, y, a);
  long long t1 = clock64();
  for (int i = 0; i < n; ++i) x = x * y;
  long long t2 = clock64();
  for (int i = 0; i < n; ++i) x = x + y;
  long long t3 = clock64();
  int idx = (int)x & 0;
  for (int i = 0; i < n; ++i) idx = (int)sm[idx + (threadIdx.x & 0)] & 0;
  long long t4 = clock64();
  out[threadIdx.x] = x + idx;
  if (threadIdx.x == 0) cyc[0] = t1 - t0, cyc[1] = t2 - t1, cyc[2] = t3 - t2, cyc[3] = t4 - t3;
}
int main() {
  double* o; long long* c; cudaMalloc(&o, 256); cudaMallocManaged(&c, 64);
  const int n = 4096;
  for (int r = 0; r < 2; ++r) { lat<<<1, 32>>>(o, c, 0.999999, 1.0000001, n); cudaDeviceSynchronize(); }
  printf("cycles per dependent op: DFMA %.2f DMUL %.2f DADD %.2f LDS+cvt %.2f\n", c[0] / (double)n, c[1] / (double)n,
         c[2] / (double)n, c[3] / (double)n);
  return 0;
}
