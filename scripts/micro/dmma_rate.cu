// DMMA m8n8k4 f64 throughput: independent accumulator chains, all SMs.
#include <cstdio>
__global__ void k(int iters, double* out) {
  const int l = threadIdx.x & 31;
  double a = 1.0 + l * 1e-3, b = 1.0 - l * 1e-3;
  double c[8][2];
  for (int q = 0; q < 8; ++q) c[q][0] = c[q][1] = 0.0;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int q = 0; q < 8; ++q)
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0, %1}, {%2}, {%3}, {%0, %1};"
                   : "+d"(c[q][0]), "+d"(c[q][1]) : "d"(a), "d"(b));
  }
  double s = 0;
  for (int q = 0; q < 8; ++q) s += c[q][0] + c[q][1];
  if (s == 1.2345) out[0] = s;
}
int main() {
  double* o; cudaMalloc(&o, 8);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  for (int warps : {4, 8, 16}) {
    const int iters = 4096, blocks = 148 * 2;
    k<<<blocks, 32 * warps>>>(iters, o);
    cudaEventRecord(e0);
    k<<<blocks, 32 * warps>>>(iters, o);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    double flops = 2.0 * 256 * 8 * (double)iters * blocks * warps;
    printf("warps/CTA %d: %.2f TFLOP/s fp64 DMMA\n", warps, flops / ms / 1e9);
  }
  return 0;
}
