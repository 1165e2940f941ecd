// Verify the mma.sync m8n8k4 f64 fragment layout on sm_100a:
//  A (8x4 row): lane l holds A[l/4][l%4]; B (4x8 col): lane l holds B[l%4][l/4];
//  C/D (8x8): lane l holds C[l/4][2(l%4)] and C[l/4][2(l%4)+1].
#include <cstdio>
__global__ void k(const double* A, const double* B, double* C) {
  const int l = threadIdx.x;
  double a = A[(l / 4) * 4 + (l % 4)];
  double b = B[(l % 4) * 8 + (l / 4)];
  double c0 = 0.0, c1 = 0.0;
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0, %1}, {%2}, {%3}, {%0, %1};"
               : "+d"(c0), "+d"(c1) : "d"(a), "d"(b));
  C[(l / 4) * 8 + 2 * (l % 4)] = c0;
  C[(l / 4) * 8 + 2 * (l % 4) + 1] = c1;
}
int main() {
  double hA[32], hB[32], hC[64], ref[64];
  for (int i = 0; i < 32; ++i) hA[i] = 0.1 * i + 1, hB[i] = 0.01 * i - 0.2;
  for (int i = 0; i < 8; ++i)
    for (int j = 0; j < 8; ++j) {
      double s = 0;
      for (int q = 0; q < 4; ++q) s += hA[i * 4 + q] * hB[q * 8 + j];
      ref[i * 8 + j] = s;
    }
  double *A, *B, *C;
  cudaMalloc(&A, 256); cudaMalloc(&B, 256); cudaMalloc(&C, 512);
  cudaMemcpy(A, hA, 256, cudaMemcpyHostToDevice);
  cudaMemcpy(B, hB, 256, cudaMemcpyHostToDevice);
  k<<<1, 32>>>(A, B, C);
  cudaMemcpy(hC, C, 512, cudaMemcpyDeviceToHost);
  double err = 0;
  for (int i = 0; i < 64; ++i) err = fmax(err, fabs(hC[i] - ref[i]));
  printf("dmma m8n8k4 layout max err %g (%s)\n", err, cudaGetErrorString(cudaGetLastError()));
  return 0;
}
