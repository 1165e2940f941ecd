// cko_node_vjp.cu — parameter VJP of the wide neural ODE (SURVEY §8d C4,
// W = 128: 18 824 parameters), where the per-thread accumulators of
// vjp_kernel do not fit. The product sum over every (step, lane) point
//   g = sum_p w_p . dh/dp(y_p, t_p)        (ode_model.cpp:135-153)
// factors into outer products of per-point vectors (models_node.cpp:109-151):
//   d3 = w (1 - o^2), d2 = (W3^T d3)(1 - z2^2), d1 = (W2^T d2)(1 - z1^2)
//   gW3 = sum d3 z2^T, gW2 = sum d2 z1^T, gW1 = sum d1 z0^T, gb_l = sum d_l.
// node_vectors_kernel writes the vectors feature-major (x[f * P + p]); the
// sums are split-K GEMMs (outer_partial_kernel, 32 x 32 output tiles, fixed
// K slices) followed by a fixed-order reduction, so the result is
// deterministic.
#include "cko_kernels.cuh"

namespace cko {

namespace {

constexpr int kOuterKS = 64;  // K slices of the split-K outer products
constexpr int kTile = 32;
constexpr int kKc = 64;

__global__ void __launch_bounds__(128) node_vectors_kernel(DevModel m, const double* states, const double* times,
                                                           const double* wq, int nb, int nt, double* vec, size_t P) {
  const int n = m.n, W = m.W, w0 = n + 1;
  const size_t row = (size_t)nb * n;
  const double* W2 = m.p + W * w0 + W;
  const double* W3 = W2 + W * W + W;
  double* Z0 = vec;
  double* Z1 = Z0 + (size_t)w0 * P;
  double* Z2 = Z1 + (size_t)W * P;
  double* D1 = Z2 + (size_t)W * P;
  double* D2 = D1 + (size_t)W * P;
  double* D3 = D2 + (size_t)W * P;
  for (size_t p = blockIdx.x * (size_t)blockDim.x + threadIdx.x; p < P; p += (size_t)gridDim.x * blockDim.x) {
    const int mm = 1 + (int)(p / nb), b = (int)(p % nb);
    const double* y = states + (size_t)mm * row + (size_t)b * n;
    const double* w = wq + (size_t)mm * row + (size_t)b * n;
    double yl[NODE_MAX_N], z0[NODE_MAX_N + 1], z1[NODE_MAX_W], z2[NODE_MAX_W], o[NODE_MAX_N];
    for (int i = 0; i < n; ++i) yl[i] = y[i];
    MNode::forward(m, times[(size_t)mm * nb + b], yl, b, z0, z1, z2, o);
    double d3[NODE_MAX_N], d2[NODE_MAX_W];
    for (int i = 0; i < n; ++i) d3[i] = w[i] * (1.0 - o[i] * o[i]);
    for (int i = 0; i < W; ++i) {
      double acc = 0.0;
      for (int l = 0; l < n; ++l) acc += W3[l * W + i] * d3[l];
      d2[i] = acc * (1.0 - z2[i] * z2[i]);
    }
    for (int i = 0; i < W; ++i) {
      double acc = 0.0;
      for (int l = 0; l < W; ++l) acc += W2[l * W + i] * d2[l];
      D1[(size_t)i * P + p] = acc * (1.0 - z1[i] * z1[i]);
      D2[(size_t)i * P + p] = d2[i];
      Z1[(size_t)i * P + p] = z1[i];
      Z2[(size_t)i * P + p] = z2[i];
    }
    for (int i = 0; i < w0; ++i) Z0[(size_t)i * P + p] = z0[i];
    for (int i = 0; i < n; ++i) D3[(size_t)i * P + p] = d3[i];
  }
}

// partial[ks][i][j] = sum_{p in slice ks} A[i][p] * B[j][p] for a 32 x 32 tile
// (B == nullptr: B[j][p] = 1, the bias column).
__global__ void __launch_bounds__(256) outer_partial_kernel(const double* A, int R, const double* B, int C, size_t P,
                                                            double* partial) {
  __shared__ double sa[kTile][kKc + 1], sb[kTile][kKc + 1];
  const int tilesC = (C + kTile - 1) / kTile;
  const int i0 = (blockIdx.x / tilesC) * kTile, j0 = (blockIdx.x % tilesC) * kTile;
  const int ks = blockIdx.y;
  const size_t per = (P + gridDim.y - 1) / gridDim.y;
  const size_t k0 = per * ks, k1 = min(P, k0 + per);
  const int tx = threadIdx.x % 16, ty = threadIdx.x / 16;  // thread owns rows ty, ty+16 and cols tx, tx+16
  double acc[2][2] = {{0.0, 0.0}, {0.0, 0.0}};
  for (size_t kc = k0; kc < k1; kc += kKc) {
    for (int e = threadIdx.x; e < kTile * kKc; e += blockDim.x) {
      const int r = e / kKc, q = e % kKc;
      const size_t k = kc + q;
      sa[r][q] = (i0 + r < R && k < k1) ? A[(size_t)(i0 + r) * P + k] : 0.0;
      sb[r][q] = (j0 + r < C && k < k1) ? (B ? B[(size_t)(j0 + r) * P + k] : 1.0) : 0.0;
    }
    __syncthreads();
    for (int q = 0; q < kKc; ++q) {
      const double a0 = sa[ty][q], a1 = sa[ty + 16][q], b0 = sb[tx][q], b1 = sb[tx + 16][q];
      acc[0][0] += a0 * b0;
      acc[0][1] += a0 * b1;
      acc[1][0] += a1 * b0;
      acc[1][1] += a1 * b1;
    }
    __syncthreads();
  }
  double* out = partial + ((size_t)ks * R) * C;
  for (int u = 0; u < 2; ++u)
    for (int v = 0; v < 2; ++v) {
      const int i = i0 + ty + 16 * u, j = j0 + tx + 16 * v;
      if (i < R && j < C) out[(size_t)i * C + j] = acc[u][v];
    }
}

// DMMA form of outer_partial_kernel for R, C multiples of 8: a 64 x 64 output
// tile per CTA (four warps of 32 x 32: 4 x 4 fragments of m8n8k4), K staged
// through shared memory 32 points at a time, fixed K slices (deterministic).
constexpr int kDT = 64, kDK = 16, kDKP = kDK + 4;
__device__ __forceinline__ void dmma884(double& c0, double& c1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0, %1}, {%2}, {%3}, {%0, %1};"
               : "+d"(c0), "+d"(c1)
               : "d"(a), "d"(b));
}
__device__ __forceinline__ void stage_tile(double (*sa)[kDKP], double (*sb)[kDKP], const double* A, int R,
                                           const double* B, int C, size_t P, int i0, int j0, size_t kc, size_t k1) {
  // 16-byte cp.async where the whole pair is inside the slice, zero-fill otherwise (rows of A / B are P long)
  for (int e = threadIdx.x; e < kDT * (kDK / 2); e += blockDim.x) {
    const int r = e / (kDK / 2), q = 2 * (e % (kDK / 2));
    const size_t k = kc + q;
    const bool full = k + 1 < k1 && (P % 2 == 0);
    if (i0 + r < R && full) {
      const unsigned s = (unsigned)__cvta_generic_to_shared(&sa[r][q]);
      asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(s), "l"(A + (size_t)(i0 + r) * P + k) : "memory");
    } else {
      sa[r][q] = (i0 + r < R && k < k1) ? A[(size_t)(i0 + r) * P + k] : 0.0;
      sa[r][q + 1] = (i0 + r < R && k + 1 < k1) ? A[(size_t)(i0 + r) * P + k + 1] : 0.0;
    }
    if (j0 + r < C && full) {
      const unsigned s = (unsigned)__cvta_generic_to_shared(&sb[r][q]);
      asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(s), "l"(B + (size_t)(j0 + r) * P + k) : "memory");
    } else {
      sb[r][q] = (j0 + r < C && k < k1) ? B[(size_t)(j0 + r) * P + k] : 0.0;
      sb[r][q + 1] = (j0 + r < C && k + 1 < k1) ? B[(size_t)(j0 + r) * P + k + 1] : 0.0;
    }
  }
  asm volatile("cp.async.commit_group;" ::: "memory");
}

__global__ void __launch_bounds__(128) outer_partial_dmma_kernel(const double* A, int R, const double* B, int C,
                                                                 size_t P, double* partial) {
  __shared__ __align__(16) double sa[2][kDT][kDKP], sb[2][kDT][kDKP];  // double-buffered K stages
  const int tilesC = (C + kDT - 1) / kDT;
  const int i0 = (blockIdx.x / tilesC) * kDT, j0 = (blockIdx.x % tilesC) * kDT;
  const int ks = blockIdx.y;
  size_t per = (P + gridDim.y - 1) / gridDim.y;
  per = (per + 1) & ~(size_t)1;  // even slice starts keep the 16-byte copies aligned
  const size_t k0 = min(P, per * ks), k1 = min(P, k0 + per);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int wr = (warp >> 1) * 32, wc = (warp & 1) * 32;  // warp's 32 x 32 block of the tile
  double acc[4][4][2] = {};
  int buf = 0;
  if (k0 < k1) stage_tile(sa[0], sb[0], A, R, B, C, P, i0, j0, k0, k1);
  for (size_t kc = k0; kc < k1; kc += kDK, buf ^= 1) {
    if (kc + kDK < k1) {
      stage_tile(sa[buf ^ 1], sb[buf ^ 1], A, R, B, C, P, i0, j0, kc + kDK, k1);
      asm volatile("cp.async.wait_group 1;" ::: "memory");
    } else {
      asm volatile("cp.async.wait_group 0;" ::: "memory");
    }
    __syncthreads();
#pragma unroll
    for (int kk = 0; kk < kDK; kk += 4) {
      double av[4], bv[4];
#pragma unroll
      for (int f = 0; f < 4; ++f) {
        av[f] = sa[buf][wr + 8 * f + lane / 4][kk + lane % 4];
        bv[f] = sb[buf][wc + 8 * f + lane / 4][kk + lane % 4];
      }
#pragma unroll
      for (int fr = 0; fr < 4; ++fr)
#pragma unroll
        for (int fc = 0; fc < 4; ++fc) dmma884(acc[fr][fc][0], acc[fr][fc][1], av[fr], bv[fc]);
    }
    __syncthreads();
  }
  double* out = partial + ((size_t)ks * R) * C;
#pragma unroll
  for (int fr = 0; fr < 4; ++fr)
#pragma unroll
    for (int fc = 0; fc < 4; ++fc) {
      const int i = i0 + wr + 8 * fr + lane / 4, j = j0 + wc + 8 * fc + 2 * (lane % 4);
      if (i < R && j < C) out[(size_t)i * C + j] = acc[fr][fc][0];
      if (i < R && j + 1 < C) out[(size_t)i * C + j + 1] = acc[fr][fc][1];
    }
}

__global__ void outer_reduce_kernel(const double* partial, int KS, int R, int C, double* out) {
  for (int e = blockIdx.x * blockDim.x + threadIdx.x; e < R * C; e += gridDim.x * blockDim.x) {
    double s = 0.0;
    for (int ks = 0; ks < KS; ++ks) s += partial[(size_t)ks * R * C + e];
    out[e] = s;
  }
}

cudaError_t outer_sum(const double* A, int R, const double* B, int C, size_t P, double* partial, double* out,
                      cudaStream_t st) {
  if (B && R % 8 == 0 && C % 8 == 0) {  // tensor cores
    const int tiles = ((R + kDT - 1) / kDT) * ((C + kDT - 1) / kDT);
    outer_partial_dmma_kernel<<<dim3(tiles, kOuterKS), 128, 0, st>>>(A, R, B, C, P, partial);
    outer_reduce_kernel<<<(R * C + 255) / 256, 256, 0, st>>>(partial, kOuterKS, R, C, out);
    return cudaGetLastError();
  }
  const int tiles = ((R + kTile - 1) / kTile) * ((C + kTile - 1) / kTile);
  outer_partial_kernel<<<dim3(tiles, kOuterKS), 256, 0, st>>>(A, R, B, C, P, partial);
  outer_reduce_kernel<<<(R * C + 255) / 256, 256, 0, st>>>(partial, kOuterKS, R, C, out);
  return cudaGetLastError();
}

}  // namespace

size_t node_vjp_scratch_doubles(const DevModel& m, int nb, int nt) {
  const size_t P = (size_t)nb * nt;
  const int n = m.n, W = m.W, w0 = n + 1;
  return P * (size_t)(w0 + 4 * W + n) + (size_t)kOuterKS * W * W;
}

cudaError_t launch_node_vjp(const DevModel& m, const double* states, const double* times, const double* wq, int nb,
                            int nt, double* scratch, double* grad, cudaStream_t st) {
  const size_t P = (size_t)nb * nt;
  const int n = m.n, W = m.W, w0 = n + 1;
  double* vec = scratch;
  double* partial = scratch + P * (size_t)(w0 + 4 * W + n);
  if (node_fast_path(m)) {  // C4 shape: the two W x W products per point on the tensor cores (cko_node.cu)
    cudaError_t e = launch_node_vectors_dmma(m, states, times, wq, nb, P, vec, st);
    if (e != cudaSuccess) return e;
  } else {
    node_vectors_kernel<<<4 * 148, 128, 0, st>>>(m, states, times, wq, nb, nt, vec, P);
  }
  const double* Z0 = vec;
  const double* Z1 = Z0 + (size_t)w0 * P;
  const double* Z2 = Z1 + (size_t)W * P;
  const double* D1 = Z2 + (size_t)W * P;
  const double* D2 = D1 + (size_t)W * P;
  const double* D3 = D2 + (size_t)W * P;
  // parameter layout [W1 (W x w0), b1, W2 (W x W), b2, W3 (n x W), b3]
  double* gW1 = grad;
  double* gb1 = gW1 + W * w0;
  double* gW2 = gb1 + W;
  double* gb2 = gW2 + W * W;
  double* gW3 = gb2 + W;
  double* gb3 = gW3 + n * W;
  cudaError_t e;
  if ((e = outer_sum(D1, W, Z0, w0, P, partial, gW1, st)) != cudaSuccess) return e;
  if ((e = outer_sum(D1, W, nullptr, 1, P, partial, gb1, st)) != cudaSuccess) return e;
  if ((e = outer_sum(D2, W, Z1, W, P, partial, gW2, st)) != cudaSuccess) return e;
  if ((e = outer_sum(D2, W, nullptr, 1, P, partial, gb2, st)) != cudaSuccess) return e;
  if ((e = outer_sum(D3, n, Z2, W, P, partial, gW3, st)) != cudaSuccess) return e;
  return outer_sum(D3, n, nullptr, 1, P, partial, gb3, st);
}

}  // namespace cko
