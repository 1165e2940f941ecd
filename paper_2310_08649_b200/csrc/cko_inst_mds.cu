// Kernel instantiations for the mds model.
#include "cko_inst.cuh"
#include "cko_pcrw.cuh"
CKO_INSTANTIATE(mds, cko::MMds)
namespace cko {
cudaError_t fwd2_run_mds(int n, const FwdLaunch* a, cudaStream_t st) {
  switch (n) {
    case 20: return v2::fwd2_launch<v2::MdsS<10>>(a, st);
    case 4: return v2::fwd2_launch<v2::MdsS<2>>(a, st);
  }
  (void)a, (void)st;
  return cudaErrorNotSupported;
}
cudaError_t adj2_run_mds(int n, const AdjLaunch* a, cudaStream_t st) {
  switch (n) {
    case 20: return v2::adj2_launch<v2::MdsS<10>>(a, st);
    case 4: return v2::adj2_launch<v2::MdsS<2>>(a, st);
  }
  (void)a, (void)st;
  return cudaErrorNotSupported;
}
}  // namespace cko
namespace cko {
cudaError_t fwdp_run_mds(int n, const FwdLaunch* a, cudaStream_t st) {
  switch (n) {
    case 20: return v2::fwd_pcrw_launch<v2::MdsS<10>>(a, st);
    case 4: return v2::fwd_pcr2_launch<v2::MdsS<2>>(a, st);
  }
  (void)a, (void)st;
  return cudaErrorNotSupported;
}
cudaError_t adjp_run_mds(int n, const AdjLaunch* a, cudaStream_t st) {
  switch (n) {
    case 20: return v2::adj_pcrw_launch<v2::MdsS<10>>(a, st);
    case 4: return v2::adj_pcr2_launch<v2::MdsS<2>>(a, st);
  }
  (void)a, (void)st;
  return cudaErrorNotSupported;
}
}  // namespace cko
namespace cko {
// Parameter VJP of the MDS chain at compile-time size (models_mds.cpp:84-113, same per-point expressions as
// MMds::vjp). Thread per lane, steps inner: the 3 (NU - 1) + 1 shared accumulators and the lane's T_b sum
// stay in registers; only w[NU..2NU) of the adjoint row is read (248 B per point at NU = 10). One row of
// `part` per block, summed by vjp_final_kernel in a fixed order (deterministic).
#ifndef CKO_VJP_MINB
#define CKO_VJP_MINB 2
#endif
template <int NU>
__global__ void __launch_bounds__(256, CKO_VJP_MINB)
    vjp_mds_kernel(DevModel m, const double* states, const double* times, const double* wq, int nb, int nt,
                   double* part) {
  constexpr int N = 2 * NU, NA = 3 * (NU - 1) + 1;
  __shared__ double red[8][NA];
  __shared__ double prm[3 * NU + 1];
  const int tid = threadIdx.x, T = blockDim.x;
  double* prow = part + (size_t)blockIdx.x * m.np;
  for (int j = tid; j < m.np; j += T) prow[j] = 0.0;
  for (int j = tid; j < 3 * NU + 1; j += T) prm[j] = m.p[j];
  __syncthreads();
  const double* K = prm;
  const double* C = prm + NU;
  const double* M = prm + 2 * NU;
  const double fa = prm[3 * NU];
  // x / M_j, x / M_j^2 and x / T_b from correctly rounded reciprocals plus one remainder correction
  // (v2::div_rn, Markstein): the quotients without the divide sequence
  double rM[NU], M2[NU], rM2[NU];
#pragma unroll
  for (int j = 1; j < NU; ++j) rM[j] = 1.0 / M[j], M2[j] = M[j] * M[j], rM2[j] = 1.0 / M2[j];
  double acc[NA];
#pragma unroll
  for (int q = 0; q < NA; ++q) acc[q] = 0.0;
  const size_t row = (size_t)nb * N;
  for (int b = tid; b < nb; b += T) {
    const double Tb = m.p[3 * NU + 1 + m.off + b];
    const double rTb = 1.0 / Tb;
    double gT = 0.0;
    for (int mm = 1 + blockIdx.x; mm <= nt; mm += gridDim.x) {
      const double* y = states + (size_t)mm * row + (size_t)b * N;
      const double* w = wq + (size_t)mm * row + (size_t)b * N + NU;
      double yv[N], wv[NU];
#pragma unroll
      for (int q = 0; q < N; q += 2) {
        const double2 v = __ldcs(reinterpret_cast<const double2*>(y + q));
        yv[q] = v.x, yv[q + 1] = v.y;
      }
#pragma unroll
      for (int q = 0; q < NU; q += 2) {
        const double2 v = __ldcs(reinterpret_cast<const double2*>(w + q));
        wv[q] = v.x, wv[q + 1] = v.y;
      }
      const double t = __ldcs(times + (size_t)mm * nb + b);
#pragma unroll
      for (int j = 1; j < NU; ++j) {
        const double om = wv[j] - wv[j - 1];
        const double dd = yv[j] - yv[j - 1], dv = yv[NU + j] - yv[NU + j - 1];
        acc[3 * (j - 1)] += v2::div_rn(om * dd, M[j], rM[j]);
        acc[3 * (j - 1) + 1] += v2::div_rn(om * dv, M[j], rM[j]);
        acc[3 * (j - 1) + 2] += -v2::div_rn(om * (K[j] * dd + C[j] * dv), M2[j], rM2[j]);
      }
      const double ph = v2::div_rn(CKO_TWO_PI * t, Tb, rTb);
      double s, c;
      sincos(ph, &s, &c);
      acc[NA - 1] += wv[0] * s;
      gT += wv[0] * fa * c * (-v2::div_rn(ph, Tb, rTb));
    }
    prow[3 * NU + 1 + m.off + b] = gT;
  }
  const int warp = tid / 32, lane = tid % 32, nw = T / 32;
#pragma unroll
  for (int q = 0; q < NA; ++q) {
    double v = acc[q];
    for (int o = 16; o > 0; o >>= 1) v += __shfl_down_sync(0xffffffffu, v, o);
    if (lane == 0) red[warp][q] = v;
  }
  __syncthreads();
  for (int q = tid; q < NA; q += T) {
    double s = 0.0;
    for (int k = 0; k < nw; ++k) s += red[k][q];
    const int j = q / 3 + 1;  // q = 3 (j - 1) + {0: K_j, 1: C_j, 2: M_j}; q = NA - 1: f_a
    prow[q == NA - 1 ? 3 * NU : (q % 3) * NU + j] = s;
  }
}

cudaError_t vjp_static_mds(const DevModel& m, const double* states, const double* times, const double* wq, int nb,
                           int nt, double* scratch, cudaStream_t st) {
#if CKO_VJP_GENERIC
  return cudaErrorNotSupported;  // A/B switch: the generic MMds kernel
#endif
  switch (m.nu) {
    case 10: vjp_mds_kernel<10><<<kVjpBlocks, 256, 0, st>>>(m, states, times, wq, nb, nt, scratch); break;
    case 2: vjp_mds_kernel<2><<<kVjpBlocks, 256, 0, st>>>(m, states, times, wq, nb, nt, scratch); break;
    default: return cudaErrorNotSupported;
  }
  return cudaGetLastError();
}
}  // namespace cko
