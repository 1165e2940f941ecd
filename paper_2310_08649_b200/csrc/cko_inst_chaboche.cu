// Kernel instantiations for the chaboche model.
#include "cko_inst.cuh"
CKO_INSTANTIATE(chaboche, cko::MChaboche)
namespace cko {
cudaError_t fwd2_run_chaboche(int n, const FwdLaunch* a, cudaStream_t st) {
  switch (n) {
    case 5: return v2::fwd2_launch<v2::ChabS<3>>(a, st);
    case 4: return v2::fwd2_launch<v2::ChabS<2>>(a, st);
    case 3: return v2::fwd2_launch<v2::ChabS<1>>(a, st);
  }
  (void)a, (void)st;
  return cudaErrorNotSupported;
}
cudaError_t adj2_run_chaboche(int n, const AdjLaunch* a, cudaStream_t st) {
  switch (n) {
    case 5: return v2::adj2_launch<v2::ChabS<3>>(a, st);
    case 4: return v2::adj2_launch<v2::ChabS<2>>(a, st);
    case 3: return v2::adj2_launch<v2::ChabS<1>>(a, st);
  }
  (void)a, (void)st;
  return cudaErrorNotSupported;
}
}  // namespace cko
namespace cko {
cudaError_t fwdp_run_chaboche(int n, const FwdLaunch* a, cudaStream_t st) {
  switch (n) {
    case 5: return v2::fwd_pcr2_launch<v2::ChabS<3>>(a, st);
    case 4: return v2::fwd_pcr2_launch<v2::ChabS<2>>(a, st);
    case 3: return v2::fwd_pcr2_launch<v2::ChabS<1>>(a, st);
  }
  (void)a, (void)st;
  return cudaErrorNotSupported;
}
cudaError_t adjp_run_chaboche(int n, const AdjLaunch* a, cudaStream_t st) {
  switch (n) {
    case 5: return v2::adj_pcr2_launch<v2::ChabS<3>>(a, st);
    case 4: return v2::adj_pcr2_launch<v2::ChabS<2>>(a, st);
    case 3: return v2::adj_pcr2_launch<v2::ChabS<1>>(a, st);
  }
  (void)a, (void)st;
  return cudaErrorNotSupported;
}
}  // namespace cko
