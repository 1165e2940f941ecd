// Kernel instantiations for the scalar model.
#include "cko_inst.cuh"
CKO_INSTANTIATE(scalar, cko::MScalarDecay)
namespace cko {
cudaError_t fwd2_run_scalar(int n, const FwdLaunch* a, cudaStream_t st) {
  switch (n) {
    case 1: return v2::fwd2_launch<v2::ScalarDecayS>(a, st);
  }
  (void)a, (void)st;
  return cudaErrorNotSupported;
}
cudaError_t adj2_run_scalar(int n, const AdjLaunch* a, cudaStream_t st) {
  switch (n) {
    case 1: return v2::adj2_launch<v2::ScalarDecayS>(a, st);
  }
  (void)a, (void)st;
  return cudaErrorNotSupported;
}
}  // namespace cko
namespace cko {
cudaError_t fwdp_run_scalar(int n, const FwdLaunch* a, cudaStream_t st) {
  switch (n) {
    case 1: return v2::fwd_pcr2_launch<v2::ScalarDecayS>(a, st);
  }
  (void)a, (void)st;
  return cudaErrorNotSupported;
}
cudaError_t adjp_run_scalar(int n, const AdjLaunch* a, cudaStream_t st) {
  switch (n) {
    case 1: return v2::adj_pcr2_launch<v2::ScalarDecayS>(a, st);
  }
  (void)a, (void)st;
  return cudaErrorNotSupported;
}
}  // namespace cko
