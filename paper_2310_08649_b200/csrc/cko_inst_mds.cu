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
