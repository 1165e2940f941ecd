// Kernel instantiations for the lin3 model.
#include "cko_inst.cuh"
CKO_INSTANTIATE(lin3, cko::MLin3)
namespace cko {
cudaError_t fwd2_run_lin3(int n, const FwdLaunch* a, cudaStream_t st) {
  switch (n) {
    case 3: return v2::fwd2_launch<v2::Lin3S>(a, st);
  }
  (void)a, (void)st;
  return cudaErrorNotSupported;
}
cudaError_t adj2_run_lin3(int n, const AdjLaunch* a, cudaStream_t st) {
  switch (n) {
    case 3: return v2::adj2_launch<v2::Lin3S>(a, st);
  }
  (void)a, (void)st;
  return cudaErrorNotSupported;
}
}  // namespace cko
namespace cko {
cudaError_t fwdp_run_lin3(int n, const FwdLaunch* a, cudaStream_t st) {
  switch (n) {
    case 3: return v2::fwd_pcr2_launch<v2::Lin3S>(a, st);
  }
  (void)a, (void)st;
  return cudaErrorNotSupported;
}
cudaError_t adjp_run_lin3(int n, const AdjLaunch* a, cudaStream_t st) {
  switch (n) {
    case 3: return v2::adj_pcr2_launch<v2::Lin3S>(a, st);
  }
  (void)a, (void)st;
  return cudaErrorNotSupported;
}
}  // namespace cko
