// Kernel instantiations for the node model.
#include "cko_inst.cuh"
CKO_INSTANTIATE(node, cko::MNode)
namespace cko {
cudaError_t fwd2_run_node(int n, const FwdLaunch* a, cudaStream_t st) {
  switch (n) {

  }
  (void)a, (void)st;
  return cudaErrorNotSupported;
}
cudaError_t adj2_run_node(int n, const AdjLaunch* a, cudaStream_t st) {
  switch (n) {

  }
  (void)a, (void)st;
  return cudaErrorNotSupported;
}
}  // namespace cko
namespace cko {
cudaError_t fwdp_run_node(int n, const FwdLaunch* a, cudaStream_t st) {
  switch (n) {

  }
  (void)a, (void)st;
  return cudaErrorNotSupported;
}
cudaError_t adjp_run_node(int n, const AdjLaunch* a, cudaStream_t st) {
  switch (n) {

  }
  (void)a, (void)st;
  return cudaErrorNotSupported;
}
}  // namespace cko
