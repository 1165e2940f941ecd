// Kernel instantiations for the neuron model (models_neuron.cpp; generic kernels only).
#include "cko_inst.cuh"
CKO_INSTANTIATE(neuron, cko::MNeuron)
namespace cko {
cudaError_t fwd2_run_neuron(int, const FwdLaunch* a, cudaStream_t st) {
  (void)a, (void)st;
  return cudaErrorNotSupported;
}
cudaError_t adj2_run_neuron(int, const AdjLaunch* a, cudaStream_t st) {
  (void)a, (void)st;
  return cudaErrorNotSupported;
}
cudaError_t fwdp_run_neuron(int, const FwdLaunch* a, cudaStream_t st) {
  (void)a, (void)st;
  return cudaErrorNotSupported;
}
cudaError_t adjp_run_neuron(int, const AdjLaunch* a, cudaStream_t st) {
  (void)a, (void)st;
  return cudaErrorNotSupported;
}
}  // namespace cko
