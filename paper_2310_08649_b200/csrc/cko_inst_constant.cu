// Kernel instantiations for the constant model.
#include "cko_inst.cuh"
CKO_INSTANTIATE(constant, cko::MConstantRate)
