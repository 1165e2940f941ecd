// Kernel instantiations for the scalar model.
#include "cko_inst.cuh"
CKO_INSTANTIATE(scalar, cko::MScalarDecay)
