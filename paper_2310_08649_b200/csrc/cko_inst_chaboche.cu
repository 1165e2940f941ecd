// Kernel instantiations for the chaboche model.
#include "cko_inst.cuh"
CKO_INSTANTIATE(chaboche, cko::MChaboche)
