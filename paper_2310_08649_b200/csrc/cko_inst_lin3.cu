// Kernel instantiations for the lin3 model.
#include "cko_inst.cuh"
CKO_INSTANTIATE(lin3, cko::MLin3)
