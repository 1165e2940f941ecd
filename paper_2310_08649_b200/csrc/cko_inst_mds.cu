// Kernel instantiations for the mds model.
#include "cko_inst.cuh"
CKO_INSTANTIATE(mds, cko::MMds)
