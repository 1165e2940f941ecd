// Kernel instantiations for the node model.
#include "cko_inst.cuh"
CKO_INSTANTIATE(node, cko::MNode)
