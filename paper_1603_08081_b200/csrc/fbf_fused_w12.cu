// fused kernel instantiation for spatial radius W=12 (one TU per radius: parallel builds)
#include "fbf_fused.cuh"
FBF_INSTANTIATE_FUSED(12)
