// fused kernel instantiations for box windows (running-sum passes), radii 2..5
#include "fbf_fused.cuh"
FBF_INSTANTIATE_FUSED_BOX(2)
FBF_INSTANTIATE_FUSED_BOX(3)
FBF_INSTANTIATE_FUSED_BOX(4)
FBF_INSTANTIATE_FUSED_BOX(5)
