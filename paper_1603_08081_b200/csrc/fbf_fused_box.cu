// fused kernel instantiations for box windows (running-sum passes), radii
// FBF_BOX_LO..FBF_BOX_HI (the Makefile builds two halves of 1..16 in parallel)
#include "fbf_fused.cuh"
#ifndef FBF_BOX_LO
#define FBF_BOX_LO 1
#define FBF_BOX_HI 16
#endif
#if FBF_BOX_LO <= 1 && 1 <= FBF_BOX_HI
FBF_INSTANTIATE_FUSED_BOX(1)
#endif
#if FBF_BOX_LO <= 2 && 2 <= FBF_BOX_HI
FBF_INSTANTIATE_FUSED_BOX(2)
#endif
#if FBF_BOX_LO <= 3 && 3 <= FBF_BOX_HI
FBF_INSTANTIATE_FUSED_BOX(3)
#endif
#if FBF_BOX_LO <= 4 && 4 <= FBF_BOX_HI
FBF_INSTANTIATE_FUSED_BOX(4)
#endif
#if FBF_BOX_LO <= 5 && 5 <= FBF_BOX_HI
FBF_INSTANTIATE_FUSED_BOX(5)
#endif
#if FBF_BOX_LO <= 6 && 6 <= FBF_BOX_HI
FBF_INSTANTIATE_FUSED_BOX(6)
#endif
#if FBF_BOX_LO <= 7 && 7 <= FBF_BOX_HI
FBF_INSTANTIATE_FUSED_BOX(7)
#endif
#if FBF_BOX_LO <= 8 && 8 <= FBF_BOX_HI
FBF_INSTANTIATE_FUSED_BOX(8)
#endif
#if FBF_BOX_LO <= 9 && 9 <= FBF_BOX_HI
FBF_INSTANTIATE_FUSED_BOX(9)
#endif
#if FBF_BOX_LO <= 10 && 10 <= FBF_BOX_HI
FBF_INSTANTIATE_FUSED_BOX(10)
#endif
#if FBF_BOX_LO <= 11 && 11 <= FBF_BOX_HI
FBF_INSTANTIATE_FUSED_BOX(11)
#endif
#if FBF_BOX_LO <= 12 && 12 <= FBF_BOX_HI
FBF_INSTANTIATE_FUSED_BOX(12)
#endif
#if FBF_BOX_LO <= 13 && 13 <= FBF_BOX_HI
FBF_INSTANTIATE_FUSED_BOX(13)
#endif
#if FBF_BOX_LO <= 14 && 14 <= FBF_BOX_HI
FBF_INSTANTIATE_FUSED_BOX(14)
#endif
#if FBF_BOX_LO <= 15 && 15 <= FBF_BOX_HI
FBF_INSTANTIATE_FUSED_BOX(15)
#endif
#if FBF_BOX_LO <= 16 && 16 <= FBF_BOX_HI
FBF_INSTANTIATE_FUSED_BOX(16)
#endif
