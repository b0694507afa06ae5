// fused kernel instantiation for one Gaussian spatial radius W = FBF_W
// (compiled once per radius by the Makefile, -DFBF_W=<W>: parallel builds)
#include "fbf_fused.cuh"
#ifndef FBF_W
#error "compile with -DFBF_W=<radius>"
#endif
FBF_INSTANTIATE_FUSED(FBF_W)
