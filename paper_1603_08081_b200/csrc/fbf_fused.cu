// fbf_fused.cu -- radius dispatch for the fused kernel (instantiations live in
// fbf_fused_w<W>.cu, one translation unit per radius).
#include "fbf_fused.cuh"

namespace fbf {

extern template cudaError_t launch_w<3>(const FusedArgs&, cudaStream_t, int*);
extern template cudaError_t launch_w<5>(const FusedArgs&, cudaStream_t, int*);
extern template cudaError_t launch_w<6>(const FusedArgs&, cudaStream_t, int*);
extern template cudaError_t launch_w<8>(const FusedArgs&, cudaStream_t, int*);
extern template cudaError_t launch_w<9>(const FusedArgs&, cudaStream_t, int*);
extern template cudaError_t launch_w<12>(const FusedArgs&, cudaStream_t, int*);
extern template cudaError_t launch_w<15>(const FusedArgs&, cudaStream_t, int*);
extern template cudaError_t launch_w<24>(const FusedArgs&, cudaStream_t, int*);

// Radii with a compiled fused kernel (the BASELINE configs' W=5,9,12,15,24 and
// the reference tests' W=3,6,8).  Other radii take the naive multi-kernel path.
bool fused_supported(int W) {
  switch (W) {
    case 3: case 5: case 6: case 8: case 9: case 12: case 15: case 24:
      return true;
    default:
      return false;
  }
}

cudaError_t launch_fused(const FusedArgs& a, cudaStream_t st, int* grid_out) {
  switch (a.k.W) {
    case 3: return launch_w<3>(a, st, grid_out);
    case 5: return launch_w<5>(a, st, grid_out);
    case 6: return launch_w<6>(a, st, grid_out);
    case 8: return launch_w<8>(a, st, grid_out);
    case 9: return launch_w<9>(a, st, grid_out);
    case 12: return launch_w<12>(a, st, grid_out);
    case 15: return launch_w<15>(a, st, grid_out);
    case 24: return launch_w<24>(a, st, grid_out);
    default: return cudaErrorInvalidValue;
  }
}

}  // namespace fbf
