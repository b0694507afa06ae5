// fbf_box2.cu -- the small-box-window fused kernel (fbf_box2.cuh), radii 1..7
#include "fbf_box2.cuh"

namespace fbf {

bool box2_supported(int W) { return W >= 1 && W <= kBox2MaxW; }

cudaError_t launch_box2_any(const FusedArgs& a, cudaStream_t st, FusedPlan* plan) {
  switch (a.k.W) {
    case 1: return launch_box2<1>(a, st, plan);
    case 2: return launch_box2<2>(a, st, plan);
    case 3: return launch_box2<3>(a, st, plan);
    case 4: return launch_box2<4>(a, st, plan);
    case 5: return launch_box2<5>(a, st, plan);
    case 6: return launch_box2<6>(a, st, plan);
    case 7: return launch_box2<7>(a, st, plan);
    default: return cudaErrorInvalidValue;
  }
}

}  // namespace fbf
