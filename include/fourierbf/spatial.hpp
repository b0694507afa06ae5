// fourierbf/spatial.hpp -- drop-in declarations for the spatial window and the
// separable convolution (reference: proj/include/fourierbf/spatial.hpp:12-112).
// convolve() runs on the B200 (fbf_convolve_* in fourierbf_b200.h).
#pragma once

#include <vector>

#include "fourierbf/image.hpp"

namespace fourierbf {

enum class SpatialKind { gaussian, box };

enum class ConvolutionBackend {
    direct,     ///< separable FIR (the B200 path)
    recursive,  ///< third-order IIR Gaussian for Gaussian windows with sigma >= 2 (GPU, fp64)
};

/// Separable symmetric window on [-W, W]^2 with a unit-sum 1-D profile.
struct SpatialKernel {
    SpatialKind kind = SpatialKind::gaussian;
    double sigma_s = 0.0;
    int radius = 1;
    std::vector<double> profile;
    double w0 = 0.0;

    double weight(int dx, int dy) const {
        return profile[static_cast<std::size_t>(dx + radius)] *
               profile[static_cast<std::size_t>(dy + radius)];
    }
};

/// W = ceil(3 sigma_s), renormalised taps; throws invalid_argument for sigma_s <= 0.
SpatialKernel make_spatial_gaussian(double sigma_s);
/// 1/(2W+1) taps; throws invalid_argument for radius < 1.
SpatialKernel make_spatial_box(int radius);

using Plane = Image;

/// Mirror-boundary separable convolution on the GPU; invalid_argument on an
/// empty plane.  The recursive backend (Gaussian, sigma >= 2) runs the IIR.
Plane convolve(const Plane& plane, const SpatialKernel& kernel,
               ConvolutionBackend backend = ConvolutionBackend::direct);

}  // namespace fourierbf
