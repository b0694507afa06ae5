// fourierbf/bilateral.hpp -- drop-in declarations of the filter entry points
// (reference: proj/include/fourierbf/bilateral.hpp:17-196).  bilateral_fast
// runs on the B200 through the C-ABI in fourierbf_b200.h; there is no CPU
// fallback: without a usable GPU it throws std::runtime_error.
#pragma once

#include <utility>

#include "fourierbf/analysis.hpp"
#include "fourierbf/image.hpp"
#include "fourierbf/kernel_approx.hpp"
#include "fourierbf/kernels.hpp"
#include "fourierbf/spatial.hpp"

namespace fourierbf {

int local_dynamic_range(const Image& image, int W);

/// O(W^2) brute-force filter (the accuracy oracle of the reference API).
Image bilateral_exact(const Image& image, const SpatialKernel& spatial, const RangeKernel& range);

/// Shiftable Fourier-kernel bilateral filter (Algorithm 1), on the GPU.
/// invalid_argument: empty image, or approx.max_pointwise_error >= spatial.w0,
/// runtime_error: "... denominator collapsed at pixel (x, y)".  The recursive
/// backend (Gaussian windows with sigma >= 2) runs the fp64 IIR path on the GPU.
Image bilateral_fast(const Image& image, const SpatialKernel& spatial,
                     const FourierKernelApprox& approx,
                     ConvolutionBackend backend = ConvolutionBackend::direct);

struct FilterConfig {
    SpatialKernel spatial;
    RangeKernel range;
    double epsilon = 1e-3;
    bool integer_intensities = true;
    ConvolutionBackend backend = ConvolutionBackend::direct;
};

std::pair<Image, AccuracyReport> filter(const Image& image, const FilterConfig& config);

}  // namespace fourierbf
