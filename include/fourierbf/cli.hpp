// fourierbf/cli.hpp -- drop-in declarations of the command-line driver
// (reference: proj/include/fourierbf/cli.hpp:24-142).  run() reads a PGM,
// filters it with filter() -- the B200 pipeline: device dynamic range, host
// QR fit, fused GPU kernel -- and writes the result and an optional
// key=value report; --bench times bilateral_fast (GPU, host buffers in and
// out) over the reference's sigma_s / sigma_r sweeps as CSV on `out`.
#pragma once
#include <ostream>
#include <string>

#include "fourierbf/kernels.hpp"
#include "fourierbf/spatial.hpp"

namespace fourierbf {

struct CliOptions {
    std::string input_path;
    std::string output_path;
    double sigma_s = 0.0;
    double sigma_r = 0.0;
    RangeFamily kernel_family = RangeFamily::gaussian;
    std::string tabulated_path;  ///< used when kernel_family is tabulated
    double epsilon = 1e-3;
    SpatialKind spatial_kind = SpatialKind::gaussian;
    ConvolutionBackend backend = ConvolutionBackend::direct;
    bool compare_exact = false;  ///< also run bilateral_exact (GPU, fp64) and report measured_linf
    std::string report_path;
    bool bench = false;
};

/// One CLI invocation: 0 on success; on failure "error: <what>" on `err` and 1.
/// `out` receives the --bench CSV only.
int run(const CliOptions& opt, std::ostream& out, std::ostream& err);

}  // namespace fourierbf
