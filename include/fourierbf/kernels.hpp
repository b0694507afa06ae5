// fourierbf/kernels.hpp -- drop-in declaration of the range kernel
// (reference: proj/include/fourierbf/kernels.hpp:14-113).
#pragma once

#include <string>
#include <vector>

namespace fourierbf {

enum class RangeFamily { gaussian, exponential, tabulated };

/// Symmetric range kernel phi(|t|) with phi(0) = 1.
class RangeKernel {
public:
    static RangeKernel gaussian(double sigma_r);
    static RangeKernel exponential(double sigma_r);
    static RangeKernel tabulated(std::vector<double> table);
    static RangeKernel tabulated_from_file(const std::string& path);

    double eval(double t) const;

    RangeFamily family() const { return family_; }
    double sigma_r() const { return sigma_r_; }
    const std::vector<double>& table() const { return table_; }

private:
    RangeKernel() = default;
    RangeFamily family_ = RangeFamily::gaussian;
    double sigma_r_ = 0.0;
    std::vector<double> table_;
};

}  // namespace fourierbf
