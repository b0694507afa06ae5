// fourierbf/kernel_approx.hpp -- drop-in declarations of the host-side
// least-squares cosine fit (reference: proj/include/fourierbf/kernel_approx.hpp:19-234).
// The fit stays on the CPU, as the north star requires.
#pragma once

#include <ostream>
#include <span>
#include <vector>

#include "fourierbf/kernels.hpp"

namespace fourierbf {

/// phi_N(t) = d_0 + sum_{n=1..N} d_n cos(n omega t), omega = pi / T.
struct FourierKernelApprox {
    int T = 0;
    double omega = 0.0;
    int N = 0;
    std::vector<double> d;
    double residual_norm = 0.0;
    double max_pointwise_error = 0;

    double evaluate(double t) const;
    /// c_{-N}..c_N with c_0 = d_0 and c_{+-n} = d_n / 2.
    std::vector<double> complex_coeffs() const;
};

/// Recursive QR of the cosine basis (two-pass modified Gram-Schmidt).
class QrState {
public:
    explicit QrState(std::vector<double> samples);
    bool append_column(std::span<const double> a);
    std::vector<double> solve() const;
    double residual(const std::vector<double>& d, double* max_abs = nullptr) const;

    std::size_t cols() const { return q_.size(); }
    std::size_t rows() const { return b_.size(); }
    const std::vector<std::vector<double>>& basis() const { return a_; }
    const std::vector<std::vector<double>>& orthonormal() const { return q_; }
    const std::vector<std::vector<double>>& triangular() const { return r_; }
    const std::vector<double>& projections() const { return p_; }
    const std::vector<double>& samples() const { return b_; }

private:
    std::vector<double> b_;
    std::vector<std::vector<double>> a_, q_, r_;
    std::vector<double> p_;
};

std::vector<double> sample_kernel(const RangeKernel& kernel, int T);

struct FitStep {
    int order;
    double residual;
    std::vector<double> coeffs;
};
using FitTrace = std::vector<FitStep>;

FourierKernelApprox progressive_fit(std::span<const double> samples, double epsilon,
                                    FitTrace* trace = nullptr);
FourierKernelApprox progressive_fit(const RangeKernel& kernel, int T, double epsilon,
                                    FitTrace* trace = nullptr);
void write_fit_trace_csv(const FitTrace& trace, std::ostream& out);

}  // namespace fourierbf
