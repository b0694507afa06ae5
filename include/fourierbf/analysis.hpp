// fourierbf/analysis.hpp -- drop-in declarations of the accuracy helpers
// (reference: proj/include/fourierbf/analysis.hpp:25-105).
#pragma once

#include <optional>
#include <ostream>
#include <string>

#include "fourierbf/image.hpp"

namespace fourierbf {

/// 2 T eps / (w0 - eps); invalid_argument unless 0 <= eps < w0 and T >= 0.
double error_bound(int T, double epsilon, double w0);
double linf_error(const Image& a, const Image& b);

struct AccuracyReport {
    int T = 0;
    double epsilon_requested = 0.0;
    double epsilon_achieved = 0.0;
    std::optional<int> N;
    double w0 = 0.0;
    double predicted_bound = 0.0;
    std::optional<double> measured_linf;
    bool weaker_guarantee_flag = false;

    void write_key_values(std::ostream& os) const;
    static std::string csv_header();
    std::string csv_row() const;
};

AccuracyReport make_report(int T, double epsilon_requested, double epsilon_achieved,
                           std::optional<int> N, double w0, bool weaker_guarantee);

}  // namespace fourierbf
