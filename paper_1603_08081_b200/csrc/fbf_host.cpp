// fbf_host.cpp -- host side of the B200 build.
//
//  * the reference's C++ API (include/fourierbf/*.hpp), re-implemented: the
//    range kernels, the recursive-QR cosine fit, the accuracy helpers and the
//    filter pipeline stay on the CPU (north star: "the coefficient fit stays in
//    host C++"); bilateral_fast and convolve call the CUDA path through the
//    C-ABI (fourierbf_b200.h).  There is no CPU fallback for either.
//  * the host-only C-ABI entry points (fit, spatial taps, synthetic images).
#include <algorithm>
#include <cmath>
#include <cstdint>
#include <cstdio>
#include <fstream>
#include <limits>
#include <numbers>
#include <sstream>
#include <stdexcept>
#include <string>
#include <thread>
#include <vector>

#include "fourierbf/fourierbf.hpp"
#include "fourierbf_b200.h"

namespace fourierbf {

// ------------------------------------------------------------------ image.hpp

Image::Image(int w, int h, double fill) : width(w), height(h) {
    if (w < 1 || h < 1) throw std::invalid_argument("Image: dimensions must be positive");
    values.assign(static_cast<std::size_t>(w) * static_cast<std::size_t>(h), fill);
}

int mirror_index(int i, int n) {
    if (i >= 0 && i < n) return i;
    const int two_n = 2 * n;
    int k = i % two_n;
    if (k < 0) k += two_n;
    return k < n ? k : two_n - 1 - k;
}

Image round_to_integers(const Image& img) {
    Image out = img;
    std::transform(out.values.begin(), out.values.end(), out.values.begin(),
                   [](double v) { return std::floor(v + 0.5); });
    return out;
}

Image mirror_horizontal(const Image& img) {
    Image out(img.width, img.height);
    for (int y = 0; y < img.height; ++y)
        std::reverse_copy(img.values.begin() + static_cast<long>(y) * img.width,
                          img.values.begin() + static_cast<long>(y + 1) * img.width,
                          out.values.begin() + static_cast<long>(y) * img.width);
    return out;
}

Image mirror_vertical(const Image& img) {
    Image out(img.width, img.height);
    for (int y = 0; y < img.height; ++y)
        std::copy_n(img.values.begin() + static_cast<long>(img.height - 1 - y) * img.width,
                    img.width, out.values.begin() + static_cast<long>(y) * img.width);
    return out;
}

// ---------------------------------------------------------------- spatial.hpp

SpatialKernel make_spatial_gaussian(double sigma_s) {
    SpatialKernel k;
    k.kind = SpatialKind::gaussian;
    k.sigma_s = sigma_s;
    int radius = 0;
    if (fbf_spatial_gaussian(sigma_s, nullptr, &radius, nullptr) != FBF_OK)
        throw std::invalid_argument("spatial sigma must be positive");
    k.profile.assign(static_cast<std::size_t>(2 * radius + 1), 0.0);
    fbf_spatial_gaussian(sigma_s, k.profile.data(), &k.radius, &k.w0);
    return k;
}

SpatialKernel make_spatial_box(int radius) {
    if (radius < 1) throw std::invalid_argument("box radius must be at least 1");
    SpatialKernel k;
    k.kind = SpatialKind::box;
    k.radius = radius;
    k.profile.assign(static_cast<std::size_t>(2 * radius + 1), 0.0);
    fbf_spatial_box(radius, k.profile.data(), &k.w0);
    return k;
}

namespace {

[[noreturn]] void rethrow_status(int rc) {
    const std::string msg = fbf_last_error();
    if (rc == FBF_EINVAL) throw std::invalid_argument(msg);
    throw std::runtime_error(msg);
}

// The reference's recursive backend substitutes an IIR Gaussian only for a
// Gaussian window with sigma >= 2 (spatial.hpp:103-105); everything else is
// the direct path.  Both run on the GPU (the IIR in fp64, csrc/fbf_iir.cu).
bool uses_iir(const SpatialKernel& k, ConvolutionBackend backend) {
    return backend == ConvolutionBackend::recursive && k.kind == SpatialKind::gaussian && k.sigma_s >= 2.0;
}

}  // namespace

Plane convolve(const Plane& plane, const SpatialKernel& kernel, ConvolutionBackend backend) {
    if (plane.width <= 0 || plane.height <= 0) throw std::invalid_argument("convolve: empty plane");
    Plane out(plane.width, plane.height);
    const int rc = uses_iir(kernel, backend)
                       ? fbf_convolve_recursive_host_f64(plane.width, plane.height, kernel.sigma_s,
                                                         plane.values.data(), out.values.data())
                       : fbf_convolve_host_f64(plane.width, plane.height, kernel.profile.data(), kernel.radius,
                                               plane.values.data(), out.values.data());
    if (rc != FBF_OK) rethrow_status(rc);
    return out;
}

// ---------------------------------------------------------------- kernels.hpp

RangeKernel RangeKernel::gaussian(double sigma_r) {
    if (!(sigma_r > 0.0)) throw std::invalid_argument("RangeKernel: sigma_r must be positive");
    RangeKernel k;
    k.family_ = RangeFamily::gaussian;
    k.sigma_r_ = sigma_r;
    return k;
}

RangeKernel RangeKernel::exponential(double sigma_r) {
    if (!(sigma_r > 0.0)) throw std::invalid_argument("RangeKernel: sigma_r must be positive");
    RangeKernel k;
    k.family_ = RangeFamily::exponential;
    k.sigma_r_ = sigma_r;
    return k;
}

RangeKernel RangeKernel::tabulated(std::vector<double> table) {
    if (table.empty()) throw std::invalid_argument("RangeKernel: table must not be empty");
    if (table.front() != 1.0) throw std::invalid_argument("RangeKernel: table[0] must equal 1.0");
    for (std::size_t t = 0; t < table.size(); ++t)
        if (!(table[t] >= 0.0 && table[t] <= 1.0))
            throw std::invalid_argument("RangeKernel: table values must lie in [0,1] (line " +
                                        std::to_string(t + 1) + ")");
    RangeKernel k;
    k.family_ = RangeFamily::tabulated;
    k.table_ = std::move(table);
    return k;
}

RangeKernel RangeKernel::tabulated_from_file(const std::string& path) {
    std::ifstream in(path);
    if (!in) throw std::runtime_error("RangeKernel: cannot open '" + path + "'");
    std::vector<double> table;
    std::string line;
    for (std::size_t lineno = 1; std::getline(in, line); ++lineno) {
        if (line.find_first_not_of(" \t\r") == std::string::npos) continue;
        std::istringstream ls(line);
        double v;
        if (!(ls >> v))
            throw std::runtime_error("RangeKernel: '" + path + "' line " + std::to_string(lineno) +
                                     ": not a number");
        table.push_back(v);
    }
    if (table.empty()) throw std::runtime_error("RangeKernel: '" + path + "' contains no samples");
    return tabulated(std::move(table));
}

double RangeKernel::eval(double t) const {
    const double a = std::abs(t);
    if (family_ == RangeFamily::tabulated) {
        const long long idx = std::llround(a);
        if (idx >= static_cast<long long>(table_.size()))
            throw std::out_of_range("RangeKernel: |t|=" + std::to_string(a) +
                                    " outside table of size " + std::to_string(table_.size()));
        return table_[static_cast<std::size_t>(idx)];
    }
    return fbf_range_eval(family_ == RangeFamily::exponential ? FBF_RANGE_EXPONENTIAL
                                                              : FBF_RANGE_GAUSSIAN,
                          sigma_r_, a);
}

// ---------------------------------------------------------- kernel_approx.hpp

double FourierKernelApprox::evaluate(double t) const {
    double acc = d[0];
    for (int n = 1; n <= N; ++n) acc += d[static_cast<std::size_t>(n)] * std::cos(n * omega * t);
    return acc;
}

std::vector<double> FourierKernelApprox::complex_coeffs() const {
    std::vector<double> c(2 * static_cast<std::size_t>(N) + 1, 0.0);
    c[static_cast<std::size_t>(N)] = d[0];
    for (int n = 1; n <= N; ++n)
        c[static_cast<std::size_t>(N - n)] = c[static_cast<std::size_t>(N + n)] =
            0.5 * d[static_cast<std::size_t>(n)];
    return c;
}

namespace {

double inner(const std::vector<double>& x, const std::vector<double>& y) {
    double s = 0.0;
    for (std::size_t i = 0; i < x.size(); ++i) s += x[i] * y[i];
    return s;
}

double length(std::span<const double> x) {
    double s = 0.0;
    for (double v : x) s += v * v;
    return std::sqrt(s);
}

}  // namespace

QrState::QrState(std::vector<double> samples) : b_(std::move(samples)) {
    if (b_.size() < 2) throw std::invalid_argument("QrState: need at least two samples");
    const double m = static_cast<double>(b_.size());
    a_.emplace_back(b_.size(), 1.0);
    q_.emplace_back(b_.size(), 1.0 / std::sqrt(m));
    r_.push_back({std::sqrt(m)});
    p_.push_back(inner(q_.back(), b_));
}

bool QrState::append_column(std::span<const double> a) {
    if (a.size() != b_.size()) throw std::invalid_argument("QrState: column length mismatch");
    std::vector<double> v(a.begin(), a.end());
    std::vector<double> coef(q_.size(), 0.0);
    // classical "twice is enough": two modified Gram-Schmidt sweeps
    for (int sweep = 0; sweep < 2; ++sweep)
        for (std::size_t j = 0; j < q_.size(); ++j) {
            const double s = inner(v, q_[j]);
            for (std::size_t t = 0; t < v.size(); ++t) v[t] += -s * q_[j][t];
            coef[j] += s;
        }
    const double nv = length(v);
    if (nv < 1e-12 * length(a)) return false;
    for (double& x : v) x /= nv;
    coef.push_back(nv);
    a_.emplace_back(a.begin(), a.end());
    p_.push_back(inner(v, b_));
    q_.push_back(std::move(v));
    r_.push_back(std::move(coef));
    return true;
}

std::vector<double> QrState::solve() const {
    const std::size_t k = r_.size();
    std::vector<double> d(k, 0.0);
    for (std::size_t i = k; i-- > 0;) {
        double s = p_[i];
        for (std::size_t j = i + 1; j < k; ++j) s -= r_[j][i] * d[j];
        d[i] = s / r_[i][i];
    }
    return d;
}

double QrState::residual(const std::vector<double>& d, double* max_abs) const {
    double ss = 0.0, worst = 0.0;
    for (std::size_t t = 0; t < b_.size(); ++t) {
        double e = b_[t];
        for (std::size_t j = 0; j < a_.size(); ++j) e -= a_[j][t] * d[j];
        ss += e * e;
        worst = std::max(worst, std::abs(e));
    }
    if (max_abs) *max_abs = worst;
    return std::sqrt(ss);
}

std::vector<double> sample_kernel(const RangeKernel& kernel, int T) {
    if (T < 1) throw std::invalid_argument("sample_kernel: T must be >= 1");
    std::vector<double> b(static_cast<std::size_t>(T) + 1);
    for (int t = 0; t <= T; ++t) b[static_cast<std::size_t>(t)] = kernel.eval(t);
    return b;
}

FourierKernelApprox progressive_fit(std::span<const double> samples, double epsilon,
                                    FitTrace* trace) {
    if (samples.size() < 2) throw std::invalid_argument("progressive_fit: T must be >= 1");
    const int T = static_cast<int>(samples.size()) - 1;
    if (!(epsilon > 0.0) || !(epsilon < std::sqrt(static_cast<double>(T) + 1.0)))
        throw std::invalid_argument(
            "progressive_fit: epsilon must lie in (0, sqrt(T+1)); larger values are met "
            "by the zero fit and carry no information");
    FourierKernelApprox fit;
    fit.T = T;
    fit.omega = std::numbers::pi / T;
    QrState qr(std::vector<double>(samples.begin(), samples.end()));
    fit.d = qr.solve();
    fit.residual_norm = qr.residual(fit.d, &fit.max_pointwise_error);
    if (trace) trace->push_back({0, fit.residual_norm, fit.d});
    std::vector<double> column(samples.size());
    while (fit.residual_norm > epsilon) {
        if (fit.N == T)
            throw std::runtime_error(
                "progressive_fit: numerical breakdown: basis spans the whole grid but the "
                "residual still exceeds epsilon");
        const int n = fit.N + 1;
        for (int t = 0; t <= T; ++t) column[static_cast<std::size_t>(t)] = std::cos(n * fit.omega * t);
        if (!qr.append_column(column))
            throw std::runtime_error(
                "progressive_fit: numerical breakdown: linearly dependent basis column at "
                "harmonic " + std::to_string(n));
        fit.N = n;
        fit.d = qr.solve();
        fit.residual_norm = qr.residual(fit.d, &fit.max_pointwise_error);
        if (trace) trace->push_back({fit.N, fit.residual_norm, fit.d});
    }
    return fit;
}

FourierKernelApprox progressive_fit(const RangeKernel& kernel, int T, double epsilon,
                                    FitTrace* trace) {
    return progressive_fit(sample_kernel(kernel, T), epsilon, trace);
}

void write_fit_trace_csv(const FitTrace& trace, std::ostream& out) {
    char buf[32];
    for (const FitStep& s : trace) {
        out << s.order;
        std::snprintf(buf, sizeof buf, "%.17g", s.residual);
        out << ',' << buf;
        for (double c : s.coeffs) {
            std::snprintf(buf, sizeof buf, "%.17g", c);
            out << ',' << buf;
        }
        out << '\n';
    }
}

// --------------------------------------------------------------- analysis.hpp

double error_bound(int T, double epsilon, double w0) {
    if (T < 0) throw std::invalid_argument("error_bound: negative dynamic range");
    if (!(epsilon >= 0.0)) throw std::invalid_argument("error_bound: negative tolerance");
    if (!(epsilon < w0))
        throw std::invalid_argument("error_bound: tolerance must stay below the center spatial weight");
    return fbf_error_bound(T, epsilon, w0);
}

double linf_error(const Image& a, const Image& b) {
    if (!a.same_size(b)) throw std::invalid_argument("linf_error: size mismatch");
    double worst = 0.0;
    for (std::size_t i = 0; i < a.values.size(); ++i)
        worst = std::max(worst, std::abs(a.values[i] - b.values[i]));
    return worst;
}

namespace {
std::string g17(double v) {
    char buf[40];
    std::snprintf(buf, sizeof buf, "%.17g", v);
    return buf;
}
}  // namespace

void AccuracyReport::write_key_values(std::ostream& os) const {
    os << "T=" << T << '\n';
    if (N) os << "N=" << *N << '\n';
    os << "epsilon_requested=" << g17(epsilon_requested) << '\n'
       << "epsilon_achieved=" << g17(epsilon_achieved) << '\n'
       << "w0=" << g17(w0) << '\n'
       << "predicted_bound=" << g17(predicted_bound) << '\n';
    if (measured_linf) os << "measured_linf=" << g17(*measured_linf) << '\n';
    os << "weaker_guarantee_flag=" << (weaker_guarantee_flag ? "true" : "false") << '\n';
}

std::string AccuracyReport::csv_header() {
    return "T,N,epsilon_requested,epsilon_achieved,w0,predicted_bound,measured_linf,"
           "weaker_guarantee_flag";
}

std::string AccuracyReport::csv_row() const {
    std::string row = std::to_string(T) + ',' + (N ? std::to_string(*N) : std::string()) + ',' +
                      g17(epsilon_requested) + ',' + g17(epsilon_achieved) + ',' + g17(w0) + ',' +
                      g17(predicted_bound) + ',' + (measured_linf ? g17(*measured_linf) : "") + ',' +
                      (weaker_guarantee_flag ? "true" : "false");
    return row;
}

AccuracyReport make_report(int T, double epsilon_requested, double epsilon_achieved,
                           std::optional<int> N, double w0, bool weaker_guarantee) {
    AccuracyReport r;
    r.T = T;
    r.epsilon_requested = epsilon_requested;
    r.epsilon_achieved = epsilon_achieved;
    r.N = N;
    r.w0 = w0;
    r.predicted_bound = epsilon_achieved < w0 ? error_bound(T, epsilon_achieved, w0)
                                              : std::numeric_limits<double>::infinity();
    r.weaker_guarantee_flag = weaker_guarantee;
    return r;
}

// -------------------------------------------------------------- bilateral.hpp

int local_dynamic_range(const Image& image, int W) {
    if (image.width <= 0 || image.height <= 0)
        throw std::invalid_argument("local_dynamic_range: empty image");
    if (W < 1) throw std::invalid_argument("local_dynamic_range: window radius must be positive");
    // on the device (fbf_ldr.cu): filter()'s T, exact in fp64
    int T = 0;
    const int rc = fbf_local_dynamic_range_host_f64(image.values.data(), image.width, image.height, W, &T);
    if (rc != FBF_OK) throw std::runtime_error("local_dynamic_range: CUDA failure");
    return T;
}

Image bilateral_exact(const Image& image, const SpatialKernel& spatial, const RangeKernel& range) {
    if (image.width <= 0 || image.height <= 0)
        throw std::invalid_argument("bilateral_exact: empty image");
    const int W = spatial.radius;
    Image out(image.width, image.height);
    // Gaussian / exponential range kernels: the fp64 brute force on the GPU
    // (fbf_exact.cu); tabulated kernels and radii above 64 stay on the CPU
    if (range.family() != RangeFamily::tabulated && W <= 64) {
        const int rc = fbf_bilateral_exact_host_f64(
            image.width, image.height, spatial.profile.data(), W,
            range.family() == RangeFamily::exponential ? FBF_RANGE_EXPONENTIAL : FBF_RANGE_GAUSSIAN,
            range.sigma_r(), image.values.data(), out.values.data());
        if (rc != FBF_OK) rethrow_status(rc);
        return out;
    }
    for (int y = 0; y < image.height; ++y)
        for (int x = 0; x < image.width; ++x) {
            const double centre = image(x, y);
            double num = 0.0, den = 0.0;
            for (int dy = -W; dy <= W; ++dy) {
                const int sy = mirror_index(y - dy, image.height);
                for (int dx = -W; dx <= W; ++dx) {
                    const double v = image(mirror_index(x - dx, image.width), sy);
                    const double wt = spatial.weight(dx, dy) * range.eval(v - centre);
                    num += wt * v;
                    den += wt;
                }
            }
            out(x, y) = num / den;
        }
    return out;
}

Image bilateral_fast(const Image& image, const SpatialKernel& spatial,
                     const FourierKernelApprox& approx, ConvolutionBackend backend) {
    if (image.width <= 0 || image.height <= 0)
        throw std::invalid_argument("bilateral_fast: empty image");
    if (!(approx.max_pointwise_error < spatial.w0))
        throw std::invalid_argument(
            "bilateral_fast: kernel approximation error must stay below the center "
            "spatial weight");
    fbf_geometry g;
    fbf_geometry_whole(&g, image.width, image.height, 1);
    fbf_filter f{};
    f.kind = spatial.kind == SpatialKind::box ? FBF_SPATIAL_BOX : FBF_SPATIAL_GAUSSIAN;
    f.radius = spatial.radius;
    f.profile = spatial.profile.data();
    f.w0 = spatial.w0;
    f.N = approx.N;
    f.d = approx.d.data();
    f.omega = approx.omega;
    f.max_pointwise_error = approx.max_pointwise_error;
    f.check_epsilon = 1;
    f.sigma_s = spatial.sigma_s;
    Image out(image.width, image.height);
    long long bad = -1;
    const int rc = fbf_bilateral_fast_host_f64(&g, &f, image.values.data(), out.values.data(),
                                               uses_iir(spatial, backend) ? FBF_VARIANT_RECURSIVE
                                                                          : FBF_VARIANT_FUSED,
                                               &bad);
    if (rc != FBF_OK) rethrow_status(rc);
    return out;
}

std::pair<Image, AccuracyReport> filter(const Image& image, const FilterConfig& config) {
    if (!(config.epsilon > 0.0)) throw std::invalid_argument("filter: tolerance must be positive");
    if (!(config.epsilon < config.spatial.w0))
        throw std::invalid_argument(
            "filter: tolerance must stay below the center spatial weight w(0); lower "
            "--epsilon or reduce the spatial radius");
    const bool weaker = !config.integer_intensities;
    const Image working = config.integer_intensities ? round_to_integers(image) : image;
    const int T = local_dynamic_range(working, config.spatial.radius);
    if (T == 0)
        return {image, make_report(0, config.epsilon, 0.0, std::nullopt, config.spatial.w0, weaker)};
    const FourierKernelApprox approx = progressive_fit(config.range, T, config.epsilon);
    Image out = bilateral_fast(working, config.spatial, approx, config.backend);
    return {std::move(out), make_report(T, config.epsilon, approx.max_pointwise_error, approx.N,
                                        config.spatial.w0, weaker)};
}

}  // namespace fourierbf

// ======================================================= host-only C-ABI pieces

namespace {

double range_value(int family, double sigma_r, double a) {
    return family == FBF_RANGE_EXPONENTIAL ? std::exp(-a / sigma_r)
                                           : std::exp(-(a * a) / (2.0 * sigma_r * sigma_r));
}

}  // namespace

extern "C" {

int fbf_spatial_gaussian(double sigma_s, double* profile, int* radius, double* w0) {
    if (!(sigma_s > 0.0)) return FBF_EINVAL;
    const int W = static_cast<int>(std::ceil(3.0 * sigma_s));
    if (radius) *radius = W;
    if (!profile) return FBF_OK;
    double total = 0.0;
    for (int j = -W; j <= W; ++j) {
        profile[j + W] = std::exp(-(static_cast<double>(j) * j) / (2.0 * sigma_s * sigma_s));
        total += profile[j + W];
    }
    for (int k = 0; k <= 2 * W; ++k) profile[k] /= total;
    if (w0) *w0 = profile[W] * profile[W];
    return FBF_OK;
}

int fbf_spatial_box(int radius, double* profile, double* w0) {
    if (radius < 1) return FBF_EINVAL;
    const double tap = 1.0 / (2.0 * radius + 1.0);
    if (profile) std::fill(profile, profile + 2 * radius + 1, tap);
    if (w0) *w0 = tap * tap;
    return FBF_OK;
}

double fbf_range_eval(int family, double sigma_r, double t) {
    return range_value(family, sigma_r, std::abs(t));
}

int fbf_fit_fixed(int family, double sigma_r, int T, int N, double* d, double* residual_norm,
                  double* max_pointwise_error) {
    if (T < 1 || N < 0 || N > T || !(sigma_r > 0.0)) return FBF_EINVAL;
    try {
        const fourierbf::RangeKernel k = family == FBF_RANGE_EXPONENTIAL
                                             ? fourierbf::RangeKernel::exponential(sigma_r)
                                             : fourierbf::RangeKernel::gaussian(sigma_r);
        fourierbf::QrState qr(fourierbf::sample_kernel(k, T));
        const double omega = std::numbers::pi / T;
        std::vector<double> col(static_cast<std::size_t>(T) + 1);
        for (int n = 1; n <= N; ++n) {
            for (int t = 0; t <= T; ++t) col[static_cast<std::size_t>(t)] = std::cos(n * omega * t);
            if (!qr.append_column(col)) return FBF_EINVAL;
        }
        const std::vector<double> sol = qr.solve();
        double mx = 0.0;
        const double rn = qr.residual(sol, &mx);
        std::copy(sol.begin(), sol.end(), d);
        if (residual_norm) *residual_norm = rn;
        if (max_pointwise_error) *max_pointwise_error = mx;
        return FBF_OK;
    } catch (...) {
        return FBF_EINVAL;
    }
}

int fbf_progressive_fit(int family, double sigma_r, int T, double epsilon, double* d, int* N,
                        double* residual_norm, double* max_pointwise_error) {
    try {
        const fourierbf::RangeKernel k = family == FBF_RANGE_EXPONENTIAL
                                             ? fourierbf::RangeKernel::exponential(sigma_r)
                                             : fourierbf::RangeKernel::gaussian(sigma_r);
        const fourierbf::FourierKernelApprox a = fourierbf::progressive_fit(k, T, epsilon);
        std::copy(a.d.begin(), a.d.end(), d);
        *N = a.N;
        if (residual_norm) *residual_norm = a.residual_norm;
        if (max_pointwise_error) *max_pointwise_error = a.max_pointwise_error;
        return FBF_OK;
    } catch (...) {
        return FBF_EINVAL;
    }
}

double fbf_error_bound(int T, double epsilon, double w0) {
    if (T < 0 || !(epsilon >= 0.0) || !(epsilon < w0)) return -1.0;
    return 2.0 * T * epsilon / (w0 - epsilon);
}

}  // extern "C"
