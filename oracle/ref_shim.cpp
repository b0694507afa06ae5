// ref_shim.cpp -- TEST INFRASTRUCTURE ONLY.
//
// A thin extern "C" wrapper that compiles the UNMODIFIED reference library
// (header-only, /root/reference/proj/include/fourierbf, included by path --
// nothing is copied) into oracle/_ref/libfbf_ref.so.  Used to pin the C
// restatement (oracle/fbf_oracle.c), to generate tests/golden/ fixtures, and
// as bench.py's reference CPU arm.  The product never links it.
//
// Threading: the reference is single-threaded.  ref_bilateral_fast_rows may
// split the requested output rows into strips, each filtered by the
// reference's own bilateral_fast on a sub-image carrying W halo rows; rows of
// a strip that lie >= W from a cut are bit-identical to the whole-image run
// (every reference operation is per-row or per-column with mirror padding
// only at the sub-image edges, which coincide with the global edges wherever
// they are reached).
#include <algorithm>
#include <cstring>
#include <sstream>
#include <exception>
#include <numbers>
#include <string>
#include <thread>
#include <vector>

#include "fourierbf/analysis.hpp"
#include "fourierbf/bilateral.hpp"
#include "fourierbf/cli.hpp"
#include "fourierbf/kernel_approx.hpp"
#include "fourierbf/kernels.hpp"
#include "fourierbf/pgm.hpp"
#include "fourierbf/spatial.hpp"

namespace fb = fourierbf;

namespace {

thread_local std::string g_err;

fb::SpatialKernel spatial_of(int kind, double param) {
    return kind == 1 ? fb::make_spatial_box(static_cast<int>(param))
                     : fb::make_spatial_gaussian(param);
}

fb::RangeKernel range_of(int family, double sigma_r) {
    return family == 1 ? fb::RangeKernel::exponential(sigma_r) : fb::RangeKernel::gaussian(sigma_r);
}

fb::Image image_of(const double* v, int w, int h, int row_lo, int row_hi) {
    fb::Image img(w, row_hi - row_lo);
    std::memcpy(img.values.data(), v + static_cast<size_t>(row_lo) * w,
                sizeof(double) * static_cast<size_t>(w) * (row_hi - row_lo));
    return img;
}

}  // namespace

extern "C" {

const char* ref_last_error() { return g_err.c_str(); }

int ref_make_spatial(int kind, double param, double* profile, int* radius, double* w0) {
    try {
        const fb::SpatialKernel k = spatial_of(kind, param);
        *radius = k.radius;
        if (w0) *w0 = k.w0;
        if (profile) std::copy(k.profile.begin(), k.profile.end(), profile);
        return 0;
    } catch (const std::exception& e) {
        g_err = e.what();
        return -1;
    }
}

double ref_range_eval(int family, double sigma_r, double t) { return range_of(family, sigma_r).eval(t); }

// Fixed-order fit through the public QrState (tests/acceptance.cpp:247-263 pattern).
int ref_fit_fixed(int family, double sigma_r, int T, int N, double* d, double* residual_norm,
                  double* max_err) {
    try {
        const std::vector<double> b = fb::sample_kernel(range_of(family, sigma_r), T);
        const double omega = std::numbers::pi / T;
        fb::QrState qr(b);
        std::vector<double> col(static_cast<size_t>(T) + 1);
        for (int n = 1; n <= N; ++n) {
            for (int t = 0; t <= T; ++t) col[static_cast<size_t>(t)] = std::cos(n * omega * t);
            if (!qr.append_column(col)) {
                g_err = "column rejected";
                return -1;
            }
        }
        const std::vector<double> sol = qr.solve();
        double mx = 0.0;
        const double rn = qr.residual(sol, &mx);
        std::copy(sol.begin(), sol.end(), d);
        if (residual_norm) *residual_norm = rn;
        if (max_err) *max_err = mx;
        return 0;
    } catch (const std::exception& e) {
        g_err = e.what();
        return -1;
    }
}

int ref_progressive_fit(int family, double sigma_r, int T, double eps, double* d, int* N,
                        double* residual_norm, double* max_err) {
    try {
        const fb::FourierKernelApprox a = fb::progressive_fit(range_of(family, sigma_r), T, eps);
        std::copy(a.d.begin(), a.d.end(), d);
        *N = a.N;
        if (residual_norm) *residual_norm = a.residual_norm;
        if (max_err) *max_err = a.max_pointwise_error;
        return 0;
    } catch (const std::exception& e) {
        g_err = e.what();
        return -1;
    }
}

int ref_convolve(const double* in, double* out, int w, int h, int kind, double param) {
    try {
        const fb::Plane p = fb::convolve(image_of(in, w, h, 0, h), spatial_of(kind, param));
        std::copy(p.values.begin(), p.values.end(), out);
        return 0;
    } catch (const std::exception& e) {
        g_err = e.what();
        return -1;
    }
}

// Reference bilateral_fast on output rows [row0, row1) of a w*h image.
// check_eps = 0 builds the approximation with max_pointwise_error = 0, the
// precondition bypass used for config c3 (precedent test_bilateral.cpp:120-129).
// Returns 0, 1 (invalid_argument), 2 (runtime_error: anomaly), -1 other.
int ref_bilateral_fast_rows(const double* img, int w, int h, int kind, double param,
                            const double* d, int N, int T, double max_err, int check_eps,
                            int row0, int row1, int nthreads, double* out) {
    const fb::SpatialKernel sk = spatial_of(kind, param);
    fb::FourierKernelApprox a;
    a.T = T;
    a.omega = std::numbers::pi / T;
    a.N = N;
    a.d.assign(d, d + N + 1);
    a.max_pointwise_error = check_eps ? max_err : 0.0;
    const int W = sk.radius;
    const int rows = row1 - row0;
    nthreads = std::max(1, std::min(nthreads, rows));
    // tiny images: one whole-image run (periodic mirror may reach any row)
    if (h <= 4 * W + 2) nthreads = 1;
    std::vector<int> rc(static_cast<size_t>(nthreads), 0);
    std::vector<std::string> msg(static_cast<size_t>(nthreads));
    auto work = [&](int t) {
        const int a0 = row0 + static_cast<int>(static_cast<long>(rows) * t / nthreads);
        const int a1 = row0 + static_cast<int>(static_cast<long>(rows) * (t + 1) / nthreads);
        const bool whole = (h <= 4 * W + 2);
        const int lo = whole ? 0 : std::max(0, a0 - W);
        const int hi = whole ? h : std::min(h, a1 + W);
        try {
            const fb::Image res = fb::bilateral_fast(image_of(img, w, h, lo, hi), sk, a);
            std::memcpy(out + static_cast<size_t>(a0 - row0) * w,
                        res.values.data() + static_cast<size_t>(a0 - lo) * w,
                        sizeof(double) * static_cast<size_t>(w) * (a1 - a0));
        } catch (const std::invalid_argument& e) {
            rc[static_cast<size_t>(t)] = 1;
            msg[static_cast<size_t>(t)] = e.what();
        } catch (const std::runtime_error& e) {
            rc[static_cast<size_t>(t)] = 2;
            msg[static_cast<size_t>(t)] = e.what();
        } catch (const std::exception& e) {
            rc[static_cast<size_t>(t)] = -1;
            msg[static_cast<size_t>(t)] = e.what();
        }
    };
    if (nthreads == 1) {
        work(0);
    } else {
        std::vector<std::thread> pool;
        for (int t = 0; t < nthreads; ++t) pool.emplace_back(work, t);
        for (auto& th : pool) th.join();
    }
    for (int t = 0; t < nthreads; ++t)
        if (rc[static_cast<size_t>(t)]) {
            g_err = msg[static_cast<size_t>(t)];
            return rc[static_cast<size_t>(t)];
        }
    return 0;
}

// Reference bilateral_exact on rows [row0, row1) (threads: strips with W halo).
int ref_bilateral_exact_rows(const double* img, int w, int h, int kind, double param, int family,
                             double sigma_r, int row0, int row1, int nthreads, double* out) {
    const fb::SpatialKernel sk = spatial_of(kind, param);
    const fb::RangeKernel rk = range_of(family, sigma_r);
    const int W = sk.radius;
    const int rows = row1 - row0;
    nthreads = std::max(1, std::min(nthreads, rows));
    const bool whole = (h <= 4 * W + 2);
    if (whole) nthreads = 1;
    auto work = [&](int t) {
        const int a0 = row0 + static_cast<int>(static_cast<long>(rows) * t / nthreads);
        const int a1 = row0 + static_cast<int>(static_cast<long>(rows) * (t + 1) / nthreads);
        const int lo = whole ? 0 : std::max(0, a0 - W);
        const int hi = whole ? h : std::min(h, a1 + W);
        const fb::Image res = fb::bilateral_exact(image_of(img, w, h, lo, hi), sk, rk);
        std::memcpy(out + static_cast<size_t>(a0 - row0) * w,
                    res.values.data() + static_cast<size_t>(a0 - lo) * w,
                    sizeof(double) * static_cast<size_t>(w) * (a1 - a0));
    };
    try {
        if (nthreads == 1) {
            work(0);
        } else {
            std::vector<std::thread> pool;
            for (int t = 0; t < nthreads; ++t) pool.emplace_back(work, t);
            for (auto& th : pool) th.join();
        }
    } catch (const std::exception& e) {
        g_err = e.what();
        return -1;
    }
    return 0;
}

int ref_local_dynamic_range(const double* img, int w, int h, int W) {
    try {
        return fb::local_dynamic_range(image_of(img, w, h, 0, h), W);
    } catch (const std::exception& e) {
        g_err = e.what();
        return -1;
    }
}

double ref_error_bound(int T, double eps, double w0) {
    try {
        return fb::error_bound(T, eps, w0);
    } catch (const std::exception& e) {
        g_err = e.what();
        return -1.0;
    }
}

// pgm.hpp decode_pgm: 0 and the raster (up to cap values), or -1 with the
// reference's message in ref_last_error()
int ref_decode_pgm(const char* bytes, size_t len, double* values, size_t cap, int* w, int* h) {
    try {
        const fb::Image img = fb::decode_pgm(std::string_view(bytes, len));
        *w = img.width;
        *h = img.height;
        std::memcpy(values, img.values.data(), sizeof(double) * std::min(cap, img.values.size()));
        return 0;
    } catch (const std::exception& e) {
        g_err = e.what();
        return -1;
    }
}

// pgm.hpp encode_pgm: byte count (bytes copied up to cap), or -1
long ref_encode_pgm(const double* values, int w, int h, char* out, size_t cap) {
    try {
        fb::Image img(w, h);
        std::memcpy(img.values.data(), values, sizeof(double) * static_cast<size_t>(w) * h);
        const std::string bytes = fb::encode_pgm(img);
        std::memcpy(out, bytes.data(), std::min(cap, bytes.size()));
        return static_cast<long>(bytes.size());
    } catch (const std::exception& e) {
        g_err = e.what();
        return -1;
    }
}

// cli.hpp run(): the reference command-line driver on files (family 0 gaussian,
// 1 exponential, 2 tabulated:<table>; spatial 0 gaussian, 1 box).  Returns
// run()'s code; its stdout / stderr text is copied into out / err (cap bytes).
int ref_cli_run(const char* input, const char* output, double sigma_s, double sigma_r, double epsilon,
                int family, const char* table, int spatial, int compare_exact, const char* report, int bench,
                char* out, size_t out_cap, char* err, size_t err_cap, int backend) {
    fb::CliOptions opt;
    opt.backend = backend == 1 ? fb::ConvolutionBackend::recursive : fb::ConvolutionBackend::direct;
    opt.input_path = input ? input : "";
    opt.output_path = output ? output : "";
    opt.sigma_s = sigma_s;
    opt.sigma_r = sigma_r;
    opt.epsilon = epsilon;
    opt.kernel_family = family == 2 ? fb::RangeFamily::tabulated
                        : family == 1 ? fb::RangeFamily::exponential : fb::RangeFamily::gaussian;
    opt.tabulated_path = table ? table : "";
    opt.spatial_kind = spatial == 1 ? fb::SpatialKind::box : fb::SpatialKind::gaussian;
    opt.compare_exact = compare_exact != 0;
    opt.report_path = report ? report : "";
    opt.bench = bench != 0;
    std::ostringstream o, e;
    const int rc = fb::run(opt, o, e);
    const std::string so = o.str(), se = e.str();
    std::memset(out, 0, out_cap);
    std::memset(err, 0, err_cap);
    std::memcpy(out, so.data(), std::min(out_cap - 1, so.size()));
    std::memcpy(err, se.data(), std::min(err_cap - 1, se.size()));
    return rc;
}

// convolve / bilateral_fast with ConvolutionBackend::recursive (the IIR Gaussian,
// recursive_gaussian.hpp) on a whole w*h image; Gaussian window of sigma.
int ref_convolve_recursive(const double* in, double* out, int w, int h, double sigma) {
    try {
        const fb::Plane p = fb::convolve(image_of(in, w, h, 0, h), fb::make_spatial_gaussian(sigma),
                                         fb::ConvolutionBackend::recursive);
        std::copy(p.values.begin(), p.values.end(), out);
        return 0;
    } catch (const std::exception& e) {
        g_err = e.what();
        return -1;
    }
}

int ref_bilateral_fast_recursive(const double* img, int w, int h, double sigma, const double* d, int N, int T,
                                 double max_err, double* out) {
    try {
        fb::FourierKernelApprox a;
        a.T = T;
        a.omega = std::numbers::pi / T;
        a.N = N;
        a.d.assign(d, d + N + 1);
        a.max_pointwise_error = max_err;
        const fb::Image res = fb::bilateral_fast(image_of(img, w, h, 0, h), fb::make_spatial_gaussian(sigma), a,
                                                 fb::ConvolutionBackend::recursive);
        std::copy(res.values.begin(), res.values.end(), out);
        return 0;
    } catch (const std::exception& e) {
        g_err = e.what();
        return -1;
    }
}

}  // extern "C"
