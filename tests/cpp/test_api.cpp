// test_api.cpp -- the drop-in C++ API (include/fourierbf/*.hpp) exercised the
// way the reference's own suites do (proj/tests/test_bilateral.cpp,
// test_spatial.cpp, test_kernel_approx.cpp, test_analysis.cpp), linked against
// libfourierbf_b200.so.  Fast-path tolerances are fp32-level (the B200 path
// computes in fp32; BASELINE parity bar 1e-3 on [0,255]).
//
//   test_api            all checks (needs a GPU for bilateral_fast / convolve)
//   test_api --host     host-only checks (fit, kernels, analysis, validation)
#include <cmath>
#include <cstdio>
#include <cstring>
#include <fstream>
#include <random>
#include <sstream>
#include <stdexcept>
#include <string>
#include <vector>

#include "fourierbf/fourierbf.hpp"

using namespace fourierbf;

static int g_fail = 0, g_pass = 0;
#define CHECK(cond)                                                         \
  do {                                                                      \
    if (cond) {                                                             \
      ++g_pass;                                                             \
    } else {                                                                \
      ++g_fail;                                                             \
      std::fprintf(stderr, "FAIL %s:%d: %s\n", __FILE__, __LINE__, #cond); \
    }                                                                       \
  } while (0)
#define CHECK_NEAR(a, b, tol) CHECK(std::abs((a) - (b)) <= (tol))
template <class E, class F>
static bool throws(F f, const char* needle = nullptr) {
  try {
    f();
  } catch (const E& e) {
    return !needle || std::string(e.what()).find(needle) != std::string::npos;
  } catch (...) {
    return false;
  }
  return false;
}

static Image random_integer_image(int w, int h, unsigned seed) {
  std::mt19937 rng(seed);
  std::uniform_int_distribution<int> dist(0, 255);
  Image img(w, h);
  for (double& v : img.values) v = dist(rng);
  return img;
}

static FourierKernelApprox identity_approx(int T) {
  FourierKernelApprox a;
  a.T = T;
  a.omega = 3.14159265358979323846 / T;
  a.N = 0;
  a.d = {1.0};
  return a;
}

static void host_checks() {
  // test_spatial.cpp:48-75
  const SpatialKernel k1 = make_spatial_gaussian(1.0), k2 = make_spatial_gaussian(2.0),
                      k3 = make_spatial_gaussian(3.0);
  CHECK(k1.radius == 3 && k2.radius == 6 && k3.radius == 9);
  CHECK_NEAR(k1.w0, 0.159241125690702, 1e-14);
  CHECK_NEAR(k2.w0, 0.039870356216689, 1e-14);
  CHECK_NEAR(k3.w0, 0.017735845914730, 1e-14);
  CHECK(make_spatial_gaussian(2.5).radius == 8);
  const SpatialKernel b = make_spatial_box(2);
  CHECK(b.kind == SpatialKind::box && b.radius == 2);
  CHECK(throws<std::invalid_argument>([] { make_spatial_gaussian(0.0); }));
  CHECK(throws<std::invalid_argument>([] { make_spatial_box(0); }));
  // test_kernel_approx.cpp:62-80: two-point grid
  QrState st({1.0, 0.5});
  CHECK(st.append_column(std::vector<double>{1.0, -1.0}));
  const std::vector<double> d = st.solve();
  CHECK_NEAR(d[0], 0.75, 1e-15);
  CHECK_NEAR(d[1], 0.25, 1e-15);
  CHECK_NEAR(st.residual(d), 0.0, 1e-15);
  QrState dep({1.0, 2.0, 3.0, 4.0});
  CHECK(dep.append_column(std::vector<double>{1.0, -1.0, 1.0, -1.0}));
  CHECK(!dep.append_column(std::vector<double>{1.0, -1.0, 1.0, -1.0}));
  // test_kernel_approx.cpp:139-158
  FitTrace trace;
  const FourierKernelApprox fit = progressive_fit(RangeKernel::gaussian(30.0), 217, 1e-3, &trace);
  CHECK(fit.N == 9 && fit.T == 217 && fit.residual_norm <= 1e-3);
  CHECK(fit.max_pointwise_error <= fit.residual_norm);
  CHECK(trace.size() == 10u);
  std::ostringstream csv;
  write_fit_trace_csv(trace, csv);
  CHECK(csv.str().rfind("0,", 0) == 0);
  // kernels.hpp
  CHECK(RangeKernel::gaussian(30.0).eval(0.0) == 1.0);
  CHECK_NEAR(RangeKernel::exponential(20.0).eval(-40.0), std::exp(-2.0), 1e-15);
  CHECK(throws<std::invalid_argument>([] { RangeKernel::tabulated({0.5}); }));
  CHECK(throws<std::out_of_range>([] { RangeKernel::tabulated({1.0, 0.5}).eval(3.0); }));
  // analysis.hpp
  CHECK_NEAR(error_bound(217, 1e-3, 0.017735845914730), 2.0 * 217 * 1e-3 / (0.017735845914730 - 1e-3),
             1e-12);
  CHECK(throws<std::invalid_argument>([] { error_bound(10, 0.5, 0.1); }));
  const AccuracyReport r = make_report(10, 1e-3, 0.5, 4, 0.1, false);
  CHECK(std::isinf(r.predicted_bound));
  std::ostringstream kv;
  make_report(208, 1e-3, 1e-4, 8, 0.0177, true).write_key_values(kv);
  CHECK(kv.str().find("N=8\n") != std::string::npos && kv.str().find("weaker_guarantee_flag=true") != std::string::npos);
  // image.hpp
  CHECK(mirror_index(-1, 5) == 0 && mirror_index(5, 5) == 4 && mirror_index(-6, 5) == 4);
  CHECK(throws<std::invalid_argument>([] { Image(0, 3); }));
  CHECK(round_to_integers(Image(2, 2, 2.5)).values[0] == 3.0);
  // bilateral.hpp argument validation (no device work)
  CHECK(throws<std::invalid_argument>([] { bilateral_fast(Image(), make_spatial_gaussian(1.0), identity_approx(255)); }));
  FourierKernelApprox bad = identity_approx(255);
  bad.max_pointwise_error = 0.5;
  CHECK(throws<std::invalid_argument>(
      [&] { bilateral_fast(random_integer_image(8, 8, 7), make_spatial_gaussian(3.0), bad); }));
  CHECK(throws<std::invalid_argument>([] { local_dynamic_range(Image(), 1); }));
  CHECK(throws<std::invalid_argument>([] { local_dynamic_range(Image(4, 4, 0.0), 0); }));
}

// test_pgm.cpp / test_cli.cpp restated (host-only parts: the codec, run()'s diagnostics)
static void pgm_cli_host_checks() {
  const Image one = decode_pgm(std::string("P5\n1 1\n255\n") + static_cast<char>(0x80));
  CHECK(one.width == 1 && one.height == 1 && one(0, 0) == 128.0);
  const Image c = decode_pgm(std::string("P5 # c\n# line\n  2 1 # dims\n255\n") + static_cast<char>(3) +
                             static_cast<char>(250));
  CHECK(c.width == 2 && c(0, 0) == 3.0 && c(1, 0) == 250.0);
  CHECK(decode_pgm("P2\n2 1\n255\n7 9\n")(1, 0) == 9.0);
  CHECK(throws<std::runtime_error>([] { decode_pgm("P6\n1 1\n255\nx"); }, "not a P5 or P2"));
  CHECK(throws<std::runtime_error>([] { decode_pgm("P5\n2 2\n255\nab"); }, "truncated raster"));
  CHECK(throws<std::runtime_error>([] { decode_pgm("P2\n1 1\n100\n101"); }, "exceeds maxval"));
  Image r(5, 1);
  r.values = {0.5, 1.49, 254.5, -3.0, 300.0};
  const Image back = decode_pgm(encode_pgm(r));
  CHECK(back.values == (std::vector<double>{1.0, 1.0, 255.0, 0.0, 255.0}));
  CHECK(throws<std::invalid_argument>([] { encode_pgm(Image()); }));
  CHECK(throws<std::runtime_error>([] { read_pgm("/nonexistent/file.pgm"); }));
  CliOptions opt;  // run(): diagnostics before any pixel work
  std::ostringstream out, err;
  CHECK(run(opt, out, err) == 1 && err.str().find("--input") != std::string::npos);
  opt.input_path = "/nonexistent/in.pgm";
  opt.output_path = "/tmp/unused.pgm";
  opt.sigma_s = 1.0;
  opt.sigma_r = 30.0;
  err.str("");
  CHECK(run(opt, out, err) == 1 && err.str().find("error:") != std::string::npos);
}

static void gpu_checks() {
  // test_bilateral.cpp:133-162 local_dynamic_range (now on the device, fp64)
  {
    CHECK(local_dynamic_range(Image(5, 4, 9.0), 2) == 0);
    Image two(2, 2);
    two(1, 0) = two(1, 1) = 255.0;
    CHECK(local_dynamic_range(two, 1) == 255);
    Image frac(3, 1, 0.0);
    frac(1, 0) = 1.25;
    CHECK(local_dynamic_range(frac, 1) == 2);
    for (unsigned seed = 0; seed < 6; ++seed) {
      const Image img = random_integer_image(seed % 2 ? 7 : 16, seed % 3 ? 5 : 12, seed);
      for (const int W : {1, 2, 5}) {
        double spread = 0.0;  // brute force, test_bilateral.cpp:68-83
        for (int y = 0; y < img.height; ++y)
          for (int x = 0; x < img.width; ++x) {
            double hi = -1e300, lo = 1e300;
            for (int jy = -W; jy <= W; ++jy)
              for (int jx = -W; jx <= W; ++jx) {
                const double v = img(mirror_index(x - jx, img.width), mirror_index(y - jy, img.height));
                hi = std::max(hi, v);
                lo = std::min(lo, v);
              }
            spread = std::max(spread, hi - lo);
          }
        CHECK(local_dynamic_range(img, W) == static_cast<int>(std::ceil(spread)));
      }
    }
  }
  // test_bilateral.cpp:218-224 constant pass-through
  {
    const Image img(8, 8, 120.0);
    const Image out = bilateral_fast(img, make_spatial_gaussian(1.0),
                                     progressive_fit(RangeKernel::gaussian(30.0), 255, 1e-3));
    for (double v : out.values) CHECK_NEAR(v, 120.0, 1e-4);
  }
  // :226-232 N=0 identity == convolve
  {
    const Image img = random_integer_image(14, 9, 77);
    const SpatialKernel s = make_spatial_gaussian(2.0);
    const Image a = bilateral_fast(img, s, identity_approx(255));
    const Image c = convolve(img, s);
    for (size_t i = 0; i < a.values.size(); ++i) CHECK_NEAR(a.values[i], c.values[i], 1e-4);
  }
  // :247-257 within the guaranteed bound
  {
    const Image img = random_integer_image(64, 64, 99);
    const SpatialKernel s = make_spatial_gaussian(2.0);
    const RangeKernel phi = RangeKernel::gaussian(30.0);
    const int T = local_dynamic_range(img, s.radius);
    const FourierKernelApprox approx = progressive_fit(phi, T, 1e-3);
    const Image fast = bilateral_fast(img, s, approx);
    const Image exact = bilateral_exact(img, s, phi);
    CHECK(linf_error(exact, fast) <= error_bound(T, approx.max_pointwise_error, s.w0));
  }
  // :259-269 shift equivariance
  {
    const Image img = random_integer_image(12, 12, 101);
    Image shifted = img;
    for (double& v : shifted.values) v += 10.0;
    const SpatialKernel s = make_spatial_gaussian(1.0);
    const FourierKernelApprox approx = progressive_fit(RangeKernel::gaussian(25.0), 255, 1e-4);
    const Image a = bilateral_fast(shifted, s, approx), b = bilateral_fast(img, s, approx);
    for (size_t i = 0; i < a.values.size(); ++i) CHECK_NEAR(a.values[i], b.values[i] + 10.0, 2e-3);
  }
  // :271-282 mirror commutation
  {
    const Image img = random_integer_image(13, 9, 111);
    const SpatialKernel s = make_spatial_gaussian(1.5);
    const FourierKernelApprox approx =
        progressive_fit(RangeKernel::gaussian(30.0), local_dynamic_range(img, s.radius), 1e-3);
    const Image a = bilateral_fast(mirror_horizontal(img), s, approx);
    const Image b = mirror_horizontal(bilateral_fast(img, s, approx));
    for (size_t i = 0; i < a.values.size(); ++i) CHECK_NEAR(a.values[i], b.values[i], 2e-3);
    const Image c = bilateral_fast(mirror_vertical(img), s, approx);
    const Image e = mirror_vertical(bilateral_fast(img, s, approx));
    for (size_t i = 0; i < c.values.size(); ++i) CHECK_NEAR(c.values[i], e.values[i], 2e-3);
  }
  // :302-312 collapsed denominator names the pixel
  {
    FourierKernelApprox lying = identity_approx(255);
    lying.d = {0.0};
    CHECK(throws<std::runtime_error>(
        [&] { bilateral_fast(random_integer_image(6, 6, 8), make_spatial_gaussian(1.0), lying); },
        "pixel (0, 0)"));
  }
  // :314-375 filter(): short circuit, report, rounding, flags, tolerance check
  {
    const Image flat(8, 8, 42.0);
    const FilterConfig cfg{make_spatial_gaussian(2.0), RangeKernel::gaussian(30.0), 1e-3, true,
                           ConvolutionBackend::direct};
    const auto [out, rep] = filter(flat, cfg);
    CHECK(out.values == flat.values && rep.T == 0 && !rep.N.has_value());
    const Image img = random_integer_image(24, 24, 200);
    const auto [o2, r2] = filter(img, cfg);
    CHECK(r2.T == local_dynamic_range(img, 6) && r2.N.has_value());
    const Image exact = bilateral_exact(img, cfg.spatial, cfg.range);
    CHECK(linf_error(exact, o2) <= r2.predicted_bound);
    const FilterConfig too_loose{make_spatial_gaussian(3.0), RangeKernel::gaussian(30.0), 0.02, true,
                                 ConvolutionBackend::direct};
    CHECK(throws<std::invalid_argument>([&] { filter(img, too_loose); }));
  }
  // test_spatial.cpp:91-107 separable == brute force (fp32 path)
  {
    std::mt19937 rng(1);
    std::uniform_real_distribution<double> dist(0.0, 255.0);
    Image img(16, 16);
    for (double& v : img.values) v = dist(rng);
    const SpatialKernel k = make_spatial_gaussian(2.0);
    const Plane fast = convolve(img, k);
    for (int y = 0; y < 16; ++y)
      for (int x = 0; x < 16; ++x) {
        double acc = 0.0;
        for (int dy = -k.radius; dy <= k.radius; ++dy)
          for (int dx = -k.radius; dx <= k.radius; ++dx)
            acc += k.weight(dx, dy) * img(mirror_index(x - dx, 16), mirror_index(y - dy, 16));
        CHECK_NEAR(fast(x, y), acc, 1e-11);  // test_spatial.cpp:91-107 (fp64 on the device)
      }
    CHECK(throws<std::invalid_argument>([&] { convolve(Plane(), k); }));
  }
  // the recursive backend (spatial.hpp:98-112 dispatch, recursive_gaussian.hpp)
  {
    const Image img = random_integer_image(24, 20, 31);
    const SpatialKernel narrow = make_spatial_gaussian(1.5), wide = make_spatial_gaussian(3.0);
    CHECK(convolve(img, narrow, ConvolutionBackend::recursive).values == convolve(img, narrow).values);
    const Plane iir = convolve(img, wide, ConvolutionBackend::recursive), fir = convolve(img, wide);
    CHECK(linf_error(iir, fir) > 1e-6 && linf_error(iir, fir) < 5.0);
    const FourierKernelApprox a = progressive_fit(RangeKernel::gaussian(30.0), 255, 1e-3);
    const Image bi = bilateral_fast(img, make_spatial_gaussian(2.5), a, ConvolutionBackend::recursive);
    CHECK(linf_error(bi, bilateral_fast(img, make_spatial_gaussian(2.5), a)) < 5.0);
  }
  // cli.hpp run() end to end: PGM in, report out
  {
    const std::string in = "/tmp/fbf_test_api_in.pgm", outp = "/tmp/fbf_test_api_out.pgm",
                      rep = "/tmp/fbf_test_api_report.txt";
    write_pgm(random_integer_image(20, 14, 5), in);
    CliOptions opt;
    opt.input_path = in;
    opt.output_path = outp;
    opt.report_path = rep;
    opt.sigma_s = 1.0;
    opt.sigma_r = 30.0;
    opt.compare_exact = true;
    std::ostringstream o, e;
    CHECK(run(opt, o, e) == 0);
    CHECK(read_pgm(outp).width == 20);
    std::ifstream f(rep);
    std::stringstream txt;
    txt << f.rdbuf();
    CHECK(txt.str().find("measured_linf=") != std::string::npos);
  }
}

int main(int argc, char** argv) {
  const bool host_only = argc > 1 && std::strcmp(argv[1], "--host") == 0;
  host_checks();
  pgm_cli_host_checks();
  if (!host_only) gpu_checks();
  std::printf("%d passed, %d failed\n", g_pass, g_fail);
  return g_fail ? 1 : 0;
}
