// fbf_synth.cpp -- the seeded synthetic image generator of the BASELINE
// configs.  Input generation only, not
// part of the filter: it is compiled into the product library (fbf_synth_image
// in include/fourierbf_b200.h) and, from this same source, into the standalone
// oracle/_synth/libfbf_synth.so that bench.py's reference arm loads, so both
// arms read identical bytes without the reference arm touching the product.
#include <algorithm>
#include <cmath>
#include <cstdint>
#include <thread>
#include <vector>

#include "fourierbf_b200.h"

namespace {

constexpr double kPi = 3.14159265358979323846;

// splitmix64 output function; stream j of key k is mix(k + j * golden)
inline uint64_t mix64(uint64_t z) {
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
    return z ^ (z >> 31);
}
inline double unit(uint64_t key, uint64_t j) {
    return static_cast<double>(mix64(key + (j + 1) * 0x9E3779B97F4A7C15ULL) >> 11) * 0x1.0p-53;
}

}  // namespace

extern "C" {

// BASELINE.json generator: gradient 0->128 along x, `rects` axis-aligned
// rectangles (later ones on top) of uniform intensity in [0,255), iid
// Gaussian noise (Box-Muller), clipped to [0,255], stored as fp32.
int fbf_synth_image(unsigned long long seed, int width, int height, int rects, double noise_sigma,
                    int row0, int rows, float* out, int nthreads) {
    if (width < 1 || height < 1 || rects < 0 || row0 < 0 || rows < 1 || row0 + rows > height)
        return FBF_EINVAL;
    struct Rect {
        int x0, y0, x1, y1;
        double v;
    };
    const uint64_t krect = mix64(seed ^ 0x5EED0001ULL);
    const uint64_t knoise = mix64(seed ^ 0x5EED0002ULL);
    std::vector<Rect> rs(static_cast<std::size_t>(rects));
    for (int r = 0; r < rects; ++r) {
        const uint64_t b = 8ULL * static_cast<uint64_t>(r);
        const int rw = 1 + static_cast<int>(unit(krect, b + 0) * (width / 4.0));
        const int rh = 1 + static_cast<int>(unit(krect, b + 1) * (height / 4.0));
        const int cw = std::min(rw, width), ch = std::min(rh, height);
        const int x0 = static_cast<int>(unit(krect, b + 2) * (width - cw + 1));
        const int y0 = static_cast<int>(unit(krect, b + 3) * (height - ch + 1));
        rs[static_cast<std::size_t>(r)] = {x0, y0, x0 + cw, y0 + ch, 255.0 * unit(krect, b + 4)};
    }
    auto work = [&](int ya, int yb) {
        std::vector<double> line(static_cast<std::size_t>(width));
        for (int y = ya; y < yb; ++y) {
            for (int x = 0; x < width; ++x)
                line[static_cast<std::size_t>(x)] = width > 1 ? 128.0 * x / (width - 1) : 0.0;
            for (const Rect& r : rs)
                if (y >= r.y0 && y < r.y1)
                    std::fill(line.begin() + r.x0, line.begin() + r.x1, r.v);
            float* o = out + static_cast<std::size_t>(y - row0) * width;
            for (int x = 0; x < width; ++x) {
                const uint64_t i = static_cast<uint64_t>(y) * width + x;
                const double u1 = unit(knoise, 2 * i), u2 = unit(knoise, 2 * i + 1);
                const double z = std::sqrt(-2.0 * std::log(1.0 - u1)) * std::cos(2.0 * kPi * u2);
                const double v = line[static_cast<std::size_t>(x)] + noise_sigma * z;
                o[x] = static_cast<float>(std::min(255.0, std::max(0.0, v)));
            }
        }
    };
    nthreads = std::max(1, std::min(nthreads, rows));
    if (nthreads == 1) {
        work(row0, row0 + rows);
    } else {
        std::vector<std::thread> pool;
        for (int t = 0; t < nthreads; ++t)
            pool.emplace_back(work, row0 + static_cast<int>(static_cast<long>(rows) * t / nthreads),
                              row0 + static_cast<int>(static_cast<long>(rows) * (t + 1) / nthreads));
        for (auto& th : pool) th.join();
    }
    return FBF_OK;
}

}  // extern "C"
