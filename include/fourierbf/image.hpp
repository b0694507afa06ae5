// fourierbf/image.hpp -- drop-in declaration of the reference's image type
// (reference: proj/include/fourierbf/image.hpp:11-63).  Same names, members,
// indexing and exceptions; the definitions live in libfourierbf_b200.so.
#pragma once

#include <cstddef>
#include <vector>

namespace fourierbf {

/// Row-major real image; also the type of every intermediate plane.
struct Image {
    int width = 0;
    int height = 0;
    std::vector<double> values;

    Image() = default;
    /// throws std::invalid_argument unless both dimensions are positive
    Image(int w, int h, double fill = 0.0);

    double& operator()(int x, int y) { return values[static_cast<std::size_t>(y) * width + x]; }
    double operator()(int x, int y) const { return values[static_cast<std::size_t>(y) * width + x]; }
    bool empty() const { return values.empty(); }
    std::size_t size() const { return values.size(); }
    bool same_size(const Image& o) const { return width == o.width && height == o.height; }
};

/// Half-sample symmetric reflection onto [0, n), periodic for any offset.
int mirror_index(int i, int n);
/// floor(v + 0.5) on every pixel.
Image round_to_integers(const Image& img);
Image mirror_horizontal(const Image& img);
Image mirror_vertical(const Image& img);

}  // namespace fourierbf
