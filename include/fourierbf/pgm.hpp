// fourierbf/pgm.hpp -- drop-in declarations of the 8-bit graymap codec
// (reference: proj/include/fourierbf/pgm.hpp:62-133).  Reading accepts binary
// P5 and ASCII P2 with maxval in [1, 255]; writing emits binary P5, maxval
// 255, samples rounded half-up and clamped to [0, 255].  Parse failures throw
// std::runtime_error("pgm parse error at byte <offset>: <what>").
#pragma once
#include <string>
#include <string_view>

#include "fourierbf/image.hpp"

namespace fourierbf {

Image decode_pgm(std::string_view bytes);
std::string encode_pgm(const Image& img);  ///< invalid_argument on an empty image
Image read_pgm(const std::string& path);   ///< runtime_error when unreadable
void write_pgm(const Image& img, const std::string& path);

}  // namespace fourierbf
