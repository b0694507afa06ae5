// pgm_probe.cpp -- test driver for the drop-in PGM codec (include/fourierbf/pgm.hpp).
//   pgm_probe decode < bytes            -> "ok W H" + one value per line, or "error <what>"
//   pgm_probe encode W H < values (text) -> the encoded bytes
// tests/test_pgm.py compares it against the reference codec (oracle/_ref).
#include <cstdio>
#include <iostream>
#include <iterator>
#include <sstream>
#include <string>

#include "fourierbf/pgm.hpp"

int main(int argc, char** argv) {
    const std::string mode = argc > 1 ? argv[1] : "";
    if (mode == "decode") {
        const std::string bytes((std::istreambuf_iterator<char>(std::cin)), std::istreambuf_iterator<char>());
        try {
            const fourierbf::Image img = fourierbf::decode_pgm(bytes);
            std::printf("ok %d %d\n", img.width, img.height);
            for (const double v : img.values) std::printf("%.17g\n", v);
        } catch (const std::exception& e) {
            std::printf("error %s\n", e.what());
        }
        return 0;
    }
    if (mode == "encode" && argc == 4) {
        fourierbf::Image img(std::stoi(argv[2]), std::stoi(argv[3]));
        for (double& v : img.values) std::cin >> v;
        const std::string out = fourierbf::encode_pgm(img);
        std::fwrite(out.data(), 1, out.size(), stdout);
        return 0;
    }
    std::fprintf(stderr, "usage: pgm_probe decode|encode W H\n");
    return 2;
}
