// fbf_main.cpp -- the `fourierbf` command-line tool (reference:
// proj/tools/main.cpp): same flags, parsed here without CLI11, then
// fourierbf::run() on the B200 pipeline.
//
//   fourierbf --input in.pgm --output out.pgm --sigma-s 5 --sigma-r 20
//             [--epsilon 1e-3] [--kernel gaussian|exponential|tabulated:<path>]
//             [--spatial gaussian|box] [--backend direct|recursive]
//             [--compare-exact] [--report r.txt] [--bench]
#include <cstdlib>
#include <iostream>
#include <string>

#include "fourierbf/cli.hpp"

namespace {

const char* kUsage =
    "Fast bilateral filter via a cosine decomposition of the range kernel (B200)\n"
    "usage: fourierbf --input PGM [--output PGM] --sigma-s S [--sigma-r R] [--epsilon E]\n"
    "                 [--kernel gaussian|exponential|tabulated:<path>] [--spatial gaussian|box]\n"
    "                 [--backend direct|recursive] [--compare-exact] [--report PATH] [--bench]\n";

int usage_error(const std::string& msg) {
    std::cerr << "error: " << msg << "\n" << kUsage;
    return 2;
}

bool to_double(const std::string& s, double& v) {
    char* end = nullptr;
    v = std::strtod(s.c_str(), &end);
    return !s.empty() && end && *end == '\0';
}

}  // namespace

int main(int argc, char** argv) {
    fourierbf::CliOptions opt;
    bool have_input = false, have_sigma_s = false;
    for (int i = 1; i < argc; ++i) {
        std::string arg = argv[i], val;
        const bool is_flag = arg == "--compare-exact" || arg == "--bench" || arg == "--help" || arg == "-h";
        const std::string name = arg.substr(0, arg.find('='));
        const bool takes_value = name == "--input" || name == "--output" || name == "--report" ||
                                 name == "--sigma-s" || name == "--sigma-r" || name == "--epsilon" ||
                                 name == "--kernel" || name == "--spatial" || name == "--backend";
        if (!is_flag && !takes_value) return usage_error("unknown option " + arg);
        if (!is_flag) {
            const auto eq = arg.find('=');
            if (arg.rfind("--", 0) == 0 && eq != std::string::npos) {
                val = arg.substr(eq + 1);
                arg = arg.substr(0, eq);
            } else if (i + 1 < argc) {
                val = argv[++i];
            } else {
                return usage_error(arg + " needs a value");
            }
        }
        double d = 0.0;
        if (arg == "--help" || arg == "-h") {
            std::cout << kUsage;
            return 0;
        } else if (arg == "--compare-exact") {
            opt.compare_exact = true;
        } else if (arg == "--bench") {
            opt.bench = true;
        } else if (arg == "--input") {
            opt.input_path = val;
            have_input = true;
        } else if (arg == "--output") {
            opt.output_path = val;
        } else if (arg == "--report") {
            opt.report_path = val;
        } else if (arg == "--sigma-s" || arg == "--sigma-r" || arg == "--epsilon") {
            if (!to_double(val, d)) return usage_error(arg + ": not a number: " + val);
            (arg == "--sigma-s" ? opt.sigma_s : arg == "--sigma-r" ? opt.sigma_r : opt.epsilon) = d;
            have_sigma_s |= arg == "--sigma-s";
        } else if (arg == "--kernel") {
            if (val == "gaussian") {
                opt.kernel_family = fourierbf::RangeFamily::gaussian;
            } else if (val == "exponential") {
                opt.kernel_family = fourierbf::RangeFamily::exponential;
            } else if (val.rfind("tabulated:", 0) == 0 && val.size() > 10) {
                opt.kernel_family = fourierbf::RangeFamily::tabulated;
                opt.tabulated_path = val.substr(10);
            } else {
                std::cerr << "error: --kernel must be gaussian, exponential, or tabulated:<path>\n";
                return 1;
            }
        } else if (arg == "--spatial") {
            if (val != "gaussian" && val != "box") return usage_error("--spatial must be gaussian or box");
            opt.spatial_kind = val == "box" ? fourierbf::SpatialKind::box : fourierbf::SpatialKind::gaussian;
        } else if (arg == "--backend") {
            if (val != "direct" && val != "recursive") return usage_error("--backend must be direct or recursive");
            opt.backend = val == "recursive" ? fourierbf::ConvolutionBackend::recursive
                                             : fourierbf::ConvolutionBackend::direct;
        } else {
            return usage_error("unknown option " + arg);
        }
    }
    if (!have_input) return usage_error("--input is required");
    if (!have_sigma_s) return usage_error("--sigma-s is required");
    return fourierbf::run(opt, std::cout, std::cerr);
}
