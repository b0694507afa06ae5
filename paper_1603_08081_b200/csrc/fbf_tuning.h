// fbf_tuning.h -- the measured tuning constants of the product library.
//
// The product build compiles every constant in: results and launch shapes do
// not depend on the process environment.  The experiment build
// (`make exp` -> _lib/libfourierbf_b200_exp.so, loaded by the A/B tools
// through FBF_LIBRARY) reads an FBF_<NAME> environment override for each, so
// the sweeps behind the defaults (profiles/r01_notes.md, r02_notes.md) can be
// re-run without rebuilding.
#pragma once
#include <cstdlib>

namespace fbf {

#ifdef FBF_EXPERIMENTS
inline double tunable(const char* env, double dflt) {
  const char* v = std::getenv(env);
  return v ? std::atof(v) : dflt;
}
#define FBF_TUNABLE(name, dflt) ::fbf::tunable("FBF_" #name, (dflt))
#else
#define FBF_TUNABLE(name, dflt) (dflt)
#endif

// the fused kernel's cut coordinate: a unit's prologue in rows of one harmonic
// per 2W (fbf_fused.cuh); the margin a larger harmonic-group count must win by
// in the group cost model (fbf_capi.cu pick_groups; the finish pass is in the model)
constexpr double kUnitCostFrac = 0.55;
constexpr double kGroupMargin = 0.99;
// host pipeline (fbf_hostpath.cpp plan_chunks)
constexpr double kPipelineMinPx = 1.0e6;  // calls below this many pixels run as one launch
constexpr int kBatchChunks = 16;          // image chunks of a batch call
constexpr double kStripPx = 0.3e6;        // strips K = round(sqrt(px / kStripPx)), at most 4
constexpr int kEdgeSmallPct = 35;         // first / last strip rows, % of a middle strip (<= 16 Mpixel)
constexpr int kEdgeLargePct = 20;         // ... above 16 Mpixel

}  // namespace fbf
