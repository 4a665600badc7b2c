// Scene construction shared by the host renderers (synth_host.cpp) and the
// device renderers (synth.cu) of the synthetic generator (fscan_synth.h).
// Harness code: it builds inputs for tests and the bench outside any timed region.
#pragma once

#include <vector>

#include "fscan_synth.h"
#include "synth_common.h"

namespace fsynth {

struct PairScene {
    std::vector<Object> a, b;
    double theta = 0, tx = 0, ty = 0;
};

// Objects of pair `pair` (scan A) and the same objects moved by its pose (scan B).
void build_scene(const fscan_synth_spec& s, int pair, PairScene* out);

// Scan k of the generated drive `seq` (odometry workload): the scene of pair
// `seq` with its objects moved by pose P_k (P_0 = identity).
void sequence_scan(const fscan_synth_spec& s, int seq, int k, const PairScene& base, std::vector<Object>* out,
                   double* pose);

}  // namespace fsynth
