// Host-side scene (SoA) shared by the scene generators and the scene IO of
// the host library (libsfmcov_synth.so); the C ABI hands it out as the
// opaque sfmcov_synth_scene.
#pragma once

#include <cstdint>
#include <vector>

namespace sfmhost {
struct Scene {
    int P = 8;
    std::vector<double> cams;   // n × P
    std::vector<double> pts;    // m × 3
    std::vector<int32_t> oc, op;
    std::vector<double> u;      // t × 2
    std::vector<double> sigma;  // t × 4
    int64_t n() const { return (int64_t)cams.size() / P; }
    int64_t m() const { return (int64_t)pts.size() / 3; }
    int64_t t() const { return (int64_t)oc.size(); }
};
}  // namespace sfmhost

struct sfmcov_synth_scene {
    sfmhost::Scene s;
};
