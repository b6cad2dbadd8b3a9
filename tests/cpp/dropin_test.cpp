// C++ drop-in check: a reference-style caller (tests/test_covariance.cpp:16-40
// of the reference) compiled against include/sfmcov_b200.hpp.  Exit 0 = pass.
#include "sfmcov_b200.hpp"

#include <cmath>
#include <cstdio>
#include <string>
#include <vector>

using namespace sfmcov;

static Reconstruction cube_scene(uint64_t seed, double noise) {
    sfmcov_synth_scene* h = sfmcov_synth_cube(seed, noise, 8);
    int64_t n, m, t;
    int32_t P;
    sfmcov_synth_sizes(h, &n, &m, &t, &P);
    std::vector<double> cams(n * P), pts(m * 3), u(t * 2), sg(t * 4);
    std::vector<int32_t> oc(t), op(t);
    sfmcov_synth_export(h, cams.data(), pts.data(), oc.data(), op.data(), u.data(), sg.data());
    sfmcov_synth_free(h);
    Reconstruction rec;
    for (int64_t i = 0; i < n; ++i) {
        Camera c;
        for (int a = 0; a < 3; ++a) { c.r[a] = cams[P * i + a]; c.C[a] = cams[P * i + 3 + a]; }
        c.c = cams[P * i + 6];
        c.k = cams[P * i + 7];
        rec.cameras.push_back(c);
    }
    for (int64_t j = 0; j < m; ++j) rec.points.push_back(Point3D{{pts[3 * j], pts[3 * j + 1], pts[3 * j + 2]}});
    for (int64_t k = 0; k < t; ++k) {
        Observation o;
        o.cam_index = oc[k];
        o.point_index = op[k];
        o.u = {u[2 * k], u[2 * k + 1]};
        o.sigma = {sg[4 * k], sg[4 * k + 1], sg[4 * k + 2], sg[4 * k + 3]};
        rec.observations.push_back(o);
    }
    return rec;
}

#define CHECK(c) do { if (!(c)) { std::printf("FAIL %s:%d %s\n", __FILE__, __LINE__, #c); return 1; } } while (0)

int main() {
    const Reconstruction rec = cube_scene(1, 0.5);
    const CovarianceResult result = compute_covariance(rec);
    CHECK(result.camera_cov.size() == 6);
    const CovarianceDiagnostics& d = result.diagnostics;
    CHECK(d.inertia_positive == 48 && d.inertia_negative == 7);
    CHECK(d.largest_dense_dim == 55);
    CHECK(d.flagged_columns.empty() && d.negative_eigenvalue_warnings == 0);
    CHECK(d.min_pivot > 1e-12 * d.max_pivot);
    for (const Mat8& c : result.camera_cov) {
        double mx = 0.0;
        for (double v : c) mx = std::fmax(mx, std::fabs(v));
        for (int p = 0; p < 8; ++p) {
            CHECK(c[9 * p] > 0.0);
            // unscaling multiplies mirrored triangles in opposite order: symmetric to the ulp
            for (int q = 0; q < 8; ++q) CHECK(std::fabs(c[8 * p + q] - c[8 * q + p]) <= 1e-14 * mx);
        }
    }
    // optional outputs (test_covariance.cpp:42-68 shape): point blocks, full camera matrix whose
    // diagonal blocks are the camera blocks bitwise
    CovarianceOptions opts;
    opts.point_covariances = true;
    opts.camera_cross_covariances = true;
    const CovarianceResult full = compute_covariance(rec, opts);
    CHECK(full.point_cov.size() == (size_t)rec.num_points());
    CHECK(full.camera_matrix_rows == 48);
    for (Index i = 0; i < 6; ++i) CHECK(full.cross_block(i, i) == full.camera_cov[i]);
    for (const Mat3& pc : full.point_cov) CHECK(pc[0] > 0.0 && pc[4] > 0.0 && pc[8] > 0.0);
    // errors keep the reference's kind / stage / message fragments
    Reconstruction bad = rec;
    bad.cameras[1].c = -1.0;
    try {
        compute_covariance(bad);
        CHECK(false);
    } catch (const Error& e) {
        CHECK(e.kind() == ErrorKind::invariant && e.stage() == "validate");
        CHECK(std::string(e.what()).find("camera 1 has non-positive focal length") != std::string::npos);
    }
    // print the first block so the Python test can compare against the oracle
    for (int q = 0; q < 64; ++q) std::printf("%.17g%c", result.camera_cov[0][q], q == 63 ? '\n' : ' ');
    std::printf("PASS\n");
    return 0;
}
