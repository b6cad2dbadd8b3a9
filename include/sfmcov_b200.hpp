// sfmcov_b200.hpp — C++ drop-in for the reference `sfmcov` covariance entry
// point, over the C ABI of sfmcov_b200.h (no Eigen, no torch).
//
// Mirrors include/sfmcov/types.hpp, error.hpp and covariance.hpp of the
// reference with Eigen-free value types of the same field names, so callers
// of sfmcov::compute_covariance (tools/sfmcov_cli.cpp:100,
// src/subrec.cpp:207, tests) switch by changing the include and linking
// libsfmcov_b200.so.  Camera blocks are returned as row-major 8x8 arrays
// (the reference's Mat8 is column-major but symmetric blocks read the same).
#pragma once

#include "sfmcov_b200.h"

#include <array>
#include <cstdint>
#include <memory>
#include <stdexcept>
#include <string>
#include <utility>
#include <vector>

namespace sfmcov {

using Vec2 = std::array<double, 2>;
using Vec3 = std::array<double, 3>;
using Mat2 = std::array<double, 4>;  // row-major
using Mat8 = std::array<double, 64>; // row-major
using Mat3 = std::array<double, 9>;  // row-major
using Index = std::int64_t;

inline constexpr int kCameraParams = 8;
inline constexpr int kPointParams = 3;
inline constexpr int kGaugeDim = 7;

// include/sfmcov/types.hpp:28-66
struct Camera {
    Vec3 r{0, 0, 0};
    Vec3 C{0, 0, 0};
    double c = 1.0;
    double k = 0.0;
};
struct Point3D {
    Vec3 X{0, 0, 0};
};
struct Observation {
    std::int32_t cam_index = 0;
    std::int32_t point_index = 0;
    Vec2 u{0, 0};
    Mat2 sigma{1, 0, 0, 1};
};
struct Reconstruction {
    std::vector<Camera> cameras;
    std::vector<Point3D> points;
    std::vector<Observation> observations;
    Index num_cameras() const { return (Index)cameras.size(); }
    Index num_points() const { return (Index)points.size(); }
    Index num_observations() const { return (Index)observations.size(); }
    Index num_parameters() const { return kCameraParams * num_cameras() + kPointParams * num_points(); }
};

// include/sfmcov/error.hpp:9-33
enum class ErrorKind { io = 1, parse, invariant, degenerate, dimension, size_guard, device };

class Error : public std::runtime_error {
public:
    Error(ErrorKind kind, std::string stage, const std::string& what)
        : std::runtime_error(what), kind_(kind), stage_(std::move(stage)) {}
    ErrorKind kind() const { return kind_; }
    const std::string& stage() const { return stage_; }

private:
    ErrorKind kind_;
    std::string stage_;
};

// include/sfmcov/covariance.hpp:49-75
struct CovarianceDiagnostics {
    double scale_min = 0.0;
    double scale_max = 0.0;
    std::vector<Index> flagged_columns;
    double min_pivot = 0.0;
    double max_pivot = 0.0;
    int inertia_positive = 0;
    int inertia_negative = 0;
    int negative_eigenvalue_warnings = 0;
    std::size_t peak_dense_bytes = 0;
    Index largest_dense_dim = 0;
};

struct CovarianceResult {
    std::vector<Mat8> camera_cov;
    std::vector<Mat3> point_cov;        // filled when options.point_covariances
    std::vector<double> camera_matrix;  // (8n x 8n, column-major) when options.camera_cross_covariances
    Index camera_matrix_rows = 0;
    CovarianceDiagnostics diagnostics;

    // block (i, j) of the camera matrix (covariance.hpp:67), row-major 8 x 8
    Mat8 cross_block(Index i, Index j) const {
        Mat8 b{};
        for (int p = 0; p < 8; ++p)
            for (int q = 0; q < 8; ++q) b[8 * p + q] = camera_matrix[(size_t)(8 * j + q) * camera_matrix_rows + 8 * i + p];
        return b;
    }
};

struct CovarianceOptions {
    int threads = 0;
    bool point_covariances = false;
    bool camera_cross_covariances = false;
};

namespace b200 {

inline void check(int32_t code, const sfmcov_error& e) {
    if (code) throw Error(static_cast<ErrorKind>(code), e.stage, e.message);
}

// One CUDA handle per thread of use; created lazily on device 0.
inline sfmcov_handle* default_handle() {
    struct Holder {
        sfmcov_handle* h = nullptr;
        ~Holder() { if (h) sfmcov_cuda_destroy(h); }
    };
    thread_local Holder holder;
    if (!holder.h) {
        sfmcov_error e{};
        holder.h = sfmcov_cuda_create(0, &e);
        if (!holder.h) throw Error(ErrorKind::device, "device", e.message);
    }
    return holder.h;
}

}  // namespace b200

// compute_covariance (include/sfmcov/covariance.hpp:110-111): validation,
// Jacobian, gauge nullspace, Fisher blocks, conditioning, Schur reduction and
// the gauge-fixed inversion all run on the GPU.
inline CovarianceResult compute_covariance(const Reconstruction& rec, const CovarianceOptions& options = {}) {
    const Index n = rec.num_cameras(), m = rec.num_points(), t = rec.num_observations();
    std::vector<double> cams(8 * n), pts(3 * m), u(2 * t), sigma(4 * t);
    std::vector<std::int32_t> oc(t), op(t);
    for (Index i = 0; i < n; ++i) {
        const Camera& c = rec.cameras[i];
        double* o = &cams[8 * i];
        o[0] = c.r[0]; o[1] = c.r[1]; o[2] = c.r[2];
        o[3] = c.C[0]; o[4] = c.C[1]; o[5] = c.C[2];
        o[6] = c.c; o[7] = c.k;
    }
    for (Index j = 0; j < m; ++j)
        for (int a = 0; a < 3; ++a) pts[3 * j + a] = rec.points[j].X[a];
    for (Index k = 0; k < t; ++k) {
        const Observation& ob = rec.observations[k];
        oc[k] = ob.cam_index;
        op[k] = ob.point_index;
        u[2 * k] = ob.u[0];
        u[2 * k + 1] = ob.u[1];
        for (int a = 0; a < 4; ++a) sigma[4 * k + a] = ob.sigma[a];
    }
    sfmcov_scene s{(int32_t)n, (int32_t)m, (int32_t)t, 8, cams.data(), pts.data(), oc.data(), op.data(),
                   u.data(), sigma.data()};
    sfmcov_options o{options.threads, options.point_covariances ? 1 : 0, options.camera_cross_covariances ? 1 : 0, 0};
    CovarianceResult result;
    result.camera_cov.resize(n);
    std::vector<int64_t> flagged(8 * n + 3 * m + 1);
    sfmcov_diagnostics d{};
    d.flagged = flagged.data();
    d.flagged_capacity = (int64_t)flagged.size();
    sfmcov_error e{};
    if (options.point_covariances) result.point_cov.resize(m);
    if (options.camera_cross_covariances) {
        result.camera_matrix_rows = 8 * n;
        result.camera_matrix.resize((size_t)(8 * n) * (8 * n));
    }
    b200::check(sfmcov_cuda_compute_covariance_full(
                    b200::default_handle(), &s, &o, result.camera_cov.empty() ? nullptr : result.camera_cov[0].data(),
                    result.point_cov.empty() ? nullptr : result.point_cov[0].data(),
                    result.camera_matrix.empty() ? nullptr : result.camera_matrix.data(), &d, &e),
                e);
    CovarianceDiagnostics& g = result.diagnostics;
    g.scale_min = d.scale_min;
    g.scale_max = d.scale_max;
    g.flagged_columns.assign(flagged.begin(), flagged.begin() + d.n_flagged);
    g.min_pivot = d.min_pivot;
    g.max_pivot = d.max_pivot;
    g.inertia_positive = d.inertia_positive;
    g.inertia_negative = d.inertia_negative;
    g.negative_eigenvalue_warnings = d.negative_eigenvalue_warnings;
    g.peak_dense_bytes = (std::size_t)d.peak_dense_bytes;
    g.largest_dense_dim = d.largest_dense_dim;
    return result;
}

}  // namespace sfmcov
