// sfmcov_b200.hpp — C++ drop-in for the reference `sfmcov` hot-path API, over
// the C ABI of sfmcov_b200.h (no Eigen, no torch).
//
// Mirrors the reference headers include/sfmcov/{types,error,projection,
// nullspace,covariance}.hpp with Eigen-free value types of the same names and
// fields, so a caller (tools/sfmcov_cli.cpp:100, src/subrec.cpp:207, the
// reference's own tests) switches by changing the include and linking
// libsfmcov_b200.so.  Every function runs on the GPU through the C ABI.
//
// Layout conventions (the reference uses Eigen column-major matrices):
//   * fixed-size blocks (Mat2, Mat3, Mat8, Mat28, Mat23, Mat83) are
//     std::array, ROW-major: element (r, c) of an R x C block at [C r + c]
//     (symmetric blocks read the same either way);
//   * MatX is column-major like Eigen's MatrixXd: (r, c) at data[rows c + r].
// The camera model is the reference's (P = 8: r, C, c, k); the BASELINE P = 9
// camera is reachable through the C ABI (sfmcov_scene.cam_params = 9).
#pragma once

#include "sfmcov_b200.h"

#include <array>
#include <cmath>
#include <cstdint>
#include <cstring>
#include <map>
#include <memory>
#include <mutex>
#include <stdexcept>
#include <string>
#include <utility>
#include <vector>

namespace sfmcov {

using Index = std::int64_t;
using Vec2 = std::array<double, 2>;
using Vec3 = std::array<double, 3>;
using Mat2 = std::array<double, 4>;    // row-major 2 x 2
using Mat3 = std::array<double, 9>;    // row-major 3 x 3
using Mat8 = std::array<double, 64>;   // row-major 8 x 8
using Mat28 = std::array<double, 16>;  // row-major 2 x 8 (camera Jacobian block)
using Mat23 = std::array<double, 6>;   // row-major 2 x 3 (point Jacobian block)
using Mat83 = std::array<double, 24>;  // row-major 8 x 3 (coupling block)
using VecX = std::vector<double>;

inline constexpr int kCameraParams = 8;
inline constexpr int kPointParams = 3;
inline constexpr int kGaugeDim = 7;
inline constexpr double kPivotRtol = 1e-12;  // covariance.hpp:14
inline constexpr double kPsdTol = 1e-9;      // covariance.hpp:18

// Dense column-major matrix (the reference's MatX = Eigen::MatrixXd).
class MatX {
public:
    MatX() = default;
    MatX(Index rows, Index cols) : rows_(rows), cols_(cols), data_((size_t)(rows * cols), 0.0) {}
    static MatX Zero(Index rows, Index cols) { return MatX(rows, cols); }
    static MatX Identity(Index rows, Index cols) {
        MatX m(rows, cols);
        for (Index i = 0; i < std::min(rows, cols); ++i) m(i, i) = 1.0;
        return m;
    }
    Index rows() const { return rows_; }
    Index cols() const { return cols_; }
    double& operator()(Index r, Index c) { return data_[(size_t)(c * rows_ + r)]; }
    double operator()(Index r, Index c) const { return data_[(size_t)(c * rows_ + r)]; }
    double* data() { return data_.data(); }
    const double* data() const { return data_.data(); }
    bool operator==(const MatX& o) const { return rows_ == o.rows_ && cols_ == o.cols_ && data_ == o.data_; }

private:
    Index rows_ = 0, cols_ = 0;
    std::vector<double> data_;
};

// ---- error.hpp:9-33 -----------------------------------------------------------
enum class ErrorKind {
    io,          // unreadable or unwritable files
    parse,       // malformed input files
    invariant,   // reconstruction invariant violations, bad arguments
    degenerate,  // numerically degenerate scenes
    dimension,   // mismatched shapes between arguments
    size_guard,  // dense computation requested above its parameter limit
    device,      // (B200 only) no usable CUDA device / CUDA failure
};

class Error : public std::runtime_error {
public:
    Error(ErrorKind kind, std::string stage, const std::string& message)
        : std::runtime_error(stage + ": " + message), kind_(kind), stage_(std::move(stage)) {}
    ErrorKind kind() const { return kind_; }
    const std::string& stage() const { return stage_; }

private:
    ErrorKind kind_;
    std::string stage_;
};

// ---- types.hpp:28-80 ------------------------------------------------------------
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
struct ObservationIndex {
    std::vector<std::vector<std::int32_t>> by_camera;
    std::vector<std::vector<std::int32_t>> by_point;
};
struct Reconstruction {
    std::vector<Camera> cameras;
    std::vector<Point3D> points;
    std::vector<Observation> observations;
    Index num_cameras() const { return (Index)cameras.size(); }
    Index num_points() const { return (Index)points.size(); }
    Index num_observations() const { return (Index)observations.size(); }
    Index num_parameters() const { return kCameraParams * num_cameras() + kPointParams * num_points(); }
    // Throws Error(invariant) naming the offending camera/point/observation (on the GPU).
    inline void validate() const;
};

namespace b200 {

// Error kinds: C code k (1..6) is the reference's ErrorKind k - 1; 7 = device.
inline ErrorKind kind_of(int32_t code) {
    return (code >= 1 && code <= 6) ? static_cast<ErrorKind>(code - 1) : ErrorKind::device;
}
inline void check(int32_t code, const sfmcov_error& e) {
    if (!code) return;
    std::string msg = e.message;
    const std::string pre = std::string(e.stage) + ": ";
    if (msg.compare(0, pre.size(), pre) == 0) msg = msg.substr(pre.size());
    throw Error(kind_of(code), e.stage, msg);
}

// One shared handle per device for the process (the handle serialises its
// calls with its own mutex; device memory is allocated once, not per thread).
inline sfmcov_handle* default_handle(int device = 0) {
    struct Registry {
        std::mutex mu;
        std::map<int, sfmcov_handle*> handles;
        ~Registry() {
            for (auto& kv : handles) sfmcov_cuda_destroy(kv.second);
        }
    };
    static Registry reg;
    std::lock_guard<std::mutex> lock(reg.mu);
    sfmcov_handle*& h = reg.handles[device];
    if (!h) {
        sfmcov_error e{};
        h = sfmcov_cuda_create(device, &e);
        if (!h) throw Error(ErrorKind::device, "device", e.message);
    }
    return h;
}

// The scene as the C ABI's structure of arrays (owned copy).
struct SceneSoA {
    int32_t n = 0, m = 0, t = 0;
    std::vector<double> cams, pts, u, sigma;
    std::vector<int32_t> oc, op;
    explicit SceneSoA(const Reconstruction& rec)
        : n((int32_t)rec.num_cameras()), m((int32_t)rec.num_points()), t((int32_t)rec.num_observations()),
          cams(8 * (size_t)n), pts(3 * (size_t)m), u(2 * (size_t)t), sigma(4 * (size_t)t), oc(t), op(t) {
        for (int32_t i = 0; i < n; ++i) {
            const Camera& c = rec.cameras[i];
            double* o = &cams[8 * (size_t)i];
            o[0] = c.r[0]; o[1] = c.r[1]; o[2] = c.r[2];
            o[3] = c.C[0]; o[4] = c.C[1]; o[5] = c.C[2];
            o[6] = c.c; o[7] = c.k;
        }
        for (int32_t j = 0; j < m; ++j)
            for (int a = 0; a < 3; ++a) pts[3 * (size_t)j + a] = rec.points[j].X[a];
        for (int32_t k = 0; k < t; ++k) {
            const Observation& ob = rec.observations[k];
            oc[k] = ob.cam_index;
            op[k] = ob.point_index;
            u[2 * (size_t)k] = ob.u[0];
            u[2 * (size_t)k + 1] = ob.u[1];
            for (int a = 0; a < 4; ++a) sigma[4 * (size_t)k + a] = ob.sigma[a];
        }
    }
    sfmcov_scene view() const {
        return sfmcov_scene{n, m, t, 8, cams.data(), pts.data(), oc.data(), op.data(), u.data(), sigma.data()};
    }
};

}  // namespace b200

// Reconstruction::validate (src/scene.cpp:19-78) and build_observation_index
// (src/scene.cpp:80-90): the device validation and CSR index.
inline ObservationIndex build_observation_index(const Reconstruction& rec) {
    const b200::SceneSoA s(rec);
    const sfmcov_scene v = s.view();
    std::vector<int64_t> oc((size_t)s.n + 1), op((size_t)s.m + 1);
    std::vector<int32_t> ic((size_t)std::max(s.t, 1)), ip((size_t)std::max(s.t, 1));
    sfmcov_error e{};
    b200::check(sfmcov_cuda_observation_index(b200::default_handle(), &v, oc.data(), ic.data(), op.data(), ip.data(), &e),
                e);
    ObservationIndex ix;
    ix.by_camera.resize(s.n);
    ix.by_point.resize(s.m);
    for (int32_t i = 0; i < s.n; ++i) ix.by_camera[i].assign(ic.begin() + oc[i], ic.begin() + oc[i + 1]);
    for (int32_t j = 0; j < s.m; ++j) ix.by_point[j].assign(ip.begin() + op[j], ip.begin() + op[j + 1]);
    return ix;
}
inline void Reconstruction::validate() const { (void)build_observation_index(*this); }

// ---- projection.hpp:31-54 ----------------------------------------------------------
struct JacobianBlock {
    std::int32_t cam_index = 0;
    std::int32_t point_index = 0;
    Mat28 cam_block{};
    Mat23 point_block{};
};
struct SparseJacobian {
    Index n_cams = 0;
    Index n_pts = 0;
    std::vector<JacobianBlock> blocks;  // observation order
    Index rows() const { return 2 * (Index)blocks.size(); }
    Index cols() const { return kCameraParams * n_cams + kPointParams * n_pts; }
    Index cam_col(Index i) const { return kCameraParams * i; }
    Index point_col(Index j) const { return kCameraParams * n_cams + kPointParams * j; }
    double max_abs() const {
        double m = 0.0;
        for (const JacobianBlock& b : blocks) {
            for (double v : b.cam_block) m = std::max(m, std::fabs(v));
            for (double v : b.point_block) m = std::max(m, std::fabs(v));
        }
        return m;
    }
    MatX dense() const {
        MatX J = MatX::Zero(rows(), cols());
        for (size_t t = 0; t < blocks.size(); ++t)
            for (int r = 0; r < 2; ++r) {
                for (int p = 0; p < 8; ++p) J(2 * (Index)t + r, cam_col(blocks[t].cam_index) + p) = blocks[t].cam_block[8 * r + p];
                for (int q = 0; q < 3; ++q) J(2 * (Index)t + r, point_col(blocks[t].point_index) + q) = blocks[t].point_block[3 * r + q];
            }
        return J;
    }
    // (B200) the scene the Jacobian was assembled from: the GPU nullspace
    // routines re-derive what they need from it
    std::shared_ptr<const b200::SceneSoA> source;
};

// assemble_jacobian (projection.hpp:54, src/projection.cpp:80-105) on the GPU.
inline SparseJacobian assemble_jacobian(const Reconstruction& rec, int threads = 1) {
    (void)threads;
    auto s = std::make_shared<const b200::SceneSoA>(rec);
    const sfmcov_scene v = s->view();
    std::vector<double> jc(16 * (size_t)s->t + 1), jp(6 * (size_t)s->t + 1);
    sfmcov_error e{};
    b200::check(sfmcov_cuda_jacobian(b200::default_handle(), &v, jc.data(), jp.data(), &e), e);
    SparseJacobian J;
    J.n_cams = s->n;
    J.n_pts = s->m;
    J.blocks.resize(s->t);
    for (int32_t k = 0; k < s->t; ++k) {
        JacobianBlock& b = J.blocks[k];
        b.cam_index = s->oc[k];
        b.point_index = s->op[k];
        std::memcpy(b.cam_block.data(), &jc[16 * (size_t)k], sizeof b.cam_block);
        std::memcpy(b.point_block.data(), &jp[6 * (size_t)k], sizeof b.point_block);
    }
    J.source = std::move(s);
    return J;
}

// ---- nullspace.hpp:22-36 ------------------------------------------------------------
namespace b200 {
inline MatX gpu_nullspace(const SceneSoA& s) {
    const sfmcov_scene v = s.view();
    const Index rows = 8 * (Index)s.n + 3 * (Index)s.m;
    std::vector<double> hr((size_t)rows * kGaugeDim + 1);
    sfmcov_error e{};
    check(sfmcov_cuda_nullspace(default_handle(), &v, hr.data(), &e), e);
    MatX h(rows, kGaugeDim);
    for (Index r = 0; r < rows; ++r)
        for (int l = 0; l < kGaugeDim; ++l) h(r, l) = hr[(size_t)(r * kGaugeDim + l)];
    return h;
}
inline std::vector<double> row_major(const MatX& h) {
    std::vector<double> out((size_t)(h.rows() * h.cols()) + 1);
    for (Index r = 0; r < h.rows(); ++r)
        for (Index c = 0; c < h.cols(); ++c) out[(size_t)(r * h.cols() + c)] = h(r, c);
    return out;
}
inline MatX from_row_major(const double* a, Index rows, Index cols) {
    MatX m(rows, cols);
    for (Index r = 0; r < rows; ++r)
        for (Index c = 0; c < cols; ++c) m(r, c) = a[r * cols + c];
    return m;
}
}  // namespace b200

// Closed-form rows [I | [C]x | C], [I | [X]x | X]; rotation rows left zero.
inline MatX fixed_nullspace_blocks(const Reconstruction& rec) {
    MatX h = b200::gpu_nullspace(b200::SceneSoA(rec));
    for (Index i = 0; i < rec.num_cameras(); ++i)
        for (int a = 0; a < 3; ++a)
            for (int l = 0; l < kGaugeDim; ++l) h(8 * i + a, l) = 0.0;
    return h;
}
// The camera-rotation 3x3 blocks from the per-camera normal equations.
inline void solve_rotation_blocks(const SparseJacobian& jac, MatX& h) {
    if (h.rows() != jac.cols() || h.cols() != kGaugeDim || !jac.source)
        throw Error(ErrorKind::dimension, "nullspace", "nullspace shape does not match Jacobian");
    const MatX full = b200::gpu_nullspace(*jac.source);
    for (Index i = 0; i < jac.n_cams; ++i)
        for (int a = 0; a < 3; ++a)
            for (int b = 0; b < 3; ++b) h(8 * i + a, 3 + b) = full(8 * i + a, 3 + b);
}
inline MatX gauge_nullspace(const SparseJacobian& jac, const Reconstruction& rec) {
    MatX h = fixed_nullspace_blocks(rec);
    solve_rotation_blocks(jac, h);
    return h;
}
// max |J H| / (max |J| max |H|) (nullspace.hpp:36), reduced on the GPU.
inline double nullspace_residual(const SparseJacobian& jac, const MatX& h) {
    if (h.rows() != jac.cols() || h.cols() < 1 || !jac.source)
        throw Error(ErrorKind::dimension, "nullspace", "nullspace shape does not match Jacobian");
    const sfmcov_scene v = jac.source->view();
    const std::vector<double> hr = b200::row_major(h);
    double res = 0.0;
    sfmcov_error e{};
    b200::check(sfmcov_cuda_nullspace_residual(b200::default_handle(), &v, hr.data(), (int32_t)h.cols(), &res, &e), e);
    return res;
}

// ---- covariance.hpp:20-115 ----------------------------------------------------------
struct ConditioningScales {
    VecX s_a;                    // parameter column scales, length 8n+3m
    VecX s_b;                    // border column scales
    std::vector<Index> flagged;  // parameter columns that fell back to scale 1
};
struct Coupling {
    std::int32_t cam_index = 0;
    std::int32_t point_index = 0;
    Mat83 block{};  // M[P_i, X_j], row-major 8 x 3
};
struct BorderedSystem {
    Index n_cams = 0;
    Index n_pts = 0;
    std::vector<Mat8> cam_blocks;
    std::vector<Mat3> point_blocks;
    std::vector<Coupling> couplings;  // observation order
    std::vector<std::vector<std::int32_t>> obs_by_point;
    MatX border;  // (8n+3m) x b
    bool conditioned = false;
    Index border_cols() const { return border.cols(); }
};
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
    std::vector<Mat3> point_cov;  // filled when options.point_covariances
    MatX camera_matrix;           // 8n x 8n, when options.camera_cross_covariances
    CovarianceDiagnostics diagnostics;
    // block (i, j) of the camera matrix (covariance.hpp:67), row-major 8 x 8
    Mat8 cross_block(Index i, Index j) const {
        Mat8 b{};
        for (int p = 0; p < 8; ++p)
            for (int q = 0; q < 8; ++q) b[8 * p + q] = camera_matrix(8 * i + p, 8 * j + q);
        return b;
    }
};
struct CovarianceOptions {
    int threads = 0;
    bool point_covariances = false;
    bool camera_cross_covariances = false;
};

namespace b200 {
// the system as the C ABI's arrays
struct SystemArrays {
    int32_t n, m, t, b;
    std::vector<double> D, A, C, border;
    std::vector<int32_t> oc, op;
    explicit SystemArrays(const BorderedSystem& sys)
        : n((int32_t)sys.n_cams), m((int32_t)sys.n_pts), t((int32_t)sys.couplings.size()),
          b((int32_t)sys.border_cols()), D(64 * (size_t)n + 1), A(9 * (size_t)m + 1), C(24 * (size_t)t + 1),
          border(row_major(sys.border)), oc((size_t)t + 1), op((size_t)t + 1) {
        for (int32_t i = 0; i < n; ++i) std::memcpy(&D[64 * (size_t)i], sys.cam_blocks[i].data(), sizeof(Mat8));
        for (int32_t j = 0; j < m; ++j) std::memcpy(&A[9 * (size_t)j], sys.point_blocks[j].data(), sizeof(Mat3));
        for (int32_t k = 0; k < t; ++k) {
            std::memcpy(&C[24 * (size_t)k], sys.couplings[k].block.data(), sizeof(Mat83));
            oc[k] = sys.couplings[k].cam_index;
            op[k] = sys.couplings[k].point_index;
        }
    }
};
}  // namespace b200

// build_fisher_blocks (covariance.hpp:80-81, src/covariance.cpp:33-82): the
// Fisher blocks of the scene on the GPU, the border attached as given.
inline BorderedSystem build_fisher_blocks(const SparseJacobian& jac, const Reconstruction& rec, MatX border,
                                          int threads = 1) {
    (void)threads;
    if (border.rows() != jac.cols())
        throw Error(ErrorKind::dimension, "fisher", "border row count does not match Jacobian");
    const b200::SceneSoA s(rec);
    const sfmcov_scene v = s.view();
    std::vector<double> D(64 * (size_t)s.n + 1), A(9 * (size_t)s.m + 1), C(24 * (size_t)s.t + 1);
    sfmcov_error e{};
    b200::check(sfmcov_cuda_fisher(b200::default_handle(), &v, D.data(), A.data(), C.data(), nullptr, nullptr, nullptr, &e),
                e);
    BorderedSystem sys;
    sys.n_cams = s.n;
    sys.n_pts = s.m;
    sys.border = std::move(border);
    sys.cam_blocks.resize(s.n);
    sys.point_blocks.resize(s.m);
    sys.couplings.resize(s.t);
    for (int32_t i = 0; i < s.n; ++i) std::memcpy(sys.cam_blocks[i].data(), &D[64 * (size_t)i], sizeof(Mat8));
    for (int32_t j = 0; j < s.m; ++j) std::memcpy(sys.point_blocks[j].data(), &A[9 * (size_t)j], sizeof(Mat3));
    sys.obs_by_point.assign(s.m, {});
    for (int32_t k = 0; k < s.t; ++k) {
        Coupling& c = sys.couplings[k];
        c.cam_index = s.oc[k];
        c.point_index = s.op[k];
        std::memcpy(c.block.data(), &C[24 * (size_t)k], sizeof(Mat83));
        sys.obs_by_point[s.op[k]].push_back(k);  // ascending observation order
    }
    return sys;
}

inline ConditioningScales condition_columns(const BorderedSystem& sys) {
    const b200::SystemArrays a(sys);
    const Index rows = 8 * (Index)a.n + 3 * (Index)a.m;
    ConditioningScales sc;
    sc.s_a.resize(rows);
    sc.s_b.resize(a.b);
    std::vector<int64_t> fl((size_t)rows + 1);
    int64_t nf = 0;
    sfmcov_error e{};
    b200::check(sfmcov_cuda_condition_columns(b200::default_handle(), a.n, a.m, 8, a.b, a.D.data(), a.A.data(),
                                              a.border.data(), sc.s_a.data(), sc.s_b.data(), fl.data(),
                                              (int64_t)fl.size(), &nf, &e),
                e);
    sc.flagged.assign(fl.begin(), fl.begin() + nf);
    return sc;
}

inline void apply_conditioning(BorderedSystem& sys, const ConditioningScales& scales) {
    b200::SystemArrays a(sys);
    sfmcov_error e{};
    b200::check(sfmcov_cuda_apply_conditioning(b200::default_handle(), a.n, a.m, a.t, 8, a.b, a.D.data(), a.A.data(),
                                               a.C.data(), a.oc.data(), a.op.data(), a.border.data(), scales.s_a.data(),
                                               scales.s_b.data(), &e),
                e);
    for (int32_t i = 0; i < a.n; ++i) std::memcpy(sys.cam_blocks[i].data(), &a.D[64 * (size_t)i], sizeof(Mat8));
    for (int32_t j = 0; j < a.m; ++j) std::memcpy(sys.point_blocks[j].data(), &a.A[9 * (size_t)j], sizeof(Mat3));
    for (int32_t k = 0; k < a.t; ++k) std::memcpy(sys.couplings[k].block.data(), &a.C[24 * (size_t)k], sizeof(Mat83));
    sys.border = b200::from_row_major(a.border.data(), sys.border.rows(), sys.border.cols());
    sys.conditioned = true;
}

// schur_reduce (covariance.hpp:94-95): Z_p = D_p - B_p^T A_p^-1 B_p, dense
// (8n+b) square, exactly symmetric; point_block_inverses = the A_j^-1.
inline MatX schur_reduce(const BorderedSystem& sys, CovarianceDiagnostics* diag = nullptr, int threads = 1,
                         std::vector<Mat3>* point_block_inverses = nullptr) {
    (void)threads;
    const b200::SystemArrays a(sys);
    const Index dim = 8 * (Index)a.n + a.b;
    MatX z(dim, dim);
    std::vector<double> ainv(point_block_inverses ? 9 * (size_t)a.m + 1 : 0);
    sfmcov_error e{};
    b200::check(sfmcov_cuda_schur_system(b200::default_handle(), a.n, a.m, a.t, 8, a.b, a.D.data(), a.A.data(),
                                         a.C.data(), a.oc.data(), a.op.data(), a.border.data(), z.data(),
                                         point_block_inverses ? ainv.data() : nullptr, &e),
                e);
    if (point_block_inverses) {
        point_block_inverses->resize(a.m);
        for (int32_t j = 0; j < a.m; ++j) std::memcpy((*point_block_inverses)[j].data(), &ainv[9 * (size_t)j], sizeof(Mat3));
    }
    if (diag) {
        diag->largest_dense_dim = std::max(diag->largest_dense_dim, dim);
        diag->peak_dense_bytes = std::max<std::size_t>(diag->peak_dense_bytes, sizeof(double) * (size_t)dim * (size_t)dim);
    }
    return z;
}

// invert_schur (covariance.hpp:100): inverse of a symmetric nonsingular
// matrix on the GPU (Jacobi eigendecomposition); pivots = |eigenvalues|.
inline MatX invert_schur(MatX z_p, CovarianceDiagnostics& diag) {
    const Index n = z_p.rows();
    if (z_p.cols() != n || n < 1) throw Error(ErrorKind::dimension, "factorization", "matrix must be square");
    MatX inv(n, n);
    int32_t pos = 0, neg = 0;
    sfmcov_error e{};
    b200::check(sfmcov_cuda_invert_symmetric(b200::default_handle(), z_p.data(), n, inv.data(), &diag.min_pivot,
                                             &diag.max_pivot, &pos, &neg, &e),
                e);
    diag.inertia_positive = pos;
    diag.inertia_negative = neg;
    diag.peak_dense_bytes = std::max<std::size_t>(diag.peak_dense_bytes, 2 * sizeof(double) * (size_t)n * (size_t)n);
    return inv;
}

// extract_camera_covariances (covariance.hpp:104-105).
inline CovarianceResult extract_camera_covariances(const MatX& z_inv, const ConditioningScales& scales, Index n_cams,
                                                   CovarianceDiagnostics diag = {}) {
    CovarianceResult result;
    result.camera_cov.resize(n_cams);
    int32_t warn = 0;
    sfmcov_error e{};
    b200::check(sfmcov_cuda_extract_camera_blocks(b200::default_handle(), z_inv.data(), z_inv.rows(), (int32_t)n_cams, 8,
                                                  scales.s_a.empty() ? nullptr : scales.s_a.data(),
                                                  n_cams ? result.camera_cov[0].data() : nullptr, &warn, &e),
                e);
    diag.negative_eigenvalue_warnings += warn;
    if (scales.s_a.empty()) {
        diag.scale_min = diag.scale_max = 1.0;
    } else {
        diag.scale_min = diag.scale_max = scales.s_a[0];
        for (double v : scales.s_a) {
            diag.scale_min = std::min(diag.scale_min, v);
            diag.scale_max = std::max(diag.scale_max, v);
        }
    }
    diag.flagged_columns = scales.flagged;
    result.diagnostics = std::move(diag);
    return result;
}

// compute_covariance (covariance.hpp:110-111): validation, Jacobian, gauge
// nullspace, Fisher blocks, conditioning, Schur reduction and the
// gauge-fixed inversion, fused on the GPU.
inline CovarianceResult compute_covariance(const Reconstruction& rec, const CovarianceOptions& options = {}) {
    const b200::SceneSoA s(rec);
    const sfmcov_scene v = s.view();
    const Index n = s.n, m = s.m;
    sfmcov_options o{options.threads, options.point_covariances ? 1 : 0, options.camera_cross_covariances ? 1 : 0, 0};
    CovarianceResult result;
    result.camera_cov.resize(n);
    std::vector<int64_t> flagged(8 * n + 3 * m + 1);
    sfmcov_diagnostics d{};
    d.flagged = flagged.data();
    d.flagged_capacity = (int64_t)flagged.size();
    sfmcov_error e{};
    if (options.point_covariances) result.point_cov.resize(m);
    if (options.camera_cross_covariances) result.camera_matrix = MatX(8 * n, 8 * n);
    b200::check(sfmcov_cuda_compute_covariance_full(
                    b200::default_handle(), &v, &o, result.camera_cov.empty() ? nullptr : result.camera_cov[0].data(),
                    result.point_cov.empty() ? nullptr : result.point_cov[0].data(),
                    options.camera_cross_covariances ? result.camera_matrix.data() : nullptr, &d, &e),
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

// full_covariance (covariance.hpp:115): the (8n+3m)^2 parameter covariance.
inline MatX full_covariance(const Reconstruction& rec, Index max_params = 2000) {
    if (rec.num_parameters() > max_params)
        throw Error(ErrorKind::size_guard, "full-covariance",
                    "scene has " + std::to_string(rec.num_parameters()) + " parameters, guard is " +
                        std::to_string(max_params));
    const b200::SceneSoA s(rec);
    const sfmcov_scene v = s.view();
    MatX sigma(rec.num_parameters(), rec.num_parameters());
    sfmcov_error e{};
    b200::check(sfmcov_cuda_full_covariance(b200::default_handle(), &v, max_params, sigma.data(), &e), e);
    return sigma;
}

// ---- covariance_io.hpp:10-24 (host library libsfmcov_synth.so) ---------------
inline std::array<double, 36> pack_upper_triangle(const Mat8& m) {
    std::array<double, 36> tri{};
    sfmcov_covio_pack_upper_triangle(m.data(), 8, tri.data());
    return tri;
}
inline Mat8 unpack_upper_triangle(const std::array<double, 36>& tri) {
    Mat8 m{};
    sfmcov_covio_unpack_upper_triangle(tri.data(), 8, m.data());
    return m;
}
inline void save_covariance_json(const CovarianceResult& result, const std::string& path) {
    const CovarianceDiagnostics& g = result.diagnostics;
    std::vector<int64_t> fl(g.flagged_columns.begin(), g.flagged_columns.end());
    sfmcov_diagnostics d{g.scale_min, g.scale_max, g.min_pivot, g.max_pivot, g.inertia_positive, g.inertia_negative,
                         g.negative_eigenvalue_warnings, (int32_t)fl.size(), (int64_t)g.peak_dense_bytes,
                         g.largest_dense_dim, fl.data(), (int64_t)fl.size()};
    sfmcov_error e{};
    b200::check(sfmcov_covio_save_json(path.c_str(), (int64_t)result.camera_cov.size(), 8,
                                       result.camera_cov.empty() ? nullptr : result.camera_cov[0].data(), &d, &e),
                e);
}
inline CovarianceResult load_covariance_json(const std::string& path) {
    sfmcov_error e{};
    int64_t n = 0;
    sfmcov_diagnostics d{};
    b200::check(sfmcov_covio_load_json(path.c_str(), 8, 0, nullptr, &n, &d, &e), e);
    CovarianceResult r;
    r.camera_cov.resize(n);
    std::vector<int64_t> fl((size_t)d.n_flagged + 1);
    d.flagged = fl.data();
    d.flagged_capacity = (int64_t)fl.size();
    b200::check(sfmcov_covio_load_json(path.c_str(), 8, n, n ? r.camera_cov[0].data() : nullptr, &n, &d, &e), e);
    CovarianceDiagnostics& g = r.diagnostics;
    g.scale_min = d.scale_min;
    g.scale_max = d.scale_max;
    g.flagged_columns.assign(fl.begin(), fl.begin() + d.n_flagged);
    g.min_pivot = d.min_pivot;
    g.max_pivot = d.max_pivot;
    g.inertia_positive = d.inertia_positive;
    g.inertia_negative = d.inertia_negative;
    g.negative_eigenvalue_warnings = d.negative_eigenvalue_warnings;
    g.peak_dense_bytes = (std::size_t)d.peak_dense_bytes;
    g.largest_dense_dim = d.largest_dense_dim;
    return r;
}
inline void save_covariance_csv(const CovarianceResult& result, const std::string& path) {
    sfmcov_error e{};
    b200::check(sfmcov_covio_save_csv(path.c_str(), (int64_t)result.camera_cov.size(), 8,
                                      result.camera_cov.empty() ? nullptr : result.camera_cov[0].data(), &e),
                e);
}

}  // namespace sfmcov
