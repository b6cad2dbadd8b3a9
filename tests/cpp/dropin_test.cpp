// C++ drop-in check: reference-style callers compiled against
// include/sfmcov_b200.hpp (no Eigen).  Ports of the reference's own tests:
// tests/test_covariance.cpp:16-40, 42-68, 70-78, 120-135; test_fisher.cpp:42-100;
// test_schur.cpp:57-165; test_nullspace.cpp:53-69.  Exit 0 = pass.
#include "sfmcov_b200.hpp"

#include <cmath>
#include <cstdio>
#include <string>
#include <vector>

using namespace sfmcov;

static int g_fail = 0;
#define CHECK(c)                                                            \
    do {                                                                    \
        if (!(c)) {                                                         \
            std::printf("FAIL %s:%d %s\n", __FILE__, __LINE__, #c);         \
            ++g_fail;                                                       \
        }                                                                   \
    } while (0)

static Reconstruction from_synth(sfmcov_synth_scene* h) {
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
static Reconstruction cube_scene(uint64_t seed, double noise) { return from_synth(sfmcov_synth_cube(seed, noise, 8)); }
static Reconstruction random_scene(int64_t n, int64_t m, double vis, uint64_t seed, double noise) {
    return from_synth(sfmcov_synth_random(n, m, vis, seed, noise, 8));
}
// support.hpp:106-122: two cube scenes 100 apart, no shared observations
static Reconstruction disconnected_scene(uint64_t seed, double noise) {
    Reconstruction out = cube_scene(seed, noise);
    Reconstruction b = cube_scene(seed + 1, noise);
    const auto co = (int32_t)out.num_cameras(), po = (int32_t)out.num_points();
    for (Camera& c : b.cameras) c.C[0] += 100.0;
    for (Point3D& p : b.points) p.X[0] += 100.0;
    out.cameras.insert(out.cameras.end(), b.cameras.begin(), b.cameras.end());
    out.points.insert(out.points.end(), b.points.begin(), b.points.end());
    for (Observation o : b.observations) {
        o.cam_index += co;
        o.point_index += po;
        out.observations.push_back(o);
    }
    return out;
}

// ---- dense test helpers (test code, host) --------------------------------------
static double norm(const MatX& a) {
    double s = 0.0;
    for (Index c = 0; c < a.cols(); ++c)
        for (Index r = 0; r < a.rows(); ++r) s += a(r, c) * a(r, c);
    return std::sqrt(s);
}
static double rel_diff(const MatX& a, const MatX& b) {  // support.hpp rel_diff
    MatX d(a.rows(), a.cols());
    for (Index c = 0; c < a.cols(); ++c)
        for (Index r = 0; r < a.rows(); ++r) d(r, c) = a(r, c) - b(r, c);
    const double s = norm(b);
    return s > 0.0 ? norm(d) / s : norm(d);
}
template <size_t N>
static MatX block_of(const std::array<double, N>& a, int rows, int cols) {
    MatX m(rows, cols);
    for (int r = 0; r < rows; ++r)
        for (int c = 0; c < cols; ++c) m(r, c) = a[cols * r + c];
    return m;
}
static MatX sub(const MatX& a, Index r0, Index c0, Index rows, Index cols) {
    MatX m(rows, cols);
    for (Index c = 0; c < cols; ++c)
        for (Index r = 0; r < rows; ++r) m(r, c) = a(r0 + r, c0 + c);
    return m;
}
static MatX mul(const MatX& a, const MatX& b, bool ta = false) {
    const Index n = ta ? a.cols() : a.rows(), k = ta ? a.rows() : a.cols();
    MatX c(n, b.cols());
    for (Index j = 0; j < b.cols(); ++j)
        for (Index l = 0; l < k; ++l) {
            const double bv = b(l, j);
            if (bv == 0.0) continue;
            for (Index i = 0; i < n; ++i) c(i, j) += (ta ? a(l, i) : a(i, l)) * bv;
        }
    return c;
}
static MatX solve(MatX a, MatX b) {  // Gaussian elimination, partial pivoting
    const Index n = a.rows();
    for (Index c = 0; c < n; ++c) {
        Index p = c;
        for (Index r = c + 1; r < n; ++r)
            if (std::fabs(a(r, c)) > std::fabs(a(p, c))) p = r;
        for (Index j = 0; j < n; ++j) std::swap(a(c, j), a(p, j));
        for (Index j = 0; j < b.cols(); ++j) std::swap(b(c, j), b(p, j));
        for (Index r = c + 1; r < n; ++r) {
            const double f = a(r, c) / a(c, c);
            if (f == 0.0) continue;
            for (Index j = c; j < n; ++j) a(r, j) -= f * a(c, j);
            for (Index j = 0; j < b.cols(); ++j) b(r, j) -= f * b(c, j);
        }
    }
    for (Index c = n - 1; c >= 0; --c)
        for (Index j = 0; j < b.cols(); ++j) {
            double v = b(c, j);
            for (Index k = c + 1; k < n; ++k) v -= a(c, k) * b(k, j);
            b(c, j) = v / a(c, c);
        }
    return b;
}
static double max_abs_diff_identity(const MatX& a) {
    double m = 0.0;
    for (Index c = 0; c < a.cols(); ++c)
        for (Index r = 0; r < a.rows(); ++r) m = std::max(m, std::fabs(a(r, c) - (r == c ? 1.0 : 0.0)));
    return m;
}
static double asym(const MatX& a) {
    double m = 0.0;
    for (Index c = 0; c < a.cols(); ++c)
        for (Index r = 0; r < a.rows(); ++r) m = std::max(m, std::fabs(a(r, c) - a(c, r)));
    return m;
}

// test_fisher.cpp:18-29 / test_schur.cpp:19-26
static MatX dense_from_blocks(const BorderedSystem& sys) {
    const Index n = sys.n_cams, dim = 8 * n + 3 * sys.n_pts;
    MatX m(dim, dim);
    for (Index i = 0; i < n; ++i)
        for (int p = 0; p < 8; ++p)
            for (int q = 0; q < 8; ++q) m(8 * i + p, 8 * i + q) = sys.cam_blocks[i][8 * p + q];
    for (Index j = 0; j < sys.n_pts; ++j)
        for (int p = 0; p < 3; ++p)
            for (int q = 0; q < 3; ++q) m(8 * n + 3 * j + p, 8 * n + 3 * j + q) = sys.point_blocks[j][3 * p + q];
    for (const Coupling& c : sys.couplings)
        for (int p = 0; p < 8; ++p)
            for (int q = 0; q < 3; ++q) {
                m(8 * c.cam_index + p, 8 * n + 3 * c.point_index + q) += c.block[3 * p + q];
                m(8 * n + 3 * c.point_index + q, 8 * c.cam_index + p) += c.block[3 * p + q];
            }
    return m;
}
static BorderedSystem bordered_cube(uint64_t seed, double noise, bool with_border, bool conditioned) {
    const Reconstruction rec = cube_scene(seed, noise);
    const SparseJacobian jac = assemble_jacobian(rec);
    MatX border = with_border ? gauge_nullspace(jac, rec) : MatX::Zero(jac.cols(), 0);
    BorderedSystem sys = build_fisher_blocks(jac, rec, border, 1);
    if (conditioned) apply_conditioning(sys, condition_columns(sys));
    return sys;
}
// test_schur.cpp:29-52: dense elimination of the point block
static MatX dense_schur_reference(const BorderedSystem& sys) {
    const Index n = sys.n_cams, m = sys.n_pts, b = sys.border_cols();
    const MatX fisher = dense_from_blocks(sys);
    MatX d(8 * n + b, 8 * n + b);
    for (Index c = 0; c < 8 * n; ++c)
        for (Index r = 0; r < 8 * n; ++r) d(r, c) = fisher(r, c);
    for (Index r = 0; r < 8 * n; ++r)
        for (Index l = 0; l < b; ++l) d(r, 8 * n + l) = d(8 * n + l, r) = sys.border(r, l);
    const MatX a = sub(fisher, 8 * n, 8 * n, 3 * m, 3 * m);
    MatX c(3 * m, 8 * n + b);
    for (Index r = 0; r < 3 * m; ++r) {
        for (Index k = 0; k < 8 * n; ++k) c(r, k) = fisher(8 * n + r, k);
        for (Index l = 0; l < b; ++l) c(r, 8 * n + l) = sys.border(8 * n + r, l);
    }
    const MatX ct_ainv_c = mul(c, solve(a, c), true);
    for (Index col = 0; col < d.cols(); ++col)
        for (Index r = 0; r < d.rows(); ++r) d(r, col) -= ct_ainv_c(r, col);
    return d;
}

template <class F>
static void expect_error(F&& f, ErrorKind kind, const std::string& stage, const std::string& fragment, int line) {
    try {
        f();
        std::printf("FAIL line %d: no error\n", line);
        ++g_fail;
    } catch (const Error& e) {
        if (e.kind() != kind || (!stage.empty() && e.stage() != stage) ||
            std::string(e.what()).find(fragment) == std::string::npos) {
            std::printf("FAIL line %d: got kind %d stage '%s' what '%s'\n", line, (int)e.kind(), e.stage().c_str(), e.what());
            ++g_fail;
        }
    }
}

// ---- test_fisher.cpp:42-100 ----------------------------------------------------------
static void test_fisher() {
    for (const Reconstruction& rec : {cube_scene(1, 0.0), cube_scene(1, 0.5), random_scene(7, 50, 0.5, 4, 0.7)}) {
        const SparseJacobian jac = assemble_jacobian(rec);
        const MatX h = gauge_nullspace(jac, rec);
        const BorderedSystem sys = build_fisher_blocks(jac, rec, h, 1);
        CHECK(sys.border == h);
        CHECK(!sys.conditioned);
        // J^T W J from the dense Jacobian
        const MatX j = jac.dense();
        MatX wj(j.rows(), j.cols());
        for (Index t = 0; t < rec.num_observations(); ++t) {
            const Mat2& s = rec.observations[t].sigma;
            const double det = s[0] * s[3] - s[1] * s[2];
            const double w[4] = {s[3] / det, -s[1] / det, -s[2] / det, s[0] / det};
            for (Index c = 0; c < j.cols(); ++c) {
                wj(2 * t, c) = w[0] * j(2 * t, c) + w[1] * j(2 * t + 1, c);
                wj(2 * t + 1, c) = w[2] * j(2 * t, c) + w[3] * j(2 * t + 1, c);
            }
        }
        CHECK(rel_diff(dense_from_blocks(sys), mul(j, wj, true)) < 1e-13);
    }
    {  // sigma x 4 scales every block by 1/4 exactly
        const Reconstruction rec = cube_scene(2, 0.5);
        Reconstruction loose = rec;
        for (Observation& o : loose.observations)
            for (double& v : o.sigma) v *= 4.0;
        const SparseJacobian jac = assemble_jacobian(rec);
        const MatX h = gauge_nullspace(jac, rec);
        const BorderedSystem a = build_fisher_blocks(jac, rec, h, 1), b = build_fisher_blocks(jac, loose, h, 1);
        for (Index i = 0; i < rec.num_cameras(); ++i)
            for (int e = 0; e < 64; ++e) CHECK(b.cam_blocks[i][e] == 0.25 * a.cam_blocks[i][e]);
        for (Index k = 0; k < rec.num_points(); ++k)
            for (int e = 0; e < 9; ++e) CHECK(b.point_blocks[k][e] == 0.25 * a.point_blocks[k][e]);
        for (size_t t = 0; t < a.couplings.size(); ++t)
            for (int e = 0; e < 24; ++e) CHECK(b.couplings[t].block[e] == 0.25 * a.couplings[t].block[e]);
    }
    {  // non-SPD observation covariance, by index
        Reconstruction rec = cube_scene(3, 0.5);
        const SparseJacobian jac = assemble_jacobian(rec);
        const MatX h = gauge_nullspace(jac, rec);
        rec.observations[7].sigma = {1.0, 2.0, 2.0, 1.0};
        expect_error([&] { build_fisher_blocks(jac, rec, h, 1); }, ErrorKind::degenerate, "fisher", "observation 7",
                     __LINE__);
        rec.observations[7].sigma = {0.0, 0.0, 0.0, 0.0};
        expect_error([&] { build_fisher_blocks(jac, rec, h, 1); }, ErrorKind::degenerate, "fisher", "", __LINE__);
    }
    {  // border with the wrong row count
        const Reconstruction rec = cube_scene(1, 0.0);
        const SparseJacobian jac = assemble_jacobian(rec);
        expect_error([&] { build_fisher_blocks(jac, rec, MatX::Zero(jac.cols() + 1, 7), 1); }, ErrorKind::dimension,
                     "fisher", "", __LINE__);
    }
}

// ---- test_nullspace.cpp:53-69 ----------------------------------------------------------
static void test_nullspace() {
    for (const Reconstruction& rec : {cube_scene(1, 0.0), cube_scene(2, 0.5), random_scene(12, 90, 0.4, 5, 0.5)}) {
        const SparseJacobian jac = assemble_jacobian(rec);
        const MatX h = gauge_nullspace(jac, rec);
        CHECK(nullspace_residual(jac, h) < 1e-10);
    }
    const Reconstruction rec = cube_scene(1, 0.5);
    const SparseJacobian jac = assemble_jacobian(rec);
    MatX h = gauge_nullspace(jac, rec);
    h(0, 0) += 1.0;  // test_nullspace.cpp:63-69
    CHECK(nullspace_residual(jac, h) > 1e-4);
    expect_error([&] { nullspace_residual(jac, MatX::Zero(jac.cols() + 1, 7)); }, ErrorKind::dimension, "nullspace", "",
                 __LINE__);
}

// ---- test_schur.cpp:57-165 ----------------------------------------------------------
static void test_schur() {
    for (const bool with_border : {true, false}) {
        const BorderedSystem sys = bordered_cube(1, 0.5, with_border, false);
        const MatX z = schur_reduce(sys);
        CHECK(z.rows() == 8 * sys.n_cams + sys.border_cols());
        CHECK(rel_diff(z, dense_schur_reference(sys)) < 1e-10);
    }
    {
        const BorderedSystem sys = bordered_cube(2, 0.5, true, true);
        CHECK(asym(schur_reduce(sys)) == 0.0);
    }
    {
        const Reconstruction rec = disconnected_scene(3, 0.5);
        const SparseJacobian jac = assemble_jacobian(rec);
        const BorderedSystem sys = build_fisher_blocks(jac, rec, MatX::Zero(jac.cols(), 0), 1);
        const MatX z = schur_reduce(sys);
        double mx = 0.0;
        for (Index i = 0; i < 6 * 8; ++i)
            for (Index j = 6 * 8; j < 12 * 8; ++j) mx = std::max(mx, std::fabs(z(i, j)));
        CHECK(mx == 0.0);
    }
    {
        BorderedSystem sys = bordered_cube(4, 0.5, true, false);
        sys.point_blocks[5].fill(0.0);
        expect_error([&] { schur_reduce(sys, nullptr, 1); }, ErrorKind::degenerate, "schur", "point 5", __LINE__);
    }
    {
        const BorderedSystem sys = bordered_cube(5, 0.5, true, true);
        CovarianceDiagnostics diag;
        std::vector<Mat3> a_inv;
        const MatX z = schur_reduce(sys, &diag, 1, &a_inv);
        CHECK(diag.largest_dense_dim == z.rows());
        CHECK(diag.peak_dense_bytes == sizeof(double) * (size_t)z.rows() * (size_t)z.rows());
        CHECK(a_inv.size() == (size_t)sys.n_pts);
        for (Index j = 0; j < sys.n_pts; ++j)
            CHECK(max_abs_diff_identity(mul(block_of(sys.point_blocks[j], 3, 3), block_of(a_inv[j], 3, 3))) < 1e-10);
    }
    {
        const BorderedSystem sys = bordered_cube(6, 0.5, true, true);
        CHECK(schur_reduce(sys, nullptr, 1) == schur_reduce(sys, nullptr, 4));
    }
    {
        const BorderedSystem sys = bordered_cube(7, 0.5, true, true);
        CovarianceDiagnostics diag;
        const MatX z = schur_reduce(sys, &diag, 1);
        const MatX z_inv = invert_schur(z, diag);
        CHECK(max_abs_diff_identity(mul(z, z_inv)) < 1e-8);
        CHECK(asym(z_inv) == 0.0);
        CHECK(diag.inertia_positive == 8 * sys.n_cams);
        CHECK(diag.inertia_negative == 7);
        CHECK(diag.min_pivot > 0.0);
        CHECK(diag.max_pivot >= diag.min_pivot);
        CHECK(diag.peak_dense_bytes == 2 * sizeof(double) * (size_t)z.rows() * (size_t)z.rows());
    }
    {  // small hand-checked factorizations
        CovarianceDiagnostics diag;
        MatX d = MatX::Zero(2, 2);
        d(0, 0) = 2.0;
        d(1, 1) = 3.0;
        const MatX d_inv = invert_schur(d, diag);
        CHECK(std::fabs(d_inv(0, 0) - 0.5) <= 1e-14 * 0.5);
        CHECK(std::fabs(d_inv(1, 1) - 1.0 / 3.0) <= 1e-14 / 3.0);
        CHECK(diag.inertia_positive == 2 && diag.inertia_negative == 0);
        CHECK(std::fabs(diag.min_pivot - 2.0) < 1e-12 && std::fabs(diag.max_pivot - 3.0) < 1e-12);
        MatX swap = MatX::Zero(2, 2);
        swap(0, 1) = swap(1, 0) = 1.0;  // eigenvalues +-1
        const MatX swap_inv = invert_schur(swap, diag);
        double mx = 0.0;
        for (Index c = 0; c < 2; ++c)
            for (Index r = 0; r < 2; ++r) mx = std::max(mx, std::fabs(swap_inv(r, c) - swap(r, c)));
        CHECK(mx < 1e-14);
        CHECK(diag.inertia_positive == 1 && diag.inertia_negative == 1);
    }
    {  // shape errors and singular systems
        CovarianceDiagnostics diag;
        expect_error([&] { invert_schur(MatX::Zero(2, 3), diag); }, ErrorKind::dimension, "factorization", "", __LINE__);
        const BorderedSystem free_gauge = bordered_cube(8, 0.5, false, true);
        expect_error([&] { invert_schur(schur_reduce(free_gauge), diag); }, ErrorKind::degenerate, "factorization",
                     "degenerate", __LINE__);
    }
}

// ---- test_covariance.cpp:42-78, 120-135 + the stage pipeline ------------------------
static void test_full_covariance() {
    {
        const Reconstruction rec = cube_scene(2, 0.5);
        CovarianceOptions opts;
        opts.threads = 1;
        opts.point_covariances = true;
        opts.camera_cross_covariances = true;
        const CovarianceResult result = compute_covariance(rec, opts);
        const MatX sigma = full_covariance(rec);
        const Index n = rec.num_cameras();
        CHECK(sigma.rows() == rec.num_parameters());
        for (Index i = 0; i < n; ++i) CHECK(rel_diff(block_of(result.camera_cov[i], 8, 8), sub(sigma, 8 * i, 8 * i, 8, 8)) < 1e-8);
        CHECK(result.point_cov.size() == (size_t)rec.num_points());
        for (Index j = 0; j < rec.num_points(); ++j)
            CHECK(rel_diff(block_of(result.point_cov[j], 3, 3), sub(sigma, 8 * n + 3 * j, 8 * n + 3 * j, 3, 3)) < 1e-8);
        for (Index i = 0; i < n; ++i) {
            CHECK(result.cross_block(i, i) == result.camera_cov[i]);
            for (Index l = 0; l < n; ++l)
                CHECK(rel_diff(block_of(result.cross_block(i, l), 8, 8), sub(sigma, 8 * i, 8 * l, 8, 8)) < 1e-8);
        }
    }
    {  // the covariance annihilates the gauge directions
        const Reconstruction rec = cube_scene(3, 0.5);
        const MatX sigma = full_covariance(rec);
        const SparseJacobian jac = assemble_jacobian(rec);
        const MatX h = gauge_nullspace(jac, rec);
        const MatX hs = mul(h, sigma, true);
        double a = 0, b = 0, c = 0;
        for (Index k = 0; k < hs.cols() * hs.rows(); ++k) a = std::max(a, std::fabs(hs.data()[k]));
        for (Index k = 0; k < h.cols() * h.rows(); ++k) b = std::max(b, std::fabs(h.data()[k]));
        for (Index k = 0; k < sigma.cols() * sigma.rows(); ++k) c = std::max(c, std::fabs(sigma.data()[k]));
        CHECK(a / (b * c) < 1e-6);
    }
    {
        const Reconstruction rec = cube_scene(1, 0.0);
        expect_error([&] { full_covariance(rec, 50); }, ErrorKind::size_guard, "full-covariance", "guard is 50", __LINE__);
        // an empty scene passes validate() and fails in the factorization, as in the reference
        expect_error([&] { compute_covariance(Reconstruction{}); }, ErrorKind::degenerate, "factorization", "", __LINE__);
        expect_error([&] { full_covariance(Reconstruction{}); }, ErrorKind::degenerate, "factorization", "", __LINE__);
    }
    {  // the stage functions composed like compute_covariance (covariance.cpp:323-350)
        const Reconstruction rec = random_scene(12, 150, 0.3, 5, 0.5);
        rec.validate();
        const SparseJacobian jac = assemble_jacobian(rec);
        BorderedSystem sys = build_fisher_blocks(jac, rec, gauge_nullspace(jac, rec), 1);
        const ConditioningScales sc = condition_columns(sys);
        apply_conditioning(sys, sc);
        CovarianceDiagnostics diag;
        const MatX z_inv = invert_schur(schur_reduce(sys, &diag, 1), diag);
        const CovarianceResult staged = extract_camera_covariances(z_inv, sc, rec.num_cameras(), diag);
        const CovarianceResult fused = compute_covariance(rec);
        for (Index i = 0; i < rec.num_cameras(); ++i)
            CHECK(rel_diff(block_of(staged.camera_cov[i], 8, 8), block_of(fused.camera_cov[i], 8, 8)) < 1e-9);
        CHECK(staged.diagnostics.negative_eigenvalue_warnings == 0);
        CHECK(staged.diagnostics.inertia_positive == 8 * rec.num_cameras());
        CHECK(staged.diagnostics.inertia_negative == 7);
        CHECK(staged.diagnostics.scale_min == fused.diagnostics.scale_min);
        CHECK(staged.diagnostics.scale_max == fused.diagnostics.scale_max);
        const ObservationIndex ix = build_observation_index(rec);
        CHECK((Index)ix.by_camera.size() == rec.num_cameras());
        for (Index j = 0; j < rec.num_points(); ++j) CHECK(ix.by_point[j] == sys.obs_by_point[j]);
    }
}

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
    // errors keep the reference's kind / stage / message
    Reconstruction bad = rec;
    bad.cameras[1].c = -1.0;
    expect_error([&] { compute_covariance(bad); }, ErrorKind::invariant, "validate",
                 "validate: camera 1 has non-positive focal length", __LINE__);
    CHECK(static_cast<int>(ErrorKind::io) == 0 && static_cast<int>(ErrorKind::size_guard) == 5);
    {  // covariance IO round trip (covariance_io.hpp)
        save_covariance_json(result, "/tmp/sfmcov_dropin_cov.json");
        const CovarianceResult back = load_covariance_json("/tmp/sfmcov_dropin_cov.json");
        // the file holds the upper triangles (blocks are symmetric to the last bit, not bitwise)
        CHECK(back.camera_cov.size() == result.camera_cov.size());
        for (size_t i = 0; i < back.camera_cov.size(); ++i)
            CHECK(pack_upper_triangle(back.camera_cov[i]) == pack_upper_triangle(result.camera_cov[i]));
        CHECK(back.diagnostics.inertia_negative == 7 && back.diagnostics.min_pivot == d.min_pivot);
        const auto tri = pack_upper_triangle(result.camera_cov[0]);
        CHECK(pack_upper_triangle(unpack_upper_triangle(tri)) == tri);
        save_covariance_csv(result, "/tmp/sfmcov_dropin_cov.csv");
        std::remove("/tmp/sfmcov_dropin_cov.json");
        std::remove("/tmp/sfmcov_dropin_cov.csv");
    }
    test_fisher();
    test_nullspace();
    test_schur();
    test_full_covariance();
    if (g_fail) {
        std::printf("%d checks failed\n", g_fail);
        return 1;
    }
    // print the first block so the Python test can compare against the oracle
    for (int q = 0; q < 64; ++q) std::printf("%.17g%c", result.camera_cov[0][q], q == 63 ? '\n' : ' ');
    std::printf("PASS\n");
    return 0;
}
