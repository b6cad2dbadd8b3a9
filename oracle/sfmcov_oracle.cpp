// =============================================================================
// TEST INFRASTRUCTURE — NOT PRODUCT CODE.
//
// CPU restatement ("oracle") of the reference NBUP covariance path of
// arXiv 1808.02414 (`sfmcov`, /root/reference/proj).  Only tests/,
// __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference leg
// may load this library, and only as the checker or the CPU baseline.  The
// product path (paper_1808_02414_b200/) never links or calls it.
//
// The reference itself cannot be built here (Eigen3, lapacke.h and the
// vendored CLI11/doctest are absent), so this file restates
// its algorithm statement by statement, Eigen-free, templated on the camera
// width P ∈ {8, 9}:
//   P = 8  — the reference camera (r, C, c, k), include/sfmcov/types.hpp:28-39
//   P = 9  — the BASELINE camera (r, C, f, k1, k2), u = f(1+k1ρ+k2ρ²)u_n
//            (not in the reference).
// The dense inversion calls the same LAPACK routines as the reference
// (dsytrf('L') + dsytrs2 against I, src/covariance.cpp:203,245) from the
// OpenBLAS 0.3.15 LP64 build bundled with the image; dgesdd for the dense
// Moore–Penrose oracle (src/oracle.cpp:47).
//
// Parity pinning: the reference ships no golden vectors; the
// restatement is pinned by the reference's own known-answer tests and
// property tests, ported in tests/test_oracle_*.py.
//
// Elementary functions.  Eigen/glibc are not bit-reproducible on the GPU, so
// the restatement fixes its own op order for every formula and uses a
// deterministic sin/cos (fdlibm-style kernels, restated below) built only
// from IEEE +,-,*,/ with FP contraction disabled (-ffp-contract=off).  The
// CUDA kernels implement the same op sequences with --fmad=false, so the
// Jacobian, the nullspace and the observation index are bit-exact between
// the two, as BASELINE.json's north_star requires.
// =============================================================================

#include <algorithm>
#include <atomic>
#include <chrono>
#include <cmath>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <exception>
#include <limits>
#include <string>
#include <thread>
#include <vector>

// ---- LAPACKE / OpenBLAS prototypes (lapacke.h is absent; LP64 ints) --------
extern "C" {
int LAPACKE_dsytrf(int layout, char uplo, int n, double* a, int lda, int* ipiv);
int LAPACKE_dsytrs2(int layout, char uplo, int n, int nrhs, const double* a, int lda,
                    const int* ipiv, double* b, int ldb);
int LAPACKE_dgesdd(int layout, char jobz, int m, int n, double* a, int lda, double* s,
                   double* u, int ldu, double* vt, int ldvt);
int LAPACKE_dpotrf(int layout, char uplo, int n, double* a, int lda);
int LAPACKE_dtrtri(int layout, char uplo, char diag, int n, double* a, int lda);
void openblas_set_num_threads(int);
char* openblas_get_corename(void);
int openblas_get_num_threads(void);
}
static constexpr int kColMajor = 102;

namespace oracle {

// ---- error convention: include/sfmcov/error.hpp:9-33 ------------------------
enum Kind { kOk = 0, kIo = 1, kParse = 2, kInvariant = 3, kDegenerate = 4, kDimension = 5,
            kSizeGuard = 6 };

struct Error {
    int kind;
    std::string stage;
    std::string message;
};

// ---- constants (reference headers) ------------------------------------------
constexpr double kDepthEps = 1e-9;            // projection.hpp:12
constexpr double kRotationTaylorEps = 1e-8;   // rotation.hpp:7
constexpr double kRotationCondTol = 1e-12;    // nullspace.hpp:13
constexpr double kPivotRtol = 1e-12;          // covariance.hpp:14
constexpr double kPsdTol = 1e-9;              // covariance.hpp:18
constexpr int kGauge = 7;                     // types.hpp:25

// ---- deterministic sin/cos --------------------------------------------------
// fdlibm/musl kernel polynomials on [-pi/4, pi/4] with a two-constant
// Cody–Waite reduction.  Same op order as csrc/detmath.cuh.
namespace dm {
constexpr double S1 = -1.66666666666666324348e-01, S2 = 8.33333333332248946124e-03,
                 S3 = -1.98412698298579493134e-04, S4 = 2.75573137070700676789e-06,
                 S5 = -2.50507602534068634195e-08, S6 = 1.58969099521155010221e-10;
constexpr double C1 = 4.16666666666666019037e-02, C2 = -1.38888888888741095749e-03,
                 C3 = 2.48015872894767294178e-05, C4 = -2.75573143513906633035e-07,
                 C5 = 2.08757232129817482790e-09, C6 = -1.13596475577881948265e-11;
constexpr double kInvPio2 = 6.36619772367581382433e-01;
constexpr double kPio2Hi = 1.57079632673412561417e+00;   // first 33 bits of pi/2
constexpr double kPio2Lo = 6.07710050650619224932e-11;   // pi/2 - kPio2Hi

inline double ksin(double x) {
    const double z = x * x;
    const double w = z * z;
    const double r = (S2 + z * (S3 + z * S4)) + (z * w) * (S5 + z * S6);
    const double v = z * x;
    return x + v * (S1 + z * r);
}
inline double kcos(double x) {
    const double z = x * x;
    const double w = z * z;
    const double r = z * (C1 + z * (C2 + z * C3)) + (w * w) * (C4 + z * (C5 + z * C6));
    const double hz = 0.5 * z;
    const double one_minus = 1.0 - hz;
    return one_minus + (((1.0 - one_minus) - hz) + z * r);
}
// sin and cos of x >= 0 (rotation angles are norms).
inline void sincos_pos(double x, double* s, double* c) {
    double n = 0.0;
    double y = x;
    if (x > 7.85398163397448278999e-01) {
        n = (double)(long long)(x * kInvPio2 + 0.5);
        y = (x - n * kPio2Hi) - n * kPio2Lo;
    }
    const double sy = ksin(y), cy = kcos(y);
    const long long q = ((long long)n) & 3;
    if (q == 0) { *s = sy; *c = cy; }
    else if (q == 1) { *s = cy; *c = -sy; }
    else if (q == 2) { *s = -sy; *c = -cy; }
    else { *s = -cy; *c = sy; }
}
}  // namespace dm

// ---- small fixed-size algebra (row-major) -----------------------------------
struct M3 { double a[9]; double& operator()(int i, int j) { return a[3 * i + j]; }
            double operator()(int i, int j) const { return a[3 * i + j]; } };

inline M3 zero3() { M3 m; for (double& v : m.a) v = 0.0; return m; }
inline M3 eye3() { M3 m = zero3(); m(0, 0) = m(1, 1) = m(2, 2) = 1.0; return m; }
inline M3 mul3(const M3& A, const M3& B) {
    M3 C;
    for (int i = 0; i < 3; ++i)
        for (int j = 0; j < 3; ++j)
            C(i, j) = (A(i, 0) * B(0, j) + A(i, 1) * B(1, j)) + A(i, 2) * B(2, j);
    return C;
}

// rotation.cpp:7-13
inline M3 skew(const double v[3]) {
    M3 s;
    s(0, 0) = 0.0;   s(0, 1) = -v[2]; s(0, 2) = v[1];
    s(1, 0) = v[2];  s(1, 1) = 0.0;   s(1, 2) = -v[0];
    s(2, 0) = -v[1]; s(2, 1) = v[0];  s(2, 2) = 0.0;
    return s;
}

// rotation.cpp:15-28 (Rodrigues, Taylor branch below kRotationTaylorEps)
inline M3 rotation_matrix(const double r[3]) {
    const double theta2 = (r[0] * r[0] + r[1] * r[1]) + r[2] * r[2];
    const M3 rx = skew(r);
    double a, b;
    if (theta2 < kRotationTaylorEps * kRotationTaylorEps) {
        a = 1.0 - theta2 / 6.0;
        b = 0.5 - theta2 / 24.0;
    } else {
        const double theta = std::sqrt(theta2);
        double s, c;
        dm::sincos_pos(theta, &s, &c);
        a = s / theta;
        b = (1.0 - c) / theta2;
    }
    const M3 rx2 = mul3(rx, rx);
    M3 R;
    for (int i = 0; i < 3; ++i)
        for (int j = 0; j < 3; ++j)
            R(i, j) = ((i == j ? 1.0 : 0.0) + a * rx(i, j)) + b * rx2(i, j);
    return R;
}

// rotation.cpp:70-77: d(R(r) w)/dr
inline M3 rotate_point_derivative(const double r[3], const double w[3]) {
    const double theta2 = (r[0] * r[0] + r[1] * r[1]) + r[2] * r[2];
    const M3 sw = skew(w);
    if (theta2 < kRotationTaylorEps * kRotationTaylorEps) {
        const double rxw[3] = {r[1] * w[2] - r[2] * w[1], r[2] * w[0] - r[0] * w[2],
                               r[0] * w[1] - r[1] * w[0]};
        const M3 s1 = skew(rxw);
        const M3 s2 = mul3(skew(r), sw);
        M3 out;
        for (int k = 0; k < 9; ++k) out.a[k] = -sw.a[k] - 0.5 * (s1.a[k] + s2.a[k]);
        return out;
    }
    const M3 R = rotation_matrix(r);
    M3 negR;
    for (int k = 0; k < 9; ++k) negR.a[k] = -R.a[k];
    const M3 t1 = mul3(negR, sw);
    const M3 sr = skew(r);
    M3 rtmi;  // R^T - I
    for (int i = 0; i < 3; ++i)
        for (int j = 0; j < 3; ++j) rtmi(i, j) = R(j, i) - (i == j ? 1.0 : 0.0);
    const M3 p = mul3(rtmi, sr);
    M3 m2;
    for (int i = 0; i < 3; ++i)
        for (int j = 0; j < 3; ++j) m2(i, j) = r[i] * r[j] + p(i, j);
    const M3 num = mul3(t1, m2);
    M3 out;
    for (int k = 0; k < 9; ++k) out.a[k] = num.a[k] / theta2;
    return out;
}

// Cyclic Jacobi for a symmetric n×n matrix (row-major, in place) with a fixed
// sweep cap; eigenvalues in d (unsorted), eigenvectors in the columns of v.
// Stands in for Eigen::SelfAdjointEigenSolver (covariance.cpp:147-153,266;
// nullspace.cpp:52-60).  Same op order as csrc/detmath.cuh.
template <int N>
inline void jacobi_eig(double* a, double* d, double* v) {
    for (int i = 0; i < N; ++i)
        for (int j = 0; j < N; ++j) v[N * i + j] = (i == j) ? 1.0 : 0.0;
    // Cyclic sweeps; an off-diagonal entry below 1e-17 sqrt|a_pp a_qq| is
    // treated as converged (set to 0, no rotation); stop after a sweep that
    // rotated nothing.
    for (int sweep = 0; sweep < 32; ++sweep) {
        bool rotated = false;
        for (int p = 0; p < N; ++p)
            for (int q = p + 1; q < N; ++q) {
                const double apq = a[N * p + q];
                if (!(std::fabs(apq) > 1e-17 * std::sqrt(std::fabs(a[N * p + p] * a[N * q + q])))) {
                    a[N * p + q] = 0.0;
                    a[N * q + p] = 0.0;
                    continue;
                }
                rotated = true;
                const double theta = (a[N * q + q] - a[N * p + p]) / (2.0 * apq);
                const double at = std::fabs(theta);
                double t;
                if (at > 1e150) {
                    t = 0.5 / theta;
                } else {
                    t = 1.0 / (at + std::sqrt(theta * theta + 1.0));
                    if (theta < 0.0) t = -t;
                }
                const double c = 1.0 / std::sqrt(t * t + 1.0);
                const double s = t * c;
                for (int k = 0; k < N; ++k) {  // columns p, q
                    const double akp = a[N * k + p], akq = a[N * k + q];
                    a[N * k + p] = c * akp - s * akq;
                    a[N * k + q] = s * akp + c * akq;
                }
                for (int k = 0; k < N; ++k) {  // rows p, q
                    const double apk = a[N * p + k], aqk = a[N * q + k];
                    a[N * p + k] = c * apk - s * aqk;
                    a[N * q + k] = s * apk + c * aqk;
                }
                a[N * p + q] = 0.0;
                a[N * q + p] = 0.0;
                for (int k = 0; k < N; ++k) {
                    const double vkp = v[N * k + p], vkq = v[N * k + q];
                    v[N * k + p] = c * vkp - s * vkq;
                    v[N * k + q] = s * vkp + c * vkq;
                }
            }
        if (!rotated) break;
    }
    for (int i = 0; i < N; ++i) d[i] = a[N * i + i];
}

// Symmetric 3×3 inverse through the eigendecomposition, with the reference's
// rank test (lam_min > 0 and lam_min >= tol * lam_max).  Returns false if the
// test fails.
inline bool eig_inverse3(const M3& m, double tol, M3* inv) {
    double a[9], d[3], v[9];
    for (int k = 0; k < 9; ++k) a[k] = m.a[k];
    jacobi_eig<3>(a, d, v);
    const double lmin = std::min(std::min(d[0], d[1]), d[2]);
    const double lmax = std::max(std::max(d[0], d[1]), d[2]);
    if (!(lmin > 0.0) || lmin < tol * lmax) return false;
    const double il[3] = {1.0 / d[0], 1.0 / d[1], 1.0 / d[2]};
    for (int i = 0; i < 3; ++i)
        for (int j = 0; j < 3; ++j)
            (*inv)(i, j) = (v[3 * i + 0] * il[0] * v[3 * j + 0] + v[3 * i + 1] * il[1] * v[3 * j + 1]) +
                           v[3 * i + 2] * il[2] * v[3 * j + 2];
    return true;
}

// ---- scene (layout-compatible with include/sfmcov_b200.h sfmcov_scene) -------
extern "C" struct oracle_scene {
    int32_t n_cams, n_pts, n_obs, cam_params;
    const double* cams;       // n × P: r(3), C(3), c|f, k|k1[, k2]
    const double* pts;        // m × 3
    const int32_t* obs_cam;   // t
    const int32_t* obs_pt;    // t
    const double* obs_u;      // t × 2 (may be null)
    const double* obs_sigma;  // t × 4 row-major 2×2 (null = identity)
};

inline double sig(const oracle_scene& s, int64_t t, int k) {
    if (!s.obs_sigma) return (k == 0 || k == 3) ? 1.0 : 0.0;
    return s.obs_sigma[4 * t + k];
}

// ---- threading: src/threading.cpp:24-52 --------------------------------------
template <typename F>
void parallel_for(int64_t count, int threads, F&& fn) {
    if (count <= 0) return;
    const int workers = std::max<int>(1, (int)std::min<int64_t>(threads, count));
    if (workers == 1) { fn(0, count); return; }
    const int64_t chunk = (count + workers - 1) / workers;
    std::vector<std::exception_ptr> errors(workers);
    std::vector<std::thread> pool;
    for (int w = 0; w < workers; ++w) {
        const int64_t b = w * chunk, e = std::min<int64_t>(b + chunk, count);
        if (b >= e) break;
        pool.emplace_back([&, w, b, e] {
            try { fn(b, e); } catch (...) { errors[w] = std::current_exception(); }
        });
    }
    for (auto& t : pool) t.join();
    for (auto& e : errors) if (e) std::rethrow_exception(e);
}

// ---- validation: src/scene.cpp:19-78 -----------------------------------------
inline bool finite3(const double* v) {
    return std::isfinite(v[0]) && std::isfinite(v[1]) && std::isfinite(v[2]);
}

inline void validate(const oracle_scene& s) {
    const int P = s.cam_params;
    const int64_t n = s.n_cams, m = s.n_pts, T = s.n_obs;
    if (P != 8 && P != 9) throw Error{kDimension, "validate", "camera width must be 8 or 9"};
    for (int64_t i = 0; i < n; ++i) {
        const double* c = s.cams + P * i;
        bool fin = finite3(c) && finite3(c + 3);
        for (int p = 6; p < P; ++p) fin = fin && std::isfinite(c[p]);
        if (!fin) throw Error{kInvariant, "validate", "camera " + std::to_string(i) + " has non-finite parameters"};
        if (!(c[6] > 0.0)) throw Error{kInvariant, "validate", "camera " + std::to_string(i) + " has non-positive focal length"};
    }
    for (int64_t j = 0; j < m; ++j)
        if (!finite3(s.pts + 3 * j))
            throw Error{kInvariant, "validate", "point " + std::to_string(j) + " has non-finite coordinates"};
    std::vector<int64_t> keys;
    keys.reserve(T);
    std::vector<int> cc(n, 0), pc(m, 0);
    for (int64_t t = 0; t < T; ++t) {
        const int32_t ci = s.obs_cam[t], pj = s.obs_pt[t];
        if (ci < 0 || ci >= n) throw Error{kInvariant, "validate", "observation " + std::to_string(t) + " camera index out of range"};
        if (pj < 0 || pj >= m) throw Error{kInvariant, "validate", "observation " + std::to_string(t) + " point index out of range"};
        const double s00 = sig(s, t, 0), s01 = sig(s, t, 1), s10 = sig(s, t, 2), s11 = sig(s, t, 3);
        const bool ufin = !s.obs_u || (std::isfinite(s.obs_u[2 * t]) && std::isfinite(s.obs_u[2 * t + 1]));
        if (!ufin || !std::isfinite(s00) || !std::isfinite(s01) || !std::isfinite(s10) || !std::isfinite(s11))
            throw Error{kInvariant, "validate", "observation " + std::to_string(t) + " has non-finite values"};
        const double scale = std::max({std::fabs(s00), std::fabs(s11), std::fabs(s01), 1e-300});
        if (std::fabs(s01 - s10) > 1e-12 * scale)
            throw Error{kInvariant, "validate", "observation " + std::to_string(t) + " covariance not symmetric"};
        const double det = s00 * s11 - s01 * s10;
        if (!(s00 > 0.0) || !(det > 0.0))
            throw Error{kInvariant, "validate", "observation " + std::to_string(t) + " covariance not positive definite"};
        keys.push_back((int64_t(ci) << 32) | int64_t(pj));
        ++cc[ci];
        ++pc[pj];
    }
    std::sort(keys.begin(), keys.end());
    if (std::adjacent_find(keys.begin(), keys.end()) != keys.end())
        throw Error{kInvariant, "validate", "duplicate (camera, point) observation pair"};
    for (int64_t i = 0; i < n; ++i)
        if (cc[i] < 4)
            throw Error{kInvariant, "validate", "camera " + std::to_string(i) + " observes " + std::to_string(cc[i]) + " points, need at least 4"};
    for (int64_t j = 0; j < m; ++j)
        if (pc[j] < 2)
            throw Error{kInvariant, "validate", "point " + std::to_string(j) + " is observed by " + std::to_string(pc[j]) + " cameras, need at least 2"};
}

// ---- observation index: src/scene.cpp:80-90 (CSR, ascending obs ids) ---------
struct Csr { std::vector<int64_t> off; std::vector<int32_t> idx; };

inline void build_index(const oracle_scene& s, Csr* by_cam, Csr* by_pt) {
    const int64_t n = s.n_cams, m = s.n_pts, T = s.n_obs;
    by_cam->off.assign(n + 1, 0);
    by_pt->off.assign(m + 1, 0);
    for (int64_t t = 0; t < T; ++t) { ++by_cam->off[s.obs_cam[t] + 1]; ++by_pt->off[s.obs_pt[t] + 1]; }
    for (int64_t i = 0; i < n; ++i) by_cam->off[i + 1] += by_cam->off[i];
    for (int64_t j = 0; j < m; ++j) by_pt->off[j + 1] += by_pt->off[j];
    by_cam->idx.resize(T);
    by_pt->idx.resize(T);
    std::vector<int64_t> fc(by_cam->off.begin(), by_cam->off.end() - 1), fp(by_pt->off.begin(), by_pt->off.end() - 1);
    for (int64_t t = 0; t < T; ++t) {
        by_cam->idx[fc[s.obs_cam[t]]++] = (int32_t)t;
        by_pt->idx[fp[s.obs_pt[t]]++] = (int32_t)t;
    }
}

// ---- Jacobian: src/projection.cpp:21-59, 80-105 -------------------------------
// cam block 2×P row-major: cols r(0..2), C(3..5), c|f (6), k|k1 (7)[, k2 (8)];
// point block 2×3 row-major.
template <int P>
inline bool observation_jacobian(const double* cam, const double* X, double* jc, double* jp, double* depth) {
    const double* r = cam;
    const double* C = cam + 3;
    const double c = cam[6];
    const double k1 = cam[7];
    const double k2 = (P == 9) ? cam[8] : 0.0;
    const M3 R = rotation_matrix(r);
    const double w[3] = {X[0] - C[0], X[1] - C[1], X[2] - C[2]};
    double v[3];
    for (int i = 0; i < 3; ++i) v[i] = (R(i, 0) * w[0] + R(i, 1) * w[1]) + R(i, 2) * w[2];
    *depth = v[2];
    if (!(v[2] > kDepthEps)) return false;
    const double un[2] = {v[0] / v[2], v[1] / v[2]};
    const double rho = un[0] * un[0] + un[1] * un[1];
    double d, dd;
    if (P == 8) { d = 1.0 + k1 * rho; dd = 2.0 * k1; }
    else { d = (1.0 + k1 * rho) + k2 * (rho * rho); dd = 2.0 * (k1 + 2.0 * k2 * rho); }
    double M[2][2];
    for (int i = 0; i < 2; ++i)
        for (int j = 0; j < 2; ++j) {
            const double e = (dd * un[i]) * un[j];
            M[i][j] = c * ((i == j) ? (d + e) : e);
        }
    const double iz = 1.0 / v[2];
    const double g02 = (-v[0] * iz) * iz, g12 = (-v[1] * iz) * iz;
    double A[2][3];
    for (int i = 0; i < 2; ++i) {
        A[i][0] = M[i][0] * iz;
        A[i][1] = M[i][1] * iz;
        A[i][2] = M[i][0] * g02 + M[i][1] * g12;
    }
    const M3 D = rotate_point_derivative(r, w);
    for (int i = 0; i < 2; ++i)
        for (int j = 0; j < 3; ++j) {
            const double dx = (A[i][0] * R(0, j) + A[i][1] * R(1, j)) + A[i][2] * R(2, j);
            const double drr = (A[i][0] * D(0, j) + A[i][1] * D(1, j)) + A[i][2] * D(2, j);
            jp[3 * i + j] = dx;
            jc[P * i + 3 + j] = -dx;
            jc[P * i + j] = drr;
        }
    const double crho = c * rho;
    for (int i = 0; i < 2; ++i) {
        jc[P * i + 6] = d * un[i];
        jc[P * i + 7] = crho * un[i];
        if (P == 9) jc[P * i + 8] = (c * (rho * rho)) * un[i];
    }
    return true;
}

template <int P>
struct Jac {
    std::vector<double> jc;  // t × 2P
    std::vector<double> jp;  // t × 6
};

template <int P>
inline Jac<P> assemble_jacobian(const oracle_scene& s, int threads) {
    Jac<P> J;
    J.jc.resize(size_t(s.n_obs) * 2 * P);
    J.jp.resize(size_t(s.n_obs) * 6);
    parallel_for(s.n_obs, threads, [&](int64_t b, int64_t e) {
        for (int64_t t = b; t < e; ++t) {
            double depth;
            if (!observation_jacobian<P>(s.cams + P * size_t(s.obs_cam[t]), s.pts + 3 * size_t(s.obs_pt[t]),
                                         &J.jc[2 * P * t], &J.jp[6 * t], &depth)) {
                char buf[64];
                std::snprintf(buf, sizeof buf, "%f", depth);
                throw Error{kDegenerate, "jacobian",
                            "observation " + std::to_string(t) + ": projection: point at camera-space depth " +
                                buf + " (behind camera or on the principal plane)"};
            }
        }
    });
    return J;
}

// ---- gauge nullspace: src/nullspace.cpp:14-83 ---------------------------------
// H is dense (P·n + 3m) × 7, row-major here.
template <int P>
inline std::vector<double> fixed_nullspace_blocks(const oracle_scene& s) {
    const int64_t n = s.n_cams, m = s.n_pts;
    std::vector<double> h(size_t(P * n + 3 * m) * kGauge, 0.0);
    auto put = [&](int64_t row, const double* X) {
        const M3 sx = skew(X);
        for (int a = 0; a < 3; ++a) {
            double* hr = &h[size_t(row + a) * kGauge];
            hr[a] = 1.0;
            for (int b = 0; b < 3; ++b) hr[3 + b] = sx(a, b);
            hr[6] = X[a];
        }
    };
    for (int64_t i = 0; i < n; ++i) put(P * i + 3, s.cams + P * i + 3);
    for (int64_t j = 0; j < m; ++j) put(P * n + 3 * j, s.pts + 3 * j);
    return h;
}

// Rotation blocks: per camera, normal = Σ d_rᵀd_r, rhs = Σ d_rᵀ(−(d_C[C]x + d_X[X]x))
// in ascending observation order, then H_r = eig-inverse(normal)·rhs.
template <int P>
inline void solve_rotation_blocks(const oracle_scene& s, const Jac<P>& J, std::vector<double>& h) {
    const int64_t n = s.n_cams;
    std::vector<M3> normal(n, zero3()), rhs(n, zero3());
    for (int64_t t = 0; t < s.n_obs; ++t) {
        const int ci = s.obs_cam[t];
        const double* jc = &J.jc[2 * P * t];
        const double* jp = &J.jp[6 * t];
        const M3 hc = skew(s.cams + P * size_t(ci) + 3);
        const M3 hx = skew(s.pts + 3 * size_t(s.obs_pt[t]));
        double tgt[2][3];
        for (int i = 0; i < 2; ++i)
            for (int j = 0; j < 3; ++j) {
                const double a = (jc[P * i + 3] * hc(0, j) + jc[P * i + 4] * hc(1, j)) + jc[P * i + 5] * hc(2, j);
                const double b = (jp[3 * i + 0] * hx(0, j) + jp[3 * i + 1] * hx(1, j)) + jp[3 * i + 2] * hx(2, j);
                tgt[i][j] = -(a + b);
            }
        for (int p = 0; p < 3; ++p)
            for (int q = 0; q < 3; ++q) {
                normal[ci](p, q) += jc[p] * jc[q] + jc[P + p] * jc[P + q];
                rhs[ci](p, q) += jc[p] * tgt[0][q] + jc[P + p] * tgt[1][q];
            }
    }
    for (int64_t i = 0; i < n; ++i) {
        M3 inv;
        if (!eig_inverse3(normal[i], kRotationCondTol, &inv))
            throw Error{kDegenerate, "nullspace", "camera " + std::to_string(i) + " has a rank-deficient rotation system"};
        const M3 hr = mul3(inv, rhs[i]);
        for (int a = 0; a < 3; ++a)
            for (int b = 0; b < 3; ++b) h[size_t(P * i + a) * kGauge + 3 + b] = hr(a, b);
    }
}

template <int P>
inline double nullspace_residual(const oracle_scene& s, const Jac<P>& J, const std::vector<double>& h) {
    const int64_t n = s.n_cams;
    double max_jh = 0.0, max_j = 0.0, max_h = 0.0;
    for (int64_t t = 0; t < s.n_obs; ++t) {
        const double* jc = &J.jc[2 * P * t];
        const double* jp = &J.jp[6 * t];
        const int64_t cr = P * int64_t(s.obs_cam[t]), pr = P * n + 3 * int64_t(s.obs_pt[t]);
        for (int i = 0; i < 2; ++i)
            for (int l = 0; l < kGauge; ++l) {
                double acc = 0.0;
                for (int p = 0; p < P; ++p) acc += jc[P * i + p] * h[size_t(cr + p) * kGauge + l];
                for (int p = 0; p < 3; ++p) acc += jp[3 * i + p] * h[size_t(pr + p) * kGauge + l];
                max_jh = std::max(max_jh, std::fabs(acc));
            }
        for (int k = 0; k < 2 * P; ++k) max_j = std::max(max_j, std::fabs(jc[k]));
        for (int k = 0; k < 6; ++k) max_j = std::max(max_j, std::fabs(jp[k]));
    }
    for (double v : h) max_h = std::max(max_h, std::fabs(v));
    const double denom = max_j * max_h;
    return denom > 0.0 ? max_jh / denom : 0.0;
}

// ---- Fisher blocks + conditioning: src/covariance.cpp:20-135 -------------------
template <int P>
struct System {
    int64_t n = 0, m = 0, T = 0;
    std::vector<double> D;   // n × P × P
    std::vector<double> A;   // m × 9
    std::vector<double> Cp;  // t × P × 3  (coupling J_cᵀWJ_p)
    std::vector<double> H;   // (Pn + 3m) × 7 row-major
    Csr by_cam, by_pt;
    std::vector<double> s_a, s_b;
    std::vector<int64_t> flagged;
};

template <int P>
inline System<P> build_fisher_blocks(const oracle_scene& s, const Jac<P>& J, std::vector<double> h, int threads) {
    System<P> sys;
    sys.n = s.n_cams; sys.m = s.n_pts; sys.T = s.n_obs;
    sys.H = std::move(h);
    std::vector<double> W(size_t(sys.T) * 4);
    parallel_for(sys.T, threads, [&](int64_t b, int64_t e) {
        for (int64_t t = b; t < e; ++t) {
            const double s00 = sig(s, t, 0), s01 = sig(s, t, 1), s10 = sig(s, t, 2), s11 = sig(s, t, 3);
            const double det = s00 * s11 - s01 * s10;
            if (!(s00 > 0.0) || !(det > 0.0))
                throw Error{kDegenerate, "fisher", "observation " + std::to_string(t) + " covariance is not positive definite"};
            W[4 * t + 0] = s11 / det;
            W[4 * t + 1] = -s01 / det;
            W[4 * t + 2] = -s10 / det;
            W[4 * t + 3] = s00 / det;
        }
    });
    build_index(s, &sys.by_cam, &sys.by_pt);
    sys.D.assign(size_t(sys.n) * P * P, 0.0);
    sys.A.assign(size_t(sys.m) * 9, 0.0);
    sys.Cp.resize(size_t(sys.T) * P * 3);
    // (Jᵀ W) J, evaluated left to right like the reference's Eigen expression.
    auto jtwj = [](const double* ja, int na, const double* w, const double* jb, int nb, double* out, bool add) {
        for (int p = 0; p < na; ++p) {
            const double t0 = ja[p] * w[0] + ja[na + p] * w[2];
            const double t1 = ja[p] * w[1] + ja[na + p] * w[3];
            for (int q = 0; q < nb; ++q) {
                const double v = t0 * jb[q] + t1 * jb[nb + q];
                if (add) out[nb * p + q] += v; else out[nb * p + q] = v;
            }
        }
    };
    parallel_for(sys.n, threads, [&](int64_t b, int64_t e) {
        for (int64_t i = b; i < e; ++i)
            for (int64_t k = sys.by_cam.off[i]; k < sys.by_cam.off[i + 1]; ++k) {
                const int64_t t = sys.by_cam.idx[k];
                jtwj(&J.jc[2 * P * t], P, &W[4 * t], &J.jc[2 * P * t], P, &sys.D[size_t(P) * P * i], true);
            }
    });
    parallel_for(sys.m, threads, [&](int64_t b, int64_t e) {
        for (int64_t j = b; j < e; ++j)
            for (int64_t k = sys.by_pt.off[j]; k < sys.by_pt.off[j + 1]; ++k) {
                const int64_t t = sys.by_pt.idx[k];
                jtwj(&J.jp[6 * t], 3, &W[4 * t], &J.jp[6 * t], 3, &sys.A[9 * j], true);
            }
    });
    parallel_for(sys.T, threads, [&](int64_t b, int64_t e) {
        for (int64_t t = b; t < e; ++t) jtwj(&J.jc[2 * P * t], P, &W[4 * t], &J.jp[6 * t], 3, &sys.Cp[size_t(P) * 3 * t], false);
    });
    return sys;
}

template <int P>
inline void condition_columns(System<P>& sys) {
    const int64_t n = sys.n, m = sys.m;
    sys.s_a.resize(P * n + 3 * m);
    sys.flagged.clear();
    for (int64_t i = 0; i < n; ++i)
        for (int p = 0; p < P; ++p) {
            const double d = sys.D[size_t(P) * P * i + P * p + p];
            if (d > 0.0) sys.s_a[P * i + p] = 1.0 / std::sqrt(d);
            else { sys.s_a[P * i + p] = 1.0; sys.flagged.push_back(P * i + p); }
        }
    for (int64_t j = 0; j < m; ++j)
        for (int p = 0; p < 3; ++p) {
            const double d = sys.A[9 * j + 4 * p];
            if (d > 0.0) sys.s_a[P * n + 3 * j + p] = 1.0 / std::sqrt(d);
            else { sys.s_a[P * n + 3 * j + p] = 1.0; sys.flagged.push_back(P * n + 3 * j + p); }
        }
    sys.s_b.resize(kGauge);
    const int64_t rows = P * n + 3 * m;
    for (int l = 0; l < kGauge; ++l) {
        double ss = 0.0;
        for (int64_t r = 0; r < rows; ++r) {
            const double v = sys.s_a[r] * sys.H[size_t(r) * kGauge + l];
            ss += v * v;
        }
        const double norm = std::sqrt(ss);
        sys.s_b[l] = norm > 0.0 ? 1.0 / norm : 1.0;
    }
}

template <int P>
inline void apply_conditioning(System<P>& sys, const oracle_scene& s) {
    const int64_t n = sys.n, m = sys.m;
    for (int64_t i = 0; i < n; ++i) {
        double* d = &sys.D[size_t(P) * P * i];
        const double* s = &sys.s_a[P * i];
        for (int p = 0; p < P; ++p)
            for (int q = 0; q < P; ++q) d[P * p + q] = (s[p] * d[P * p + q]) * s[q];
    }
    for (int64_t j = 0; j < m; ++j) {
        double* a = &sys.A[9 * j];
        const double* s = &sys.s_a[P * n + 3 * j];
        for (int p = 0; p < 3; ++p)
            for (int q = 0; q < 3; ++q) a[3 * p + q] = (s[p] * a[3 * p + q]) * s[q];
    }
    // couplings in observation order (covariance.cpp:128-132)
    for (int64_t t = 0; t < sys.T; ++t) {
        double* c = &sys.Cp[size_t(P) * 3 * t];
        const double* dc = &sys.s_a[P * int64_t(s.obs_cam[t])];
        const double* dp = &sys.s_a[P * n + 3 * int64_t(s.obs_pt[t])];
        for (int p = 0; p < P; ++p)
            for (int q = 0; q < 3; ++q) c[3 * p + q] = (dc[p] * c[3 * p + q]) * dp[q];
    }
    const int64_t rows = P * n + 3 * sys.m;
    for (int64_t r = 0; r < rows; ++r)
        for (int l = 0; l < kGauge; ++l) sys.H[size_t(r) * kGauge + l] = (sys.s_a[r] * sys.H[size_t(r) * kGauge + l]) * sys.s_b[l];
}

// ---- Schur reduction: src/covariance.cpp:137-194 ------------------------------
// Output: dense col-major (Pn+7)², full symmetric (upper accumulated, then
// mirrored like selfadjointView<Upper>).
template <int P>
inline std::vector<double> schur_reduce(const System<P>& sys, const oracle_scene& s, int threads, std::vector<M3>* a_inv_out) {
    const int64_t n = sys.n, m = sys.m;
    const int64_t dim = P * n + kGauge;
    std::vector<M3> a_inv(m);
    parallel_for(m, threads, [&](int64_t b, int64_t e) {
        for (int64_t j = b; j < e; ++j) {
            M3 a;
            for (int k = 0; k < 9; ++k) a.a[k] = sys.A[9 * j + k];
            if (!eig_inverse3(a, kPivotRtol, &a_inv[j]))
                throw Error{kDegenerate, "schur", "point " + std::to_string(j) + " has a singular 3x3 block"};
        }
    });
    std::vector<double> z(size_t(dim) * dim, 0.0);
    auto Z = [&](int64_t r, int64_t c) -> double& { return z[size_t(c) * dim + r]; };
    for (int64_t i = 0; i < n; ++i) {
        for (int p = 0; p < P; ++p)
            for (int q = 0; q < P; ++q) Z(P * i + p, P * i + q) = sys.D[size_t(P) * P * i + P * p + q];
        for (int p = 0; p < P; ++p)
            for (int l = 0; l < kGauge; ++l) Z(P * i + p, P * n + l) = sys.H[size_t(P * i + p) * kGauge + l];
    }
    std::vector<double> tb;  // per-obs P×3 blocks C·A⁻¹
    for (int64_t j = 0; j < m; ++j) {
        const int64_t o0 = sys.by_pt.off[j], o1 = sys.by_pt.off[j + 1];
        const int64_t k = o1 - o0;
        const double* br = &sys.H[size_t(P * n + 3 * j) * kGauge];  // 3×7
        tb.resize(size_t(k) * P * 3);
        for (int64_t a = 0; a < k; ++a) {
            const double* c = &sys.Cp[size_t(P) * 3 * sys.by_pt.idx[o0 + a]];
            double* t = &tb[size_t(P) * 3 * a];
            for (int p = 0; p < P; ++p)
                for (int q = 0; q < 3; ++q)
                    t[3 * p + q] = (c[3 * p] * a_inv[j](0, q) + c[3 * p + 1] * a_inv[j](1, q)) + c[3 * p + 2] * a_inv[j](2, q);
        }
        for (int64_t a = 0; a < k; ++a) {
            const int64_t ta = sys.by_pt.idx[o0 + a];
            const int64_t ca = s.obs_cam[ta];
            const double* t = &tb[size_t(P) * 3 * a];
            for (int64_t o = 0; o < k; ++o) {
                const int64_t to = sys.by_pt.idx[o0 + o];
                const int64_t cb = s.obs_cam[to];
                if (o != a && !(cb > ca)) continue;
                if (o == a && cb != ca) continue;
                const double* c = &sys.Cp[size_t(P) * 3 * to];
                for (int p = 0; p < P; ++p)
                    for (int q = 0; q < P; ++q)
                        Z(P * ca + p, P * cb + q) -= (t[3 * p] * c[3 * q] + t[3 * p + 1] * c[3 * q + 1]) + t[3 * p + 2] * c[3 * q + 2];
            }
            for (int p = 0; p < P; ++p)
                for (int l = 0; l < kGauge; ++l)
                    Z(P * ca + p, P * n + l) -= (t[3 * p] * br[l] + t[3 * p + 1] * br[kGauge + l]) + t[3 * p + 2] * br[2 * kGauge + l];
        }
        double ab[3][kGauge];  // A⁻¹ · border rows
        for (int q = 0; q < 3; ++q)
            for (int l = 0; l < kGauge; ++l)
                ab[q][l] = (a_inv[j](q, 0) * br[l] + a_inv[j](q, 1) * br[kGauge + l]) + a_inv[j](q, 2) * br[2 * kGauge + l];
        for (int l1 = 0; l1 < kGauge; ++l1)
            for (int l2 = 0; l2 < kGauge; ++l2)
                Z(P * n + l1, P * n + l2) -= (br[l1] * ab[0][l2] + br[kGauge + l1] * ab[1][l2]) + br[2 * kGauge + l1] * ab[2][l2];
    }
    for (int64_t c = 0; c < dim; ++c)
        for (int64_t r = c + 1; r < dim; ++r) Z(r, c) = Z(c, r);
    if (a_inv_out) *a_inv_out = std::move(a_inv);
    return z;
}

// ---- diagnostics (include/sfmcov/covariance.hpp:49-60) ------------------------
extern "C" struct oracle_diag {
    double scale_min, scale_max;
    double min_pivot, max_pivot;
    int32_t inertia_positive, inertia_negative;
    int32_t negative_eigenvalue_warnings;
    int32_t n_flagged;
    int64_t peak_dense_bytes;
    int64_t largest_dense_dim;
};

// ---- bordered inversion: src/covariance.cpp:196-257 ---------------------------
// BLAS threads for invert_schur: 1 = the reference's pin_blas_single_thread
// (threading.cpp:54-57); the CPU-baseline harness may raise it.
static int g_blas_threads = 1;
// Timing sample for the CPU baseline (bench.py only): instead of all n
// columns of the identity, dsytrs2 solves the first c1 = ceil(n / k) columns,
// then (from the identity again) the first c2 = 2 c1; its time is affine in
// the number of right-hand sides (a fixed cost for the pivots and the D
// blocks, then a per-column cost), so the two samples give the time of all n
// columns: t(n) = t2 + (t2 - t1) (n - c2) / (c2 - c1) (measured at config 3,
// one thread: 21.1 s predicted, 21.9 s for the full solve).  The blocks
// extracted after a sampled solve are not valid covariances.
static int g_trs_sample = 1;
static double g_trs_t[2] = {0, 0};
static int64_t g_trs_c[2] = {0, 0};

inline std::vector<double> invert_schur(std::vector<double> z, int64_t n, oracle_diag* diag, double* t_trf, double* t_trs) {
    openblas_set_num_threads(g_blas_threads);
    std::vector<int> ipiv(n);
    auto t0 = std::chrono::steady_clock::now();
    int info = LAPACKE_dsytrf(kColMajor, 'L', (int)n, z.data(), (int)n, ipiv.data());
    auto t1 = std::chrono::steady_clock::now();
    if (t_trf) *t_trf = std::chrono::duration<double>(t1 - t0).count();
    if (info < 0) throw Error{kDegenerate, "factorization", "factorization argument error " + std::to_string(info)};
    if (info > 0)
        throw Error{kDegenerate, "factorization", "exactly singular pivot at index " + std::to_string(info) +
                                                     "; the scene is likely disconnected or its gauge degenerate"};
    auto Z = [&](int64_t r, int64_t c) -> double& { return z[size_t(c) * n + r]; };
    double mn = std::numeric_limits<double>::infinity(), mx = 0.0;
    int pos = 0, neg = 0;
    for (int64_t i = 0; i < n;) {
        if (ipiv[i] > 0) {
            const double d = Z(i, i);
            mn = std::min(mn, std::fabs(d)); mx = std::max(mx, std::fabs(d));
            (d >= 0.0 ? pos : neg)++;
            ++i;
        } else {
            const double a = Z(i, i), c = Z(i + 1, i + 1), bb = Z(i + 1, i);
            const double mean = 0.5 * (a + c);
            const double disc = std::sqrt(0.25 * (a - c) * (a - c) + bb * bb);
            for (const double lam : {mean + disc, mean - disc}) {
                mn = std::min(mn, std::fabs(lam)); mx = std::max(mx, std::fabs(lam));
                (lam >= 0.0 ? pos : neg)++;
            }
            i += 2;
        }
    }
    diag->min_pivot = mn; diag->max_pivot = mx;
    diag->inertia_positive = pos; diag->inertia_negative = neg;
    if (!(mn > kPivotRtol * mx)) {
        char buf[64];
        std::snprintf(buf, sizeof buf, "%f", mn / mx);
        throw Error{kDegenerate, "factorization", std::string("near-singular pivot (ratio ") + buf +
                                                     "); the scene is likely disconnected or its gauge degenerate"};
    }
    std::vector<double> inv(size_t(n) * n, 0.0);
    for (int64_t i = 0; i < n; ++i) inv[size_t(i) * n + i] = 1.0;
    diag->peak_dense_bytes = std::max<int64_t>(diag->peak_dense_bytes, 2 * 8 * int64_t(n) * n);
    if (g_trs_sample > 1 && n >= 4 * g_trs_sample) {
        const int64_t c1 = (n + g_trs_sample - 1) / g_trs_sample, c2 = 2 * c1;
        for (int pass = 0; pass < 2; ++pass) {
            const int64_t c = pass ? c2 : c1;
            for (int64_t k = 0; k < c; ++k) {
                std::fill(inv.begin() + size_t(k) * n, inv.begin() + size_t(k + 1) * n, 0.0);
                inv[size_t(k) * n + k] = 1.0;
            }
            t0 = std::chrono::steady_clock::now();
            info = LAPACKE_dsytrs2(kColMajor, 'L', (int)n, (int)c, z.data(), (int)n, ipiv.data(), inv.data(), (int)n);
            t1 = std::chrono::steady_clock::now();
            g_trs_t[pass] = std::chrono::duration<double>(t1 - t0).count();
            g_trs_c[pass] = c;
        }
        if (t_trs) *t_trs = g_trs_t[1] + (g_trs_t[1] - g_trs_t[0]) * double(n - c2) / double(c2 - c1);
    } else {
        t0 = std::chrono::steady_clock::now();
        info = LAPACKE_dsytrs2(kColMajor, 'L', (int)n, (int)n, z.data(), (int)n, ipiv.data(), inv.data(), (int)n);
        t1 = std::chrono::steady_clock::now();
        if (t_trs) *t_trs = std::chrono::duration<double>(t1 - t0).count();
    }
    if (info != 0) throw Error{kDegenerate, "factorization", "solve against identity failed with status " + std::to_string(info)};
    for (int64_t c = 0; c < n; ++c)
        for (int64_t r = c + 1; r < n; ++r) {
            const double v = 0.5 * (inv[size_t(c) * n + r] + inv[size_t(r) * n + c]);
            inv[size_t(c) * n + r] = v;
            inv[size_t(r) * n + c] = v;
        }
    return inv;
}

// ---- extraction: src/covariance.cpp:259-279 -----------------------------------
template <int P>
inline void extract_camera_covariances(const std::vector<double>& zinv, int64_t dim, const std::vector<double>& s_a,
                                       int64_t n, double* cam_cov, oracle_diag* diag) {
    int warnings = 0;
    for (int64_t i = 0; i < n; ++i) {
        const double* s = &s_a[P * i];
        double* out = cam_cov + size_t(P) * P * i;
        for (int p = 0; p < P; ++p)
            for (int q = 0; q < P; ++q) out[P * p + q] = (s[p] * zinv[size_t(P * i + q) * dim + P * i + p]) * s[q];
        double a[P * P], d[P], v[P * P];
        for (int k = 0; k < P * P; ++k) a[k] = out[k];
        jacobi_eig<P>(a, d, v);
        double tr = 0.0, lmin = d[0];
        for (int p = 0; p < P; ++p) { tr += out[P * p + p]; lmin = std::min(lmin, d[p]); }
        if (lmin < -kPsdTol * tr) ++warnings;
    }
    diag->negative_eigenvalue_warnings = warnings;
    if (s_a.empty()) { diag->scale_min = diag->scale_max = 1.0; }
    else {
        diag->scale_min = *std::min_element(s_a.begin(), s_a.end());
        diag->scale_max = *std::max_element(s_a.begin(), s_a.end());
    }
}

// ---- point covariances: src/covariance.cpp:283-319 ----------------------------
// Sigma_X[j] = S_j (A_j^-1 + W Z_sub W^T) S_j, W = A_j^-1 [C_a^T ... | H_pj],
// Z_sub the bordered inverse restricted to the point's cameras and the border.
template <int P>
inline void extract_point_covariances(const System<P>& sys, const oracle_scene& s, const std::vector<M3>& a_inv,
                                      const std::vector<double>& zinv, int64_t dim, double* point_cov, int threads) {
    const int64_t n = sys.n;
    const int b = kGauge;
    parallel_for(sys.m, threads, [&](int64_t lo, int64_t hi) {
        std::vector<double> wj, zs, tmp;
        for (int64_t j = lo; j < hi; ++j) {
            const int64_t o0 = sys.by_pt.off[j], w = sys.by_pt.off[j + 1] - o0;
            const int64_t cols = P * w + b;
            wj.assign(size_t(3) * cols, 0.0);  // row-major 3 x cols
            for (int64_t a = 0; a < w; ++a) {
                const int64_t t = sys.by_pt.idx[o0 + a];
                const double* c = &sys.Cp[size_t(P) * 3 * t];  // P x 3, c[3p + q]
                for (int r = 0; r < 3; ++r)
                    for (int p = 0; p < P; ++p)
                        wj[size_t(r) * cols + P * a + p] =
                            (a_inv[j](r, 0) * c[3 * p] + a_inv[j](r, 1) * c[3 * p + 1]) + a_inv[j](r, 2) * c[3 * p + 2];
            }
            for (int r = 0; r < 3; ++r)
                for (int l = 0; l < b; ++l) {
                    const double* hr = &sys.H[size_t(P * n + 3 * j) * kGauge];
                    wj[size_t(r) * cols + P * w + l] =
                        (a_inv[j](r, 0) * hr[l] + a_inv[j](r, 1) * hr[kGauge + l]) + a_inv[j](r, 2) * hr[2 * kGauge + l];
                }
            // z_sub (cols x cols, row-major) from the bordered inverse
            zs.assign(size_t(cols) * cols, 0.0);
            auto gidx = [&](int64_t k) -> int64_t {  // global row/col of local index k
                if (k < P * w) {
                    const int64_t a = k / P;
                    return P * int64_t(s.obs_cam[sys.by_pt.idx[o0 + a]]) + (k - P * a);
                }
                return P * n + (k - P * w);
            };
            for (int64_t r = 0; r < cols; ++r) {
                const int64_t gr = gidx(r);
                for (int64_t c = 0; c < cols; ++c) zs[size_t(r) * cols + c] = zinv[size_t(gidx(c)) * dim + gr];
            }
            // cov = a_inv + (wj zs) wj^T
            tmp.assign(size_t(3) * cols, 0.0);
            for (int r = 0; r < 3; ++r)
                for (int64_t c = 0; c < cols; ++c) {
                    double v = 0.0;
                    for (int64_t k = 0; k < cols; ++k) v += wj[size_t(r) * cols + k] * zs[size_t(k) * cols + c];
                    tmp[size_t(r) * cols + c] = v;
                }
            const double* sp = &sys.s_a[P * n + 3 * j];
            for (int r = 0; r < 3; ++r)
                for (int q = 0; q < 3; ++q) {
                    double v = 0.0;
                    for (int64_t k = 0; k < cols; ++k) v += tmp[size_t(r) * cols + k] * wj[size_t(q) * cols + k];
                    point_cov[9 * j + 3 * r + q] = (sp[r] * (a_inv[j](r, q) + v)) * sp[q];
                }
        }
    });
}

// camera_matrix = S_c Z_inv[cams, cams] S_c (covariance.cpp:346-348), col-major N x N
template <int P>
inline void extract_camera_matrix(const std::vector<double>& zinv, int64_t dim, const std::vector<double>& s_a, int64_t n,
                                  double* cm) {
    const int64_t N = P * n;
    for (int64_t c = 0; c < N; ++c)
        for (int64_t r = 0; r < N; ++r) cm[size_t(c) * N + r] = (s_a[r] * zinv[size_t(c) * dim + r]) * s_a[c];
}

struct Timings { double validate = 0, jacobian = 0, nullspace = 0, fisher = 0, conditioning = 0, schur = 0, dsytrf = 0, dsytrs2 = 0, extract = 0, total = 0; };

inline double since(std::chrono::steady_clock::time_point t0) {
    return std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
}

// ---- pipeline: src/covariance.cpp:323-350 --------------------------------------
template <int P>
inline void compute_covariance(const oracle_scene& s, int threads, double* cam_cov, oracle_diag* diag,
                               int64_t* flagged, int64_t flagged_cap, Timings* tm, double* point_cov = nullptr,
                               double* camera_matrix = nullptr) {
    auto T0 = std::chrono::steady_clock::now();
    auto t0 = T0;
    validate(s);
    tm->validate = since(t0); t0 = std::chrono::steady_clock::now();
    const Jac<P> J = assemble_jacobian<P>(s, threads);
    tm->jacobian = since(t0); t0 = std::chrono::steady_clock::now();
    std::vector<double> h = fixed_nullspace_blocks<P>(s);
    solve_rotation_blocks<P>(s, J, h);
    tm->nullspace = since(t0); t0 = std::chrono::steady_clock::now();
    System<P> sys = build_fisher_blocks<P>(s, J, std::move(h), threads);
    tm->fisher = since(t0); t0 = std::chrono::steady_clock::now();
    condition_columns<P>(sys);
    apply_conditioning<P>(sys, s);
    tm->conditioning = since(t0); t0 = std::chrono::steady_clock::now();
    std::memset(diag, 0, sizeof(*diag));
    const int64_t dim = P * sys.n + kGauge;
    diag->largest_dense_dim = dim;
    diag->peak_dense_bytes = 8 * dim * dim;
    std::vector<M3> a_inv;
    std::vector<double> z = schur_reduce<P>(sys, s, threads, point_cov ? &a_inv : nullptr);
    tm->schur = since(t0); t0 = std::chrono::steady_clock::now();
    const std::vector<double> zinv = invert_schur(std::move(z), dim, diag, &tm->dsytrf, &tm->dsytrs2);
    t0 = std::chrono::steady_clock::now();
    extract_camera_covariances<P>(zinv, dim, sys.s_a, sys.n, cam_cov, diag);
    if (point_cov) extract_point_covariances<P>(sys, s, a_inv, zinv, dim, point_cov, threads);
    if (camera_matrix) extract_camera_matrix<P>(zinv, dim, sys.s_a, sys.n, camera_matrix);
    diag->n_flagged = (int32_t)sys.flagged.size();
    for (int64_t k = 0; k < std::min<int64_t>(flagged_cap, (int64_t)sys.flagged.size()); ++k) flagged[k] = sys.flagged[k];
    tm->extract = since(t0);
    tm->total = since(T0);
}

// ---- dense Moore–Penrose oracle: src/oracle.cpp:16-72 ---------------------------
template <int P>
inline std::vector<double> dense_fisher(const oracle_scene& s) {
    const Jac<P> J = assemble_jacobian<P>(s, 1);
    System<P> sys = build_fisher_blocks<P>(s, J, std::vector<double>(), 1);
    const int64_t n = sys.n, m = sys.m, N = P * n + 3 * m;
    std::vector<double> f(size_t(N) * N, 0.0);
    auto F = [&](int64_t r, int64_t c) -> double& { return f[size_t(c) * N + r]; };
    for (int64_t i = 0; i < n; ++i)
        for (int p = 0; p < P; ++p)
            for (int q = 0; q < P; ++q) F(P * i + p, P * i + q) = sys.D[size_t(P) * P * i + P * p + q];
    for (int64_t j = 0; j < m; ++j)
        for (int p = 0; p < 3; ++p)
            for (int q = 0; q < 3; ++q) F(P * n + 3 * j + p, P * n + 3 * j + q) = sys.A[9 * j + 3 * p + q];
    for (int64_t t = 0; t < sys.T; ++t) {
        const int64_t ci = s.obs_cam[t], pj = s.obs_pt[t];
        for (int p = 0; p < P; ++p)
            for (int q = 0; q < 3; ++q) {
                const double v = sys.Cp[size_t(P) * 3 * t + 3 * p + q];
                F(P * ci + p, P * n + 3 * pj + q) = v;
                F(P * n + 3 * pj + q, P * ci + p) = v;
            }
    }
    return f;
}

// Camera blocks of the inverse of the bordered Fisher matrix
// K = [[F, H], [H^T, 0]] (F the dense unconditioned Fisher matrix, H the
// gauge basis, both in FP64 as the restatement forms them), solved in long
// double: LU with partial pivoting plus two refinement steps with long-double
// residuals.  An independent CPU truth for small scenes, to validate the
// GPU's double-double refinement (sfmcov_cuda_refine_covariance).  The
// Jacobi scaling of the reference (src/covariance.cpp:84-135) cancels
// exactly, so it is not applied.
template <int P>
void exact_camera_blocks(const oracle_scene& s, int64_t max_params, double* cam_cov) {
    const int64_t n = s.n_cams, m = s.n_pts, Nf = P * n + 3 * m, dim = Nf + kGauge;
    if (Nf > max_params)
        throw Error{kSizeGuard, "oracle", "scene has " + std::to_string(Nf) + " parameters, guard is " +
                                              std::to_string(max_params)};
    const std::vector<double> F = dense_fisher<P>(s);
    const Jac<P> J = assemble_jacobian<P>(s, 1);
    std::vector<double> H = fixed_nullspace_blocks<P>(s);
    solve_rotation_blocks<P>(s, J, H);
    std::vector<long double> K(size_t(dim) * dim, 0.0L);  // column-major
    auto k = [&](int64_t r, int64_t c) -> long double& { return K[size_t(c) * dim + r]; };
    for (int64_t c = 0; c < Nf; ++c)
        for (int64_t r = 0; r < Nf; ++r) k(r, c) = F[size_t(c) * Nf + r];
    for (int64_t r = 0; r < Nf; ++r)
        for (int l = 0; l < kGauge; ++l) {
            k(r, Nf + l) = H[size_t(r) * kGauge + l];
            k(Nf + l, r) = H[size_t(r) * kGauge + l];
        }
    std::vector<long double> LU = K;
    std::vector<int64_t> piv(dim);
    auto lu = [&](int64_t r, int64_t c) -> long double& { return LU[size_t(c) * dim + r]; };
    for (int64_t c = 0; c < dim; ++c) {
        int64_t pr = c;
        for (int64_t r = c + 1; r < dim; ++r)
            if (std::fabs((double)lu(r, c)) > std::fabs((double)lu(pr, c))) pr = r;
        piv[c] = pr;
        if (pr != c)
            for (int64_t cc = 0; cc < dim; ++cc) std::swap(lu(c, cc), lu(pr, cc));
        const long double d = lu(c, c);
        if (d == 0.0L) throw Error{kDegenerate, "oracle", "singular bordered Fisher matrix"};
        for (int64_t r = c + 1; r < dim; ++r) lu(r, c) /= d;
        for (int64_t cc = c + 1; cc < dim; ++cc) {
            const long double f = lu(c, cc);
            if (f == 0.0L) continue;
            long double* col = &LU[size_t(cc) * dim];
            const long double* lc = &LU[size_t(c) * dim];
            for (int64_t r = c + 1; r < dim; ++r) col[r] -= lc[r] * f;
        }
    }
    auto solve = [&](std::vector<long double>& x) {
        for (int64_t c = 0; c < dim; ++c) std::swap(x[c], x[piv[c]]);
        for (int64_t c = 0; c < dim; ++c) {
            const long double v = x[c];
            if (v == 0.0L) continue;
            const long double* lc = &LU[size_t(c) * dim];
            for (int64_t r = c + 1; r < dim; ++r) x[r] -= lc[r] * v;
        }
        for (int64_t c = dim - 1; c >= 0; --c) {
            x[c] /= lu(c, c);
            const long double v = x[c];
            const long double* uc = &LU[size_t(c) * dim];
            for (int64_t r = 0; r < c; ++r) x[r] -= uc[r] * v;
        }
    };
    std::vector<long double> x(dim), r(dim);
    for (int64_t i = 0; i < n; ++i)
        for (int q = 0; q < P; ++q) {
            const int64_t col = P * i + q;
            std::fill(x.begin(), x.end(), 0.0L);
            x[col] = 1.0L;
            solve(x);
            for (int it = 0; it < 2; ++it) {
                std::fill(r.begin(), r.end(), 0.0L);
                r[col] = 1.0L;
                for (int64_t c = 0; c < dim; ++c) {
                    const long double v = x[c];
                    const long double* kc = &K[size_t(c) * dim];
                    for (int64_t rr = 0; rr < dim; ++rr) r[rr] -= kc[rr] * v;
                }
                solve(r);
                for (int64_t c = 0; c < dim; ++c) x[c] += r[c];
            }
            for (int p = 0; p < P; ++p) cam_cov[size_t(P) * P * i + P * p + q] = (double)x[P * i + p];
        }
}

}  // namespace oracle

// =============================================================================
// C ABI for ctypes (tests / bench cpu leg only)
// =============================================================================
using namespace oracle;

extern "C" struct oracle_error {
    int32_t kind;
    char stage[32];
    char message[480];
};

static int fail(oracle_error* e, const Error& x) {
    if (e) {
        e->kind = x.kind;
        std::snprintf(e->stage, sizeof e->stage, "%s", x.stage.c_str());
        std::snprintf(e->message, sizeof e->message, "%s: %s", x.stage.c_str(), x.message.c_str());
    }
    return x.kind;
}
static int ok(oracle_error* e) {
    if (e) { e->kind = 0; e->stage[0] = 0; e->message[0] = 0; }
    return 0;
}

#define ORACLE_DISPATCH(P_, BODY)                    \
    do {                                             \
        if ((P_) == 8) { constexpr int P = 8; BODY; } \
        else if ((P_) == 9) { constexpr int P = 9; BODY; } \
        else throw Error{kDimension, "validate", "camera width must be 8 or 9"}; \
    } while (0)

extern "C" {

const char* oracle_blas_corename(void) { return openblas_get_corename(); }
void oracle_blas_threads(int n) { g_blas_threads = n > 0 ? n : 1; openblas_set_num_threads(g_blas_threads); }
void oracle_trs_sample(int k) { g_trs_sample = k > 0 ? k : 1; }
// the last sampled dsytrs2: columns and seconds of the two passes
void oracle_trs_sample_info(int64_t* cols, double* secs) {
    cols[0] = g_trs_c[0]; cols[1] = g_trs_c[1]; secs[0] = g_trs_t[0]; secs[1] = g_trs_t[1];
}

int oracle_validate(const oracle_scene* s, oracle_error* e) {
    try { validate(*s); return ok(e); } catch (const Error& x) { return fail(e, x); }
}

// CSR: off_cam (n+1), idx_cam (t), off_pt (m+1), idx_pt (t)
int oracle_observation_index(const oracle_scene* s, int64_t* off_cam, int32_t* idx_cam, int64_t* off_pt, int32_t* idx_pt) {
    Csr a, b;
    build_index(*s, &a, &b);
    std::memcpy(off_cam, a.off.data(), 8 * a.off.size());
    std::memcpy(idx_cam, a.idx.data(), 4 * a.idx.size());
    std::memcpy(off_pt, b.off.data(), 8 * b.off.size());
    std::memcpy(idx_pt, b.idx.data(), 4 * b.idx.size());
    return 0;
}

void oracle_rotation_matrix(const double* r, double* R) { const M3 m = rotation_matrix(r); std::memcpy(R, m.a, 72); }
void oracle_rotate_point_derivative(const double* r, const double* w, double* D) {
    const M3 m = rotate_point_derivative(r, w); std::memcpy(D, m.a, 72);
}
void oracle_sincos(double x, double* s, double* c) { dm::sincos_pos(x, s, c); }

// One (camera, point) Jacobian: jc 2×P, jp 2×3.  Returns 4 (degenerate) when
// the point is behind the camera, with the reference's "projection" message.
int oracle_observation_jacobian(int P_, const double* cam, const double* X, double* jc, double* jp, oracle_error* e) {
    try {
        double depth = 0.0;
        bool good = false;
        ORACLE_DISPATCH(P_, good = observation_jacobian<P>(cam, X, jc, jp, &depth));
        if (!good) {
            char buf[64];
            std::snprintf(buf, sizeof buf, "%f", depth);
            throw Error{kDegenerate, "projection", std::string("point at camera-space depth ") + buf +
                                                     " (behind camera or on the principal plane)"};
        }
        return ok(e);
    } catch (const Error& x) { return fail(e, x); }
}

// u = c(1 + kρ[+k2ρ²]) u_n (projection.cpp:36-39)
int oracle_project(int P_, const double* cam, const double* X, double* u, oracle_error* e) {
    const M3 R = rotation_matrix(cam);
    const double w[3] = {X[0] - cam[3], X[1] - cam[4], X[2] - cam[5]};
    double v[3];
    for (int i = 0; i < 3; ++i) v[i] = (R(i, 0) * w[0] + R(i, 1) * w[1]) + R(i, 2) * w[2];
    if (!(v[2] > kDepthEps)) {
        char buf[64];
        std::snprintf(buf, sizeof buf, "%f", v[2]);
        return fail(e, Error{kDegenerate, "projection", std::string("point at camera-space depth ") + buf +
                                                           " (behind camera or on the principal plane)"});
    }
    const double un0 = v[0] / v[2], un1 = v[1] / v[2];
    const double rho = un0 * un0 + un1 * un1;
    double d = 1.0 + cam[7] * rho;
    if (P_ == 9) d = d + cam[8] * (rho * rho);
    u[0] = cam[6] * d * un0;
    u[1] = cam[6] * d * un1;
    return ok(e);
}

int oracle_jacobian(const oracle_scene* s, int threads, double* jc, double* jp, oracle_error* e) {
    try {
        ORACLE_DISPATCH(s->cam_params, {
            const Jac<P> J = assemble_jacobian<P>(*s, threads);
            std::memcpy(jc, J.jc.data(), 8 * J.jc.size());
            std::memcpy(jp, J.jp.data(), 8 * J.jp.size());
        });
        return ok(e);
    } catch (const Error& x) { return fail(e, x); }
}

// H: (P·n + 3m) × 7 row-major.  Also returns the |JH| residual.
int oracle_nullspace(const oracle_scene* s, double* h, double* residual, oracle_error* e) {
    try {
        ORACLE_DISPATCH(s->cam_params, {
            const Jac<P> J = assemble_jacobian<P>(*s, 1);
            std::vector<double> H = fixed_nullspace_blocks<P>(*s);
            solve_rotation_blocks<P>(*s, J, H);
            std::memcpy(h, H.data(), 8 * H.size());
            if (residual) *residual = nullspace_residual<P>(*s, J, H);
        });
        return ok(e);
    } catch (const Error& x) { return fail(e, x); }
}

// Residual of an arbitrary basis h (rows × 7 row-major).
double oracle_nullspace_residual(const oracle_scene* s, const double* h) {
    double r = -1.0;
    try {
        ORACLE_DISPATCH(s->cam_params, {
            const Jac<P> J = assemble_jacobian<P>(*s, 1);
            std::vector<double> H(h, h + size_t(P * s->n_cams + 3 * s->n_pts) * kGauge);
            r = nullspace_residual<P>(*s, J, H);
        });
    } catch (...) {}
    return r;
}

// Unconditioned Fisher blocks and the conditioning scales.
// D n×P×P, A m×9, Cp t×P×3 (row-major blocks); s_a (Pn+3m), s_b (7).
int oracle_fisher(const oracle_scene* s, double* D, double* A, double* Cp, double* s_a, double* s_b,
                  int64_t* flagged, int64_t flagged_cap, int64_t* n_flagged, oracle_error* e) {
    try {
        // like build_fisher_blocks (covariance.cpp:33-82): no scene validation,
        // only the index ranges the restatement needs to stay in bounds
        for (int64_t t = 0; t < s->n_obs; ++t)
            if (s->obs_cam[t] < 0 || s->obs_cam[t] >= s->n_cams || s->obs_pt[t] < 0 || s->obs_pt[t] >= s->n_pts)
                throw Error{kInvariant, "validate", "observation " + std::to_string(t) + " index out of range"};
        ORACLE_DISPATCH(s->cam_params, {
            const Jac<P> J = assemble_jacobian<P>(*s, 1);
            std::vector<double> H = fixed_nullspace_blocks<P>(*s);
            solve_rotation_blocks<P>(*s, J, H);
            System<P> sys = build_fisher_blocks<P>(*s, J, std::move(H), 1);
            if (D) std::memcpy(D, sys.D.data(), 8 * sys.D.size());
            if (A) std::memcpy(A, sys.A.data(), 8 * sys.A.size());
            if (Cp) std::memcpy(Cp, sys.Cp.data(), 8 * sys.Cp.size());
            condition_columns<P>(sys);
            if (s_a) std::memcpy(s_a, sys.s_a.data(), 8 * sys.s_a.size());
            if (s_b) std::memcpy(s_b, sys.s_b.data(), 8 * sys.s_b.size());
            if (n_flagged) *n_flagged = (int64_t)sys.flagged.size();
            for (int64_t k = 0; k < std::min<int64_t>(flagged_cap, (int64_t)sys.flagged.size()); ++k) flagged[k] = sys.flagged[k];
        });
        return ok(e);
    } catch (const Error& x) { return fail(e, x); }
}

// Conditioned bordered Schur matrix Z_p, dense col-major (Pn+7)².
int oracle_schur(const oracle_scene* s, int threads, double* z_out, oracle_error* e) {
    try {
        validate(*s);
        ORACLE_DISPATCH(s->cam_params, {
            const Jac<P> J = assemble_jacobian<P>(*s, threads);
            std::vector<double> H = fixed_nullspace_blocks<P>(*s);
            solve_rotation_blocks<P>(*s, J, H);
            System<P> sys = build_fisher_blocks<P>(*s, J, std::move(H), threads);
            condition_columns<P>(sys);
            apply_conditioning<P>(sys, *s);
            const std::vector<double> z = schur_reduce<P>(sys, *s, threads, nullptr);
            std::memcpy(z_out, z.data(), 8 * z.size());
        });
        return ok(e);
    } catch (const Error& x) { return fail(e, x); }
}

// invert_schur on an arbitrary symmetric col-major n×n matrix.
int oracle_invert_schur(const double* z, int64_t n, double* z_inv, oracle_diag* diag, oracle_error* e) {
    try {
        std::memset(diag, 0, sizeof(*diag));
        std::vector<double> a(z, z + size_t(n) * n);
        const std::vector<double> inv = invert_schur(std::move(a), n, diag, nullptr, nullptr);
        std::memcpy(z_inv, inv.data(), 8 * inv.size());
        return ok(e);
    } catch (const Error& x) { return fail(e, x); }
}

// Full pipeline.  cam_cov: n × P × P row-major blocks.  times (10 doubles):
// validate, jacobian, nullspace, fisher, conditioning, schur, dsytrf, dsytrs2,
// extract, total.
int oracle_compute_covariance(const oracle_scene* s, int threads, double* cam_cov, oracle_diag* diag,
                              int64_t* flagged, int64_t flagged_cap, double* times, oracle_error* e) {
    try {
        Timings tm;
        if (s->cam_params != 8 && s->cam_params != 9) throw Error{kDimension, "validate", "camera width must be 8 or 9"};
        if (s->cam_params == 8) compute_covariance<8>(*s, threads, cam_cov, diag, flagged, flagged_cap, &tm);
        else compute_covariance<9>(*s, threads, cam_cov, diag, flagged, flagged_cap, &tm);
        if (times) {
            const double v[10] = {tm.validate, tm.jacobian, tm.nullspace, tm.fisher, tm.conditioning,
                                  tm.schur, tm.dsytrf, tm.dsytrs2, tm.extract, tm.total};
            std::memcpy(times, v, sizeof v);
        }
        return ok(e);
    } catch (const Error& x) { return fail(e, x); }
}

// compute_covariance with CovarianceOptions::point_covariances /
// camera_cross_covariances: point_cov m x 3 x 3 (row-major blocks),
// camera_matrix P n x P n col-major; either may be NULL.
int oracle_compute_covariance_full(const oracle_scene* s, int threads, double* cam_cov, double* point_cov,
                                   double* camera_matrix, oracle_diag* diag, int64_t* flagged, int64_t flagged_cap,
                                   oracle_error* e) {
    try {
        Timings tm;
        if (s->cam_params != 8 && s->cam_params != 9) throw Error{kDimension, "validate", "camera width must be 8 or 9"};
        if (s->cam_params == 8)
            compute_covariance<8>(*s, threads, cam_cov, diag, flagged, flagged_cap, &tm, point_cov, camera_matrix);
        else
            compute_covariance<9>(*s, threads, cam_cov, diag, flagged, flagged_cap, &tm, point_cov, camera_matrix);
        return ok(e);
    } catch (const Error& x) { return fail(e, x); }
}

// Dense Fisher JᵀWJ, col-major (Pn+3m)².
int oracle_dense_fisher(const oracle_scene* s, double* f, oracle_error* e) {
    try {
        ORACLE_DISPATCH(s->cam_params, {
            const std::vector<double> F = dense_fisher<P>(*s);
            std::memcpy(f, F.data(), 8 * F.size());
        });
        return ok(e);
    } catch (const Error& x) { return fail(e, x); }
}

int oracle_exact_camera_blocks(const oracle_scene* s, int64_t max_params, double* cam_cov, oracle_error* e) {
    try {
        ORACLE_DISPATCH(s->cam_params, exact_camera_blocks<P>(*s, max_params, cam_cov));
        return ok(e);
    } catch (const Error& x) { return fail(e, x); }
}

// pseudoinverse_covariance (src/oracle.cpp:34-72): dgesdd, exactly the 7
// trailing singular values dropped (count-based), symmetrised.
int oracle_pseudoinverse(const oracle_scene* s, int64_t max_params, double* cam_cov, double* sigma_full,
                         double* singular_values, double* gauge_gap, oracle_error* e) {
    try {
        const int P_ = s->cam_params;
        const int64_t params = int64_t(P_) * s->n_cams + 3 * int64_t(s->n_pts);
        if (params > max_params)
            throw Error{kSizeGuard, "oracle", "scene has " + std::to_string(params) + " parameters, guard is " + std::to_string(max_params)};
        validate(*s);
        openblas_set_num_threads(1);
        std::vector<double> f;
        ORACLE_DISPATCH(P_, f = dense_fisher<P>(*s));
        const int n = (int)params;
        std::vector<double> u(size_t(n) * n), vt(size_t(n) * n), sv(n);
        const int info = LAPACKE_dgesdd(kColMajor, 'A', n, n, f.data(), n, sv.data(), u.data(), n, vt.data(), n);
        if (info != 0) throw Error{kDegenerate, "oracle", "SVD failed with status " + std::to_string(info)};
        std::vector<double> sinv(n, 0.0);
        for (int i = 0; i + kGauge < n; ++i) sinv[i] = 1.0 / sv[i];
        if (gauge_gap) *gauge_gap = sv[n - kGauge - 1] / sv[n - kGauge];
        // sigma = V S⁺ Uᵀ  (col-major): sigma(r,c) = Σ_k vt(k,r) sinv_k u(c,k)
        std::vector<double> sg(size_t(n) * n, 0.0);
        for (int c = 0; c < n; ++c)
            for (int k = 0; k < n - kGauge; ++k) {
                const double uck = u[size_t(k) * n + c] * sinv[k];
                for (int r = 0; r < n; ++r) sg[size_t(c) * n + r] += vt[size_t(r) * n + k] * uck;
            }
        for (int c = 0; c < n; ++c)
            for (int r = c + 1; r < n; ++r) {
                const double v = 0.5 * (sg[size_t(c) * n + r] + sg[size_t(r) * n + c]);
                sg[size_t(c) * n + r] = v;
                sg[size_t(r) * n + c] = v;
            }
        if (singular_values) std::memcpy(singular_values, sv.data(), 8 * sv.size());
        if (sigma_full) std::memcpy(sigma_full, sg.data(), 8 * sg.size());
        if (cam_cov)
            for (int64_t i = 0; i < s->n_cams; ++i)
                for (int p = 0; p < P_; ++p)
                    for (int q = 0; q < P_; ++q)
                        cam_cov[size_t(P_) * P_ * i + P_ * p + q] = sg[size_t(P_ * i + q) * n + P_ * i + p];
        return ok(e);
    } catch (const Error& x) { return fail(e, x); }
}

// Cholesky-route restatement of the gauge-fixed inversion (SURVEY.md appendix
// A, "route A"): from the conditioned bordered Z_p, Z_aug = Z − Γ E⁻¹ Γᵀ,
// dpotrf + dtrtri, Σ_ii = Σ_k (L⁻¹)_kiᵀ (L⁻¹)_ki, unscaled by s_a.  Used as
// the "CPU-best" comparison line and to cross-check the GPU algorithm.
int oracle_cholesky_route(const double* zp, int64_t n_cams, int P_, const double* s_a_cams, int blas_threads,
                          double* cam_cov, oracle_error* e) {
    try {
        const int64_t N = int64_t(P_) * n_cams, dim = N + kGauge;
        openblas_set_num_threads(blas_threads);
        // E⁻¹ via dpotrf of −E
        std::vector<double> F(kGauge * kGauge);
        for (int c = 0; c < kGauge; ++c)
            for (int r = 0; r < kGauge; ++r) F[c * kGauge + r] = -zp[size_t(N + c) * dim + N + r];
        if (LAPACKE_dpotrf(kColMajor, 'L', kGauge, F.data(), kGauge) != 0)
            throw Error{kDegenerate, "factorization", "border block is not negative definite; the scene is likely disconnected or its gauge degenerate"};
        // G = Γ L_F⁻ᵀ  → Z_aug = Z + G Gᵀ
        std::vector<double> G(size_t(N) * kGauge);
        for (int64_t r = 0; r < N; ++r) {
            double g[kGauge];
            for (int l = 0; l < kGauge; ++l) {
                double acc = zp[size_t(N + l) * dim + r];
                for (int k = 0; k < l; ++k) acc -= g[k] * F[k * kGauge + l];
                g[l] = acc / F[l * kGauge + l];
            }
            for (int l = 0; l < kGauge; ++l) G[size_t(l) * N + r] = g[l];
        }
        std::vector<double> a(size_t(N) * N);
        for (int64_t c = 0; c < N; ++c)
            for (int64_t r = 0; r < N; ++r) {
                double acc = zp[size_t(c) * dim + r];
                for (int l = 0; l < kGauge; ++l) acc += G[size_t(l) * N + r] * G[size_t(l) * N + c];
                a[size_t(c) * N + r] = acc;
            }
        if (LAPACKE_dpotrf(kColMajor, 'L', (int)N, a.data(), (int)N) != 0)
            throw Error{kDegenerate, "factorization", "Cholesky failed; the scene is likely disconnected or its gauge degenerate"};
        if (LAPACKE_dtrtri(kColMajor, 'L', 'N', (int)N, a.data(), (int)N) != 0)
            throw Error{kDegenerate, "factorization", "triangular inverse failed"};
        for (int64_t i = 0; i < n_cams; ++i)
            for (int p = 0; p < P_; ++p)
                for (int q = 0; q < P_; ++q) {
                    const int64_t cp = P_ * i + p, cq = P_ * i + q;
                    double acc = 0.0;
                    for (int64_t r = std::max(cp, cq); r < N; ++r) acc += a[size_t(cp) * N + r] * a[size_t(cq) * N + r];
                    cam_cov[size_t(P_) * P_ * i + P_ * p + q] = (s_a_cams[cp] * acc) * s_a_cams[cq];
                }
        openblas_set_num_threads(1);
        return ok(e);
    } catch (const Error& x) { return fail(e, x); }
}

}  // extern "C"
