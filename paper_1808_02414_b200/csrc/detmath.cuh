// Deterministic small-matrix math shared by the stage-(a)/(c) kernels.
//
// Every formula fixes its operation order so that, compiled with
// --fmad=false (no FMA contraction) and IEEE div/sqrt, the device results
// are bit-identical to the CPU restatement in oracle/ (which uses the same
// op sequences with -ffp-contract=off).  This is what makes the Jacobian,
// the gauge nullspace rotation blocks and the per-camera Fisher blocks
// bit-exact against the reference restatement (BASELINE.json north_star).
//
// Reference formulas: rotation.cpp:7-28,70-77 (skew, Rodrigues,
// d(Rw)/dr); projection.cpp:41-59 (analytic Jacobian); nullspace.cpp:40-61
// (rotation normal equations); covariance.cpp:147-153 (3x3 eigen-inverse
// with the lam_min < 1e-12 lam_max singularity test).
#pragma once

#include <cstdint>

#ifndef SFM_HD
#define SFM_HD __host__ __device__ __forceinline__
#endif

namespace sfm {

constexpr double kDepthEps = 1e-9;
constexpr double kRotationTaylorEps = 1e-8;
constexpr double kRotationCondTol = 1e-12;
constexpr double kPivotRtol = 1e-12;
constexpr double kPsdTol = 1e-9;
constexpr int kGauge = 7;

// ---- sin/cos: fdlibm-style kernels on [-pi/4, pi/4], Cody–Waite reduction --
SFM_HD double ksin(double x) {
    const double S1 = -1.66666666666666324348e-01, S2 = 8.33333333332248946124e-03,
                 S3 = -1.98412698298579493134e-04, S4 = 2.75573137070700676789e-06,
                 S5 = -2.50507602534068634195e-08, S6 = 1.58969099521155010221e-10;
    const double z = x * x;
    const double w = z * z;
    const double r = (S2 + z * (S3 + z * S4)) + (z * w) * (S5 + z * S6);
    const double v = z * x;
    return x + v * (S1 + z * r);
}

SFM_HD double kcos(double x) {
    const double C1 = 4.16666666666666019037e-02, C2 = -1.38888888888741095749e-03,
                 C3 = 2.48015872894767294178e-05, C4 = -2.75573143513906633035e-07,
                 C5 = 2.08757232129817482790e-09, C6 = -1.13596475577881948265e-11;
    const double z = x * x;
    const double w = z * z;
    const double r = z * (C1 + z * (C2 + z * C3)) + (w * w) * (C4 + z * (C5 + z * C6));
    const double hz = 0.5 * z;
    const double one_minus = 1.0 - hz;
    return one_minus + (((1.0 - one_minus) - hz) + z * r);
}

SFM_HD void sincos_pos(double x, double* s, double* c) {
    const double kInvPio2 = 6.36619772367581382433e-01;
    const double kPio2Hi = 1.57079632673412561417e+00;
    const double kPio2Lo = 6.07710050650619224932e-11;
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

// ---- 3x3 (row-major) ---------------------------------------------------------
struct M3 { double a[9]; };

SFM_HD void mul3(const double* A, const double* B, double* C) {
    for (int i = 0; i < 3; ++i)
        for (int j = 0; j < 3; ++j)
            C[3 * i + j] = (A[3 * i + 0] * B[0 + j] + A[3 * i + 1] * B[3 + j]) + A[3 * i + 2] * B[6 + j];
}

SFM_HD void skew(const double* v, double* s) {
    s[0] = 0.0;   s[1] = -v[2]; s[2] = v[1];
    s[3] = v[2];  s[4] = 0.0;   s[5] = -v[0];
    s[6] = -v[1]; s[7] = v[0];  s[8] = 0.0;
}

SFM_HD void rotation_matrix(const double* r, double* R) {
    const double theta2 = (r[0] * r[0] + r[1] * r[1]) + r[2] * r[2];
    double rx[9], rx2[9];
    skew(r, rx);
    double a, b;
    if (theta2 < kRotationTaylorEps * kRotationTaylorEps) {
        a = 1.0 - theta2 / 6.0;
        b = 0.5 - theta2 / 24.0;
    } else {
        const double theta = sqrt(theta2);
        double s, c;
        sincos_pos(theta, &s, &c);
        a = s / theta;
        b = (1.0 - c) / theta2;
    }
    mul3(rx, rx, rx2);
    for (int i = 0; i < 3; ++i)
        for (int j = 0; j < 3; ++j)
            R[3 * i + j] = ((i == j ? 1.0 : 0.0) + a * rx[3 * i + j]) + b * rx2[3 * i + j];
}

// d(R(r) w)/dr given R = rotation_matrix(r).
SFM_HD void rotate_point_derivative(const double* r, const double* w, const double* R, double* out) {
    const double theta2 = (r[0] * r[0] + r[1] * r[1]) + r[2] * r[2];
    double sw[9];
    skew(w, sw);
    if (theta2 < kRotationTaylorEps * kRotationTaylorEps) {
        const double rxw[3] = {r[1] * w[2] - r[2] * w[1], r[2] * w[0] - r[0] * w[2], r[0] * w[1] - r[1] * w[0]};
        double s1[9], sr[9], s2[9];
        skew(rxw, s1);
        skew(r, sr);
        mul3(sr, sw, s2);
        for (int k = 0; k < 9; ++k) out[k] = -sw[k] - 0.5 * (s1[k] + s2[k]);
        return;
    }
    double negR[9], t1[9], sr[9], rtmi[9], p[9], m2[9], num[9];
    for (int k = 0; k < 9; ++k) negR[k] = -R[k];
    mul3(negR, sw, t1);
    skew(r, sr);
    for (int i = 0; i < 3; ++i)
        for (int j = 0; j < 3; ++j) rtmi[3 * i + j] = R[3 * j + i] - (i == j ? 1.0 : 0.0);
    mul3(rtmi, sr, p);
    for (int i = 0; i < 3; ++i)
        for (int j = 0; j < 3; ++j) m2[3 * i + j] = r[i] * r[j] + p[3 * i + j];
    mul3(t1, m2, num);
    for (int k = 0; k < 9; ++k) out[k] = num[k] / theta2;
}

// Cyclic Jacobi (same sweeps/order as the oracle); eigenvalues in d
// (unsorted), eigenvectors in columns of v.
template <int N>
SFM_HD void jacobi_eig(double* a, double* d, double* v) {
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
                if (!(fabs(apq) > 1e-17 * sqrt(fabs(a[N * p + p] * a[N * q + q])))) {
                    a[N * p + q] = 0.0;
                    a[N * q + p] = 0.0;
                    continue;
                }
                rotated = true;
                const double theta = (a[N * q + q] - a[N * p + p]) / (2.0 * apq);
                const double at = fabs(theta);
                double t;
                if (at > 1e150) {
                    t = 0.5 / theta;
                } else {
                    t = 1.0 / (at + sqrt(theta * theta + 1.0));
                    if (theta < 0.0) t = -t;
                }
                const double c = 1.0 / sqrt(t * t + 1.0);
                const double s = t * c;
                for (int k = 0; k < N; ++k) {
                    const double akp = a[N * k + p], akq = a[N * k + q];
                    a[N * k + p] = c * akp - s * akq;
                    a[N * k + q] = s * akp + c * akq;
                }
                for (int k = 0; k < N; ++k) {
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

// Eigen-inverse of a symmetric 3x3 with the reference rank test.
SFM_HD bool eig_inverse3(const double* m, double tol, double* inv) {
    double a[9], d[3], v[9];
    for (int k = 0; k < 9; ++k) a[k] = m[k];
    jacobi_eig<3>(a, d, v);
    const double lmin = fmin(fmin(d[0], d[1]), d[2]);
    const double lmax = fmax(fmax(d[0], d[1]), d[2]);
    if (!(lmin > 0.0) || lmin < tol * lmax) return false;
    const double il[3] = {1.0 / d[0], 1.0 / d[1], 1.0 / d[2]};
    for (int i = 0; i < 3; ++i)
        for (int j = 0; j < 3; ++j)
            inv[3 * i + j] = (v[3 * i + 0] * il[0] * v[3 * j + 0] + v[3 * i + 1] * il[1] * v[3 * j + 1]) +
                             v[3 * i + 2] * il[2] * v[3 * j + 2];
    return true;
}

// Rank/condition test only (point blocks in the Schur stage).
SFM_HD bool eig_ok3(const double* m, double tol) {
    double a[9], d[3], v[9];
    for (int k = 0; k < 9; ++k) a[k] = m[k];
    jacobi_eig<3>(a, d, v);
    const double lmin = fmin(fmin(d[0], d[1]), d[2]);
    const double lmax = fmax(fmax(d[0], d[1]), d[2]);
    return (lmin > 0.0) && !(lmin < tol * lmax);
}

// ---- analytic observation Jacobian (projection.cpp:41-59) --------------------
// cam: r(3), C(3), c|f, k|k1[, k2]; R = rotation_matrix(r) (precomputed per
// camera; identical bits to recomputing it).  jc: 2 x P row-major, jp: 2 x 3.
template <int P>
SFM_HD bool observation_jacobian(const double* cam, const double* R, const double* X, double* jc, double* jp,
                                 double* depth) {
    const double* r = cam;
    const double* C = cam + 3;
    const double c = cam[6];
    const double k1 = cam[7];
    const double k2 = (P == 9) ? cam[8] : 0.0;
    const double w[3] = {X[0] - C[0], X[1] - C[1], X[2] - C[2]};
    double v[3];
    for (int i = 0; i < 3; ++i) v[i] = (R[3 * i + 0] * w[0] + R[3 * i + 1] * w[1]) + R[3 * i + 2] * w[2];
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
    double D[9];
    rotate_point_derivative(r, w, R, D);
    for (int i = 0; i < 2; ++i)
        for (int j = 0; j < 3; ++j) {
            const double dx = (A[i][0] * R[0 + j] + A[i][1] * R[3 + j]) + A[i][2] * R[6 + j];
            const double drr = (A[i][0] * D[0 + j] + A[i][1] * D[3 + j]) + A[i][2] * D[6 + j];
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

}  // namespace sfm
