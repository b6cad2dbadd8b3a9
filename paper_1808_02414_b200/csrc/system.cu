// Stage functions of the reference API on caller-supplied block systems
// (include/sfmcov/covariance.hpp:80-105, nullspace.hpp:36): the C++ drop-in
// header passes a BorderedSystem's arrays through these, so a caller can
// build, modify, condition and reduce a system step by step exactly like the
// reference's own tests do (tests/test_schur.cpp, test_fisher.cpp).  The
// full pipeline (capi.cu run()) does not use them: it fuses the same steps.
//
//   nullspace_residual   src/nullspace.cpp:70-83
//   condition_columns    src/covariance.cpp:84-116
//   apply_conditioning   src/covariance.cpp:118-135
//   schur_reduce         src/covariance.cpp:137-194 (any border width b)
//   extract_camera_covariances  src/covariance.cpp:259-279
//   full_covariance      src/covariance.cpp:352-397 (dense bordered K)
#include "common.cuh"
#include "detmath.cuh"
#include "kernels.cuh"

#include <algorithm>
#include <vector>

namespace sfm {

namespace {

__device__ __forceinline__ void atomic_max_nonneg(unsigned long long* a, double v) {
    atomicMax(a, (unsigned long long)__double_as_longlong(v));  // v >= 0: bit order = value order
}

// ---- nullspace_residual: max |J H| over observations, max |J|, max |H| -------
template <int P>
__global__ void k_nullres_obs(int t, int n, const int* oc, const int* op, const int* pos_cam, const double* rec,
                              const double* H, int b, unsigned long long* mx) {
    const int k = blockIdx.x * blockDim.x + threadIdx.x;
    if (k >= t) return;
    const double* jc = rec + (size_t)kRec * pos_cam[k];
    const double* jp = jc + 2 * P;
    const size_t rc = (size_t)P * oc[k], rp = (size_t)P * n + 3 * (size_t)op[k];
    double mjh = 0.0, mj = 0.0;
    for (int e = 0; e < 2 * P; ++e) mj = fmax(mj, fabs(jc[e]));
    for (int e = 0; e < 6; ++e) mj = fmax(mj, fabs(jp[e]));
    for (int l = 0; l < b; ++l)
        for (int row = 0; row < 2; ++row) {
            double v = 0.0;
            for (int p = 0; p < P; ++p) v += jc[P * row + p] * H[(rc + p) * b + l];
            double w = 0.0;
            for (int q = 0; q < 3; ++q) w += jp[3 * row + q] * H[(rp + q) * b + l];
            mjh = fmax(mjh, fabs(v + w));
        }
    atomic_max_nonneg(mx, mjh);
    atomic_max_nonneg(mx + 1, mj);
}
__global__ void k_absmax(const double* x, long long count, unsigned long long* mx) {
    double m = 0.0;
    for (long long e = (long long)blockIdx.x * blockDim.x + threadIdx.x; e < count; e += (long long)gridDim.x * blockDim.x)
        m = fmax(m, fabs(x[e]));
    atomic_max_nonneg(mx, m);
}

// ---- condition_columns ----------------------------------------------------------
template <int P>
__global__ void k_cond_sa(int n, int m, const double* D, const double* A, double* s_a, unsigned char* flags) {
    const long long c = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    const long long N = (long long)P * n;
    if (c >= N + 3LL * m) return;
    double d;
    if (c < N) {
        const long long i = c / P, p = c - i * P;
        d = D[(size_t)P * P * i + (P + 1) * p];
    } else {
        const long long j = (c - N) / 3, q = (c - N) - 3 * j;
        d = A[9 * (size_t)j + 4 * q];
    }
    if (d > 0.0) {
        s_a[c] = 1.0 / sqrt(d);
        flags[c] = 0;
    } else {
        s_a[c] = 1.0;
        flags[c] = 1;
    }
}
// per-block sums of (s_a[r] border[r, l])^2, then a fixed-order final sum
constexpr int kRowsPerBlock = 1024;
__global__ void k_cond_sb_part(long long rows, int b, const double* s_a, const double* border, double* part) {
    const int l = threadIdx.x;
    if (l >= b) return;
    const long long r0 = (long long)blockIdx.x * kRowsPerBlock, r1 = min(rows, r0 + kRowsPerBlock);
    double acc = 0.0;
    for (long long r = r0; r < r1; ++r) {
        const double v = s_a[r] * border[r * b + l];
        acc += v * v;
    }
    part[(size_t)blockIdx.x * b + l] = acc;
}
__global__ void k_cond_sb_final(int nblocks, int b, const double* part, double* s_b) {
    const int l = threadIdx.x;
    if (l >= b) return;
    double acc = 0.0;
    for (int k = 0; k < nblocks; ++k) acc += part[(size_t)k * b + l];
    const double norm = sqrt(acc);
    s_b[l] = norm > 0.0 ? 1.0 / norm : 1.0;
}

// ---- apply_conditioning (diag(d) M diag(d), evaluated (d_p M_pq) d_q) ----------
template <int P>
__global__ void k_apply_cond(int n, int m, int t, int b, double* D, double* A, double* Cp, const int* oc,
                             const int* op, double* border, const double* s_a, const double* s_b) {
    const long long e = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    const long long nD = (long long)P * P * n, nA = 9LL * m, nC = (long long)P * 3 * t;
    const long long rows = (long long)P * n + 3LL * m, nB = rows * b;
    if (e < nD) {
        const long long i = e / (P * P), pq = e - i * P * P, p = pq / P, q = pq - p * P;
        D[e] = (s_a[P * i + p] * D[e]) * s_a[P * i + q];
    } else if (e < nD + nA) {
        const long long f = e - nD, j = f / 9, pq = f - 9 * j, p = pq / 3, q = pq - 3 * p;
        const size_t base = (size_t)P * n + 3 * (size_t)j;
        A[f] = (s_a[base + p] * A[f]) * s_a[base + q];
    } else if (e < nD + nA + nC) {
        const long long f = e - nD - nA, k = f / (P * 3), pq = f - k * P * 3, p = pq / 3, q = pq - 3 * p;
        Cp[f] = (s_a[(size_t)P * oc[k] + p] * Cp[f]) * s_a[(size_t)P * n + 3 * (size_t)op[k] + q];
    } else if (e < nD + nA + nC + nB) {
        const long long f = e - nD - nA - nC, r = f / b, l = f - r * b;
        border[f] = (s_a[r] * border[f]) * s_b[l];
    }
}

// ---- schur_reduce on a given system -------------------------------------------
// per point: the reference's singularity test, L = chol(A_j), V_j = L^-1 H_pj
// (3 x b), optional A_j^-1 = L^-T L^-1
template <int P>
__global__ void k_sys_point(int m, int n, const double* A, const double* border, int b, double* Lpt, double* V,
                            double* a_inv, Status* st) {
    const int j = blockIdx.x * blockDim.x + threadIdx.x;
    if (j >= m) return;
    double as[9];
    for (int k = 0; k < 9; ++k) as[k] = A[9 * (size_t)j + k];
    bool good = eig_ok3(as, kPivotRtol);
    double l00 = 1, l10 = 0, l11 = 1, l20 = 0, l21 = 0, l22 = 1;
    if (good) {
        l00 = sqrt(as[0]);
        l10 = as[3] / l00;
        l20 = as[6] / l00;
        const double d11 = as[4] - l10 * l10;
        l11 = sqrt(d11);
        l21 = (as[7] - l20 * l10) / l11;
        const double d22 = as[8] - l20 * l20 - l21 * l21;
        l22 = sqrt(d22);
        if (!(d11 > 0.0) || !(d22 > 0.0)) good = false;
    }
    if (!good) {
        atomicMin(&st->pt_sing_bad, j);
        l00 = 1; l10 = 0; l11 = 1; l20 = 0; l21 = 0; l22 = 1;
    }
    double* lo = Lpt + 8 * (size_t)j;
    lo[0] = l00; lo[1] = l10; lo[2] = l11; lo[3] = l20; lo[4] = l21; lo[5] = l22; lo[6] = good ? 1.0 : 0.0; lo[7] = 0.0;
    const size_t r0 = (size_t)P * n + 3 * (size_t)j;
    for (int l = 0; l < b; ++l) {
        const double h0 = border[(r0 + 0) * b + l], h1 = border[(r0 + 1) * b + l], h2 = border[(r0 + 2) * b + l];
        const double v0 = h0 / l00;
        const double v1 = (h1 - l10 * v0) / l11;
        const double v2 = (h2 - l20 * v0 - l21 * v1) / l22;
        V[(3 * (size_t)j + 0) * b + l] = v0;
        V[(3 * (size_t)j + 1) * b + l] = v1;
        V[(3 * (size_t)j + 2) * b + l] = v2;
    }
    if (a_inv) {  // L^-1 columns, then L^-T L^-1
        const double i00 = 1.0 / l00, i11 = 1.0 / l11, i22 = 1.0 / l22;
        const double i10 = -l10 * i00 * i11;
        const double i21 = -l21 * i11 * i22;
        const double i20 = -(l20 * i00 + l21 * i10) * i22;
        const double Li[9] = {i00, 0, 0, i10, i11, 0, i20, i21, i22};  // row-major lower
        double* o = a_inv + 9 * (size_t)j;
        for (int p = 0; p < 3; ++p)
            for (int q = 0; q < 3; ++q) {
                double v = 0.0;
                for (int k = 0; k < 3; ++k) v += Li[3 * k + p] * Li[3 * k + q];
                o[3 * p + q] = v;
            }
    }
}

// per by-camera slot: W = C L^-T (P x 3), stride kWStride
template <int P>
__global__ void k_sys_obs(int t, const int* idx_cam, const int* op, const double* Cp, const double* Lpt, double* Wb) {
    const int k = blockIdx.x * blockDim.x + threadIdx.x;
    if (k >= t) return;
    const int tt = idx_cam[k];
    const double* L = Lpt + 8 * (size_t)op[tt];
    const double* c = Cp + (size_t)P * 3 * tt;
    double* w = Wb + (size_t)kWStride * k;
    for (int p = 0; p < P; ++p) {
        const double w0 = c[3 * p] / L[0];
        const double w1 = (c[3 * p + 1] - L[1] * w0) / L[2];
        const double w2 = (c[3 * p + 2] - L[3] * w0 - L[4] * w1) / L[5];
        w[3 * p] = w0;
        w[3 * p + 1] = w1;
        w[3 * p + 2] = w2;
    }
    for (int z = 3 * P; z < kWStride; ++z) w[z] = 0.0;
}

// Z (N x N, ld N): the camera blocks D_i on the diagonal, zero elsewhere
template <int P>
__global__ void k_sys_zinit(int n, const double* D, double* Z) {
    const long long N = (long long)P * n;
    const long long e = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (e >= N * N) return;
    const long long r = e % N, c = e / N;
    Z[e] = (r / P == c / P) ? D[(size_t)P * P * (r / P) + P * (r % P) + (c % P)] : 0.0;
}

// Γ (N x b) = border_c - Σ_{slots of cam i} W V_j, in slot order
template <int P>
__global__ void k_sys_gamma(int n, int b, const int* off_cam, const int* idx_cam, const int* op, const double* Wb,
                            const double* V, const double* border, double* Gamma) {
    const long long e = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (e >= (long long)P * n * b) return;
    const long long row = e / b, l = e - row * b;
    const int i = (int)(row / P), p = (int)(row - (long long)i * P);
    double acc = 0.0;
    for (int k = off_cam[i]; k < off_cam[i + 1]; ++k) {
        const double* w = Wb + (size_t)kWStride * k;
        const size_t vj = 3 * (size_t)op[idx_cam[k]];
        acc += (w[3 * p] * V[vj * b + l] + w[3 * p + 1] * V[(vj + 1) * b + l]) + w[3 * p + 2] * V[(vj + 2) * b + l];
    }
    Gamma[e] = border[row * b + l] - acc;
}

// E (b x b) = -Σ_j V_j^T V_j: block partials of 1024 points, fixed-order final sum
__global__ void k_sys_e_part(int m, int b, const double* V, double* part) {
    const int e = threadIdx.x;
    if (e >= b * b) return;
    const int l1 = e / b, l2 = e - l1 * b;
    const long long j0 = (long long)blockIdx.x * kRowsPerBlock, j1 = min((long long)m, j0 + kRowsPerBlock);
    double acc = 0.0;
    for (long long j = j0; j < j1; ++j)
        acc += (V[(3 * j) * b + l1] * V[(3 * j) * b + l2] + V[(3 * j + 1) * b + l1] * V[(3 * j + 1) * b + l2]) +
               V[(3 * j + 2) * b + l1] * V[(3 * j + 2) * b + l2];
    part[(size_t)blockIdx.x * b * b + e] = acc;
}

// z_p (dim x dim, col-major, full): mirrored lower Z, Γ, Γ^T, E
__global__ void k_sys_assemble(int N, int b, const double* Z, const double* Gamma, const double* epart, int nparts,
                               double* zp) {
    const long long dim = (long long)N + b;
    const long long e = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (e >= dim * dim) return;
    const long long r = e % dim, c = e / dim;
    double v;
    if (r < N && c < N) v = r >= c ? Z[c * N + r] : Z[r * N + c];
    else if (r < N) v = Gamma[r * b + (c - N)];
    else if (c < N) v = Gamma[c * b + (r - N)];
    else {
        const long long l1 = r - N, l2 = c - N;
        const long long a = min(l1, l2), bb = max(l1, l2);  // one triangle: exact symmetry
        double s = 0.0;
        for (int k = 0; k < nparts; ++k) s += epart[(size_t)k * b * b + a * b + bb];
        v = -s;
    }
    zp[e] = v;
}

// ---- extract_camera_covariances from a given Z^-1 -------------------------------
template <int P>
__global__ void k_sys_extract(int n, const double* Zi, long long ld, const double* s_a, double* cov, int* warn) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    double out[P * P];
    for (int p = 0; p < P; ++p)
        for (int q = 0; q < P; ++q) {
            const double sp = s_a ? s_a[P * i + p] : 1.0, sq = s_a ? s_a[P * i + q] : 1.0;
            out[P * p + q] = (sp * Zi[(size_t)(P * i + q) * ld + P * i + p]) * sq;
        }
    for (int e = 0; e < P * P; ++e) cov[(size_t)P * P * i + e] = out[e];
    double tr = 0.0;
    for (int p = 0; p < P; ++p) tr += out[P * p + p];
    const double tau = kPsdTol * tr;  // lam_min > -tau  <=>  chol(out + tau I) exists
    double L[P * P];
    bool pd = true;
    for (int c = 0; c < P && pd; ++c) {
        double s = out[P * c + c] + tau;
        for (int kk = 0; kk < c; ++kk) s -= L[P * c + kk] * L[P * c + kk];
        if (!(s > 0.0)) { pd = false; break; }
        const double lcc = sqrt(s);
        L[P * c + c] = lcc;
        for (int r = c + 1; r < P; ++r) {
            double x = 0.5 * (out[P * r + c] + out[P * c + r]);
            for (int kk = 0; kk < c; ++kk) x -= L[P * r + kk] * L[P * c + kk];
            L[P * r + c] = x / lcc;
        }
    }
    if (!pd) atomicAdd(warn, 1);
}

// ---- full_covariance: the scaled bordered Fisher matrix K, dense -----------------
template <int P>
__global__ void k_full_k(int n, int m, int t, const double* D, const double* A, const double* rec, const int* oc,
                         const int* op, const int* pos_cam, const double* H, const double* s_a, const double* s_b,
                         double* K, long long ld) {
    const long long e = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    const long long nD = (long long)P * P * n, nA = 9LL * m, nC = (long long)P * 3 * t;
    const long long rows = (long long)P * n + 3LL * m, nH = rows * 7;
    if (e < nD) {
        const long long i = e / (P * P), pq = e - i * P * P, p = pq / P, q = pq - p * P;
        const long long r = P * i + p, c = P * i + q;
        K[c * ld + r] = (s_a[r] * D[e]) * s_a[c];
    } else if (e < nD + nA) {
        const long long f = e - nD, j = f / 9, pq = f - 9 * j, p = pq / 3, q = pq - 3 * p;
        const long long r = (long long)P * n + 3 * j + p, c = (long long)P * n + 3 * j + q;
        K[c * ld + r] = (s_a[r] * A[f]) * s_a[c];
    } else if (e < nD + nA + nC) {
        const long long f = e - nD - nA, k = f / (P * 3), pq = f - k * P * 3, p = pq / 3, q = pq - 3 * p;
        const double* jc = rec + (size_t)kRec * pos_cam[k];
        const double* jp = jc + 2 * P;
        const double* W = jp + 6;
        const double t0 = jc[p] * W[0] + jc[P + p] * W[2];
        const double t1 = jc[p] * W[1] + jc[P + p] * W[3];
        const double cpl = t0 * jp[q] + t1 * jp[3 + q];
        const long long r = (long long)P * oc[k] + p, c = (long long)P * n + 3LL * op[k] + q;
        const double v = (s_a[r] * cpl) * s_a[c];
        K[c * ld + r] = v;
        K[r * ld + c] = v;
    } else if (e < nD + nA + nC + nH) {
        const long long f = e - nD - nA - nC, r = f / 7, l = f - r * 7;
        const double v = (s_a[r] * H[f]) * s_b[l];
        K[(rows + l) * ld + r] = v;
        K[r * ld + rows + l] = v;
    }
}

// sigma (params x params, ld params) = 0.5 (S_s + S_s^T), S_s = diag(s_a) S diag(s_a)
__global__ void k_full_unscale(long long params, const double* S, long long lds, const double* s_a, double* sigma) {
    const long long e = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (e >= params * params) return;
    const long long r = e % params, c = e / params;
    // rounded products (no contraction into the sum): exact symmetry
    const double a = __dmul_rn(__dmul_rn(s_a[r], S[c * lds + r]), s_a[c]);
    const double b = __dmul_rn(__dmul_rn(s_a[c], S[r * lds + c]), s_a[r]);
    sigma[e] = 0.5 * (a + b);
}

}  // namespace

void launch_nullspace_residual(int P, int t, int n, int m, const int* oc, const int* op, const int* pos_cam,
                               const double* rec, const double* H, int b, unsigned long long* mx, cudaStream_t s) {
    SFM_CUDA(cudaMemsetAsync(mx, 0, 3 * sizeof(unsigned long long), s));
    if (t) {
        if (P == 8) k_nullres_obs<8><<<cdiv(t, 128), 128, 0, s>>>(t, n, oc, op, pos_cam, rec, H, b, mx);
        else k_nullres_obs<9><<<cdiv(t, 128), 128, 0, s>>>(t, n, oc, op, pos_cam, rec, H, b, mx);
        SFM_LAUNCH_CHECK();
    }
    const long long cnt = ((long long)P * n + 3LL * m) * b;
    if (cnt) {
        k_absmax<<<(unsigned)std::min<long long>(1184, cdiv(cnt, 256)), 256, 0, s>>>(H, cnt, mx + 2);
        SFM_LAUNCH_CHECK();
    }
}

void launch_condition_columns(int P, int n, int m, int b, const double* D, const double* A, const double* border,
                              double* s_a, unsigned char* flags, double* part, double* s_b, cudaStream_t s) {
    const long long rows = (long long)P * n + 3LL * m;
    if (rows) {
        if (P == 8) k_cond_sa<8><<<cdiv(rows, 256), 256, 0, s>>>(n, m, D, A, s_a, flags);
        else k_cond_sa<9><<<cdiv(rows, 256), 256, 0, s>>>(n, m, D, A, s_a, flags);
        SFM_LAUNCH_CHECK();
    }
    if (b) {
        const int nb = (int)std::max<long long>(1, cdiv(rows, kRowsPerBlock));
        k_cond_sb_part<<<nb, 64, 0, s>>>(rows, b, s_a, border, part);
        SFM_LAUNCH_CHECK();
        k_cond_sb_final<<<1, 64, 0, s>>>(rows ? nb : 0, b, part, s_b);
        SFM_LAUNCH_CHECK();
    }
}
size_t condition_part_doubles(int P, int n, int m, int b) {
    const long long rows = (long long)P * n + 3LL * m;
    return (size_t)std::max<long long>(1, cdiv(rows, kRowsPerBlock)) * (size_t)std::max(b, 1);
}

void launch_apply_conditioning(int P, int n, int m, int t, int b, double* D, double* A, double* Cp, const int* oc,
                               const int* op, double* border, const double* s_a, const double* s_b, cudaStream_t s) {
    const long long tot = (long long)P * P * n + 9LL * m + (long long)P * 3 * t + ((long long)P * n + 3LL * m) * b;
    if (!tot) return;
    if (P == 8) k_apply_cond<8><<<cdiv(tot, 256), 256, 0, s>>>(n, m, t, b, D, A, Cp, oc, op, border, s_a, s_b);
    else k_apply_cond<9><<<cdiv(tot, 256), 256, 0, s>>>(n, m, t, b, D, A, Cp, oc, op, border, s_a, s_b);
    SFM_LAUNCH_CHECK();
}

void schur_system(const SysSchurArgs& a, cudaStream_t s) {
    const int P = a.P, n = a.n, m = a.m, t = a.t, b = a.b, N = P * n;
    if (m) {
        if (P == 8) k_sys_point<8><<<cdiv(m, 128), 128, 0, s>>>(m, n, a.A, a.border, b, a.Lpt, a.V, a.a_inv, a.st);
        else k_sys_point<9><<<cdiv(m, 128), 128, 0, s>>>(m, n, a.A, a.border, b, a.Lpt, a.V, a.a_inv, a.st);
        SFM_LAUNCH_CHECK();
    }
    if (t) {
        if (P == 8) k_sys_obs<8><<<cdiv(t, 128), 128, 0, s>>>(t, a.ix->idx_cam, a.op, a.Cp, a.Lpt, a.Wb);
        else k_sys_obs<9><<<cdiv(t, 128), 128, 0, s>>>(t, a.ix->idx_cam, a.op, a.Cp, a.Lpt, a.Wb);
        SFM_LAUNCH_CHECK();
    }
    if (N) {
        if (P == 8) k_sys_zinit<8><<<cdiv((long long)N * N, 256), 256, 0, s>>>(n, a.D, a.Z);
        else k_sys_zinit<9><<<cdiv((long long)N * N, 256), 256, 0, s>>>(n, a.D, a.Z);
        SFM_LAUNCH_CHECK();
    }
    launch_pair_reduce(P, *a.pairs, a.Wb, n, a.Z, N, s);
    if (b && N) {
        const long long cnt = (long long)N * b;
        if (P == 8) k_sys_gamma<8><<<cdiv(cnt, 128), 128, 0, s>>>(n, b, a.ix->off_cam, a.ix->idx_cam, a.op, a.Wb, a.V, a.border, a.Gamma);
        else k_sys_gamma<9><<<cdiv(cnt, 128), 128, 0, s>>>(n, b, a.ix->off_cam, a.ix->idx_cam, a.op, a.Wb, a.V, a.border, a.Gamma);
        SFM_LAUNCH_CHECK();
    }
    const int nparts = m ? (int)cdiv(m, kRowsPerBlock) : 0;
    if (b && nparts) {
        k_sys_e_part<<<nparts, std::max(32, ((b * b + 31) / 32) * 32), 0, s>>>(m, b, a.V, a.epart);
        SFM_LAUNCH_CHECK();
    }
    const long long dim = (long long)N + b;
    if (dim) {
        k_sys_assemble<<<cdiv(dim * dim, 256), 256, 0, s>>>(N, b, a.Z, a.Gamma, a.epart, nparts, a.zp);
        SFM_LAUNCH_CHECK();
    }
}
size_t schur_system_epart_doubles(int m, int b) { return (size_t)std::max<long long>(1, cdiv(m, kRowsPerBlock)) * b * b + 1; }

void launch_extract_given(int P, int n, const double* Zi, long long ld, const double* s_a, double* cov, int* warn,
                          cudaStream_t s) {
    SFM_CUDA(cudaMemsetAsync(warn, 0, sizeof(int), s));
    if (!n) return;
    if (P == 8) k_sys_extract<8><<<cdiv(n, 64), 64, 0, s>>>(n, Zi, ld, s_a, cov, warn);
    else k_sys_extract<9><<<cdiv(n, 64), 64, 0, s>>>(n, Zi, ld, s_a, cov, warn);
    SFM_LAUNCH_CHECK();
}

void launch_full_k(int P, int n, int m, int t, const double* D, const double* A, const double* rec, const int* oc,
                   const int* op, const int* pos_cam, const double* H, const double* s_a, const double* s_b, double* K,
                   long long ld, cudaStream_t s) {
    const long long dimK = (long long)P * n + 3LL * m + 7;
    SFM_CUDA(cudaMemsetAsync(K, 0, 8 * (size_t)ld * dimK, s));
    const long long tot = (long long)P * P * n + 9LL * m + (long long)P * 3 * t + ((long long)P * n + 3LL * m) * 7;
    if (!tot) return;
    if (P == 8) k_full_k<8><<<cdiv(tot, 256), 256, 0, s>>>(n, m, t, D, A, rec, oc, op, pos_cam, H, s_a, s_b, K, ld);
    else k_full_k<9><<<cdiv(tot, 256), 256, 0, s>>>(n, m, t, D, A, rec, oc, op, pos_cam, H, s_a, s_b, K, ld);
    SFM_LAUNCH_CHECK();
}

void launch_full_unscale(long long params, const double* S, long long lds, const double* s_a, double* sigma,
                         cudaStream_t s) {
    if (!params) return;
    k_full_unscale<<<cdiv(params * params, 256), 256, 0, s>>>(params, S, lds, s_a, sigma);
    SFM_LAUNCH_CHECK();
}

}  // namespace sfm
