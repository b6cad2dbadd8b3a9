// Iterative refinement of selected camera covariance blocks against the
// exact bordered Fisher system, with double-double residuals.
//
// What is refined: the reference's covariance is the camera block of the
// inverse of the bordered Fisher matrix
//     K = [[M, H], [H^T, 0]],   M = [[D, C], [C^T, A]]
// (src/covariance.cpp:33-82 builds D, A and the couplings C, src/nullspace.cpp
// the gauge basis H; src/covariance.cpp:137-279 reduces and inverts it; the
// Jacobi scaling of src/covariance.cpp:84-135 cancels exactly).  Taking the
// FP64 values of D, A, C and H as exact data (they are bit-identical to the
// CPU restatement's), the camera blocks of K^-1 are a well-defined target.
// For the camera columns e_i of the selected cameras this solves K y = e_i by
//     y_0 = 0,  r_k = e_i - K y_k  (double-double),  y_{k+1} = y_k + K~^-1 r_k
// where K~^-1 is the FP64 solve through the pipeline's own factors (3x3
// point Cholesky factors, W = C_s L^-T, V = L^-1 H_s, L_F, G and X = L^-1 of
// Z_aug).  K~^-1 has relative accuracy ~kappa u, so every step gains ~8
// digits until the double-double residual (~1e-32 relative) limits it: two
// to three steps reach an accuracy far below the 1e-9 parity bar.
//
// Verification only: the product path never calls this; it answers "how far
// is the FP64 pipeline (and the reference's own route) from the exact
// inverse" at sizes where no CPU reference can run (configs 4 and 5).
//
// Vectors are row-major [row][R] (R right-hand sides contiguous), so a warp's
// 32 lanes are 32 right-hand sides of one camera / point and every vector
// access is coalesced.  Compiled with --fmad=false: the couplings are formed
// with the restatement's operation order; double-double products use
// explicit fma().
#include "common.cuh"
#include "detmath.cuh"
#include "kernels.cuh"

#include <algorithm>
#include <cmath>
#include <vector>

namespace sfm {

namespace {

struct dd {
    double hi, lo;
};
__device__ __forceinline__ dd quick_two_sum(double a, double b) {
    const double s = a + b;
    return {s, b - (s - a)};
}
__device__ __forceinline__ dd two_sum(double a, double b) {
    const double s = a + b;
    const double bb = s - a;
    return {s, (a - (s - bb)) + (b - bb)};
}
__device__ __forceinline__ dd dd_add(dd a, dd b) {
    dd s = two_sum(a.hi, b.hi);
    const dd t = two_sum(a.lo, b.lo);
    s.lo += t.hi;
    s = quick_two_sum(s.hi, s.lo);
    s.lo += t.lo;
    return quick_two_sum(s.hi, s.lo);
}
// a += c * y (c exact double, y double-double)
__device__ __forceinline__ void dd_fma(dd& a, double c, dd y) {
    const double p = y.hi * c;
    double e = fma(y.hi, c, -p);
    e = fma(y.lo, c, e);
    a = dd_add(a, quick_two_sum(p, e));
}
__device__ __forceinline__ dd ld_dd(const double* hi, const double* lo, size_t i) { return {hi[i], lo[i]}; }

// H rows of camera i, parameter p (src/nullspace.cpp:14-31 closed form plus
// the solved rotation rows): h[7]
template <int P>
__device__ void cam_h_row(const double* cams, const double* Hr, int i, int p, double* h) {
    for (int l = 0; l < 7; ++l) h[l] = 0.0;
    if (p < 3) {
        for (int b = 0; b < 3; ++b) h[3 + b] = Hr[9 * (size_t)i + 3 * p + b];
    } else if (p < 6) {
        const int a = p - 3;
        const double* C = cams + (size_t)P * i + 3;
        double sx[9];
        skew(C, sx);
        h[a] = 1.0;
        h[3] = sx[3 * a]; h[4] = sx[3 * a + 1]; h[5] = sx[3 * a + 2];
        h[6] = C[a];
    }
}
__device__ void pt_h_row(const double* pts, int j, int q, double* h) {
    const double* X = pts + 3 * (size_t)j;
    double sx[9];
    skew(X, sx);
    for (int l = 0; l < 7; ++l) h[l] = 0.0;
    h[q] = 1.0;
    h[3] = sx[3 * q]; h[4] = sx[3 * q + 1]; h[5] = sx[3 * q + 2];
    h[6] = X[q];
}

// Unscaled couplings C_t = (J_c^T W) J_p at the by-camera slot, in the
// restatement's operation order (no contraction: --fmad=false).
template <int P>
__global__ void k_ref_coupling(const double* rec, int t, double* Cb) {
    const int k = blockIdx.x * blockDim.x + threadIdx.x;
    if (k >= t) return;
    const double* jc = rec + (size_t)kRec * k;
    const double* jp = jc + 2 * P;
    const double* W = jp + 6;
    double* c = Cb + (size_t)27 * k;
    for (int p = 0; p < P; ++p) {
        const double t0 = jc[p] * W[0] + jc[P + p] * W[2];
        const double t1 = jc[p] * W[1] + jc[P + p] * W[3];
        for (int q = 0; q < 3; ++q) c[3 * p + q] = t0 * jp[q] + t1 * jp[3 + q];
    }
}

// ---- residual r = e - K y (double-double) -------------------------------------
// Camera rows: r_c[i] = e - D_i y_c[i] - Σ_{a in cam i} C_a y_p[pt a] - H_ci λ.
// One warp per (camera, 32 columns); lane = column.
template <int P>
__global__ void k_ref_res_cam(int n, int R, const int* off_cam, const int* idx_cam, const int* op, const double* Cb,
                              const double* D, const double* cams, const double* Hr, const int* col_cam,
                              const double* ych, const double* ycl, const double* yph, const double* ypl,
                              const double* ylh, const double* yll, double* rc) {
    const int w = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, lane = threadIdx.x & 31;
    const int chunks = R / 32;
    if (w >= n * chunks) return;
    const int i = w / chunks, col = (w - i * chunks) * 32 + lane;
    dd acc[P];
    const int ccam = col_cam[col];  // camera of this column (-1: padding)
    const int cp = col % P;
#pragma unroll
    for (int p = 0; p < P; ++p) acc[p] = {(ccam == i && cp == p) ? 1.0 : 0.0, 0.0};
    const size_t base_c = (size_t)P * i;
    for (int q = 0; q < P; ++q) {
        const dd y = ld_dd(ych, ycl, (base_c + q) * R + col);
#pragma unroll
        for (int p = 0; p < P; ++p) dd_fma(acc[p], -D[(size_t)P * P * i + P * p + q], y);
    }
    for (int k = off_cam[i]; k < off_cam[i + 1]; ++k) {
        const int j = op[idx_cam[k]];
        const double* c = Cb + (size_t)27 * k;
        const size_t bp = (size_t)3 * j;
        const dd y0 = ld_dd(yph, ypl, (bp + 0) * R + col);
        const dd y1 = ld_dd(yph, ypl, (bp + 1) * R + col);
        const dd y2 = ld_dd(yph, ypl, (bp + 2) * R + col);
#pragma unroll
        for (int p = 0; p < P; ++p) {
            dd_fma(acc[p], -c[3 * p], y0);
            dd_fma(acc[p], -c[3 * p + 1], y1);
            dd_fma(acc[p], -c[3 * p + 2], y2);
        }
    }
    dd lam[7];
#pragma unroll
    for (int l = 0; l < 7; ++l) lam[l] = ld_dd(ylh, yll, (size_t)l * R + col);
#pragma unroll
    for (int p = 0; p < P; ++p) {
        double h[7];
        cam_h_row<P>(cams, Hr, i, p, h);
        for (int l = 0; l < 7; ++l)
            if (h[l] != 0.0) dd_fma(acc[p], -h[l], lam[l]);
        rc[(base_c + p) * R + col] = acc[p].hi + acc[p].lo;
    }
}

// Point rows: r_p[j] = -A_j y_p[j] - Σ_{a in pt j} C_a^T y_c[cam a] - H_pj λ.
template <int P>
__global__ void k_ref_res_pt(int m, int R, const int* off_pt, const int* idx_pt, const int* oc, const int* pos_cam,
                             const double* Cb, const double* A, const double* pts, const double* ych, const double* ycl,
                             const double* yph, const double* ypl, const double* ylh, const double* yll, double* rp) {
    const int w = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, lane = threadIdx.x & 31;
    const int chunks = R / 32;
    if (w >= m * chunks) return;
    const int j = w / chunks, col = (w - j * chunks) * 32 + lane;
    dd acc[3] = {{0.0, 0.0}, {0.0, 0.0}, {0.0, 0.0}};
    const size_t bp = (size_t)3 * j;
    for (int q2 = 0; q2 < 3; ++q2) {
        const dd y = ld_dd(yph, ypl, (bp + q2) * R + col);
        for (int q = 0; q < 3; ++q) dd_fma(acc[q], -A[9 * (size_t)j + 3 * q + q2], y);
    }
    for (int k = off_pt[j]; k < off_pt[j + 1]; ++k) {
        const int tt = idx_pt[k];
        const int i = oc[tt];
        const double* c = Cb + (size_t)27 * pos_cam[tt];
        const size_t bc = (size_t)P * i;
        for (int p = 0; p < P; ++p) {
            const dd y = ld_dd(ych, ycl, (bc + p) * R + col);
            dd_fma(acc[0], -c[3 * p], y);
            dd_fma(acc[1], -c[3 * p + 1], y);
            dd_fma(acc[2], -c[3 * p + 2], y);
        }
    }
    for (int q = 0; q < 3; ++q) {
        double h[7];
        pt_h_row(pts, j, q, h);
        for (int l = 0; l < 7; ++l)
            if (h[l] != 0.0) dd_fma(acc[q], -h[l], ld_dd(ylh, yll, (size_t)l * R + col));
        rp[(bp + q) * R + col] = acc[q].hi + acc[q].lo;
    }
}

// r_λ = -Σ_i H_ci^T y_c[i] - Σ_j H_pj^T y_p[j]: per-chunk partials
// (thread = column, a fixed range of cameras / points), then a fixed-order
// final sum.  Partials are double-double.
constexpr int kLamChunk = 256;
template <int P>
__global__ void k_ref_res_lam_part(int n, int m, int R, const double* cams, const double* Hr, const double* pts,
                                   const double* ych, const double* ycl, const double* yph, const double* ypl,
                                   double* part_hi, double* part_lo) {
    const int col = blockIdx.y * blockDim.x + threadIdx.x;
    if (col >= R) return;
    const int ent0 = blockIdx.x * kLamChunk, ent1 = min(ent0 + kLamChunk, n + m);
    dd acc[7];
    for (int l = 0; l < 7; ++l) acc[l] = {0.0, 0.0};
    for (int g = ent0; g < ent1; ++g) {
        if (g < n) {
            for (int p = 0; p < 6; ++p) {
                double h[7];
                cam_h_row<P>(cams, Hr, g, p, h);
                const dd y = ld_dd(ych, ycl, ((size_t)P * g + p) * R + col);
                for (int l = 0; l < 7; ++l)
                    if (h[l] != 0.0) dd_fma(acc[l], -h[l], y);
            }
        } else {
            const int j = g - n;
            for (int q = 0; q < 3; ++q) {
                double h[7];
                pt_h_row(pts, j, q, h);
                const dd y = ld_dd(yph, ypl, ((size_t)3 * j + q) * R + col);
                for (int l = 0; l < 7; ++l)
                    if (h[l] != 0.0) dd_fma(acc[l], -h[l], y);
            }
        }
    }
    for (int l = 0; l < 7; ++l) {
        part_hi[((size_t)blockIdx.x * 7 + l) * R + col] = acc[l].hi;
        part_lo[((size_t)blockIdx.x * 7 + l) * R + col] = acc[l].lo;
    }
}
__global__ void k_ref_res_lam_final(int nchunk, int R, const double* part_hi, const double* part_lo, double* rl) {
    const int e = blockIdx.x * blockDim.x + threadIdx.x;  // l * R + col
    if (e >= 7 * R) return;
    const int l = e / R, col = e - l * R;
    dd acc = {0.0, 0.0};
    for (int c = 0; c < nchunk; ++c) {
        const size_t o = ((size_t)c * 7 + l) * R + col;
        acc = dd_add(acc, {part_hi[o], part_lo[o]});
    }
    rl[e] = acc.hi + acc.lo;
}

// ---- approximate solve K~^-1 r through the pipeline's factors (FP64) -------------
// u_j = L_j^-1 (s_p ∘ r_p[j])
template <int P>
__global__ void k_ref_u(int m, int n, int R, const double* s_a, const double* Lpt, const double* rp, double* u) {
    const long long e = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (e >= (long long)m * R) return;
    const int j = (int)(e / R), col = (int)(e - (long long)j * R);
    const double* L = Lpt + 8 * (size_t)j;
    const double* sp = s_a + (size_t)P * n + 3 * (size_t)j;
    const size_t b = (size_t)3 * j;
    const double r0 = sp[0] * rp[(b + 0) * R + col], r1 = sp[1] * rp[(b + 1) * R + col], r2 = sp[2] * rp[(b + 2) * R + col];
    const double u0 = r0 / L[0];
    const double u1 = (r1 - L[1] * u0) / L[2];
    const double u2 = (r2 - L[3] * u0 - L[4] * u1) / L[5];
    u[(b + 0) * R + col] = u0;
    u[(b + 1) * R + col] = u1;
    u[(b + 2) * R + col] = u2;
}

// f_i = s_c ∘ r_c[i] - Σ_{slots k of cam i} W_k u[pt k]   -> B rows P i .. P i + P - 1
template <int P>
__global__ void k_ref_f(int n, int R, const int* off_cam, const int* idx_cam, const int* op, const double* s_a,
                        const double* Wb, const double* rc, const double* u, double* B) {
    const int w = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, lane = threadIdx.x & 31;
    const int chunks = R / 32;
    if (w >= n * chunks) return;
    const int i = w / chunks, col = (w - i * chunks) * 32 + lane;
    double acc[P];
    const size_t bc = (size_t)P * i;
#pragma unroll
    for (int p = 0; p < P; ++p) acc[p] = s_a[bc + p] * rc[(bc + p) * R + col];
    for (int k = off_cam[i]; k < off_cam[i + 1]; ++k) {
        const int j = op[idx_cam[k]];
        const double* W = Wb + (size_t)kWStride * k;
        const size_t b = (size_t)3 * j;
        const double u0 = u[b * R + col], u1 = u[(b + 1) * R + col], u2 = u[(b + 2) * R + col];
#pragma unroll
        for (int p = 0; p < P; ++p) acc[p] -= fma(W[3 * p], u0, fma(W[3 * p + 1], u1, W[3 * p + 2] * u2));
    }
#pragma unroll
    for (int p = 0; p < P; ++p) B[(bc + p) * R + col] = acc[p];
}

// g = s_b ∘ r_λ - Σ_j V_j^T u_j: per-chunk partials, then the final kernel
// forms h = L_F^-1 g.
template <int P>
__global__ void k_ref_g_part(int m, int R, const double* V, const double* u, double* part) {
    const int col = blockIdx.y * blockDim.x + threadIdx.x;
    if (col >= R) return;
    const int j0 = blockIdx.x * kLamChunk, j1 = min(j0 + kLamChunk, m);
    double acc[7] = {0, 0, 0, 0, 0, 0, 0};
    for (int j = j0; j < j1; ++j) {
        const size_t b = (size_t)3 * j;
        const double u0 = u[b * R + col], u1 = u[(b + 1) * R + col], u2 = u[(b + 2) * R + col];
        const double* v = V + 21 * (size_t)j;
        for (int l = 0; l < 7; ++l) acc[l] += fma(v[l], u0, fma(v[7 + l], u1, v[14 + l] * u2));
    }
    for (int l = 0; l < 7; ++l) part[((size_t)blockIdx.x * 7 + l) * R + col] = acc[l];
}
__global__ void k_ref_h(int nchunk, int R, const double* part, const double* s_b, const double* rl, const double* LF,
                        double* h) {
    const int col = blockIdx.x * blockDim.x + threadIdx.x;
    if (col >= R) return;
    double g[7];
    for (int l = 0; l < 7; ++l) {
        double s = 0.0;
        for (int c = 0; c < nchunk; ++c) s += part[((size_t)c * 7 + l) * R + col];
        g[l] = s_b[l] * rl[(size_t)l * R + col] - s;
    }
    for (int l = 0; l < 7; ++l) {
        double x = g[l];
        for (int k = 0; k < l; ++k) x -= LF[7 * l + k] * g[k];
        g[l] = x / LF[7 * l + l];
        h[(size_t)l * R + col] = g[l];
    }
}

// B[row] += G[row] h  (rows < N)
__global__ void k_ref_add_gh(int N, int R, const double* G, const double* h, double* B) {
    const long long e = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (e >= (long long)N * R) return;
    const int row = (int)(e / R), col = (int)(e - (long long)row * R);
    double s = 0.0;
    for (int l = 0; l < 7; ++l) s = fma(G[(size_t)row * 7 + l], h[(size_t)l * R + col], s);
    B[e] += s;
}

// Triangular products with X = L^-1 (lower, column-major in the Z buffer):
//   trans = 0: T = X B   (T[r] = Σ_{c <= r} X(r, c) B[c])
//   trans = 1: T = X^T B (T[c] = Σ_{r >= c} X(r, c) B[r])
// 64 x 32 output tiles (rows x columns), 256 threads, 8 outputs each.
constexpr int kTR = 64, kTC = 32, kTK = 32;
__global__ void __launch_bounds__(256) k_ref_trmm(int Npad, int R, const double* X, long long ld, const double* B,
                                                  double* T, int trans) {
    __shared__ double xs[kTK][kTR + 1];  // xs[k][r] = op(X)(r0 + r, k0 + k)
    __shared__ double bs[kTK][kTC];
    const int r0 = blockIdx.x * kTR, c0 = blockIdx.y * kTC;
    const int tid = threadIdx.x;
    const int tr = tid / 8, tc = tid % 8;  // 32 x 8 threads: rows tr, tr + 32; columns tc + 8 v
    double acc[2][4] = {{0, 0, 0, 0}, {0, 0, 0, 0}};
    // K range: trans 0 -> columns 0 .. r0 + 63; trans 1 -> rows r0 .. Npad
    const int kb = trans ? r0 : 0, ke = trans ? Npad : min(Npad, r0 + kTR);
    for (int k0 = kb; k0 < ke; k0 += kTK) {
        for (int e = tid; e < kTK * kTR; e += 256) {
            double v;
            if (!trans) {  // X(r0 + r, k0 + k), column-major: coalesced along r
                const int r = e % kTR, k = e / kTR;
                const int gr = r0 + r, gc = k0 + k;
                v = (gr >= gc) ? X[(size_t)gc * ld + gr] : 0.0;
                xs[k][r] = v;
            } else {  // X^T(r0 + r, k0 + k) = X(k0 + k, r0 + r): coalesced along k
                const int k = e % kTK, r = e / kTK;
                const int gr = k0 + k, gc = r0 + r;
                v = (gr >= gc) ? X[(size_t)gc * ld + gr] : 0.0;
                xs[k][r] = v;
            }
        }
        for (int e = tid; e < kTK * kTC; e += 256) {
            const int k = e / kTC, c = e % kTC;
            bs[k][c] = B[(size_t)(k0 + k) * R + c0 + c];
        }
        __syncthreads();
#pragma unroll 8
        for (int k = 0; k < kTK; ++k) {
            const double a0 = xs[k][tr], a1 = xs[k][tr + 32];
#pragma unroll
            for (int v = 0; v < 4; ++v) {
                const double b = bs[k][tc + 8 * v];
                acc[0][v] = fma(a0, b, acc[0][v]);
                acc[1][v] = fma(a1, b, acc[1][v]);
            }
        }
        __syncthreads();
    }
#pragma unroll
    for (int v = 0; v < 4; ++v) {
        T[(size_t)(r0 + tr) * R + c0 + tc + 8 * v] = acc[0][v];
        T[(size_t)(r0 + tr + 32) * R + c0 + tc + 8 * v] = acc[1][v];
    }
}

// λ_s = -L_F^-T (h - G^T x_c): G^T x_c partials over row chunks, then final.
__global__ void k_ref_gtx_part(int N, int R, const double* G, const double* xc, double* part) {
    const int col = blockIdx.y * blockDim.x + threadIdx.x;
    if (col >= R) return;
    const int r0 = blockIdx.x * kLamChunk, r1 = min(r0 + kLamChunk, N);
    double acc[7] = {0, 0, 0, 0, 0, 0, 0};
    for (int r = r0; r < r1; ++r) {
        const double x = xc[(size_t)r * R + col];
        for (int l = 0; l < 7; ++l) acc[l] = fma(G[(size_t)r * 7 + l], x, acc[l]);
    }
    for (int l = 0; l < 7; ++l) part[((size_t)blockIdx.x * 7 + l) * R + col] = acc[l];
}
__global__ void k_ref_lambda(int nchunk, int R, const double* part, const double* h, const double* LF, double* lam) {
    const int col = blockIdx.x * blockDim.x + threadIdx.x;
    if (col >= R) return;
    double w[7];
    for (int l = 0; l < 7; ++l) {
        double s = 0.0;
        for (int c = 0; c < nchunk; ++c) s += part[((size_t)c * 7 + l) * R + col];
        w[l] = h[(size_t)l * R + col] - s;
    }
    for (int l = 6; l >= 0; --l) {  // L_F^T x = w
        double x = w[l];
        for (int k = l + 1; k < 7; ++k) x -= LF[7 * k + l] * w[k];
        w[l] = x / LF[7 * l + l];
    }
    for (int l = 0; l < 7; ++l) lam[(size_t)l * R + col] = -w[l];
}

// Points: x_p = L^-T (u - Σ_a W_a^T x_c[cam a] - V λ_s), then y_p += s_p ∘ x_p (dd).
template <int P>
__global__ void k_ref_points(int m, int n, int R, const int* off_pt, const int* idx_pt, const int* oc,
                             const int* pos_cam, const double* Wb, const double* Lpt, const double* V,
                             const double* s_a, const double* u, const double* xc, const double* lam, double* yph,
                             double* ypl) {
    const int w = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, lane = threadIdx.x & 31;
    const int chunks = R / 32;
    if (w >= m * chunks) return;
    const int j = w / chunks, col = (w - j * chunks) * 32 + lane;
    const size_t b = (size_t)3 * j;
    double v0 = u[b * R + col], v1 = u[(b + 1) * R + col], v2 = u[(b + 2) * R + col];
    for (int k = off_pt[j]; k < off_pt[j + 1]; ++k) {
        const int tt = idx_pt[k];
        const int i = oc[tt];
        const double* W = Wb + (size_t)kWStride * pos_cam[tt];
        const size_t bc = (size_t)P * i;
        for (int p = 0; p < P; ++p) {
            const double x = xc[(bc + p) * R + col];
            v0 -= W[3 * p] * x;
            v1 -= W[3 * p + 1] * x;
            v2 -= W[3 * p + 2] * x;
        }
    }
    const double* Vj = V + 21 * (size_t)j;
    for (int l = 0; l < 7; ++l) {
        const double lm = lam[(size_t)l * R + col];
        v0 -= Vj[l] * lm;
        v1 -= Vj[7 + l] * lm;
        v2 -= Vj[14 + l] * lm;
    }
    const double* L = Lpt + 8 * (size_t)j;  // L^T x = v
    const double x2 = v2 / L[5];
    const double x1 = (v1 - L[4] * x2) / L[2];
    const double x0 = (v0 - L[1] * x1 - L[3] * x2) / L[0];
    const double* sp = s_a + (size_t)P * n + b;
    const double xs[3] = {x0, x1, x2};
    for (int q = 0; q < 3; ++q) {
        const size_t o = (b + q) * R + col;
        const dd y = dd_add({yph[o], ypl[o]}, {sp[q] * xs[q], 0.0});
        yph[o] = y.hi;
        ypl[o] = y.lo;
    }
}

// y_c += s_a ∘ x_c, y_λ += s_b ∘ λ_s (dd)
__global__ void k_ref_update(int N, int R, const double* s_a, const double* xc, const double* s_b, const double* lam,
                             double* ych, double* ycl, double* ylh, double* yll) {
    const long long e = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    const long long nc = (long long)N * R;
    if (e < nc) {
        const int row = (int)(e / R);
        const dd y = dd_add({ych[e], ycl[e]}, {s_a[row] * xc[e], 0.0});
        ych[e] = y.hi;
        ycl[e] = y.lo;
    } else if (e < nc + 7LL * R) {
        const long long f = e - nc;
        const int l = (int)(f / R);
        const dd y = dd_add({ylh[f], yll[f]}, {s_b[l] * lam[f], 0.0});
        ylh[f] = y.hi;
        yll[f] = y.lo;
    }
}

// camera blocks of the selection: out[c][p][q] = y_c[P cam + p][P c + q] (hi + lo)
__global__ void k_ref_blocks(int P, int R, int nsel, const int* sel, const double* ych, const double* ycl,
                             double* out) {
    const int e = blockIdx.x * blockDim.x + threadIdx.x;
    if (e >= nsel * P * P) return;
    const int c = e / (P * P), pq = e - c * P * P, p = pq / P, q = pq - p * P;
    const size_t o = ((size_t)P * sel[c] + p) * R + (size_t)P * c + q;
    out[e] = ych[o] + ycl[o];
}

template <typename T>
T* carve(DBuf& b, size_t& off, size_t count) {
    T* p = reinterpret_cast<T*>(static_cast<char*>(b.p) + off);
    off += ((sizeof(T) * count + 255) / 256) * 256;
    return p;
}

}  // namespace

size_t refine_bytes(int N, int Npad, int m, int R) {
    const size_t rows_p = (size_t)3 * m;
    size_t b = 0;
    auto add = [&](size_t bytes) { b += ((bytes + 255) / 256) * 256; };
    add(8 * (size_t)N * R * 3);            // rc, ych, ycl
    add(8 * rows_p * R * 4);               // rp, yph, ypl, u
    add(8 * 7 * (size_t)R * 4);            // rl, ylh, yll, h
    add(8 * 7 * (size_t)R);                // lam
    add(8 * (size_t)Npad * R * 2);         // B, T
    const size_t nchunk = (size_t)(std::max(N, m) + kLamChunk) / kLamChunk + ((size_t)N + m) / kLamChunk + 2;
    add(8 * nchunk * 7 * R * 2);           // partials (hi, lo)
    add(4 * (size_t)R);                    // col_cam
    return b;
}

void refine_camera_blocks(const RefineArgs& a, const std::vector<int>& sel, int iters, double* out_blocks,
                          double* history, cudaStream_t s) {
    const int P = a.P, n = a.n, m = a.m, N = P * n, Npad = a.Npad;
    const int nsel = (int)sel.size();
    const int R = ((P * nsel + 31) / 32) * 32;
    size_t off = 0;
    a.scratch->get(refine_bytes(N, Npad, m, R) + 4096);
    DBuf& W = *a.scratch;
    const size_t rows_p = (size_t)3 * m;
    double* rc = carve<double>(W, off, (size_t)N * R);
    double* ych = carve<double>(W, off, (size_t)N * R);
    double* ycl = carve<double>(W, off, (size_t)N * R);
    double* rp = carve<double>(W, off, rows_p * R);
    double* yph = carve<double>(W, off, rows_p * R);
    double* ypl = carve<double>(W, off, rows_p * R);
    double* u = carve<double>(W, off, rows_p * R);
    double* rl = carve<double>(W, off, 7 * (size_t)R);
    double* ylh = carve<double>(W, off, 7 * (size_t)R);
    double* yll = carve<double>(W, off, 7 * (size_t)R);
    double* h = carve<double>(W, off, 7 * (size_t)R);
    double* lam = carve<double>(W, off, 7 * (size_t)R);
    double* B = carve<double>(W, off, (size_t)Npad * R);
    double* T = carve<double>(W, off, (size_t)Npad * R);
    const int nchunk_l = (n + m + kLamChunk - 1) / kLamChunk;
    const int nchunk_g = (std::max(m, 1) + kLamChunk - 1) / kLamChunk;
    const int nchunk_x = (std::max(N, 1) + kLamChunk - 1) / kLamChunk;
    const size_t nchunk = (size_t)std::max(nchunk_l, std::max(nchunk_g, nchunk_x));
    double* part_hi = carve<double>(W, off, nchunk * 7 * R);
    double* part_lo = carve<double>(W, off, nchunk * 7 * R);
    int* col_cam = carve<int>(W, off, R);
    {
        std::vector<int> cc(R, -1);
        for (int c = 0; c < nsel; ++c)
            for (int p = 0; p < P; ++p) cc[(size_t)P * c + p] = sel[c];
        SFM_CUDA(cudaMemcpyAsync(col_cam, cc.data(), 4 * (size_t)R, cudaMemcpyHostToDevice, s));
    }
    for (double* z : {ych, ycl}) SFM_CUDA(cudaMemsetAsync(z, 0, 8 * (size_t)N * R, s));
    for (double* z : {yph, ypl}) SFM_CUDA(cudaMemsetAsync(z, 0, 8 * rows_p * R, s));
    for (double* z : {ylh, yll}) SFM_CUDA(cudaMemsetAsync(z, 0, 8 * 7 * (size_t)R, s));
    SFM_CUDA(cudaMemsetAsync(B, 0, 8 * (size_t)Npad * R, s));  // padding rows stay zero
    double* Cb = a.coupling;
    if (a.t) {
        if (P == 8) k_ref_coupling<8><<<cdiv(a.t, 128), 128, 0, s>>>(a.rec, a.t, Cb);
        else k_ref_coupling<9><<<cdiv(a.t, 128), 128, 0, s>>>(a.rec, a.t, Cb);
        SFM_LAUNCH_CHECK();
    }
    const int chunks = R / 32;
    std::vector<double> prev((size_t)nsel * P * P, 0.0), cur((size_t)nsel * P * P);
    int* dsel_buf = nullptr;
    SFM_CUDA(cudaMallocAsync((void**)&dsel_buf, 4 * (size_t)std::max(nsel, 1), s));
    SFM_CUDA(cudaMemcpyAsync(dsel_buf, sel.data(), 4 * (size_t)nsel, cudaMemcpyHostToDevice, s));
    double* dout = nullptr;
    SFM_CUDA(cudaMallocAsync((void**)&dout, 8 * (size_t)std::max(nsel, 1) * P * P, s));
    for (int it = 0; it < iters; ++it) {
        // residual r = e - K y
        const unsigned wb_c = cdiv((long long)n * chunks * 32, 256), wb_p = cdiv((long long)m * chunks * 32, 256);
        if (n) {
            if (P == 8)
                k_ref_res_cam<8><<<wb_c, 256, 0, s>>>(n, R, a.off_cam, a.idx_cam, a.op, Cb, a.D, a.cams, a.Hr, col_cam,
                                                      ych, ycl, yph, ypl, ylh, yll, rc);
            else
                k_ref_res_cam<9><<<wb_c, 256, 0, s>>>(n, R, a.off_cam, a.idx_cam, a.op, Cb, a.D, a.cams, a.Hr, col_cam,
                                                      ych, ycl, yph, ypl, ylh, yll, rc);
            SFM_LAUNCH_CHECK();
        }
        if (m) {
            if (P == 8)
                k_ref_res_pt<8><<<wb_p, 256, 0, s>>>(m, R, a.off_pt, a.idx_pt, a.oc, a.pos_cam, Cb, a.A, a.pts, ych, ycl,
                                                     yph, ypl, ylh, yll, rp);
            else
                k_ref_res_pt<9><<<wb_p, 256, 0, s>>>(m, R, a.off_pt, a.idx_pt, a.oc, a.pos_cam, Cb, a.A, a.pts, ych, ycl,
                                                     yph, ypl, ylh, yll, rp);
            SFM_LAUNCH_CHECK();
        }
        {
            const dim3 g(nchunk_l, cdiv(R, 128));
            if (P == 8) k_ref_res_lam_part<8><<<g, 128, 0, s>>>(n, m, R, a.cams, a.Hr, a.pts, ych, ycl, yph, ypl, part_hi, part_lo);
            else k_ref_res_lam_part<9><<<g, 128, 0, s>>>(n, m, R, a.cams, a.Hr, a.pts, ych, ycl, yph, ypl, part_hi, part_lo);
            SFM_LAUNCH_CHECK();
            k_ref_res_lam_final<<<cdiv(7 * R, 128), 128, 0, s>>>(nchunk_l, R, part_hi, part_lo, rl);
            SFM_LAUNCH_CHECK();
        }
        // correction through the FP64 factors
        if (m) {
            if (P == 8) k_ref_u<8><<<cdiv((long long)m * R, 256), 256, 0, s>>>(m, n, R, a.s_a, a.Lpt, rp, u);
            else k_ref_u<9><<<cdiv((long long)m * R, 256), 256, 0, s>>>(m, n, R, a.s_a, a.Lpt, rp, u);
            SFM_LAUNCH_CHECK();
        }
        if (n) {
            if (P == 8) k_ref_f<8><<<wb_c, 256, 0, s>>>(n, R, a.off_cam, a.idx_cam, a.op, a.s_a, a.Wb, rc, u, B);
            else k_ref_f<9><<<wb_c, 256, 0, s>>>(n, R, a.off_cam, a.idx_cam, a.op, a.s_a, a.Wb, rc, u, B);
            SFM_LAUNCH_CHECK();
        }
        {
            const dim3 g(nchunk_g, cdiv(R, 128));
            if (P == 8) k_ref_g_part<8><<<g, 128, 0, s>>>(m, R, a.V, u, part_hi);
            else k_ref_g_part<9><<<g, 128, 0, s>>>(m, R, a.V, u, part_hi);
            SFM_LAUNCH_CHECK();
            k_ref_h<<<cdiv(R, 128), 128, 0, s>>>(m ? nchunk_g : 0, R, part_hi, a.s_b, rl, a.LF, h);
            SFM_LAUNCH_CHECK();
        }
        k_ref_add_gh<<<cdiv((long long)N * R, 256), 256, 0, s>>>(N, R, a.G, h, B);
        SFM_LAUNCH_CHECK();
        {
            const dim3 g(Npad / kTR, R / kTC);
            k_ref_trmm<<<g, 256, 0, s>>>(Npad, R, a.X, a.ld, B, T, 0);
            SFM_LAUNCH_CHECK();
            k_ref_trmm<<<g, 256, 0, s>>>(Npad, R, a.X, a.ld, T, B, 1);  // B <- x_c (scaled)
            SFM_LAUNCH_CHECK();
        }
        {
            const dim3 g(nchunk_x, cdiv(R, 128));
            k_ref_gtx_part<<<g, 128, 0, s>>>(N, R, a.G, B, part_hi);
            SFM_LAUNCH_CHECK();
            k_ref_lambda<<<cdiv(R, 128), 128, 0, s>>>(nchunk_x, R, part_hi, h, a.LF, lam);
            SFM_LAUNCH_CHECK();
        }
        if (m) {
            if (P == 8)
                k_ref_points<8><<<wb_p, 256, 0, s>>>(m, n, R, a.off_pt, a.idx_pt, a.oc, a.pos_cam, a.Wb, a.Lpt, a.V, a.s_a,
                                                     u, B, lam, yph, ypl);
            else
                k_ref_points<9><<<wb_p, 256, 0, s>>>(m, n, R, a.off_pt, a.idx_pt, a.oc, a.pos_cam, a.Wb, a.Lpt, a.V, a.s_a,
                                                     u, B, lam, yph, ypl);
            SFM_LAUNCH_CHECK();
        }
        k_ref_update<<<cdiv((long long)N * R + 7LL * R, 256), 256, 0, s>>>(N, R, a.s_a, B, a.s_b, lam, ych, ycl, ylh,
                                                                              yll);
        SFM_LAUNCH_CHECK();
        // B's padding rows were overwritten by the products (X has identity
        // padding): clear them for the next right-hand side
        if (Npad > N) SFM_CUDA(cudaMemsetAsync(B + (size_t)N * R, 0, 8 * (size_t)(Npad - N) * R, s));
        if (nsel) {
            k_ref_blocks<<<cdiv(nsel * P * P, 128), 128, 0, s>>>(P, R, nsel, dsel_buf, ych, ycl, dout);
            SFM_LAUNCH_CHECK();
            SFM_CUDA(cudaMemcpyAsync(cur.data(), dout, 8 * cur.size(), cudaMemcpyDeviceToHost, s));
        }
        SFM_CUDA(cudaStreamSynchronize(s));
        double worst = 0.0;
        for (int c = 0; c < nsel; ++c) {
            double dn = 0.0, yn = 0.0;
            for (int e = 0; e < P * P; ++e) {
                const double d = cur[(size_t)c * P * P + e] - prev[(size_t)c * P * P + e];
                dn += d * d;
                yn += cur[(size_t)c * P * P + e] * cur[(size_t)c * P * P + e];
            }
            worst = std::max(worst, yn > 0 ? std::sqrt(dn / yn) : 0.0);
        }
        if (history) history[it] = worst;
        prev = cur;
    }
    if (nsel) std::copy(cur.begin(), cur.end(), out_blocks);
    SFM_CUDA(cudaFreeAsync(dsel_buf, s));
    SFM_CUDA(cudaFreeAsync(dout, s));
    SFM_CUDA(cudaStreamSynchronize(s));
}

}  // namespace sfm
