// Optional outputs of compute_covariance (CovarianceOptions::point_covariances
// and camera_cross_covariances; reference src/covariance.cpp:283-348).
//
// With X = L^-1 from the sweep (Z_aug = L L^T), the camera block of the
// bordered inverse is Zi = Z_aug^-1 = X^T X (one K-major GEMM over the lower
// tiles, K from the row tile on: "LAUUM").  The other blocks of the bordered
// inverse M^-1, M = [[Z, Γ], [Γ^T, E]], E = -F = -L_F L_F^T, G = Γ L_F^-T:
//     (M^-1)_12 = Zi G L_F^-1                  (N x 7)
//     (M^-1)_22 = L_F^-T (G^T Zi G - I) L_F^-1 (7 x 7)
// A point's covariance (the reference's S (A^-1 + W Z_sub W^T) S with
// W = A^-1 [C_a^T .. | H_pj]) becomes, with A = L L^T, Wb_a = C_a L^-T and
// V = L^-1 H_pj (both from the Schur stage),
//     Σ_X = S L^-T (I + Q) L^-1 S,
//     Q = Σ_ab Wb_a^T Zi_ab Wb_b + Σ_a (Wb_a^T Y_a V^T + transpose) + V Eb V^T.

#include "common.cuh"
#include "kernels.cuh"

namespace sfm {

// Zi(c, r) := Zi(r, c) for r > c (lower -> upper), 32 x 32 tiles via smem.
__global__ void k_mirror_lower(double* Z, long long ld, int N) {
    __shared__ double t[32][33];
    const int bi = blockIdx.y, bj = blockIdx.x;  // source tile: rows bi, cols bj, bi >= bj
    if (bi < bj) return;
    const int tx = threadIdx.x, ty = threadIdx.y;  // 32 x 8
    for (int k = ty; k < 32; k += 8) {
        const int r = bi * 32 + tx, c = bj * 32 + k;
        t[k][tx] = (r < N && c < N) ? Z[(size_t)c * ld + r] : 0.0;
    }
    __syncthreads();
    for (int k = ty; k < 32; k += 8) {
        const int r = bj * 32 + tx, c = bi * 32 + k;  // destination (r, c) = source (c, r)
        if (r < N && c < N && c > r) Z[(size_t)c * ld + r] = t[tx][k];
    }
}

// T = Zi G (N x 7), Zi full symmetric: per (row block, column chunk) partial
// sums, then the chunks in fixed order.
constexpr int kSymvChunk = 256;
__global__ void k_symv7_partial(const double* Z, long long ld, int N, const double* G, double* part) {
    const int r = blockIdx.x * blockDim.x + threadIdx.x;
    const int c0 = blockIdx.y * kSymvChunk, c1 = min(N, c0 + kSymvChunk);
    if (r >= N) return;
    double acc[7] = {0, 0, 0, 0, 0, 0, 0};
    for (int c = c0; c < c1; ++c) {
        const double z = Z[(size_t)c * ld + r];
#pragma unroll
        for (int l = 0; l < 7; ++l) acc[l] += z * __ldg(G + (size_t)c * 7 + l);
    }
    double* o = part + ((size_t)blockIdx.y * N + r) * 7;
#pragma unroll
    for (int l = 0; l < 7; ++l) o[l] = acc[l];
}

// Y = T L_F^-1 per row; partial G^T T per block (fixed-order tree).
__global__ void __launch_bounds__(64) k_border_rows(const double* part, int nchunks, int N, const double* G,
                                                    const double* LF, double* Y, double* gtt_part) {
    __shared__ double red[64][49];
    const int r = blockIdx.x * blockDim.x + threadIdx.x;
    double t[7] = {0, 0, 0, 0, 0, 0, 0};
    double loc[49];
#pragma unroll
    for (int k = 0; k < 49; ++k) loc[k] = 0.0;
    if (r < N) {
        for (int ch = 0; ch < nchunks; ++ch)
#pragma unroll
            for (int l = 0; l < 7; ++l) t[l] += part[((size_t)ch * N + r) * 7 + l];
        // y L_F = t  (backward substitution, L_F lower row-major)
        double y[7];
        for (int l = 6; l >= 0; --l) {
            double v = t[l];
            for (int k = l + 1; k < 7; ++k) v -= y[k] * LF[7 * k + l];
            y[l] = v / LF[7 * l + l];
        }
#pragma unroll
        for (int l = 0; l < 7; ++l) Y[(size_t)r * 7 + l] = y[l];
#pragma unroll
        for (int a = 0; a < 7; ++a)
#pragma unroll
            for (int b = 0; b < 7; ++b) loc[7 * a + b] = G[(size_t)r * 7 + a] * t[b];
    }
    for (int k = 0; k < 49; ++k) red[threadIdx.x][k] = loc[k];
    __syncthreads();
    for (int w = 32; w > 0; w >>= 1) {
        if (threadIdx.x < w)
            for (int k = 0; k < 49; ++k) red[threadIdx.x][k] += red[threadIdx.x + w][k];
        __syncthreads();
    }
    if (threadIdx.x < 49) gtt_part[(size_t)blockIdx.x * 49 + threadIdx.x] = red[0][threadIdx.x];
}

// Eb = L_F^-T (G^T T - I) L_F^-1 (single thread; 7 x 7).
__global__ void k_border_corner(const double* gtt_part, int nblocks, const double* LF, double* Eb) {
    if (threadIdx.x || blockIdx.x) return;
    double M[49];
    for (int k = 0; k < 49; ++k) M[k] = 0.0;
    for (int b = 0; b < nblocks; ++b)
        for (int k = 0; k < 49; ++k) M[k] += gtt_part[(size_t)b * 49 + k];
    for (int l = 0; l < 7; ++l) M[8 * l] -= 1.0;
    // Li = L_F^-1 (lower)
    double Li[49];
    for (int k = 0; k < 49; ++k) Li[k] = 0.0;
    for (int c = 0; c < 7; ++c) {
        Li[7 * c + c] = 1.0 / LF[7 * c + c];
        for (int r = c + 1; r < 7; ++r) {
            double v = 0.0;
            for (int k = c; k < r; ++k) v += LF[7 * r + k] * Li[7 * k + c];
            Li[7 * r + c] = -v / LF[7 * r + r];
        }
    }
    // Eb = Li^T M Li
    double ML[49];
    for (int a = 0; a < 7; ++a)
        for (int b = 0; b < 7; ++b) {
            double v = 0.0;
            for (int k = 0; k < 7; ++k) v += M[7 * a + k] * Li[7 * k + b];
            ML[7 * a + b] = v;
        }
    for (int a = 0; a < 7; ++a)
        for (int b = 0; b < 7; ++b) {
            double v = 0.0;
            for (int k = 0; k < 7; ++k) v += Li[7 * k + a] * ML[7 * k + b];
            Eb[7 * a + b] = v;
        }
}

// One thread per point.
template <int P>
__global__ void __launch_bounds__(128) k_point_cov(int m, int n, const int* off_pt, const int* idx_pt, const int* oc,
                                                   const int* pos_cam, const double* Lpt, const double* V,
                                                   const double* Wb, const double* Zi, long long ld, const double* Y,
                                                   const double* Eb, const double* s_a, double* out) {
    const int j = blockIdx.x * blockDim.x + threadIdx.x;
    if (j >= m) return;
    double Q[9] = {0, 0, 0, 0, 0, 0, 0, 0, 0};
    double v[21];
#pragma unroll
    for (int k = 0; k < 21; ++k) v[k] = V[21 * (size_t)j + k];
    const int b0 = off_pt[j], b1 = off_pt[j + 1];
    for (int ia = b0; ia < b1; ++ia) {
        const int ta = idx_pt[ia];
        const int ca = oc[ta];
        const double* wa = Wb + (size_t)pos_cam[ta] * kWStride;  // P x 3
        double acc[P * 3];  // Σ_b Zi_(ca, cb) Wb_b  (P x 3)
#pragma unroll
        for (int k = 0; k < P * 3; ++k) acc[k] = 0.0;
        for (int ib = b0; ib < b1; ++ib) {
            const int tb = idx_pt[ib];
            const int cb = oc[tb];
            const double* wb = Wb + (size_t)pos_cam[tb] * kWStride;
            double w[P * 3];
#pragma unroll
            for (int k = 0; k < P * 3; ++k) w[k] = __ldg(wb + k);
            const double* zc = Zi + (size_t)P * cb * ld + (size_t)P * ca;  // (P ca + p, P cb + q)
#pragma unroll
            for (int q = 0; q < P; ++q) {
#pragma unroll
                for (int p = 0; p < P; ++p) {
                    const double z = __ldg(zc + (size_t)q * ld + p);
#pragma unroll
                    for (int s = 0; s < 3; ++s) acc[3 * p + s] += z * w[3 * q + s];
                }
            }
        }
        // Q += Wb_a^T acc ; cross term with the border: u = Wb_a^T Y_ca (3 x 7)
        double u[21];
#pragma unroll
        for (int k = 0; k < 21; ++k) u[k] = 0.0;
        const double* ya = Y + (size_t)P * ca * 7;
#pragma unroll
        for (int p = 0; p < P; ++p) {
            const double a0 = __ldg(wa + 3 * p), a1 = __ldg(wa + 3 * p + 1), a2 = __ldg(wa + 3 * p + 2);
#pragma unroll
            for (int s = 0; s < 3; ++s) {
                Q[s] += a0 * acc[3 * p + s];
                Q[3 + s] += a1 * acc[3 * p + s];
                Q[6 + s] += a2 * acc[3 * p + s];
            }
#pragma unroll
            for (int l = 0; l < 7; ++l) {
                const double yv = __ldg(ya + 7 * p + l);
                u[l] += a0 * yv;
                u[7 + l] += a1 * yv;
                u[14 + l] += a2 * yv;
            }
        }
        // Q += u V^T + (u V^T)^T
#pragma unroll
        for (int r = 0; r < 3; ++r)
#pragma unroll
            for (int s = 0; s < 3; ++s) {
                double x = 0.0, y = 0.0;
#pragma unroll
                for (int l = 0; l < 7; ++l) {
                    x += u[7 * r + l] * v[7 * s + l];
                    y += u[7 * s + l] * v[7 * r + l];
                }
                Q[3 * r + s] += x + y;
            }
    }
    // Q += V Eb V^T
    double ve[21];
#pragma unroll
    for (int r = 0; r < 3; ++r)
#pragma unroll
        for (int l = 0; l < 7; ++l) {
            double x = 0.0;
#pragma unroll
            for (int k = 0; k < 7; ++k) x += v[7 * r + k] * __ldg(Eb + 7 * k + l);
            ve[7 * r + l] = x;
        }
#pragma unroll
    for (int r = 0; r < 3; ++r)
#pragma unroll
        for (int s = 0; s < 3; ++s) {
            double x = 0.0;
#pragma unroll
            for (int l = 0; l < 7; ++l) x += ve[7 * r + l] * v[7 * s + l];
            Q[3 * r + s] += x;
        }
    // Σ = S Li^T (I + Q) Li S, Li = L^-1
    const double* L = Lpt + 8 * (size_t)j;
    const double l00 = L[0], l10 = L[1], l11 = L[2], l20 = L[3], l21 = L[4], l22 = L[5];
    double Li[9] = {0, 0, 0, 0, 0, 0, 0, 0, 0};
    Li[0] = 1.0 / l00;
    Li[4] = 1.0 / l11;
    Li[8] = 1.0 / l22;
    Li[3] = -(l10 * Li[0]) / l11;
    Li[7] = -(l21 * Li[4]) / l22;
    Li[6] = -(l20 * Li[0] + l21 * Li[3]) / l22;
    double Mq[9];
#pragma unroll
    for (int k = 0; k < 9; ++k) Mq[k] = Q[k] + ((k % 4) == 0 ? 1.0 : 0.0);
    double ML[9], R[9];
#pragma unroll
    for (int a = 0; a < 3; ++a)
#pragma unroll
        for (int b = 0; b < 3; ++b) ML[3 * a + b] = (Mq[3 * a] * Li[b] + Mq[3 * a + 1] * Li[3 + b]) + Mq[3 * a + 2] * Li[6 + b];
#pragma unroll
    for (int a = 0; a < 3; ++a)
#pragma unroll
        for (int b = 0; b < 3; ++b) R[3 * a + b] = (Li[a] * ML[b] + Li[3 + a] * ML[3 + b]) + Li[6 + a] * ML[6 + b];
    const double* sp = s_a + (size_t)P * n + 3 * (size_t)j;
#pragma unroll
    for (int a = 0; a < 3; ++a)
#pragma unroll
        for (int b = 0; b < 3; ++b) out[9 * (size_t)j + 3 * a + b] = (sp[a] * R[3 * a + b]) * sp[b];
}

// Camera blocks from the full Zi (unscaled): cov_i = S_i Zi_ii S_i + PSD test.
template <int P>
__global__ void k_extract_from_full(const double* Zi, long long ld, int n, const double* s_a, double* cov, int* psd_warn) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    double out[P * P];
    for (int p = 0; p < P; ++p)
        for (int q = 0; q < P; ++q)
            out[P * p + q] = (s_a[P * i + p] * Zi[(size_t)(P * i + q) * ld + P * i + p]) * s_a[P * i + q];
    for (int k = 0; k < P * P; ++k) cov[(size_t)P * P * i + k] = out[k];
    double tr = 0.0;
    for (int p = 0; p < P; ++p) tr += out[P * p + p];
    const double tau = 1e-9 * tr;
    double L[P * P];
    bool pd = true;
    for (int c = 0; c < P && pd; ++c) {
        double sd = out[P * c + c] + tau;
        for (int k = 0; k < c; ++k) sd -= L[P * c + k] * L[P * c + k];
        if (!(sd > 0.0)) { pd = false; break; }
        const double lcc = sqrt(sd);
        L[P * c + c] = lcc;
        for (int r = c + 1; r < P; ++r) {
            double x = 0.5 * (out[P * r + c] + out[P * c + r]);
            for (int k = 0; k < c; ++k) x -= L[P * r + k] * L[P * c + k];
            L[P * r + c] = x / lcc;
        }
    }
    if (!pd) atomicAdd(psd_warn, 1);
}

// Zi(r, c) := (s_r Zi(r, c)) s_c on the N x N camera part (the camera matrix).
__global__ void k_scale_sym(double* Z, long long ld, int N, const double* s_a) {
    const long long e = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (e >= (long long)N * N) return;
    const int r = (int)(e % N), c = (int)(e / N);
    double* z = Z + (size_t)c * ld + r;
    *z = (s_a[r] * *z) * s_a[c];
}

// ---- driver -------------------------------------------------------------------------
void full_covariance(const FullCovArgs& a, cudaStream_t s) {
    const int N = a.P * a.n;
    const long long ld = a.Npad;
    const int K = a.Npad / kNB;
    // Zi = X^T X on the lower tiles
    GemmArgs g = gemm_args(a.Zi, ld, a.X, ld, a.X, ld, K, K, a.Npad);
    g.tri = 1; g.a_kmajor = 1; g.b_kmajor = 1; g.k_from_row = 1;
    launch_gemm(g, s);
    const int nb32 = (a.Npad + 31) / 32;
    k_mirror_lower<<<dim3(nb32, nb32), dim3(32, 8), 0, s>>>(a.Zi, ld, a.Npad);
    SFM_LAUNCH_CHECK();
    if (a.point_cov && a.m) {
        const int nch = (N + kSymvChunk - 1) / kSymvChunk;
        k_symv7_partial<<<dim3(cdiv(N, 128), nch), 128, 0, s>>>(a.Zi, ld, N, a.G, a.part);
        SFM_LAUNCH_CHECK();
        const int rb = (int)cdiv(N, 64);
        k_border_rows<<<rb, 64, 0, s>>>(a.part, nch, N, a.G, a.LF, a.Y, a.gtt_part);
        SFM_LAUNCH_CHECK();
        k_border_corner<<<1, 32, 0, s>>>(a.gtt_part, rb, a.LF, a.Eb);
        SFM_LAUNCH_CHECK();
        if (a.P == 8)
            k_point_cov<8><<<cdiv(a.m, 128), 128, 0, s>>>(a.m, a.n, a.off_pt, a.idx_pt, a.oc, a.pos_cam, a.Lpt, a.V, a.Wb,
                                                          a.Zi, ld, a.Y, a.Eb, a.s_a, a.point_cov);
        else
            k_point_cov<9><<<cdiv(a.m, 128), 128, 0, s>>>(a.m, a.n, a.off_pt, a.idx_pt, a.oc, a.pos_cam, a.Lpt, a.V, a.Wb,
                                                          a.Zi, ld, a.Y, a.Eb, a.s_a, a.point_cov);
        SFM_LAUNCH_CHECK();
    }
    if (a.cross) {
        if (a.P == 8) k_extract_from_full<8><<<cdiv(a.n, 64), 64, 0, s>>>(a.Zi, ld, a.n, a.s_a, a.cam_cov, a.psd);
        else k_extract_from_full<9><<<cdiv(a.n, 64), 64, 0, s>>>(a.Zi, ld, a.n, a.s_a, a.cam_cov, a.psd);
        SFM_LAUNCH_CHECK();
        const long long tot = (long long)N * N;
        if (tot) k_scale_sym<<<cdiv(tot, 256), 256, 0, s>>>(a.Zi, ld, N, a.s_a);
        SFM_LAUNCH_CHECK();
    }
}

size_t full_cov_part_doubles(int N) { return (size_t)((N + kSymvChunk - 1) / kSymvChunk) * N * 7 + 16; }

}  // namespace sfm
