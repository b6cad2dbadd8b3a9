// Many small covariance problems in one pipeline run (the sub-reconstruction
// batches of src/subrec.cpp:184-229, 258-297, which the reference runs one
// compute_covariance at a time).
//
// The sub-scenes of a batch are concatenated into one scene whose cameras and
// points are disjoint per sub-scene, gathered on the device from the resident
// full scene by the sub-scenes' camera / point / observation id lists.  The
// single-scene stage-A and Schur kernels then run on it unchanged (everything
// they compute is per observation, per point, per camera or per camera pair,
// and a pair never crosses sub-scenes); what is per sub-scene is the gauge --
// its border scales s_b, F = Σ V^T V, L_F -- and the dense inversion: one
// identity-padded Z per sub-scene (ZMap routes the pair blocks there), each
// factored and inverted by the fused sweep of dense.cu on worker streams.
// Kernels here: the gather, the per-scene gauge reductions, the batched fill
// and the per-scene pivot test.  Orchestration: capi.cu run_batch.
#include "common.cuh"
#include "detmath.cuh"
#include "kernels.cuh"

#include <algorithm>

namespace sfm {

namespace {

__device__ __forceinline__ int upper_scene(const int* off, int B, int idx) {  // off[s] <= idx < off[s+1]
    int lo = 0, hi = B;
    while (hi - lo > 1) {
        const int mid = (lo + hi) >> 1;
        if (off[mid] <= idx) lo = mid;
        else hi = mid;
    }
    return lo;
}
__device__ __forceinline__ int lower_in(const int* a, int n, int key) {
    int lo = 0, hi = n;
    while (lo < hi) {
        const int mid = (lo + hi) >> 1;
        if (a[mid] < key) lo = mid + 1;
        else hi = mid;
    }
    return lo;
}

__global__ void k_batch_scene_of(const int* off, int B, int count, int* out) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i < count) out[i] = upper_scene(off, B, i);
}

// batch observation k <- global observation obs[k] of scene s, renumbered
// into the scene's sorted camera / point lists
__global__ void k_batch_gather_obs(const int* obs, int tb, const int* toff, int B, const int* cams, const int* coff,
                                   const int* pts, const int* poff, const int* oc, const int* op, const double* sigma,
                                   int* oc_b, int* op_b, double* sigma_b) {
    const int k = blockIdx.x * blockDim.x + threadIdx.x;
    if (k >= tb) return;
    const int s = upper_scene(toff, B, k);
    const int t = obs[k];
    const int c0 = coff[s], p0 = poff[s];
    oc_b[k] = c0 + lower_in(cams + c0, coff[s + 1] - c0, oc[t]);
    op_b[k] = p0 + lower_in(pts + p0, poff[s + 1] - p0, op[t]);
    if (sigma)
        for (int e = 0; e < 4; ++e) sigma_b[4 * (size_t)k + e] = sigma[4 * (size_t)t + e];
}

__global__ void k_batch_gather_rows(const int* ids, int count, int width, const double* src, double* dst) {
    const long long e = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (e >= (long long)count * width) return;
    const int i = (int)(e / width), w = (int)(e - (long long)i * width);
    dst[e] = src[(size_t)ids[i] * width + w];
}

// s_b of every scene: one CTA per scene, squares of s_a ∘ h_l over its camera
// rows then its point rows (fixed order), then 1 / norm
template <int P>
__global__ void __launch_bounds__(256) k_batch_border(const int* coff, const int* poff, const double* cams,
                                                      const double* Hr, const double* pts, const double* s_a, int nb,
                                                      double* s_b) {
    __shared__ double red[256][7];
    const int s = blockIdx.x;
    const int c0 = coff[s], c1 = coff[s + 1], p0 = poff[s], p1 = poff[s + 1];
    const int ncam = c1 - c0, total = ncam + (p1 - p0);
    double acc[7] = {0, 0, 0, 0, 0, 0, 0};
    for (int e = threadIdx.x; e < total; e += 256) {
        const bool is_cam = e < ncam;
        const int g = is_cam ? c0 + e : p0 + (e - ncam);
        const double* X = is_cam ? cams + (size_t)P * g + 3 : pts + 3 * (size_t)g;
        const size_t row0 = is_cam ? (size_t)P * g + 3 : (size_t)P * nb + 3 * (size_t)g;
        double sx[9];
        skew(X, sx);
        for (int a = 0; a < 3; ++a) {
            const double sc = s_a[row0 + a];
            double h[7] = {0, 0, 0, 0, 0, 0, 0};
            h[a] = 1.0;
            h[3] = sx[3 * a]; h[4] = sx[3 * a + 1]; h[5] = sx[3 * a + 2];
            h[6] = X[a];
            for (int l = 0; l < 7; ++l) { const double v = sc * h[l]; acc[l] += v * v; }
        }
        if (is_cam)
            for (int a = 0; a < 3; ++a) {
                const double sc = s_a[(size_t)P * g + a];
                for (int b = 0; b < 3; ++b) { const double v = sc * Hr[9 * (size_t)g + 3 * a + b]; acc[3 + b] += v * v; }
            }
    }
    for (int l = 0; l < 7; ++l) red[threadIdx.x][l] = acc[l];
    __syncthreads();
    for (int w = 128; w > 0; w >>= 1) {
        if (threadIdx.x < w)
            for (int l = 0; l < 7; ++l) red[threadIdx.x][l] += red[threadIdx.x + w][l];
        __syncthreads();
    }
    if (threadIdx.x < 7) {
        const double norm = sqrt(red[0][threadIdx.x]);
        s_b[7 * s + threadIdx.x] = norm > 0.0 ? 1.0 / norm : 1.0;
    }
}

// F = Σ_j V_j^T V_j of every scene (28 upper entries), one CTA per scene
__global__ void __launch_bounds__(128) k_batch_F(const int* poff, const double* V, double* F28) {
    __shared__ double red[128][29];
    const int s = blockIdx.x;
    double f[28];
    for (int k = 0; k < 28; ++k) f[k] = 0.0;
    for (int j = poff[s] + threadIdx.x; j < poff[s + 1]; j += 128) {
        const double* v = V + 21 * (size_t)j;
        int k = 0;
        for (int l1 = 0; l1 < 7; ++l1)
            for (int l2 = l1; l2 < 7; ++l2, ++k) f[k] += (v[l1] * v[l2] + v[7 + l1] * v[7 + l2]) + v[14 + l1] * v[14 + l2];
    }
    for (int k = 0; k < 28; ++k) red[threadIdx.x][k] = f[k];
    __syncthreads();
    for (int w = 64; w > 0; w >>= 1) {
        if (threadIdx.x < w)
            for (int k = 0; k < 28; ++k) red[threadIdx.x][k] += red[threadIdx.x + w][k];
        __syncthreads();
    }
    if (threadIdx.x < 28) F28[28 * (size_t)s + threadIdx.x] = red[0][threadIdx.x];
}

// Σ_{a in cam i} W_a V_j(a) per camera, one CTA per camera summing its slots in
// order: unlike k_obs_factor's per-warp partials the grouping does not depend
// on where the camera's slots start in the batch, so identical sub-scenes give
// bitwise identical blocks (the aggregation's trace ties then resolve to the
// earliest subset, as with one sub-scene at a time)
template <int P>
__global__ void __launch_bounds__(64) k_batch_wv(const int* off_cam, const int* idx_cam, const int* op,
                                                 const double* Wb, const double* V, double* sums) {
    const int i = blockIdx.x, tid = threadIdx.x;
    if (tid >= P * 7) return;
    const int p = tid / 7, l = tid - 7 * (tid / 7);
    double acc = 0.0;
    for (int k = off_cam[i]; k < off_cam[i + 1]; ++k) {
        const double* w = Wb + (size_t)kWStride * k;
        const double* v = V + 21 * (size_t)op[idx_cam[k]];
        acc += (w[3 * p] * v[l] + w[3 * p + 1] * v[7 + l]) + w[3 * p + 2] * v[14 + l];
    }
    sums[(size_t)P * 7 * i + tid] = acc;
}

// Z_s (Npad x Npad per scene, lower 64-tiles): [same camera] (s_a D) s_a + Σ_l G G,
// identity on the padding
template <int P>
__global__ void k_batch_fill(double* Zb, int Npad, const int* coff, const double* D, const double* s_a,
                             const double* G) {
    __shared__ double gc[64][8];
    const int s = blockIdx.y;
    const int c0 = coff[s];
    const int N = P * (coff[s + 1] - c0);
    double* Z = Zb + (size_t)s * Npad * Npad;
    const long long l = blockIdx.x;
    int ti = (int)((sqrt(8.0 * (double)l + 1.0) - 1.0) * 0.5);
    while ((long long)(ti + 1) * (ti + 2) / 2 <= l) ++ti;
    while ((long long)ti * (ti + 1) / 2 > l) --ti;
    const int tj = (int)(l - (long long)ti * (ti + 1) / 2);
    const int r0 = ti * 64, cb = tj * 64, tid = threadIdx.x;
    const size_t g0 = (size_t)P * c0;  // the scene's first row in the batch's G / s_a
    for (int e = tid; e < 64 * 7; e += blockDim.x) {
        const int rr = e / 7, ll = e % 7;
        gc[rr][ll] = (cb + rr < N) ? G[(g0 + cb + rr) * 7 + ll] : 0.0;
    }
    __syncthreads();
    const int rr = tid & 63, r = r0 + rr;
    double g[7];
    for (int q = 0; q < 7; ++q) g[q] = (r < N) ? G[(g0 + r) * 7 + q] : 0.0;
    const double sr = (r < N) ? s_a[g0 + r] : 0.0;
    const int ir = r / P;
    for (int cc = tid >> 6; cc < 64; cc += blockDim.x >> 6) {
        const int c = cb + cc;
        double v;
        if (r < N && c < N) {
            v = 0.0;
            const int ic = c / P;
            if (ir == ic) v = (sr * D[(size_t)P * P * (c0 + ir) + P * (r - P * ir) + (c - P * ic)]) * s_a[g0 + c];
            double gg = 0.0;
            for (int q = 0; q < 7; ++q) gg += g[q] * gc[cc][q];
            v += gg;
        } else {
            v = (r == c) ? 1.0 : 0.0;
        }
        Z[(size_t)c * Npad + r] = v;
    }
}

// the invert_schur ratio test per scene: min / max over the scene's Cholesky
// pivots and its 7 border pivots; bad[s] = 1 when min <= 1e-12 max
__global__ void __launch_bounds__(256) k_batch_ratio(const double* piv, int Npad, const int* coff, int P,
                                                     const double* eigE, int* bad) {
    __shared__ double mn[256], mx[256];
    const int s = blockIdx.x;
    const int N = P * (coff[s + 1] - coff[s]);
    double a = INFINITY, b = 0.0;
    for (int i = threadIdx.x; i < N; i += 256) {
        const double v = fabs(piv[(size_t)s * Npad + i]);
        a = fmin(a, v);
        b = fmax(b, v);
    }
    if (threadIdx.x < 7) {
        const double v = fabs(eigE[8 * s + threadIdx.x]);
        a = fmin(a, v);
        b = fmax(b, v);
    }
    mn[threadIdx.x] = a;
    mx[threadIdx.x] = b;
    __syncthreads();
    for (int w = 128; w > 0; w >>= 1) {
        if (threadIdx.x < w) {
            mn[threadIdx.x] = fmin(mn[threadIdx.x], mn[threadIdx.x + w]);
            mx[threadIdx.x] = fmax(mx[threadIdx.x], mx[threadIdx.x + w]);
        }
        __syncthreads();
    }
    if (threadIdx.x == 0) bad[s] = (mn[0] > kPivotRtol * mx[0]) ? 0 : 1;
}

}  // namespace

void launch_batch_scene_of(const int* off, int B, int count, int* out, cudaStream_t s) {
    if (count <= 0) return;
    k_batch_scene_of<<<cdiv(count, 256), 256, 0, s>>>(off, B, count, out);
    SFM_LAUNCH_CHECK();
}

void launch_batch_gather(const BatchLists& L, int P, const double* cams_full, const double* pts_full, const int* oc,
                         const int* op, const double* sigma, double* cams_b, double* pts_b, int* oc_b, int* op_b,
                         double* sigma_b, cudaStream_t s) {
    if (L.nb) {
        k_batch_gather_rows<<<cdiv((long long)L.nb * P, 256), 256, 0, s>>>(L.cams, L.nb, P, cams_full, cams_b);
        SFM_LAUNCH_CHECK();
    }
    if (L.mb) {
        k_batch_gather_rows<<<cdiv((long long)L.mb * 3, 256), 256, 0, s>>>(L.pts, L.mb, 3, pts_full, pts_b);
        SFM_LAUNCH_CHECK();
    }
    if (L.tb) {
        k_batch_gather_obs<<<cdiv(L.tb, 256), 256, 0, s>>>(L.obs, L.tb, L.toff, L.B, L.cams, L.coff, L.pts, L.poff, oc,
                                                           op, sigma, oc_b, op_b, sigma_b);
        SFM_LAUNCH_CHECK();
    }
}

void launch_batch_border(int P, const BatchLists& L, const double* cams_b, const double* Hr, const double* pts_b,
                         const double* s_a, double* s_b, cudaStream_t s) {
    if (!L.B) return;
    if (P == 8) k_batch_border<8><<<L.B, 256, 0, s>>>(L.coff, L.poff, cams_b, Hr, pts_b, s_a, L.nb, s_b);
    else k_batch_border<9><<<L.B, 256, 0, s>>>(L.coff, L.poff, cams_b, Hr, pts_b, s_a, L.nb, s_b);
    SFM_LAUNCH_CHECK();
}

void launch_batch_F(const BatchLists& L, const double* V, double* F28, cudaStream_t s) {
    if (!L.B) return;
    k_batch_F<<<L.B, 128, 0, s>>>(L.poff, V, F28);
    SFM_LAUNCH_CHECK();
}

void launch_batch_wv(int P, int nb, const int* off_cam, const int* idx_cam, const int* op, const double* Wb,
                     const double* V, double* sums, cudaStream_t s) {
    if (!nb) return;
    if (P == 8) k_batch_wv<8><<<nb, 64, 0, s>>>(off_cam, idx_cam, op, Wb, V, sums);
    else k_batch_wv<9><<<nb, 64, 0, s>>>(off_cam, idx_cam, op, Wb, V, sums);
    SFM_LAUNCH_CHECK();
}

void launch_batch_fill(int P, const BatchLists& L, double* Zb, int Npad, const double* D, const double* s_a,
                       const double* G, cudaStream_t s) {
    if (!L.B) return;
    const long long T = Npad / 64, tiles = T * (T + 1) / 2;
    const dim3 grid((unsigned)tiles, L.B);
    if (P == 8) k_batch_fill<8><<<grid, 256, 0, s>>>(Zb, Npad, L.coff, D, s_a, G);
    else k_batch_fill<9><<<grid, 256, 0, s>>>(Zb, Npad, L.coff, D, s_a, G);
    SFM_LAUNCH_CHECK();
}

void launch_batch_ratio(const BatchLists& L, const double* piv, int Npad, int P, const double* eigE, int* bad,
                        cudaStream_t s) {
    if (!L.B) return;
    k_batch_ratio<<<L.B, 256, 0, s>>>(piv, Npad, L.coff, P, eigE, bad);
    SFM_LAUNCH_CHECK();
}

}  // namespace sfm
