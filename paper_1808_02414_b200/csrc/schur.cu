// Stage (b): point-block Schur reduction into the gauge-augmented dense
// camera matrix, without global atomics in the accumulation.
//
// Reference: schur_reduce, src/covariance.cpp:137-194 (serial point loop
// accumulating C_a A_j^-1 C_b^T into camera-pair blocks, border rows
// C_a A_j^-1 H_pj and corner H_pj^T A_j^-1 H_pj), with the conditioning of
// src/covariance.cpp:84-135 applied on the fly.
//
// B200 formulation (all in conditioned coordinates):
//   A_s,j = L_j L_j^T                       (3x3 Cholesky per point)
//   W_a   = C_s,a L_j^-T                    (P x 3 per observation)
//   V_j   = L_j^-1 H_s,pj                   (3 x 7 per point)
//   Z     = D_s - Σ_pairs W_b W_a^T         (camera-pair blocks)
//   Γ_i   = H_s,ci - Σ_{a in cam i} W_a V_j (P x 7 per camera)
//   F     = Σ_j V_j^T V_j = -E              (7 x 7, SPD)
//   G     = Γ L_F^-T,  Z_aug = Z + G G^T = Z - Γ E^-1 Γ^T
// Z_aug is SPD and its inverse is the camera block of the inverse of the
// bordered matrix [[Z, Γ], [Γ^T, E]], so the dense
// stage is a plain Cholesky.
//
// Pair accumulation: observation pairs (a, b) of each point are keyed by
// camera-pair block (lo * n + hi), stably radix-sorted, and each block is
// reduced by one warp with register accumulators — one write per nonzero
// block, deterministic order, no atomics.
#include "common.cuh"
#include "detmath.cuh"
#include "kernels.cuh"

#include <cub/cub.cuh>
#include <cstdlib>
#include <string>

namespace sfm {

// ---- per-point preparation (thread per point) -----------------------------------
// A_s = S A S, the reference's singularity test on it (covariance.cpp:147-151),
// L_j = chol(A_s) (stored as l00 l10 l11 l20 l21 l22), V_j = L_j^-1 H_s,pj and
// the block-partial of F = Σ V_j^T V_j (fixed-order tree).
template <int P>
__global__ void __launch_bounds__(128) k_point_prep(const double* A, const double* s_a, const double* pts,
                                                    const double* s_b, int m, int n, double* Lpt, double* V,
                                                    double* Fpart, Status* st, const int* scene_of_pt) {
    __shared__ double red[128][29];
    const int j = blockIdx.x * blockDim.x + threadIdx.x;
    if (scene_of_pt && j < m) s_b += 7 * scene_of_pt[j];  // batched sub-scenes: the point's own scales
    double f[28];
#pragma unroll
    for (int k = 0; k < 28; ++k) f[k] = 0.0;
    if (j < m) {
        const double* sp = s_a + (size_t)P * n + 3 * (size_t)j;
        double as[9];
        for (int p = 0; p < 3; ++p)
            for (int q = 0; q < 3; ++q) as[3 * p + q] = (sp[p] * A[9 * (size_t)j + 3 * p + q]) * sp[q];
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
        lo[0] = l00; lo[1] = l10; lo[2] = l11; lo[3] = l20; lo[4] = l21; lo[5] = l22;
        lo[6] = good ? 1.0 : 0.0;
        lo[7] = 0.0;
        // H_s rows of the point: (s_p[q] * [e_q | [X]x row q | X_q]) * s_b
        const double* X = pts + 3 * (size_t)j;
        double sx[9];
        skew(X, sx);
        double hs[3][7];
        for (int q = 0; q < 3; ++q) {
            double h[7] = {0, 0, 0, 0, 0, 0, 0};
            h[q] = 1.0;
            h[3] = sx[3 * q]; h[4] = sx[3 * q + 1]; h[5] = sx[3 * q + 2];
            h[6] = X[q];
            for (int l = 0; l < 7; ++l) hs[q][l] = (sp[q] * h[l]) * s_b[l];
        }
        double v[3][7];
        for (int l = 0; l < 7; ++l) {
            v[0][l] = hs[0][l] / l00;
            v[1][l] = (hs[1][l] - l10 * v[0][l]) / l11;
            v[2][l] = (hs[2][l] - l20 * v[0][l] - l21 * v[1][l]) / l22;
        }
        double* vo = V + 21 * (size_t)j;
        for (int q = 0; q < 3; ++q)
            for (int l = 0; l < 7; ++l) vo[7 * q + l] = good ? v[q][l] : 0.0;
        if (good) {
            int k = 0;
            for (int l1 = 0; l1 < 7; ++l1)
                for (int l2 = l1; l2 < 7; ++l2, ++k)
                    f[k] = (v[0][l1] * v[0][l2] + v[1][l1] * v[1][l2]) + v[2][l1] * v[2][l2];
        }
    }
    for (int k = 0; k < 28; ++k) red[threadIdx.x][k] = f[k];
    __syncthreads();
    for (int w = blockDim.x / 2; w > 0; w >>= 1) {
        if (threadIdx.x < w)
            for (int k = 0; k < 28; ++k) red[threadIdx.x][k] += red[threadIdx.x + w][k];
        __syncthreads();
    }
    if (threadIdx.x < 28) Fpart[28 * (size_t)blockIdx.x + threadIdx.x] = red[0][threadIdx.x];
}

// W_a = C_s,a L_j^-T (P x 3) per observation, one thread per by-camera slot.
// The CTA's records and factors are contiguous: both move through shared
// memory (odd pitch) with coalesced 16-byte loads and stores.
//
// Fused with the camera border sums Σ_{a in cam i} W_a V_j(a): each warp (32
// consecutive slots, so one or a few cameras) reduces W_a V_j per camera
// segment with a shuffle tree; the segment of the warp's first camera goes to
// Pfirst[warp], that of its last camera to Plast[warp], and a camera lying
// wholly inside the warp straight to Gsum[camera].  k_camera_border then adds
// a camera's warp partials in warp order (deterministic), so the factors are
// not read back from HBM for the border.
template <int P>
__global__ void __launch_bounds__(128, 5) k_obs_factor(const int* oc, const int* op, const int* idx_cam, const double* rec,
                                                    const double* s_a, const double* Lpt, const double* V, int t_count,
                                                    int n, double* Wb, double* Pfirst, double* Plast, double* Gsum) {
    constexpr int NE = P * 7;
    constexpr int PITCH = kWStride + 1;  // odd: conflict-free per-thread rows
    static_assert(PITCH % 2 == 1 && PITCH >= kWStride, "staging pitch");
    __shared__ double buf[128 * PITCH];
    const int k0 = blockIdx.x * blockDim.x;
    const int nv = min(128, t_count - k0);
    {
        const double2* in = reinterpret_cast<const double2*>(rec + (size_t)k0 * kRec);
        constexpr int NP = (Layout<P>::WO + 4 + 1) / 2;  // double2 parts of the record that are used
        // all NP loads of a thread in flight before the first shared store
        // (a load -> store loop serialises the HBM latency per iteration)
        double2 v[NP];
#pragma unroll
        for (int u = 0; u < NP; ++u) {
            const int w = threadIdx.x + 128 * u;
            const int o = w / NP, part = w - o * NP;
            if (w < nv * NP) v[u] = __ldcs(in + (size_t)o * (kRec / 2) + part);
        }
#pragma unroll
        for (int u = 0; u < NP; ++u) {
            const int w = threadIdx.x + 128 * u;
            const int o = w / NP, part = w - o * NP;
            if (w < nv * NP) {
                buf[o * PITCH + 2 * part] = v[u].x;
                buf[o * PITCH + 2 * part + 1] = v[u].y;
            }
        }
    }
    __syncthreads();
    const int k = k0 + threadIdx.x;
    double wo[kWStride];
    int ci = -1, pj = 0;
    if (k < t_count) {
        const int t = idx_cam[k];
        ci = oc[t];
        pj = op[t];
        const double* rr = buf + threadIdx.x * PITCH;
        const double* jc = rr + Layout<P>::JC;
        const double* jp = rr + Layout<P>::JP;
        const double* W = rr + Layout<P>::WO;
        const double* sc = s_a + (size_t)P * ci;
        const double* sp = s_a + (size_t)P * n + 3 * (size_t)pj;
        const double* L = Lpt + 8 * (size_t)pj;
        const double l00 = L[0], l10 = L[1], l11 = L[2], l20 = L[3], l21 = L[4], l22 = L[5];
        const bool good = L[6] != 0.0;
        // three reciprocals per observation instead of 3P divisions (a DDIV
        // is a reciprocal iteration plus a slow-path check)
        const double i00 = 1.0 / l00, i11 = 1.0 / l11, i22 = 1.0 / l22;
#pragma unroll
        for (int p = 0; p < P; ++p) {
            const double t0 = jc[p] * W[0] + jc[P + p] * W[2];
            const double t1 = jc[p] * W[1] + jc[P + p] * W[3];
            double c[3];
#pragma unroll
            for (int q = 0; q < 3; ++q) c[q] = (sc[p] * (t0 * jp[q] + t1 * jp[3 + q])) * sp[q];
            const double w0 = c[0] * i00;
            const double w1 = (c[1] - l10 * w0) * i11;
            const double w2 = (c[2] - l20 * w0 - l21 * w1) * i22;
            wo[3 * p + 0] = good ? w0 : 0.0;
            wo[3 * p + 1] = good ? w1 : 0.0;
            wo[3 * p + 2] = good ? w2 : 0.0;
        }
#pragma unroll
        for (int z = 3 * P; z < kWStride; ++z) wo[z] = 0.0;
    }
    // ---- border partials: Σ W_a V_j per camera segment of the warp ----
    // In batches of 3 rows p (21 entries): each lane writes its products to
    // the warp's smem rows, then lane e sums column e over the warp's slots in
    // slot order, flushing at camera changes.
    __syncthreads();  // every thread has read its record: buf is reused
    {
        constexpr int BR = 3, BE = 7 * BR;  // rows per batch, entries per batch (odd pitch)
        const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
        const size_t gw = (size_t)(k >> 5);
        double* wbuf = buf + wib * 32 * BE;
        __shared__ int wcam[4][32];
        double v[21];
#pragma unroll
        for (int z = 0; z < 21; ++z) v[z] = (ci >= 0) ? __ldg(V + 21 * (size_t)pj + z) : 0.0;
        wcam[wib][lane] = ci;
        const unsigned vmask = __ballot_sync(0xffffffffu, ci >= 0);
        const int lastl = vmask ? 31 - __clz(vmask) : -1;
        const int cfirst = __shfl_sync(0xffffffffu, ci, 0);
        const int clast = lastl >= 0 ? __shfl_sync(0xffffffffu, ci, lastl) : -1;
#pragma unroll
        for (int p0 = 0; p0 < P; p0 += BR) {
            const int nr = (P - p0 < BR) ? P - p0 : BR;
            __syncwarp();
            if (ci >= 0) {
#pragma unroll
                for (int pr = 0; pr < BR; ++pr) {
                    if (pr < nr) {
                        const int p = p0 + pr;
#pragma unroll
                        for (int l = 0; l < 7; ++l)
                            wbuf[lane * BE + 7 * pr + l] = (wo[3 * p] * v[l] + wo[3 * p + 1] * v[7 + l]) + wo[3 * p + 2] * v[14 + l];
                    }
                }
            }
            __syncwarp();
            if (lane < 7 * nr && lastl >= 0) {
                const int eo = 7 * p0 + lane;  // entry (p, l) = (p0 + lane / 7, lane % 7)
                int cur = wcam[wib][0];
                double acc = 0.0;
                for (int o = 0; o <= lastl; ++o) {
                    const int c = wcam[wib][o];
                    if (c != cur) {
                        double* dst = (cur == cfirst) ? Pfirst + gw * NE : ((cur == clast) ? Plast + gw * NE : Gsum + (size_t)cur * NE);
                        dst[eo] = acc;
                        acc = 0.0;
                        cur = c;
                    }
                    acc += wbuf[o * BE + lane];
                }
                double* dst = (cur == cfirst) ? Pfirst + gw * NE : ((cur == clast) ? Plast + gw * NE : Gsum + (size_t)cur * NE);
                dst[eo] = acc;
            }
        }
    }
    __syncthreads();
    if (k < t_count) {
#pragma unroll
        for (int z = 0; z < kWStride; ++z) buf[threadIdx.x * PITCH + z] = wo[z];
    }
    __syncthreads();
    double2* out = reinterpret_cast<double2*>(Wb + (size_t)k0 * kWStride);
    for (int w = threadIdx.x; w < nv * (kWStride / 2); w += 128) {
        const int o = w / (kWStride / 2), part = w - o * (kWStride / 2);
        out[w] = make_double2(buf[o * PITCH + 2 * part], buf[o * PITCH + 2 * part + 1]);
    }
}

// F = Σ partials; L_F = chol(F); E = -F and E's pivots (-diag(L_F)^2) for
// the diagnostics.  One warp per entry of F's upper triangle (28 warps):
// lanes stride over the block partials (4 independent chains each), then a
// shuffle tree -- a fixed order, so the result is deterministic.
__global__ void __launch_bounds__(28 * 32) k_border_factor(const double* Fpart, int nblocks, double* LF, double* Eout,
                                                           double* eigE, Status* st) {
    __shared__ double red[28];
    // a grid of B blocks: B independent gauge blocks (batched sub-scenes),
    // each from its own nblocks partials
    Fpart += 28 * (size_t)nblocks * blockIdx.x;
    LF += 49 * blockIdx.x;
    Eout += 49 * blockIdx.x;
    eigE += 8 * blockIdx.x;
    const int e = threadIdx.x >> 5, lane = threadIdx.x & 31;
    double a0 = 0.0, a1 = 0.0, a2 = 0.0, a3 = 0.0;
    int b = lane;
    for (; b + 96 < nblocks; b += 128) {
        a0 += Fpart[28 * (size_t)b + e];
        a1 += Fpart[28 * (size_t)(b + 32) + e];
        a2 += Fpart[28 * (size_t)(b + 64) + e];
        a3 += Fpart[28 * (size_t)(b + 96) + e];
    }
    for (; b < nblocks; b += 32) a0 += Fpart[28 * (size_t)b + e];
    double acc = (a0 + a1) + (a2 + a3);
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
    if (lane == 0) red[e] = acc;
    __syncthreads();
    if (threadIdx.x != 0) return;
    double F[49];
    int k = 0;
    for (int l1 = 0; l1 < 7; ++l1)
        for (int l2 = l1; l2 < 7; ++l2, ++k) {
            F[7 * l1 + l2] = red[k];
            F[7 * l2 + l1] = red[k];
        }
    for (int q = 0; q < 49; ++q) Eout[q] = -F[q];
    double L[49];
    for (int q = 0; q < 49; ++q) L[q] = 0.0;
    bool ok = true;
    for (int c = 0; c < 7; ++c) {
        double s = F[7 * c + c];
        for (int kk = 0; kk < c; ++kk) s -= L[7 * c + kk] * L[7 * c + kk];
        if (!(s > 0.0)) { ok = false; s = 1.0; }
        const double lcc = sqrt(s);
        L[7 * c + c] = lcc;
        for (int r = c + 1; r < 7; ++r) {
            double x = F[7 * r + c];
            for (int kk = 0; kk < c; ++kk) x -= L[7 * r + kk] * L[7 * c + kk];
            L[7 * r + c] = x / lcc;
        }
    }
    if (!ok) st->border_bad = 1;
    for (int q = 0; q < 49; ++q) LF[q] = L[q];
    // border pivots for the diagnostics: the Cholesky pivots of -E (their
    // magnitudes are the |pivots| of E's LDL^T with D = -diag(L_F)^2)
    for (int c = 0; c < 7; ++c) eigE[c] = -L[7 * c + c] * L[7 * c + c];
}

// ---- camera border rows -----------------------------------------------------------
// Γ_i[p][l] = H_s,ci[p][l] - Σ_{a in cam i} (W_a V_j(a))[p][l] from the warp
// partials of k_obs_factor (added in warp order); then G_i = Γ_i L_F^-T.
// One 64-thread CTA per camera, one thread per entry (p, l).
template <int P>
__global__ void __launch_bounds__(64) k_camera_border(const int* off_cam, int t_count, const double* Pfirst,
                                                      const double* Plast, const double* Gsum, const double* cams,
                                                      const double* Hr, const double* s_a, const double* s_b,
                                                      const double* LF, int n, double* Gamma, double* G,
                                                      double* sums_out, const double* sums_in,
                                                      const int* scene_of_cam) {
    constexpr int NE = P * 7;
    __shared__ double sh[NE];
    const int i = blockIdx.x, tid = threadIdx.x;
    if (scene_of_cam) {  // batched sub-scenes: the camera's own gauge scales and factor
        const int scn = scene_of_cam[i];
        s_b += 7 * scn;
        LF += 49 * scn;
    }
    const int p = tid / 7, l = tid % 7;
    if (tid < NE) {
        double sum = 0.0;
        if (sums_in) {  // point-sharded stage A: the all-reduced sums
            sum = sums_in[(size_t)i * NE + tid];
        } else {
            const int b = off_cam[i], e = off_cam[i + 1];
            if (e > b) {
                bool any = false;
                for (int w = b >> 5; w <= (e - 1) >> 5; ++w) {
                    const int fs = 32 * w, ls = min(32 * w + 31, t_count - 1);
                    if (fs >= b && fs < e) { sum += Pfirst[(size_t)w * NE + tid]; any = true; }
                    else if (ls >= b && ls < e) { sum += Plast[(size_t)w * NE + tid]; any = true; }
                }
                if (!any) sum = Gsum[(size_t)i * NE + tid];  // the camera lies inside one warp
            }
        }
        if (sums_out) {  // this rank's partial, finished after the all-reduce
            sums_out[(size_t)i * NE + tid] = sum;
        } else {
        const double* C = cams + (size_t)P * i + 3;
        double h = 0.0;
        if (p < 3) h = (l >= 3 && l < 6) ? Hr[9 * (size_t)i + 3 * p + (l - 3)] : 0.0;
        else if (p < 6) {
            const int a = p - 3;
            double sx[9];
            skew(C, sx);
            h = (l < 3) ? (l == a ? 1.0 : 0.0) : (l < 6 ? sx[3 * a + (l - 3)] : C[a]);
        }
        const double hs = (s_a[(size_t)P * i + p] * h) * s_b[l];
        const double g = hs - sum;
        sh[tid] = g;
        Gamma[(size_t)P * 7 * i + tid] = g;
        }
    }
    if (sums_out) return;  // uniform over the CTA
    __syncthreads();
    if (tid < P) {
        const double* gr = &sh[7 * tid];
        double out[7];
        for (int ll = 0; ll < 7; ++ll) {
            double x = gr[ll];
            for (int kk = 0; kk < ll; ++kk) x -= LF[7 * ll + kk] * out[kk];
            out[ll] = x / LF[7 * ll + ll];
        }
        for (int ll = 0; ll < 7; ++ll) G[((size_t)P * i + tid) * 7 + ll] = out[ll];
    }
}

// ---- dense fill of the lower triangle --------------------------------------------
// Z(r, c) = [cam(r)==cam(c)] (s_a[r] D(r,c)) s_a[c] + add_gg * Σ_l G(r,l) G(c,l)
// for r, c < N; identity on the padding.  64x64 tiles with tile_r >= tile_c.
template <int P>
__global__ void k_fill(double* Z, long long ld, int N, int Npad, const double* D, const double* s_a, const double* G,
                       int add_gg) {
    __shared__ double gr[64][8], gc[64][8];
    const int T = Npad / 64;
    // lower-triangular tile index
    const long long l = blockIdx.x;
    int ti = (int)((sqrt(8.0 * (double)l + 1.0) - 1.0) * 0.5);
    while ((long long)(ti + 1) * (ti + 2) / 2 <= l) ++ti;
    while ((long long)ti * (ti + 1) / 2 > l) --ti;
    const int tj = (int)(l - (long long)ti * (ti + 1) / 2);
    (void)T;
    const int r0 = ti * 64, c0 = tj * 64;
    const int tid = threadIdx.x;
    if (add_gg) {
        for (int e = tid; e < 64 * 7; e += blockDim.x) {
            const int rr = e / 7, ll = e % 7;
            gr[rr][ll] = (r0 + rr < N) ? G[(size_t)(r0 + rr) * 7 + ll] : 0.0;
            gc[rr][ll] = (c0 + rr < N) ? G[(size_t)(c0 + rr) * 7 + ll] : 0.0;
        }
        __syncthreads();
    }
    const int rr = tid & 63;
    const int r = r0 + rr;
    double g[7];
#pragma unroll
    for (int q = 0; q < 7; ++q) g[q] = add_gg ? gr[rr][q] : 0.0;  // this thread's row, once
    const int ir = r / P;
    const double sr = (r < N) ? s_a[r] : 0.0;
    for (int cc = tid >> 6; cc < 64; cc += blockDim.x >> 6) {
        const int c = c0 + cc;
        double v;
        if (r < N && c < N) {
            v = 0.0;
            const int ic = c / P;
            if (ir == ic) v = (sr * D[(size_t)P * P * ir + P * (r - P * ir) + (c - P * ic)]) * s_a[c];
            if (add_gg) {
                double gg = 0.0;
#pragma unroll
                for (int q = 0; q < 7; ++q) gg += g[q] * gc[cc][q];  // gc row: warp-uniform broadcast
                v += gg;
            }
        } else {
            v = (r == c) ? 1.0 : 0.0;
        }
        Z[(size_t)c * ld + r] = v;
    }
}

// ---- observation pairs -----------------------------------------------------------
__global__ void k_pair_count(const int* off_pt, int m, long long* cnt) {
    const int j = blockIdx.x * blockDim.x + threadIdx.x;
    if (j > m) return;
    if (j == m) { cnt[m] = 0; return; }
    const long long k = off_pt[j + 1] - off_pt[j];
    cnt[j] = k * (k + 1) / 2;
}

// One warp per point: lanes read the track's cameras and by-camera slots
// once (tracks up to 32), then enumerate the k(k+1)/2 pairs (a <= c, the
// reference's order) with coalesced key / value stores.  Longer tracks: one
// lane, straight from global memory.
__global__ void __launch_bounds__(256) k_pair_gen(const int* off_pt, const int* idx_pt, const int* oc, const int* pos_cam,
                                                  int m, int n, const long long* poff, unsigned int* keys,
                                                  unsigned long long* vals) {
    const int j = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int lane = threadIdx.x & 31;
    if (j >= m) return;
    const long long o = poff[j];
    const int b = off_pt[j], e = off_pt[j + 1];
    const int k = e - b;
    if (k <= 32) {
        int mc = 0, ms = 0;
        if (lane < k) {
            const int ta = __ldg(idx_pt + b + lane);
            mc = __ldg(oc + ta);
            ms = __ldg(pos_cam + ta);
        }
        const int np = k * (k + 1) / 2;
        for (int q0 = 0; q0 < np; q0 += 32) {
            const int q = q0 + lane;
            int a = 0, r = q;
            while (a < k && r >= k - a) { r -= k - a; ++a; }  // row a, column c = a + r
            const int c = (a < k) ? a + r : 0;
            const int ca = __shfl_sync(0xffffffffu, mc, a & 31), sa = __shfl_sync(0xffffffffu, ms, a & 31);
            const int cb = __shfl_sync(0xffffffffu, mc, c & 31), sbb = __shfl_sync(0xffffffffu, ms, c & 31);
            if (q < np) {
                const bool le = ca <= cb;
                const unsigned lo = le ? ca : cb, hi = le ? cb : ca;
                const unsigned slo = le ? sa : sbb, shi = le ? sbb : sa;
                keys[o + q] = lo * (unsigned)n + hi;
                vals[o + q] = ((unsigned long long)shi << 32) | slo;
            }
        }
        return;
    }
    if (lane) return;
    long long w = o;
    for (int a = b; a < e; ++a) {
        const int ta = idx_pt[a];
        const int ca = oc[ta];
        for (int c = a; c < e; ++c) {
            const int tb = idx_pt[c];
            const int cb = oc[tb];
            int lo, hi, slo, shi;
            if (ca <= cb) { lo = ca; hi = cb; slo = pos_cam[ta]; shi = pos_cam[tb]; }
            else { lo = cb; hi = ca; slo = pos_cam[tb]; shi = pos_cam[ta]; }
            keys[w] = (unsigned int)lo * (unsigned int)n + (unsigned int)hi;
            vals[w] = ((unsigned long long)(unsigned int)shi << 32) | (unsigned int)slo;
            ++w;
        }
    }
}

// Tensor-core pair reduction: one warp per chunk (<= chunk pairs of one
// camera-pair block).  out = Σ_pairs W_hi W_lo^T is one product over the
// concatenated K dimension (3 entries per pair), so the FP64 m8n8k4 MMA runs
// on packed K: step s takes elements 4s .. 4s+3 of the chunk, lane (r, k)
// (r = lane/4, k = lane%4) loading W_hi[r][·] and W_lo[r][·] of element
// 4s + k (pair (4s+k)/3, entry (4s+k)%3) — 3 MMAs per 4 pairs, no zero pad.
// The MMA yields out(p, q) for p, q < 8 with lane holding (p = lane/4,
// q = 2(lane%4) + {0,1}).  For P = 9 row 8 and column 8 are FP64 FMAs on the
// same operands: lane (q, k) adds W_hi[8][e] W_lo[q][e] (W_hi[8][e] shuffled
// from lane k, which loads row 8) and W_hi[q][e] W_lo[8][e]; the four
// k-partials are summed once per chunk.  The pair list is read 32 at a time
// with one coalesced load and distributed by shuffles; U steps are gathered
// ahead of their MMAs.
__device__ __forceinline__ void dmma_pr(double& d0, double& d1, double a, double b) {
    asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                 : "+d"(d0), "+d"(d1)
                 : "d"(a), "d"(b));
}

template <int P, int U, int MINB>
__global__ void __launch_bounds__(256, MINB) k_pair_reduce_mma(const unsigned int* ukeys, const long long* seg_off,
                                                         const int* seg_of, const int* chunk_off, int nchunks,
                                                         int chunk, const unsigned long long* vals, const double* Wb,
                                                         int n, double* Z, long long ld, double* part, int cfirst,
                                                         int always_part, int lo_min, int lo_max, ZMap zm) {
    const int warp = cfirst + ((blockIdx.x * blockDim.x + threadIdx.x) >> 5);
    const int lane = threadIdx.x & 31;
    if (warp >= nchunks) return;
    const int sg = __ldg(seg_of + warp);  // (a binary search over chunk_off was ~16 dependent loads)
    const unsigned int key = ukeys[sg];
    const int lo = (int)(key / (unsigned int)n), hi = (int)(key - (unsigned int)lo * (unsigned int)n);
    if (lo < lo_min || lo >= lo_max) return;  // block column outside this launch's camera range
    const int c0 = __ldg(chunk_off + sg), nch = __ldg(chunk_off + sg + 1) - c0;
    const int r = lane >> 2, k = lane & 3;
    const long long sb = seg_off[sg], se = seg_off[sg + 1];
    const long long b = sb + (long long)(warp - c0) * chunk;
    const long long e = min(se, b + chunk);
    double c0v = 0.0, c1v = 0.0;                 // MMA tile (rows 0..7, cols 0..7)
    double r8 = 0.0, cl8 = 0.0, x88 = 0.0;       // P = 9: row 8, column 8, corner (k-partials)
    for (long long base = b; base < e; base += 32) {
        const int cnt = (int)min(32LL, e - base);
        const unsigned long long mine = (lane < cnt) ? __ldg(vals + base + lane) : 0ULL;
        const int nel = 3 * cnt, nsteps = (nel + 3) >> 2;
        for (int s0 = 0; s0 < nsteps; s0 += U) {
            double ah[U], al[U], a8[U], b8[U];
#pragma unroll
            for (int u = 0; u < U; ++u) {
                const int el = 4 * (s0 + u) + k;
                const int pi = el / 3, kk = el - 3 * pi;
                const bool ok = el < nel;
                const unsigned long long v = __shfl_sync(0xffffffffu, mine, pi & 31);
                const double* wh = Wb + (size_t)(v >> 32) * kWStride;
                const double* wl = Wb + (size_t)(v & 0xffffffffULL) * kWStride;
                ah[u] = ok ? __ldg(wh + 3 * r + kk) : 0.0;
                al[u] = ok ? __ldg(wl + 3 * r + kk) : 0.0;
                if (P == 9) {
                    a8[u] = (ok && r == 0) ? __ldg(wh + 24 + kk) : 0.0;
                    b8[u] = (ok && r == 0) ? __ldg(wl + 24 + kk) : 0.0;
                }
            }
#pragma unroll
            for (int u = 0; u < U; ++u) {
                dmma_pr(c0v, c1v, ah[u], al[u]);
                if (P == 9) {
                    const double h8 = __shfl_sync(0xffffffffu, a8[u], k);  // W_hi[8][e] from lane k
                    const double l8 = __shfl_sync(0xffffffffu, b8[u], k);  // W_lo[8][e] from lane k
                    r8 = fma(h8, al[u], r8);
                    cl8 = fma(ah[u], l8, cl8);
                    x88 = fma(a8[u], b8[u], x88);
                }
            }
        }
    }
    if (P == 9) {  // sum the four k-partials (fixed order)
        r8 += __shfl_xor_sync(0xffffffffu, r8, 1);
        r8 += __shfl_xor_sync(0xffffffffu, r8, 2);
        cl8 += __shfl_xor_sync(0xffffffffu, cl8, 1);
        cl8 += __shfl_xor_sync(0xffffffffu, cl8, 2);
        x88 += __shfl_xor_sync(0xffffffffu, x88, 1);
        x88 += __shfl_xor_sync(0xffffffffu, x88, 2);
    }
    const bool diag = lo == hi;
    // single chunk: Z(P hi + p, P lo + q) -= out(p, q) (diagonal blocks: lower
    // part only); else the chunk's partial block, combined by k_pair_combine
    double* pp = part + (size_t)warp * 81;
    double* Zs = Z;
    int lz = lo, hz = hi;
    if (zm.scene_of_cam) {  // batched sub-scenes: the scene's own Z, local camera indices
        const int scn = zm.scene_of_cam[lo];
        Zs = Z + scn * zm.zstride;
        lz -= zm.coff[scn];
        hz -= zm.coff[scn];
    }
    auto put = [&](int p, int q, double v) {
        if (nch > 1 || always_part) { pp[P * p + q] = v; return; }
        if (diag && p < q) return;
        double* z = Zs + ((size_t)P * lz + q) * ld + (size_t)P * hz + p;
        *z = *z - v;
    };
    const int q0 = 2 * k;
    put(r, q0, c0v);
    put(r, q0 + 1, c1v);
    if (P == 9) {
        if (k == 0) {
            put(8, r, r8);   // lane (q = r, k = 0): row 8, column r
            put(r, 8, cl8);  // row r, column 8
        }
        if (lane == 0) put(8, 8, x88);
    }
}

// The same reduction with the operands staged through shared memory: each
// warp copies the two factor rows of 8 pairs at a time (16 rows x 224 B,
// coalesced 16-byte cp.async, two stages in flight) and feeds the MMA
// fragments from shared memory.  The register-gather version above keeps
// every lane's scattered 8-byte loads on the critical path (ncu: 50-65 %
// long-scoreboard stalls, 3.2 GB of L2 sectors for 0.36 GB of operands);
// here a lane has 7 16-byte copies in flight per stage.  SFMCOV_PAIR_KERNEL=gather
// selects the register-gather kernel (A/B measurements).  Same chunking,
// same per-lane accumulation order, same output / partial layout.
constexpr int kCpRowParts = kWStride / 2; // 16-byte parts per factor row
template <int BP, int NW>
constexpr size_t pair_cp_smem_bytes() { return (size_t)NW * 2 * (2 * BP) * kWStride * sizeof(double); }

template <int P, int kCpPairs, int kCpWarps, int MINB>
__global__ void __launch_bounds__(kCpWarps * 32, MINB) k_pair_reduce_cp(const unsigned int* ukeys, const long long* seg_off,
                                                                   const int* seg_of, const int* chunk_off, int nchunks,
                                                                   int chunk, const unsigned long long* vals,
                                                                   const double* Wb, int n, double* Z, long long ld,
                                                                   double* part, int cfirst, int always_part,
                                                                   int lo_min, int lo_max, ZMap zm) {
    extern __shared__ __align__(16) double sm_pairs[];
    const int wib = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int warp = cfirst + blockIdx.x * kCpWarps + wib;
    if (warp >= nchunks) return;
    const int sg = __ldg(seg_of + warp);
    const unsigned int key = ukeys[sg];
    const int lo = (int)(key / (unsigned int)n), hi = (int)(key - (unsigned int)lo * (unsigned int)n);
    if (lo < lo_min || lo >= lo_max) return;
    const int c0 = __ldg(chunk_off + sg), nch = __ldg(chunk_off + sg + 1) - c0;
    const int r = lane >> 2, k = lane & 3;
    const long long sb = seg_off[sg], se = seg_off[sg + 1];
    const long long b = sb + (long long)(warp - c0) * chunk;
    const long long e = min(se, b + chunk);
    double* stage_base = sm_pairs + (size_t)wib * 2 * (2 * kCpPairs) * kWStride;
    auto stage = [&](int st) { return stage_base + (size_t)st * (2 * kCpPairs) * kWStride; };
    const int nb = (int)((e - b + kCpPairs - 1) / kCpPairs);
    auto issue = [&](int bi) {
        double* dst = stage(bi & 1);
        const long long pb = b + (long long)bi * kCpPairs;
        const int cnt = (int)min((long long)kCpPairs, e - pb);
        // lane i < cnt holds pair i's slots; the copies fetch them by shuffle
        const unsigned long long mine = lane < cnt ? __ldg(vals + pb + lane) : 0ULL;
#pragma unroll
        for (int c0 = 0; c0 < 2 * kCpPairs * kCpRowParts; c0 += 32) {
            const int c = c0 + lane;
            const int row = c / kCpRowParts, prt = c - row * kCpRowParts;
            const int pi = row >> 1;
            const unsigned long long v = __shfl_sync(0xffffffffu, mine, pi & 31);
            if (c < 2 * kCpPairs * kCpRowParts && pi < cnt) {
                const unsigned int slot = (row & 1) ? (unsigned int)(v & 0xffffffffULL) : (unsigned int)(v >> 32);
                cpa16(dst + (size_t)row * kWStride + 2 * prt, Wb + (size_t)slot * kWStride + 2 * prt);
            }
        }
        cpa_commit();
    };
    double c0v = 0.0, c1v = 0.0;            // MMA tile (rows 0..7, cols 0..7)
    double r8 = 0.0, cl8 = 0.0, x88 = 0.0;  // P = 9: row 8, column 8, corner (k-partials)
    if (nb > 0) issue(0);
    for (int bi = 0; bi < nb; ++bi) {
        if (bi + 1 < nb) {
            issue(bi + 1);
            cpa_wait<1>();
        } else {
            cpa_wait<0>();
        }
        __syncwarp();
        const double* src = stage(bi & 1);
        const int cnt = (int)min((long long)kCpPairs, e - (b + (long long)bi * kCpPairs));
        const int nel = 3 * cnt, nsteps = (nel + 3) >> 2;
#pragma unroll 4
        for (int st = 0; st < nsteps; ++st) {
            const int el = 4 * st + k;
            const int pi = el / 3, kk = el - 3 * pi;
            const bool ok = el < nel;
            const double* wh = src + (size_t)(2 * pi) * kWStride;
            const double* wl = wh + kWStride;
            const double ah = ok ? wh[3 * r + kk] : 0.0;
            const double al = ok ? wl[3 * r + kk] : 0.0;
            dmma_pr(c0v, c1v, ah, al);
            if (P == 9) {
                const double h8 = ok ? wh[24 + kk] : 0.0;
                const double l8 = ok ? wl[24 + kk] : 0.0;
                r8 = fma(h8, al, r8);
                cl8 = fma(ah, l8, cl8);
                if (r == 0) x88 = fma(h8, l8, x88);
            }
        }
        __syncwarp();  // the stage is refilled two batches later
    }
    if (P == 9) {  // sum the four k-partials (fixed order)
        r8 += __shfl_xor_sync(0xffffffffu, r8, 1);
        r8 += __shfl_xor_sync(0xffffffffu, r8, 2);
        cl8 += __shfl_xor_sync(0xffffffffu, cl8, 1);
        cl8 += __shfl_xor_sync(0xffffffffu, cl8, 2);
        x88 += __shfl_xor_sync(0xffffffffu, x88, 1);
        x88 += __shfl_xor_sync(0xffffffffu, x88, 2);
    }
    const bool diag = lo == hi;
    double* pp = part + (size_t)warp * 81;
    double* Zs = Z;
    int lz = lo, hz = hi;
    if (zm.scene_of_cam) {  // batched sub-scenes: the scene's own Z, local camera indices
        const int scn = zm.scene_of_cam[lo];
        Zs = Z + scn * zm.zstride;
        lz -= zm.coff[scn];
        hz -= zm.coff[scn];
    }
    auto put = [&](int p, int q, double v) {
        if (nch > 1 || always_part) { pp[P * p + q] = v; return; }
        if (diag && p < q) return;
        double* z = Zs + ((size_t)P * lz + q) * ld + (size_t)P * hz + p;
        *z = *z - v;
    };
    const int q0 = 2 * k;
    put(r, q0, c0v);
    put(r, q0 + 1, c1v);
    if (P == 9) {
        if (k == 0) {
            put(8, r, r8);
            put(r, 8, cl8);
        }
        if (lane == 0) put(8, 8, x88);
    }
}

static bool pair_kernel_old() {
    static bool v = [] { const char* e = std::getenv("SFMCOV_PAIR_KERNEL"); return e && std::string(e) == "gather"; }();
    return v;
}

static void launch_pair_mma(int P, const PairDev& pd, const double* Wb, int n, double* Z, long long ld, int cfirst,
                            int clast, int always_part, int lo_min, int lo_max, cudaStream_t s, ZMap zm = ZMap{}) {
    const int cnt = clast - cfirst;
    if (cnt <= 0) return;
    if (pair_kernel_old()) {
        const unsigned cblocks = cdiv(cnt, 8);
        if (P == 8)
            k_pair_reduce_mma<8, 4, 4><<<cblocks, 256, 0, s>>>(pd.ukeys, pd.seg_off, pd.seg_of, pd.chunk_off, clast,
                                                                pd.chunk, pd.vals, Wb, n, Z, ld, pd.part, cfirst,
                                                                always_part, lo_min, lo_max, zm);
        else
            k_pair_reduce_mma<9, 4, 4><<<cblocks, 256, 0, s>>>(pd.ukeys, pd.seg_off, pd.seg_of, pd.chunk_off, clast,
                                                                pd.chunk, pd.vals, Wb, n, Z, ld, pd.part, cfirst,
                                                                always_part, lo_min, lo_max, zm);
        SFM_LAUNCH_CHECK();
        return;
    }
    // 8 pairs per stage, 4 warps per CTA, 6 CTAs per SM (24 warps): config 3
    // pair stage 0.78 ms against 0.82 for the register gathers; 16 pairs x 4
    // warps (12 warps / SM) 0.91, 8 x 8 warps 0.79, one zero-padded MMA per
    // pair (no index division) 1.06 -- the kernel is issue-bound (IPC 2.3,
    // 58 % issue slots, ncu profiles/r02_ncu_pair_reduce.txt)
    auto go = [&](auto kern, size_t smem) {
        SFM_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
        kern<<<cdiv(cnt, 4), 4 * 32, smem, s>>>(pd.ukeys, pd.seg_off, pd.seg_of, pd.chunk_off, clast, pd.chunk,
                                                pd.vals, Wb, n, Z, ld, pd.part, cfirst, always_part, lo_min, lo_max, zm);
        SFM_LAUNCH_CHECK();
    };
    if (P == 8) go(k_pair_reduce_cp<8, 8, 4, 6>, pair_cp_smem_bytes<8, 4>());
    else go(k_pair_reduce_cp<9, 8, 4, 6>, pair_cp_smem_bytes<8, 4>());
}

// Multi-chunk segments: partial blocks summed in chunk order, then written.
template <int P>
__global__ void __launch_bounds__(256) k_pair_combine(const unsigned int* ukeys, int nseg, const int* chunk_off,
                                                      const double* part, int n, double* Z, long long ld, int lo_min,
                                                      int lo_max, ZMap zm) {
    const int sg = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int lane = threadIdx.x & 31;
    if (sg >= nseg) return;
    const int c0 = chunk_off[sg], c1 = chunk_off[sg + 1];
    if (c1 - c0 < 2) return;
    const unsigned int key = ukeys[sg];
    const int lo = (int)(key / (unsigned int)n), hi = (int)(key - (unsigned int)lo * (unsigned int)n);
    if (lo < lo_min || lo >= lo_max) return;
    double* Zs = Z;
    int lz = lo, hz = hi;
    if (zm.scene_of_cam) {
        const int scn = zm.scene_of_cam[lo];
        Zs = Z + scn * zm.zstride;
        lz -= zm.coff[scn];
        hz -= zm.coff[scn];
    }
    for (int en = lane; en < P * P; en += 32) {
        const int p = en / P, q = en - P * (en / P);
        if (lo == hi && p < q) continue;
        double v = 0.0;
        for (int c = c0; c < c1; ++c) v += part[(size_t)c * 81 + en];
        double* z = Zs + ((size_t)P * lz + q) * ld + (size_t)P * hz + p;
        *z = *z - v;
    }
}

// Segment blocks from the chunk partials in [c_begin, c_end) (chunk order;
// zero for segments without such chunks).  seg_out[sg * 81 + P p + q].
template <int P>
__global__ void __launch_bounds__(256) k_pair_combine_seg(int nseg, const int* chunk_off, const double* part,
                                                          int c_begin, int c_end, double* seg_out) {
    const int sg = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int lane = threadIdx.x & 31;
    if (sg >= nseg) return;
    const int c0 = max(chunk_off[sg], c_begin), c1 = min(chunk_off[sg + 1], c_end);
    for (int en = lane; en < P * P; en += 32) {
        double v = 0.0;
        for (int c = c0; c < c1; ++c) v += part[(size_t)c * 81 + en];
        seg_out[(size_t)sg * 81 + en] = v;
    }
}

// ---- host launchers ----------------------------------------------------------------
int point_prep_blocks(int m) { return (int)cdiv(m > 0 ? m : 1, 128); }

void launch_point_prep(const SceneDev& sc, const IndexDev& ix, const double* rec, const double* A, const double* s_a,
                       const double* s_b, double* Lpt, double* Wb, double* V, double* Fpart, double* Pfirst,
                       double* Plast, double* Gsum, Status* st, cudaStream_t s, const int* scene_of_pt) {
    const int nb = point_prep_blocks(sc.m);
    if (sc.P == 8) k_point_prep<8><<<nb, 128, 0, s>>>(A, s_a, sc.pts, s_b, sc.m, sc.n, Lpt, V, Fpart, st, scene_of_pt);
    else k_point_prep<9><<<nb, 128, 0, s>>>(A, s_a, sc.pts, s_b, sc.m, sc.n, Lpt, V, Fpart, st, scene_of_pt);
    SFM_LAUNCH_CHECK();
    if (sc.t) {
        if (sc.P == 8) k_obs_factor<8><<<cdiv(sc.t, 128), 128, 0, s>>>(sc.oc, sc.op, ix.idx_cam, rec, s_a, Lpt, V, sc.t, sc.n, Wb, Pfirst, Plast, Gsum);
        else k_obs_factor<9><<<cdiv(sc.t, 128), 128, 0, s>>>(sc.oc, sc.op, ix.idx_cam, rec, s_a, Lpt, V, sc.t, sc.n, Wb, Pfirst, Plast, Gsum);
        SFM_LAUNCH_CHECK();
    }
}

void launch_border_factor(const double* Fpart, int nblocks, double* LF, double* E, double* eigE, Status* st,
                          cudaStream_t s, int batch) {
    if (batch < 1) return;
    k_border_factor<<<batch, 28 * 32, 0, s>>>(Fpart, nblocks, LF, E, eigE, st);
    SFM_LAUNCH_CHECK();
}

void launch_camera_border(const SceneDev& sc, const IndexDev& ix, const double* Pfirst, const double* Plast,
                          const double* Gsum, const double* Hr, const double* s_a, const double* s_b, const double* LF,
                          double* Gamma, double* G, cudaStream_t s, double* sums_out, const double* sums_in,
                          const int* scene_of_cam) {
    if (!sc.n) return;
    if (sc.P == 8) k_camera_border<8><<<sc.n, 64, 0, s>>>(ix.off_cam, sc.t, Pfirst, Plast, Gsum, sc.cams, Hr, s_a, s_b, LF, sc.n, Gamma, G, sums_out, sums_in, scene_of_cam);
    else k_camera_border<9><<<sc.n, 64, 0, s>>>(ix.off_cam, sc.t, Pfirst, Plast, Gsum, sc.cams, Hr, s_a, s_b, LF, sc.n, Gamma, G, sums_out, sums_in, scene_of_cam);
    SFM_LAUNCH_CHECK();
}

// Σ of the point-preparation blocks' F partials (28 entries, fixed order):
// this rank's part of F, all-reduced before launch_border_factor(F, 1, ...).
__global__ void k_fpart_sum(const double* Fpart, int nblocks, double* F28) {
    const int e = threadIdx.x;
    if (e >= 28) return;
    double acc = 0.0;
    for (int b = 0; b < nblocks; ++b) acc += Fpart[28 * (size_t)b + e];
    F28[e] = acc;
}
void launch_fpart_sum(const double* Fpart, int nblocks, double* F28, cudaStream_t s) {
    k_fpart_sum<<<1, 32, 0, s>>>(Fpart, nblocks, F28);
    SFM_LAUNCH_CHECK();
}

void launch_fill(int P, double* Z, long long ld, int N, int Npad, const double* D, const double* s_a, const double* G,
                 int add_gg, cudaStream_t s) {
    const long long T = Npad / 64;
    const long long tiles = T * (T + 1) / 2;
    if (!tiles) return;
    if (P == 8) k_fill<8><<<(unsigned)tiles, 256, 0, s>>>(Z, ld, N, Npad, D, s_a, G, add_gg);
    else k_fill<9><<<(unsigned)tiles, 256, 0, s>>>(Z, ld, N, Npad, D, s_a, G, add_gg);
    SFM_LAUNCH_CHECK();
}

// Pairs per work item of the pair reduction (SFMCOV_PAIR_CHUNK, default 128).
static int pair_chunk() {
    static int c = [] {
        const char* e = std::getenv("SFMCOV_PAIR_CHUNK");
        const int v = e ? std::atoi(e) : 128;
        return (v >= 4 && v <= (1 << 20)) ? v : 128;
    }();
    return c;
}

__global__ void k_chunk_segment(const int* chunk_off, int nseg, int* seg_of) {
    const int sg = blockIdx.x * blockDim.x + threadIdx.x;
    if (sg >= nseg) return;
    for (int c = chunk_off[sg]; c < chunk_off[sg + 1]; ++c) seg_of[c] = sg;
}

__global__ void k_chunk_count(const int* counts, int nseg, int chunk, int* ccnt) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i < nseg) ccnt[i] = (counts[i] + chunk - 1) / chunk;
    else if (i == nseg) ccnt[i] = 0;
}

static int bits_for64(unsigned long long v) { int b = 1; while (b < 64 && (1ULL << b) <= v) ++b; return b; }

// Builds the sorted pair list and the block segments; returns #pairs and
// #segments through the handle-owned PairDev.
void build_pairs(const SceneDev& sc, const IndexDev& ix, PairDev& pd, Workspace& ws, cudaStream_t s) {
    const int m = sc.m;
    pd.cnt = (long long*)pd.buf_cnt.get(sizeof(long long) * (size_t)(m + 1));
    pd.off = (long long*)pd.buf_off.get(sizeof(long long) * (size_t)(m + 1));
    k_pair_count<<<cdiv(m + 1, 256), 256, 0, s>>>(ix.off_pt, m, pd.cnt);
    SFM_LAUNCH_CHECK();
    size_t bytes = 0;
    cub::DeviceScan::ExclusiveSum(nullptr, bytes, pd.cnt, pd.off, m + 1, s);
    SFM_CUDA(cub::DeviceScan::ExclusiveSum(ws.get_tmp(bytes), bytes, pd.cnt, pd.off, m + 1, s));
    long long npairs = 0;
    SFM_CUDA(cudaMemcpyAsync(&npairs, pd.off + m, sizeof(long long), cudaMemcpyDeviceToHost, s));
    SFM_CUDA(cudaStreamSynchronize(s));
    pd.npairs = npairs;
    // CUB's sort / run-length encode take int item counts
    if (npairs > (long long)INT_MAX)
        throw SizeGuard("schur", std::to_string(npairs) + " observation pairs exceed the 2^31-1 pair-list limit");
    const size_t np = (size_t)npairs;
    unsigned int* k0 = (unsigned int*)pd.buf_k0.get(4 * np + 16);
    unsigned int* k1 = (unsigned int*)pd.buf_k1.get(4 * np + 16);
    unsigned long long* v0 = (unsigned long long*)pd.buf_v0.get(8 * np + 16);
    unsigned long long* v1 = (unsigned long long*)pd.buf_v1.get(8 * np + 16);
    if (m) k_pair_gen<<<cdiv((long long)m * 32, 256), 256, 0, s>>>(ix.off_pt, ix.idx_pt, sc.oc, ix.pos_cam, m, sc.n, pd.off, k0, v0);
    SFM_LAUNCH_CHECK();
    const int kbits = bits_for64((unsigned long long)sc.n * (unsigned long long)sc.n);
    cub::DoubleBuffer<unsigned int> dk(k0, k1);
    cub::DoubleBuffer<unsigned long long> dv(v0, v1);
    size_t sb = 0;
    cub::DeviceRadixSort::SortPairs(nullptr, sb, dk, dv, (int)np, 0, kbits, s);
    SFM_CUDA(cub::DeviceRadixSort::SortPairs(ws.get_tmp(sb), sb, dk, dv, (int)np, 0, kbits, s));
    pd.keys = dk.Current();
    pd.vals = dv.Current();
    // run-length encode the sorted keys into block segments
    unsigned int* ukeys = (unsigned int*)pd.buf_ukeys.get(4 * np + 16);
    int* counts = (int*)pd.buf_counts.get(4 * np + 16);
    int* nruns = (int*)pd.buf_nruns.get(16);
    size_t rb = 0;
    cub::DeviceRunLengthEncode::Encode(nullptr, rb, pd.keys, ukeys, counts, nruns, (int)np, s);
    SFM_CUDA(cub::DeviceRunLengthEncode::Encode(ws.get_tmp(rb), rb, pd.keys, ukeys, counts, nruns, (int)np, s));
    int nseg = 0;
    SFM_CUDA(cudaMemcpyAsync(&nseg, nruns, sizeof(int), cudaMemcpyDeviceToHost, s));
    SFM_CUDA(cudaStreamSynchronize(s));
    pd.nseg = nseg;
    pd.ukeys = ukeys;
    long long* seg_off = (long long*)pd.buf_seg.get(8 * ((size_t)nseg + 1) + 16);
    // widen counts to int64 offsets
    size_t eb = 0;
    cub::DeviceScan::ExclusiveSum(nullptr, eb, counts, seg_off, nseg + 1, s);
    // counts[nseg] must be 0 for the trailing total: set it
    SFM_CUDA(cudaMemsetAsync(counts + nseg, 0, sizeof(int), s));
    SFM_CUDA(cub::DeviceScan::ExclusiveSum(ws.get_tmp(eb), eb, counts, seg_off, nseg + 1, s));
    pd.seg_off = seg_off;
    // split segments into chunks of at most pair_chunk() pairs (load balance:
    // diagonal blocks carry ~10x the pairs of an off-diagonal one)
    pd.chunk = pair_chunk();
    int* ccnt = (int*)pd.buf_chunk.get(8 * ((size_t)nseg + 1) + 16);
    int* coff = ccnt + (nseg + 1);
    k_chunk_count<<<cdiv(nseg + 1, 256), 256, 0, s>>>(counts, nseg, pd.chunk, ccnt);
    SFM_LAUNCH_CHECK();
    size_t cb = 0;
    cub::DeviceScan::ExclusiveSum(nullptr, cb, ccnt, coff, nseg + 1, s);
    SFM_CUDA(cub::DeviceScan::ExclusiveSum(ws.get_tmp(cb), cb, ccnt, coff, nseg + 1, s));
    int nch = 0;
    SFM_CUDA(cudaMemcpyAsync(&nch, coff + nseg, sizeof(int), cudaMemcpyDeviceToHost, s));
    SFM_CUDA(cudaStreamSynchronize(s));
    pd.chunk_off = coff;
    pd.nchunks = nch;
    pd.seg_of = (int*)pd.buf_segof.get(4 * ((size_t)nch + 1));
    if (nseg) {
        k_chunk_segment<<<cdiv(nseg, 256), 256, 0, s>>>(coff, nseg, pd.seg_of);
        SFM_LAUNCH_CHECK();
    }
    pd.part = (double*)pd.buf_part.get(8 * 81 * ((size_t)nch + 1));
}

// Segments whose block column (camera lo) lies in [lo_min, lo_max): the
// sweep's first panel needs only its own columns, so the pipeline reduces
// those first and the rest beside the first panel's factorisation.
void launch_pair_reduce(int P, const PairDev& pd, const double* Wb, int n, double* Z, long long ld, cudaStream_t s,
                        int lo_min, int lo_max, ZMap zm) {
    if (!pd.nseg) return;
    const unsigned blocks = cdiv(pd.nseg, 8);
    launch_pair_mma(P, pd, Wb, n, Z, ld, 0, pd.nchunks, 0, lo_min, lo_max, s, zm);
    if (P == 8) k_pair_combine<8><<<blocks, 256, 0, s>>>(pd.ukeys, pd.nseg, pd.chunk_off, pd.part, n, Z, ld, lo_min, lo_max, zm);
    else k_pair_combine<9><<<blocks, 256, 0, s>>>(pd.ukeys, pd.nseg, pd.chunk_off, pd.part, n, Z, ld, lo_min, lo_max, zm);
    SFM_LAUNCH_CHECK();
}

void launch_pair_reduce_segments(int P, const PairDev& pd, const double* Wb, int n, int c_begin, int c_end,
                                 double* seg_out, cudaStream_t s) {
    if (!pd.nseg) return;
    launch_pair_mma(P, pd, Wb, n, nullptr, 0, c_begin, c_end, 1, 0, n, s);
    const unsigned blocks = cdiv(pd.nseg, 8);
    if (P == 8) k_pair_combine_seg<8><<<blocks, 256, 0, s>>>(pd.nseg, pd.chunk_off, pd.part, c_begin, c_end, seg_out);
    else k_pair_combine_seg<9><<<blocks, 256, 0, s>>>(pd.nseg, pd.chunk_off, pd.part, c_begin, c_end, seg_out);
    SFM_LAUNCH_CHECK();
}

}  // namespace sfm
