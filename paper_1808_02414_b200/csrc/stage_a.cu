// Stage (a) + (c): validation, observation index, analytic Jacobian,
// per-camera / per-point Fisher reductions, gauge-nullspace rotation blocks
// and Jacobi conditioning scales.
//
// Compiled with --fmad=false: these kernels follow the CPU restatement
// (oracle/) operation for operation, so the Jacobian, the nullspace and the
// unconditioned Fisher blocks are bit-exact against it.  Reductions run in
// ascending observation order per camera / per point, exactly like the
// reference (src/covariance.cpp:57-71, src/nullspace.cpp:40-50), which also
// makes every result bitwise reproducible run to run.
#include "common.cuh"
#include "detmath.cuh"
#include "kernels.cuh"

#include <cub/cub.cuh>

namespace sfm {

__global__ void k_status_init(Status* st) {
    if (threadIdx.x == 0 && blockIdx.x == 0) {
        st->cam_bad = INT_MAX; st->pt_bad = INT_MAX; st->obs_bad = LLONG_MAX; st->dup = 0;
        st->cam_count_bad = INT_MAX; st->pt_count_bad = INT_MAX; st->jac_bad = INT_MAX;
        st->fisher_bad = INT_MAX; st->rot_bad = INT_MAX; st->pt_sing_bad = INT_MAX;
        st->border_bad = 0; st->chol_bad = INT_MAX; st->nflag = 0; st->pad = 0;
    }
}

// ---- validation: src/scene.cpp:19-78 -------------------------------------------
__device__ __forceinline__ bool finite_d(double v) { return isfinite(v); }

__global__ void k_validate_cams(const double* cams, int n, int P, Status* st) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const double* c = cams + (size_t)P * i;
    bool fin = true;
    for (int p = 0; p < P; ++p) fin = fin && finite_d(c[p]);
    int code = 0;
    if (!fin) code = 1;
    else if (!(c[6] > 0.0)) code = 2;
    if (code) atomicMin(&st->cam_bad, i * 4 + code);
}

__global__ void k_validate_pts(const double* pts, int m, Status* st) {
    const int j = blockIdx.x * blockDim.x + threadIdx.x;
    if (j >= m) return;
    const double* X = pts + 3 * (size_t)j;
    if (!(finite_d(X[0]) && finite_d(X[1]) && finite_d(X[2]))) atomicMin(&st->pt_bad, j);
}

// Finiteness / symmetry / definiteness of one observation (codes 3, 4, 5 of
// scene.cpp validate; 0 = fine).  u may be null (checked on the host).
__device__ __forceinline__ int obs_value_code(const double* u, const double* sigma, int t) {
    double s00 = 1.0, s01 = 0.0, s10 = 0.0, s11 = 1.0;
    if (sigma) { s00 = sigma[4 * (size_t)t]; s01 = sigma[4 * (size_t)t + 1]; s10 = sigma[4 * (size_t)t + 2]; s11 = sigma[4 * (size_t)t + 3]; }
    const bool ufin = !u || (finite_d(u[2 * (size_t)t]) && finite_d(u[2 * (size_t)t + 1]));
    if (!ufin || !finite_d(s00) || !finite_d(s01) || !finite_d(s10) || !finite_d(s11)) return 3;
    const double scale = fmax(fmax(fmax(fabs(s00), fabs(s11)), fabs(s01)), 1e-300);
    if (fabs(s01 - s10) > 1e-12 * scale) return 4;
    const double det = s00 * s11 - s01 * s10;
    if (!(s00 > 0.0) || !(det > 0.0)) return 5;
    return 0;
}

// check_sigma = 1: full scene validation; 0: only index ranges (stage APIs
// that, like the reference functions, do not validate, and host-API scenes
// whose covariances are still uploading: k_validate_values checks them).
__global__ void k_validate_obs(const int* oc, const int* op, const double* u, const double* sigma, int t_count,
                               int n, int m, int check_sigma, Status* st) {
    const int t = blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= t_count) return;
    const int ci = oc[t], pj = op[t];
    int code = 0;
    if (ci < 0 || ci >= n) code = 1;
    else if (pj < 0 || pj >= m) code = 2;
    else if (check_sigma) code = obs_value_code(u, sigma, t);
    if (code) atomicMin(&st->obs_bad, (long long)t * 8 + code);
}

// The value checks alone (codes 3-5), once the covariances have arrived; an
// observation with a bad index keeps its smaller code through atomicMin.
__global__ void k_validate_values(const double* u, const double* sigma, int t_count, Status* st) {
    const int t = blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= t_count) return;
    const int code = obs_value_code(u, sigma, t);
    if (code) atomicMin(&st->obs_bad, (long long)t * 8 + code);
}

__global__ void k_iota(int* v, int count) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i < count) v[i] = i;
}

// CSR offsets from keys sorted ascending (all in [0, bins)): off[c] = first
// position with key >= c, off[bins] = count.  Replaces per-observation count
// atomics (hot cameras serialised them: 130 us at config 3).
__global__ void k_offsets_from_sorted(const int* keys, int count, int bins, int* off) {
    const int k = blockIdx.x * blockDim.x + threadIdx.x;
    if (k >= count) return;
    const int key = keys[k];
    const int prev = k > 0 ? keys[k - 1] : -1;
    for (int c = prev + 1; c <= key; ++c) off[c] = k;
    if (k == count - 1)
        for (int c = key + 1; c <= bins; ++c) off[c] = count;
}

__global__ void k_pos_scatter(const int* idx, int count, int* pos) {
    const int k = blockIdx.x * blockDim.x + threadIdx.x;
    if (k < count) pos[idx[k]] = k;
}

// Duplicate (camera, point) pairs are repeated cameras inside one point's
// observation list; >= 4 per camera, >= 2 per point.
__global__ void k_structure_check(const int* off_cam, int n, const int* off_pt, const int* idx_pt, const int* oc,
                                  int m, Status* st) {
    const int g = blockIdx.x * blockDim.x + threadIdx.x;
    if (g < m) {
        const int b = off_pt[g], e = off_pt[g + 1];
        if (e - b < 2) atomicMin(&st->pt_count_bad, g);
        for (int a = b; a < e; ++a)
            for (int c = a + 1; c < e; ++c)
                if (oc[idx_pt[a]] == oc[idx_pt[c]]) st->dup = 1;
    }
    if (g < n && off_cam[g + 1] - off_cam[g] < 4) atomicMin(&st->cam_count_bad, g);
}

// ---- Jacobian: src/projection.cpp:41-59, 80-105 ----------------------------
__global__ void k_camera_rot(const double* cams, int n, int P, double* R) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    rotation_matrix(cams + (size_t)P * i, R + 9 * (size_t)i);
}

// One thread per observation; writes the AoS record [jc | jp | 0 | tg] (the
// geometry only: it runs while a host scene's σ is still uploading; k_weights
// fills W once σ has arrived).  The CTA's 128
// records are contiguous (by-camera slots): they are assembled in shared
// memory (odd pitch: conflict-free) and written with coalesced 16-byte stores.
template <int P>
__global__ void __launch_bounds__(128, 5) k_jacobian(const double* cams, const double* Rc, const double* pts, const int* oc,
                                                  const int* op, const int* idx_cam, int t_count, double* rec,
                                                  Status* st) {
    constexpr int PITCH = kRec + 1;
    __shared__ double buf[128 * PITCH];
    const int k0 = blockIdx.x * blockDim.x;
    const int k = k0 + threadIdx.x;  // by-camera slot
    if (k < t_count) {
        const int t = idx_cam[k];
        const int ci = oc[t], pj = op[t];
        double jc[2 * P], jp[6], depth;
        const bool ok = observation_jacobian<P>(cams + (size_t)P * ci, Rc + 9 * (size_t)ci, pts + 3 * (size_t)pj, jc, jp, &depth);
        if (!ok) atomicMin(&st->jac_bad, t);
        double* rr = buf + threadIdx.x * PITCH;
        for (int z = 0; z < kRec; ++z) rr[z] = 0.0;  // W (k_weights) stays 0 here
        for (int z = 0; z < 2 * P; ++z) rr[Layout<P>::JC + z] = jc[z];
        for (int z = 0; z < 6; ++z) rr[Layout<P>::JP + z] = jp[z];
        // rotation-rhs factors of this observation (the camera_reduce rhs entries):
        // tg[ii][q] = -((d_C row ii . [C]x col q) + (d_X row ii . [X]x col q))
        double hc[9], hx[9];
        skew(cams + (size_t)P * ci + 3, hc);
        skew(pts + 3 * (size_t)pj, hx);
        for (int ii = 0; ii < 2; ++ii)
            for (int q = 0; q < 3; ++q) {
                const double a = (jc[P * ii + 3] * hc[0 + q] + jc[P * ii + 4] * hc[3 + q]) + jc[P * ii + 5] * hc[6 + q];
                const double bb = (jp[3 * ii + 0] * hx[0 + q] + jp[3 * ii + 1] * hx[3 + q]) + jp[3 * ii + 2] * hx[6 + q];
                rr[Layout<P>::TG + 3 * ii + q] = -(a + bb);
            }
    }
    __syncthreads();
    const int nv = min(128, t_count - k0);
    double2* out = reinterpret_cast<double2*>(rec + (size_t)k0 * kRec);
    for (int w = threadIdx.x; w < nv * (kRec / 2); w += 128) {
        const int o = w / (kRec / 2), part = w - o * (kRec / 2);
        out[w] = make_double2(buf[o * PITCH + 2 * part], buf[o * PITCH + 2 * part + 1]);
    }
}

// W = σ^-1 into each record, the explicit 2x2 inverse (covariance.cpp:20-29),
// and the reference's Fisher-stage check (covariance.cpp:50-53).
__global__ void k_weights(const int* idx_cam, const double* sigma, int t_count, int wo, double* rec, Status* st) {
    const int k = blockIdx.x * blockDim.x + threadIdx.x;
    if (k >= t_count) return;
    const int t = idx_cam[k];
    double s00 = 1.0, s01 = 0.0, s10 = 0.0, s11 = 1.0;
    if (sigma) {
        const double2 a = reinterpret_cast<const double2*>(sigma)[2 * (size_t)t];
        const double2 b = reinterpret_cast<const double2*>(sigma)[2 * (size_t)t + 1];
        s00 = a.x; s01 = a.y; s10 = b.x; s11 = b.y;
    }
    const double det = s00 * s11 - s01 * s10;
    if (!(s00 > 0.0) || !(det > 0.0)) atomicMin(&st->fisher_bad, t);
    double2* w = reinterpret_cast<double2*>(rec + (size_t)k * kRec + wo);
    w[0] = make_double2(s11 / det, -s01 / det);
    w[1] = make_double2(-s10 / det, s00 / det);
}

// Depth of one observation (error message path only).
__global__ void k_depth_of(const double* cams, const double* Rc, const double* pts, const int* oc, const int* op,
                           int P, int t, double* out) {
    const int ci = oc[t], pj = op[t];
    const double* C = cams + (size_t)P * ci + 3;
    const double* R = Rc + 9 * (size_t)ci;
    const double* X = pts + 3 * (size_t)pj;
    const double w[3] = {X[0] - C[0], X[1] - C[1], X[2] - C[2]};
    *out = (R[6] * w[0] + R[7] * w[1]) + R[8] * w[2];
}

// ---- per-camera reduction (warp per camera) -----------------------------------
// D_i = Σ (J_cᵀW)J_c (covariance.cpp:57-63) and the rotation normal equations
// normal = Σ d_rᵀd_r, rhs = Σ d_rᵀ(−(d_C[C]x + d_X[X]x)) (nullspace.cpp:40-50),
// ascending observation order; lane-owned entries keep each sum sequential.
// Then H_r = eig-inverse(normal)·rhs (nullspace.cpp:52-61) and s_a = 1/sqrt(diag D).
template <int P>
__global__ void __launch_bounds__(128) k_camera_reduce(const int* off_cam, const double* rec, int n, double* D,
                                                       double* Hr, double* s_a, unsigned char* flags, Status* st,
                                                       double* raw) {
    // one CTA per camera, one thread per output entry: D (P*P), rotation
    // normal (9) and rhs (9); each entry is a sequential sum over the
    // camera's observations in ascending order.  The camera's records are
    // contiguous (by-camera slots) and staged 32 at a time in shared memory
    // by cp.async, the next chunk in flight while this one is summed; the
    // D-row factors t0, t1 are formed once per (observation, row).
    constexpr int NE = P * P + 18;
    // 48 observations per staged chunk (41 KB of static smem): fewer
    // load / barrier rounds than 32 (config-3 reduce stage 0.516 -> 0.481 ms)
    constexpr int CH = 48, T01 = kRec, RS = T01 + 2 * P;  // RS * 8 B is a multiple of 16
    __shared__ __align__(16) double stage[2][CH][RS];     // double-buffered: chunk c + 1 loads during chunk c
    __shared__ double sh[NE];
    const int i = blockIdx.x;
    const int tid = threadIdx.x;
    // entry decode (fixed per thread).  D entries (kind 0) on threads < P^2;
    // the rotation normal and rhs entries (kinds 1, 2: one formula,
    // jc[p] y1 + jc[P+p] y2) start at the next warp, so no warp runs two code
    // paths (a divergent warp would hold every other warp at the barrier).
    constexpr int B12 = ((P * P + 31) / 32) * 32;
    const int e12 = tid - B12;
    const int kind = tid < P * P ? 0 : ((e12 >= 0 && e12 < 9) ? 1 : ((e12 >= 9 && e12 < 18) ? 2 : 3));
    const int slot = kind == 0 ? tid : P * P + e12;  // entry index in sh[]
    int p = 0, q = 0, i1 = 0, i2 = 0;
    if (kind == 0) { p = tid / P; q = tid % P; }
    else if (kind == 1) { p = e12 / 3; q = e12 % 3; i1 = Layout<P>::JC + q; i2 = Layout<P>::JC + P + q; }
    else if (kind == 2) { p = (e12 - 9) / 3; q = (e12 - 9) % 3; i1 = Layout<P>::TG + q; i2 = Layout<P>::TG + 3 + q; }
    double acc = 0.0;
    const int b = off_cam[i], e = off_cam[i + 1];
    auto load = [&](int buf, int k0) {
        const int nc = min(CH, e - k0);
        for (int w = tid; w < nc * (kRec / 2); w += 128) {
            const int o = w / (kRec / 2), part = w - o * (kRec / 2);
            cpa16(&stage[buf][o][2 * part], rec + (size_t)(k0 + o) * kRec + 2 * part);
        }
    };
    if (b < e) load(0, b);
    cpa_commit();
    for (int k0 = b, c = 0; k0 < e; k0 += CH, ++c) {
        const int nc = min(CH, e - k0);
        const int cur = c & 1;
        if (k0 + CH < e) load(cur ^ 1, k0 + CH);
        cpa_commit();
        cpa_wait<1>();
        __syncthreads();
        // D row factors: t0 = jc_p W00 + jc_P+p W10, t1 = jc_p W01 + jc_P+p W11
        for (int w = tid; w < nc * P; w += 128) {
            const int o = w / P, pp = w - P * o;
            double* r = stage[cur][o];
            const double* jc = r + Layout<P>::JC;
            const double* W = r + Layout<P>::WO;
            r[T01 + 2 * pp] = jc[pp] * W[0] + jc[P + pp] * W[2];
            r[T01 + 2 * pp + 1] = jc[pp] * W[1] + jc[P + pp] * W[3];
        }
        __syncthreads();
        // ordered sums over the chunk; terms of 4 observations are formed
        // independently and added in observation order (bit-identical to a
        // plain sequential loop)
        if (kind == 0) {
            int o = 0;
            for (; o + 4 <= nc; o += 4) {
                double tv[4];
#pragma unroll
                for (int u = 0; u < 4; ++u) {
                    const double* r = stage[cur][o + u];
                    tv[u] = r[T01 + 2 * p] * r[Layout<P>::JC + q] + r[T01 + 2 * p + 1] * r[Layout<P>::JC + P + q];
                }
#pragma unroll
                for (int u = 0; u < 4; ++u) acc += tv[u];
            }
            for (; o < nc; ++o) {
                const double* r = stage[cur][o];
                acc += r[T01 + 2 * p] * r[Layout<P>::JC + q] + r[T01 + 2 * p + 1] * r[Layout<P>::JC + P + q];
            }
        } else if (kind < 3) {
            int o = 0;
            for (; o + 4 <= nc; o += 4) {
                double tv[4];
#pragma unroll
                for (int u = 0; u < 4; ++u) {
                    const double* r = stage[cur][o + u];
                    tv[u] = r[Layout<P>::JC + p] * r[i1] + r[Layout<P>::JC + P + p] * r[i2];
                }
#pragma unroll
                for (int u = 0; u < 4; ++u) acc += tv[u];
            }
            for (; o < nc; ++o) {
                const double* r = stage[cur][o];
                acc += r[Layout<P>::JC + p] * r[i1] + r[Layout<P>::JC + P + p] * r[i2];
            }
        }
        __syncthreads();  // stage[cur] is refilled by the next iteration's prefetch
    }
    if (raw) {  // point-sharded stage A: this rank's partial sums, finished after the all-reduce
        if (kind < 3) raw[(size_t)NE * i + slot] = acc;
        return;
    }
    if (kind < 3) sh[slot] = acc;
    __syncthreads();
    if (tid < P * P) D[(size_t)P * P * i + tid] = acc;
    if (tid < P) {
        const double d = sh[tid * (P + 1)];
        if (d > 0.0) s_a[(size_t)P * i + tid] = 1.0 / sqrt(d);
        else { s_a[(size_t)P * i + tid] = 1.0; flags[(size_t)P * i + tid] = 1; atomicAdd(&st->nflag, 1); }
    }
    if (tid == 0) {
        double inv[9], hr[9];
        if (!eig_inverse3(&sh[P * P], kRotationCondTol, inv)) {
            atomicMin(&st->rot_bad, i);
            for (int k = 0; k < 9; ++k) Hr[9 * (size_t)i + k] = 0.0;
        } else {
            mul3(inv, &sh[P * P + 9], hr);
            for (int k = 0; k < 9; ++k) Hr[9 * (size_t)i + k] = hr[k];
        }
    }
}

// The end of k_camera_reduce from summed partials (point-sharded stage A):
// D, the Jacobi scales of the camera columns and the rotation blocks.
template <int P>
__global__ void k_camera_finish(const double* raw, int n, double* D, double* Hr, double* s_a, unsigned char* flags,
                                Status* st) {
    constexpr int NE = P * P + 18;
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const double* r = raw + (size_t)NE * i;
    for (int e = 0; e < P * P; ++e) D[(size_t)P * P * i + e] = r[e];
    for (int p = 0; p < P; ++p) {
        const double d = r[p * (P + 1)];
        if (d > 0.0) s_a[(size_t)P * i + p] = 1.0 / sqrt(d);
        else { s_a[(size_t)P * i + p] = 1.0; flags[(size_t)P * i + p] = 1; atomicAdd(&st->nflag, 1); }
    }
    double inv[9], hr[9];
    if (!eig_inverse3(r + P * P, kRotationCondTol, inv)) {
        atomicMin(&st->rot_bad, i);
        for (int k = 0; k < 9; ++k) Hr[9 * (size_t)i + k] = 0.0;
    } else {
        mul3(inv, r + P * P + 9, hr);
        for (int k = 0; k < 9; ++k) Hr[9 * (size_t)i + k] = hr[k];
    }
}

// Sums of squares of s_a ∘ h_l over the camera rows (with_cams) and the
// point rows of this (sub-)scene: the point-sharded s_b, finished after the
// all-reduce by k_border_scale.
__global__ void __launch_bounds__(256) k_border_sums(const double* partial, int nblocks, double* sq) {
    __shared__ double red[256][7];
    double acc[7] = {0, 0, 0, 0, 0, 0, 0};
    for (int b = threadIdx.x; b < nblocks; b += 256)
        for (int l = 0; l < 7; ++l) acc[l] += partial[7 * (size_t)b + l];
    for (int l = 0; l < 7; ++l) red[threadIdx.x][l] = acc[l];
    __syncthreads();
    for (int w = 128; w > 0; w >>= 1) {
        if (threadIdx.x < w)
            for (int l = 0; l < 7; ++l) red[threadIdx.x][l] += red[threadIdx.x + w][l];
        __syncthreads();
    }
    if (threadIdx.x < 7) sq[threadIdx.x] = red[0][threadIdx.x];
}
__global__ void k_border_scale(const double* sq, double* s_b) {
    const int l = threadIdx.x;
    if (l >= 7) return;
    const double norm = sqrt(sq[l]);
    s_b[l] = norm > 0.0 ? 1.0 / norm : 1.0;
}

// ---- per-point reduction: A_j = Σ (J_pᵀW)J_p (covariance.cpp:64-71) ---------
template <int P>
__global__ void k_point_reduce(const int* off_pt, const int* idx_pt, const int* pos_cam, const double* rec, int m, int n, double* A,
                               double* s_a, unsigned char* flags, Status* st) {
    const int j = blockIdx.x * blockDim.x + threadIdx.x;
    if (j >= m) return;
    double a[9];
    for (int k = 0; k < 9; ++k) a[k] = 0.0;
    for (int k = off_pt[j]; k < off_pt[j + 1]; ++k) {
        const double* r = rec + (size_t)pos_cam[idx_pt[k]] * kRec;
        const double* jp = r + Layout<P>::JP;
        const double* W = r + Layout<P>::WO;
        for (int p = 0; p < 3; ++p) {
            const double t0 = jp[p] * W[0] + jp[3 + p] * W[2];
            const double t1 = jp[p] * W[1] + jp[3 + p] * W[3];
            for (int q = 0; q < 3; ++q) a[3 * p + q] += t0 * jp[q] + t1 * jp[3 + q];
        }
    }
    for (int k = 0; k < 9; ++k) A[9 * (size_t)j + k] = a[k];
    const size_t base = (size_t)P * n + 3 * (size_t)j;
    for (int p = 0; p < 3; ++p) {
        const double d = a[4 * p];
        if (d > 0.0) s_a[base + p] = 1.0 / sqrt(d);
        else { s_a[base + p] = 1.0; flags[base + p] = 1; atomicAdd(&st->nflag, 1); }
    }
}

// ---- border column scales: s_b[l] = 1/‖s_a ∘ h_l‖ (covariance.cpp:110-114) ----
// Rows of H: camera r-rows (H_r in columns 3..5), camera C-rows [I|[C]x|C],
// zero intrinsic rows, point rows [I|[X]x|X].  Deterministic two-level sum.
template <int P>
__global__ void k_border_partial(const double* cams, const double* Hr, const double* pts, const double* s_a, int n,
                                 int m, double* partial, int with_cams = 1) {
    __shared__ double red[256][7];
    const int g = blockIdx.x * blockDim.x + threadIdx.x;
    double acc[7] = {0, 0, 0, 0, 0, 0, 0};
    if (g < n + m && (with_cams || g >= n)) {
        const bool is_cam = g < n;
        const double* X = is_cam ? cams + (size_t)P * g + 3 : pts + 3 * (size_t)(g - n);
        const size_t row0 = is_cam ? (size_t)P * g + 3 : (size_t)P * n + 3 * (size_t)(g - n);
        double sx[9];
        skew(X, sx);
        for (int a = 0; a < 3; ++a) {
            const double s = s_a[row0 + a];
            double h[7] = {0, 0, 0, 0, 0, 0, 0};
            h[a] = 1.0;
            h[3] = sx[3 * a]; h[4] = sx[3 * a + 1]; h[5] = sx[3 * a + 2];
            h[6] = X[a];
            for (int l = 0; l < 7; ++l) { const double v = s * h[l]; acc[l] += v * v; }
        }
        if (is_cam) {
            for (int a = 0; a < 3; ++a) {
                const double s = s_a[(size_t)P * g + a];
                for (int b = 0; b < 3; ++b) { const double v = s * Hr[9 * (size_t)g + 3 * a + b]; acc[3 + b] += v * v; }
            }
        }
    }
    for (int l = 0; l < 7; ++l) red[threadIdx.x][l] = acc[l];
    __syncthreads();
    for (int w = blockDim.x / 2; w > 0; w >>= 1) {
        if (threadIdx.x < w)
            for (int l = 0; l < 7; ++l) red[threadIdx.x][l] += red[threadIdx.x + w][l];
        __syncthreads();
    }
    if (threadIdx.x == 0)
        for (int l = 0; l < 7; ++l) partial[7 * (size_t)blockIdx.x + l] = red[0][l];
}

__global__ void __launch_bounds__(256) k_border_final(const double* partial, int nblocks, double* s_b) {
    __shared__ double red[256][7];
    double acc[7] = {0, 0, 0, 0, 0, 0, 0};
    for (int b = threadIdx.x; b < nblocks; b += 256)
        for (int l = 0; l < 7; ++l) acc[l] += partial[7 * (size_t)b + l];
    for (int l = 0; l < 7; ++l) red[threadIdx.x][l] = acc[l];
    __syncthreads();
    for (int w = 128; w > 0; w >>= 1) {
        if (threadIdx.x < w)
            for (int l = 0; l < 7; ++l) red[threadIdx.x][l] += red[threadIdx.x + w][l];
        __syncthreads();
    }
    if (threadIdx.x < 7) {
        const double norm = sqrt(red[0][threadIdx.x]);
        s_b[threadIdx.x] = norm > 0.0 ? 1.0 / norm : 1.0;
    }
}

// ---- full H (nullspace API) ---------------------------------------------------
template <int P>
__global__ void k_write_h(const double* cams, const double* Hr, const double* pts, int n, int m, double* H) {
    const int g = blockIdx.x * blockDim.x + threadIdx.x;
    if (g >= n + m) return;
    const bool is_cam = g < n;
    const double* X = is_cam ? cams + (size_t)P * g + 3 : pts + 3 * (size_t)(g - n);
    const size_t row0 = is_cam ? (size_t)P * g + 3 : (size_t)P * n + 3 * (size_t)(g - n);
    double sx[9];
    skew(X, sx);
    for (int a = 0; a < 3; ++a) {
        double* h = H + (row0 + a) * 7;
        for (int l = 0; l < 7; ++l) h[l] = 0.0;
        h[a] = 1.0;
        h[3] = sx[3 * a]; h[4] = sx[3 * a + 1]; h[5] = sx[3 * a + 2];
        h[6] = X[a];
    }
    if (is_cam) {
        for (int a = 0; a < 3; ++a) {
            double* h = H + ((size_t)P * g + a) * 7;
            for (int l = 0; l < 7; ++l) h[l] = 0.0;
            for (int b = 0; b < 3; ++b) h[3 + b] = Hr[9 * (size_t)g + 3 * a + b];
        }
        for (int a = 6; a < P; ++a) {
            double* h = H + ((size_t)P * g + a) * 7;
            for (int l = 0; l < 7; ++l) h[l] = 0.0;
        }
    }
}

// ---- host launchers ------------------------------------------------------------
void launch_status_init(Status* st, cudaStream_t s) { k_status_init<<<1, 1, 0, s>>>(st); SFM_LAUNCH_CHECK(); }

void launch_validate(const SceneDev& sc, int check_sigma, Status* st, cudaStream_t s) {
    if (check_sigma) {
        if (sc.n) { k_validate_cams<<<cdiv(sc.n, 256), 256, 0, s>>>(sc.cams, sc.n, sc.P, st); SFM_LAUNCH_CHECK(); }
        if (sc.m) { k_validate_pts<<<cdiv(sc.m, 256), 256, 0, s>>>(sc.pts, sc.m, st); SFM_LAUNCH_CHECK(); }
    }
    // value checks here unless the scene's covariances are still uploading
    const int values = check_sigma && !sc.sigma_ready;
    if (sc.t) { k_validate_obs<<<cdiv(sc.t, 256), 256, 0, s>>>(sc.oc, sc.op, sc.u, sc.sigma, sc.t, sc.n, sc.m, values, st); SFM_LAUNCH_CHECK(); }
}

void launch_validate_values(const SceneDev& sc, Status* st, cudaStream_t s) {
    if (sc.t) { k_validate_values<<<cdiv(sc.t, 256), 256, 0, s>>>(sc.u, sc.sigma, sc.t, st); SFM_LAUNCH_CHECK(); }
}

static int bits_for(int v) { int b = 1; while ((1LL << b) <= v) ++b; return b; }

// Runs after the index ranges have been validated (every key in range).
void launch_build_index(const SceneDev& sc, IndexDev& ix, Workspace& ws, cudaStream_t s) {
    const int t = sc.t;
    if (t == 0) {
        SFM_CUDA(cudaMemsetAsync(ix.off_cam, 0, sizeof(int) * (size_t)(sc.n + 1), s));
        SFM_CUDA(cudaMemsetAsync(ix.off_pt, 0, sizeof(int) * (size_t)(sc.m + 1), s));
        return;
    }
    size_t bytes = 0;
    cub::DeviceRadixSort::SortPairs(nullptr, bytes, (const int*)nullptr, (int*)nullptr, (const int*)nullptr, (int*)nullptr, t, 0, 32, s);
    void* tmp = ws.get_tmp(bytes);
    int* iota = ix.pos_cam;  // scratch before pos is filled
    k_iota<<<cdiv(t, 256), 256, 0, s>>>(iota, t);
    SFM_LAUNCH_CHECK();
    // stable sorts: ascending observation ids within a camera / point
    size_t bb = bytes;
    SFM_CUDA(cub::DeviceRadixSort::SortPairs(tmp, bb, sc.oc, ix.key_scratch, iota, ix.idx_cam, t, 0, bits_for(sc.n), s));
    k_offsets_from_sorted<<<cdiv(t, 256), 256, 0, s>>>(ix.key_scratch, t, sc.n, ix.off_cam);
    SFM_LAUNCH_CHECK();
    bb = bytes;
    SFM_CUDA(cub::DeviceRadixSort::SortPairs(tmp, bb, sc.op, ix.key_scratch, iota, ix.idx_pt, t, 0, bits_for(sc.m), s));
    k_offsets_from_sorted<<<cdiv(t, 256), 256, 0, s>>>(ix.key_scratch, t, sc.m, ix.off_pt);
    SFM_LAUNCH_CHECK();
    k_pos_scatter<<<cdiv(t, 256), 256, 0, s>>>(ix.idx_cam, t, ix.pos_cam);
    SFM_LAUNCH_CHECK();
}

void launch_structure_check(const SceneDev& sc, const IndexDev& ix, Status* st, cudaStream_t s) {
    const int g = sc.n > sc.m ? sc.n : sc.m;
    if (g) { k_structure_check<<<cdiv(g, 256), 256, 0, s>>>(ix.off_cam, sc.n, ix.off_pt, ix.idx_pt, sc.oc, sc.m, st); SFM_LAUNCH_CHECK(); }
}

void launch_jacobian(const SceneDev& sc, const int* idx_cam, double* R, double* rec, Status* st, cudaStream_t s) {
    if (sc.n) { k_camera_rot<<<cdiv(sc.n, 128), 128, 0, s>>>(sc.cams, sc.n, sc.P, R); SFM_LAUNCH_CHECK(); }
    if (sc.t) {
        if (sc.P == 8) k_jacobian<8><<<cdiv(sc.t, 128), 128, 0, s>>>(sc.cams, R, sc.pts, sc.oc, sc.op, idx_cam, sc.t, rec, st);
        else k_jacobian<9><<<cdiv(sc.t, 128), 128, 0, s>>>(sc.cams, R, sc.pts, sc.oc, sc.op, idx_cam, sc.t, rec, st);
        SFM_LAUNCH_CHECK();
    }
}

void launch_weights(const SceneDev& sc, const int* idx_cam, double* rec, Status* st, cudaStream_t s) {
    if (!sc.t) return;
    const int wo = sc.P == 8 ? Layout<8>::WO : Layout<9>::WO;
    k_weights<<<cdiv(sc.t, 256), 256, 0, s>>>(idx_cam, sc.sigma, sc.t, wo, rec, st);
    SFM_LAUNCH_CHECK();
}

void launch_depth_of(const SceneDev& sc, const double* R, int t, double* out, cudaStream_t s) {
    k_depth_of<<<1, 1, 0, s>>>(sc.cams, R, sc.pts, sc.oc, sc.op, sc.P, t, out);
    SFM_LAUNCH_CHECK();
}

// The per-camera reduction (one CTA per camera, a sequential chain over its
// observations) leaves most of each SM idle, so the independent per-point
// reduction runs beside it on `side` (fork / join through the two events).
void launch_reductions(const SceneDev& sc, const IndexDev& ix, const double* rec, double* D, double* Hr, double* A,
                       double* s_a, unsigned char* flags, Status* st, cudaStream_t s, cudaStream_t side,
                       cudaEvent_t fork, cudaEvent_t join, double* raw) {
    const size_t ncols = (size_t)sc.P * sc.n + 3 * (size_t)sc.m;
    SFM_CUDA(cudaMemsetAsync(flags, 0, ncols, s));
    SFM_CUDA(cudaEventRecord(fork, s));
    SFM_CUDA(cudaStreamWaitEvent(side, fork, 0));
    if (sc.m) {
        if (sc.P == 8) k_point_reduce<8><<<cdiv(sc.m, 128), 128, 0, side>>>(ix.off_pt, ix.idx_pt, ix.pos_cam, rec, sc.m, sc.n, A, s_a, flags, st);
        else k_point_reduce<9><<<cdiv(sc.m, 128), 128, 0, side>>>(ix.off_pt, ix.idx_pt, ix.pos_cam, rec, sc.m, sc.n, A, s_a, flags, st);
        SFM_LAUNCH_CHECK();
    }
    SFM_CUDA(cudaEventRecord(join, side));
    if (sc.n) {
        if (sc.P == 8) k_camera_reduce<8><<<sc.n, 128, 0, s>>>(ix.off_cam, rec, sc.n, D, Hr, s_a, flags, st, raw);
        else k_camera_reduce<9><<<sc.n, 128, 0, s>>>(ix.off_cam, rec, sc.n, D, Hr, s_a, flags, st, raw);
        SFM_LAUNCH_CHECK();
    }
    SFM_CUDA(cudaStreamWaitEvent(s, join, 0));
}

void launch_border_scales(const SceneDev& sc, const double* Hr, const double* s_a, double* partial, double* s_b,
                          cudaStream_t s) {
    const int g = sc.n + sc.m;
    const int nb = (int)cdiv(g > 0 ? g : 1, 256);
    if (sc.P == 8) k_border_partial<8><<<nb, 256, 0, s>>>(sc.cams, Hr, sc.pts, s_a, sc.n, sc.m, partial);
    else k_border_partial<9><<<nb, 256, 0, s>>>(sc.cams, Hr, sc.pts, s_a, sc.n, sc.m, partial);
    SFM_LAUNCH_CHECK();
    k_border_final<<<1, 256, 0, s>>>(partial, nb, s_b);
    SFM_LAUNCH_CHECK();
}

void launch_camera_finish(int P, const double* raw, int n, double* D, double* Hr, double* s_a, unsigned char* flags,
                          Status* st, cudaStream_t s) {
    if (!n) return;
    if (P == 8) k_camera_finish<8><<<cdiv(n, 128), 128, 0, s>>>(raw, n, D, Hr, s_a, flags, st);
    else k_camera_finish<9><<<cdiv(n, 128), 128, 0, s>>>(raw, n, D, Hr, s_a, flags, st);
    SFM_LAUNCH_CHECK();
}

void launch_border_sums(const SceneDev& sc, const double* Hr, const double* s_a, int with_cams, double* partial,
                        double* sq, cudaStream_t s) {
    const int g = sc.n + sc.m;
    const int nb = (int)cdiv(g > 0 ? g : 1, 256);
    if (sc.P == 8) k_border_partial<8><<<nb, 256, 0, s>>>(sc.cams, Hr, sc.pts, s_a, sc.n, sc.m, partial, with_cams);
    else k_border_partial<9><<<nb, 256, 0, s>>>(sc.cams, Hr, sc.pts, s_a, sc.n, sc.m, partial, with_cams);
    SFM_LAUNCH_CHECK();
    k_border_sums<<<1, 256, 0, s>>>(partial, nb, sq);
    SFM_LAUNCH_CHECK();
}

void launch_border_scale(const double* sq, double* s_b, cudaStream_t s) {
    k_border_scale<<<1, 32, 0, s>>>(sq, s_b);
    SFM_LAUNCH_CHECK();
}

int border_partial_blocks(int n, int m) { const int g = n + m; return (int)cdiv(g > 0 ? g : 1, 256); }

void launch_write_h(const SceneDev& sc, const double* Hr, double* H, cudaStream_t s) {
    const int g = sc.n + sc.m;
    if (!g) return;
    if (sc.P == 8) k_write_h<8><<<cdiv(g, 128), 128, 0, s>>>(sc.cams, Hr, sc.pts, sc.n, sc.m, H);
    else k_write_h<9><<<cdiv(g, 128), 128, 0, s>>>(sc.cams, Hr, sc.pts, sc.n, sc.m, H);
    SFM_LAUNCH_CHECK();
}

}  // namespace sfm
