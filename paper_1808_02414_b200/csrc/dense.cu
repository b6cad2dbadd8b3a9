// Stage (d): gauge-fixed inversion of the reduced camera system.
//
// Replaces invert_schur + extract_camera_covariances (src/covariance.cpp:
// 196-279: Bunch–Kaufman dsytrf + dsytrs2 against I on the bordered matrix,
// N^3/3 + 2N^3 flops) by the equivalent SPD route on Z_aug = Z - Γ E^-1 Γ^T
// (SURVEY.md appendix A): blocked right-looking Cholesky (N^3/3), blocked
// triangular inverse X = L^-1 (N^3/3), and the diagonal camera blocks
// Σ_ii = Σ_k X_ki^T X_ki, unscaled by the Jacobi scales.
//
// All trailing updates go through one FP64 tensor-core GEMM
// (mma.sync m8n8k4 f64 -> SASS DMMA; sm_100a has no tcgen05 kind::f64):
//     C = beta * C + alpha * A * B^T,   K = kNB = 128, alpha = +-1
// CTA tile 128x128, 16 warps of 32x32, 3-stage cp.async pipeline over K.
// The accumulator fragment is laid out so each lane owns two consecutive
// rows of one column: C tiles move with 16-byte loads/stores.
#include "common.cuh"
#include "detmath.cuh"
#include "kernels.cuh"

namespace sfm {

// ----------------------------------------------------------------------------
// DMMA GEMM
// ----------------------------------------------------------------------------
namespace gemm {
constexpr int BM = 128, BN = 128, BK = 16, STAGES = 3, PAD = 8, LDS = BM + PAD;
constexpr int LDB_K = BK + 4;  // K-major B tile pitch (conflict-free fragment reads)
constexpr int THREADS = 512;
constexpr int SMEM = STAGES * (BK * LDS + BN * LDB_K) * 8;  // 113664 B
}  // namespace gemm

__device__ __forceinline__ void cp_async16(void* smem, const void* gmem) {
    const unsigned s = (unsigned)__cvta_generic_to_shared(smem);
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(s), "l"(gmem));
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::); }
template <int N>
__device__ __forceinline__ void cp_async_wait() { asm volatile("cp.async.wait_group %0;\n" ::"n"(N)); }

__device__ __forceinline__ void dmma(double& d0, double& d1, double a, double b) {
    asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                 : "+d"(d0), "+d"(d1)
                 : "d"(a), "d"(b));
}

// C[m, n] = beta C[m, n] + alpha Σ_k A[m, k] B[n, k]
//   A: element (m, k) at A[k * lda + m]                      (M-contiguous)
//   B: BK_MAJOR = false: (n, k) at B[k * ldb + n]            (N-contiguous)
//      BK_MAJOR = true : (n, k) at B[n * ldb + k]            (K-contiguous)
// MMA mapping: the m8n8k4 "A" operand carries B rows (n), its "B" operand
// carries A rows (m), so each lane's two accumulators are C rows
// m0 + 2(lane&3) + {0,1} of column n0 + (lane>>2): 16-byte C accesses.
template <bool BK_MAJOR>
__global__ void __launch_bounds__(gemm::THREADS, 1) k_gemm(GemmArgs g) {
    using namespace gemm;
    extern __shared__ __align__(16) double smem[];
    double* As = smem;                      // [STAGES][BK][LDS]
    double* Bs = smem + STAGES * BK * LDS;  // [STAGES][BK][LDS] or [STAGES][BN][LDB_K]
    constexpr int BSTAGE = BK_MAJOR ? BN * LDB_K : BK * LDS;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    int ti, tj;
    const long long l = blockIdx.x;
    if (g.tri) {
        int t = (int)((sqrt(8.0 * (double)l + 1.0) - 1.0) * 0.5);
        while ((long long)(t + 1) * (t + 2) / 2 <= l) ++t;
        while ((long long)t * (t + 1) / 2 > l) --t;
        ti = t;
        tj = (int)(l - (long long)t * (t + 1) / 2);
    } else {
        ti = (int)(l % g.tm);
        tj = (int)(l / g.tm);
    }
    const double* A = g.A + (size_t)ti * BM;
    const double* B = BK_MAJOR ? g.B + (size_t)tj * BN * g.ldb : g.B + (size_t)tj * BN;
    double* C = g.C + (size_t)tj * BN * g.ldc + (size_t)ti * BM;
    const int wm = warp & 3, wn = warp >> 2;  // 4 x 4 warps of 32 x 32
    const int beta = (g.beta && tj != g.beta0_tile) ? 1 : 0;

    auto load_stage = [&](int st, int kc) {
        double* as = As + st * BK * LDS;
        double* bs = Bs + st * BSTAGE;
#pragma unroll
        for (int u = 0; u < 2; ++u) {
            const int idx = tid + THREADS * u;  // 0..1023
            {
                const int k = idx >> 6, m2 = (idx & 63) * 2;
                cp_async16(as + k * LDS + m2, A + (size_t)(kc * BK + k) * g.lda + m2);
            }
            if (BK_MAJOR) {
                const int n = idx >> 3, k2 = (idx & 7) * 2;
                cp_async16(bs + n * LDB_K + k2, B + (size_t)n * g.ldb + kc * BK + k2);
            } else {
                const int k = idx >> 6, n2 = (idx & 63) * 2;
                cp_async16(bs + k * LDS + n2, B + (size_t)(kc * BK + k) * g.ldb + n2);
            }
        }
    };

    constexpr int NK = kNB / BK;  // 8
    load_stage(0, 0);
    cp_async_commit();
    load_stage(1, 1);
    cp_async_commit();

    double acc[4][4][2];
    const int rq = 2 * (lane & 3), cq = lane >> 2;
#pragma unroll
    for (int mi = 0; mi < 4; ++mi)
#pragma unroll
        for (int ni = 0; ni < 4; ++ni) {
            if (beta) {
                const double2 c = *reinterpret_cast<const double2*>(C + (size_t)(wn * 32 + ni * 8 + cq) * g.ldc + wm * 32 + mi * 8 + rq);
                acc[mi][ni][0] = c.x;
                acc[mi][ni][1] = c.y;
            } else {
                acc[mi][ni][0] = 0.0;
                acc[mi][ni][1] = 0.0;
            }
        }
    const double sgn = g.alpha_neg ? -1.0 : 1.0;

#pragma unroll 1
    for (int kc = 0; kc < NK; ++kc) {
        cp_async_wait<1>();
        __syncthreads();
        if (kc + 2 < NK) load_stage((kc + 2) % STAGES, kc + 2);
        cp_async_commit();
        const double* as = As + (kc % STAGES) * BK * LDS;
        const double* bs = Bs + (kc % STAGES) * BSTAGE;
#pragma unroll
        for (int kk = 0; kk < BK / 4; ++kk) {
            const int krow = kk * 4 + (lane & 3);
            double af[4], bf[4];
#pragma unroll
            for (int mi = 0; mi < 4; ++mi) af[mi] = sgn * as[krow * LDS + wm * 32 + mi * 8 + cq];
#pragma unroll
            for (int ni = 0; ni < 4; ++ni)
                bf[ni] = BK_MAJOR ? bs[(wn * 32 + ni * 8 + cq) * LDB_K + krow] : bs[krow * LDS + wn * 32 + ni * 8 + cq];
#pragma unroll
            for (int mi = 0; mi < 4; ++mi)
#pragma unroll
                for (int ni = 0; ni < 4; ++ni) dmma(acc[mi][ni][0], acc[mi][ni][1], bf[ni], af[mi]);
        }
    }
#pragma unroll
    for (int mi = 0; mi < 4; ++mi)
#pragma unroll
        for (int ni = 0; ni < 4; ++ni) {
            double2 c;
            c.x = acc[mi][ni][0];
            c.y = acc[mi][ni][1];
            *reinterpret_cast<double2*>(C + (size_t)(wn * 32 + ni * 8 + cq) * g.ldc + wm * 32 + mi * 8 + rq) = c;
        }
}

void launch_gemm(const GemmArgs& g, cudaStream_t s) {
    const long long tiles = g.tri ? (long long)g.tm * (g.tm + 1) / 2 : (long long)g.tm * g.tn;
    if (tiles <= 0) return;
    static bool attr = false;
    if (!attr) {
        SFM_CUDA(cudaFuncSetAttribute(k_gemm<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, gemm::SMEM));
        SFM_CUDA(cudaFuncSetAttribute(k_gemm<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, gemm::SMEM));
        attr = true;
    }
    if (g.b_kmajor) k_gemm<true><<<(unsigned)tiles, gemm::THREADS, gemm::SMEM, s>>>(g);
    else k_gemm<false><<<(unsigned)tiles, gemm::THREADS, gemm::SMEM, s>>>(g);
    SFM_LAUNCH_CHECK();
}

// ----------------------------------------------------------------------------
// Diagonal tile: Cholesky + triangular inverse of one kNB x kNB tile in smem.
// ----------------------------------------------------------------------------
namespace potrf {
constexpr int LDT = kNB + 1;
constexpr int THREADS = 512;
constexpr int SMEM = (kNB * LDT + kNB) * 8;
}  // namespace potrf

// A: tile (k0, k0) of the matrix (col-major, ld).  Writes L (lower) back,
// Linv (kNB x kNB col-major, zeros above), pivots[col0 + j] = L_jj^2.
__global__ void __launch_bounds__(potrf::THREADS, 1) k_potrf_diag(double* A, long long ld, double* Linv, double* pivots,
                                                                 int col0, Status* st) {
    using namespace potrf;
    extern __shared__ double T[];  // T[c * LDT + r]
    double* col = T + kNB * LDT;
    const int tid = threadIdx.x;
    for (int e = tid; e < kNB * kNB; e += THREADS) {
        const int r = e & (kNB - 1), c = e >> 7;
        T[c * LDT + r] = (r >= c) ? A[(size_t)c * ld + r] : 0.0;
    }
    __syncthreads();
    // right-looking unblocked Cholesky
    for (int j = 0; j < kNB; ++j) {
        if (tid == 0) {
            double d = T[j * LDT + j];
            pivots[col0 + j] = d;
            if (!(d > 0.0) || !isfinite(d)) {
                atomicMin(&st->chol_bad, col0 + j);
                d = 1.0;
            }
            T[j * LDT + j] = sqrt(d);
        }
        __syncthreads();
        const double ljj = T[j * LDT + j];
        for (int i = j + 1 + tid; i < kNB; i += THREADS) T[j * LDT + i] = T[j * LDT + i] / ljj;
        __syncthreads();
        const int warp = tid >> 5, lane = tid & 31;
        for (int c = j + 1 + warp; c < kNB; c += THREADS / 32) {
            const double lcj = T[j * LDT + c];
            for (int i = c + lane; i < kNB; i += 32) T[c * LDT + i] -= T[j * LDT + i] * lcj;
        }
        __syncthreads();
    }
    for (int e = tid; e < kNB * kNB; e += THREADS) {
        const int r = e & (kNB - 1), c = e >> 7;
        if (r >= c) A[(size_t)c * ld + r] = T[c * LDT + r];
    }
    // in-place inverse: solve L X = I, right-looking; X(i,c) for c <= j
    // overwrites L(i,c) once column c of L is consumed.
    for (int j = 0; j < kNB; ++j) {
        // copy column j of L (rows >= j) before it is overwritten
        for (int i = j + tid; i < kNB; i += THREADS) col[i] = T[j * LDT + i];
        __syncthreads();
        const double ljj = col[j];
        // row j of X: X(j, c) = X(j, c) / ljj for c < j; X(j, j) = 1 / ljj
        for (int c = tid; c <= j; c += THREADS) T[c * LDT + j] = (c == j) ? 1.0 / ljj : T[c * LDT + j] / ljj;
        __syncthreads();
        // X(i, c) -= L(i, j) X(j, c), i > j, c <= j (X(i, j) starts at 0)
        const int rows = kNB - 1 - j;
        const int cols = j + 1;
        for (int e = tid; e < rows * cols; e += THREADS) {
            const int i = j + 1 + e % rows, c = e / rows;
            const double base = (c == j) ? 0.0 : T[c * LDT + i];
            T[c * LDT + i] = base - col[i] * T[c * LDT + j];
        }
        __syncthreads();
    }
    for (int e = tid; e < kNB * kNB; e += THREADS) {
        const int r = e & (kNB - 1), c = e >> 7;
        Linv[(size_t)c * kNB + r] = (r >= c) ? T[c * LDT + r] : 0.0;
    }
}

void launch_potrf_diag(double* A, long long ld, double* Linv, double* pivots, int col0, Status* st, cudaStream_t s) {
    static bool attr = false;
    if (!attr) {
        SFM_CUDA(cudaFuncSetAttribute(k_potrf_diag, cudaFuncAttributeMaxDynamicSharedMemorySize, potrf::SMEM));
        attr = true;
    }
    k_potrf_diag<<<1, potrf::THREADS, potrf::SMEM, s>>>(A, ld, Linv, pivots, col0, st);
    SFM_LAUNCH_CHECK();
}

// ----------------------------------------------------------------------------
// Triangular inverse helpers (forward substitution X = L^-1, in place).
// ----------------------------------------------------------------------------
// X[k, k] = Linv_k (full tile, zeros above the diagonal).
__global__ void k_copy_diag(double* X, long long ld, int k, const double* Linv) {
    const int e = blockIdx.x * blockDim.x + threadIdx.x;
    if (e >= kNB * kNB) return;
    const int r = e & (kNB - 1), c = e >> 7;
    X[(size_t)(k * kNB + c) * ld + (size_t)k * kNB + r] = Linv[(size_t)c * kNB + r];
}

void launch_copy_diag(double* X, long long ld, int k, const double* Linv, cudaStream_t s) {
    k_copy_diag<<<kNB * kNB / 256, 256, 0, s>>>(X, ld, k, Linv);
    SFM_LAUNCH_CHECK();
}

// Copy the L panel below the diagonal block k into a contiguous buffer.
__global__ void k_copy_panel(const double* X, long long ld, int k, int rows, double* Lp) {
    const long long e = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    const long long total = (long long)rows * kNB;
    if (e >= total) return;
    const int r = (int)(e % rows), c = (int)(e / rows);
    Lp[(size_t)c * rows + r] = X[(size_t)(k * kNB + c) * ld + (size_t)(k + 1) * kNB + r];
}

void launch_copy_panel(const double* X, long long ld, int k, int rows, double* Lp, cudaStream_t s) {
    const long long total = (long long)rows * kNB;
    if (!total) return;
    k_copy_panel<<<cdiv(total, 256), 256, 0, s>>>(X, ld, k, rows, Lp);
    SFM_LAUNCH_CHECK();
}

// ----------------------------------------------------------------------------
// Diagonal blocks of Z^-1 = X^T X (X = L^-1 lower), unscaled + PSD check.
// One CTA (8 warps) per camera; each lane accumulates the P(P+1)/2 unique
// products over a strided set of rows, then a fixed-order tree reduction.
// ----------------------------------------------------------------------------
template <int P>
__global__ void __launch_bounds__(256) k_extract(const double* X, long long ld, int N, const double* s_a, int scale,
                                                 double* cov, Status* st, int* psd_warn) {
    constexpr int U = P * (P + 1) / 2;
    __shared__ double red[8][U];
    const int i = blockIdx.x;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int c0 = P * i;
    double acc[U];
#pragma unroll
    for (int u = 0; u < U; ++u) acc[u] = 0.0;
    for (int r = c0 + threadIdx.x; r < N; r += 256) {
        double x[P];
#pragma unroll
        for (int p = 0; p < P; ++p) x[p] = (r >= c0 + p) ? X[(size_t)(c0 + p) * ld + r] : 0.0;
        int u = 0;
#pragma unroll
        for (int p = 0; p < P; ++p)
#pragma unroll
            for (int q = p; q < P; ++q, ++u) acc[u] += x[p] * x[q];
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
        double v = acc[u];
        for (int o = 16; o > 0; o >>= 1) v += __shfl_down_sync(0xffffffffu, v, o);
        if (lane == 0) red[warp][u] = v;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        double b[P * P];
        int u = 0;
        for (int p = 0; p < P; ++p)
            for (int q = p; q < P; ++q, ++u) {
                double v = 0.0;
                for (int w = 0; w < 8; ++w) v += red[w][u];
                b[P * p + q] = v;
                b[P * q + p] = v;
            }
        double out[P * P];
        for (int p = 0; p < P; ++p)
            for (int q = 0; q < P; ++q) {
                const double sp = scale ? s_a[c0 + p] : 1.0, sq = scale ? s_a[c0 + q] : 1.0;
                out[P * p + q] = (sp * b[P * p + q]) * sq;
            }
        double* o = cov + (size_t)P * P * i;
        for (int k = 0; k < P * P; ++k) o[k] = out[k];
        double a[P * P], d[P], v[P * P];
        for (int k = 0; k < P * P; ++k) a[k] = out[k];
        jacobi_eig<P>(a, d, v);
        double tr = 0.0, lmin = d[0];
        for (int p = 0; p < P; ++p) { tr += out[P * p + p]; lmin = fmin(lmin, d[p]); }
        if (lmin < -kPsdTol * tr) atomicAdd(psd_warn, 1);
    }
}

void launch_extract(int P, const double* X, long long ld, int N, int nblocks, const double* s_a, int scale, double* cov,
                    Status* st, int* psd_warn, cudaStream_t s) {
    if (!nblocks) return;
    if (P == 8) k_extract<8><<<nblocks, 256, 0, s>>>(X, ld, N, s_a, scale, cov, st, psd_warn);
    else if (P == 9) k_extract<9><<<nblocks, 256, 0, s>>>(X, ld, N, s_a, scale, cov, st, psd_warn);
    else throw CudaError("extract: unsupported block size");
    SFM_LAUNCH_CHECK();
}

// Pivot range of the Cholesky (first N pivots) on device.
__global__ void k_pivot_range(const double* piv, int N, double* out) {
    __shared__ double mn[256], mx[256];
    double a = INFINITY, b = 0.0;
    for (int i = threadIdx.x; i < N; i += 256) { const double v = fabs(piv[i]); a = fmin(a, v); b = fmax(b, v); }
    mn[threadIdx.x] = a; mx[threadIdx.x] = b;
    __syncthreads();
    for (int w = 128; w > 0; w >>= 1) {
        if (threadIdx.x < w) { mn[threadIdx.x] = fmin(mn[threadIdx.x], mn[threadIdx.x + w]); mx[threadIdx.x] = fmax(mx[threadIdx.x], mx[threadIdx.x + w]); }
        __syncthreads();
    }
    if (threadIdx.x == 0) { out[0] = mn[0]; out[1] = mx[0]; }
}

void launch_pivot_range(const double* piv, int N, double* out, cudaStream_t s) {
    k_pivot_range<<<1, 256, 0, s>>>(piv, N, out);
    SFM_LAUNCH_CHECK();
}

// ----------------------------------------------------------------------------
// Drivers
// ----------------------------------------------------------------------------
// Blocked right-looking Cholesky of the Npad x Npad lower triangle (Npad =
// K kNB) with one-panel lookahead.  Step k on stream s: potrf(k), trsm(k)
// [L21 = A21 Linv_k^T], then the next panel column's update; the rest of the
// trailing SYRK (columns >= k+2) runs on s2 and overlaps potrf/trsm of step
// k+1.  Ordering: rest(k) waits trsm(k) (e1); next-panel(k) waits rest(k-1)
// (e2), since both update column block k+1.
int dense_cholesky(double* Z, long long ld, int Npad, double* Linv, double* pivots, Status* st, cudaStream_t s,
                   cudaStream_t s2, cudaEvent_t e1, cudaEvent_t e2) {
    const int K = Npad / kNB;
    int launches = 0;
    bool rest_pending = false;
    for (int k = 0; k < K; ++k) {
        double* Akk = Z + (size_t)k * kNB * ld + (size_t)k * kNB;
        launch_potrf_diag(Akk, ld, Linv + (size_t)k * kNB * kNB, pivots, k * kNB, st, s);
        ++launches;
        const int rows = Npad - (k + 1) * kNB;
        if (rows == 0) break;
        double* panel = Akk + kNB;
        GemmArgs t{};
        t.C = panel; t.ldc = ld; t.A = panel; t.lda = ld; t.B = Linv + (size_t)k * kNB * kNB; t.ldb = kNB;
        t.tm = rows / kNB; t.tn = 1; t.beta0_tile = -1;
        launch_gemm(t, s);
        ++launches;
        const int T2 = rows / kNB;
        if (T2 > 1) {
            SFM_CUDA(cudaEventRecord(e1, s));
            SFM_CUDA(cudaStreamWaitEvent(s2, e1, 0));
            GemmArgs r{};
            r.C = Z + (size_t)(k + 2) * kNB * ld + (size_t)(k + 2) * kNB; r.ldc = ld;
            r.A = panel + kNB; r.lda = ld; r.B = panel + kNB; r.ldb = ld;
            r.tm = T2 - 1; r.tn = T2 - 1; r.tri = 1; r.alpha_neg = 1; r.beta = 1; r.beta0_tile = -1;
            launch_gemm(r, s2);
            ++launches;
        }
        if (rest_pending) SFM_CUDA(cudaStreamWaitEvent(s, e2, 0));
        GemmArgs u{};
        u.C = Z + (size_t)(k + 1) * kNB * ld + (size_t)(k + 1) * kNB; u.ldc = ld;
        u.A = panel; u.lda = ld; u.B = panel; u.ldb = ld;
        u.tm = T2; u.tn = 1; u.alpha_neg = 1; u.beta = 1; u.beta0_tile = -1;
        launch_gemm(u, s);
        ++launches;
        rest_pending = false;
        if (T2 > 1) {
            SFM_CUDA(cudaEventRecord(e2, s2));
            rest_pending = true;
        }
    }
    if (rest_pending) SFM_CUDA(cudaStreamWaitEvent(s, e2, 0));
    return launches;
}

// Blocked triangular inverse X = L^-1 in place (forward substitution by row
// blocks), with the same lookahead split.  Step k:
//   (1) X[k, 0:k] = Linv_k X[k, 0:k] (GEMM, B K-major), X[k, k] = Linv_k
//   (2) Lp = L[k+1:, k] (copy; column block k is overwritten below)
//   (3) X[k+1:, 0:k+1] -= Lp X[k, 0:k+1]   (column block k with beta = 0)
// (3) is split into row block k+1 (stream s, feeds step k+1) and the rest
// (stream s2).
int dense_trtri(double* X, long long ld, int Npad, const double* Linv, double* Lp, cudaStream_t s, cudaStream_t s2,
                cudaEvent_t e1, cudaEvent_t e2) {
    const int K = Npad / kNB;
    int launches = 0;
    bool rest_pending = false;
    for (int k = 0; k < K; ++k) {
        const double* Lk = Linv + (size_t)k * kNB * kNB;
        if (k > 0) {
            GemmArgs g{};
            g.C = X + (size_t)k * kNB; g.ldc = ld;
            g.A = Lk; g.lda = kNB;
            g.B = X + (size_t)k * kNB; g.ldb = ld; g.b_kmajor = 1;
            g.tm = 1; g.tn = k; g.beta0_tile = -1;
            launch_gemm(g, s);
            ++launches;
        }
        launch_copy_diag(X, ld, k, Lk, s);
        ++launches;
        const int rows = Npad - (k + 1) * kNB;
        if (rows == 0) break;
        // Lp must not be overwritten while rest(k-1) on s2 still reads it
        if (rest_pending) SFM_CUDA(cudaStreamWaitEvent(s, e2, 0));
        rest_pending = false;
        launch_copy_panel(X, ld, k, rows, Lp + (size_t)(k & 1) * (size_t)Npad * kNB, s);
        ++launches;
        const double* lp = Lp + (size_t)(k & 1) * (size_t)Npad * kNB;
        const int T2 = rows / kNB;
        GemmArgs a{};
        a.C = X + (size_t)(k + 1) * kNB; a.ldc = ld;
        a.A = lp; a.lda = rows;
        a.B = X + (size_t)k * kNB; a.ldb = ld; a.b_kmajor = 1;
        a.tm = 1; a.tn = k + 1; a.alpha_neg = 1; a.beta = 1; a.beta0_tile = k;
        if (T2 > 1) {
            SFM_CUDA(cudaEventRecord(e1, s));
            SFM_CUDA(cudaStreamWaitEvent(s2, e1, 0));
            GemmArgs r = a;
            r.C = X + (size_t)(k + 2) * kNB;
            r.A = lp + kNB;
            r.tm = T2 - 1;
            launch_gemm(r, s2);
            ++launches;
            SFM_CUDA(cudaEventRecord(e2, s2));
            rest_pending = true;
        }
        launch_gemm(a, s);
        ++launches;
    }
    if (rest_pending) SFM_CUDA(cudaStreamWaitEvent(s, e2, 0));
    return launches;
}

}  // namespace sfm
