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
#include <cstdio>
#include <cstdlib>
#include <utility>
#include <vector>

#include "common.cuh"
#include "detmath.cuh"
#include "kernels.cuh"

namespace sfm {

const void* k_potrf_diag_ptr();
int potrf_smem_bytes_impl();
static inline const void* k_potrf_diag_fwd() { return k_potrf_diag_ptr(); }
static inline int potrf_smem_bytes() { return potrf_smem_bytes_impl(); }

// ----------------------------------------------------------------------------
// DMMA GEMM
// ----------------------------------------------------------------------------
namespace gemm {
// PAD: pitch 64 + 4 doubles keeps a half-warp's FP64 fragment reads (rows g,
// k = t + 4 i: bank pairs 8 t + g) conflict-free and a 3-stage 64 x 64 CTA at
// <= 56 KB, so that four fit an SM; pitch + 8 (round 1) was 2-way conflicted
// and, with the stage size taken as the larger of the two B layouts, 57 KB:
// three CTAs per SM (ncu: 12 warps active), not the four intended.  Measured
// equal in the sweep and per launch (31.2-31.4 TF/s for the bulk updates with
// three or four resident CTAs): the kernel is not occupancy-bound.
#ifndef SFM_GEMM_REGS
#define SFM_GEMM_REGS 128  // register budget per thread behind the launch bounds (A/B builds: 168 = three 64 x 64 CTAs per SM)
#endif
#ifndef SFM_GEMM_PAD
#define SFM_GEMM_PAD 4
#endif
constexpr int BM = 128, BN = 128, PAD = SFM_GEMM_PAD, LDS = BM + PAD;
// CTA tile CM x CN of (CM/32) x (CN/32) warps of 32 x 32; the grid
// enumerates 128 x 128 tiles x (128/CM)(128/CN) CTAs.  Used: 64 x 64 (four
// CTAs per SM: independent output tiles), 128 x 64 (two per SM; C aliasing
// B: a CTA must own all rows of its columns -- 128 x 32 measured slower),
// 128 x 128 (whole_tile: C aliasing A).
template <int BK, int STAGES, int CM, int CN>
struct Cfg {
    static constexpr int THREADS = (CM / 32) * (CN / 32) * 32;
    static constexpr int BMC = CM;           // CTA rows
    static constexpr int LDSA = BMC + PAD;   // M-contiguous A tile pitch
    static constexpr int BNT = CN;           // CTA columns
    static constexpr int LDSB = BNT + PAD;   // N-contiguous B tile pitch
    static constexpr int LDB_K = BK + 4;     // K-major B tile pitch (conflict-free fragment reads)
    static constexpr int BSTAGE_N = BK * LDSB, BSTAGE_K = BNT * LDB_K;
    static constexpr int ASTAGE_M = BK * LDSA, ASTAGE_K = BMC * LDB_K;  // A: M- or K-contiguous
    static constexpr int BSTAGE = BSTAGE_N > BSTAGE_K ? BSTAGE_N : BSTAGE_K;
    static constexpr int SMEM = STAGES * (ASTAGE_M + BSTAGE) * 8;     // A M-contiguous (upper bound over B layouts)
    static constexpr int SMEM_AK = STAGES * (ASTAGE_K + BSTAGE) * 8;  // A K-contiguous
    // the exact size per B layout: what a launch asks for (occupancy)
    static constexpr int smem(bool b_kmajor) { return STAGES * (ASTAGE_M + (b_kmajor ? BSTAGE_K : BSTAGE_N)) * 8; }
};
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
// Warps of 32x32, STAGES-deep cp.async pipeline of BK-wide K chunks.
__device__ __forceinline__ void dmma16(double& d0, double& d1, double& d2, double& d3, const double* a,
                                       const double* b) {
    asm volatile(
        "mma.sync.aligned.m16n8k16.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5,%6,%7,%8,%9,%10,%11}, "
        "{%12,%13,%14,%15}, {%0,%1,%2,%3};\n"
        : "+d"(d0), "+d"(d1), "+d"(d2), "+d"(d3)
        : "d"(a[0]), "d"(a[1]), "d"(a[2]), "d"(a[3]), "d"(a[4]), "d"(a[5]), "d"(a[6]), "d"(a[7]), "d"(b[0]),
          "d"(b[1]), "d"(b[2]), "d"(b[3]));
}

// M16: the 32 x 32 warp tile as 2 x 4 m16n8k16 MMAs per 16-deep chunk (8
// instructions) instead of 4 x 4 m8n8k4 MMAs per 4-deep step (64); same
// shared-memory loads, same accumulator -> C mapping (fragment layouts:
// tools/probe/dmma16_layout.cu).
template <bool BK_MAJOR, int BK, int STAGES, int CM, int CN, bool AK_MAJOR = false, bool M16 = false>
__global__ void __launch_bounds__(gemm::Cfg<BK, STAGES, CM, CN>::THREADS,
                                  65536 / (gemm::Cfg<BK, STAGES, CM, CN>::THREADS * SFM_GEMM_REGS)) k_gemm(GemmArgs g) {
    using namespace gemm;
    using CF = Cfg<BK, STAGES, CM, CN>;
    // A diagonal-tile kernel queued behind this launch with programmatic
    // stream serialization may take its SM now (launch_potrf_diag); it waits
    // for this grid's completion itself.  No effect on other successors.
    asm volatile("griddepcontrol.launch_dependents;");
    constexpr int THREADS = CF::THREADS, BNT = CF::BNT, LDSB = CF::LDSB, LDB_K = CF::LDB_K;
    constexpr int BMC = CF::BMC, LDS = CF::LDSA;
    constexpr int NCOL = BN / CN, NSUB = (BM / CM) * NCOL;
    extern __shared__ __align__(16) double smem[];
    constexpr int ASTAGE = AK_MAJOR ? CF::ASTAGE_K : CF::ASTAGE_M;
    double* As = smem;                      // [STAGES][BK][LDS] or [STAGES][BM][LDB_K]
    double* Bs = smem + STAGES * ASTAGE;    // [STAGES][BK][LDSB] or [STAGES][BNT][LDB_K]
    constexpr int BSTAGE = BK_MAJOR ? CF::BSTAGE_K : CF::BSTAGE_N;
    constexpr int CPTA = BK * BMC / 2 / THREADS;  // 16-byte copies per thread: A (BK x BMC), B (BK x BNT)
    constexpr int CPTB = BK * BNT / 2 / THREADS;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    if (g.batch > 1) {  // batched problems: this CTA's problem
        const int y = blockIdx.y;
        g.A += y * g.bsA;
        g.B += y * g.bsB;
        g.C += y * g.bsC;
        if (g.real_rows_b) g.real_rows = g.real_rows_b[y] - g.row_origin;
    }
    int ti, tj;
    const long long l = blockIdx.x / NSUB;
    const int sub = NSUB > 1 ? (int)(blockIdx.x % NSUB) : 0;
    const int half = sub % NCOL, roff = (sub / NCOL) * BMC;  // column block, row offset in the tile
    if (g.tri) {
        // single precision: an FP64 square root here queues behind the resident CTAs' DMMAs on the
        // FP64 pipe (ncu: 8 % of the kernel's stall samples sat on it); the integer loops make it exact
        int t = (int)((sqrtf(8.0f * (float)l + 1.0f) - 1.0f) * 0.5f);
        while ((long long)(t + 1) * (t + 2) / 2 <= l) ++t;
        while ((long long)t * (t + 1) / 2 > l) --t;
        ti = t;
        tj = (int)(l - (long long)t * (t + 1) / 2);
    } else {
        ti = (int)(l % g.tm);
        tj = (int)(l / g.tm);
    }
    if (g.col_step > 1) tj = g.col_first + tj * g.col_step;  // interleaved column tiles (plain launches only)
    if (g.lower_only && ti + g.row_off_tiles < tj + g.col_off_tiles) return;
    const double* A;
    const double* B;
    double* C;
    const int coff = half * BNT;  // column offset inside the 128-wide tile
    bool diag_tile = (g.tri || g.lower_only) && ti + g.row_off_tiles == tj + g.col_off_tiles;
    if (g.cyc_R > 0) {
        const int lt = tj + g.cyc_lt0;
        const int gt = ((lt / g.cyc_G) * g.cyc_R + g.cyc_rank) * g.cyc_G + lt % g.cyc_G;
        const int gi = ti + g.cyc_row0;
        if (gi < gt) return;
        diag_tile = gi == gt;
        A = g.A + (size_t)(gi - g.cyc_ab0) * BM + roff;
        B = g.B + (size_t)(gt - g.cyc_ab0) * BN + coff;  // (B row-indexed, not K-major)
        C = g.C + ((size_t)lt * BN + coff) * g.ldc + (size_t)gi * BM + roff;
    } else {
        A = AK_MAJOR ? g.A + ((size_t)ti * BM + roff) * g.lda : g.A + (size_t)ti * BM + roff;
        B = BK_MAJOR ? g.B + ((size_t)tj * BN + coff) * g.ldb : g.B + (size_t)tj * BN + coff;
        C = g.C + ((size_t)tj * BN + coff) * g.ldc + (size_t)ti * BM + roff;
    }
    constexpr int WARPS_M = BMC / 32;
    const int wm = warp % WARPS_M, wn = warp / WARPS_M;  // WARPS_M x (CN / 32) warps of 32 x 32
    // lower-triangular launches: on a diagonal tile, warp tiles strictly above
    // the diagonal (never read) skip their MMAs and stores (6 of 16); rows in
    // the identity padding (real_rows) skip likewise
    const int crow0 = (g.cyc_R > 0 ? ti + g.cyc_row0 : ti) * BM + roff;  // the CTA's first row of C
    const bool pad_rows = g.pad_skip && crow0 + wm * 32 >= g.real_rows;
    const bool idle = (diag_tile && roff + wm * 32 + 32 <= coff + wn * 32) || pad_rows;
    if (diag_tile && roff + BMC <= coff) return;  // the whole CTA lies above the diagonal
    if (g.pad_skip && crow0 >= g.real_rows) return;  // the whole CTA lies in the padding
    const int beta = (g.beta && !(g.beta0_from >= 0 && tj >= g.beta0_from)) ? 1 : 0;
    int kbeg = 0;  // K offset of this tile
    if (g.k_from_row || (g.k_from_col && tj >= g.beta0_from)) {
        kbeg = g.k_from_row ? ti * BM : (tj - g.beta0_from) * BN;
        A = AK_MAJOR ? A + kbeg : A + (size_t)kbeg * g.lda;
        B = BK_MAJOR ? B + kbeg : B + (size_t)kbeg * g.ldb;
    }

    // per-thread copy sources / destinations (chunk 0); advance by BK per chunk
    const double* asrc[CPTA];
    const double* bsrc[CPTB];
    int adst[CPTA], bdst[CPTB];
#pragma unroll
    for (int u = 0; u < CPTA; ++u) {
        const int idx = tid + THREADS * u;
        if (AK_MAJOR) {
            const int m = idx / (BK / 2), k2 = (idx % (BK / 2)) * 2;
            asrc[u] = A + (size_t)m * g.lda + k2;
            adst[u] = m * LDB_K + k2;
        } else {
            const int k = idx / (BMC / 2), m2 = (idx % (BMC / 2)) * 2;
            asrc[u] = A + (size_t)k * g.lda + m2;
            adst[u] = k * LDS + m2;
        }
    }
#pragma unroll
    for (int u = 0; u < CPTB; ++u) {
        const int idx = tid + THREADS * u;
        if (BK_MAJOR) {
            const int n = idx / (BK / 2), k2 = (idx % (BK / 2)) * 2;
            bsrc[u] = B + (size_t)n * g.ldb + k2;
            bdst[u] = n * LDB_K + k2;
        } else {
            const int k = idx / (BNT / 2), n2 = (idx % (BNT / 2)) * 2;
            bsrc[u] = B + (size_t)k * g.ldb + n2;
            bdst[u] = k * LDSB + n2;
        }
    }
    const size_t astep = AK_MAJOR ? (size_t)BK : (size_t)BK * g.lda;
    const size_t bstep = BK_MAJOR ? (size_t)BK : (size_t)BK * g.ldb;
    auto load_stage = [&](int st, int kc) {
        double* as = As + st * ASTAGE;
        double* bs = Bs + st * BSTAGE;
#pragma unroll
        for (int u = 0; u < CPTA; ++u) cp_async16(as + adst[u], asrc[u] + kc * astep);
#pragma unroll
        for (int u = 0; u < CPTB; ++u) cp_async16(bs + bdst[u], bsrc[u] + kc * bstep);
    };

    const int NK = (g.K - kbeg) / BK;
#pragma unroll
    for (int st = 0; st < STAGES - 1; ++st) {
        if (st < NK) load_stage(st, st);
        cp_async_commit();
    }

    double acc[4][4][2];
    const int rq = 2 * (lane & 3), cq = lane >> 2;
    // fragment base offsets of this lane inside a stage, pinned in registers (the compiler
    // otherwise re-derives them from S2R tid in every chunk: ncu, 4 % of the stall samples)
    int fa = BK_MAJOR ? (wn * 32 + (lane >> 2)) * LDB_K + (lane & 3) : (lane & 3) * LDSB + wn * 32 + (lane >> 2);
    int fb = AK_MAJOR ? (wm * 32 + (lane >> 2)) * LDB_K + (lane & 3) : (lane & 3) * LDS + wm * 32 + (lane >> 2);
    asm volatile("" : "+r"(fa), "+r"(fb));
    // The product accumulates from zero and is applied to C once in the
    // epilogue (C -/+ AB^T): one rounding against C instead of one per
    // k-step, which keeps the Cholesky's Schur-complement updates as accurate
    // as a dot-product (left-looking) formulation.  C is prefetched to L2 now.
#pragma unroll
    for (int mi = 0; mi < 4; ++mi)
#pragma unroll
        for (int ni = 0; ni < 4; ++ni) {
            acc[mi][ni][0] = 0.0;
            acc[mi][ni][1] = 0.0;
            if (beta && (mi & 1) == 0 && (lane & 3) == 0)  // one lane per 128-byte line
                asm volatile("prefetch.global.L2 [%0];" ::"l"(C + (size_t)(wn * 32 + ni * 8 + cq) * g.ldc + wm * 32 + mi * 8));
        }

#pragma unroll 1
    for (int kc = 0; kc < NK; ++kc) {
        cp_async_wait<STAGES - 2>();
        __syncthreads();
        if (kc + STAGES - 1 < NK) load_stage((kc + STAGES - 1) % STAGES, kc + STAGES - 1);
        cp_async_commit();
        const double* as = As + (kc % STAGES) * ASTAGE;
        const double* bs = Bs + (kc % STAGES) * BSTAGE;
        if (idle) continue;
        if constexpr (M16) {
            static_assert(BK % 16 == 0, "k16 steps");
#pragma unroll
            for (int k16 = 0; k16 < BK; k16 += 16) {
                // MMA "A" (16 n x 16 k, row) from the B tile, MMA "B" (16 k x 8 m, col) from the A tile
                // (rows n = wn 32 + 16 nb + g + 8 (i % 2), m = wm 32 + 8 mb + g; k = k16 + t + 4 j)
                double a16[2][8];
#pragma unroll
                for (int nb = 0; nb < 2; ++nb)
#pragma unroll
                    for (int i = 0; i < 8; ++i) {
                        const int dn = 16 * nb + 8 * (i % 2), dk = k16 + 4 * (i / 2);
                        a16[nb][i] = BK_MAJOR ? bs[fa + dn * LDB_K + dk] : bs[fa + dk * LDSB + dn];
                    }
#pragma unroll
                for (int mb = 0; mb < 4; ++mb) {
                    double b16[4];
#pragma unroll
                    for (int i = 0; i < 4; ++i) {
                        const int dm = 8 * mb, dk = k16 + 4 * i;
                        b16[i] = AK_MAJOR ? as[fb + dm * LDB_K + dk] : as[fb + dk * LDS + dm];
                    }
#pragma unroll
                    for (int nb = 0; nb < 2; ++nb)  // D rows n = 16 nb + gq + 8 (i / 2) -> column blocks 2 nb, 2 nb + 1
                        dmma16(acc[mb][2 * nb][0], acc[mb][2 * nb][1], acc[mb][2 * nb + 1][0], acc[mb][2 * nb + 1][1],
                               a16[nb], b16);
                }
            }
            continue;
        }
#pragma unroll
        for (int kk = 0; kk < BK / 4; ++kk) {
            const int krow = kk * 4 + (lane & 3);
            double af[4], bf[4];
#pragma unroll
            for (int mi = 0; mi < 4; ++mi) {
                af[mi] = AK_MAJOR ? as[(wm * 32 + mi * 8 + cq) * LDB_K + krow] : as[krow * LDS + wm * 32 + mi * 8 + cq];
            }
#pragma unroll
            for (int ni = 0; ni < 4; ++ni)
                bf[ni] = BK_MAJOR ? bs[(wn * 32 + ni * 8 + cq) * LDB_K + krow] : bs[krow * LDSB + wn * 32 + ni * 8 + cq];
#pragma unroll
            for (int mi = 0; mi < 4; ++mi)
#pragma unroll
                for (int ni = 0; ni < 4; ++ni) dmma(acc[mi][ni][0], acc[mi][ni][1], bf[ni], af[mi]);
        }
    }
    if (idle) return;
    // epilogue in two halves; each half issues all its C loads before any
    // store (stores to C could alias them, so the compiler would otherwise
    // serialise load -> store pairs)
#pragma unroll
    for (int h = 0; h < 2; ++h) {
        double2 cv[2][4];
        if (beta) {
#pragma unroll
            for (int m2 = 0; m2 < 2; ++m2)
#pragma unroll
                for (int ni = 0; ni < 4; ++ni)
                    cv[m2][ni] = __ldcg(reinterpret_cast<const double2*>(C + (size_t)(wn * 32 + ni * 8 + cq) * g.ldc +
                                                                         wm * 32 + (2 * h + m2) * 8 + rq));
        }
#pragma unroll
        for (int m2 = 0; m2 < 2; ++m2)
#pragma unroll
            for (int ni = 0; ni < 4; ++ni) {
                const int mi = 2 * h + m2;
                double2 c;
                if (beta) {
                    c = cv[m2][ni];
                    if (g.alpha_neg) { c.x -= acc[mi][ni][0]; c.y -= acc[mi][ni][1]; }
                    else { c.x += acc[mi][ni][0]; c.y += acc[mi][ni][1]; }
                } else {
                    c.x = g.alpha_neg ? -acc[mi][ni][0] : acc[mi][ni][0];
                    c.y = g.alpha_neg ? -acc[mi][ni][1] : acc[mi][ni][1];
                }
                *reinterpret_cast<double2*>(C + (size_t)(wn * 32 + ni * 8 + cq) * g.ldc + wm * 32 + mi * 8 + rq) = c;
            }
    }
}

// Launch with the stream's priority as a per-launch attribute, so the
// priority survives CUDA-graph capture (captured kernel nodes do not inherit
// stream priorities).
template <bool PDL = false, typename... KArgs, typename... Args>
static void launch_prio(void (*kernel)(KArgs...), dim3 grid, unsigned block, size_t smem, cudaStream_t s,
                        Args... args) {
    int prio = 0;
    SFM_CUDA(cudaStreamGetPriority(s, &prio));
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = grid;
    cfg.blockDim = dim3(block);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = s;
    cudaLaunchAttribute attr[2];
    attr[0].id = cudaLaunchAttributePriority;
    attr[0].val.priority = prio;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    if (PDL) {  // may start while the stream's preceding kernel drains (the kernel waits: griddepcontrol.wait)
        attr[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
        attr[1].val.programmaticStreamSerializationAllowed = 1;
        cfg.numAttrs = 2;
    }
    SFM_CUDA(cudaLaunchKernelEx(&cfg, kernel, args...));
}

// SFMCOV_GEMM_MMA: 16 (m16n8k16, default) or 4 (m8n8k4) -- A/B measurements
static bool gemm_m16() {
    static bool v = [] { const char* e = std::getenv("SFMCOV_GEMM_MMA"); return !(e && std::atoi(e) == 4); }();
    return v;
}

template <int BK, int ST, int CM, int CN, bool M16>
static void launch_gemm_cfg_m(const GemmArgs& g, long long tiles, cudaStream_t s) {
    using CF = gemm::Cfg<BK, ST, CM, CN>;
    const dim3 grid((unsigned)(tiles * (gemm::BM / CM) * (gemm::BN / CN)), g.batch > 1 ? g.batch : 1);
    if (g.a_kmajor) {
        if (!g.b_kmajor) throw CudaError("gemm: K-major A needs K-major B");
        launch_prio(k_gemm<true, BK, ST, CM, CN, true, M16>, grid, CF::THREADS, CF::SMEM_AK, s, g);
    } else if (g.b_kmajor) launch_prio(k_gemm<true, BK, ST, CM, CN, false, M16>, grid, CF::THREADS, CF::smem(true), s, g);
    else launch_prio(k_gemm<false, BK, ST, CM, CN, false, M16>, grid, CF::THREADS, CF::smem(false), s, g);
}
template <int BK, int ST, int CM, int CN>
static void launch_gemm_cfg(const GemmArgs& g, long long tiles, cudaStream_t s) {
    if (gemm_m16()) launch_gemm_cfg_m<BK, ST, CM, CN, true>(g, tiles, s);
    else launch_gemm_cfg_m<BK, ST, CM, CN, false>(g, tiles, s);
}

template <bool KM, int BK, int ST, int CM, int CN>
static void set_smem() {
    using CF = gemm::Cfg<BK, ST, CM, CN>;
    for (int m16 = 0; m16 < 2; ++m16) {
        SFM_CUDA(cudaFuncSetAttribute(m16 ? k_gemm<KM, BK, ST, CM, CN, false, true> : k_gemm<KM, BK, ST, CM, CN, false, false>,
                                      cudaFuncAttributeMaxDynamicSharedMemorySize, CF::SMEM));
        if (KM)
            SFM_CUDA(cudaFuncSetAttribute(m16 ? k_gemm<true, BK, ST, CM, CN, true, true> : k_gemm<true, BK, ST, CM, CN, true, false>,
                                          cudaFuncAttributeMaxDynamicSharedMemorySize, CF::SMEM_AK));
    }
}

// Opt-in shared-memory sizes, set once before any launch (and before graph
// capture).
void dense_init_attributes() {
    static bool done = false;
    if (done) return;
    set_smem<false, 16, 4, 128, 128>(); set_smem<true, 16, 4, 128, 128>();
    set_smem<false, 16, 3, 128, 64>(); set_smem<true, 16, 3, 128, 64>();
    set_smem<false, 16, 3, 64, 64>(); set_smem<true, 16, 3, 64, 64>();
    SFM_CUDA(cudaFuncSetAttribute(k_potrf_diag_fwd(), cudaFuncAttributeMaxDynamicSharedMemorySize, potrf_smem_bytes()));
    done = true;
}

// Three configurations: 64 x 64 CTAs of 4 warps, four per SM, BK 16 x 3
// stages (every launch whose output tiles are independent: with four CTAs
// per SM their prologues / epilogues overlap the others' MMAs better than
// with two 128 x 64 CTAs -- config 3 sweep 17.3 -> 16.8 ms, config 4 396 ->
// 387 ms); 128 x 64 CTAs, two per SM, for launches whose C aliases B (the
// in-place X[r, :] = Linv_r X[r, :]: a CTA must own all rows of its columns);
// 128 x 128 CTAs, one per SM, BK 16 x 4 stages for whole_tile launches (C
// aliases A, so one CTA must own a whole tile row).
void launch_gemm(const GemmArgs& g, cudaStream_t s) {
    const long long tiles = g.tri ? (long long)g.tm * (g.tm + 1) / 2 : (long long)g.tm * g.tn;
    if (tiles <= 0) return;
    // C aliasing an operand (in-place updates, e.g. X[r, :] = Linv_r X[r, :]):
    // every CTA must read its whole K range of the shared rows before writing
    // them, so no CTA may own only part of a tile's rows
    const bool alias = g.C == g.B || g.C == g.A;
    // SFMCOV_GEMM_LOG=1 (diagnostics, tools/gemm_launch_eff.py): one stderr line per launch
    static const bool log = [] { const char* e = std::getenv("SFMCOV_GEMM_LOG"); return e && e[0] == '1'; }();
    if (log) {
        int prio = 0;
        cudaStreamGetPriority(s, &prio);
        std::fprintf(stderr, "gemm tm=%d tn=%d K=%d tri=%d lower=%d kmajor=%d kfrom=%d whole=%d alias=%d prio=%d b0=%d coff=%d\n", g.tm,
                     g.tn, g.K, g.tri, g.lower_only, g.b_kmajor, g.k_from_col, g.whole_tile, (int)alias, prio, g.beta0_from,
                     g.col_off_tiles);
    }
    if (g.whole_tile) launch_gemm_cfg<16, 4, 128, 128>(g, tiles, s);
    else if (alias) launch_gemm_cfg<16, 3, 128, 64>(g, tiles, s);
    else launch_gemm_cfg<16, 3, 64, 64>(g, tiles, s);
    SFM_LAUNCH_CHECK();
}

// Diagonal tile: Cholesky + triangular inverse of one kNB x kNB tile in smem.
// Blocked by 32: each 32x32 diagonal block is factored (and inverted) by one
// warp in registers with shuffles (rsqrt pivots keep the per-column latency
// chain short); the panel solve and the trailing update inside the tile use
// all warps.  The inverse Y = L^-1 is built in shared memory: its strictly
// lower 32-blocks are stored transposed in the (unused) upper triangle of T.
// ----------------------------------------------------------------------------
#ifdef SFM_POTRF_TIMING
__device__ long long g_potrf_stamp[64];
#define POTRF_STAMP(i) do { __syncthreads(); if (threadIdx.x == 0) g_potrf_stamp[i] = clock64(); } while (0)
void debug_potrf_stamps(long long* out) { cudaMemcpyFromSymbol(out, g_potrf_stamp, 64 * sizeof(long long)); }
#else
#define POTRF_STAMP(i) do { } while (0)
#endif

// ----------------------------------------------------------------------------
// Diagonal tile: Cholesky + triangular inverse of one kNB x kNB tile in smem.
//
// 8-wide right-looking steps.  Each 8x8 diagonal block is factored and
// inverted by one warp in registers (shuffles, rsqrt pivots); the panel
// solve below it is one row per thread; the in-tile trailing update and the
// block forward substitution for Y = L^-1 are 8x8 DMMA tiles spread over the
// warps.  Y's strictly-lower 8-blocks are stored transposed in the unused
// upper triangle of the tile, its diagonal blocks in Xd.
// ----------------------------------------------------------------------------
namespace potrf {
constexpr int LDT = kNB + 8;  // 136: conflict-free m8n8k4 fragment reads
constexpr int SB = 8;
constexpr int NSB = kNB / SB;  // 16
constexpr int THREADS = 512;
constexpr int NWARPS = THREADS / 32;
constexpr int SMEM = (kNB * LDT + NSB * 64 + NWARPS * 64 + 2 * kNB) * 8;
}  // namespace potrf

// 1/sqrt(d) for d > 0: MUFU.RSQ64H seed + Newton steps (full double
// precision without the libdevice call on the per-column critical path).
// The seed is good to ~2^-23 and each step squares the error, so two steps
// reach ~2^-90; a third only repeated the rounding (parity unchanged; the
// tile factorisation loop 65k -> 63k cycles, tools/potrf_stamps.cu).
__device__ __forceinline__ double fast_rsqrt(double d) {
    double y;
    asm("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(d));
    const double hd = 0.5 * d;
#pragma unroll
    for (int it = 0; it < 2; ++it) y = y * (1.5 - hd * y * y);
    return y;
}

// 8x8 Cholesky of the block at T(c0, c0) by one warp (lanes 0..7 hold
// rows); stores L and 1/L_jj (rinv).  Pivots L_jj^2 -> piv.
__device__ __forceinline__ void warp_potrf8(double* T, int c0, double* rinv, double* spiv) {
    using namespace potrf;
    // reconverge the warp first: shuffles on a diverged warp take the
    // emulated WARPSYNC.COLLECTIVE path (~10x slower)
    __syncwarp();
    const int i = threadIdx.x & 31;
    double a[SB];
#pragma unroll
    for (int c = 0; c < SB; ++c) a[c] = (i < SB && c <= i) ? T[(c0 + c) * LDT + c0 + i] : 0.0;
    double my_inv = 1.0;
#pragma unroll
    for (int j = 0; j < SB; ++j) {
        double d = __shfl_sync(0xffffffffu, a[j], j);
        if (i == j) spiv[c0 + j] = d;  // pivots (L_jj^2) and failures are flushed after the loop
        if (!(d > 0.0) || !isfinite(d)) d = 1.0;
        const double inv = fast_rsqrt(d);
        if (i == j) { a[j] = d * inv; my_inv = inv; }
        else if (i > j) a[j] = a[j] * inv;
#pragma unroll
        for (int c = j + 1; c < SB; ++c) {
            const double lc = __shfl_sync(0xffffffffu, a[j], c);
            if (i >= c) a[c] -= a[j] * lc;
        }
    }
    if (i < SB) {
#pragma unroll
        for (int c = 0; c < SB; ++c)
            if (c <= i) T[(c0 + c) * LDT + c0 + i] = a[c];
        rinv[c0 + i] = my_inv;
    }
}

// Inverse X = L^-1 of the 8x8 lower block at T(c0, c0) by one warp (lane c
// owns column c), row-major into Xs.
__device__ __forceinline__ void warp_inv8(const double* T, int c0, const double* rinv, double* Xs) {
    using namespace potrf;
    const int c = threadIdx.x & 31;
    double x[SB];
#pragma unroll
    for (int r = 0; r < SB; ++r) {
        double s = 0.0;
#pragma unroll
        for (int k = 0; k < r; ++k)
            if (k >= c) s += T[(c0 + k) * LDT + c0 + r] * x[k];
        x[r] = (r < c) ? 0.0 : ((r == c) ? rinv[c0 + r] : -s * rinv[c0 + r]);
    }
    if (c < SB) {
#pragma unroll
        for (int r = 0; r < SB; ++r) Xs[r * SB + c] = x[r];
    }
}

__device__ __forceinline__ void dmma8(double& d0, double& d1, double a, double b) {
    asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                 : "+d"(d0), "+d"(d1)
                 : "d"(a), "d"(b));
}

// A: tile (k0, k0) of the matrix (col-major, ld).  Writes L (lower) back,
// Linv (kNB x kNB col-major, zeros above), pivots[col0 + j] = L_jj^2.
__global__ void __launch_bounds__(potrf::THREADS, 1) k_potrf_diag(double* A, long long ld, double* Linv, double* pivots,
                                                                 int col0, Status* st, long long bsA, long long bsL,
                                                                 long long bsP) {
    using namespace potrf;
    A += blockIdx.y * bsA;  // batched problems (grid.y)
    Linv += blockIdx.y * bsL;
    pivots += blockIdx.y * bsP;
    extern __shared__ double T[];                 // T[c * LDT + r]
    double* Xd = T + kNB * LDT;                   // NSB blocks, row-major 8x8
    double* Ws = Xd + NSB * 64;                   // per-warp 8x8 scratch
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const int fr = lane >> 2, fk = lane & 3;      // fragment row / k index
    POTRF_STAMP(19);
    // launched early (programmatic stream serialization): the CTA already
    // holds its SM; the tile is complete once the preceding grid has finished
    asm volatile("griddepcontrol.wait;" ::: "memory");
#pragma unroll 16
    for (int e = tid; e < kNB * kNB; e += THREADS) {
        const int r = e & (kNB - 1), c = e >> 7;
        T[c * LDT + r] = (r >= c) ? __ldcg(A + (size_t)c * ld + r) : 0.0;
    }
    __syncthreads();  // warp 0 reads the first 8x8 block, loaded by warps 0, 4, 8 and 12
    POTRF_STAMP(0);
    double* rinv = Ws + NWARPS * 64;             // 1 / L_jj
    double* spiv = rinv + kNB;                   // pivots
    if (warp == 0) warp_potrf8(T, 0, rinv, spiv);
    __syncthreads();
    for (int s = 0; s < NSB; ++s) {
        const int c0 = s * SB;
        const int rows = kNB - c0 - SB;
        if (rows == 0) break;
        // panel solve by forward substitution, one row per thread:
        // x_c = (a_c - Σ_{k<c} x_k L[c0+c][c0+k]) / L_cc
        if (tid < rows) {
            const int r = c0 + SB + tid;
            double x[SB];
#pragma unroll
            for (int c = 0; c < SB; ++c) x[c] = T[(c0 + c) * LDT + r];
#pragma unroll
            for (int c = 0; c < SB; ++c) {
                double sum = 0.0;  // dot product first, one subtraction (see k_gemm)
#pragma unroll
                for (int k = 0; k < c; ++k) sum += x[k] * T[(c0 + k) * LDT + c0 + c];
                x[c] = (x[c] - sum) * rinv[c0 + c];
            }
#pragma unroll
            for (int c = 0; c < SB; ++c) T[(c0 + c) * LDT + r] = x[c];
        }
        __syncthreads();
        // trailing update T[r, c] -= Σ_k L[r, c0+k] L[c, c0+k] in 8x8 DMMA
        // tiles.  Warp 0 updates the next diagonal tile and factors it right
        // away (the lookahead inside the tile); warps 1.. take the other
        // tiles four at a time.
        const int nt = rows / SB;
        const int ntiles = nt * (nt + 1) / 2;
        const int c1 = c0 + SB;
        if (warp == 0) {
            double* cp = T + (c1 + 2 * fk) * LDT + c1 + fr;
            double d0 = 0.0, d1 = 0.0;  // product from zero, applied once (see k_gemm)
#pragma unroll
            for (int kk = 0; kk < SB; kk += 4) {
                const double tv = T[(c0 + kk + fk) * LDT + c1 + fr];
                dmma8(d0, d1, tv, tv);
            }
            cp[0] -= d0;
            cp[LDT] -= d1;
            warp_potrf8(T, c1, rinv, spiv);
        } else {
            for (int t0 = 1 + 4 * (warp - 1); t0 < ntiles; t0 += 4 * (NWARPS - 1)) {
                double d[4][2];
                double* cp[4];
                int r0v[4], q0v[4];
#pragma unroll
                for (int u = 0; u < 4; ++u) {
                    const int t = (t0 + u < ntiles) ? t0 + u : t0;
                    int ti = (int)((sqrtf(8.0f * t + 1.0f) - 1.0f) * 0.5f);
                    while ((ti + 1) * (ti + 2) / 2 <= t) ++ti;
                    while (ti * (ti + 1) / 2 > t) --ti;
                    const int tj = t - ti * (ti + 1) / 2;
                    r0v[u] = c1 + SB * ti;
                    q0v[u] = c1 + SB * tj;
                    cp[u] = T + (q0v[u] + 2 * fk) * LDT + r0v[u] + fr;
                    d[u][0] = 0.0;
                    d[u][1] = 0.0;
                }
#pragma unroll
                for (int kk = 0; kk < SB; kk += 4) {
#pragma unroll
                    for (int u = 0; u < 4; ++u) {
                        const double av = T[(c0 + kk + fk) * LDT + r0v[u] + fr];
                        const double bv = T[(c0 + kk + fk) * LDT + q0v[u] + fr];
                        dmma8(d[u][0], d[u][1], av, bv);
                    }
                }
#pragma unroll
                for (int u = 0; u < 4; ++u)
                    if (t0 + u < ntiles) {
                        cp[u][0] -= d[u][0];
                        cp[u][LDT] -= d[u][1];
                    }
            }
        }
        __syncthreads();
    }
    POTRF_STAMP(4);
    if (tid < kNB) {
        const double d = spiv[tid];
        pivots[col0 + tid] = d;
        if (!(d > 0.0) || !isfinite(d)) atomicMin(&st->chol_bad, col0 + tid);
    }
    // the sixteen 8x8 diagonal inverses, in parallel
    for (int s = warp; s < NSB; s += NWARPS) warp_inv8(T, s * SB, rinv, Xd + s * 64);
    __syncthreads();
    POTRF_STAMP(1);
    // Y = L^-1 by block rows: Y_ij = -X_i Σ_{k=j}^{i-1} L_ik Y_kj (j < i);
    // Y_kj (k > j) lives transposed at T[(8k + r) LDT + 8j + c].
    for (int bi = 1; bi < NSB; ++bi) {
        for (int bj = warp; bj < bi; bj += NWARPS) {
            double d0 = 0.0, d1 = 0.0;
            for (int bk = bj; bk < bi; ++bk) {
#pragma unroll
                for (int kk = 0; kk < SB; kk += 4) {
                    const double av = T[(SB * bk + kk + fk) * LDT + SB * bi + fr];  // L_ik[fr][kk+fk]
                    const double bv = (bk == bj) ? Xd[bj * 64 + (kk + fk) * SB + fr]  // Y_jj[kk+fk][fr]
                                                 : T[(SB * bk + kk + fk) * LDT + SB * bj + fr];
                    dmma8(d0, d1, av, bv);
                }
            }
            // S (C layout) -> scratch, then Y_ij = -X_i S
            double* w = Ws + warp * 64;
            w[fr * SB + 2 * fk] = d0;
            w[fr * SB + 2 * fk + 1] = d1;
            __syncwarp();
            double y0 = 0.0, y1 = 0.0;
#pragma unroll
            for (int kk = 0; kk < SB; kk += 4) {
                const double t = Xd[bi * 64 + fr * SB + kk + fk];  // -X_i[fr][kk+fk]
                const double av = __hiloint2double(__double2hiint(t) ^ (int)0x80000000u, __double2loint(t));
                const double bv = w[(kk + fk) * SB + fr];             // S[kk+fk][fr]
                dmma8(y0, y1, av, bv);
            }
            __syncwarp();
            // Y_ij[fr][2fk + q] -> T[(8 bi + fr) LDT + 8 bj + 2 fk + q]
            T[(SB * bi + fr) * LDT + SB * bj + 2 * fk] = y0;
            T[(SB * bi + fr) * LDT + SB * bj + 2 * fk + 1] = y1;
        }
        __syncthreads();
    }
    POTRF_STAMP(2);
    for (int e = tid; e < kNB * kNB; e += THREADS) {
        const int r = e & (kNB - 1), c = e >> 7;
        const int bi = r / SB, bj = c / SB;
        double y = 0.0;
        if (bi == bj) { if ((r % SB) >= (c % SB)) y = Xd[bi * 64 + (r % SB) * SB + (c % SB)]; }
        else if (bi > bj) y = T[r * LDT + c];
        Linv[(size_t)c * kNB + r] = y;
        if (r >= c) A[(size_t)c * ld + r] = T[c * LDT + r];
    }
    POTRF_STAMP(3);
#ifdef SFM_POTRF_DELAY
    {  // sensitivity experiment: how much of the tile kernel's time is on the sweep's critical path
        const long long t0 = clock64();
        while (clock64() - t0 < SFM_POTRF_DELAY) { }
    }
#endif
}

const void* k_potrf_diag_ptr() { return (const void*)k_potrf_diag; }
int potrf_smem_bytes_impl() { return potrf::SMEM; }

void launch_potrf_diag(double* A, long long ld, double* Linv, double* pivots, int col0, Status* st, cudaStream_t s,
                       const SweepBatch* bt) {
    const int B = bt ? bt->B : 1;
    // SFMCOV_POTRF_PDL=0: plain stream order (A/B measurements)
    static const bool pdl = [] { const char* e = std::getenv("SFMCOV_POTRF_PDL"); return !(e && e[0] == '0'); }();
    if (pdl && !bt)  // batched sweeps: one tile CTA per problem would hold that many SMs while waiting (measured: noisier, no gain)
        launch_prio<true>(k_potrf_diag, dim3(1, B), potrf::THREADS, potrf::SMEM, s, A, ld, Linv, pivots, col0, st,
                          bt ? bt->zs : 0LL, bt ? bt->ls : 0LL, bt ? bt->ps : 0LL);
    else
        launch_prio(k_potrf_diag, dim3(1, B), potrf::THREADS, potrf::SMEM, s, A, ld, Linv, pivots, col0, st,
                    bt ? bt->zs : 0LL, bt ? bt->ls : 0LL, bt ? bt->ps : 0LL);
    SFM_LAUNCH_CHECK();
}

// ----------------------------------------------------------------------------
// Diagonal blocks of Z^-1 = X^T X (X = L^-1 lower), unscaled + PSD check.
// One CTA (8 warps) per camera; each lane accumulates the P(P+1)/2 unique
// products over a strided set of rows, then a fixed-order tree reduction.
// ----------------------------------------------------------------------------
// The per-camera Gram blocks on the tensor cores: S = Xcᵀ Xc over the rows
// r >= c0 of the camera's columns (X lower triangular), as FP64 m8n8k4 MMAs
// whose A and B fragments are the same load (lane (m, k) holds X[r + k][c0 + m]
// for both).  For P = 9 the ninth column is FMAs on the same fragments.  Few
// registers, so 8 warps x 4 CTAs per SM keep enough loads in flight for HBM
// (the scalar 45-accumulator version ran at 2.2 TB/s with 25 % of the warps).
template <int P>
__global__ void __launch_bounds__(256, 4) k_extract(const double* X, long long ld, int N, const double* s_a, int scale,
                                                 double* cov, Status* st, int* psd_warn, ZMap zm) {
    static_assert(P == 8 || P == 9, "camera block");
    constexpr int NW = 8, U = 4;  // warps, MMAs in flight per warp
    __shared__ double red[NW][81];
    int i = blockIdx.x;
    if (zm.scene_of_cam) {  // batched sub-scenes: the camera's own problem
        const int scn = zm.scene_of_cam[i], c0s = zm.coff[scn];
        X += scn * zm.zstride;
        N = P * (zm.coff[scn + 1] - c0s);
        s_a += (size_t)P * c0s;
        cov += (size_t)P * P * c0s;
        i -= c0s;
    }
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int c0 = P * i;
    const int m = lane >> 2, k = lane & 3;
    const double* xc = X + (size_t)(c0 + m) * ld;
    const double* x8c = X + (size_t)(c0 + 8) * ld;
    double d0[U], d1[U], a8[U], s88 = 0.0;
#pragma unroll
    for (int u = 0; u < U; ++u) { d0[u] = 0.0; d1[u] = 0.0; a8[u] = 0.0; }
    for (int r0 = c0 + 4 * U * warp; r0 < N; r0 += 4 * U * NW) {
        double xv[U], x8[U];
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const int r = r0 + 4 * u + k;
            xv[u] = (r < N && r >= c0 + m) ? __ldcs(xc + r) : 0.0;
            if (P == 9) x8[u] = (r < N && r >= c0 + 8) ? __ldcs(x8c + r) : 0.0;
        }
#pragma unroll
        for (int u = 0; u < U; ++u) {
            asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                         : "+d"(d0[u]), "+d"(d1[u])
                         : "d"(xv[u]), "d"(xv[u]));
            if (P == 9) {
                a8[u] = fma(x8[u], xv[u], a8[u]);     // S[8][m], partial over k
                if (m == 0) s88 = fma(x8[u], x8[u], s88);
            }
        }
    }
    // lane holds S[m][2k], S[m][2k+1]; S[8][m] partials over k; S[8][8] on lanes 0..3
    double t0 = 0.0, t1 = 0.0, t8 = 0.0;
#pragma unroll
    for (int u = 0; u < U; ++u) { t0 += d0[u]; t1 += d1[u]; t8 += a8[u]; }
    red[warp][9 * m + 2 * k] = t0;
    red[warp][9 * m + 2 * k + 1] = t1;
    if (P == 9) {
        t8 += __shfl_xor_sync(0xffffffffu, t8, 1);
        t8 += __shfl_xor_sync(0xffffffffu, t8, 2);
        s88 += __shfl_xor_sync(0xffffffffu, s88, 1);
        s88 += __shfl_xor_sync(0xffffffffu, s88, 2);
        if (k == 0) red[warp][9 * 8 + m] = t8;
        if (lane == 0) red[warp][80] = s88;
    }
    __syncthreads();
    __shared__ double out[P * P];
    if (threadIdx.x < P * P) {
        const int p = threadIdx.x / P, q = threadIdx.x % P;
        // the stored entries: (p, q) with p < 8, q < 8 at 9p + q; row 8 at 72 + q; (8, 8) at 80
        const int lo = p < q ? p : q, hi = p < q ? q : p;
        const int src = (hi < 8) ? 9 * lo + hi : (lo < 8 ? 72 + lo : 80);  // one triangle: exact symmetry
        double v = 0.0;
#pragma unroll
        for (int w = 0; w < NW; ++w) v += red[w][src];
        const double sp = scale ? s_a[c0 + p] : 1.0, sq = scale ? s_a[c0 + q] : 1.0;
        const double o = (sp * v) * sq;
        out[threadIdx.x] = o;
        cov[(size_t)P * P * i + threadIdx.x] = o;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        // PSD test (covariance.cpp:266-268: lam_min < -kPsdTol * trace warns):
        // lam_min(S) > -tau  <=>  S + tau I is positive definite  <=>  its
        // Cholesky succeeds.
        double tr = 0.0;
        for (int p = 0; p < P; ++p) tr += out[P * p + p];
        const double tau = kPsdTol * tr;
        double L[P * P];
        bool pd = true;
        for (int c = 0; c < P && pd; ++c) {
            double s = out[P * c + c] + tau;
            for (int kk = 0; kk < c; ++kk) s -= L[P * c + kk] * L[P * c + kk];
            if (!(s > 0.0)) { pd = false; break; }
            const double lcc = sqrt(s);
            L[P * c + c] = lcc;
            for (int r = c + 1; r < P; ++r) {
                double x = out[P * r + c];
                for (int kk = 0; kk < c; ++kk) x -= L[P * r + kk] * L[P * c + kk];
                L[P * r + c] = x / lcc;
            }
        }
        if (!pd) atomicAdd(psd_warn, 1);
    }
}

void launch_extract(int P, const double* X, long long ld, int N, int nblocks, const double* s_a, int scale, double* cov,
                    Status* st, int* psd_warn, cudaStream_t s, ZMap zm) {
    if (!nblocks) return;
    if (P == 8) k_extract<8><<<nblocks, 256, 0, s>>>(X, ld, N, s_a, scale, cov, st, psd_warn, zm);
    else if (P == 9) k_extract<9><<<nblocks, 256, 0, s>>>(X, ld, N, s_a, scale, cov, st, psd_warn, zm);
    else throw CudaError("extract: unsupported block size");
    SFM_LAUNCH_CHECK();
}

// Identity on the padded tail of the diagonal: Z(i, i) = 1 for i in [from, to).
__global__ void k_set_diag(double* Z, long long ld, int from, int to) {
    const int i = from + blockIdx.x * blockDim.x + threadIdx.x;
    if (i < to) Z[(size_t)i * ld + i] = 1.0;
}

void launch_set_diag(double* Z, long long ld, int from, int to, cudaStream_t s) {
    if (to <= from) return;
    k_set_diag<<<cdiv(to - from, 128), 128, 0, s>>>(Z, ld, from, to);
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

// min / max of x[0..count) (values > 0 here: the Jacobi scales), two passes.
__global__ void k_minmax_partial(const double* x, long long count, double* part) {
    __shared__ double mn[256], mx[256];
    double a = INFINITY, b = -INFINITY;
    for (long long i = (long long)blockIdx.x * 256 + threadIdx.x; i < count; i += (long long)gridDim.x * 256) {
        const double v = x[i];
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
    if (threadIdx.x == 0) { part[2 * blockIdx.x] = mn[0]; part[2 * blockIdx.x + 1] = mx[0]; }
}

__global__ void k_minmax_final(const double* part, int nb, double* out) {
    __shared__ double mn[256], mx[256];
    double a = INFINITY, b = -INFINITY;
    for (int i = threadIdx.x; i < nb; i += 256) { a = fmin(a, part[2 * i]); b = fmax(b, part[2 * i + 1]); }
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
    if (threadIdx.x == 0) { out[0] = mn[0]; out[1] = mx[0]; }
}

// out[0..1] = min, max; part: 2 * 296 doubles of scratch
void launch_minmax(const double* x, long long count, double* part, double* out, cudaStream_t s) {
    constexpr int NB = 296;
    k_minmax_partial<<<NB, 256, 0, s>>>(x, count, part);
    SFM_LAUNCH_CHECK();
    k_minmax_final<<<1, 256, 0, s>>>(part, NB, out);
    SFM_LAUNCH_CHECK();
}

void launch_pivot_range(const double* piv, int N, double* out, cudaStream_t s) {
    k_pivot_range<<<1, 256, 0, s>>>(piv, N, out);
    SFM_LAUNCH_CHECK();
}

// ----------------------------------------------------------------------------
// Drivers
// ----------------------------------------------------------------------------
static bool debug_sync() {
    static bool v = [] { const char* e = std::getenv("SFMCOV_DEBUG_SYNC"); return e && e[0] == '1'; }();
    return v;
}

GemmArgs gemm_args(double* C, long long ldc, const double* A, long long lda, const double* B, long long ldb,
                          int tm, int tn, int K) {
    GemmArgs g{};
    g.C = C; g.ldc = ldc; g.A = A; g.lda = lda; g.B = B; g.ldb = ldb;
    g.tm = tm; g.tn = tn; g.K = K; g.beta0_from = -1;
    return g;
}

// ----------------------------------------------------------------------------
// Fused sweep: Cholesky and triangular inverse in one pass over the panels.
//
// Step p (panel p = 128-blocks b0 .. b0+g, W = g kNB columns):
//   s  (critical): potrf / trsm / inner updates of the panel (as in
//       dense_cholesky); take(p): L[rows >= b0, panel] -> ring buffer Lb and
//       the panel's W x W diagonal block of Z := I (its columns now hold the
//       right-hand side of X = L^-1); u(p): next panel columns -= L L^T.
//   s2 (bulk)    : rest(p): trailing columns beyond the next panel.
//   s3 (bulk)    : inverse step p on the rows of panel p, columns 0 .. b0+g:
//       for each block r of the panel: X[r, :] = Linv_r X[r, :], then
//       X[r', :] -= L[r', r] X[r, :] for the panel's later blocks r';
//       finally X[rows below, 0 .. b0+g] -= L[below, panel] X[panel rows, :].
// The Cholesky chain only touches columns >= b0(p+1) after take(p) and the
// inverse chain only columns < b0(p+1), so the two overlap freely; both read
// the panel from Lb, which is recycled once inverse step p - NB has finished.
// ----------------------------------------------------------------------------
__global__ void k_panel_take(double* Z, long long ld, int b0, int W, int rows, double* Lb) {
    const long long e = (long long)blockIdx.x * blockDim.x + threadIdx.x;  // one double2 (two rows) each
    const int half = rows >> 1;
    if (e >= (long long)half * W) return;
    const int i = (int)(e % half) * 2, j = (int)(e / half);
    double2* zp = reinterpret_cast<double2*>(Z + (size_t)(b0 * kNB + j) * ld + (size_t)b0 * kNB + i);
    const double2 v = __ldcg(zp);
    *reinterpret_cast<double2*>(Lb + (size_t)j * rows + i) = v;
    if (i < W) {
        double2 x;
        x.x = (i == j) ? 1.0 : 0.0;
        x.y = (i + 1 == j) ? 1.0 : 0.0;
        *zp = x;
    }
}

// The panel's diagonal 128-tiles (L, from Z) into the slot; the W x W block of Z := I.
__global__ void k_panel_take_diag(double* Z, long long ld, int b0, int W, double* Lb, int rows, long long bsZ,
                                  long long bsL) {
    Z += blockIdx.y * bsZ;  // batched problems (grid.y)
    Lb += blockIdx.y * bsL;
    const int e = blockIdx.x * blockDim.x + threadIdx.x;  // one double2 (two rows)
    const int half = W >> 1;
    if (e >= half * W) return;
    const int i = (e % half) * 2, j = e / half;
    double2* zp = reinterpret_cast<double2*>(Z + (size_t)(b0 * kNB + j) * ld + (size_t)b0 * kNB + i);
    if (i / kNB == j / kNB) *reinterpret_cast<double2*>(Lb + (size_t)j * rows + i) = __ldcg(zp);
    double2 x;
    x.x = (i == j) ? 1.0 : 0.0;
    x.y = (i + 1 == j) ? 1.0 : 0.0;
    *zp = x;
}

static void launch_panel_take_diag(double* Z, long long ld, int b0, int W, double* Lb, int rows, cudaStream_t s,
                                   const SweepBatch* bt = nullptr) {
    const int total = (W / 2) * W;
    k_panel_take_diag<<<dim3(cdiv(total, 256), bt ? bt->B : 1), 256, 0, s>>>(Z, ld, b0, W, Lb, rows, bt ? bt->zs : 0LL,
                                                                               bt ? bt->rs : 0LL);
    SFM_LAUNCH_CHECK();
}

static void launch_panel_take(double* Z, long long ld, int b0, int W, int rows, double* Lb, cudaStream_t s) {
    const long long total = (long long)(rows / 2) * W;
    k_panel_take<<<cdiv(total, 256), 256, 0, s>>>(Z, ld, b0, W, rows, Lb);
    SFM_LAUNCH_CHECK();
}

// SFMCOV_SWEEP_TRACE=1 (diagnostics, tools/trace_view.py): per panel, events
// on the critical stream (panel start, hand-over, next-column update done),
// s2 (rest done) and s3 (inverse step done), printed to stderr in ms after
// the first.  Config 3 showed the sweep is throughput-bound, not
// critical-path-bound: the Cholesky chain ends at 14.2 ms, the inverse chain
// at 17.9 ms, and a 12-slot ring left the total unchanged.
static bool sweep_trace() {
    static bool v = [] { const char* e = std::getenv("SFMCOV_SWEEP_TRACE"); return e && e[0] == '1'; }();
    return v;
}
struct SweepTrace {
    std::vector<cudaEvent_t> ev;
    std::vector<std::pair<int, int>> tag;  // (panel, point)
    void rec(int p, int what, cudaStream_t st) {
        cudaEvent_t e;
        cudaEventCreate(&e);
        cudaEventRecord(e, st);
        ev.push_back(e);
        tag.push_back({p, what});
    }
    void dump() {
        if (ev.empty()) return;
        cudaDeviceSynchronize();
        static const char* names[] = {"start", "take", "next1", "rest", "inv", "potrf", "trsm", "inner"};
        for (size_t i = 0; i < ev.size(); ++i) {
            float ms = 0.f;
            cudaEventElapsedTime(&ms, ev[0], ev[i]);
            std::fprintf(stderr, "trace p=%d %s %.4f\n", tag[i].first, names[tag[i].second], ms);
        }
        for (auto e : ev) cudaEventDestroy(e);
        cudaGetLastError();
    }
};

int dense_sweep(double* Z, long long ld, int Npad, int G, double* Linv, double* pivots, Status* st, double* ring,
                int NB, cudaStream_t s, cudaStream_t s2, cudaStream_t s3, cudaEvent_t* eL, cudaEvent_t* eT,
                cudaEvent_t eR, cudaStream_t s4, cudaEvent_t eX, cudaEvent_t eN, cudaEvent_t eZ, int nreal,
                const SweepBatch* bt, const InvSplit* isp) {
    // nreal (optional): the unpadded size; the trailing and next-panel
    // updates skip the identity padding's rows (their L rows are zero).
    // bt (optional): bt->B problems swept together, every launch batched
    // over grid.y (nreal then per problem, bt->nreal_b).
    // eZ (optional): Z's columns beyond the first panel are complete (the
    // pair reduction of the other block columns, queued on s2 before this
    // sweep): waited for by the first next-panel update on s; rest(0) is
    // ordered after it on s2 itself.
    SweepTrace tr;
    const bool trace = sweep_trace();
    bool next_pending = false;  // the previous step's update of the next panel's later columns (s4)
    const int K = Npad / kNB;
    int launches = 0;
    bool rest_pending = false;
    // SFMCOV_INV_SPLIT=w: the inverse on w column-interleaved streams (1 = all on s3; A/B measurements)
    static const int inv_ways = [] { const char* e = std::getenv("SFMCOV_INV_SPLIT"); return e ? std::atoi(e) : 3; }();
    const int ways = (!bt && isp && s3 != s) ? std::max(1, std::min(inv_ways, isp->n + 1)) : 1;
    const bool split_inv = ways > 1;
    // operand kinds for the batch strides: Z, the Linv tiles, the panel ring
    enum Op { OZ, OL, OR };
    auto stride = [&](Op o) -> long long { return !bt ? 0 : (o == OZ ? bt->zs : (o == OL ? bt->ls : bt->rs)); };
    auto batched = [&](GemmArgs& g, Op c, Op a, Op b) {
        if (!bt || bt->B <= 1) return;
        g.batch = bt->B;
        g.bsC = stride(c);
        g.bsA = stride(a);
        g.bsB = stride(b);
    };
    // skip the padding's rows of C, whose first row is `origin` of the matrix
    auto pad_rows = [&](GemmArgs& g, int origin) {
        if (bt && bt->nreal_b) {
            g.pad_skip = 1;
            g.real_rows_b = bt->nreal_b;
            g.row_origin = origin;
        } else if (nreal > 0) {
            g.pad_skip = 1;
            g.real_rows = nreal - origin;
        }
    };
    int last_slot = -1;
    for (int b0 = 0, p = 0; b0 < K; b0 += G, ++p) {
        const int g_here = (b0 + G <= K) ? G : K - b0;
        const int W = g_here * kNB;
        // --- panel factorisation (critical path) ---
        // The off-diagonal L tiles go straight into the ring slot (trsm out of
        // place, so two CTAs per 128-wide tile may split it); the diagonal
        // tiles stay in Z until the hand-over.
        const int slot = p % NB;
        const int rows = Npad - b0 * kNB;
        double* Lb = ring + (size_t)slot * Npad * G * kNB;
        if (trace) tr.rec(p, 0, s);
        for (int g = 0; g < g_here; ++g) {
            const int c = b0 + g;
            double* Acc = Z + (size_t)c * kNB * ld + (size_t)c * kNB;
            launch_potrf_diag(Acc, ld, Linv + (size_t)c * kNB * kNB, pivots, c * kNB, st, s, bt);
            ++launches;
            if (trace) tr.rec(p, 5, s);
            // the slot is written from here on (trsm, or the hand-over of a last one-tile panel):
            // inverse step p - NB must be done with it (waited for after the first tile kernel,
            // which then directly follows the last update)
            if (g == 0 && p >= NB) {
                SFM_CUDA(cudaStreamWaitEvent(s, eT[slot], 0));
                for (int q = 1; q < ways; ++q) SFM_CUDA(cudaStreamWaitEvent(s, isp->eT[q - 1][slot], 0));
            }
            const int below = K - c - 1;
            if (below == 0) break;
            double* Lc = Lb + (size_t)g * kNB * rows + (size_t)(g + 1) * kNB;  // L[rows > c, c] in the slot
            GemmArgs t = gemm_args(Lc, rows, Acc + kNB, ld, Linv + (size_t)c * kNB * kNB, kNB, below, 1, kNB);
            batched(t, OR, OZ, OL);
            launch_gemm(t, s);
            ++launches;
            if (trace) tr.rec(p, 6, s);
            const int inner = b0 + g_here - c - 1;
            if (inner > 0) {
                if (g == 0 && next_pending) SFM_CUDA(cudaStreamWaitEvent(s, eN, 0));  // same columns
                GemmArgs u = gemm_args(Z + (size_t)(c + 1) * kNB * ld + (size_t)(c + 1) * kNB, ld, Lc, rows, Lc, rows,
                                       below, inner, kNB);
                u.alpha_neg = 1; u.beta = 1; u.lower_only = 1;
                batched(u, OZ, OR, OR);
                launch_gemm(u, s);
                ++launches;
                if (trace) tr.rec(p, 7, s);
            }
        }
        // --- hand the panel over to the inverse: diagonal tiles into the slot,
        // the panel's W x W block of Z := I ---
        launch_panel_take_diag(Z, ld, b0, W, Lb, rows, s, bt);
        ++launches;
        SFM_CUDA(cudaEventRecord(eL[slot], s));
        if (trace) tr.rec(p, 1, s);
        const int nb0 = b0 + g_here;
        const int T2 = K - nb0;
        const int gn = (T2 < G) ? T2 : G;
        // --- Cholesky trailing update ---
        if (T2 > gn) {
            SFM_CUDA(cudaStreamWaitEvent(s2, eL[slot], 0));
            const int r0 = nb0 + gn;
            const double* Lr = Lb + W + (size_t)gn * kNB;
            GemmArgs r = gemm_args(Z + (size_t)r0 * kNB * ld + (size_t)r0 * kNB, ld, Lr, rows, Lr, rows, T2 - gn,
                                   T2 - gn, W);
            r.tri = 1; r.alpha_neg = 1; r.beta = 1;
            pad_rows(r, r0 * kNB);
            batched(r, OZ, OR, OR);
            launch_gemm(r, s2);
            ++launches;
            if (trace) tr.rec(p, 3, s2);
        }
        next_pending = false;
        if (T2 > 0) {
            // next panel: its first block column on the critical stream (the next
            // potrf / trsm need only it), the later columns on s4 concurrently
            // (the next panel's first inner update waits for them)
            if (rest_pending) SFM_CUDA(cudaStreamWaitEvent(s, eR, 0));
            if (p == 0 && eZ) SFM_CUDA(cudaStreamWaitEvent(s, eZ, 0));
            const bool split = gn > 1 && s4 != s;
            if (split) SFM_CUDA(cudaEventRecord(eX, s));
            GemmArgs u = gemm_args(Z + (size_t)nb0 * kNB * ld + (size_t)nb0 * kNB, ld, Lb + W, rows, Lb + W, rows, T2,
                                   split ? 1 : gn, W);
            u.alpha_neg = 1; u.beta = 1; u.lower_only = 1;
            pad_rows(u, nb0 * kNB);
            batched(u, OZ, OR, OR);
            launch_gemm(u, s);
            ++launches;
            if (trace) tr.rec(p, 2, s);
            if (split) {
                SFM_CUDA(cudaStreamWaitEvent(s4, eX, 0));
                GemmArgs v = gemm_args(Z + (size_t)(nb0 + 1) * kNB * ld + (size_t)nb0 * kNB, ld, Lb + W, rows,
                                       Lb + W + kNB, rows, T2, gn - 1, W);
                v.alpha_neg = 1; v.beta = 1; v.lower_only = 1; v.col_off_tiles = 1;
                pad_rows(v, nb0 * kNB);
                batched(v, OZ, OR, OR);
                launch_gemm(v, s4);
                ++launches;
                SFM_CUDA(cudaEventRecord(eN, s4));
                next_pending = true;
            }
        }
        rest_pending = false;
        if (T2 > gn) {
            SFM_CUDA(cudaEventRecord(eR, s2));
            rest_pending = true;
        }
        // --- inverse step p (rows of panel p) ---
        // The columns of X are independent: with extra inverse streams the column tiles are dealt
        // round-robin to s3 and isp->s[], so that one share's narrow in-panel launches overlap
        // another's bulk update.
        for (int q = 0; q < ways; ++q) {
            cudaStream_t si = q ? isp->s[q - 1] : s3;
            const int step = ways;
            auto ncol = [&](int cols) { return cols > q ? (cols - q + step - 1) / step : 0; };  // this half's tiles of [0, cols)
            auto half = [&](GemmArgs& a) {
                if (split_inv) { a.col_step = step; a.col_first = q; }
            };
            SFM_CUDA(cudaStreamWaitEvent(si, eL[slot], 0));
            for (int g = 0; g < g_here; ++g) {
                const int r = b0 + g;
                if (ncol(r + 1) == 0) continue;
                GemmArgs a = gemm_args(Z + (size_t)r * kNB, ld, Linv + (size_t)r * kNB * kNB, kNB, Z + (size_t)r * kNB, ld,
                                       1, ncol(r + 1), kNB);
                a.b_kmajor = 1;
                half(a);
                batched(a, OZ, OL, OZ);
                launch_gemm(a, si);
                ++launches;
                const int later = g_here - g - 1;
                if (later > 0) {
                    GemmArgs u = gemm_args(Z + (size_t)(r + 1) * kNB, ld, Lb + (size_t)g * kNB * rows + (size_t)(g + 1) * kNB,
                                           rows, Z + (size_t)r * kNB, ld, later, ncol(r + 1), kNB);
                    u.b_kmajor = 1; u.alpha_neg = 1; u.beta = 1;
                    half(u);
                    batched(u, OZ, OR, OZ);
                    launch_gemm(u, si);
                    ++launches;
                }
            }
            if (T2 > 0 && ncol(nb0) > 0) {
                GemmArgs x = gemm_args(Z + (size_t)nb0 * kNB, ld, Lb + W, rows, Z + (size_t)b0 * kNB, ld, T2, ncol(nb0), W);
                x.b_kmajor = 1; x.alpha_neg = 1; x.beta = 1; x.beta0_from = b0;
                x.k_from_col = 1;  // X[panel rows, panel columns] is lower triangular: skip its zero K range
                half(x);
                batched(x, OZ, OR, OZ);
                launch_gemm(x, si);
                ++launches;
            }
            SFM_CUDA(cudaEventRecord(q ? isp->eT[q - 1][slot] : eT[slot], si));
        }
        if (trace) tr.rec(p, 4, s3);
        last_slot = slot;
        if (debug_sync()) {
            SFM_CUDA(cudaStreamSynchronize(s));
            SFM_CUDA(cudaStreamSynchronize(s2));
            SFM_CUDA(cudaStreamSynchronize(s3));
        }
    }
    if (rest_pending) SFM_CUDA(cudaStreamWaitEvent(s, eR, 0));
    if (next_pending) SFM_CUDA(cudaStreamWaitEvent(s, eN, 0));
    if (last_slot >= 0) SFM_CUDA(cudaStreamWaitEvent(s, eT[last_slot], 0));
    for (int q = 1; q < ways && last_slot >= 0; ++q) SFM_CUDA(cudaStreamWaitEvent(s, isp->eT[q - 1][last_slot], 0));
    if (trace) tr.dump();
    return launches;
}

}  // namespace sfm
