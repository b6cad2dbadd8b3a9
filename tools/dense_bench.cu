// Standalone micro-benchmark of the dense kernels (development aid).
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -DSFM_POTRF_TIMING -I include -I paper_1808_02414_b200/csrc \
//      tools/dense_bench.cu paper_1808_02414_b200/csrc/dense.cu -o tools/dense_bench
#include "common.cuh"
#include "kernels.cuh"
#include <cstdio>
#include <vector>
#include <random>
namespace sfm { long long g_kernel_launches = 0; }
#ifdef SFM_POTRF_TIMING
namespace sfm { void debug_potrf_stamps(long long* out); }
#endif
using namespace sfm;

int main(int argc, char** argv) {
    const int N = argc > 1 ? atoi(argv[1]) : 9088;
    std::vector<double> h((size_t)N * N);
    std::mt19937_64 rng(1);
    std::uniform_real_distribution<double> u(-1, 1);
    for (int c = 0; c < N; ++c) for (int r = c; r < N; ++r) { double v = u(rng) * 0.01; h[(size_t)c * N + r] = v; h[(size_t)r * N + c] = v; }
    for (int i = 0; i < N; ++i) h[(size_t)i * N + i] = 4.0;
    double *Z, *Linv, *piv, *Lp; Status* st;
    SFM_CUDA(cudaMalloc(&Z, 8ull * N * N));
    SFM_CUDA(cudaMalloc(&Linv, 8ull * N * kNB));
    SFM_CUDA(cudaMalloc(&piv, 8ull * N));
    SFM_CUDA(cudaMalloc(&Lp, 8ull * trtri_lp_doubles(N, 8)));
    SFM_CUDA(cudaMalloc(&st, sizeof(Status)));
    cudaStream_t s, s2; int lo, hi; cudaDeviceGetStreamPriorityRange(&lo, &hi);
    cudaStreamCreateWithPriority(&s, cudaStreamNonBlocking, hi); cudaStreamCreateWithPriority(&s2, cudaStreamNonBlocking, lo);
    cudaEvent_t e1, e2, a, b; cudaEventCreateWithFlags(&e1, cudaEventDisableTiming); cudaEventCreateWithFlags(&e2, cudaEventDisableTiming);
    cudaEventCreate(&a); cudaEventCreate(&b);
    // potrf alone
    SFM_CUDA(cudaMemcpy(Z, h.data(), 8ull * N * N, cudaMemcpyHostToDevice));
    for (int rep = 0; rep < 3; ++rep) {
        cudaEventRecord(a, s);
        launch_potrf_diag(Z, N, Linv, piv, 0, st, s);
        cudaEventRecord(b, s); cudaEventSynchronize(b);
        float ms; cudaEventElapsedTime(&ms, a, b);
        printf("potrf_diag: %.1f us\n", ms * 1e3);
        SFM_CUDA(cudaMemcpy(Z, h.data(), 8ull * kNB * N, cudaMemcpyHostToDevice));
    }
#ifdef SFM_POTRF_TIMING
    long long stamps[64];
    debug_potrf_stamps(stamps);
    printf("  load: %lld cycles\n", stamps[0] - stamps[19]);
    for (int i = 1; i <= 3; ++i) printf("  stamp %2d: +%lld cycles\n", i, stamps[i] - stamps[i - 1]);
    for (int s = 0; s < 15; ++s) printf("  step %2d: potrf8+sync %lld, rest %lld\n", s, stamps[28 + s] - stamps[44 + s], stamps[45 + s] - stamps[28 + s]);
#endif
    // GEMM shapes
    for (int K : {128, 256, 384, 512}) {
        const int T = (N / kNB) - 8;
        GemmArgs g{}; g.C = Z + 8ull * kNB * N + 8 * kNB; g.ldc = N; g.A = Z + 8 * kNB; g.lda = N; g.B = Z + 8 * kNB; g.ldb = N;
        g.tm = T; g.tn = T; g.K = K; g.tri = 1; g.alpha_neg = 1; g.beta = 1; g.beta0_from = -1;
        launch_gemm(g, s); cudaStreamSynchronize(s);
        cudaEventRecord(a, s);
        for (int r = 0; r < 3; ++r) launch_gemm(g, s);
        cudaEventRecord(b, s); cudaEventSynchronize(b);
        float ms; cudaEventElapsedTime(&ms, a, b); ms /= 3;
        const double fl = 2.0 * K * (double)T * (T + 1) / 2 * kNB * kNB;
        printf("syrk-tiles T=%d K=%d: %.3f ms  %.2f TF/s\n", T, K, ms, fl / ms / 1e9);
    }
    for (int G : {1, 2, 3, 4, 6}) {
        SFM_CUDA(cudaMemcpy(Z, h.data(), 8ull * N * N, cudaMemcpyHostToDevice));
        cudaEventRecord(a, s);
        dense_cholesky(Z, N, N, G, Linv, piv, st, s, s2, e1, e2);
        cudaEventRecord(b, s);
        dense_trtri(Z, N, N, G, Linv, Lp, s, s2, e1, e2);
        cudaEvent_t c2; cudaEventCreate(&c2); cudaEventRecord(c2, s); cudaEventSynchronize(c2);
        float ms1, ms2; cudaEventElapsedTime(&ms1, a, b); cudaEventElapsedTime(&ms2, b, c2);
        const double f = (double)N * N * N / 3.0;
        printf("G=%d: cholesky %.2f ms (%.1f TF/s)  trtri %.2f ms (%.1f TF/s)\n", G, ms1, f / ms1 / 1e9, ms2, f / ms2 / 1e9);
    }
    return 0;
}
