// Diagonal-tile kernel check (development aid): accuracy of L, L^-1 and the
// pivots against a long-double Cholesky on the host, and the launch time.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 [-DSFM_POTRF_TIMING] -I include \
//      -I paper_1808_02414_b200/csrc tools/potrf_check.cu paper_1808_02414_b200/csrc/dense.cu -o tools/potrf_check
#include "common.cuh"
#include "kernels.cuh"
#include <cmath>
#include <cstdio>
#include <random>
#include <vector>
namespace sfm {
thread_local long long g_kernel_launches = 0;
#ifdef SFM_POTRF_TIMING
void debug_potrf_stamps(long long* out);
#endif
}
using namespace sfm;

static void host_chol(const std::vector<double>& a, int n, std::vector<long double>& L, std::vector<long double>& X) {
    L.assign((size_t)n * n, 0.0L);
    for (int j = 0; j < n; ++j) {
        long double d = a[(size_t)j * n + j];
        for (int k = 0; k < j; ++k) d -= L[(size_t)j * n + k] * L[(size_t)j * n + k];
        const long double ljj = sqrtl(d);
        L[(size_t)j * n + j] = ljj;
        for (int i = j + 1; i < n; ++i) {
            long double s = a[(size_t)j * n + i];
            for (int k = 0; k < j; ++k) s -= L[(size_t)i * n + k] * L[(size_t)j * n + k];
            L[(size_t)i * n + j] = s / ljj;
        }
    }
    X.assign((size_t)n * n, 0.0L);  // row-major X = L^-1
    for (int c = 0; c < n; ++c)
        for (int r = c; r < n; ++r) {
            long double s = (r == c) ? 1.0L : 0.0L;
            for (int k = c; k < r; ++k) s -= L[(size_t)r * n + k] * X[(size_t)k * n + c];
            X[(size_t)r * n + c] = s / L[(size_t)r * n + r];
        }
}

int main(int argc, char** argv) {
    const int N = 1024, n = kNB;
    const int kind = argc > 1 ? atoi(argv[1]) : 0;
    std::mt19937_64 rng(7 + kind);
    std::uniform_real_distribution<double> u(-1, 1);
    std::vector<double> h((size_t)N * N, 0.0), t((size_t)n * n);
    if (kind == 0) {  // diagonally dominant
        for (int c = 0; c < n; ++c)
            for (int r = c; r < n; ++r) { const double v = u(rng) * 0.05; t[(size_t)c * n + r] = v; t[(size_t)r * n + c] = v; }
        for (int i = 0; i < n; ++i) t[(size_t)i * n + i] = 4.0;
    } else {  // B B^T + eps I: condition ~1e8
        std::vector<double> B((size_t)n * n);
        for (auto& x : B) x = u(rng);
        for (int c = 0; c < n; ++c)
            for (int r = 0; r < n; ++r) {
                double s = 0;
                for (int k = 0; k < n; ++k) s += B[(size_t)r * n + k] * B[(size_t)c * n + k];
                t[(size_t)c * n + r] = s + (r == c ? 1e-6 : 0.0);
            }
    }
    for (int c = 0; c < n; ++c)
        for (int r = 0; r < n; ++r) h[(size_t)c * N + r] = t[(size_t)c * n + r];
    std::vector<long double> L, X;
    host_chol(t, n, L, X);
    double *Z, *Linv, *piv;
    Status* st;
    SFM_CUDA(cudaMalloc(&Z, 8ull * N * N));
    SFM_CUDA(cudaMalloc(&Linv, 8ull * n * n));
    SFM_CUDA(cudaMalloc(&piv, 8ull * N));
    SFM_CUDA(cudaMalloc(&st, sizeof(Status)));
    SFM_CUDA(cudaMemset(st, 0x7f, sizeof(Status)));
    dense_init_attributes();
    cudaStream_t s;
    cudaStreamCreate(&s);
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    float best = 1e9f;
    for (int rep = 0; rep < 10; ++rep) {
        SFM_CUDA(cudaMemcpy(Z, h.data(), 8ull * N * N, cudaMemcpyHostToDevice));
        cudaEventRecord(a, s);
        launch_potrf_diag(Z, N, Linv, piv, 0, st, s);
        cudaEventRecord(b, s);
        SFM_CUDA(cudaEventSynchronize(b));
        float ms;
        cudaEventElapsedTime(&ms, a, b);
        if (ms < best) best = ms;
#ifdef SFM_POTRF_TIMING
        long long tt[64];
        debug_potrf_stamps(tt);
        if (rep == 9)
            printf("cycles: load %lld | factor %lld | pivots %lld | Y %lld | write %lld\n", tt[0] - tt[19], tt[4] - tt[0],
                   tt[1] - tt[4], tt[2] - tt[1], tt[3] - tt[2]);
#endif
    }
    std::vector<double> hz((size_t)N * N), hl((size_t)n * n), hp(n);
    SFM_CUDA(cudaMemcpy(hz.data(), Z, 8ull * N * N, cudaMemcpyDeviceToHost));
    SFM_CUDA(cudaMemcpy(hl.data(), Linv, 8ull * n * n, cudaMemcpyDeviceToHost));
    SFM_CUDA(cudaMemcpy(hp.data(), piv, 8ull * n, cudaMemcpyDeviceToHost));
    long double eL = 0, mL = 0, eX = 0, mX = 0, eP = 0;
    bool upper_ok = true, rest_ok = true;
    for (int c = 0; c < n; ++c)
        for (int r = 0; r < n; ++r) {
            const long double lr = L[(size_t)r * n + c], xr = X[(size_t)r * n + c];
            if (r >= c) { eL = fmaxl(eL, fabsl(hz[(size_t)c * N + r] - lr)); mL = fmaxl(mL, fabsl(lr)); }
            else if (hz[(size_t)c * N + r] != h[(size_t)c * N + r]) upper_ok = false;  // upper triangle untouched
            eX = fmaxl(eX, fabsl(hl[(size_t)c * n + r] - xr));
            mX = fmaxl(mX, fabsl(xr));
        }
    for (int c = n; c < N; ++c)
        if (hz[(size_t)c * N] != 0.0) rest_ok = false;
    for (int j = 0; j < n; ++j) {
        const long double p = L[(size_t)j * n + j] * L[(size_t)j * n + j];
        eP = fmaxl(eP, fabsl(hp[j] - p) / p);
    }
    printf("kind %d  %.2f us  |L err| %.3Le  |Linv err| %.3Le  pivot rel %.3Le  upper %s rest %s\n", kind, best * 1e3,
           eL / mL, eX / mX, eP, upper_ok ? "kept" : "CHANGED", rest_ok ? "kept" : "CHANGED");
    return 0;
}
