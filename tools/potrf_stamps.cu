// Phase timing of one diagonal-tile Cholesky + inverse (development aid).
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -DSFM_POTRF_TIMING -I include -I paper_1808_02414_b200/csrc \
//      tools/potrf_stamps.cu paper_1808_02414_b200/csrc/dense.cu -o tools/potrf_stamps
#include "common.cuh"
#include "kernels.cuh"
#include <cstdio>
#include <random>
#include <vector>
namespace sfm {
thread_local long long g_kernel_launches = 0;
void debug_potrf_stamps(long long* out);
}
using namespace sfm;

int main() {
    const int N = 1024;
    std::vector<double> h((size_t)N * N);
    std::mt19937_64 rng(1);
    std::uniform_real_distribution<double> u(-1, 1);
    for (int c = 0; c < N; ++c)
        for (int r = c; r < N; ++r) { const double v = u(rng) * 0.01; h[(size_t)c * N + r] = v; h[(size_t)r * N + c] = v; }
    for (int i = 0; i < N; ++i) h[(size_t)i * N + i] = 4.0;
    double *Z, *Linv, *piv;
    Status* st;
    SFM_CUDA(cudaMalloc(&Z, 8ull * N * N));
    SFM_CUDA(cudaMalloc(&Linv, 8ull * kNB * kNB));
    SFM_CUDA(cudaMalloc(&piv, 8ull * N));
    SFM_CUDA(cudaMalloc(&st, sizeof(Status)));
    dense_init_attributes();
    cudaStream_t s;
    cudaStreamCreate(&s);
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    for (int rep = 0; rep < 5; ++rep) {
        SFM_CUDA(cudaMemcpy(Z, h.data(), 8ull * N * N, cudaMemcpyHostToDevice));
        cudaEventRecord(a, s);
        launch_potrf_diag(Z, N, Linv, piv, 0, st, s);
        cudaEventRecord(b, s);
        cudaEventSynchronize(b);
        float ms;
        cudaEventElapsedTime(&ms, a, b);
        long long t[64];
        debug_potrf_stamps(t);
        printf("potrf_diag %.1f us | load %lld | factor %lld | diag-inverses+ %lld | Y %lld | write %lld cycles\n", ms * 1e3,
               t[0] - t[19], t[4] - t[0], t[1] - t[4], t[2] - t[1], t[3] - t[2]);
    }
    return 0;
}
