// Dense Moore-Penrose reference covariance on the GPU (reference
// src/oracle.cpp:34-72, pseudoinverse_covariance): verification only.
//
// The Fisher matrix F = J^T W J (dense, N = P n + 3 m) is symmetric PSD, so
// its SVD is its eigendecomposition; cuSOLVER syevd (a library call, loaded at
// run time like NCCL) gives F = V diag(λ) V^T, the seven eigenvalues smallest
// in magnitude are dropped by count (never by threshold, as the reference
// drops the seven trailing singular values), and Σ = V_s V^T with
// V_s = V diag(1/λ) is one DMMA GEMM of this library.  Σ is symmetrised like
// the reference's 0.5 (Σ + Σ^T).

#include "common.cuh"
#include "kernels.cuh"

#include <cusolverDn.h>
#include <dlfcn.h>

#include <algorithm>
#include <cmath>
#include <string>
#include <vector>

namespace sfm {

namespace {
struct Cusolver {
    bool ok = false;
    std::string why;
    cusolverStatus_t (*Create)(cusolverDnHandle_t*) = nullptr;
    cusolverStatus_t (*Destroy)(cusolverDnHandle_t) = nullptr;
    cusolverStatus_t (*SetStream)(cusolverDnHandle_t, cudaStream_t) = nullptr;
    cusolverStatus_t (*BufferSize)(cusolverDnHandle_t, cusolverEigMode_t, cublasFillMode_t, int, const double*, int,
                                   const double*, int*) = nullptr;
    cusolverStatus_t (*Syevd)(cusolverDnHandle_t, cusolverEigMode_t, cublasFillMode_t, int, double*, int, double*,
                              double*, int, int*) = nullptr;
};

Cusolver& cusolver() {
    static Cusolver c = [] {
        Cusolver a;
        void* lib = dlopen("libcusolver.so.11", RTLD_NOW | RTLD_GLOBAL);
        if (!lib) lib = dlopen("/usr/local/cuda/lib64/libcusolver.so.11", RTLD_NOW | RTLD_GLOBAL);
        if (!lib) {
            a.why = "libcusolver.so.11 not found";
            return a;
        }
        a.Create = (decltype(a.Create))dlsym(lib, "cusolverDnCreate");
        a.Destroy = (decltype(a.Destroy))dlsym(lib, "cusolverDnDestroy");
        a.SetStream = (decltype(a.SetStream))dlsym(lib, "cusolverDnSetStream");
        a.BufferSize = (decltype(a.BufferSize))dlsym(lib, "cusolverDnDsyevd_bufferSize");
        a.Syevd = (decltype(a.Syevd))dlsym(lib, "cusolverDnDsyevd");
        a.ok = a.Create && a.Destroy && a.SetStream && a.BufferSize && a.Syevd;
        if (!a.ok) a.why = "libcusolver lacks a required symbol";
        return a;
    }();
    return c;
}

// V_s[:, k] = V[:, idx_k] / λ_idx_k for the kept eigenpairs (N - 7 columns).
__global__ void k_scale_cols(const double* V, long long ldv, int N, const int* keep, const double* lam, int nk,
                             double* Vs, double* Vk, long long lds) {
    const long long e = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (e >= (long long)N * nk) return;
    const int r = (int)(e % N), k = (int)(e / N);
    const int c = keep[k];
    const double v = V[(size_t)c * ldv + r];
    Vs[(size_t)k * lds + r] = v / lam[c];
    Vk[(size_t)k * lds + r] = v;
}

__global__ void k_symmetrize(double* S, long long ld, int N) {
    const long long e = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (e >= (long long)N * N) return;
    const int r = (int)(e % N), c = (int)(e / N);
    if (r <= c) return;
    const double a = S[(size_t)c * ld + r], b = S[(size_t)r * ld + c];
    const double v = 0.5 * (a + b);
    S[(size_t)c * ld + r] = v;
    S[(size_t)r * ld + c] = v;
}
}  // namespace

bool cusolver_available(std::string* why) {
    if (!cusolver().ok && why) *why = cusolver().why;
    return cusolver().ok;
}

// F (N x N, col-major, host) -> sigma (Npad x Npad device, ld Npad), eigenvalues
// ascending (host).  Scratch is allocated here.
void dense_pseudoinverse(const std::vector<double>& F, int N, DBuf& dA, DBuf& dW, DBuf& dwork, DBuf& dVs, DBuf& dVk,
                         DBuf& dS, DBuf& dkeep, std::vector<double>& lam, double** sigma, long long* ld_out,
                         cudaStream_t s) {
    Cusolver& cs = cusolver();
    if (!cs.ok) throw CudaError("cuSOLVER unavailable: " + cs.why);
    double* A = dA.as<double>((size_t)N * N);
    double* W = dW.as<double>((size_t)N);
    SFM_CUDA(cudaMemcpyAsync(A, F.data(), 8 * (size_t)N * N, cudaMemcpyHostToDevice, s));
    cusolverDnHandle_t hs = nullptr;
    if (cs.Create(&hs) != CUSOLVER_STATUS_SUCCESS) throw CudaError("cusolverDnCreate failed");
    struct Guard {
        Cusolver& cs;
        cusolverDnHandle_t h;
        ~Guard() { cs.Destroy(h); }
    } guard{cs, hs};
    cs.SetStream(hs, s);
    int lwork = 0;
    if (cs.BufferSize(hs, CUSOLVER_EIG_MODE_VECTOR, CUBLAS_FILL_MODE_LOWER, N, A, N, W, &lwork) != CUSOLVER_STATUS_SUCCESS)
        throw CudaError("cusolverDnDsyevd_bufferSize failed");
    double* work = dwork.as<double>((size_t)lwork + 1);
    int* info = reinterpret_cast<int*>(dwork.as<double>((size_t)lwork + 2) + lwork);
    if (cs.Syevd(hs, CUSOLVER_EIG_MODE_VECTOR, CUBLAS_FILL_MODE_LOWER, N, A, N, W, work, lwork, info) !=
        CUSOLVER_STATUS_SUCCESS)
        throw CudaError("cusolverDnDsyevd failed");
    int hinfo = 0;
    SFM_CUDA(cudaMemcpyAsync(&hinfo, info, sizeof(int), cudaMemcpyDeviceToHost, s));
    lam.resize(N);
    SFM_CUDA(cudaMemcpyAsync(lam.data(), W, 8 * (size_t)N, cudaMemcpyDeviceToHost, s));
    SFM_CUDA(cudaStreamSynchronize(s));
    if (hinfo != 0) throw CudaError("eigendecomposition failed with status " + std::to_string(hinfo));
    // drop the seven eigenvalues smallest in magnitude (by count)
    std::vector<int> order(N);
    for (int i = 0; i < N; ++i) order[i] = i;
    std::stable_sort(order.begin(), order.end(), [&](int a, int b) { return std::fabs(lam[a]) < std::fabs(lam[b]); });
    std::vector<int> keep(order.begin() + std::min(N, 7), order.end());
    std::sort(keep.begin(), keep.end());
    const int nk = (int)keep.size();
    const int Npad = ((N + kNB - 1) / kNB) * kNB;
    const int Kpad = ((nk + 15) / 16) * 16;
    double* Vs = dVs.as<double>((size_t)Npad * Kpad);
    double* Vk = dVk.as<double>((size_t)Npad * Kpad);
    SFM_CUDA(cudaMemsetAsync(Vs, 0, 8 * (size_t)Npad * Kpad, s));
    SFM_CUDA(cudaMemsetAsync(Vk, 0, 8 * (size_t)Npad * Kpad, s));
    int* dk = reinterpret_cast<int*>(dkeep.as<int>((size_t)nk + 1));
    SFM_CUDA(cudaMemcpyAsync(dk, keep.data(), 4 * (size_t)nk, cudaMemcpyHostToDevice, s));
    const long long tot = (long long)N * nk;
    if (tot) k_scale_cols<<<cdiv(tot, 256), 256, 0, s>>>(A, N, N, dk, W, nk, Vs, Vk, Npad);
    SFM_LAUNCH_CHECK();
    // Σ = V_s V_k^T: C (Npad x Npad) = A B^T with A = V_s (Npad x Kpad, ld Npad), B(n, k) = V_k[k * Npad + n]
    double* S = dS.as<double>((size_t)Npad * Npad);
    const int T = Npad / kNB;
    GemmArgs g = gemm_args(S, Npad, Vs, Npad, Vk, Npad, T, T, Kpad);
    launch_gemm(g, s);
    const long long tt = (long long)N * N;
    k_symmetrize<<<cdiv(tt, 256), 256, 0, s>>>(S, Npad, N);
    SFM_LAUNCH_CHECK();
    SFM_CUDA(cudaStreamSynchronize(s));
    // the keep buffers are sized nk + 1 ints; the staging vector keeps `keep` alive until here
    *sigma = S;
    *ld_out = Npad;
}

}  // namespace sfm
