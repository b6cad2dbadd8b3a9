// Dense Moore-Penrose reference covariance on the GPU (reference
// src/oracle.cpp:34-72, pseudoinverse_covariance): verification only.
//
// The Fisher matrix F = J^T W J (dense, N = P n + 3 m) is symmetric PSD, so
// its SVD is its eigendecomposition; this library's Jacobi eigensolver
// (eigen.cu) gives F = V diag(λ) V^T, the seven eigenvalues smallest in
// magnitude are dropped by count (never by threshold, as the reference drops
// the seven trailing singular values), and Σ = V diag(1/λ) V^T over the kept
// pairs is one DMMA GEMM of this library.  Σ is symmetrised like the
// reference's 0.5 (Σ + Σ^T).

#include "common.cuh"
#include "kernels.cuh"

#include <algorithm>
#include <cmath>
#include <string>
#include <vector>

namespace sfm {

// F (N x N, col-major, host) -> sigma (Npad x Npad device, ld Npad), eigenvalues
// (host, in the eigensolver's order).  Scratch is allocated here.
void dense_pseudoinverse(const std::vector<double>& F, int N, DBuf& dA, DBuf& dW, DBuf& dwork, DBuf& dVs, DBuf& dVk,
                         DBuf& dS, DBuf& dkeep, std::vector<double>& lam, double** sigma, long long* ld_out,
                         cudaStream_t s) {
    double* src = dS.as<double>((size_t)N * N + 1);
    SFM_CUDA(cudaMemcpyAsync(src, F.data(), 8 * (size_t)N * N, cudaMemcpyHostToDevice, s));
    double* V = nullptr;
    int ldv = 0;
    sym_eigen(src, N, N, dA, dW, dwork, lam, &V, &ldv, s);
    // drop the seven eigenvalues smallest in magnitude (by count)
    std::vector<int> order(N);
    for (int i = 0; i < N; ++i) order[i] = i;
    std::stable_sort(order.begin(), order.end(), [&](int a, int b) { return std::fabs(lam[a]) < std::fabs(lam[b]); });
    std::vector<int> keep(order.begin() + std::min(N, 7), order.end());
    std::sort(keep.begin(), keep.end());
    std::vector<double> w(keep.size());
    for (size_t k = 0; k < keep.size(); ++k) w[k] = 1.0 / lam[keep[k]];
    eig_reconstruct(V, ldv, N, keep, w, dVs, dVk, dS, dkeep, sigma, ld_out, s);
}

}  // namespace sfm
