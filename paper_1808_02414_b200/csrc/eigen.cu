// Symmetric eigendecomposition on the GPU: parallel cyclic Jacobi.
//
// Used where the reference needs a dense symmetric solve that is not the
// product path's SPD Cholesky route:
//   * pseudoinverse_covariance (src/oracle.cpp:34-72): SVD of the PSD Fisher
//     matrix = its eigendecomposition, the 7 smallest dropped by count;
//   * invert_schur on an arbitrary symmetric (indefinite) matrix
//     (src/covariance.cpp:196-257): A^-1 = V diag(1/λ) V^T, inertia from the
//     signs of λ;
//   * full_covariance (src/covariance.cpp:352-397): the parameter block of
//     the bordered Fisher inverse.
//
// Algorithm: two-sided Jacobi with the round-robin (circle) ordering, so
// every step rotates n/2 disjoint planes at once.  Per step one kernel forms
// the n/2 rotations from the current 2x2 diagonal blocks, a second applies
// A <- R^T A R block by block (thread per pair of planes, upper triangle,
// mirrored) and V <- V R.  Sweeps repeat until no off-diagonal entry exceeds
// max(1e-16 sqrt|a_pp a_qq|, 1e-18 ||A||_F).  Jacobi is accurate for the
// small eigenvalues that decide a gauge (relative, not just ||A||-absolute,
// accuracy on graded matrices), which is what the oracle's count-based cut
// of the 7 gauge directions relies on.  Odd orders are padded with a zero row
// and column that never rotates.
#include "common.cuh"
#include "kernels.cuh"

#include <algorithm>
#include <cmath>
#include <string>
#include <vector>

namespace sfm {

namespace {

// circle method: m = n2 - 1 (odd) positions rotate, player m is fixed;
// round r pairs (m, r) and ((r + k) mod m, (r - k) mod m), k = 1 .. n2/2 - 1
__device__ __forceinline__ void rr_pair(int n2, int r, int i, int* p, int* q) {
    const int m = n2 - 1;
    int a, b;
    if (i == 0) {
        a = m;
        b = r;
    } else {
        a = (r + i) % m;
        b = (r - i + m) % m;
    }
    *p = min(a, b);
    *q = max(a, b);
}

__global__ void k_jac_angles(const double* A, int n2, int r, double tol_abs, double* cs, int* rotated) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n2 / 2) return;
    int p, q;
    rr_pair(n2, r, i, &p, &q);
    const double app = A[(size_t)p * n2 + p], aqq = A[(size_t)q * n2 + q], apq = A[(size_t)q * n2 + p];
    double c = 1.0, s = 0.0;
    if (fabs(apq) > fmax(1e-16 * sqrt(fabs(app * aqq)), tol_abs)) {
        const double theta = (aqq - app) / (2.0 * apq);
        const double t = (theta >= 0.0 ? 1.0 : -1.0) / (fabs(theta) + sqrt(1.0 + theta * theta));
        c = 1.0 / sqrt(1.0 + t * t);
        s = t * c;
        atomicAdd(rotated, 1);
    }
    cs[2 * i] = c;
    cs[2 * i + 1] = s;
}

// Thread per (plane i, plane j), i <= j: the 2x2 block A[{p_i, q_i}, {p_j, q_j}]
// <- R_i^T B R_j, written to both triangles; then V rows.  R = [[c, s], [-s, c]].
__global__ void k_jac_apply(double* A, double* V, int n2, int r, const double* cs) {
    const int h = n2 / 2;
    const long long npairs = (long long)h * (h + 1) / 2;
    const long long e = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (e < npairs) {
        // triangular index e -> (i, j), i <= j
        int j = (int)((sqrt(8.0 * (double)e + 1.0) - 1.0) * 0.5);
        while ((long long)(j + 1) * (j + 2) / 2 <= e) ++j;
        while ((long long)j * (j + 1) / 2 > e) --j;
        const int i = (int)(e - (long long)j * (j + 1) / 2);
        int pi, qi, pj, qj;
        rr_pair(n2, r, i, &pi, &qi);
        rr_pair(n2, r, j, &pj, &qj);
        const double ci = cs[2 * i], si = cs[2 * i + 1], cj = cs[2 * j], sj = cs[2 * j + 1];
        if (si == 0.0 && sj == 0.0) return;
        const double b00 = A[(size_t)pj * n2 + pi], b01 = A[(size_t)qj * n2 + pi];
        const double b10 = A[(size_t)pj * n2 + qi], b11 = A[(size_t)qj * n2 + qi];
        // B R_j
        const double c00 = cj * b00 - sj * b01, c01 = sj * b00 + cj * b01;
        const double c10 = cj * b10 - sj * b11, c11 = sj * b10 + cj * b11;
        // R_i^T (B R_j)
        double d00 = ci * c00 - si * c10, d01 = ci * c01 - si * c11;
        double d10 = si * c00 + ci * c10, d11 = si * c01 + ci * c11;
        if (i == j) {  // the rotated plane itself: exact zero off the diagonal
            d01 = 0.0;
            d10 = 0.0;
        }
        A[(size_t)pj * n2 + pi] = d00;
        A[(size_t)qj * n2 + pi] = d01;
        A[(size_t)pj * n2 + qi] = d10;
        A[(size_t)qj * n2 + qi] = d11;
        if (i != j) {
            A[(size_t)pi * n2 + pj] = d00;
            A[(size_t)qi * n2 + pj] = d10;
            A[(size_t)pi * n2 + qj] = d01;
            A[(size_t)qi * n2 + qj] = d11;
        }
        return;
    }
    const long long f = e - npairs;  // V: thread per (row, plane)
    if (f >= (long long)n2 * h) return;
    const int row = (int)(f % n2), i = (int)(f / n2);
    const double c = cs[2 * i], s = cs[2 * i + 1];
    if (s == 0.0) return;
    int p, q;
    rr_pair(n2, r, i, &p, &q);
    const double vp = V[(size_t)p * n2 + row], vq = V[(size_t)q * n2 + row];
    V[(size_t)p * n2 + row] = c * vp - s * vq;
    V[(size_t)q * n2 + row] = s * vp + c * vq;
}

__global__ void k_jac_init(const double* src, long long lds, int n, int n2, double* A, double* V) {
    const long long e = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (e >= (long long)n2 * n2) return;
    const int r = (int)(e % n2), c = (int)(e / n2);
    A[e] = (r < n && c < n) ? src[(size_t)c * lds + r] : 0.0;
    V[e] = r == c ? 1.0 : 0.0;
}

__global__ void k_jac_diag(const double* A, int n2, double* lam) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n2) lam[i] = A[(size_t)i * n2 + i];
}

__global__ void k_fro2(const double* A, long long count, double* out) {
    __shared__ double red[256];
    double acc = 0.0;
    for (long long e = blockIdx.x * 256LL + threadIdx.x; e < count; e += 256LL * gridDim.x) acc += A[e] * A[e];
    red[threadIdx.x] = acc;
    __syncthreads();
    for (int w = 128; w > 0; w >>= 1) {
        if (threadIdx.x < w) red[threadIdx.x] += red[threadIdx.x + w];
        __syncthreads();
    }
    if (threadIdx.x == 0) out[blockIdx.x] = red[0];
}

// out[:, k] = V[:, keep_k] * w_k (w = 1/λ or 1), columns padded to ldo rows
__global__ void k_eig_cols(const double* V, int n2, int n, const int* keep, const double* w, int nk, double* out,
                           long long ldo) {
    const long long e = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (e >= (long long)n * nk) return;
    const int r = (int)(e % n), k = (int)(e / n);
    out[(size_t)k * ldo + r] = V[(size_t)keep[k] * n2 + r] * w[k];
}

__global__ void k_sym_avg(double* S, long long ld, int n) {
    const long long e = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (e >= (long long)n * n) return;
    const int r = (int)(e % n), c = (int)(e / n);
    if (r <= c) return;
    const double v = 0.5 * (S[(size_t)c * ld + r] + S[(size_t)r * ld + c]);
    S[(size_t)c * ld + r] = v;
    S[(size_t)r * ld + c] = v;
}

}  // namespace

int sym_eigen(const double* src, long long lds, int n, DBuf& dA, DBuf& dV, DBuf& dwork, std::vector<double>& lam,
              double** V_out, int* ld_out, cudaStream_t s) {
    const int n2 = n + (n & 1);
    double* A = dA.as<double>((size_t)n2 * n2 + 1);
    double* V = dV.as<double>((size_t)n2 * n2 + 1);
    double* w = dwork.as<double>(4 * (size_t)n2 + 512);
    double* cs = w;
    double* dl = w + n2;
    double* fro = w + 2 * (size_t)n2;
    int* rotated = reinterpret_cast<int*>(w + 2 * (size_t)n2 + 300);
    if (n2)
        k_jac_init<<<cdiv((long long)n2 * n2, 256), 256, 0, s>>>(src, lds, n, n2, A, V);
    SFM_LAUNCH_CHECK();
    double norm = 0.0;
    {
        const int nb = (int)std::min<long long>(256, cdiv((long long)n2 * n2 + 1, 256));
        k_fro2<<<nb, 256, 0, s>>>(A, (long long)n2 * n2, fro);
        SFM_LAUNCH_CHECK();
        std::vector<double> part(nb);
        SFM_CUDA(cudaMemcpyAsync(part.data(), fro, 8 * (size_t)nb, cudaMemcpyDeviceToHost, s));
        SFM_CUDA(cudaStreamSynchronize(s));
        for (double v : part) norm += v;
        norm = std::sqrt(norm);
    }
    const double tol_abs = std::max(1e-18 * norm, 1e-300);
    int sweeps = 0;
    const int h = n2 / 2;
    const long long work = (long long)h * (h + 1) / 2 + (long long)n2 * h;
    for (; n2 >= 2 && sweeps < 40; ++sweeps) {
        SFM_CUDA(cudaMemsetAsync(rotated, 0, sizeof(int), s));
        for (int r = 0; r < n2 - 1; ++r) {
            k_jac_angles<<<cdiv(h, 128), 128, 0, s>>>(A, n2, r, tol_abs, cs, rotated);
            SFM_LAUNCH_CHECK();
            k_jac_apply<<<cdiv(work, 256), 256, 0, s>>>(A, V, n2, r, cs);
            SFM_LAUNCH_CHECK();
        }
        int hrot = 0;
        SFM_CUDA(cudaMemcpyAsync(&hrot, rotated, sizeof(int), cudaMemcpyDeviceToHost, s));
        SFM_CUDA(cudaStreamSynchronize(s));
        if (hrot == 0) break;
    }
    if (n2) {
        k_jac_diag<<<cdiv(n2, 256), 256, 0, s>>>(A, n2, dl);
        SFM_LAUNCH_CHECK();
    }
    lam.resize(n);
    SFM_CUDA(cudaMemcpyAsync(lam.data(), dl, 8 * (size_t)n, cudaMemcpyDeviceToHost, s));
    SFM_CUDA(cudaStreamSynchronize(s));
    *V_out = V;
    *ld_out = n2;
    return sweeps;
}

void eig_reconstruct(const double* V, int ldv, int n, const std::vector<int>& keep, const std::vector<double>& wts,
                     DBuf& dL, DBuf& dR, DBuf& dS, DBuf& dkeep, double** S_out, long long* ld_out, cudaStream_t s) {
    const int nk = (int)keep.size();
    const int Npad = ((n + kNB - 1) / kNB) * kNB;
    const int Kpad = std::max(16, ((nk + 15) / 16) * 16);
    double* L = dL.as<double>((size_t)Npad * Kpad);
    double* R = dR.as<double>((size_t)Npad * Kpad);
    SFM_CUDA(cudaMemsetAsync(L, 0, 8 * (size_t)Npad * Kpad, s));
    SFM_CUDA(cudaMemsetAsync(R, 0, 8 * (size_t)Npad * Kpad, s));
    // weights, unit weights, then the kept column ids (as ints)
    double* buf = dkeep.as<double>(3 * (size_t)nk + 4);
    double* dw = buf;
    double* dones = buf + nk;
    int* dk = reinterpret_cast<int*>(buf + 2 * (size_t)nk + 2);
    const std::vector<double> ones(nk, 1.0);
    SFM_CUDA(cudaMemcpyAsync(dk, keep.data(), 4 * (size_t)nk, cudaMemcpyHostToDevice, s));
    SFM_CUDA(cudaMemcpyAsync(dw, wts.data(), 8 * (size_t)nk, cudaMemcpyHostToDevice, s));
    SFM_CUDA(cudaMemcpyAsync(dones, ones.data(), 8 * (size_t)nk, cudaMemcpyHostToDevice, s));
    const long long tot = (long long)n * nk;
    if (tot) {
        k_eig_cols<<<cdiv(tot, 256), 256, 0, s>>>(V, ldv, n, dk, dw, nk, L, Npad);
        SFM_LAUNCH_CHECK();
        k_eig_cols<<<cdiv(tot, 256), 256, 0, s>>>(V, ldv, n, dk, dones, nk, R, Npad);
        SFM_LAUNCH_CHECK();
    }
    double* S = dS.as<double>((size_t)Npad * Npad);
    const int T = Npad / kNB;
    if (T) {
        GemmArgs g = gemm_args(S, Npad, L, Npad, R, Npad, T, T, Kpad);
        launch_gemm(g, s);
        k_sym_avg<<<cdiv((long long)n * n, 256), 256, 0, s>>>(S, Npad, n);
        SFM_LAUNCH_CHECK();
    }
    SFM_CUDA(cudaStreamSynchronize(s));
    *S_out = S;
    *ld_out = Npad;
}

}  // namespace sfm
