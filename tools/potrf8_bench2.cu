// In-context microbenchmark: the 8x8 warp Cholesky with the big-kernel layout.
#include <cstdio>
#include <cuda_runtime.h>
constexpr int kNB = 128, LDT = 136, SB = 8;
__device__ __forceinline__ double fast_rsqrt(double d) {
    double y;
    asm("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(d));
    const double hd = 0.5 * d;
#pragma unroll
    for (int it = 0; it < 3; ++it) y = y * (1.5 - hd * y * y);
    return y;
}
__device__ __forceinline__ void warp_potrf8(double* T, int c0, double* rinv, double* spiv) {
    const int i = threadIdx.x & 31;
    double a[SB];
#pragma unroll
    for (int c = 0; c < SB; ++c) a[c] = (i < SB && c <= i) ? T[(c0 + c) * LDT + c0 + i] : 0.0;
    double my_inv = 1.0;
#pragma unroll
    for (int j = 0; j < SB; ++j) {
        double d = __shfl_sync(0xffffffffu, a[j], j);
        if (i == j) spiv[c0 + j] = d;
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
template <int THREADS>
__global__ void __launch_bounds__(THREADS, 1) k(const double* A, long long* cyc) {
    extern __shared__ double T[];
    double* rinv = T + kNB * LDT;
    double* spiv = rinv + kNB;
    for (int e = threadIdx.x; e < kNB * kNB; e += THREADS) {
        const int r = e & (kNB - 1), c = e >> 7;
        T[c * LDT + r] = (r >= c) ? A[(size_t)c * kNB + r] : 0.0;
    }
    __syncthreads();
    const int warp = threadIdx.x >> 5;
    for (int s = 0; s < 4; ++s) {
        __syncthreads();
        long long t0 = clock64();
        if (warp == 0) warp_potrf8(T, s * SB, rinv, spiv);
        __syncthreads();
        if (threadIdx.x == 0) cyc[s] = clock64() - t0;
    }
}
int main() {
    double h[kNB * kNB];
    for (int c = 0; c < kNB; ++c) for (int r = 0; r < kNB; ++r) h[c * kNB + r] = (r == c) ? 4.0 : 0.01 / (1 + r + c);
    double* A; cudaMalloc(&A, sizeof h); cudaMemcpy(A, h, sizeof h, cudaMemcpyHostToDevice);
    long long* c; cudaMalloc(&c, 64);
    const int smem = (kNB * LDT + 2 * kNB) * 8;
    cudaFuncSetAttribute(k<512>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    cudaFuncSetAttribute(k<32>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    long long o[4];
    k<512><<<1, 512, smem>>>(A, c); cudaMemcpy(o, c, 32, cudaMemcpyDeviceToHost);
    printf("512 threads: %lld %lld %lld %lld\n", o[0], o[1], o[2], o[3]);
    k<32><<<1, 32, smem>>>(A, c); cudaMemcpy(o, c, 32, cudaMemcpyDeviceToHost);
    printf("32 threads: %lld %lld %lld %lld\n", o[0], o[1], o[2], o[3]);
    printf("%s\n", cudaGetErrorString(cudaGetLastError()));
}
