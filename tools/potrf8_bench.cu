// Microbenchmark of the 8x8 warp Cholesky variants (development aid).
#include <cstdio>
#include <cuda_runtime.h>
__device__ __forceinline__ double fast_rsqrt(double d) {
    double y;
    asm("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(d));
    const double hd = 0.5 * d;
#pragma unroll
    for (int it = 0; it < 3; ++it) y = y * (1.5 - hd * y * y);
    return y;
}
template <int MODE>
__device__ __forceinline__ void chol8(double* T, int ld, double* piv, int* flag) {
    const int i = threadIdx.x & 31;
    double a[8];
#pragma unroll
    for (int c = 0; c < 8; ++c) a[c] = (i < 8 && c <= i) ? T[c * ld + i] : 0.0;
#pragma unroll
    for (int j = 0; j < 8; ++j) {
        double d = __shfl_sync(0xffffffffu, a[j], j);
        if (MODE == 0) {
            if (i == 0) { piv[j] = d; if (!(d > 0.0) || !isfinite(d)) atomicMin(flag, j); }
            if (!(d > 0.0) || !isfinite(d)) d = 1.0;
        }
        const double inv = (MODE == 2) ? 1.0 / sqrt(d) : fast_rsqrt(d);
        if (i == j) a[j] = d * inv;
        else if (i > j) a[j] = a[j] * inv;
#pragma unroll
        for (int c = j + 1; c < 8; ++c) {
            const double lc = __shfl_sync(0xffffffffu, a[j], c);
            if (i >= c) a[c] -= a[j] * lc;
        }
    }
    if (i < 8)
#pragma unroll
        for (int c = 0; c < 8; ++c) if (c <= i) T[c * ld + i] = a[c];
}
template <int MODE>
__global__ void k(double* out, long long* cyc, int reps, double* gpiv) {
    __shared__ double T[8 * 9], B[8 * 9];
    __shared__ double piv[8];
    __shared__ int flag;
    if (threadIdx.x < 64) { int r = threadIdx.x % 8, c = threadIdx.x / 8; B[c * 9 + r] = (r == c) ? 4.0 : 0.1 / (1 + r + c); }
    __syncthreads();
    long long t0 = clock64();
    for (int it = 0; it < reps; ++it) {
        if (threadIdx.x < 72) T[threadIdx.x] = B[threadIdx.x];
        __syncthreads();
        if (threadIdx.x < 32) chol8<MODE>(T, 9, gpiv ? gpiv : piv, &flag);
        __syncthreads();
    }
    long long t1 = clock64();
    if (threadIdx.x == 0) { cyc[MODE + 3 * (reps == 1)] = (t1 - t0) / reps; out[0] = T[0] + T[63]; }
}
int main() {
    double* o; long long* c; cudaMalloc(&o, 64); cudaMalloc(&c, 128);
    double* gp; cudaMalloc(&gp, 64);
    k<0><<<1, 512>>>(o, c, 1000, gp); k<1><<<1, 512>>>(o, c, 1000, gp); k<2><<<1, 512>>>(o, c, 1000, gp);
    k<0><<<1, 512>>>(o, c, 1, gp); k<1><<<1, 512>>>(o, c, 1, gp); k<2><<<1, 512>>>(o, c, 1, gp);
    long long h[6]; cudaMemcpy(h, c, 48, cudaMemcpyDeviceToHost);
    printf("warm chol8 cycles/call: full %lld, no-piv %lld, ieee-rsqrt %lld\n", h[0], h[1], h[2]);
    printf("cold chol8 cycles/call: full %lld, no-piv %lld, ieee-rsqrt %lld\n", h[3], h[4], h[5]);
}
