// Checks the fragment layout assumed for mma.sync.m16n8k16.row.col.f64 against
// a host product (development aid for k_gemm's MMA shape).
// nvcc -gencode arch=compute_100a,code=sm_100a -O2 -o /tmp/dmma16 tools/probe/dmma16_layout.cu
#include <cstdio>
#include <cmath>
__global__ void k(const double* A, const double* B, double* C) {  // A 16x16 row-major, B 16x8 (k x n) row-major
    const int lane = threadIdx.x, g = lane >> 2, t = lane & 3;
    double a[8], b[4], c[4] = {0, 0, 0, 0};
    for (int i = 0; i < 8; ++i) a[i] = A[(g + 8 * (i % 2)) * 16 + t + 4 * (i / 2)];
    for (int i = 0; i < 4; ++i) b[i] = B[(t + 4 * i) * 8 + g];
    asm volatile("mma.sync.aligned.m16n8k16.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5,%6,%7,%8,%9,%10,%11}, "
                 "{%12,%13,%14,%15}, {%0,%1,%2,%3};\n"
                 : "+d"(c[0]), "+d"(c[1]), "+d"(c[2]), "+d"(c[3])
                 : "d"(a[0]), "d"(a[1]), "d"(a[2]), "d"(a[3]), "d"(a[4]), "d"(a[5]), "d"(a[6]), "d"(a[7]),
                   "d"(b[0]), "d"(b[1]), "d"(b[2]), "d"(b[3]));
    for (int i = 0; i < 4; ++i) C[(g + 8 * (i / 2)) * 8 + 2 * t + (i % 2)] = c[i];
}
int main() {
    double hA[256], hB[128], hC[128], ref[128];
    for (int i = 0; i < 256; ++i) hA[i] = std::sin(0.37 * i + 1.0);
    for (int i = 0; i < 128; ++i) hB[i] = std::cos(0.11 * i + 0.5);
    for (int r = 0; r < 16; ++r)
        for (int c = 0; c < 8; ++c) {
            double s = 0;
            for (int q = 0; q < 16; ++q) s += hA[r * 16 + q] * hB[q * 8 + c];
            ref[r * 8 + c] = s;
        }
    double *dA, *dB, *dC;
    cudaMalloc(&dA, sizeof hA); cudaMalloc(&dB, sizeof hB); cudaMalloc(&dC, sizeof hC);
    cudaMemcpy(dA, hA, sizeof hA, cudaMemcpyHostToDevice);
    cudaMemcpy(dB, hB, sizeof hB, cudaMemcpyHostToDevice);
    k<<<1, 32>>>(dA, dB, dC);
    cudaMemcpy(hC, dC, sizeof hC, cudaMemcpyDeviceToHost);
    double e = 0;
    for (int i = 0; i < 128; ++i) e = std::fmax(e, std::fabs(hC[i] - ref[i]));
    std::printf("m16n8k16 f64 layout: max |err| %.3e (%s)\n", e, e < 1e-12 ? "ok" : "WRONG");
    return e < 1e-12 ? 0 : 1;
}
