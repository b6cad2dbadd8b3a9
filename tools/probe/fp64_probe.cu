// FP64 throughput probe: DMMA shapes vs DFMA, plus cuBLAS DGEMM and cuSOLVER dpotrf + dtrtri yardsticks
// (the library pair against which the fused Cholesky / inverse sweep is judged).
// build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/probe/fp64_probe tools/probe/fp64_probe.cu -lcublas -lcusolver
#include <cstdio>
#include <cstdlib>
#include <vector>
#include <cuda_runtime.h>
#include <cublas_v2.h>
#include <cusolverDn.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("CUDA %s at %d\n", cudaGetErrorString(e), __LINE__); exit(1);} } while (0)

template <int ACC>
__global__ void dmma_m8n8k4(double* out, int iters) {
  double a = threadIdx.x * 1e-3, b = 1.0 + threadIdx.x * 1e-4;
  double c[ACC][2];
  for (int i = 0; i < ACC; ++i) c[i][0] = c[i][1] = 0.0;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < ACC; ++i)
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                   : "+d"(c[i][0]), "+d"(c[i][1]) : "d"(a), "d"(b));
  }
  double s = 0; for (int i = 0; i < ACC; ++i) s += c[i][0] + c[i][1];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

template <int ACC>
__global__ void dmma_m16n8k16(double* out, int iters) {
  double a[8], b[4];
  for (int i = 0; i < 8; ++i) a[i] = threadIdx.x * 1e-3 + i;
  for (int i = 0; i < 4; ++i) b[i] = 1.0 + threadIdx.x * 1e-4 + i;
  double c[ACC][4];
  for (int i = 0; i < ACC; ++i) c[i][0] = c[i][1] = c[i][2] = c[i][3] = 0.0;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < ACC; ++i)
      asm volatile("mma.sync.aligned.m16n8k16.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5,%6,%7,%8,%9,%10,%11}, {%12,%13,%14,%15}, {%0,%1,%2,%3};"
                   : "+d"(c[i][0]), "+d"(c[i][1]), "+d"(c[i][2]), "+d"(c[i][3])
                   : "d"(a[0]), "d"(a[1]), "d"(a[2]), "d"(a[3]), "d"(a[4]), "d"(a[5]), "d"(a[6]), "d"(a[7]),
                     "d"(b[0]), "d"(b[1]), "d"(b[2]), "d"(b[3]));
  }
  double s = 0; for (int i = 0; i < ACC; ++i) s += c[i][0] + c[i][1] + c[i][2] + c[i][3];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

template <int ACC>
__global__ void dmma_m16n8k4(double* out, int iters) {
  double a0 = threadIdx.x * 1e-3, a1 = a0 + 1, b = 1.0 + threadIdx.x * 1e-4;
  double c[ACC][4];
  for (int i = 0; i < ACC; ++i) c[i][0] = c[i][1] = c[i][2] = c[i][3] = 0.0;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < ACC; ++i)
      asm volatile("mma.sync.aligned.m16n8k4.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5}, {%6}, {%0,%1,%2,%3};"
                   : "+d"(c[i][0]), "+d"(c[i][1]), "+d"(c[i][2]), "+d"(c[i][3]) : "d"(a0), "d"(a1), "d"(b));
  }
  double s = 0; for (int i = 0; i < ACC; ++i) s += c[i][0] + c[i][1] + c[i][2] + c[i][3];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

template <int ACC>
__global__ void dfma_loop(double* out, int iters) {
  double a = threadIdx.x * 1e-3, b = 1.0 - threadIdx.x * 1e-7;
  double c[ACC];
  for (int i = 0; i < ACC; ++i) c[i] = i;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < ACC; ++i) c[i] = fma(c[i], b, a);
  }
  double s = 0; for (int i = 0; i < ACC; ++i) s += c[i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

template <typename K>
void timeit(const char* name, K kern, int blocks, int threads, int iters, double flops_per_warp_iter) {
  double* d; CK(cudaMalloc(&d, sizeof(double) * blocks * threads));
  kern<<<blocks, threads>>>(d, 10); CK(cudaDeviceSynchronize());
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  cudaEventRecord(e0);
  kern<<<blocks, threads>>>(d, iters);
  cudaEventRecord(e1); CK(cudaEventSynchronize(e1));
  float ms; cudaEventElapsedTime(&ms, e0, e1);
  double fl = flops_per_warp_iter * (double)iters * blocks * (threads / 32);
  printf("%-28s blocks=%d thr=%d : %.3f ms  %.2f TFLOP/s\n", name, blocks, threads, ms, fl / ms / 1e9);
  cudaFree(d);
}

int main() {
  int dev = 0; cudaDeviceProp p; cudaGetDeviceProperties(&p, dev);
  printf("%s SMs=%d clock=%d kHz l2=%d MB\n", p.name, p.multiProcessorCount, p.clockRate, p.l2CacheSize >> 20);
  int sms = p.multiProcessorCount;
  for (int thr : {128, 256, 512}) {
    timeit("dmma m8n8k4 acc8", dmma_m8n8k4<8>, sms * 4, thr, 20000, 8 * 8 * 4 * 2 * 8);
    timeit("dmma m16n8k4 acc8", dmma_m16n8k4<8>, sms * 4, thr, 10000, 16 * 8 * 4 * 2 * 8);
    timeit("dmma m16n8k16 acc4", dmma_m16n8k16<4>, sms * 4, thr, 5000, 16 * 8 * 16 * 2 * 4);
    timeit("dfma acc8", dfma_loop<8>, sms * 4, thr, 20000, 32 * 2 * 8);
  }
  // cuBLAS DGEMM sustained
  cublasHandle_t h; cublasCreate(&h);
  for (int n : {4096, 8192, 16384}) {
    double *A, *B, *C;
    CK(cudaMalloc(&A, sizeof(double) * n * n)); CK(cudaMalloc(&B, sizeof(double) * n * n)); CK(cudaMalloc(&C, sizeof(double) * n * n));
    cudaMemset(A, 0, sizeof(double) * n * n); cudaMemset(B, 0, sizeof(double) * n * n);
    double one = 1.0, zero = 0.0;
    cublasDgemm(h, CUBLAS_OP_N, CUBLAS_OP_N, n, n, n, &one, A, n, B, n, &zero, C, n);
    CK(cudaDeviceSynchronize());
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    int reps = n >= 16384 ? 5 : 20;
    cudaEventRecord(e0);
    for (int r = 0; r < reps; ++r) cublasDgemm(h, CUBLAS_OP_N, CUBLAS_OP_N, n, n, n, &one, A, n, B, n, &zero, C, n);
    cudaEventRecord(e1); CK(cudaEventSynchronize(e1));
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    printf("cublasDgemm n=%d: %.2f TFLOP/s (%d reps, %.1f ms)\n", n, 2.0 * n * n * (double)n * reps / ms / 1e9, reps, ms);
    cudaFree(A); cudaFree(B); cudaFree(C);
  }
  // cuSOLVER dpotrf + dtrtri yardstick on an SPD matrix
  cusolverDnHandle_t sh; cusolverDnCreate(&sh);
  for (int n : {9000, 9088, 27000}) {
    double* A; CK(cudaMalloc(&A, sizeof(double) * (size_t)n * n));
    std::vector<double> hA((size_t)n * n, 0.0);
    // diagonally dominant SPD: I*n + small off-diagonal
    for (size_t j = 0; j < (size_t)n; ++j) for (size_t i = 0; i < (size_t)n; ++i) hA[j * n + i] = (i == j) ? n : 1.0 / (1.0 + (i > j ? i - j : j - i));
    int lwork = 0; cusolverDnDpotrf_bufferSize(sh, CUBLAS_FILL_MODE_LOWER, n, A, n, &lwork);
    double* work; CK(cudaMalloc(&work, sizeof(double) * lwork)); int* info; CK(cudaMalloc(&info, sizeof(int)));
    for (int rep = 0; rep < 2; ++rep) {
      CK(cudaMemcpy(A, hA.data(), sizeof(double) * (size_t)n * n, cudaMemcpyHostToDevice));
      cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
      cudaEventRecord(e0);
      cusolverDnDpotrf(sh, CUBLAS_FILL_MODE_LOWER, n, A, n, work, lwork, info);
      cudaEventRecord(e1); CK(cudaEventSynchronize(e1));
      float ms; cudaEventElapsedTime(&ms, e0, e1);
      // the triangular inverse of the factor (what the fused sweep also computes)
      size_t dws = 0, hws = 0;
      cusolverDnXtrtri_bufferSize(sh, CUBLAS_FILL_MODE_LOWER, CUBLAS_DIAG_NON_UNIT, n, CUDA_R_64F, A, n, &dws, &hws);
      void* dbuf; CK(cudaMalloc(&dbuf, dws + 16)); std::vector<char> hbuf(hws + 16);
      cudaEvent_t e2; cudaEventCreate(&e2);
      cusolverDnXtrtri(sh, CUBLAS_FILL_MODE_LOWER, CUBLAS_DIAG_NON_UNIT, n, CUDA_R_64F, A, n, dbuf, dws, hbuf.data(), hws, info);
      cudaEventRecord(e2); CK(cudaEventSynchronize(e2));
      float ms2; cudaEventElapsedTime(&ms2, e1, e2);
      printf("cusolver dpotrf n=%d: %.2f ms  %.2f TFLOP/s | dtrtri %.2f ms  %.2f TFLOP/s | potrf+trtri %.2f ms = %.2f TFLOP/s (2n^3/3)\n",
             n, ms, (double)n * n * n / 3.0 / ms / 1e9, ms2, (double)n * n * n / 3.0 / ms2 / 1e9, ms + ms2,
             2.0 * n * n * (double)n / 3.0 / (ms + ms2) / 1e9);
      cudaFree(dbuf);
    }
    cudaFree(A); cudaFree(work); cudaFree(info);
  }
  return 0;
}
