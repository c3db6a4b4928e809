// FP64 pipe microbenchmark for B200 (sm_100a): DFMA vs DMMA (mma.sync f64 shapes),
// plus cuBLAS DGEMM and cuSOLVER DPOTRF yardsticks. Used once to pick the GEMM
// micro-architecture of the Cholesky/solve kernels; results go to profiles/.
#include <cstdio>
#include <cstdlib>
#include <vector>
#include <cuda_runtime.h>
#include <cublas_v2.h>
#include <cusolverDn.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("CUDA %s @%d\n", cudaGetErrorString(e), __LINE__); exit(1);} } while (0)

__global__ void dfma_kernel(double* out, int iters) {
  double a0 = threadIdx.x * 1e-9, a1 = a0 + 1, a2 = a0 + 2, a3 = a0 + 3, a4 = a0 + 4, a5 = a0 + 5, a6 = a0 + 6, a7 = a0 + 7;
  const double b = 0.999999, c = 1e-7;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int u = 0; u < 16; ++u) {
      a0 = fma(a0, b, c); a1 = fma(a1, b, c); a2 = fma(a2, b, c); a3 = fma(a3, b, c);
      a4 = fma(a4, b, c); a5 = fma(a5, b, c); a6 = fma(a6, b, c); a7 = fma(a7, b, c);
    }
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = a0 + a1 + a2 + a3 + a4 + a5 + a6 + a7;
}

__global__ void dmma_m8n8k4(double* out, int iters) {
  double a = threadIdx.x * 1e-3, b = 1.0 + threadIdx.x * 1e-4;
  double c[8][2] = {};
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int u = 0; u < 8; ++u)
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                   : "+d"(c[u][0]), "+d"(c[u][1]) : "d"(a), "d"(b));
  }
  double s = 0; for (int u = 0; u < 8; ++u) s += c[u][0] + c[u][1];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

__global__ void dmma_m16n8k4(double* out, int iters) {
  double a0 = threadIdx.x * 1e-3, a1 = a0 + 1, b = 1.0 + threadIdx.x * 1e-4;
  double c[4][4] = {};
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int u = 0; u < 4; ++u)
      asm volatile("mma.sync.aligned.m16n8k4.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5}, {%6}, {%0,%1,%2,%3};"
                   : "+d"(c[u][0]), "+d"(c[u][1]), "+d"(c[u][2]), "+d"(c[u][3]) : "d"(a0), "d"(a1), "d"(b));
  }
  double s = 0; for (int u = 0; u < 4; ++u) s += c[u][0] + c[u][1] + c[u][2] + c[u][3];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

__global__ void dmma_m16n8k8(double* out, int iters) {
  double a[4], b[2];
  for (int k = 0; k < 4; ++k) a[k] = threadIdx.x * 1e-3 + k;
  for (int k = 0; k < 2; ++k) b[k] = 1.0 + threadIdx.x * 1e-4 + k;
  double c[4][4] = {};
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int u = 0; u < 4; ++u)
      asm volatile("mma.sync.aligned.m16n8k8.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};"
                   : "+d"(c[u][0]), "+d"(c[u][1]), "+d"(c[u][2]), "+d"(c[u][3])
                   : "d"(a[0]), "d"(a[1]), "d"(a[2]), "d"(a[3]), "d"(b[0]), "d"(b[1]));
  }
  double s = 0; for (int u = 0; u < 4; ++u) s += c[u][0] + c[u][1] + c[u][2] + c[u][3];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

__global__ void dmma_m16n8k16(double* out, int iters) {
  double a[8], b[4];
  for (int k = 0; k < 8; ++k) a[k] = threadIdx.x * 1e-3 + k;
  for (int k = 0; k < 4; ++k) b[k] = 1.0 + threadIdx.x * 1e-4 + k;
  double c[4][4] = {};
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int u = 0; u < 4; ++u)
      asm volatile("mma.sync.aligned.m16n8k16.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5,%6,%7,%8,%9,%10,%11}, {%12,%13,%14,%15}, {%0,%1,%2,%3};"
                   : "+d"(c[u][0]), "+d"(c[u][1]), "+d"(c[u][2]), "+d"(c[u][3])
                   : "d"(a[0]), "d"(a[1]), "d"(a[2]), "d"(a[3]), "d"(a[4]), "d"(a[5]), "d"(a[6]), "d"(a[7]),
                     "d"(b[0]), "d"(b[1]), "d"(b[2]), "d"(b[3]));
  }
  double s = 0; for (int u = 0; u < 4; ++u) s += c[u][0] + c[u][1] + c[u][2] + c[u][3];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

template <typename F>
float time_it(F f, int reps) {
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  f(); CK(cudaDeviceSynchronize());
  float best = 1e30f;
  for (int r = 0; r < reps; ++r) {
    cudaEventRecord(a); f(); cudaEventRecord(b); cudaEventSynchronize(b);
    float ms; cudaEventElapsedTime(&ms, a, b); if (ms < best) best = ms;
  }
  return best;
}

int main() {
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  double* out; CK(cudaMalloc(&out, 1 << 26));
  const int iters = 4096;
  for (int threads : {128, 256, 512}) {
    for (int bps : {1, 2, 4}) {
      int blocks = sms * bps;
      double fl = 2.0 * 16 * 8 * (double)iters * blocks * threads;
      float ms = time_it([&] { dfma_kernel<<<blocks, threads>>>(out, iters); }, 5);
      printf("DFMA        thr=%d blk/SM=%d: %.2f TFLOP/s\n", threads, bps, fl / ms / 1e9);
      double warps = (double)blocks * threads / 32;
      ms = time_it([&] { dmma_m8n8k4<<<blocks, threads>>>(out, iters / 4); }, 5);
      printf("DMMA m8n8k4 thr=%d blk/SM=%d: %.2f TFLOP/s\n", threads, bps, warps * (iters / 4) * 8 * 2.0 * 8 * 8 * 4 / ms / 1e9);
      ms = time_it([&] { dmma_m16n8k4<<<blocks, threads>>>(out, iters / 4); }, 5);
      printf("DMMA m16n8k4 thr=%d blk/SM=%d: %.2f TFLOP/s\n", threads, bps, warps * (iters / 4) * 4 * 2.0 * 16 * 8 * 4 / ms / 1e9);
      ms = time_it([&] { dmma_m16n8k8<<<blocks, threads>>>(out, iters / 4); }, 5);
      printf("DMMA m16n8k8 thr=%d blk/SM=%d: %.2f TFLOP/s\n", threads, bps, warps * (iters / 4) * 4 * 2.0 * 16 * 8 * 8 / ms / 1e9);
      ms = time_it([&] { dmma_m16n8k16<<<blocks, threads>>>(out, iters / 8); }, 5);
      printf("DMMA m16n8k16 thr=%d blk/SM=%d: %.2f TFLOP/s\n", threads, bps, warps * (iters / 8) * 4 * 2.0 * 16 * 8 * 16 / ms / 1e9);
    }
  }
  // cuBLAS DGEMM yardstick
  cublasHandle_t h; cublasCreate(&h);
  for (int n : {4096, 8192, 16384}) {
    double *A, *B, *C; size_t bytes = (size_t)n * n * 8;
    CK(cudaMalloc(&A, bytes)); CK(cudaMalloc(&B, bytes)); CK(cudaMalloc(&C, bytes));
    cudaMemset(A, 0, bytes); cudaMemset(B, 0, bytes); cudaMemset(C, 0, bytes);
    double one = 1, zero = 0;
    float ms = time_it([&] { cublasDgemm(h, CUBLAS_OP_N, CUBLAS_OP_T, n, n, n, &one, A, n, B, n, &zero, C, n); }, 10);
    printf("cuBLAS DGEMM n=%d: %.2f TFLOP/s (%.3f ms)\n", n, 2.0 * n * n * (double)n / ms / 1e9, ms);
    float ms2 = time_it([&] { cublasDsyrk(h, CUBLAS_FILL_MODE_LOWER, CUBLAS_OP_N, n, 256, &one, A, n, &one, C, n); }, 10);
    printf("cuBLAS DSYRK n=%d k=256: %.2f TFLOP/s\n", n, 1.0 * n * n * 256.0 / ms2 / 1e9);
    cudaFree(A); cudaFree(B); cudaFree(C);
  }
  // cuSOLVER potrf yardstick on a diagonally dominant SPD matrix
  cusolverDnHandle_t sh; cusolverDnCreate(&sh);
  for (int n : {3600, 16384}) {
    size_t bytes = (size_t)n * n * 8;
    std::vector<double> hA((size_t)n * n);
    for (int j = 0; j < n; ++j) for (int i = 0; i < n; ++i) hA[(size_t)j * n + i] = (i == j) ? n : 1.0 / (1 + abs(i - j));
    double* A; double* A0; CK(cudaMalloc(&A, bytes)); CK(cudaMalloc(&A0, bytes));
    cudaMemcpy(A0, hA.data(), bytes, cudaMemcpyHostToDevice);
    int lwork; cusolverDnDpotrf_bufferSize(sh, CUBLAS_FILL_MODE_LOWER, n, A, n, &lwork);
    double* work; int* info; cudaMalloc(&work, (size_t)lwork * 8); cudaMalloc(&info, 4);
    float best = 1e30f;
    for (int r = 0; r < 4; ++r) {
      cudaMemcpy(A, A0, bytes, cudaMemcpyDeviceToDevice);
      cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
      cudaEventRecord(a);
      cusolverDnDpotrf(sh, CUBLAS_FILL_MODE_LOWER, n, A, n, work, lwork, info);
      cudaEventRecord(b); cudaEventSynchronize(b);
      float ms; cudaEventElapsedTime(&ms, a, b); if (r > 0 && ms < best) best = ms;
    }
    printf("cuSOLVER DPOTRF n=%d: %.3f ms, %.2f TFLOP/s\n", n, best, (double)n * n * n / 3.0 / best / 1e9);
    // trsm yardstick: L^{-1} B with B n x 2n
    double* Bm; CK(cudaMalloc(&Bm, bytes * 2)); cudaMemset(Bm, 0, bytes * 2);
    double one = 1;
    float ms = time_it([&] { cublasDtrsm(h, CUBLAS_SIDE_LEFT, CUBLAS_FILL_MODE_LOWER, CUBLAS_OP_N, CUBLAS_DIAG_NON_UNIT, n, 2 * n, &one, A, n, Bm, n); }, 3);
    printf("cuBLAS DTRSM n=%d nrhs=%d: %.3f ms, %.2f TFLOP/s\n", n, 2 * n, ms, 2.0 * n * (double)n * n / ms / 1e9);
    cudaFree(Bm); cudaFree(A); cudaFree(A0); cudaFree(work); cudaFree(info);
  }
  printf("done\n");
  return 0;
}
