// Latency microbenchmark (one warp): dependent DFMA, DMUL, SHFL.IDX (double), MUFU.RSQ64H,
// and the full pivot step of the 16x16 Cholesky (shfl + rsqrt refine + scale + fma).
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/microbench/fp64_lat tools/microbench/fp64_lat.cu
#include <cstdio>

__global__ void lat(double* out, long long* cyc, double seed) {
  double x = seed + threadIdx.x * 1e-3;
  const int N = 1024;
  long long t0, t1;
  // DFMA chain
  t0 = clock64();
#pragma unroll 16
  for (int i = 0; i < N; ++i) x = fma(x, 0.999999, 1e-7);
  t1 = clock64();
  cyc[0] = t1 - t0;
  t0 = clock64();
#pragma unroll 16
  for (int i = 0; i < N; ++i) x = x * 1.0000001;
  t1 = clock64();
  cyc[1] = t1 - t0;
  // shfl chain
  t0 = clock64();
#pragma unroll 16
  for (int i = 0; i < N; ++i) x = __shfl_sync(0xffffffffu, x, (threadIdx.x + 1) & 31);
  t1 = clock64();
  cyc[2] = t1 - t0;
  // MUFU.RSQ64H chain
  t0 = clock64();
#pragma unroll 16
  for (int i = 0; i < N; ++i) {
    double y;
    asm volatile("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(x));
    x = y;
  }
  t1 = clock64();
  cyc[3] = t1 - t0;
  // 32-bit shfl chain
  float f = x;
  t0 = clock64();
#pragma unroll 16
  for (int i = 0; i < N; ++i) f = __shfl_sync(0xffffffffu, f, (threadIdx.x + 1) & 31);
  t1 = clock64();
  cyc[4] = t1 - t0;
  // FFMA chain
  t0 = clock64();
#pragma unroll 16
  for (int i = 0; i < N; ++i) f = fmaf(f, 0.999f, 1e-3f);
  t1 = clock64();
  cyc[5] = t1 - t0;
  // smem round trip chain (st + ld)
  __shared__ double sm[64];
  t0 = clock64();
#pragma unroll 16
  for (int i = 0; i < N; ++i) {
    sm[threadIdx.x] = x;
    __syncwarp();
    x = sm[(threadIdx.x + 1) & 31];
    __syncwarp();
  }
  t1 = clock64();
  cyc[6] = t1 - t0;
  out[threadIdx.x] = x + f;
}

int main() {
  double* o;
  long long* c;
  cudaMalloc(&o, 32 * 8);
  cudaMalloc(&c, 16 * 8);
  for (int r = 0; r < 2; ++r) lat<<<1, 32>>>(o, c, 1.0);
  long long h[16];
  cudaMemcpy(h, c, sizeof(h), cudaMemcpyDeviceToHost);
  const char* names[] = {"DFMA", "DMUL", "SHFL f64 (2x SHFL)", "MUFU.RSQ64H", "SHFL f32", "FFMA",
                         "STS+LDS f64 round trip (syncwarp)"};
  for (int i = 0; i < 7; ++i) printf("%-36s %.1f cycles\n", names[i], h[i] / 1024.0);
  return 0;
}
