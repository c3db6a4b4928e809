// Markstein quotient vs IEEE division on random h, alpha (the generation kernel's u = h / alpha).
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/div_check tools/div_check.cu
#include <cstdio>
#include <cuda_runtime.h>
__global__ void k(unsigned long long seed, unsigned long long* bad, long long m) {
  long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  unsigned long long x = seed ^ (i * 0x9E3779B97F4A7C15ull);
  for (int r = 0; r < 64 && i < m; ++r) {
    x ^= x << 13; x ^= x >> 7; x ^= x << 17;
    const double h = (double)(x >> 11) * 0x1.0p-53 * 2.0;           // (0, 2)
    x ^= x << 13; x ^= x >> 7; x ^= x << 17;
    const double alpha = 1e-3 + (double)(x >> 11) * 0x1.0p-53 * 5.0; // (0.001, 5)
    const double ia = 1.0 / alpha;
    const double q = h * ia;
    const double u = fma(fma(-alpha, q, h), ia, q);
    if (u != h / alpha) atomicAdd(bad, 1ull);
  }
}
int main() {
  unsigned long long* d; cudaMalloc(&d, 8); cudaMemset(d, 0, 8);
  const long long m = 1ll << 24;
  k<<<(unsigned)(m / 256), 256>>>(12345, d, m);
  unsigned long long b; cudaMemcpy(&b, d, 8, cudaMemcpyDeviceToHost);
  printf("markstein vs division: %llu mismatches in %lld quotients\n", b, m * 64);
  return 0;
}
