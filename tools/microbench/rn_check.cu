// Branch-free correctly rounded sqrt / reciprocal (the diag kernel's pivot arithmetic) vs
// the IEEE intrinsics, on random doubles over a wide exponent range.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/microbench/rn_check tools/microbench/rn_check.cu
#include <cstdio>
#include <cstdint>

#include "../../paper_2601_11437_b200/csrc/pivot_math.cuh"

__global__ void check(unsigned long long seed, unsigned long long n, unsigned long long* bad) {
  unsigned long long i = blockIdx.x * (unsigned long long)blockDim.x + threadIdx.x;
  unsigned long long nb_s = 0, nb_r = 0, nb_c = 0;
  for (; i < n; i += (unsigned long long)gridDim.x * blockDim.x) {
    unsigned long long x = (i + 1) * 0x9E3779B97F4A7C15ull ^ seed;
    x ^= x >> 31; x *= 0xBF58476D1CE4E5B9ull; x ^= x >> 29;
    // exponent in [-700, 700] around 1, random mantissa
    const int ex = (int)((x >> 52) % 1400) - 700;
    const unsigned long long bits = (x & 0xFFFFFFFFFFFFFull) | ((unsigned long long)(1023 + ex) << 52);
    const double d = __longlong_as_double((long long)bits);
    const double s = mle::pivot_sqrt_rn(d);
    if (s != __dsqrt_rn(d)) ++nb_s;
    const double r = mle::pivot_rcp_rn(d);
    if (r != __drcp_rn(d)) ++nb_r;
    // the pair as used: 1 / sqrt(d) from the rsqrt-seeded refinement
    const double c = mle::pivot_rcp_of_sqrt(s, mle::pivot_rsqrt_seed(d));
    if (c != __drcp_rn(__dsqrt_rn(d))) ++nb_c;
  }
  atomicAdd(&bad[0], nb_s);
  atomicAdd(&bad[1], nb_r);
  atomicAdd(&bad[2], nb_c);
}

int main() {
  unsigned long long* bad;
  cudaMalloc(&bad, 24);
  cudaMemset(bad, 0, 24);
  const unsigned long long n = 1ull << 30;
  check<<<148 * 8, 256>>>(12345, n, bad);
  unsigned long long h[3];
  cudaMemcpy(h, bad, 24, cudaMemcpyDeviceToHost);
  printf("%llu values: sqrt mismatches %llu, rcp mismatches %llu, rcp(sqrt) mismatches %llu (%s)\n",
         n, h[0], h[1], h[2], cudaGetErrorString(cudaGetLastError()));
  return 0;
}
