// Throughput microbenchmark: what a warp-wide table-coefficient load costs the SM's L1 /
// shared-memory pipe, by width, address pattern and memory space.  Decides whether staging
// the generation tables' intervals in shared memory (or the constant bank) can lift the
// L1-wavefront bound of gen_engine_kernel.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/microbench/ld_bcast tools/microbench/ld_bcast.cu
// Output: cycles per warp-load instruction per SM (SM-wide steady state, 32 warps per SM).
#include <cstdio>
#include <cstdlib>

constexpr int kTabWords = 1024;  // 16-byte words: 16 KB table
__constant__ uint4 c_tab[kTabWords / 4];  // 4 KB in the constant bank

enum Space { kGlobal = 0, kShared = 1, kConst = 2 };

// pattern: 0 = every lane the same address; 1 = two addresses (lane parity) 336 B apart;
// 2 = one address per quarter-warp, 336 B apart; 3 = lane-consecutive (fully coalesced)
__device__ __forceinline__ int lane_offset(int pattern, int lane) {
  switch (pattern) {
    case 0: return 0;
    case 1: return (lane & 1) * 21;
    case 2: return (lane >> 3) * 21;
    case 4: return (lane >> 4) * 21;  // two addresses, half-warps
    default: return lane;
  }
}

template <int kSpace, int kBytes>
__global__ void __launch_bounds__(256) bench(const uint4* __restrict__ gtab, unsigned* out,
                                             long long* cyc, int iters, int pattern) {
  __shared__ uint4 s_tab[kTabWords];
  for (int w = threadIdx.x; w < kTabWords; w += blockDim.x) s_tab[w] = gtab[w];
  __syncthreads();
  const int lane = threadIdx.x & 31;
  const int lofs = lane_offset(pattern, lane);
  unsigned acc0 = 0, acc1 = 0, acc2 = 0, acc3 = 0;
  const int mask = (kSpace == kConst ? kTabWords / 4 : kTabWords) - 64;
  const long long t0 = clock64();
  for (int i = 0; i < iters; ++i) {
    const int base = ((i * 8 + (int)(acc0 & 0)) & (mask - 1)) + lofs;
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      const int idx = base + j;
      if (kBytes == 16) {
        uint4 v;
        if (kSpace == kGlobal) v = __ldg(gtab + idx);
        else if (kSpace == kShared) v = s_tab[idx];
        else v = c_tab[idx];
        acc0 ^= v.x; acc1 ^= v.y; acc2 ^= v.z; acc3 ^= v.w;
      } else if (kBytes == 8) {
        uint2 v;
        if (kSpace == kGlobal) v = __ldg(reinterpret_cast<const uint2*>(gtab) + 2 * idx);
        else if (kSpace == kShared) v = reinterpret_cast<const uint2*>(s_tab)[2 * idx];
        else v = reinterpret_cast<const uint2*>(c_tab)[2 * idx];
        acc0 ^= v.x; acc1 ^= v.y;
      } else {
        unsigned v;
        if (kSpace == kGlobal) v = __ldg(reinterpret_cast<const unsigned*>(gtab) + 4 * idx);
        else if (kSpace == kShared) v = reinterpret_cast<const unsigned*>(s_tab)[4 * idx];
        else v = reinterpret_cast<const unsigned*>(c_tab)[4 * idx];
        acc0 ^= v;
      }
    }
  }
  const long long t1 = clock64();
  out[blockIdx.x * blockDim.x + threadIdx.x] = acc0 ^ acc1 ^ acc2 ^ acc3;
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}

template <int kSpace, int kBytes>
void run(const char* name, const uint4* gtab, unsigned* out, long long* cyc, int pattern) {
  const int iters = 4096, ctas = 148 * 4;
  bench<kSpace, kBytes><<<ctas, 256>>>(gtab, out, cyc, iters, pattern);
  bench<kSpace, kBytes><<<ctas, 256>>>(gtab, out, cyc, iters, pattern);
  cudaDeviceSynchronize();
  long long h[148 * 4];
  cudaMemcpy(h, cyc, sizeof(h), cudaMemcpyDeviceToHost);
  double mean = 0;
  for (int i = 0; i < ctas; ++i) mean += (double)h[i];
  mean /= ctas;
  // 4 CTAs x 8 warps per SM, each issuing iters * 8 loads in `mean` cycles
  const double per = mean / ((double)iters * 8 * 32);
  printf("%-8s %2d B pattern %d: %.3f cycles per warp-load per SM (%s)\n", name, kBytes, pattern,
         per, cudaGetErrorString(cudaGetLastError()));
}

int main() {
  uint4* gtab;
  unsigned* out;
  long long* cyc;
  cudaMalloc(&gtab, kTabWords * sizeof(uint4));
  cudaMalloc(&out, 148 * 4 * 256 * sizeof(unsigned));
  cudaMalloc(&cyc, 148 * 4 * sizeof(long long));
  uint4* h = (uint4*)malloc(kTabWords * sizeof(uint4));
  for (int i = 0; i < kTabWords; ++i) h[i] = make_uint4(i, 2 * i, 3 * i, 5 * i);
  cudaMemcpy(gtab, h, kTabWords * sizeof(uint4), cudaMemcpyHostToDevice);
  cudaMemcpyToSymbol(c_tab, h, sizeof(c_tab));
  for (int p = 0; p <= 4; ++p) {
    run<kGlobal, 16>("global", gtab, out, cyc, p);
    run<kGlobal, 8>("global", gtab, out, cyc, p);
    run<kGlobal, 4>("global", gtab, out, cyc, p);
    run<kShared, 16>("shared", gtab, out, cyc, p);
    run<kShared, 8>("shared", gtab, out, cyc, p);
    run<kShared, 4>("shared", gtab, out, cyc, p);
    if (p < 3 || p == 4) {
      run<kConst, 16>("const", gtab, out, cyc, p);
      run<kConst, 8>("const", gtab, out, cyc, p);
    }
  }
  return 0;
}
