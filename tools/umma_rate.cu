// Developer microbenchmark: cycles per tcgen05.mma.kind::i8 (M=128, SS operands, K=32) as a
// function of N, one CTA per SM, operands resident in shared memory (no loads).
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o tools/umma_rate tools/umma_rate.cu
#include <cstdint>
#include <cstdio>

#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return (uint32_t)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ uint64_t sdesc(uint32_t saddr) {
  return ((uint64_t)((saddr >> 4) & 0x3FFF)) | ((uint64_t)(128 >> 4) << 16) |
         ((uint64_t)(256 >> 4) << 32) | (1ull << 46);
}

template <int kN, int kKind>  // kKind 0: int8 (K=32), 1: bf16 (K=16), both 32 bytes of K
__global__ void __launch_bounds__(128, 1) umma_loop(int iters, long long* cycles) {
  extern __shared__ __align__(1024) uint8_t sm[];  // A 4 KB + B kN*32 B
  __shared__ __align__(8) uint64_t bar;
  __shared__ uint32_t tmem_base;
  const int warp = threadIdx.x >> 5;
  for (int i = threadIdx.x; i < (4096 + kN * 32) / 4; i += blockDim.x)
    reinterpret_cast<uint32_t*>(sm)[i] = 0x01010101u * (i & 3);
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&bar)));
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(
        smem_u32(&tmem_base)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("fence.proxy.async.shared::cta;");
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t tmem = tmem_base;
  if (threadIdx.x == 0) {
    const uint32_t idesc = kKind == 0
        ? (2u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(kN >> 3) << 17) | ((uint32_t)(128 >> 4) << 24)
        : (1u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(kN >> 3) << 17) | ((uint32_t)(128 >> 4) << 24);
    const uint64_t da = sdesc(smem_u32(sm)), db = sdesc(smem_u32(sm + 4096));
    const long long t0 = clock64();
    for (int i = 0; i < iters; ++i) {
      const uint32_t acc = i > 0 ? 1u : 0u;
      if (kKind == 0)
        asm volatile("{ .reg .pred pp; setp.ne.b32 pp, %4, 0;\n"
                     "tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, pp; }" ::"r"(tmem),
                     "l"(da), "l"(db), "r"(idesc), "r"(acc));
      else
        asm volatile("{ .reg .pred pp; setp.ne.b32 pp, %4, 0;\n"
                     "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, pp; }" ::"r"(tmem),
                     "l"(da), "l"(db), "r"(idesc), "r"(acc));
    }
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
        smem_u32(&bar)));
    uint32_t done = 0;
    while (!done)
      asm volatile("{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], 0; "
                   "selp.u32 %0, 1, 0, p; }" : "=r"(done) : "r"(smem_u32(&bar)) : "memory");
    cycles[blockIdx.x] = clock64() - t0;
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tmem));
}

template <int kN, int kKind>
void run(int sms) {
  const int iters = 20000;
  long long* d;
  cudaMalloc(&d, sizeof(long long) * sms);
  const int smem = 4096 + kN * 32;
  cudaFuncSetAttribute(umma_loop<kN, kKind>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  umma_loop<kN, kKind><<<sms, 128, smem>>>(100, d);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  cudaEventRecord(a);
  umma_loop<kN, kKind><<<sms, 128, smem>>>(iters, d);
  cudaEventRecord(b);
  cudaEventSynchronize(b);
  float ms;
  cudaEventElapsedTime(&ms, a, b);
  long long h[148];
  cudaMemcpy(h, d, sizeof(long long) * sms, cudaMemcpyDeviceToHost);
  double macs = 128.0 * kN * 32.0 * iters * sms;
  printf("%s N=%3d: %.1f cycles/MMA (ideal %s %.0f) | %.1f T MAC/s -> %.0f TOPS  (%s)\n",
         kKind == 0 ? "i8  " : "bf16", kN, (double)h[0] / iters, "N/2 =", kN / 2.0,
         macs / (ms * 1e-3) / 1e12, 2 * macs / (ms * 1e-3) / 1e12,
         cudaGetErrorString(cudaGetLastError()));
  cudaFree(d);
}


// The ozgemm_persistent_kernel<64> per-k-block MMA sequence: for p = 1..8 one MMA over the
// B rows [B_1 .. B_{9-p}] (64 (9 - p) rows, split at 256) at TMEM column (p - 1) 64.
// kCommit: tcgen05.commit to an mbarrier after every k block (as the kernel does).
template <int kCommit, int kVaryA, int kS = 8, int kSplit = 256>
__global__ void __launch_bounds__(128, 1) umma_seq(int kblocks, long long* cycles) {
  extern __shared__ __align__(1024) uint8_t sm[];  // A 8 x 4 KB + B 16 KB
  __shared__ __align__(8) uint64_t bar;
  __shared__ uint32_t tmem_base;
  const int warp = threadIdx.x >> 5;
  for (int i = threadIdx.x; i < (32768 + 16384) / 4; i += blockDim.x)
    reinterpret_cast<uint32_t*>(sm)[i] = 0x01010101u * (i & 3);
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&bar)));
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(
        smem_u32(&tmem_base)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("fence.proxy.async.shared::cta;");
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t tmem = tmem_base;
  if (threadIdx.x == 0) {
    const uint32_t sa = smem_u32(sm), sb = sa + 32768;
    const long long t0 = clock64();
    for (int kb = 0; kb < kblocks; ++kb) {
#pragma unroll
      for (int p = 1; p <= kS; ++p) {
        const int rows = 64 * (kS + 1 - p);
        const uint32_t accum = (kb > 0 || p > 1) ? 1u : 0u;
        // kSplit > 0: pieces of at most kSplit rows; kSplit < 0: |kSplit| equal pieces
        const int pieces = kSplit > 0 ? (rows + kSplit - 1) / kSplit
                                      : (rows > 256 ? -kSplit : 1);
        const int step = ((rows / pieces + 15) / 16) * 16;
#pragma unroll
        for (int r0 = 0; r0 < rows; r0 += step) {
          const int nr = rows - r0 < step ? rows - r0 : step;
          const uint32_t idesc = (2u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(nr >> 3) << 17) |
                                 ((uint32_t)(128 >> 4) << 24);
          asm volatile("{ .reg .pred pp; setp.ne.b32 pp, %4, 0;\n"
                       "tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, pp; }" ::"r"(
                           tmem + (uint32_t)((p - 1) * 64 + r0)),
                       "l"(sdesc(sa + (kVaryA ? (p - 1) * 4096 : 0))), "l"(sdesc(sb + r0 * 32)),
                       "r"(idesc), "r"(accum));
        }
      }
      if (kCommit)
        asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];"
                     ::"r"(smem_u32(&bar)));
    }
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
        smem_u32(&bar)));
    // wait for the final phase: total arrivals = kblocks * kCommit + 1
    const uint32_t last = (uint32_t)((kblocks * kCommit) & 1);
    uint32_t done = 0;
    while (!done)
      asm volatile("{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; "
                   "selp.u32 %0, 1, 0, p; }" : "=r"(done) : "r"(smem_u32(&bar)), "r"(last) : "memory");
    cycles[blockIdx.x] = clock64() - t0;
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tmem));
}

template <int kCommit, int kVaryA, int kS = 8, int kSplit = 256>
void run_seq(int sms, int kb = 2000) {
  long long* d;
  cudaMalloc(&d, sizeof(long long) * sms);
  const int smem = 32768 + 16384;
  cudaFuncSetAttribute(umma_seq<kCommit, kVaryA, kS, kSplit>,
                       cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  umma_seq<kCommit, kVaryA, kS, kSplit><<<sms, 128, smem>>>(10, d);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  cudaEventRecord(e0);
  umma_seq<kCommit, kVaryA, kS, kSplit><<<sms, 128, smem>>>(kb, d);
  cudaEventRecord(e1);
  cudaDeviceSynchronize();
  float ms;
  cudaEventElapsedTime(&ms, e0, e1);
  long long h[148];
  cudaMemcpy(h, d, sizeof(long long) * sms, cudaMemcpyDeviceToHost);
  printf("ozgemm<64> k-block sequence S=%d split %d (commit %d, vary A %d, %d k blocks, %.1f ms):"
         " %.0f cycles per k block (compute bound %d), effective SM clock %.0f MHz, %.0f int8 "
         "TOPS (%s)\n", kS, kSplit,
         kCommit, kVaryA, kb, ms, (double)h[0] / kb, 32 * kS * (kS + 1) / 2,
         (double)h[0] / (ms * 1e3),
         2.0 * (kS * (kS + 1) / 2) * 128 * 64 * 32 * (double)kb * sms / (ms * 1e-3) / 1e12,
         cudaGetErrorString(cudaGetLastError()));
  cudaFree(d);
}


__device__ __forceinline__ void mwait(uint64_t* bar, uint32_t ph) {
  uint32_t done = 0;
  while (!done)
    asm volatile("{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; "
                 "selp.u32 %0, 1, 0, p; }" : "=r"(done) : "r"(smem_u32(bar)), "r"(ph) : "memory");
}
__device__ __forceinline__ void marrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}

// Kernel-shaped MMA loop: producer warp (no data, arrives full after empty), MMA warp with the
// 4-stage full/empty ring, optional per-tile accumulator handshake with 8 epilogue warps.
template <int kTileSync, int kRandom = 0, int kS = 8>
__global__ void __launch_bounds__(320, 1) umma_ring(int tiles, int kblocks, long long* cycles) {
  extern __shared__ __align__(1024) uint8_t sm[];  // 4 stages x 48 KB
  __shared__ __align__(8) uint64_t full[4], empty[4], accf, acce;
  __shared__ uint32_t tmem_base;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    for (int i = 0; i < 4; ++i) {
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&full[i])));
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&empty[i])));
    }
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&accf)));
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 8;" ::"r"(smem_u32(&acce)));
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(
        smem_u32(&tmem_base)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t tmem = tmem_base;
  if (kRandom >= 1) {
    uint32_t x = 2463534242u + threadIdx.x * 7919u + blockIdx.x * 104729u;
    for (int i = threadIdx.x; i < 4 * 49152 / 4; i += blockDim.x) {
      x ^= x << 13; x ^= x >> 17; x ^= x << 5;
      reinterpret_cast<uint32_t*>(sm)[i] = kRandom == 1 ? (x & 0x7F7F7F7Fu) : kRandom == 2 ? x : 0u;
    }
    asm volatile("fence.proxy.async.shared::cta;");
    __syncthreads();
  }
  long long g0;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(g0));
  const long long t0 = clock64();
  if (warp == 0) {
    if (lane == 0) {
      long long gk = 0;
      for (int t = 0; t < tiles; ++t)
        for (int kb = 0; kb < kblocks; ++kb, ++gk) {
          const int st = (int)(gk % 4);
          if (gk >= 4) mwait(&empty[st], (uint32_t)(((gk / 4) - 1) & 1));
          marrive(&full[st]);
        }
    }
    __syncwarp();
  } else if (warp == 1) {
    long long gk = 0;
    for (int t = 0; t < tiles; ++t) {
      if (kTileSync && t >= 1) mwait(&acce, (uint32_t)((t - 1) & 1));
      asm volatile("tcgen05.fence::after_thread_sync;");
      for (int kb = 0; kb < kblocks; ++kb, ++gk) {
        const int st = (int)(gk % 4);
        mwait(&full[st], (uint32_t)((gk / 4) & 1));
        asm volatile("tcgen05.fence::after_thread_sync;");
        if (lane == 0) {
          const uint32_t sa = smem_u32(sm + st * 49152), sb = sa + 32768;
#pragma unroll
          for (int p = 1; p <= kS; ++p) {
            const int rows = 64 * (kS + 1 - p);
            const uint32_t accum = (kb > 0 || p > 1) ? 1u : 0u;
#pragma unroll
            for (int r0 = 0; r0 < rows; r0 += 256) {
              const int nr = rows - r0 < 256 ? rows - r0 : 256;
              const uint32_t idesc = (2u << 4) | (1u << 7) | (1u << 10) |
                                     ((uint32_t)(nr >> 3) << 17) | ((uint32_t)(128 >> 4) << 24);
              asm volatile("{ .reg .pred pp; setp.ne.b32 pp, %4, 0;\n"
                           "tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, pp; }" ::"r"(
                               tmem + (uint32_t)((p - 1) * 64 + r0)),
                           "l"(sdesc(sa + (p - 1) * 4096)), "l"(sdesc(sb + r0 * 32)), "r"(idesc),
                           "r"(accum));
            }
          }
          asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];"
                       ::"r"(smem_u32(&empty[st])));
        }
        __syncwarp();
      }
      if (lane == 0)
        asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];"
                     ::"r"(smem_u32(&accf)));
      __syncwarp();
    }
  } else if (kTileSync) {
    for (int t = 0; t < tiles; ++t) {
      mwait(&accf, (uint32_t)(t & 1));
      asm volatile("tcgen05.fence::after_thread_sync;");
      __syncwarp();
      if (lane == 0) marrive(&acce);
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (threadIdx.x == 32) {
    long long g1;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(g1));
    cycles[blockIdx.x] = clock64() - t0;
    cycles[148 + blockIdx.x] = g1 - g0;
  }
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tmem));
}

template <int kTileSync, int kRandom = 0, int kS = 8>
void run_ring(int sms, int tiles, int kblocks) {
  long long* d;
  cudaMalloc(&d, sizeof(long long) * 296);
  const int smem = 4 * 49152;
  cudaFuncSetAttribute(umma_ring<kTileSync, kRandom, kS>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                       smem);
  umma_ring<kTileSync, kRandom, kS><<<sms, 320, smem>>>(2, kblocks, d);
  umma_ring<kTileSync, kRandom, kS><<<sms, 320, smem>>>(tiles, kblocks, d);
  cudaDeviceSynchronize();
  long long h[296];
  cudaMemcpy(h, d, sizeof(long long) * 296, cudaMemcpyDeviceToHost);
  printf("ring S=%d (tile sync %d, random %d, %d tiles x %d k blocks): %.0f cycles per k block, "
         "%.1f ms, clock %.0f MHz, %.0f int8 TOPS (%s)\n", kS, kTileSync, kRandom,
         tiles, kblocks, (double)h[0] / ((double)tiles * kblocks), h[148] * 1e-6,
         (double)h[0] / (h[148] * 1e-3), 2.0 * 36 * 128 * 64 * 32 * (double)tiles * kblocks * sms /
         (h[148] * 1e-9) / 1e12, cudaGetErrorString(cudaGetLastError()));
  cudaFree(d);
}

int main(int argc, char** argv) {
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  if (argc > 1) {  // the S = 7 / 6 sequences, split variants
    run_seq<1, 1, 8, 256>(sms);
    run_seq<1, 1, 7, 256>(sms);
    run_seq<1, 1, 7, 128>(sms);
    run_seq<1, 1, 7, -2>(sms);
    run_seq<1, 1, 6, 256>(sms);
    run_seq<1, 1, 6, -2>(sms);
    run_ring<1, 0, 7>(sms, 2000, 16);
    run_ring<0, 0, 7>(sms, 2000, 16);
    run_ring<1, 2, 7>(sms, 2000, 16);
    run_ring<1, 0, 8>(sms, 2000, 16);
    return 0;
  }
  run<32, 0>(sms);
  run<64, 0>(sms);
  run<128, 0>(sms);
  run<256, 0>(sms);
  run<64, 1>(sms);
  run<256, 1>(sms);
  run_seq<0, 0>(sms);
  run_seq<0, 1>(sms);
  run_seq<1, 1>(sms);
  run_ring<1, 3>(sms, 2000, 16);
  run_ring<1>(sms, 2000, 16);
  run_ring<1, 1>(sms, 2000, 16);
  run_ring<1, 2>(sms, 2000, 16);
  run_ring<1, 2>(sms, 20000, 16);
  return 0;
}
