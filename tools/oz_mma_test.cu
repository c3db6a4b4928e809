// Developer harness: validate a hand-written tcgen05.mma kind::i8 tile (M=128, N=64, K-major,
// SWIZZLE_NONE canonical layout, TMEM accumulator, bulk-copy + mbarrier staging).
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o tools/oz_mma_test tools/oz_mma_test.cu
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <vector>

#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e_ = (x); if (e_ != cudaSuccess) { printf("CUDA %s @%d\n", cudaGetErrorString(e_), __LINE__); exit(1);} } while (0)

constexpr int M = 128, N = 64, KB = 32;  // one MMA: 128 x 64 x 32 (int8)

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return (uint32_t)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
               : "memory");
}
// bounded wait: traps after ~2^26 polls instead of hanging the GPU
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t phase) {
  uint32_t done = 0;
  for (uint32_t it = 0; it < (1u << 26) && !done; ++it) {
    asm volatile(
        "{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0, 1, 0, p; }"
        : "=r"(done) : "r"(smem_u32(bar)), "r"(phase) : "memory");
  }
  if (!done) asm volatile("trap;");
}
__device__ __forceinline__ void bulk_g2s(void* smem, const void* gmem, uint32_t bytes, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
      ::"r"(smem_u32(smem)), "l"(gmem), "r"(bytes), "r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ uint64_t sdesc(const void* smem, uint32_t lbo, uint32_t sbo) {
  const uint64_t a = smem_u32(smem);
  return ((a >> 4) & 0x3FFF) | ((uint64_t)((lbo >> 4) & 0x3FFF) << 16) |
         ((uint64_t)((sbo >> 4) & 0x3FFF) << 32) | (1ull << 46);
}

__global__ void __launch_bounds__(192, 1) oz_tile_test(const int8_t* __restrict__ A,
                                                      const int8_t* __restrict__ B, int kblocks,
                                                      int* __restrict__ D) {
  __shared__ __align__(1024) int8_t sA[M * KB];
  __shared__ __align__(1024) int8_t sB[N * KB];
  __shared__ __align__(8) uint64_t full_bar, empty_bar, acc_bar;
  __shared__ uint32_t tmem_base;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    mbar_init(&full_bar, 1);
    mbar_init(&empty_bar, 1);
    mbar_init(&acc_bar, 1);
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                     smem_u32(&tmem_base)), "n"(64));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t tmem = tmem_base;
  const uint32_t idesc = (2u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(N >> 3) << 17) |
                         ((uint32_t)(M >> 4) << 24);
  for (int kb = 0; kb < kblocks; ++kb) {
    if (threadIdx.x == 0) {
      if (kb > 0) mbar_wait(&empty_bar, (kb - 1) & 1);
      mbar_expect_tx(&full_bar, M * KB + N * KB);
      bulk_g2s(sA, A + (size_t)kb * M * KB, M * KB, &full_bar);
      bulk_g2s(sB, B + (size_t)kb * N * KB, N * KB, &full_bar);
    }
    if (warp == 1) {
      mbar_wait(&full_bar, kb & 1);
      asm volatile("tcgen05.fence::after_thread_sync;");
      if (lane == 0) {
        const uint64_t da = sdesc(sA, 128, 256), db = sdesc(sB, 128, 256);
        const uint32_t acc = kb > 0 ? 1u : 0u;
        asm volatile(
            "{ .reg .pred p; setp.ne.b32 p, %4, 0;\n"
            "tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p; }"
            ::"r"(tmem), "l"(da), "l"(db), "r"(idesc), "r"(acc));
        asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];"
                     ::"r"(smem_u32(&empty_bar)));
      }
      __syncwarp();
    }
  }
  if (warp == 1 && lane == 0)
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];"
                 ::"r"(smem_u32(&acc_bar)));
  if (warp >= 2) {
    mbar_wait(&acc_bar, 0);
    asm volatile("tcgen05.fence::after_thread_sync;");
    const int q = warp & 3;  // TMEM lane quadrant this warp may access
    const int row = q * 32 + lane;
    for (int c0 = 0; c0 < N; c0 += 16) {
      uint32_t v[16];
      asm volatile(
          "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
          : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]),
            "=r"(v[7]), "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]),
            "=r"(v[13]), "=r"(v[14]), "=r"(v[15])
          : "r"(tmem + ((uint32_t)(q * 32) << 16) + (uint32_t)c0));
      asm volatile("tcgen05.wait::ld.sync.aligned;");
      for (int j = 0; j < 16; ++j) D[row * N + c0 + j] = (int)v[j];
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (warp == 0)
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "n"(64));
}

// canonical K-major SWIZZLE_NONE offset of (row r, k byte c) inside one rows x 32 block
static size_t canon(int r, int c) { return (size_t)(r >> 3) * 256 + (c >> 4) * 128 + (r & 7) * 16 + (c & 15); }

int main() {
  const int kblocks = 4, K = kblocks * KB;
  std::vector<int8_t> a((size_t)M * K), b((size_t)N * K);
  srand(1);
  for (auto& x : a) x = (int8_t)(rand() % 255 - 127);
  for (auto& x : b) x = (int8_t)(rand() % 255 - 127);
  std::vector<int8_t> ca((size_t)M * K), cb((size_t)N * K);
  for (int kb = 0; kb < kblocks; ++kb) {
    for (int r = 0; r < M; ++r)
      for (int c = 0; c < KB; ++c) ca[(size_t)kb * M * KB + canon(r, c)] = a[(size_t)r * K + kb * KB + c];
    for (int r = 0; r < N; ++r)
      for (int c = 0; c < KB; ++c) cb[(size_t)kb * N * KB + canon(r, c)] = b[(size_t)r * K + kb * KB + c];
  }
  int8_t *dA, *dB;
  int* dD;
  CK(cudaMalloc(&dA, ca.size()));
  CK(cudaMalloc(&dB, cb.size()));
  CK(cudaMalloc(&dD, sizeof(int) * M * N));
  CK(cudaMemcpy(dA, ca.data(), ca.size(), cudaMemcpyHostToDevice));
  CK(cudaMemcpy(dB, cb.data(), cb.size(), cudaMemcpyHostToDevice));
  oz_tile_test<<<1, 192>>>(dA, dB, kblocks, dD);
  CK(cudaGetLastError());
  CK(cudaDeviceSynchronize());
  std::vector<int> d((size_t)M * N);
  CK(cudaMemcpy(d.data(), dD, sizeof(int) * M * N, cudaMemcpyDeviceToHost));
  long bad = 0;
  for (int i = 0; i < M; ++i)
    for (int j = 0; j < N; ++j) {
      long ref = 0;
      for (int k = 0; k < K; ++k) ref += (long)a[(size_t)i * K + k] * b[(size_t)j * K + k];
      if (ref != d[(size_t)i * N + j]) {
        if (bad < 5) printf("mismatch (%d,%d): got %d want %ld\n", i, j, d[(size_t)i * N + j], ref);
        ++bad;
      }
    }
  printf("tcgen05 kind::i8 tile test: %ld mismatches of %d\n", bad, M * N);
  return bad != 0;
}
