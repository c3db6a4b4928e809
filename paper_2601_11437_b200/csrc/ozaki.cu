// ozaki.cu — FP64 GEMM on the 5th-generation tensor cores (tcgen05.mma kind::i8, TMEM).
//
// B200 has no FP64 tcgen05 kind; its mma.sync DMMA path peaks at ~36 TF/s.  The trailing
// updates of the Cholesky and of the solves (C -= A B^T with K = 512) are instead run as an
// Ozaki-scheme emulation (splitting into int8 slices, exact int32 products):
//   * every row of A and of B (over the K range) is scaled by a power of two to (-1, 1) and
//     split into S = 8 signed 7-bit digits:  A(i,:) = 2^ea_i sum_p 2^-7p A_p(i,:)
//   * C(i,j) = 2^(ea_i + eb_j) sum_{d=2..S+1} 2^-7d  sum_{p+q=d} (A_p B_q^T)(i,j)
//     (the 36 slice products with p + q <= S + 1; each is an exact int8 x int8 -> int32
//     tensor-core GEMM, the 8 diagonals d accumulate in 8 TMEM accumulators)
//   * the FP64 epilogue converts, scales (exact powers of two) and accumulates into C.
// With S = 8 the error is within a few units of DGEMM's (56 mantissa bits per row before
// dropped terms; tools/ozaki accuracy study in DESIGN.md), at 4.5 POPS int8 peak / 36.
//
// Layouts.  Slices are written by oz_slice_kernel in the UMMA canonical K-major
// SWIZZLE_NONE layout: for each 128-row tile and each 32-wide k block, 8 slices of a
// 128 x 32 int8 block (4 KB; core matrices of 8 rows x 16 B, LBO = 128 B, SBO = 256 B).  The
// first / second 64 rows of a block are its first / second 2 KB, which the GEMM uses as the
// 64-row B operand.
#include <cuda_runtime.h>
#include <stdint.h>

#include "kernels.h"

namespace mle {

namespace {

constexpr int OZ_S = 8;             // slices per operand
constexpr int OZ_KB = 32;           // k per MMA (int8)
constexpr int OZ_BLK = 128 * OZ_KB; // bytes of one slice block (128 rows x 32)
constexpr int OZ_A_STAGE = OZ_S * OZ_BLK;        // 32 KB: the 8 A slices of one k block
constexpr int OZ_THREADS = 192;                  // warp 0 producer, 1 MMA, 2-5 epilogue

// CTA tile 128 x kN.  TMEM holds the 8 diagonal accumulators (8 kN columns); kN = 32 fits
// two CTAs per SM so one CTA's epilogue overlaps the other's main loop.
template <int kN>
struct OzCfg {
  static constexpr int kStages = kN == 64 ? 4 : 2;
  static constexpr int kBStage = OZ_S * kN * OZ_KB;           // 8 B slices, kN rows each
  static constexpr int kStage = OZ_A_STAGE + kBStage;
  static constexpr int kSmem = kStages * kStage;
  static constexpr int kTmemCols = OZ_S * kN;                 // 512 / 256
  static constexpr int kCtasPerSm = kN == 64 ? 1 : 2;
};

__device__ __forceinline__ double pow2i(int e) {  // exact 2^e
  return (e > -1023 && e < 1024) ? __longlong_as_double((long long)(e + 1023) << 52)
                                 : ldexp(1.0, e);
}

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return (uint32_t)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
               "r"(bytes)
               : "memory");
}
// Bounded wait: a lost arrival traps (kernel error) instead of hanging the GPU.
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t phase) {
  uint32_t done = 0;
  for (uint32_t it = 0; it < (1u << 28) && !done; ++it) {
    asm volatile(
        "{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; "
        "selp.u32 %0, 1, 0, p; }"
        : "=r"(done)
        : "r"(smem_u32(bar)), "r"(phase)
        : "memory");
  }
  if (!done) asm volatile("trap;");
}
__device__ __forceinline__ void bulk_g2s(void* smem, const void* gmem, uint32_t bytes,
                                         uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
      ::"r"(smem_u32(smem)), "l"(gmem), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}
// UMMA shared-memory descriptor: K-major, SWIZZLE_NONE, LBO = 128 B, SBO = 256 B, sm_100.
__device__ __forceinline__ uint64_t sdesc(uint32_t saddr) {
  return ((uint64_t)((saddr >> 4) & 0x3FFF)) | ((uint64_t)(128 >> 4) << 16) |
         ((uint64_t)(256 >> 4) << 32) | (1ull << 46);
}

}  // namespace

// Slicing.  CTA = 32 rows x all K (<= kOzSliceMaxK) of one operand, staged once in shared
// memory (grid rows/32 x batch): coalesced load, per-row max -> exponent e with
// |X(r,:)| < 2^e, then each thread turns 16 elements of one row into 8 digits each (exact:
// x 2^7, trunc, subtract) and writes one 16-byte word per slice in the canonical layout.
// (32 consecutive rows of a 128-row block are 1 KB contiguous in every slice block.)
constexpr int kOzSliceRows = 32;
constexpr int kOzSliceMaxK = 512;
constexpr int kOzSliceStride = kOzSliceMaxK + 1;  // odd stride: conflict-free row access
constexpr int kOzSliceSmem = kOzSliceRows * kOzSliceStride * 8;

template <int kRowContig>
__global__ void __launch_bounds__(256) oz_slice_kernel(OzSliceArgs sa) {
  const int z = blockIdx.z;
  if (sa.fail_flag[z] && *sa.fail_flag[z]) return;
  extern __shared__ double tile[];  // [32][kOzSliceStride]
  __shared__ int ex[kOzSliceRows];
  const double* X = sa.X[z];
  const long long ld = sa.ld;
  const int K = sa.K, t = threadIdx.x, w = t >> 5, l = t & 31;
  const long long r0 = (long long)blockIdx.x * kOzSliceRows;
  if (kRowContig) {  // X(r,k) = X[r + k ld]: lanes along r
    for (int k = w; k < K; k += 8) tile[l * kOzSliceStride + k] = X[r0 + l + (long long)k * ld];
  } else {           // X(r,k) = X[k + r ld]: lanes along k
    for (int r = w; r < kOzSliceRows; r += 8) {
      const double* row = X + (r0 + r) * ld;
      for (int k = l; k < K; k += 32) tile[r * kOzSliceStride + k] = row[k];
    }
  }
  __syncthreads();
  for (int r = w; r < kOzSliceRows; r += 8) {
    double mx = 0.0;
    for (int k = l; k < K; k += 32) mx = fmax(mx, fabs(tile[r * kOzSliceStride + k]));
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) mx = fmax(mx, __shfl_xor_sync(0xffffffffu, mx, o));
    if (l == 0) {
      int e = 0;
      if (mx > 0.0) frexp(mx, &e);
      ex[r] = e;
      sa.e[z][r0 + r] = e;
    }
  }
  __syncthreads();
  int8_t* out = sa.slices[z];
  const int kblocks = K / OZ_KB;
  const long long tile128 = r0 >> 7;
  const int rsub = (int)(r0 & 127);
  // work item = (row, 16-wide k chunk); lanes on consecutive rows
  for (int item = t; item < kOzSliceRows * (K / 16); item += 256) {
    const int r = item & (kOzSliceRows - 1), ch = item / kOzSliceRows;
    // |x| 2^(56 - e) < 2^56 is exact (power-of-two scaling); its truncation holds the 8
    // base-128 digits the float recurrence (x 2^7, trunc, subtract) would produce.
    const int sh = 56 - ex[r];
    const double sc1 = pow2i(sh > 1000 ? 1000 : sh), sc2 = pow2i(sh > 1000 ? sh - 1000 : 0);
    const double* src = tile + r * kOzSliceStride + ch * 16;
    uint32_t wd[OZ_S][4];
#pragma unroll
    for (int p = 0; p < OZ_S; ++p) wd[p][0] = wd[p][1] = wd[p][2] = wd[p][3] = 0u;
#pragma unroll
    for (int c = 0; c < 16; ++c) {
      const double x = src[c];
      const unsigned long long u =
          (unsigned long long)__double2ll_rz(fabs(x) * sc1 * sc2);
      const bool neg = x < 0.0;
#pragma unroll
      for (int p = 0; p < OZ_S; ++p) {
        const uint32_t d = (uint32_t)(u >> (56 - 7 * (p + 1))) & 127u;
        const uint32_t byte = (neg ? (0u - d) : d) & 0xFFu;
        wd[p][c >> 2] |= byte << (8 * (c & 3));
      }
    }
    const int kb = ch >> 1, half = ch & 1;
    const int rl = rsub + r;
    int8_t* dst = out + ((size_t)(tile128 * kblocks + kb) * OZ_S) * OZ_BLK +
                  (size_t)(rl >> 3) * 256 + (size_t)(rl & 7) * 16 + (size_t)half * 128;
#pragma unroll
    for (int p = 0; p < OZ_S; ++p)
      *reinterpret_cast<uint4*>(dst + (size_t)p * OZ_BLK) =
          make_uint4(wd[p][0], wd[p][1], wd[p][2], wd[p][3]);
  }
}

// C(i,j) = beta C + alpha 2^(ea_i + eb_j) sum_d 2^-7d sum_{p+q=d} (A_p B_q^T)(i,j).
// MMA structure: for slice p of A, ONE MMA against the concatenation [B_1; ...; B_{9-p}]
// (kN (9-p) rows, split at 256) written at TMEM column (p-1) kN: product (p, q) then lands
// at column (p+q-2) kN, i.e. in accumulator d = p + q.  8-12 MMAs per k block instead of 36.
template <int kN>
__global__ void __launch_bounds__(OZ_THREADS, OzCfg<kN>::kCtasPerSm) ozgemm_kernel(OzGemmArgs g) {
  using Cfg = OzCfg<kN>;
  constexpr int kParts = 128 / kN;
  const int z = blockIdx.z;
  if (*g.fail_flag[z]) return;
  int tm, tn;
  const int b = blockIdx.x / kParts, part = blockIdx.x % kParts;
  if (g.lower) {
    int I = (int)((sqrtf(8.0f * (float)b + 1.0f) - 1.0f) * 0.5f);
    while (I * (I + 1) / 2 > b) --I;
    while ((I + 1) * (I + 2) / 2 <= b) ++I;
    tm = I;
    tn = b - I * (I + 1) / 2;
  } else {
    tm = b % g.tiles_m;
    tn = b / g.tiles_m;
  }
  if (g.trap && tm < tn) return;

  extern __shared__ __align__(1024) uint8_t oz_smem[];
  __shared__ __align__(8) uint64_t full_bar[Cfg::kStages], empty_bar[Cfg::kStages], acc_bar;
  __shared__ uint32_t tmem_base;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int kblocks = g.kblocks;

  if (threadIdx.x == 0) {
    for (int s = 0; s < Cfg::kStages; ++s) {
      mbar_init(&full_bar[s], 1);
      mbar_init(&empty_bar[s], 1);
    }
    mbar_init(&acc_bar, 1);
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                     smem_u32(&tmem_base)), "n"(Cfg::kTmemCols));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t tmem = tmem_base;

  const int8_t* Ablk = g.As[z] + (size_t)tm * kblocks * OZ_S * OZ_BLK;
  const int8_t* Bblk =
      g.Bs[z] + (size_t)tn * kblocks * OZ_S * OZ_BLK + (size_t)part * (kN * OZ_KB);

  if (warp == 0) {
    if (lane == 0) {
      // producer: one 32 KB bulk copy for the A slices, 8 copies for the B row range
      for (int kb = 0; kb < kblocks; ++kb) {
        const int st = kb % Cfg::kStages;
        if (kb >= Cfg::kStages) mbar_wait(&empty_bar[st], ((kb / Cfg::kStages) - 1) & 1);
        uint8_t* sa = oz_smem + (size_t)st * Cfg::kStage;
        uint8_t* sb = sa + OZ_A_STAGE;
        mbar_expect_tx(&full_bar[st], Cfg::kStage);
        bulk_g2s(sa, Ablk + (size_t)kb * OZ_S * OZ_BLK, OZ_A_STAGE, &full_bar[st]);
        const int8_t* bsrc = Bblk + (size_t)kb * OZ_S * OZ_BLK;
#pragma unroll
        for (int q = 0; q < OZ_S; ++q)
          bulk_g2s(sb + q * (kN * OZ_KB), bsrc + (size_t)q * OZ_BLK, kN * OZ_KB, &full_bar[st]);
      }
    }
    __syncwarp();
  } else if (warp == 1) {
    for (int kb = 0; kb < kblocks; ++kb) {
      const int st = kb % Cfg::kStages;
      mbar_wait(&full_bar[st], (kb / Cfg::kStages) & 1);
      asm volatile("tcgen05.fence::after_thread_sync;");
      if (lane == 0) {
        const uint32_t sa = smem_u32(oz_smem + (size_t)st * Cfg::kStage);
        const uint32_t sb = sa + OZ_A_STAGE;
#pragma unroll
        for (int p = 1; p <= OZ_S; ++p) {
          const uint64_t da = sdesc(sa + (p - 1) * OZ_BLK);
          const int rows = kN * (OZ_S + 1 - p);  // B rows [B_1 .. B_{9-p}]
          const uint32_t accum = (kb > 0 || p > 1) ? 1u : 0u;
#pragma unroll
          for (int r0 = 0; r0 < rows; r0 += 256) {
            const int nr = rows - r0 < 256 ? rows - r0 : 256;
            const uint32_t idesc = (2u << 4) | (1u << 7) | (1u << 10) |
                                   ((uint32_t)(nr >> 3) << 17) | ((uint32_t)(128 >> 4) << 24);
            const uint64_t db = sdesc(sb + r0 * OZ_KB);
            const uint32_t col = tmem + (uint32_t)((p - 1) * kN + r0);
            asm volatile(
                "{ .reg .pred pp; setp.ne.b32 pp, %4, 0;\n"
                "tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, pp; }" ::"r"(col),
                "l"(da), "l"(db), "r"(idesc), "r"(accum));
          }
        }
        asm volatile(
            "tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
                smem_u32(&empty_bar[st])));
      }
      __syncwarp();
    }
    if (lane == 0)
      asm volatile(
          "tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
              smem_u32(&acc_bar)));
    __syncwarp();
  } else {
    // epilogue: thread = one row of the tile (TMEM lane quadrant = warp % 4)
    const int qd = warp & 3;
    const int row = qd * 32 + lane;
    const long long r_glob = (long long)tm * 128 + row;
    const long long c_glob = (long long)tn * 128 + (long long)part * kN;
    double* C = g.C[z] + r_glob + c_glob * g.ldc;
    const int* eb = g.eb[z] + c_glob;
    const double alpha = g.alpha;
    const bool acc_c = g.beta != 0.0;
    const double s_row = alpha * pow2i(g.ea[z][r_glob]);
    constexpr int kPre = kN == 32 ? 32 : 16;  // C values prefetched before the main loop ends
    double cpre[kPre];
#pragma unroll
    for (int j = 0; j < kPre; ++j) cpre[j] = acc_c ? C[(long long)j * g.ldc] : 0.0;
    mbar_wait(&acc_bar, 0);
    asm volatile("tcgen05.fence::after_thread_sync;");
    double acc[kN];
#pragma unroll
    for (int j = 0; j < kN; ++j) acc[j] = 0.0;
#pragma unroll 1
    for (int d = OZ_S + 1; d >= 2; --d) {  // smallest contributions first
      const double w = pow2i(-7 * d);
#pragma unroll
      for (int c0 = 0; c0 < kN; c0 += 16) {
        uint32_t v[16];
        asm volatile(
            "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,"
            "%13,%14,%15}, [%16];"
            : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]),
              "=r"(v[6]), "=r"(v[7]), "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]),
              "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15])
            : "r"(tmem + ((uint32_t)(qd * 32) << 16) + (uint32_t)((d - 2) * kN + c0)));
        asm volatile("tcgen05.wait::ld.sync.aligned;");
#pragma unroll
        for (int j = 0; j < 16; ++j) acc[c0 + j] = fma((double)(int)v[j], w, acc[c0 + j]);
      }
    }
    // C = C + (alpha 2^ea) 2^eb acc: exact power-of-two scalings, one rounding in the add
#pragma unroll
    for (int c0 = 0; c0 < kN; c0 += kPre) {
      double cv[kPre];
      int ev[kPre];
#pragma unroll
      for (int j = 0; j < kPre; ++j) {
        cv[j] = c0 == 0 ? cpre[j] : (acc_c ? C[(long long)(c0 + j) * g.ldc] : 0.0);
        ev[j] = eb[c0 + j];
      }
#pragma unroll
      for (int j = 0; j < kPre; ++j)
        C[(long long)(c0 + j) * g.ldc] = cv[j] + (acc[c0 + j] * s_row) * pow2i(ev[j]);
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (warp == 0)
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem),
                 "n"(Cfg::kTmemCols));
}

cudaError_t init_ozaki_attributes() {
  cudaError_t e = cudaFuncSetAttribute(oz_slice_kernel<0>,
                                       cudaFuncAttributeMaxDynamicSharedMemorySize, kOzSliceSmem);
  if (e != cudaSuccess) return e;
  e = cudaFuncSetAttribute(oz_slice_kernel<1>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                           kOzSliceSmem);
  if (e != cudaSuccess) return e;
  e = cudaFuncSetAttribute(ozgemm_kernel<64>,
                                       cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       OzCfg<64>::kSmem);
  if (e != cudaSuccess) return e;
  return cudaFuncSetAttribute(ozgemm_kernel<32>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                              OzCfg<32>::kSmem);
}

cudaError_t launch_oz_slice(const OzSliceArgs& a, int rows, bool row_contig, int batch,
                            cudaStream_t s) {
  if (a.K > kOzSliceMaxK || a.K % OZ_KB || rows % 128) return cudaErrorInvalidValue;
  const dim3 grid((unsigned)(rows / kOzSliceRows), 1, (unsigned)batch);
  if (row_contig)
    oz_slice_kernel<1><<<grid, 256, kOzSliceSmem, s>>>(a);
  else
    oz_slice_kernel<0><<<grid, 256, kOzSliceSmem, s>>>(a);
  return cudaGetLastError();
}

cudaError_t launch_ozgemm(const OzGemmArgs& g, int batch, cudaStream_t s, int n_tile) {
  const long long tiles =
      g.lower ? (long long)g.tiles_m * (g.tiles_m + 1) / 2 : (long long)g.tiles_m * g.tiles_n;
  if (tiles <= 0) return cudaSuccess;
  if (n_tile == 64) {
    ozgemm_kernel<64><<<dim3((unsigned)(2 * tiles), 1, (unsigned)batch), OZ_THREADS,
                        OzCfg<64>::kSmem, s>>>(g);
  } else {
    ozgemm_kernel<32><<<dim3((unsigned)(4 * tiles), 1, (unsigned)batch), OZ_THREADS,
                        OzCfg<32>::kSmem, s>>>(g);
  }
  return cudaGetLastError();
}

}  // namespace mle
