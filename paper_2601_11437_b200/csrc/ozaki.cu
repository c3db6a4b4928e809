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

#include <algorithm>

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

// Epilogue combine for 16 columns of one TMEM lane: the 8 int32 diagonal accumulators v_d
// (d = 2..9, at column offsets (d - 2) * stride from `addr`) fold exactly into two int64
// Horner sums  hi = sum_{d=2..5} v_d 2^(7 (5 - d)),  lo = sum_{d=6..9} v_d 2^(7 (9 - d))
// (|v_d| < 2^26 for K <= 512, so |hi|, |lo| < 2^48 convert to double exactly), and
//   sum_d v_d 2^(-7 d) = hi 2^-35 + lo 2^-63
// is formed with a single rounding (one FMA).  2 conversions per element instead of 8.
__device__ __forceinline__ void oz_tmem_ld16(uint32_t addr, uint32_t (&v)[16]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,"
      "%13,%14,%15}, [%16];"
      : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]),
        "=r"(v[7]), "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]),
        "=r"(v[13]), "=r"(v[14]), "=r"(v[15])
      : "r"(addr));
}

__device__ __forceinline__ void oz_horner4(uint32_t addr, uint32_t stride, long long (&h)[16]) {
  uint32_t v0[16], v1[16], v2[16], v3[16];
  oz_tmem_ld16(addr, v0);
  oz_tmem_ld16(addr + stride, v1);
  oz_tmem_ld16(addr + 2 * stride, v2);
  oz_tmem_ld16(addr + 3 * stride, v3);
  asm volatile("tcgen05.wait::ld.sync.aligned;");
#pragma unroll
  for (int j = 0; j < 16; ++j)
    h[j] = ((((long long)(int)v0[j] * 128 + (int)v1[j]) * 128 + (int)v2[j]) * 128) +
           (int)v3[j];
}

__device__ __forceinline__ void oz_horner3(uint32_t addr, uint32_t stride, long long (&h)[16]) {
  uint32_t v0[16], v1[16], v2[16];
  oz_tmem_ld16(addr, v0);
  oz_tmem_ld16(addr + stride, v1);
  oz_tmem_ld16(addr + 2 * stride, v2);
  asm volatile("tcgen05.wait::ld.sync.aligned;");
#pragma unroll
  for (int j = 0; j < 16; ++j)
    h[j] = (((long long)(int)v0[j] * 128 + (int)v1[j]) * 128) + (int)v2[j];
}

// kS slices: diagonals d = 2..kS+1; hi over d = 2..5, lo over d = 6..kS+1.
template <int kS>
__device__ __forceinline__ void oz_combine16(uint32_t addr, uint32_t stride, double (&out)[16]) {
  static_assert(kS == 7 || kS == 8, "7 or 8 slices");
  long long hi[16], lo[16];
  oz_horner4(addr, stride, hi);
  if (kS == 8)
    oz_horner4(addr + 4 * stride, stride, lo);
  else
    oz_horner3(addr + 4 * stride, stride, lo);
  const double s_hi = pow2i(-35), s_lo = pow2i(-7 * (kS + 1));
#pragma unroll
  for (int j = 0; j < 16; ++j) out[j] = fma((double)hi[j], s_hi, (double)lo[j] * s_lo);
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

constexpr int kOzSliceThreads = 512;
constexpr int kOzSliceWarps = kOzSliceThreads / 32;

template <int kRowContig, int kS>
__global__ void __launch_bounds__(kOzSliceThreads) oz_slice_kernel(OzSliceArgs sa) {
  const int z = blockIdx.z;
  if (sa.fail_flag[z] && *sa.fail_flag[z]) return;
  extern __shared__ double tile[];  // [32][kOzSliceStride]
  __shared__ int ex[kOzSliceRows];
  const double* X = sa.X[z];
  const long long ld = sa.ld;
  const int K = sa.K, t = threadIdx.x, w = t >> 5, l = t & 31;
  const long long r0 = (long long)blockIdx.x * kOzSliceRows;
  if (sa.rows_z[z] > 0 && r0 >= sa.rows_z[z]) return;
  // loads: 16 independent 8-byte loads in flight per lane, then the shared-memory stores
  if (kRowContig) {  // X(r,k) = X[r + k ld]: lanes along r, warps over k
    constexpr int kStep = kOzSliceWarps * 16;
    for (int k0 = w; k0 < K; k0 += kStep) {
      double v[16];
#pragma unroll
      for (int q = 0; q < 16; ++q) {
        const int k = k0 + q * kOzSliceWarps;
        v[q] = k < K ? X[r0 + l + (long long)k * ld] : 0.0;
      }
#pragma unroll
      for (int q = 0; q < 16; ++q) {
        const int k = k0 + q * kOzSliceWarps;
        if (k < K) tile[l * kOzSliceStride + k] = v[q];
      }
    }
  } else {           // X(r,k) = X[k + r ld]: lanes along k, warps over rows
    for (int r = w; r < kOzSliceRows; r += kOzSliceWarps) {
      const double* row = X + (r0 + r) * ld;
      double v[16];
#pragma unroll
      for (int q = 0; q < 16; ++q) {
        const int k = l + 32 * q;
        v[q] = k < K ? row[k] : 0.0;
      }
#pragma unroll
      for (int q = 0; q < 16; ++q) {
        const int k = l + 32 * q;
        if (k < K) tile[r * kOzSliceStride + k] = v[q];
      }
    }
  }
  if (sa.upper_zero) {  // only the lower trapezoid k <= r is valid: zero the rest
    __syncthreads();
    for (int r = w; r < kOzSliceRows; r += kOzSliceWarps)
      for (int k = l; k < K; k += 32)
        if (k > r0 + r) tile[r * kOzSliceStride + k] = 0.0;
  }
  __syncthreads();
  for (int r = w; r < kOzSliceRows; r += kOzSliceWarps) {
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
  for (int item = t; item < kOzSliceRows * (K / 16); item += kOzSliceThreads) {
    const int r = item & (kOzSliceRows - 1), ch = item / kOzSliceRows;
    // |x| 2^(7 kS - e) < 2^(7 kS) is exact (power-of-two scaling); its truncation holds the
    // kS base-128 digits the float recurrence (x 2^7, trunc, subtract) would produce.
    const int sh = 7 * kS - ex[r];
    const double sc1 = pow2i(sh > 1000 ? 1000 : sh), sc2 = pow2i(sh > 1000 ? sh - 1000 : 0);
    const double* src = tile + r * kOzSliceStride + ch * 16;
    uint32_t wd[kS][4];
#pragma unroll
    for (int p = 0; p < kS; ++p) wd[p][0] = wd[p][1] = wd[p][2] = wd[p][3] = 0u;
#pragma unroll
    for (int c = 0; c < 16; ++c) {
      const double x = src[c];
      const unsigned long long u =
          (unsigned long long)__double2ll_rz(fabs(x) * sc1 * sc2);
      const bool neg = x < 0.0;
#pragma unroll
      for (int p = 0; p < kS; ++p) {
        const uint32_t d = (uint32_t)(u >> (7 * kS - 7 * (p + 1))) & 127u;
        const uint32_t byte = (neg ? (0u - d) : d) & 0xFFu;
        wd[p][c >> 2] |= byte << (8 * (c & 3));
      }
    }
    const int kb = ch >> 1, half = ch & 1;
    const int rl = rsub + r;
    int8_t* dst = out + ((size_t)(tile128 * kblocks + kb) * kS) * OZ_BLK +
                  (size_t)(rl >> 3) * 256 + (size_t)(rl & 7) * 16 + (size_t)half * 128;
#pragma unroll
    for (int p = 0; p < kS; ++p)
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
    const bool acc_c = g.beta != 0.0 && tm >= g.beta0_tm && tn >= g.beta0_tn;
    const double s_row = alpha * pow2i(g.ea[z][r_glob]);
    constexpr int kPre = kN == 32 ? 32 : 16;  // C values prefetched before the main loop ends
    double cpre[kPre];
#pragma unroll
    for (int j = 0; j < kPre; ++j) cpre[j] = acc_c ? C[(long long)j * g.ldc] : 0.0;
    mbar_wait(&acc_bar, 0);
    asm volatile("tcgen05.fence::after_thread_sync;");
    double acc[kN];
#pragma unroll
    for (int c0 = 0; c0 < kN; c0 += 16) {
      double part[16];
      oz_combine16<OZ_S>(tmem + ((uint32_t)(qd * 32) << 16) + (uint32_t)c0, kN, part);
#pragma unroll
      for (int j = 0; j < 16; ++j) acc[c0 + j] = part[j];
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


// Persistent variant: one CTA per SM walks the tile list (tile t, t + gridDim.x, ...).
// The kernel is bound by the shared-memory ingress of the slices (L2 -> SMEM, ~29 B/clk/SM
// measured), not by the tensor pipe: a 128 x kN tile needs 8 x 32 (128 + kN) bytes per k
// block for 36 x 128 x kN x 32 MACs, so kN = 64 halves the ingress per MAC of kN = 32.
//   kN = 32: 5-stage ring of 40 KB, two TMEM accumulator sets (2 x 256 columns): the
//            epilogue of one tile overlaps the main loop of the next.
//   kN = 64: 4-stage ring of 48 KB, one accumulator set (512 columns): the producer keeps
//            streaming the next tile's stages while the epilogue drains TMEM.
// 8 epilogue warps (two per TMEM lane quadrant, kN / 2 columns each).  Per-tile arithmetic
// is that of ozgemm_kernel, so every variant gives bit-identical results.
template <int kN, int kS = OZ_S>
struct OzP {
  static constexpr int kAStage = kS * OZ_BLK;
  static constexpr int kStage = kAStage + kS * kN * OZ_KB;
  static constexpr int kStages = kN == 32 ? 5 : (kS == 8 ? 4 : 5);
  static constexpr int kSmem = kStages * kStage;
  static constexpr int kAcc = kS * kN;              // TMEM columns per accumulator set
  static constexpr int kSets = kN == 32 ? 2 : 1;
};
constexpr int OZP_EPI_WARPS = 8;
constexpr int OZP_THREADS = 64 + 32 * OZP_EPI_WARPS;

struct OzTile {
  int z, tm, tn, part;
};

// Tile t of the launch -> coordinates; false if the tile is skipped (trapezoid / failed item).
template <int kN>
__device__ __forceinline__ bool oz_tile(const OzGemmArgs& g, long long per_z, long long t,
                                        OzTile& o) {
  constexpr int kParts = 128 / kN;
  o.z = (int)(t / per_z);
  const long long r = t - (long long)o.z * per_z;
  const int b = (int)(r / kParts);
  o.part = (int)(r % kParts);
  if (g.lower) {
    int I = (int)((sqrtf(8.0f * (float)b + 1.0f) - 1.0f) * 0.5f);
    while (I * (I + 1) / 2 > b) --I;
    while ((I + 1) * (I + 2) / 2 <= b) ++I;
    o.tm = I;
    o.tn = b - I * (I + 1) / 2;
  } else {
    o.tm = b % g.tiles_m;
    o.tn = b / g.tiles_m;
    if (g.tiles_m_z[o.z] > 0 && o.tm >= g.tiles_m_z[o.z]) return false;
  }
  if (g.trap && o.tm < o.tn) return false;
  return *g.fail_flag[o.z] == 0;
}

template <int kN, int kS>
__global__ void __launch_bounds__(OZP_THREADS, 1) ozgemm_persistent_kernel(OzGemmArgs g,
                                                                           long long per_z,
                                                                           long long total) {
  using Cfg = OzP<kN, kS>;
  extern __shared__ __align__(1024) uint8_t oz_smem[];
  __shared__ __align__(8) uint64_t full_bar[Cfg::kStages], empty_bar[Cfg::kStages];
  __shared__ __align__(8) uint64_t acc_full[Cfg::kSets], acc_empty[Cfg::kSets];
  __shared__ uint32_t tmem_base;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int kblocks = g.kblocks;

  if (threadIdx.x == 0) {
    for (int s = 0; s < Cfg::kStages; ++s) {
      mbar_init(&full_bar[s], 1);
      mbar_init(&empty_bar[s], 1);
    }
    for (int b = 0; b < Cfg::kSets; ++b) {
      mbar_init(&acc_full[b], 1);
      mbar_init(&acc_empty[b], OZP_EPI_WARPS);
    }
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

  if (warp == 0) {
    if (lane == 0) {  // producer
      long long gk = 0;
      for (long long t = blockIdx.x; t < total; t += gridDim.x) {
        OzTile o;
        if (!oz_tile<kN>(g, per_z, t, o)) continue;
        const int8_t* Ablk = g.As[o.z] + (size_t)o.tm * kblocks * kS * OZ_BLK;
        const int8_t* Bblk = g.Bs[o.z] + (size_t)o.tn * kblocks * kS * OZ_BLK +
                             (size_t)o.part * (kN * OZ_KB);
        for (int kb = 0; kb < kblocks; ++kb, ++gk) {
          const int st = (int)(gk % Cfg::kStages);
          const long long use = gk / Cfg::kStages;
          if (use >= 1) mbar_wait(&empty_bar[st], (uint32_t)((use - 1) & 1));
          uint8_t* sa = oz_smem + (size_t)st * Cfg::kStage;
          uint8_t* sb = sa + Cfg::kAStage;
          if (g.diag_mode == 2 || g.diag_mode >= 5) {
            asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(
                smem_u32(&full_bar[st])) : "memory");
            continue;
          }
          mbar_expect_tx(&full_bar[st], Cfg::kStage);
          bulk_g2s(sa, Ablk + (size_t)kb * kS * OZ_BLK, Cfg::kAStage, &full_bar[st]);
          const int8_t* bsrc = Bblk + (size_t)kb * kS * OZ_BLK;
#pragma unroll
          for (int q = 0; q < kS; ++q)
            bulk_g2s(sb + q * (kN * OZ_KB), bsrc + (size_t)q * OZ_BLK, kN * OZ_KB,
                     &full_bar[st]);
        }
      }
    }
    __syncwarp();
  } else if (warp == 1) {  // MMA issuer
    long long gk = 0, local = 0;
    long long c_start = clock64(), c_full = 0, c_acc = 0, g_start = 0;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(g_start));
    for (long long t = blockIdx.x; t < total; t += gridDim.x) {
      OzTile o;
      if (!oz_tile<kN>(g, per_z, t, o)) continue;
      const int ab = (int)(local % Cfg::kSets);
      const long long use = local / Cfg::kSets;
      {
        const long long c0 = clock64();
        if (use >= 1) mbar_wait(&acc_empty[ab], (uint32_t)((use - 1) & 1));
        c_acc += clock64() - c0;
      }
      asm volatile("tcgen05.fence::after_thread_sync;");
      const uint32_t acc = tmem + (uint32_t)(ab * Cfg::kAcc);
      for (int kb = 0; kb < kblocks; ++kb, ++gk) {
        const int st = (int)(gk % Cfg::kStages);
        {
          const long long c0 = clock64();
          mbar_wait(&full_bar[st], (uint32_t)((gk / Cfg::kStages) & 1));
          c_full += clock64() - c0;
        }
        asm volatile("tcgen05.fence::after_thread_sync;");
        if (lane == 0) {
          const uint32_t sa = smem_u32(oz_smem + (size_t)st * Cfg::kStage);
          const uint32_t sb = sa + Cfg::kAStage;
#pragma unroll
          for (int p = 1; p <= kS; ++p) {
            if (g.diag_mode == 1 && !(kb == 0 && p == 1)) continue;
            const int rows = kN * (kS + 1 - p);  // B rows [B_1 .. B_{kS+1-p}]
            const uint32_t accum = (kb > 0 || p > 1) ? 1u : 0u;
#pragma unroll
            for (int r0 = 0; r0 < rows; r0 += 256) {
              const int nr = rows - r0 < 256 ? rows - r0 : 256;
              const uint32_t idesc = (2u << 4) | (1u << 7) | (1u << 10) |
                                     ((uint32_t)(nr >> 3) << 17) | ((uint32_t)(128 >> 4) << 24);
              asm volatile(
                  "{ .reg .pred pp; setp.ne.b32 pp, %4, 0;\n"
                  "tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, pp; }" ::"r"(
                      acc + (uint32_t)((p - 1) * kN + r0)),
                  "l"(sdesc(sa + (p - 1) * OZ_BLK)), "l"(sdesc(sb + r0 * OZ_KB)), "r"(idesc),
                  "r"(accum));
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
                smem_u32(&acc_full[ab])));
      __syncwarp();
      ++local;
    }
    if (g.diag_out && blockIdx.x == 0 && lane == 0) {
      long long g_end;
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(g_end));
      g.diag_out[0] = clock64() - c_start;
      g.diag_out[1] = c_full;
      g.diag_out[2] = c_acc;
      g.diag_out[3] = g_end - g_start;
      g.diag_out[4] = local;
      g.diag_out[5] = gk;
    }
  } else {  // epilogue: warp pair per TMEM lane quadrant, kN / 2 columns each
    constexpr int kCols = kN / 2;
    const int ew = warp - 2;
    const int qd = warp & 3;           // lane quadrant this warp may access
    const int ch = ew >> 2;            // column half
    const int row = qd * 32 + lane;
    long long local = 0;
    for (long long t = blockIdx.x; t < total; t += gridDim.x) {
      OzTile o;
      if (!oz_tile<kN>(g, per_z, t, o)) continue;
      const int ab = (int)(local % Cfg::kSets);
      const long long use = local / Cfg::kSets;
      const long long r_glob = (long long)o.tm * 128 + row;
      const long long c_glob = (long long)o.tn * 128 + (long long)o.part * kN + ch * kCols;
      double* C = g.C[o.z] + r_glob + c_glob * g.ldc;
      const bool acc_c = g.beta != 0.0 && o.tm >= g.beta0_tm && o.tn >= g.beta0_tn;
      // C prefetch before the accumulator wait (kN = 32; at kN = 64 it would spill: C is
      // then read after TMEM is released, overlapping the next tile's MMAs)
      constexpr int kPre = kN == 32 ? kCols : 0;
      double cv[kPre > 0 ? kPre : 1];
#pragma unroll
      for (int j = 0; j < kPre; ++j) cv[j] = acc_c ? __ldcg(C + (long long)j * g.ldc) : 0.0;
      const double s_row = g.alpha * pow2i(g.ea[o.z][r_glob]);
      mbar_wait(&acc_full[ab], (uint32_t)(use & 1));
      asm volatile("tcgen05.fence::after_thread_sync;");
      double acc[kCols];
#pragma unroll
      for (int c0 = 0; c0 < kCols; c0 += 16) {
        double part[16];
        if (g.diag_mode != 3 && g.diag_mode < 5)
          oz_combine16<kS>(tmem + ((uint32_t)(qd * 32) << 16) +
                           (uint32_t)(ab * Cfg::kAcc + ch * kCols + c0),
                       kN, part);
#pragma unroll
        for (int j = 0; j < 16; ++j)
          acc[c0 + j] = (g.diag_mode != 3 && g.diag_mode < 5) ? part[j] : 0.0;
      }
      asm volatile("tcgen05.fence::before_thread_sync;");
      __syncwarp();
      if (lane == 0)
        asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(&acc_empty[ab]))
                     : "memory");
      const int* eb = g.eb[o.z] + c_glob;
      if (g.diag_mode == 6) {
        ++local;
        continue;
      }
#pragma unroll
      for (int c0 = 0; c0 < kCols; c0 += 16) {
        double cw[16];
#pragma unroll
        for (int j = 0; j < 16; ++j)
          cw[j] = kPre > 0 ? cv[(c0 + j) % (kPre > 0 ? kPre : 1)]
                           : (acc_c ? __ldcg(C + (long long)(c0 + j) * g.ldc) : 0.0);
#pragma unroll
        for (int j = 0; j < 16; ++j)
          __stcg(C + (long long)(c0 + j) * g.ldc,
                 cw[j] + (acc[c0 + j] * s_row) * pow2i(__ldg(eb + c0 + j)));
      }
      ++local;
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (warp == 0)
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tmem));
}

int g_num_sms = 148;

cudaError_t init_ozaki_attributes() {
  int dev = 0;
  if (cudaGetDevice(&dev) == cudaSuccess)
    cudaDeviceGetAttribute(&g_num_sms, cudaDevAttrMultiProcessorCount, dev);
  cudaError_t e0 = cudaFuncSetAttribute(ozgemm_persistent_kernel<32, 8>,
                                        cudaFuncAttributeMaxDynamicSharedMemorySize,
                                        OzP<32, 8>::kSmem);
  if (e0 != cudaSuccess) return e0;
  e0 = cudaFuncSetAttribute(ozgemm_persistent_kernel<64, 8>,
                            cudaFuncAttributeMaxDynamicSharedMemorySize, OzP<64, 8>::kSmem);
  if (e0 != cudaSuccess) return e0;
  e0 = cudaFuncSetAttribute(ozgemm_persistent_kernel<64, 7>,
                            cudaFuncAttributeMaxDynamicSharedMemorySize, OzP<64, 7>::kSmem);
  if (e0 != cudaSuccess) return e0;
  cudaError_t e = cudaSuccess;
#define MLE_SLICE_ATTR(RC, S)                                                              \
  e = cudaFuncSetAttribute(oz_slice_kernel<RC, S>, cudaFuncAttributeMaxDynamicSharedMemorySize, \
                           kOzSliceSmem);                                                  \
  if (e != cudaSuccess) return e;
  MLE_SLICE_ATTR(0, 8)
  MLE_SLICE_ATTR(1, 8)
  MLE_SLICE_ATTR(0, 7)
  MLE_SLICE_ATTR(1, 7)
#undef MLE_SLICE_ATTR
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
  const bool seven = a.nslices == 7;
  if (row_contig && seven)
    oz_slice_kernel<1, 7><<<grid, kOzSliceThreads, kOzSliceSmem, s>>>(a);
  else if (row_contig)
    oz_slice_kernel<1, 8><<<grid, kOzSliceThreads, kOzSliceSmem, s>>>(a);
  else if (seven)
    oz_slice_kernel<0, 7><<<grid, kOzSliceThreads, kOzSliceSmem, s>>>(a);
  else
    oz_slice_kernel<0, 8><<<grid, kOzSliceThreads, kOzSliceSmem, s>>>(a);
  return cudaGetLastError();
}

cudaError_t launch_ozgemm(const OzGemmArgs& g, int batch, cudaStream_t s, int n_tile) {
  const long long tiles =
      g.lower ? (long long)g.tiles_m * (g.tiles_m + 1) / 2 : (long long)g.tiles_m * g.tiles_n;
  if (tiles <= 0) return cudaSuccess;
  if (n_tile == 0 || n_tile == 1) {  // persistent: 0 -> 128 x 64 tiles, 1 -> 128 x 32
    const int kn = n_tile == 0 ? 64 : 32;
    const long long per_z = tiles * (128 / kn), total = per_z * batch;
    const long long cap = g.max_ctas > 0 ? std::min(g.max_ctas, g_num_sms) : g_num_sms;
    const long long grid = std::min<long long>(total, cap);
    if (kn == 64 && g.nslices == 7)
      ozgemm_persistent_kernel<64, 7><<<(unsigned)grid, OZP_THREADS, OzP<64, 7>::kSmem, s>>>(
          g, per_z, total);
    else if (kn == 64)
      ozgemm_persistent_kernel<64, 8><<<(unsigned)grid, OZP_THREADS, OzP<64, 8>::kSmem, s>>>(
          g, per_z, total);
    else
      ozgemm_persistent_kernel<32, 8><<<(unsigned)grid, OZP_THREADS, OzP<32, 8>::kSmem, s>>>(
          g, per_z, total);
  } else if (n_tile == 64) {
    ozgemm_kernel<64><<<dim3((unsigned)(2 * tiles), 1, (unsigned)batch), OZ_THREADS,
                        OzCfg<64>::kSmem, s>>>(g);
  } else {
    ozgemm_kernel<32><<<dim3((unsigned)(4 * tiles), 1, (unsigned)batch), OZ_THREADS,
                        OzCfg<32>::kSmem, s>>>(g);
  }
  return cudaGetLastError();
}

}  // namespace mle
