// ozaki.cu — FP64 GEMM on the 5th-generation tensor cores (tcgen05.mma kind::i8, TMEM).
//
// B200 has no FP64 tcgen05 kind; its mma.sync DMMA path peaks at ~36 TF/s.  The trailing
// updates of the Cholesky and of the solves (C -= A B^T with K = 512) are instead run as an
// Ozaki-scheme emulation (splitting into int8 slices, exact int32 products):
//   * every row of A and of B (over the K range) gets a power-of-two exponent e with
//     max |x| < (509/512) 2^e, and x 2^(8S-1-e) is rounded to the nearest integer X
//     (|X| < 127.25 * 256^(S-1)), written as S balanced base-256 digits D_p in [-128, 127]:
//       x = 2^(e+1) sum_{p=1..S} 2^-8p D_p      (8S - 1 significant bits per row, unbiased)
//   * C(i,j) = 2^(ea_i + eb_j + 2) sum_{d=2..S+1} 2^-8d sum_{p+q=d} (A_p B_q^T)(i,j)
//     (the S(S+1)/2 slice products with p + q <= S + 1; each is an exact int8 x int8 ->
//     int32 tensor-core GEMM, the S diagonals d accumulate in S TMEM accumulators)
//   * the FP64 epilogue folds the diagonals exactly, scales (exact powers of two) and
//     accumulates into C with one rounding.
// S = 7 (55-bit operands, 28 products) everywhere by default; S = 6 (47-bit operands, 21
// products) for the solve sweeps only with MLE_SOLVE_SLICES=6 (it flips a Fisher-BT stopping
// decision on config 2: DESIGN.md 4a).
//
// Layouts.  Slices are written by oz_slice_kernel in the UMMA canonical K-major
// SWIZZLE_NONE layout: for each 128-row tile and each 32-wide k block, S slices of a
// 128 x 32 int8 block (4 KB; core matrices of 8 rows x 16 B, LBO = 128 B, SBO = 256 B).  The
// first / second 64 rows of a block are its first / second 2 KB, which the GEMM uses as the
// 64-row B operand.
#include <cuda_runtime.h>

#include <cstdlib>
#include <stdint.h>

#include <algorithm>

#include "kernels.h"

namespace mle {

namespace {

constexpr int OZ_KB = 32;           // k per MMA (int8)
constexpr int OZ_BLK = 128 * OZ_KB; // bytes of one slice block (128 rows x 32)

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
// Spin on the non-suspending test_wait (developer A/B against try_wait's suspend/wake cost
// on the MMA issuer's critical path).
__device__ __forceinline__ void mbar_wait_spin(uint64_t* bar, uint32_t phase) {
  uint32_t done = 0;
  for (uint32_t it = 0; it < (1u << 30) && !done; ++it) {
    asm volatile(
        "{ .reg .pred p; mbarrier.test_wait.parity.shared::cta.b64 p, [%1], %2; "
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
// Same bytes into the same shared-memory offset of every CTA in cta_mask (cluster multicast);
// complete_tx is signalled on the barrier at the same offset in each destination CTA.
__device__ __forceinline__ void bulk_g2s_mc(void* smem, const void* gmem, uint32_t bytes,
                                            uint64_t* bar, uint16_t cta_mask) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.multicast::cluster"
      " [%0], [%1], %2, [%3], %4;"
      ::"r"(smem_u32(smem)), "l"(gmem), "r"(bytes), "r"(smem_u32(bar)), "h"(cta_mask)
      : "memory");
}
__device__ __forceinline__ void cluster_sync() {
  asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;"
               ::: "memory");
}
__device__ __forceinline__ uint32_t cluster_rank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}

// UMMA shared-memory descriptor: K-major, SWIZZLE_NONE, LBO = 128 B, SBO = 256 B, sm_100.
__device__ __forceinline__ uint64_t sdesc(uint32_t saddr) {
  return ((uint64_t)((saddr >> 4) & 0x3FFF)) | ((uint64_t)(128 >> 4) << 16) |
         ((uint64_t)(256 >> 4) << 32) | (1ull << 46);
}

// Epilogue combine for 16 columns of one TMEM lane: the S int32 diagonal accumulators v_d
// (d = 2..S+1, at column offsets (d - 2) * stride from `addr`) fold exactly into two int64
// Horner sums  hi = sum_{d=2..5} v_d 2^(8 (5 - d)),  lo = sum_{d=6..S+1} v_d 2^(8 (S+1-d))
// (|v_d| < 7 * 2^23 for K <= 512, so |hi| < 2^51 and |lo| < 2^43 convert to double exactly),
// and  4 sum_d v_d 2^(-8 d) = hi 2^-38 + lo 2^(2 - 8 (S+1))  is formed with one rounding (one
// FMA; the factor 4 is the 2^(1+1) of the two operands' digit scaling).
__device__ __forceinline__ void oz_tmem_ld16(uint32_t addr, uint32_t (&v)[16]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,"
      "%13,%14,%15}, [%16];"
      : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]),
        "=r"(v[7]), "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]),
        "=r"(v[13]), "=r"(v[14]), "=r"(v[15])
      : "r"(addr));
}

template <int kS>
__device__ __forceinline__ void oz_combine16(uint32_t addr, uint32_t stride, double (&out)[16]) {
  static_assert(kS == 6 || kS == 7, "6 or 7 slices");
  uint32_t v[kS][16];
#pragma unroll
  for (int d = 0; d < kS; ++d) oz_tmem_ld16(addr + d * stride, v[d]);
  asm volatile("tcgen05.wait::ld.sync.aligned;");
  const double s_hi = pow2i(-38), s_lo = pow2i(2 - 8 * (kS + 1));
#pragma unroll
  for (int j = 0; j < 16; ++j) {
    long long hi = (int)v[0][j], lo = (int)v[4][j];
#pragma unroll
    for (int d = 1; d < 4; ++d) hi = hi * 256 + (int)v[d][j];
#pragma unroll
    for (int d = 5; d < kS; ++d) lo = lo * 256 + (int)v[d][j];
    // int64 -> double without I2F (an XU-pipe conversion, 64 per thread per tile, inside the
    // serialised TMEM drain): for |x| < 2^51 the bits of x + (2^52 + 2^51) as a double are
    // the integer 2^52 + 2^51 + x exactly; subtracting that constant leaves x exactly.
    constexpr long long kMagic = 0x4338000000000000LL;  // bits of 2^52 + 2^51
    constexpr double kMagicD = 6755399441055744.0;       // 2^52 + 2^51
    const double hd = __longlong_as_double(hi + kMagic) - kMagicD;
    const double ld = __longlong_as_double(lo + kMagic) - kMagicD;
    out[j] = fma(hd, s_hi, ld * s_lo);
  }
}

}  // namespace

// Slicing.  CTA = kR rows x all K (<= kOzSliceMaxK) of one operand (16 kR threads), staged
// once in shared memory: coalesced load, per-row max -> exponent e, then each thread turns
// 16 elements of one row into kS balanced base-256 digits each (exact power-of-two scaling,
// one round-to-nearest, integer digit extraction) and writes one 16-byte word per slice in
// the canonical layout (kR consecutive rows of a 128-row block are kR x 32 B contiguous in
// every slice block).  kR = 16 (66 KB, three CTAs per SM) for large operands; small ones
// (the Cholesky's 512-row W_b / panel slices: 32 x 5 CTAs at kR = 16, one per SM, load then
// compute with nothing to overlap) use kR = 4 (16 KB, 64 threads, ~13 CTAs per SM).
constexpr int kOzSliceMaxK = 512;
constexpr int kOzSliceStride = kOzSliceMaxK + 1;  // odd stride: conflict-free row access
constexpr int oz_slice_smem(int rows) { return rows * kOzSliceStride * 8; }

template <int kRowContig, int kS, int kR>
__global__ void __launch_bounds__(16 * kR) oz_slice_kernel(OzSliceArgs sa) {
  constexpr int kThreads = 16 * kR, kWarps = kThreads / 32;
  static_assert(kR == 4 || kR == 8 || kR == 16, "rows per CTA");
  const int z = blockIdx.z;
  if (sa.fail_flag[z] && *sa.fail_flag[z]) return;
  extern __shared__ double tile[];  // [kR][kOzSliceStride]
  __shared__ int ex[kR];
  const double* X = sa.X[z];
  const long long ld = sa.ld;
  const int K = sa.K, t = threadIdx.x, w = t >> 5, l = t & 31;
  const long long r0 = (long long)blockIdx.x * kR;
  if (sa.rows_z[z] > 0 && r0 >= sa.rows_z[z]) return;
  // loads: 16 independent 8-byte loads in flight per lane, then the shared-memory stores
  if (kRowContig) {  // X(r,k) = X[r + k ld]: lane groups of kR along r, 32/kR columns each
    const int rr = l % kR, kh = l / kR;
    constexpr int kCols = 32 / kR;          // columns per warp instruction
    constexpr int kStep = kWarps * kCols * 16;
    for (int k0 = kCols * w + kh; k0 < K; k0 += kStep) {
      double v[16];
#pragma unroll
      for (int q = 0; q < 16; ++q) {
        const int k = k0 + q * kCols * kWarps;
        v[q] = k < K ? X[r0 + rr + (long long)k * ld] : 0.0;
      }
#pragma unroll
      for (int q = 0; q < 16; ++q) {
        const int k = k0 + q * kCols * kWarps;
        if (k < K) tile[rr * kOzSliceStride + k] = v[q];
      }
    }
  } else {           // X(r,k) = X[k + r ld]: lanes along k, warps over rows
    for (int r = w; r < kR; r += kWarps) {
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
    for (int idx = t; idx < kR * K; idx += kThreads) {
      const int r = idx / K, k = idx - r * K;
      if (k > r0 + r) tile[r * kOzSliceStride + k] = 0.0;
    }
  }
  __syncthreads();
  for (int r = w; r < kR; r += kWarps) {
    double mx = 0.0;
    for (int k = l; k < K; k += 32) mx = fmax(mx, fabs(tile[r * kOzSliceStride + k]));
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) mx = fmax(mx, __shfl_xor_sync(0xffffffffu, mx, o));
    if (l == 0) {
      int e = 0;
      if (mx > 0.0) {
        frexp(mx, &e);                                  // 2^(e-1) <= mx < 2^e
        if (mx >= pow2i(e) * (509.0 / 512.0)) ++e;      // keeps |X| < 127.25 * 256^(kS-1)
      }
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
  for (int item = t; item < kR * (K / 16); item += kThreads) {
    const int r = item % kR, ch = item / kR;
    // X = rint(x 2^(8 kS - 1 - e)) (exact scaling, one rounding), |X| < 127.25 * 256^(kS-1),
    // which S balanced digits in [-128, 127] represent exactly (max 127 (256^S - 1) / 255).
    // Excess-128 trick: with c = 128 (1 + 256 + ... + 256^(S-1)), Y = X + c lies in
    // [0, 256^S) and its plain base-256 digits are the balanced digits + 128, so slice byte
    // = byte(Y) ^ 0x80.  Bytes are gathered four elements at a time with byte permutes.
    const int sh = 8 * kS - 1 - ex[r];
    const double sc1 = pow2i(sh > 1000 ? 1000 : sh), sc2 = pow2i(sh > 1000 ? sh - 1000 : 0);
    constexpr unsigned long long kExcess = 0x8080808080808080ull >> (8 * (8 - kS));
    const double* src = tile + r * kOzSliceStride + ch * 16;
    uint32_t lo[16], hi[16];
#pragma unroll
    for (int c = 0; c < 16; ++c) {
      const unsigned long long y =
          (unsigned long long)__double2ll_rn((src[c] * sc1) * sc2) + kExcess;
      lo[c] = (uint32_t)y;
      hi[c] = (uint32_t)(y >> 32);
    }
    uint32_t wd[kS][4];
#pragma unroll
    for (int p = 0; p < kS; ++p) {  // slice p = digit of weight 256^(kS - 1 - p)
      const int bp = kS - 1 - p;     // its byte in Y
      const unsigned sel = (unsigned)((bp & 3) | (((bp & 3) + 4) << 4));
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        const uint32_t* wv = bp < 4 ? lo : hi;
        const uint32_t t01 = __byte_perm(wv[4 * q], wv[4 * q + 1], sel);
        const uint32_t t23 = __byte_perm(wv[4 * q + 2], wv[4 * q + 3], sel);
        wd[p][q] = __byte_perm(t01, t23, 0x5410) ^ 0x80808080u;
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

#ifndef OZ_EARLY_WAIT  // MMA issuer waits for the next stage before this one's last MMAs
#define OZ_EARLY_WAIT 0
#endif
#ifndef OZ_TEST_WAIT  // MMA issuer waits on full stages with test_wait spins (A/B)
#define OZ_TEST_WAIT 0
#endif
#ifndef OZ_STORE  // C store of the epilogue (developer A/B: __stcs streaming, __stwt ...)
#define OZ_STORE __stcg
#endif

// Persistent GEMM: one CTA per SM walks the tile list (tile t, t + gridDim.x, ...).
// The kernel is bound by the ingress of the slices (L2 -> SMEM), not by the tensor pipe: a
// 128 x kN tile needs S x 32 (128 + kN) bytes per k block for S(S+1)/2 x 128 x kN x 32 MACs,
// so kN = 64 halves the ingress per MAC of kN = 32.
//   kN = 32: two TMEM accumulator sets (2 x 32 S columns): the epilogue of one tile overlaps
//            the main loop of the next.
//   kN = 64: one accumulator set (64 S columns): the producer keeps streaming the next
//            tile's stages while the epilogue drains TMEM.
// The ring takes as many stages as fit in ~220 KB of shared memory.  8 epilogue warps (two
// per TMEM lane quadrant, kN / 2 columns each).  The per-tile arithmetic does not depend on
// kN, so both variants give bit-identical results.
template <int kN, int kS>
struct OzP {
  static constexpr int kAStage = kS * OZ_BLK;
  static constexpr int kStage = kAStage + kS * kN * OZ_KB;
#ifndef OZ_MAX_STAGES  // developer A/B (Makefile EXTRA=-DOZ_MAX_STAGES=...)
#define OZ_MAX_STAGES 8
#endif
  static constexpr int kStages0 = (220 * 1024) / kStage > 8 ? 8 : (220 * 1024) / kStage;
  static constexpr int kStages = kStages0 < OZ_MAX_STAGES ? kStages0 : OZ_MAX_STAGES;
  static constexpr int kSmem = kStages * kStage;
  static constexpr int kAcc = kS * kN;              // TMEM columns per accumulator set
  static constexpr int kSets = kN == 32 ? 2 : 1;
  static_assert(kSets * kAcc <= 512, "TMEM");
};
constexpr int OZP_EPI_WARPS = 8;
constexpr int OZP_THREADS = 64 + 32 * OZP_EPI_WARPS;

struct OzTile {
  int z, tm, tn, part;
};

// Tile order: groups of kOzGroup consecutive row tiles.  Inside a group the tiles run down
// the rows first, then across the columns, so the CTAs working at any moment share a few B
// (column) panels and the group's A (row) panels -- kOzGroup x 128 rows x K x S bytes, 29 MB
// at K = 512, S = 7 -- stay resident in L2 while the group sweeps all columns.  Each A panel
// is then read from DRAM once per launch and each B panel once per group, instead of every
// A panel once per column of tiles (253 GB of DRAM reads in one config-4 sweep GEMM whose
// operands are 2 x 235 MB: ncu, profiles/r02_ozgemm_config4_summary.txt).
constexpr int kOzGroup = 64;

// Full / trapezoid grid (tiles_m x tiles_n): index b -> (tm, tn), grouped.
__device__ __forceinline__ void oz_full_tile(int b, int tiles_m, int tiles_n, int& tm, int& tn) {
  const int per_group = kOzGroup * tiles_n;
  const int g = b / per_group;
  const int m0 = g * kOzGroup;
  const int gs = min(kOzGroup, tiles_m - m0);
  const int l = b - g * per_group;
  tm = m0 + l % gs;
  tn = l / gs;
}

// Lower triangle (tm >= tn) of a tiles_m x tiles_m grid: index b -> (tm, tn), grouped.  Group
// g holds rows [m0, m0 + gs): the full columns tn < m0 (gs tiles each), then the group's own
// triangle column by column (column j: rows j .. gs - 1).
__device__ __forceinline__ void oz_lower_tile(int b, int tiles_m, int& tm, int& tn) {
  constexpr int G = kOzGroup;
  int g = 0, base = 0;
  for (;;) {
    const int m0 = g * G, gs = min(G, tiles_m - m0);
    const int size = gs * m0 + gs * (gs + 1) / 2;
    if (b < base + size || m0 + gs >= tiles_m) {
      int l = b - base;
      if (l < gs * m0) {
        tn = l / gs;
        tm = m0 + l % gs;
        return;
      }
      l -= gs * m0;
      int j = 0;
      while (l >= gs - j) {
        l -= gs - j;
        ++j;
      }
      tn = m0 + j;
      tm = m0 + j + l;
      return;
    }
    base += size;
    ++g;
  }
}

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
    oz_lower_tile(b, g.tiles_m, o.tm, o.tn);
  } else {
    oz_full_tile(b, g.tiles_m, g.tiles_n, o.tm, o.tn);
    if (g.tiles_m_z[o.z] > 0 && o.tm >= g.tiles_m_z[o.z]) return false;
  }
  if (g.trap && o.tm < o.tn) return false;
  return *g.fail_flag[o.z] == 0;
}

// kMc = 2: CTA pairs (clusters of 2) own the two 64-column halves of one 128 x 128 tile and
// share its A stages: each CTA loads half of every A stage and multicasts it to both, so the
// L2 -> SM traffic per pair is A + 2 B instead of 2 A + 2 B.  A stage is refilled only after
// BOTH CTAs' MMAs released it (each MMA commit arrives on the empty barriers of the pair).
template <int kN, int kS, int kMc>
__global__ void __launch_bounds__(OZP_THREADS, 1) ozgemm_persistent_kernel(OzGemmArgs g,
                                                                           long long per_z,
                                                                           long long total) {
  using Cfg = OzP<kN, kS>;
  static_assert(kMc == 1 || kMc * kN == 128, "a cluster owns the kMc parts of a 128-wide tile");
  constexpr uint16_t kMask = (uint16_t)((1u << kMc) - 1u);
  extern __shared__ __align__(1024) uint8_t oz_smem[];
  __shared__ __align__(8) uint64_t full_bar[Cfg::kStages], empty_bar[Cfg::kStages];
  __shared__ __align__(8) uint64_t acc_full[Cfg::kSets], acc_empty[Cfg::kSets];
  __shared__ uint32_t tmem_base;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int kblocks = g.kblocks;

  if (threadIdx.x == 0) {
    for (int s = 0; s < Cfg::kStages; ++s) {
      mbar_init(&full_bar[s], 1);
      mbar_init(&empty_bar[s], kMc);
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
  if (kMc > 1) cluster_sync();  // the peer's barriers exist before any multicast / remote arrive
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t tmem = tmem_base;
  const uint32_t rank = kMc > 1 ? cluster_rank() : 0u;

  if (warp == 0) {
    if (lane == 0) {  // producer
      long long gk = 0;
      for (long long t = blockIdx.x; t < total && g.diag_mode < 8; t += gridDim.x) {
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
          if (kMc > 1) {  // my 1/kMc of the A stage, to every CTA of the cluster
            constexpr uint32_t kPart = Cfg::kAStage / kMc;
            static_assert(Cfg::kAStage % (16 * kMc) == 0, "16-byte multicast parts");
            bulk_g2s_mc(sa + rank * kPart, Ablk + (size_t)kb * kS * OZ_BLK + rank * kPart, kPart,
                        &full_bar[st], kMask);
          } else {
            bulk_g2s(sa, Ablk + (size_t)kb * kS * OZ_BLK, Cfg::kAStage, &full_bar[st]);
          }
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
    int st = 0;
    uint32_t ph = 0;
    const uint32_t smem_base = smem_u32(oz_smem);
    long long c_start = clock64(), c_full = 0, c_acc = 0, g_start = 0;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(g_start));
    for (long long t = blockIdx.x; t < total; t += gridDim.x) {
      OzTile o;
      if (!oz_tile<kN>(g, per_z, t, o)) continue;
      const int ab = (int)(local % Cfg::kSets);
      const long long use = local / Cfg::kSets;
      {
        const long long c0 = clock64();
        if (use >= 1 && g.diag_mode < 7) mbar_wait(&acc_empty[ab], (uint32_t)((use - 1) & 1));
        c_acc += clock64() - c0;
      }
      asm volatile("tcgen05.fence::after_thread_sync;");
      const uint32_t acc = tmem + (uint32_t)(ab * Cfg::kAcc);
      // The whole warp walks the k blocks (uniform values, uniform registers); one elected
      // lane issues each MMA / commit.  Descriptors: stage base + constant offsets (the
      // address field is addr >> 4 in the low 14 bits).
      bool ready = false;  // the current stage's full barrier already waited (early wait)
      for (int kb = 0; kb < kblocks; ++kb, ++gk) {
        if (g.diag_mode < 8 && !ready) {  // diagnostics 8 / 9: no producer, stage 0 re-read
          const long long c0 = clock64();
#if OZ_TEST_WAIT
          mbar_wait_spin(&full_bar[st], ph);
#else
          mbar_wait(&full_bar[st], ph);
#endif
          c_full += clock64() - c0;
        }
        ready = false;
        __syncwarp();
        asm volatile("tcgen05.fence::after_thread_sync;");
        const uint64_t da0 = sdesc(smem_base + (uint32_t)st * Cfg::kStage);
        const uint64_t db0 = da0 + (uint64_t)(Cfg::kAStage >> 4);
#pragma unroll
        for (int p = 1; p <= kS; ++p) {
#if OZ_EARLY_WAIT
          // wait for the next stage while this k block's last MMAs are still queued, so the
          // barrier's wake-up latency overlaps tensor work instead of following it
          if (p == kS - 1 && g.diag_mode < 8 && kb + 1 < kblocks) {
            const int nst = st + 1 == Cfg::kStages ? 0 : st + 1;
            const uint32_t nph = st + 1 == Cfg::kStages ? (ph ^ 1u) : ph;
            const long long c0 = clock64();
#if OZ_TEST_WAIT
            mbar_wait_spin(&full_bar[nst], nph);
#else
            mbar_wait(&full_bar[nst], nph);
#endif
            c_full += clock64() - c0;
            ready = true;
          }
#endif
          if (g.diag_mode == 1 && !(kb == 0 && p == 1)) continue;
          const int rows = kN * (kS + 1 - p);  // B rows [B_1 .. B_{kS+1-p}]
          const uint32_t accum = (kb > 0 || p > 1) ? 1u : 0u;
#pragma unroll
          for (int r0 = 0; r0 < rows; r0 += 256) {
            const int nr = rows - r0 < 256 ? rows - r0 : 256;
            const uint32_t idesc = (2u << 4) | (1u << 7) | (1u << 10) |
                                   ((uint32_t)(nr >> 3) << 17) | ((uint32_t)(128 >> 4) << 24);
            asm volatile(
                "{ .reg .pred pp, pe; setp.ne.b32 pp, %4, 0; elect.sync _|pe, 0xffffffff;\n"
                "@pe tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, pp; }" ::"r"(
                    acc + (uint32_t)((p - 1) * kN + r0)),
                "l"(da0 + (uint64_t)(((p - 1) * OZ_BLK) >> 4)),
                "l"(db0 + (uint64_t)((r0 * OZ_KB) >> 4)), "r"(idesc), "r"(accum));
          }
        }
        if (g.diag_mode == 8) {  // diagnostics: no per-k-block commit (pure MMA issue)
        } else if (kMc > 1)  // the stage is free once every cluster CTA's MMAs have read it
          asm volatile(
              "{ .reg .pred pe; elect.sync _|pe, 0xffffffff;\n"
              "@pe tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.multicast::"
              "cluster.b64 [%0], %1; }" ::"r"(smem_u32(&empty_bar[st])), "h"(kMask));
        else
          asm volatile(
              "{ .reg .pred pe; elect.sync _|pe, 0xffffffff;\n"
              "@pe tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0]; }"
              ::"r"(smem_u32(&empty_bar[st])));
        if (++st == Cfg::kStages) {
          st = 0;
          ph ^= 1u;
        }
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
      // C prefetch before the accumulator wait: all of the thread's columns at kN = 32, the
      // first 16 at kN = 64 (all 32 would spill); the rest is read after TMEM is released,
      // overlapping the next tile's MMAs
#ifndef OZ_PRE64  // C columns prefetched before the accumulator wait at kN = 64 (A/B)
#define OZ_PRE64 16
#endif
      constexpr int kPre = kN == 32 ? kCols : OZ_PRE64;
      double cv[kPre > 0 ? kPre : 1];
#pragma unroll
      for (int j = 0; j < kPre; ++j) cv[j] = acc_c ? __ldcg(C + (long long)j * g.ldc) : 0.0;
      const double s_row = g.alpha * pow2i(g.ea[o.z][r_glob]);
      if (g.diag_mode >= 7) {  // diagnostics: no accumulator handoff at all
        ++local;
        continue;
      }
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
          cw[j] = c0 + j < kPre ? cv[(c0 + j) % kPre]
                                : (acc_c ? __ldcg(C + (long long)(c0 + j) * g.ldc) : 0.0);
#pragma unroll
        for (int j = 0; j < 16; ++j)
          OZ_STORE(C + (long long)(c0 + j) * g.ldc,
                 cw[j] + (acc[c0 + j] * s_row) * pow2i(__ldg(eb + c0 + j)));
      }
      ++local;
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (kMc > 1) cluster_sync();  // no CTA leaves while its peer may still signal / fill it
  if (warp == 0)
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tmem));
}

int g_num_sms = 148;

template <int kN, int kS, int kMc>
static cudaError_t oz_attr() {
  cudaError_t e = cudaFuncSetAttribute(ozgemm_persistent_kernel<kN, kS, kMc>,
                                       cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       OzP<kN, kS>::kSmem);
  if (e != cudaSuccess || kMc == 1) return e;
  return cudaFuncSetAttribute(ozgemm_persistent_kernel<kN, kS, kMc>,
                              cudaFuncAttributeNonPortableClusterSizeAllowed, 0);
}

cudaError_t init_ozaki_attributes() {
  int dev = 0;
  if (cudaGetDevice(&dev) == cudaSuccess)
    cudaDeviceGetAttribute(&g_num_sms, cudaDevAttrMultiProcessorCount, dev);
  cudaError_t e = cudaSuccess;
  if ((e = oz_attr<64, 7, 2>()) != cudaSuccess) return e;
  if ((e = oz_attr<64, 6, 2>()) != cudaSuccess) return e;
  if ((e = oz_attr<64, 7, 1>()) != cudaSuccess) return e;
  if ((e = oz_attr<64, 6, 1>()) != cudaSuccess) return e;
  if ((e = oz_attr<32, 7, 1>()) != cudaSuccess) return e;
  if ((e = oz_attr<32, 6, 1>()) != cudaSuccess) return e;
  if ((e = oz_attr<32, 7, 4>()) != cudaSuccess) return e;
  if ((e = oz_attr<32, 6, 4>()) != cudaSuccess) return e;
#define MLE_SLICE_ATTR(RC, S, R)                                                           \
  e = cudaFuncSetAttribute(oz_slice_kernel<RC, S, R>,                                       \
                           cudaFuncAttributeMaxDynamicSharedMemorySize, oz_slice_smem(R));  \
  if (e != cudaSuccess) return e;
  MLE_SLICE_ATTR(0, 7, 16)
  MLE_SLICE_ATTR(1, 7, 16)
  MLE_SLICE_ATTR(0, 6, 16)
  MLE_SLICE_ATTR(1, 6, 16)
  MLE_SLICE_ATTR(0, 7, 4)
  MLE_SLICE_ATTR(1, 7, 4)
  MLE_SLICE_ATTR(0, 6, 4)
  MLE_SLICE_ATTR(1, 6, 4)
#undef MLE_SLICE_ATTR
  return cudaSuccess;
}

template <int kR>
static void oz_slice_launch(const OzSliceArgs& a, int rows, bool row_contig, bool six, int batch,
                            cudaStream_t s) {
  const dim3 grid((unsigned)(rows / kR), 1, (unsigned)batch);
  const int smem = oz_slice_smem(kR);
  if (row_contig && six)
    oz_slice_kernel<1, 6, kR><<<grid, 16 * kR, smem, s>>>(a);
  else if (row_contig)
    oz_slice_kernel<1, 7, kR><<<grid, 16 * kR, smem, s>>>(a);
  else if (six)
    oz_slice_kernel<0, 6, kR><<<grid, 16 * kR, smem, s>>>(a);
  else
    oz_slice_kernel<0, 7, kR><<<grid, 16 * kR, smem, s>>>(a);
}

cudaError_t launch_oz_slice(const OzSliceArgs& a, int rows, bool row_contig, int batch,
                            cudaStream_t s) {
  if (a.K > kOzSliceMaxK || a.K % OZ_KB || rows % 128) return cudaErrorInvalidValue;
  const bool six = oz_nslices(a.nslices) == 6;
  // 16-row CTAs, except row-major operands too small to give three per SM: 4-row CTAs
  // there (measured: 11.6 -> 9.8 us for the 512-row W_b slices; no gain for column-major)
  if (row_contig || (long long)(rows / 16) * batch >= 3LL * 148)
    oz_slice_launch<16>(a, rows, row_contig, six, batch, s);
  else
    oz_slice_launch<4>(a, rows, row_contig, six, batch, s);
  return cudaGetLastError();
}

template <int kN, int kS, int kMc>
static cudaError_t oz_launch(const OzGemmArgs& g, long long per_z, long long total,
                             long long grid, cudaStream_t s) {
  if (kMc == 1) {
    ozgemm_persistent_kernel<kN, kS, kMc><<<(unsigned)grid, OZP_THREADS, OzP<kN, kS>::kSmem,
                                            s>>>(g, per_z, total);
    return cudaGetLastError();
  }
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3((unsigned)grid, 1, 1);
  cfg.blockDim = dim3(OZP_THREADS, 1, 1);
  cfg.dynamicSmemBytes = OzP<kN, kS>::kSmem;
  cfg.stream = s;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = kMc;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, ozgemm_persistent_kernel<kN, kS, kMc>, g, per_z, total);
}

// n_tile: 0 -> 128 x 64 tiles in CTA pairs sharing A (default), 1 -> 128 x 32 tiles,
// 2 -> 128 x 64 tiles without pairing (A/B comparisons), 3 -> 128 x 32 tiles in clusters of
// four sharing A (double-buffered TMEM accumulators: the epilogue of one tile overlaps the
// MMAs of the next).  All give bit-identical results.
cudaError_t launch_ozgemm(const OzGemmArgs& g, int batch, cudaStream_t s, int n_tile) {
  const long long tiles =
      g.lower ? (long long)g.tiles_m * (g.tiles_m + 1) / 2 : (long long)g.tiles_m * g.tiles_n;
  if (tiles <= 0) return cudaSuccess;
  if (n_tile < 0 || n_tile > 3) return cudaErrorInvalidValue;
  const int kn = (n_tile == 1 || n_tile == 3) ? 32 : 64;
  const long long per_z = tiles * (128 / kn), total = per_z * batch;
  const long long cap = g.max_ctas > 0 ? std::min(g.max_ctas, g_num_sms) : g_num_sms;
  long long grid = std::min<long long>(total, cap);
  const bool six = oz_nslices(g.nslices) == 6;
  if (n_tile == 0) {
    grid &= ~1LL;  // whole pairs (total is even: two halves per 128-wide tile)
    if (grid < 2) grid = 2;
    return (six ? oz_launch<64, 6, 2> : oz_launch<64, 7, 2>)(g, per_z, total, grid, s);
  }
  if (n_tile == 2) return (six ? oz_launch<64, 6, 1> : oz_launch<64, 7, 1>)(g, per_z, total, grid, s);
  if (n_tile == 3) {
    grid &= ~3LL;  // whole clusters (total is a multiple of 4: four parts per 128-wide tile)
    if (grid < 4) grid = 4;
    return (six ? oz_launch<32, 6, 4> : oz_launch<32, 7, 4>)(g, per_z, total, grid, s);
  }
  return (six ? oz_launch<32, 6, 1> : oz_launch<32, 7, 1>)(g, per_z, total, grid, s);
}

}  // namespace mle
