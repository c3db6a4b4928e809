// linalg.cu — FP64 dense linear algebra for the likelihood engine on sm_100a.
//
// Replaces the LAPACK/BLAS calls of the reference (likelihood.py:75 dpotrf,
// likelihood.py:84,121,125,134-135 solve_triangular) and the Frobenius reductions of
// trace_product (likelihood.py:92-104).
//
//  * dgemm_kernel: 128x128x16 CTA tiles, 8 warps of 64x32, FP64 tensor-core MMA
//    (mma.sync.m8n8k4.f64 -> DMMA); operand stages by bulk copies (cp.async.bulk on an mbarrier
//    ring, a producer warp ahead of eight DMMA warps) or cp.async.  Used for every
//    panel product and trailing update: Cholesky (panel x Linv^T, lower SYRK), forward
//    solve X = L^-1 S (row panel, full update), lower-only right solve B = X L^-T.
//  * potrf_diag_kernel: one CTA factors a 128x128 diagonal tile in shared memory (16-wide
//    blocked right-looking) and inverts it (blocked by 16), reporting the first failing
//    pivot with LAPACK dpotrf semantics (info - 1, likelihood.py:76-77).
//  * reduce kernels: deterministic two-pass FP64 sums of log L_jj, y^T y, tr B_i,
//    <B_i, B_j>_F and y^T B_i y (the augmented entry B_i[n, n]).
#include <cuda_runtime.h>

#include <cstdlib>

#include "kernels.h"
#include "pivot_math.cuh"

namespace mle {

// Programmatic dependent launch for the Cholesky's latency-bound chain (diagonal tile ->
// panel rows -> next tile's update -> next diagonal tile): a kernel launched with
// cudaLaunchAttributeProgrammaticStreamSerialization may be scheduled once its predecessor
// signals (pdl_trigger, issued near the predecessor's end); it waits in pdl_wait until the
// predecessor has completed and its writes are visible.  Without the attribute both are
// no-ops.
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void pdl_trigger() {
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
}

static cudaError_t launch_pdl(const void* fn, dim3 grid, dim3 block, size_t smem,
                              cudaStream_t s, void** args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  return cudaLaunchKernelExC(&cfg, fn, args);
}

namespace {

constexpr int BM = 128;
constexpr int GEMM_THREADS = 256;
#ifndef MLE_DGEMM_STAGES_WIDE
#define MLE_DGEMM_STAGES_WIDE 3
#endif
#ifndef MLE_DGEMM_STAGES_NARROW
#define MLE_DGEMM_STAGES_NARROW 2
#endif
#ifndef MLE_DGEMM_BK_NARROW
#define MLE_DGEMM_BK_NARROW 32
#endif
constexpr int SA = BM + 4;   // A smem: [BK][SA], m contiguous (SA = 4 mod 16 -> conflict free)

// Per CTA-width constants.  kBN = 128: 2 x 4 warps of 64 x 32 (1 CTA / SM, used for the
// in-place panel products that need the whole 128-column panel in one CTA).  kBN = 64:
// 4 x 2 warps of 32 x 32 with <= 128 registers, so two CTAs share an SM and one CTA's
// C preload / store phases overlap the other's DMMA main loop.
template <int kBN, bool kBulk = false>
struct Tile {
  static constexpr int WM_CNT = (kBN == 128) ? 2 : 4;
  static constexpr int WN_CNT = 8 / WM_CNT;
  static constexpr int WTM = BM / WM_CNT;  // rows per warp
  static constexpr int WTN = kBN / WN_CNT; // cols per warp (32)
  static constexpr int MI = WTM / 8;       // m8 blocks per warp
  static constexpr int NI = WTN / 8;       // n8 blocks per warp
  static constexpr int SBN = kBN + 4;      // B (kBNK) smem stride
  static constexpr int MIN_BLOCKS = (kBN == 128) ? 1 : 2;
  // k-tile and pipeline depth.  Finer k-tiles with a deeper bulk-copy ring in the same
  // shared-memory budget (16 x 4 narrow, 5 wide stages) measured the same on the loglik pass
  // and slower on the kBKN sweeps, so both stagings share one shape.
  static constexpr int BK = (kBN == 128) ? 16 : (kBulk ? MLE_DGEMM_BK_NARROW : 32);
  static constexpr int STAGES = kBulk ? ((kBN == 128) ? MLE_DGEMM_STAGES_WIDE : MLE_DGEMM_STAGES_NARROW)
                                      : ((kBN == 128) ? 3 : 2);
  static constexpr int SBK = BK + 4;                    // B (kBKN) smem: [BN][SBK]
  static constexpr int A_STAGE = BK * SA;
  template <int kBL>
  static constexpr size_t smem_bytes() {
    return sizeof(double) * STAGES * (A_STAGE + (kBL == kBNK ? BK * SBN : kBN * SBK)) +
           16 * STAGES;  // + a full and an empty mbarrier per stage (bulk-copy staging)
  }
};

__device__ __forceinline__ void cp_async16(void* smem, const void* gmem) {
  const unsigned s = (unsigned)__cvta_generic_to_shared(smem);
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(s), "l"(gmem));
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::); }
template <int N>
__device__ __forceinline__ void cp_async_wait() {
  asm volatile("cp.async.wait_group %0;\n" ::"n"(N));
}

// Bulk-copy (TMA engine) staging: one warp issues whole-column cp.async.bulk copies that
// complete on a shared-memory mbarrier; no thread of the CTA computes addresses or holds the
// data in flight.  The waits are bounded (a lost completion traps instead of hanging).
__device__ __forceinline__ unsigned smem_addr(const void* p) {
  return (unsigned)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void mbar_init(unsigned long long* bar, unsigned count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_addr(bar)), "r"(count));
}
__device__ __forceinline__ void mbar_expect_tx(unsigned long long* bar, unsigned bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_addr(bar)),
               "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_wait(unsigned long long* bar, unsigned phase) {
  unsigned done = 0;
  for (unsigned it = 0; it < (1u << 28) && !done; ++it) {
    asm volatile(
        "{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; "
        "selp.u32 %0, 1, 0, p; }"
        : "=r"(done)
        : "r"(smem_addr(bar)), "r"(phase)
        : "memory");
  }
  if (!done) asm volatile("trap;");
}
__device__ __forceinline__ void bulk_g2s(void* smem, const void* gmem, unsigned bytes,
                                         unsigned long long* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
      ::"r"(smem_addr(smem)), "l"(gmem), "r"(bytes), "r"(smem_addr(bar))
      : "memory");
}

__device__ __forceinline__ void dmma_16x8x8(double (&d)[4], const double (&a)[4],
                                            const double (&b)[2]) {
  asm volatile(
      "mma.sync.aligned.m16n8k8.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5,%6,%7}, "
      "{%8,%9}, {%0,%1,%2,%3};\n"
      : "+d"(d[0]), "+d"(d[1]), "+d"(d[2]), "+d"(d[3])
      : "d"(a[0]), "d"(a[1]), "d"(a[2]), "d"(a[3]), "d"(b[0]), "d"(b[1]));
}

// 128-row tile index tm and 128-column tile index tn128 (+ 64-column half for kBN = 64).
template <int kBN>
__device__ __forceinline__ void tile_coords(const GemmArgs& g, int* tm, int* tn, int* half) {
  const int sub = (kBN == 128) ? 1 : 2;
  const int b = blockIdx.x / sub;
  *half = blockIdx.x % sub;
  if (g.lower) {
    int I = (int)((sqrtf(8.0f * (float)b + 1.0f) - 1.0f) * 0.5f);
    while (I * (I + 1) / 2 > b) --I;
    while ((I + 1) * (I + 2) / 2 <= b) ++I;
    *tm = I;
    *tn = b - I * (I + 1) / 2;
  } else {
    *tm = b % g.tiles_m;
    *tn = b / g.tiles_m;
  }
}

}  // namespace

// C[tm, tn] = alpha * sum_k A(m, k) B(n, k) + beta * C, A(m,k) = A[m + k*lda].
// kBulk: operand stages arrive by cp.async.bulk column copies (the TMA engine) on a full /
// empty mbarrier ring driven by a ninth, producer warp; otherwise by per-thread 16-byte
// cp.async with a CTA barrier per k-tile.  Same k order: the two produce identical bits.
template <int kBL, int kBN, bool kBulk>
__global__ void __launch_bounds__(kBulk ? GEMM_THREADS + 32 : GEMM_THREADS, Tile<kBN, kBulk>::MIN_BLOCKS)
    dgemm_kernel(GemmArgs g) {
  using T = Tile<kBN, kBulk>;
  constexpr int BK = T::BK, STAGES = T::STAGES, SBK = T::SBK, A_STAGE = T::A_STAGE;
  const int z = blockIdx.z;
  if (*g.fail_flag[z]) return;
  extern __shared__ __align__(16) double smem[];
  double* As = smem;
  double* Bs = smem + STAGES * A_STAGE;
  constexpr int B_STAGE = (kBL == kBNK) ? BK * T::SBN : kBN * SBK;
  unsigned long long* full_bar =
      reinterpret_cast<unsigned long long*>(smem + STAGES * (A_STAGE + B_STAGE));
  unsigned long long* empty_bar = full_bar + STAGES;

  int tm, tn, half;
  tile_coords<kBN>(g, &tm, &tn, &half);
  if (g.trap && tm + g.trap_off < tn) return;
  const long long col0 = (long long)tn * 128 + (long long)half * kBN;
  // no __restrict__: panel products run in place (C aliases A or B; see engine.cu)
  const double* A = g.A[z] + (long long)tm * BM;
  const double* Bz = g.B[z];
  const double* B = (kBL == kBNK) ? Bz + col0 : Bz + col0 * g.ldb;
  double* C = g.C[z] + (long long)tm * BM + col0 * g.ldc;
  const long long lda = g.lda, ldb = g.ldb, ldc = g.ldc;

  const int tid = threadIdx.x;
  const int warp = tid >> 5, lane = tid & 31;
  const int wm = warp % T::WM_CNT, wn = warp / T::WM_CNT;
  const int gq = lane >> 2, tq = lane & 3;

  auto load_stage = [&](int stage, int kt) {
    double* as = As + stage * A_STAGE;
    double* bs = Bs + stage * B_STAGE;
    const int k0 = kt * BK;
#pragma unroll
    for (int r = 0; r < (BM * BK / 2) / GEMM_THREADS; ++r) {
      const int c = tid + r * GEMM_THREADS;
      const int k = c >> 6, m2 = (c & 63) << 1;
      cp_async16(as + k * SA + m2, A + m2 + (long long)(k0 + k) * lda);
    }
#pragma unroll
    for (int r = 0; r < (kBN * BK / 2) / GEMM_THREADS; ++r) {
      const int c = tid + r * GEMM_THREADS;
      if (kBL == kBNK) {
        const int k = c / (kBN / 2), n2 = (c % (kBN / 2)) * 2;
        cp_async16(bs + k * T::SBN + n2, B + n2 + (long long)(k0 + k) * ldb);
      } else {
        const int nn = c / (BK / 2), k2 = (c % (BK / 2)) * 2;
        cp_async16(bs + nn * SBK + k2, B + (k0 + k2) + (long long)nn * ldb);
      }
    }
  };

  // producer warp only: one expect_tx for the stage's bytes, then one bulk copy per operand
  // column (A and kBNK B: BK columns of 128 / kBN doubles; kBKN B: kBN rows of BK doubles)
  auto load_stage_bulk = [&](int stage, int kt) {
    double* as = As + stage * A_STAGE;
    double* bs = Bs + stage * B_STAGE;
    unsigned long long* bar = full_bar + stage;
    const int k0 = kt * BK;
    if (lane == 0) mbar_expect_tx(bar, (unsigned)(sizeof(double) * (BM + kBN) * BK));
    __syncwarp();
    if (lane < BK) {
      bulk_g2s(as + lane * SA, A + (long long)(k0 + lane) * lda, BM * 8, bar);
      if (kBL == kBNK)
        bulk_g2s(bs + lane * T::SBN, B + (long long)(k0 + lane) * ldb, kBN * 8, bar);
    }
    if (kBL != kBNK) {
#pragma unroll
      for (int nn = lane; nn < kBN; nn += 32)
        bulk_g2s(bs + nn * SBK, B + k0 + (long long)nn * ldb, BK * 8, bar);
    }
  };

  const int KT = g.K / BK;
  if (kBulk) {
    // Warp 8 is the producer: it runs ahead of the eight DMMA warps through a full / empty
    // mbarrier ring, so the main loop has no CTA-wide barrier and no thread of the compute
    // warps touches an address of the operand stream.
    if (tid == 0) {
#pragma unroll
      for (int s = 0; s < STAGES; ++s) {
        mbar_init(full_bar + s, 1);
        mbar_init(empty_bar + s, GEMM_THREADS / 32);
      }
      asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    if (warp == GEMM_THREADS / 32) {
      for (int kt = 0; kt < KT; ++kt) {
        const int st = kt % STAGES, use = kt / STAGES;
        if (use >= 1) mbar_wait(empty_bar + st, (unsigned)((use - 1) & 1));
        load_stage_bulk(st, kt);
      }
      return;
    }
  } else {
#pragma unroll
    for (int s = 0; s < STAGES - 1; ++s) {
      if (s < KT) load_stage(s, s);
      cp_async_commit();
    }
  }

  // Accumulators start from C (beta = 1) so the C read overlaps the pipeline prologue and
  // the epilogue is store-only; alpha = -1 is applied by negating the A fragments.
  // m8n8k4 DMMA fragment map (f64): a0 = A(g, t), b0 = B(k = t, n = g),
  // c0 = C(g, 2t), c1 = C(g, 2t+1).
  double acc[T::MI][T::NI][2];
  if (g.beta != 0.0) {
#pragma unroll
    for (int mi = 0; mi < T::MI; ++mi)
#pragma unroll
      for (int ni = 0; ni < T::NI; ++ni) {
        const int r = wm * T::WTM + mi * 8 + gq;
        const int c = wn * T::WTN + ni * 8 + 2 * tq;
        const double* p0 = C + r + (long long)c * ldc;
        acc[mi][ni][0] = p0[0];
        acc[mi][ni][1] = p0[ldc];
      }
  } else {
#pragma unroll
    for (int mi = 0; mi < T::MI; ++mi)
#pragma unroll
      for (int ni = 0; ni < T::NI; ++ni) acc[mi][ni][0] = acc[mi][ni][1] = 0.0;
  }
  const unsigned neg = g.alpha < 0.0 ? 0x80000000u : 0u;

  for (int kt = 0; kt < KT; ++kt) {
    if (kBulk) {
      mbar_wait(full_bar + kt % STAGES, (unsigned)((kt / STAGES) & 1));
    } else {
      cp_async_wait<STAGES - 2>();
      __syncthreads();
      const int nk = kt + STAGES - 1;
      if (nk < KT) load_stage(nk % STAGES, nk);
      cp_async_commit();
    }
    const double* as = As + (kt % STAGES) * A_STAGE;
    const double* bs = Bs + (kt % STAGES) * B_STAGE;
#pragma unroll
    for (int kk = 0; kk < BK; kk += 4) {
      // k-outer ordering: MI x NI independent DMMAs per k4 step keep the tensor pipe fed
      double af[T::MI], bf[T::NI];
#pragma unroll
      for (int mi = 0; mi < T::MI; ++mi) {
        const double v = as[(kk + tq) * SA + wm * T::WTM + mi * 8 + gq];
        af[mi] = __hiloint2double(__double2hiint(v) ^ (int)neg, __double2loint(v));
      }
#pragma unroll
      for (int ni = 0; ni < T::NI; ++ni) {
        const int c0 = wn * T::WTN + ni * 8 + gq;
        bf[ni] = (kBL == kBNK) ? bs[(kk + tq) * T::SBN + c0] : bs[c0 * SBK + kk + tq];
      }
#pragma unroll
      for (int mi = 0; mi < T::MI; ++mi)
#pragma unroll
        for (int ni = 0; ni < T::NI; ++ni)
          asm volatile(
              "mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
              : "+d"(acc[mi][ni][0]), "+d"(acc[mi][ni][1])
              : "d"(af[mi]), "d"(bf[ni]));
    }
    if (kBulk) {  // this warp is done with the stage: one arrival per warp frees it
      // The stage is refilled through the async proxy: the warp's generic-proxy reads of it
      // must be ordered before that write (without this fence the refill overtook the last
      // fragment loads: wrong factors at n >= 16,384, measured).
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      __syncwarp();
      if (lane == 0)
        asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(
                         smem_addr(empty_bar + kt % STAGES))
                     : "memory");
    }
  }
  if (!kBulk) cp_async_wait<0>();

  // epilogue: store-only
#pragma unroll
  for (int mi = 0; mi < T::MI; ++mi) {
#pragma unroll
    for (int ni = 0; ni < T::NI; ++ni) {
      const int r = wm * T::WTM + mi * 8 + gq;
      const int c = wn * T::WTN + ni * 8 + 2 * tq;
      double* p0 = C + r + (long long)c * ldc;
      p0[0] = acc[mi][ni][0];
      p0[ldc] = acc[mi][ni][1];
    }
  }
}

// Operand staging of dgemm_kernel.  Default: the bulk-copy ring for kBNK products (both
// operands arrive as whole 512 B - 1 KB columns: the Cholesky's panel products and updates)
// and per-thread cp.async for kBKN products, whose B operand is 64-128 rows of only
// 128-256 B (measured: the small bulk copies cost the config-2 solve sweeps 3%).
// MLE_DGEMM_STAGE=cpasync | bulk forces one staging everywhere (A/B timing; the results are
// bit-identical either way).
static bool dgemm_bulk_staging(BLayout bl) {
  static const int mode = [] {
    const char* e = getenv("MLE_DGEMM_STAGE");
    return !e ? 0 : (e[0] == 'c' ? 1 : 2);
  }();
  return mode == 0 ? bl == kBNK : mode == 2;
}

// Opt-in shared-memory limits; must run once per device before the first launch.
cudaError_t init_kernel_attributes() {
  cudaError_t e;
#define MLE_SET_SMEM(BL, BNW, BULK)                                                        \
  e = cudaFuncSetAttribute(dgemm_kernel<BL, BNW, BULK>,                                    \
                           cudaFuncAttributeMaxDynamicSharedMemorySize,                    \
                           (int)Tile<BNW, BULK>::template smem_bytes<BL>());                     \
  if (e != cudaSuccess) return e;
  MLE_SET_SMEM(kBNK, 128, true)
  MLE_SET_SMEM(kBKN, 128, true)
  MLE_SET_SMEM(kBNK, 64, true)
  MLE_SET_SMEM(kBKN, 64, true)
  MLE_SET_SMEM(kBNK, 128, false)
  MLE_SET_SMEM(kBKN, 128, false)
  MLE_SET_SMEM(kBNK, 64, false)
  MLE_SET_SMEM(kBKN, 64, false)
#undef MLE_SET_SMEM
  return cudaSuccess;
}

template <bool kBulk>
static void launch_gemm_staged(const GemmArgs& g, BLayout bl, long long tiles, int batch,
                               cudaStream_t s) {
  const int threads = kBulk ? GEMM_THREADS + 32 : GEMM_THREADS;  // + the producer warp
  if (g.wide) {
    const dim3 grid((unsigned)tiles, 1, (unsigned)batch);
    if (bl == kBNK)
      dgemm_kernel<kBNK, 128, kBulk><<<grid, threads, Tile<128, kBulk>::template smem_bytes<kBNK>(), s>>>(g);
    else
      dgemm_kernel<kBKN, 128, kBulk><<<grid, threads, Tile<128, kBulk>::template smem_bytes<kBKN>(), s>>>(g);
  } else {
    const dim3 grid((unsigned)(2 * tiles), 1, (unsigned)batch);
    if (bl == kBNK)
      dgemm_kernel<kBNK, 64, kBulk><<<grid, threads, Tile<64, kBulk>::template smem_bytes<kBNK>(), s>>>(g);
    else
      dgemm_kernel<kBKN, 64, kBulk><<<grid, threads, Tile<64, kBulk>::template smem_bytes<kBKN>(), s>>>(g);
  }
}

// wide = 1 selects 128-column CTAs (required when C aliases A across the whole panel).
cudaError_t launch_gemm(const GemmArgs& g, BLayout bl, int batch, cudaStream_t s) {
  const long long tiles =
      g.lower ? (long long)g.tiles_m * (g.tiles_m + 1) / 2 : (long long)g.tiles_m * g.tiles_n;
  if (tiles <= 0) return cudaSuccess;
  if (dgemm_bulk_staging(bl))
    launch_gemm_staged<true>(g, bl, tiles, batch, s);
  else
    launch_gemm_staged<false>(g, bl, tiles, batch, s);
  return cudaGetLastError();
}

// ---------------------------------------------------------------------------------------
// Small-tile DMMA GEMM for the latency-critical products of the Cholesky chain (one 128 x 128
// output tile per dataset: the next diagonal tile's panel rows and its rank-128 update).  A
// 128-wide CTA does such a tile at one SM's DMMA rate (~25 us); here TM x TN CTAs (16 x 128
// for the in-place panel, whose CTAs must own whole rows; 32 x 32 for the update) spread it
// over 8-16 SMs.  K (<= 128) is staged whole in shared memory before any store, so C may
// alias A row-wise.  C(m, n) = alpha sum_k A(m, k) B(n, k) + beta C; B layout kBNK.
namespace {
constexpr int SM_K = 128;
template <int TM, int TN>
__global__ void __launch_bounds__(256) dgemm_small_kernel(GemmArgs g) {
  constexpr int SAS = TM + 4, SBS = TN + 4;  // smem strides (m / n contiguous per k)
  constexpr int TILES_M = TM / 8, TILES_N = TN / 8, PER_WARP = TILES_M * TILES_N / 8;
  static_assert(PER_WARP >= 1 && (TILES_M * TILES_N) % 8 == 0, "tile shape");
  extern __shared__ __align__(16) double sm_small[];
  double* As = sm_small;              // [K][SAS]
  double* Bs = sm_small + SM_K * SAS;  // [K][SBS]
  const int z = blockIdx.z;
  pdl_wait();
  if (__ldcv(g.fail_flag[z])) return;
  constexpr int CM = 128 / TM, CN = 128 / TN;  // CTAs per 128 x 128 tile
  const int sub = blockIdx.x % (CM * CN), tile = blockIdx.x / (CM * CN);
  const int sm_ = sub % CM, sn_ = sub / CM;
  const int tm = tile % g.tiles_m, tn = tile / g.tiles_m;
  const int r0 = tm * 128 + sm_ * TM, c0 = tn * 128 + sn_ * TN;
  if (g.trap && r0 + TM <= c0) return;  // sub-tile strictly above the diagonal
  const int K = g.K;
  const double* A = g.A[z] + r0;
  const double* B = g.B[z] + c0;
  double* C = g.C[z] + r0 + (long long)c0 * g.ldc;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  // all 16-byte copies in flight at once (cp.async), then one wait: the fill is one L2
  // round trip instead of K * (TM + TN) / 256 dependent ones
  for (int idx = tid; idx < K * (TM / 2); idx += 256) {
    const int k = idx / (TM / 2), m2 = (idx % (TM / 2)) * 2;
    cp_async16(As + k * SAS + m2, A + m2 + (long long)k * g.lda);
  }
  for (int idx = tid; idx < K * (TN / 2); idx += 256) {
    const int k = idx / (TN / 2), n2 = (idx % (TN / 2)) * 2;
    cp_async16(Bs + k * SBS + n2, B + n2 + (long long)k * g.ldb);
  }
  cp_async_commit();
  cp_async_wait<0>();
  __syncthreads();
  const int gq = lane >> 2, tq = lane & 3;
  const unsigned neg = g.alpha < 0.0 ? 0x80000000u : 0u;
  double acc[PER_WARP][2];
  int om[PER_WARP], on[PER_WARP];
#pragma unroll
  for (int q = 0; q < PER_WARP; ++q) {
    const int t = warp * PER_WARP + q;
    om[q] = (t % TILES_M) * 8;
    on[q] = (t / TILES_M) * 8;
    if (g.beta != 0.0) {
      const double* p0 = C + om[q] + gq + (long long)(on[q] + 2 * tq) * g.ldc;
      acc[q][0] = p0[0];
      acc[q][1] = p0[g.ldc];
    } else {
      acc[q][0] = acc[q][1] = 0.0;
    }
  }
  for (int kk = 0; kk < K; kk += 4) {
#pragma unroll
    for (int q = 0; q < PER_WARP; ++q) {
      const double v = As[(kk + tq) * SAS + om[q] + gq];
      const double a = __hiloint2double(__double2hiint(v) ^ (int)neg, __double2loint(v));
      const double b = Bs[(kk + tq) * SBS + on[q] + gq];
      asm volatile(
          "mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
          : "+d"(acc[q][0]), "+d"(acc[q][1])
          : "d"(a), "d"(b));
    }
  }
  pdl_trigger();  // the chain's next kernel may be scheduled during the stores
#pragma unroll
  for (int q = 0; q < PER_WARP; ++q) {
    double* p0 = C + om[q] + gq + (long long)(on[q] + 2 * tq) * g.ldc;
    p0[0] = acc[q][0];
    p0[g.ldc] = acc[q][1];
  }
}
template <int TM, int TN>
constexpr size_t small_smem() { return sizeof(double) * SM_K * ((TM + 4) + (TN + 4)); }
}  // namespace

cudaError_t init_small_gemm_attributes() {
  cudaError_t e = cudaFuncSetAttribute(dgemm_small_kernel<16, 128>,
                                       cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       (int)small_smem<16, 128>());
  if (e != cudaSuccess) return e;
  return cudaFuncSetAttribute(dgemm_small_kernel<32, 32>,
                              cudaFuncAttributeMaxDynamicSharedMemorySize,
                              (int)small_smem<32, 32>());
}

// rows_only = 1: 16 x 128 CTAs (in-place panels); 0: 32 x 32 CTAs.  K <= 128, kBNK B.
cudaError_t launch_gemm_small(const GemmArgs& g, int batch, cudaStream_t s, int rows_only) {
  const long long tiles = (long long)g.tiles_m * g.tiles_n;
  if (tiles <= 0) return cudaSuccess;
  if (g.K > SM_K || g.K % 4) return cudaErrorInvalidValue;
  GemmArgs ga = g;
  void* args[] = {&ga};
  if (rows_only) {
    const dim3 grid((unsigned)(tiles * 8), 1, (unsigned)batch);
    return launch_pdl((const void*)dgemm_small_kernel<16, 128>, grid, dim3(256),
                      small_smem<16, 128>(), s, args);
  }
  const dim3 grid((unsigned)(tiles * 16), 1, (unsigned)batch);
  return launch_pdl((const void*)dgemm_small_kernel<32, 32>, grid, dim3(256),
                    small_smem<32, 32>(), s, args);
}

// ---------------------------------------------------------------------------------------
// Diagonal tile: Cholesky + inverse of one 128x128 tile in shared memory (one CTA).
// Ls is column-major with stride DS: L(i, j) (i >= j) at Ls[j*DS + i].  The inverse
// X = L^-1 lives in the other triangle, row-major: X(i, j) (i > j) at Ls[i*DS + j], with
// its diagonal in dinv.  Only the pivot chain is scalar (16x16 blocks in one warp's
// registers) plus the 16-row panel solves; trailing updates and the inverse assembly
// (recursive doubling 16 -> 32 -> 64 -> 128) are 16x16-blocked DMMA products over smem.
namespace {
constexpr int DT = kNB;     // 128
constexpr int DS = DT + 4;  // smem stride (= 4 mod 16: conflict-free mma fragment loads)
constexpr int DB = 16;      // register block
constexpr int DTHREADS = 512;
constexpr int DWARPS = DTHREADS / 32;
// scratch of the inverse's doubling products T = L21 X11: one buffer per pair and level (four
// 16 x 16, two 32 x 32, one 64 x 64), so that a level's T can be formed as soon as its inputs
// are final, under a later pivot block; + the pivot chain's broadcast buffer (64 doubles)
constexpr int DSCR = 4 * 16 * 16 + 2 * 32 * 32 + 64 * 64 + 64;
constexpr size_t kDiagSmem = sizeof(double) * (DT * DS + DT + DSCR);

__device__ __forceinline__ double flip_sign(double x, unsigned neg) {
  return __hiloint2double(__double2hiint(x) ^ (int)neg, __double2loint(x));
}

// acc (one 16x16 output block = two n8 tiles) += sign * A(16 x K) * B(16 x K)^T, with the
// operands read through accessor functors fa(row, k), fb(col, k).
template <class FA, class FB>
__device__ __forceinline__ void mma16x16(double (&acc)[2][4], FA fa, FB fb, int K,
                                         unsigned neg) {
  const int lane = threadIdx.x & 31, g = lane >> 2, t = lane & 3;
  for (int k0 = 0; k0 < K; k0 += 8) {
    double a[4] = {fa(g, k0 + t), fa(g + 8, k0 + t), fa(g, k0 + t + 4), fa(g + 8, k0 + t + 4)};
#pragma unroll
    for (int e = 0; e < 4; ++e) a[e] = flip_sign(a[e], neg);
#pragma unroll
    for (int nt = 0; nt < 2; ++nt) {
      const double b[2] = {fb(nt * 8 + g, k0 + t), fb(nt * 8 + g, k0 + t + 4)};
      dmma_16x8x8(acc[nt], a, b);
    }
  }
}

// Lower-triangle task index -> (bi, bj), bi >= bj.
__device__ __forceinline__ void tri_index(int t, int* bi, int* bj) {
  int i = (int)((sqrtf(8.0f * (float)t + 1.0f) - 1.0f) * 0.5f);
  while (i * (i + 1) / 2 > t) --i;
  while ((i + 1) * (i + 2) / 2 <= t) ++i;
  *bi = i;
  *bj = t - i * (i + 1) / 2;
}

__device__ __forceinline__ double select_f64(int p, double a, double b) {
  double o;
  asm("{\n\t.reg .pred q;\n\tsetp.ne.s32 q, %1, 0;\n\tselp.f64 %0, %2, %3, q;\n\t}"
      : "=d"(o) : "r"(p), "d"(a), "d"(b));
  return o;
}

// One pivot step of the register-resident 16x16 Cholesky (lane r holds row r); recursion
// keeps every index of v[] a compile-time constant so the block never leaves registers.
// d is this pivot's value (already broadcast).  The next pivot only needs lane C+1's own
// update v[C+1] -= vc^2, so it is computed and broadcast first; the rest of the rank-1
// update (column values through a shared-memory broadcast, col[]) overlaps the next
// pivot's reciprocal square root.  Entries above the diagonal (s > r) are scratch: they are
// updated unconditionally (no selects) and never stored.  LAPACK dpotf2 semantics for
// failures: AJJ <= 0 or NaN stops the factorization; the first failing column is fc.
template <int C>
__device__ __forceinline__ void chol16_step(double (&v)[16], double (&rv)[16], double d, int r,
                                            long long g0, long long n_aug, int& fc,
                                            double* col) {
  if constexpr (C < 16) {
    const int aug = (g0 + C == n_aug);  // augmented index n carries y: no pivot there
    fc = (fc < 0 && !aug && !(d > 0.0)) ? C : fc;
    // LAPACK dpotf2 arithmetic, branch-free (a branch would split the unrolled chain into
    // separate basic blocks): AJJ = sqrt(AJJ), column scaled by ONE / AJJ
    const double y = pivot_rsqrt_seed(d);
    const double piv = select_f64(aug, 1.0, pivot_sqrt_from(d, y));
    const double rinv = select_f64(aug, 1.0, pivot_rcp_of_sqrt(piv, y));
    rv[C] = rinv;
    const double vc = select_f64(r == C, piv, v[C] * rinv);
    v[C] = vc;
    if constexpr (C + 1 < 16) {
      double* cb = col + (C & 1) * 32;  // double-buffered: no WAR hazard with the last step
      const int lane = threadIdx.x & 31;
      if (lane == C + 1) cb[16] = fma(-vc, vc, v[C + 1]);  // the next pivot, first
      if (lane < 16) cb[lane] = vc;
      __syncwarp();
      const double dn = cb[16];
      constexpr int s0 = (C + 1) & ~1;  // 16-byte aligned broadcast loads
#pragma unroll
      for (int s = s0; s < 16; s += 2) {
        const double2 l2 = *reinterpret_cast<const double2*>(cb + s);
        if (s >= C + 1) v[s] = fma(-vc, l2.x, v[s]);
        v[s + 1] = fma(-vc, l2.y, v[s + 1]);
      }
      chol16_step<C + 1>(v, rv, dn, r, g0, n_aug, fc, col);
    }
  }
}
}  // namespace

// Developer diagnostics (mle_diag_trace): when g_diag_trace is set, thread 0 of every
// potrf_diag_kernel CTA appends {globaltimer at entry, after the tile load, after the pivot
// blocks, after the inverse, at exit, SM id} (6 x int64) to it; g_diag_trace_n counts records.
__device__ long long* g_diag_trace = nullptr;
__device__ unsigned long long g_diag_trace_n = 0;
__device__ unsigned long long g_diag_trace_cap = 0;
__device__ __forceinline__ long long gtimer() {
  long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

#ifdef MLE_DIAG_TIMING
__device__ long long g_diag_clock[32];
#define DIAG_T(slot) \
  if (threadIdx.x == 0) g_diag_clock[slot] = clock64();
#else
#define DIAG_T(slot)
#endif

__global__ void __launch_bounds__(DTHREADS, 1) potrf_diag_kernel(DiagArgs da) {
  const int item = blockIdx.x;
  int* fail_flag = da.fail_flag[item];
  pdl_wait();
  if (*fail_flag) return;
  long long* fail_idx = da.fail_idx[item];
  double* a = da.a[item];
  double* linv = da.linv[item];
  const long long ld = da.ld, n_aug = da.n_aug[item];
  const int k0 = da.k0;
  extern __shared__ __align__(16) double dsm[];
  double* Ls = dsm;             // DT * DS
  double* dinv = Ls + DT * DS;  // DT
  double* scr = dinv + DT;      // DSCR
  __shared__ int s_fail;
  const int tid = threadIdx.x;
  const int warp = tid >> 5, lane = tid & 31;
  const int g = lane >> 2, t = lane & 3;
  double* A = a + (long long)k0 + (long long)k0 * ld;
  long long* trace = g_diag_trace;
  long long tr[5] = {0, 0, 0, 0, 0};
  if (trace && tid == 0) tr[0] = gtimer();
  for (int idx = tid; idx < DT * DT; idx += DTHREADS) {
    const int i = idx & (DT - 1), j = idx >> 7;
    Ls[j * DS + i] = A[i + (long long)j * ld];
  }
  if (tid == 0) s_fail = 0;
  __syncthreads();
  if (trace && tid == 0) tr[1] = gtimer();
  DIAG_T(0)
#define LS(i, j) Ls[(j) * DS + (i)]
#define XS(i, j) ((i) > (j) ? Ls[(i) * DS + (j)] : ((i) == (j) ? dinv[i] : 0.0))
  // ---- the inverse X = L^-1, in pieces (dinv holds the reciprocal pivots) ----
  // X lives in the other triangle of Ls.  Recursive doubling: [[X11, 0], [X21, X22]] with
  // X21 = -X22 (L21 X11), levels 16 -> 32 -> 64.  Every piece depends only on finished pivot
  // blocks, so warps 1..15 compute it under the NEXT blocks' pivot chains (warp 0), and only
  // the last block's pieces remain after the factorization (three dependent products instead
  // of the whole inverse: ~3.5 us of tail instead of ~11).  Same operands, same k order as
  // the one-shot inverse it replaces: bit-identical.
  double* colbuf = scr;                    // pivot chain broadcast (chol16_step)
  double* T16 = scr + 64;                  // [pair][16 x 16]
  double* T32 = T16 + 4 * 16 * 16;         // [pair][32 x 32]
  double* T64 = T32 + 2 * 32 * 32;         // 64 x 64
  // diagonal 16 x 16 block blk: thread c (< 16) does column c by forward substitution
  auto inv_diag = [&](int blk, int c) {
    const int o = blk * DB;
    double x[DB];
#pragma unroll
    for (int r = 0; r < DB; ++r) {
      double v = (r == c) ? 1.0 : 0.0;
#pragma unroll
      for (int m = 0; m < r; ++m) v -= LS(o + r, o + m) * x[m];
      x[r] = (r >= c) ? v * dinv[o + r] : 0.0;
    }
#pragma unroll
    for (int r = 0; r < DB; ++r)
      if (r > c) Ls[(o + r) * DS + (o + c)] = x[r];
  };
  // T = L21 X11 of the pair at offset o, level s (s x s, column-major), 16 x 16 task q
  auto inv_T = [&](double* T, int o, int sz, int q) {
    const int bps = sz / DB, bi = q % bps, bj = q / bps;
    double acc[2][4] = {};
    mma16x16(
        acc, [&](int rr, int k) { return LS(o + sz + bi * DB + rr, o + k); },
        [&](int cc, int k) { return XS(o + k, o + bj * DB + cc); }, sz, 0u);
#pragma unroll
    for (int nt = 0; nt < 2; ++nt) {
      const int cc = bj * DB + nt * 8 + 2 * t, rr = bi * DB + g;
      T[cc * sz + rr] = acc[nt][0];
      T[(cc + 1) * sz + rr] = acc[nt][1];
      T[cc * sz + rr + 8] = acc[nt][2];
      T[(cc + 1) * sz + rr + 8] = acc[nt][3];
    }
  };
  // X21 = -X22 T of the same pair, task q
  auto inv_X21 = [&](const double* T, int o, int sz, int q) {
    const int bps = sz / DB, bi = q % bps, bj = q / bps;
    double acc[2][4] = {};
    mma16x16(
        acc, [&](int rr, int k) { return XS(o + sz + bi * DB + rr, o + sz + k); },
        [&](int cc, int k) { return T[(bj * DB + cc) * sz + k]; }, sz, 0x80000000u);
#pragma unroll
    for (int nt = 0; nt < 2; ++nt) {
      const int i0 = o + sz + bi * DB + g, j1 = o + bj * DB + nt * 8 + 2 * t;
      Ls[i0 * DS + j1] = acc[nt][0];
      Ls[i0 * DS + j1 + 1] = acc[nt][1];
      Ls[(i0 + 8) * DS + j1] = acc[nt][2];
      Ls[(i0 + 8) * DS + j1 + 1] = acc[nt][3];
    }
  };
  // helper warps: the 12 warps that do not share warp 0's scheduler (warps 4, 8, 12 would
  // take issue slots from the latency-bound pivot chain)
  constexpr int HW = DWARPS - DWARPS / 4;
  const bool helper = (warp & 3) != 0;
  const int hw = warp - 1 - (warp >> 2);  // 0 .. 11 over warps 1,2,3,5,6,7,...
  auto helpers_sync = [&]() {
    __syncwarp();
    asm volatile("bar.sync 1, %0;" ::"n"(HW * 32) : "memory");
  };
#pragma unroll 1
  for (int J = 0; J < DT / DB; ++J) {
    const int j0 = J * DB;
    // (a) pivot chain of the 16x16 diagonal block in warp 0's registers
    if (warp == 0) {
      const int r = lane & (DB - 1);
      double v[DB], rv[DB];
#pragma unroll
      for (int s = 0; s < DB; ++s) v[s] = (s <= r) ? LS(j0 + r, j0 + s) : 0.0;
      int fc = -1;
      chol16_step<0>(v, rv, LS(j0, j0), r, (long long)k0 + j0, n_aug, fc, colbuf);
      if (lane < DB) {
#pragma unroll
        for (int s = 0; s < DB; ++s)
          if (s <= r) LS(j0 + r, j0 + s) = v[s];
        // reciprocal pivots (1 / L_jj as used by the factorization) for the panel rows and
        // the inverse
#pragma unroll
        for (int s = 0; s < DB; ++s)
          if (s == r) dinv[j0 + r] = rv[s];
      }
      if (fc >= 0 && lane == 0) {
        s_fail = 1;
        *fail_idx = (long long)k0 + j0 + fc;
        *fail_flag = 1;
      }
    } else if (helper && J >= 1) {
      // inverse pieces whose inputs were final before this step (prev = J - 1 is factored):
      //   stage 1: X_prev; T16 of pair (prev - 1, prev) [prev odd]; T32 of blocks 0-3 [J = 3]
      //            and 4-7 [J = 7]; T64 [J = 5]
      //   stage 2: X21 of that 16-pair [prev odd]; T16 of pair (6, 7) [J = 7, needs X_6]
      //   stage 3: X21 of the 32-pair 0-3 [J = 4]
      const int prev = J - 1;
      if (hw == HW - 1 && lane < DB) inv_diag(prev, lane);
      if (prev & 1) {
        if (hw == 0) inv_T(T16 + (prev >> 1) * 256, (prev - 1) * DB, DB, 0);
      }
      if (J == 3 || J == 7) {
        const int p = J == 3 ? 0 : 1;
        if (hw >= 1 && hw <= 4) inv_T(T32 + p * 1024, p * 64, 32, hw - 1);
      }
      if (J == 5)
        for (int q = hw; q < 16; q += HW) inv_T(T64, 0, 64, q);
      helpers_sync();
      if (prev & 1) {
        if (hw == 0) inv_X21(T16 + (prev >> 1) * 256, (prev - 1) * DB, DB, 0);
      }
      if (J == 7 && hw == 1) inv_T(T16 + 3 * 256, 6 * DB, DB, 0);
      helpers_sync();
      if (J == 4 && hw < 4) inv_X21(T32, 0, 32, hw);
    }
    __syncthreads();
    DIAG_T(1 + 3 * J)
    if (s_fail) return;
    const int rem = DT - j0 - DB;  // rows below the block
    const int base = j0 + DB;
    // (b) panel rows: x L_JJ^T = a_row, right-looking with reciprocal pivots (dtrsm order)
    if (tid < rem) {
      const int i = base + tid;
      double x[DB];
#pragma unroll
      for (int c = 0; c < DB; ++c) x[c] = LS(i, j0 + c);
#pragma unroll
      for (int c = 0; c < DB; ++c) {
        x[c] *= dinv[j0 + c];
#pragma unroll
        for (int m = c + 1; m < DB; ++m) x[m] -= x[c] * LS(j0 + m, j0 + c);
      }
#pragma unroll
      for (int c = 0; c < DB; ++c) LS(i, j0 + c) = x[c];
    }
    __syncthreads();
    DIAG_T(2 + 3 * J)
    // (c) trailing lower update A22 -= L21 L21^T on 16x16 blocks with DMMA (K = 16)
    const int nblk = rem / DB;
    for (int task = warp; task < nblk * (nblk + 1) / 2; task += DWARPS) {
      int bi, bj;
      tri_index(task, &bi, &bj);
      const int r0 = base + bi * DB, c0 = base + bj * DB;
      double acc[2][4];
#pragma unroll
      for (int nt = 0; nt < 2; ++nt) {
        acc[nt][0] = LS(r0 + g, c0 + nt * 8 + 2 * t);
        acc[nt][1] = LS(r0 + g, c0 + nt * 8 + 2 * t + 1);
        acc[nt][2] = LS(r0 + g + 8, c0 + nt * 8 + 2 * t);
        acc[nt][3] = LS(r0 + g + 8, c0 + nt * 8 + 2 * t + 1);
      }
      mma16x16(
          acc, [&](int rr, int k) { return LS(r0 + rr, j0 + k); },
          [&](int cc, int k) { return LS(c0 + cc, j0 + k); }, DB, 0x80000000u);
#pragma unroll
      for (int nt = 0; nt < 2; ++nt) {
        LS(r0 + g, c0 + nt * 8 + 2 * t) = acc[nt][0];
        LS(r0 + g, c0 + nt * 8 + 2 * t + 1) = acc[nt][1];
        LS(r0 + g + 8, c0 + nt * 8 + 2 * t) = acc[nt][2];
        LS(r0 + g + 8, c0 + nt * 8 + 2 * t + 1) = acc[nt][3];
      }
    }
    __syncthreads();
    DIAG_T(3 + 3 * J)
  }

  if (trace && tid == 0) tr[2] = gtimer();
  // ---- what is left of the inverse: the last block's pieces, three dependent products ----
  if (tid < DB) inv_diag(DT / DB - 1, tid);
  __syncthreads();
  DIAG_T(25)
  if (warp == 0) inv_X21(T16 + 3 * 256, 6 * DB, DB, 0);
  __syncthreads();
  if (warp < 4) inv_X21(T32 + 1024, 64, 32, warp);
  __syncthreads();
  inv_X21(T64, 0, 64, warp);  // 16 tasks, one per warp
  __syncthreads();
  DIAG_T(26)
  if (trace && tid == 0) tr[3] = gtimer();
  pdl_trigger();  // the chain's next kernel may be scheduled during the write-back
  // write back L (lower incl. diagonal) and Linv (dense 128x128, zero upper)
  for (int idx = tid; idx < DT * DT; idx += DTHREADS) {
    const int i = idx & (DT - 1), j = idx >> 7;
    if (i >= j) A[i + (long long)j * ld] = LS(i, j);
    linv[idx] = XS(i, j);
  }
  if (trace && tid == 0) {
    tr[4] = gtimer();
    const unsigned long long slot = atomicAdd(&g_diag_trace_n, 1ull);
    if (slot < g_diag_trace_cap) {
      unsigned sm;
      asm volatile("mov.u32 %0, %%smid;" : "=r"(sm));
      long long* o = trace + 6 * slot;
      for (int q = 0; q < 5; ++q) o[q] = tr[q];
      o[5] = (long long)sm * 1000 + k0 / 128;  // SM id, tile index
    }
  }
#undef XS
#undef LS
}

// Diagnostics: start (buf != null, cap records) or stop (buf == null) the per-CTA trace of
// potrf_diag_kernel; returns the number of records written since the last start in *count.
cudaError_t diag_trace_control(long long* buf, unsigned long long cap, unsigned long long* count) {
  cudaError_t e = cudaDeviceSynchronize();
  if (e != cudaSuccess) return e;
  if (count) {
    e = cudaMemcpyFromSymbol(count, g_diag_trace_n, sizeof(*count));
    if (e != cudaSuccess) return e;
  }
  const unsigned long long zero = 0;
  if ((e = cudaMemcpyToSymbol(g_diag_trace_n, &zero, sizeof(zero))) != cudaSuccess) return e;
  if ((e = cudaMemcpyToSymbol(g_diag_trace_cap, &cap, sizeof(cap))) != cudaSuccess) return e;
  return cudaMemcpyToSymbol(g_diag_trace, &buf, sizeof(buf));
}

cudaError_t init_diag_attributes() {
  return cudaFuncSetAttribute(potrf_diag_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                              (int)kDiagSmem);
}

cudaError_t launch_potrf_diag(const DiagArgs& d, int items, cudaStream_t s) {
  DiagArgs da = d;
  void* args[] = {&da};
  return launch_pdl((const void*)potrf_diag_kernel, dim3(items), dim3(DTHREADS), kDiagSmem, s,
                    args);
}

// ---------------------------------------------------------------------------------------
// Reductions.  Partials: per block 7 sums [logdet, quad, trA, trN, <A,A>, <A,N>, <N,N>];
// blockIdx.y = item.  Fixed grid and fixed summation order -> deterministic results, and the
// loglik-only path (Ba == null) sums log-det / y^T y in exactly the eval_all order.
namespace {
constexpr int RTHREADS = 256;
constexpr int RBLOCKS = kReduceBlocks;
constexpr int RN = kReduceSums;
constexpr int RP = kReducePartials;

__device__ __forceinline__ double block_sum(double v, double* sh) {
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  __syncthreads();
  if (lane == 0) sh[warp] = v;
  __syncthreads();
  double r = 0.0;
  if (threadIdx.x == 0)
    for (int w = 0; w < (int)(blockDim.x >> 5); ++w) r += sh[w];
  return r;
}
}  // namespace

template <int kSums>  // 7 (no nugget item) or RN = 11
__global__ void __launch_bounds__(RTHREADS) reduce_kernel(ReduceArgs ra) {
  const int item = blockIdx.y;
  if (*ra.fail_flag[item]) return;
  const double* __restrict__ L = ra.L[item];
  const double* __restrict__ Ba = ra.Ba[item];
  const double* __restrict__ Bn = ra.Bn[item];
  const double* __restrict__ Bm = kSums > 7 ? ra.Bm[item] : nullptr;
  const long long ld = ra.ld;
  const int n = ra.n;
  __shared__ double sh[RTHREADS / 32];
  double s[RN];
#pragma unroll
  for (int q = 0; q < RN; ++q) s[q] = 0.0;
  double dmin = INFINITY, dmax = 0.0;
  // One warp per column (column j on warp (j mod W) of block (j / W) mod grid, W = warps per
  // block): the diagonal terms on lane 0, the strictly lower rows coalesced across the lanes,
  // four rows' loads in flight per lane.  A fixed mapping, so the sums are deterministic and
  // the loglik-only path (Ba == null) sums log-det / y^T y exactly as eval_all does.
  const int warps = RTHREADS / 32, warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  for (int j = blockIdx.x * warps + warp; j < n; j += gridDim.x * warps) {
    const long long cj = (long long)j * ld;
    if (lane == 0) {
      s[0] += log(L[j + cj]);
      dmin = fmin(dmin, L[j + cj]);
      dmax = fmax(dmax, L[j + cj]);
      const double y = L[n + cj];
      s[1] += y * y;
      if (Ba != nullptr) {
        const double a = Ba[j + cj], b = Bn[j + cj];
        s[2] += a;
        s[3] += b;
        s[4] += a * a;
        s[5] += a * b;
        s[6] += b * b;
        if (Bm != nullptr) {
          const double c = Bm[j + cj];
          s[7] += c;
          s[8] += a * c;
          s[9] += b * c;
          s[10] += c * c;
        }
      }
    }
    if (Ba == nullptr) continue;
    int i = j + 1 + lane;
    if (Bm == nullptr) {
      for (; i + 96 < n; i += 128) {
        double a[4], b[4];
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          a[q] = Ba[i + 32 * q + cj];
          b[q] = Bn[i + 32 * q + cj];
        }
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          s[4] += 2.0 * a[q] * a[q];
          s[5] += 2.0 * a[q] * b[q];
          s[6] += 2.0 * b[q] * b[q];
        }
      }
      for (; i < n; i += 32) {
        const double a = Ba[i + cj], b = Bn[i + cj];
        s[4] += 2.0 * a * a;
        s[5] += 2.0 * a * b;
        s[6] += 2.0 * b * b;
      }
    } else {
      for (; i < n; i += 32) {
        const double a = Ba[i + cj], b = Bn[i + cj], c = Bm[i + cj];
        s[4] += 2.0 * a * a;
        s[5] += 2.0 * a * b;
        s[6] += 2.0 * b * b;
        s[8] += 2.0 * a * c;
        s[9] += 2.0 * b * c;
        s[10] += 2.0 * c * c;
      }
    }
  }
  double* partials = ra.partials[item];
  // (loglik-only items, Ba == null, have only log-det and y^T y: a block-uniform skip)
  const int live = Ba == nullptr ? 2 : kSums;
  for (int q = 0; q < RN; ++q) {
    const double t = q < live ? block_sum(s[q], sh) : 0.0;
    if (threadIdx.x == 0) partials[blockIdx.x * RP + q] = t;
  }
  if (threadIdx.x == 0) {
    partials[blockIdx.x * RP + RN] = dmin;
    partials[blockIdx.x * RP + RN + 1] = dmax;
  }
}

// out[0..RN) = fixed-order sums of the partials; out[RN..RN+3) = B_alpha, B_nu, M at [n,n];
// out[RN+3], out[RN+4] = min / max of diag(L).  One warp per output (RN + 2 warps): lane l
// folds partials l, l + 32, ... in order, then a fixed xor tree: deterministic, and ~50x
// shorter than one thread walking all RBLOCKS partials (a dependent chain of L2 round trips
// at the tail of every pass).
constexpr int kFinalWarps = RN + 2;
__global__ void __launch_bounds__(32 * kFinalWarps) reduce_final_kernel(ReduceArgs ra) {
  const int item = blockIdx.x;
  if (*ra.fail_flag[item]) return;
  const double* partials = ra.partials[item];
  double* out = ra.out[item];
  const int q = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (q < RN) {
    double v = 0.0;
    for (int b = lane; b < RBLOCKS; b += 32) v += partials[b * RP + q];
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    if (lane == 0) out[q] = v;
  } else if (q == RN) {
    double v = INFINITY;
    for (int b = lane; b < RBLOCKS; b += 32) v = fmin(v, partials[b * RP + RN]);
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v = fmin(v, __shfl_xor_sync(0xffffffffu, v, o));
    if (lane == 0) out[RN + 3] = v;
  } else {
    double v = 0.0;
    for (int b = lane; b < RBLOCKS; b += 32) v = fmax(v, partials[b * RP + RN + 1]);
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v = fmax(v, __shfl_xor_sync(0xffffffffu, v, o));
    if (lane == 0) {
      out[RN + 4] = v;
      const long long diag_n = ra.n + (long long)ra.n * ra.ld;
      out[RN] = ra.Ba[item] ? ra.Ba[item][diag_n] : 0.0;
      out[RN + 1] = ra.Bn[item] ? ra.Bn[item][diag_n] : 0.0;
      out[RN + 2] = ra.Bm[item] ? ra.Bm[item][diag_n] : 0.0;
    }
  }
}

// ---------------------------------------------------------------------------------------
// Sequential-derivative mode (contexts whose derivative blocks do not fit beside the factor:
// config 5 on one B200).  The blocks B_i = L^-1 S_i L^-T are reduced one at a time in a single
// work matrix; a finished block is parked, column by column, in the unused upper triangle of
// a resident N x (N + 513) array:
//     B(r, c), r >= c   ->   park[(r - c) + (N - c + 512) ld]
// i.e. the lower part of column c (contiguous) becomes the top of column N - c + 512
// (contiguous): rows 0 .. N - c - 1 of that column lie above the 512-wide diagonal band the
// factorization and the two-sided reduction use, so nothing else touches them.
__device__ __forceinline__ const double* parked_column(const double* park, long long ld,
                                                       long long N, long long c) {
  return park + (N - c + 512) * ld - c;  // + r addresses B(r, c)
}

__global__ void __launch_bounds__(256) park_lower_kernel(const double* __restrict__ src,
                                                         double* __restrict__ park, long long ld,
                                                         int N) {
  const long long c = blockIdx.x;
  const double* in = src + c * ld;
  double* out = park + ((long long)N - c + 512) * ld - c;
  for (long long r = c + threadIdx.x; r < N; r += 256) out[r] = in[r];
}

cudaError_t launch_park_lower(const double* src, double* park, long long ld, int N,
                              cudaStream_t s) {
  park_lower_kernel<<<(unsigned)N, 256, 0, s>>>(src, park, ld, N);
  return cudaGetLastError();
}

// S = I_n on the lower triangle and the 512-wide diagonal band of the padded matrix only (the
// full-matrix set_identity would wipe a block parked above the band).
__global__ void __launch_bounds__(256) set_identity_lower_kernel(double* S, long long ld, int n,
                                                                 int N) {
  const long long j = blockIdx.x;
  double* col = S + j * ld;
  for (long long i = (j / 512) * 512 + threadIdx.x; i < N; i += 256)
    col[i] = (i == j && i < n) ? 1.0 : 0.0;
}

cudaError_t launch_set_identity_lower(double* S, long long ld, int n, int N, cudaStream_t s) {
  set_identity_lower_kernel<<<(unsigned)N, 256, 0, s>>>(S, ld, n, N);
  return cudaGetLastError();
}

// Sums of one finished block W (lower, in the work matrix) against up to two parked blocks:
// partials per CTA [tr W, <W,W>, <W,U1>, <W,U2>] (Frobenius products of the symmetric
// matrices over [0, n)^2 from their lower triangles); one warp per column, fixed mapping and
// order -> deterministic.  out[0..4) = the sums, out[4] = W[n, n] (= y^T W y).
constexpr int SEQ_SUMS = 4;
__global__ void __launch_bounds__(RTHREADS) seq_reduce_kernel(const double* __restrict__ W,
                                                              const double* __restrict__ U1,
                                                              const double* __restrict__ U2,
                                                              long long ld, int n, int N,
                                                              double* partials) {
  __shared__ double sh[RTHREADS / 32];
  double s[SEQ_SUMS] = {0.0, 0.0, 0.0, 0.0};
  const int warps = RTHREADS / 32, warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  for (int j = blockIdx.x * warps + warp; j < n; j += gridDim.x * warps) {
    const double* w = W + (long long)j * ld;
    const double* u1 = U1 ? parked_column(U1, ld, N, j) : nullptr;
    const double* u2 = U2 ? parked_column(U2, ld, N, j) : nullptr;
    if (lane == 0) {
      const double a = w[j];
      s[0] += a;
      s[1] += a * a;
      if (u1) s[2] += a * u1[j];
      if (u2) s[3] += a * u2[j];
    }
    for (int i = j + 1 + lane; i < n; i += 32) {
      const double a = w[i];
      s[1] += 2.0 * a * a;
      if (u1) s[2] += 2.0 * a * u1[i];
      if (u2) s[3] += 2.0 * a * u2[i];
    }
  }
  for (int q = 0; q < SEQ_SUMS; ++q) {
    const double t = block_sum(s[q], sh);
    if (threadIdx.x == 0) partials[blockIdx.x * SEQ_SUMS + q] = t;
  }
}

__global__ void __launch_bounds__(32 * SEQ_SUMS) seq_reduce_final_kernel(const double* partials,
                                                                         const double* W,
                                                                         long long ld, int n,
                                                                         double* out) {
  const int q = threadIdx.x >> 5, lane = threadIdx.x & 31;
  double v = 0.0;
  for (int b = lane; b < RBLOCKS; b += 32) v += partials[b * SEQ_SUMS + q];
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  if (lane == 0) out[q] = v;
  if (threadIdx.x == 0) out[SEQ_SUMS] = W[n + (long long)n * ld];
}

// partials: >= kReduceBlocks * 4 doubles; out: 5 doubles (device).
cudaError_t launch_seq_reduce(const double* W, const double* U1, const double* U2, long long ld,
                              int n, int N, double* partials, double* out, cudaStream_t s) {
  seq_reduce_kernel<<<RBLOCKS, RTHREADS, 0, s>>>(W, U1, U2, ld, n, N, partials);
  seq_reduce_final_kernel<<<1, 32 * SEQ_SUMS, 0, s>>>(partials, W, ld, n, out);
  return cudaGetLastError();
}

cudaError_t launch_reduce(const ReduceArgs& r, int items, cudaStream_t s) {
  bool any_m = false;
  for (int i = 0; i < items; ++i) any_m = any_m || r.Bm[i] != nullptr;
  if (any_m)
    reduce_kernel<RN><<<dim3(RBLOCKS, items), RTHREADS, 0, s>>>(r);
  else
    reduce_kernel<7><<<dim3(RBLOCKS, items), RTHREADS, 0, s>>>(r);
  reduce_final_kernel<<<items, 32 * kFinalWarps, 0, s>>>(r);
  return cudaGetLastError();
}

}  // namespace mle

namespace mle {

// z = L[0:n, 0:n] w for a resident Cholesky factor (column-major, lower): the GPU half of
// the reference's simulate_grf (simulate.py:104-106, `lower @ normals`).  Thread per row;
// for every column the warp reads consecutive rows (coalesced).
__global__ void trmv_lower_kernel(const double* __restrict__ L, long long ld, int n,
                                  const double* __restrict__ w, double* __restrict__ z) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  double acc = 0.0;
  for (int j = 0; j <= i; ++j) acc = fma(L[i + (long long)j * ld], w[j], acc);
  z[i] = acc;
}

cudaError_t launch_trmv_lower(const double* L, long long ld, int n, const double* w, double* z,
                              cudaStream_t s) {
  trmv_lower_kernel<<<(n + 255) / 256, 256, 0, s>>>(L, ld, n, w, z);
  return cudaGetLastError();
}

struct LinvDinvArgs {
  double* dinv[kMaxItems];
  const double* linv[kMaxItems];
};

__global__ void __launch_bounds__(256) linv_to_dinv_kernel(LinvDinvArgs a) {
  const int k = blockIdx.x, z = blockIdx.y;
  const double* src = a.linv[z] + (size_t)k * kNB * kNB;
  double* dst = a.dinv[z] + (size_t)(k / 4) * 512 * 512 + (size_t)(k % 4) * kNB * (1 + 512);
  for (int e = threadIdx.x; e < kNB * kNB; e += 256) {
    const int r = e & (kNB - 1), c = e / kNB;
    dst[r + (size_t)c * 512] = src[e];
  }
}

cudaError_t launch_linv_to_dinv(double* const* dinv, const double* const* linv, int Nt,
                                int items, cudaStream_t s) {
  LinvDinvArgs a;
  for (int z = 0; z < items; ++z) {
    a.dinv[z] = dinv[z];
    a.linv[z] = linv[z];
  }
  linv_to_dinv_kernel<<<dim3((unsigned)Nt, (unsigned)items), 256, 0, s>>>(a);
  return cudaGetLastError();
}

struct IdentityArgs {
  double* S[kMaxItems];
};

__global__ void __launch_bounds__(256) set_identity_kernel(IdentityArgs a, long long ld, int n) {
  double* S = a.S[blockIdx.y];
  const long long total = ld * ld;
  for (long long e = (long long)blockIdx.x * 256 + threadIdx.x; e < total;
       e += (long long)gridDim.x * 256) {
    const long long i = e % ld, j = e / ld;
    S[e] = (i == j && i < n) ? 1.0 : 0.0;
  }
}

cudaError_t launch_set_identity(double* const* S, long long ld, int n, int items,
                                cudaStream_t s) {
  IdentityArgs a;
  for (int z = 0; z < items; ++z) a.S[z] = S[z];
  set_identity_kernel<<<dim3(148 * 8, (unsigned)items), 256, 0, s>>>(a, ld, n);
  return cudaGetLastError();
}

__global__ void __launch_bounds__(256) scatter_theta_kernel(PassIo io,
                                                            const ThetaParams* staged) {
  const int b = blockIdx.x;
  const unsigned long long* src = reinterpret_cast<const unsigned long long*>(staged + b);
  unsigned long long* dst = reinterpret_cast<unsigned long long*>(io.theta[b]);
  constexpr int words = (int)(sizeof(ThetaParams) / 8);
  static_assert(sizeof(ThetaParams) % 8 == 0, "ThetaParams is copied in 8-byte words");
  for (int w = threadIdx.x; w < words; w += blockDim.x) dst[w] = src[w];
  if (threadIdx.x == 0) *io.flag[b] = 0;
}

__global__ void gather_results_kernel(PassIo io, double* dst) {
  const int b = blockIdx.x, q = threadIdx.x;
  double* d = dst + (size_t)b * (kReduceOut + 2);
  if (q < kReduceOut) d[q] = io.out[b][q];
  if (q == kReduceOut) {
    int f = *io.flag[b];
    long long bits = 0;
    memcpy(&bits, &f, sizeof(int));
    reinterpret_cast<long long*>(d)[kReduceOut] = bits;
  }
  if (q == kReduceOut + 1) reinterpret_cast<long long*>(d)[kReduceOut + 1] = *io.idx[b];
}

cudaError_t launch_scatter_theta(const PassIo& io, const ThetaParams* staged, int items,
                                 cudaStream_t s) {
  scatter_theta_kernel<<<items, 256, 0, s>>>(io, staged);
  return cudaGetLastError();
}

cudaError_t launch_gather_results(const PassIo& io, double* dst, int items, cudaStream_t s) {
  gather_results_kernel<<<items, 32, 0, s>>>(io, dst);
  return cudaGetLastError();
}

// ---- distributed engine (column panels) -----------------------------------------------
__global__ void __launch_bounds__(256) linv_to_dinv_range_kernel(LinvDinvArgs a, int k_begin) {
  const int k = k_begin + blockIdx.x, z = blockIdx.y;
  const double* src = a.linv[z] + (size_t)k * kNB * kNB;
  double* dst = a.dinv[z] + (size_t)(k % 4) * kNB * (1 + 512);
  for (int e = threadIdx.x; e < kNB * kNB; e += 256) {
    const int r = e & (kNB - 1), c = e / kNB;
    dst[r + (size_t)c * 512] = src[e];
  }
}

cudaError_t launch_linv_to_dinv_block(double* const* dinv, const double* const* linv,
                                      int k_begin, int tiles, int items, cudaStream_t s) {
  LinvDinvArgs a;
  for (int z = 0; z < items; ++z) {
    a.dinv[z] = dinv[z];
    a.linv[z] = linv[z];
  }
  linv_to_dinv_range_kernel<<<dim3((unsigned)tiles, (unsigned)items), 256, 0, s>>>(a, k_begin);
  return cudaGetLastError();
}

// Upper triangle of one size x size block from its lower triangle (a[i + j ld] = a[j + i ld]
// for i < j), batched: 32 x 32 sub-tiles through shared memory (coalesced on both sides).
struct MirrorArgs {
  double* a[kMaxGemm];
};

__global__ void __launch_bounds__(256) mirror_lower_kernel(MirrorArgs m, long long ld, int size) {
  __shared__ double t[32][33];
  const int tiles = size / 32;
  const int bi = blockIdx.x % tiles, bj = blockIdx.x / tiles;  // source tile (bi >= bj)
  if (bi < bj) return;
  double* a = m.a[blockIdx.y];
  const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5;
  for (int r = ty; r < 32; r += 8)  // element (32 bi + tx, 32 bj + r)
    t[r][tx] = a[(32LL * bi + tx) + (32LL * bj + r) * ld];
  __syncthreads();
  for (int r = ty; r < 32; r += 8) {  // destination (32 bj + tx, 32 bi + r) = source (bi.., bj..)
    const int i = 32 * bj + tx, j = 32 * bi + r;
    if (i < j) a[i + (long long)j * ld] = t[tx][r];
  }
}

cudaError_t launch_mirror_lower(double* const* a, int items, long long ld, int size,
                                cudaStream_t s) {
  if (size % 32 || items > kMaxGemm) return cudaErrorInvalidValue;
  MirrorArgs m;
  for (int z = 0; z < items; ++z) m.a[z] = a[z];
  const int tiles = size / 32;
  mirror_lower_kernel<<<dim3((unsigned)(tiles * tiles), (unsigned)items), 256, 0, s>>>(m, ld,
                                                                                    size);
  return cudaGetLastError();
}

__global__ void __launch_bounds__(256) panel_identity_kernel(PanelArgs a) {
  double* S = a.p[blockIdx.y];
  const long long c0 = a.c0[blockIdx.y];
  const long long total = a.ld * a.width;
  for (long long e = (long long)blockIdx.x * 256 + threadIdx.x; e < total;
       e += (long long)gridDim.x * 256) {
    const long long i = e % a.ld, jl = e / a.ld;
    S[e] = (i == c0 + jl && i < a.n) ? 1.0 : 0.0;
  }
}

cudaError_t launch_panel_identity(const PanelArgs& a, int items, cudaStream_t s) {
  panel_identity_kernel<<<dim3(148 * 2, (unsigned)items), 256, 0, s>>>(a);
  return cudaGetLastError();
}

// One CTA per (panel column, panel): the same sums as reduce_kernel restricted to column j,
// written to partials[z][jl][0..RN) plus the three B[n, n] slots; the host adds them in a
// fixed order.
__global__ void __launch_bounds__(RTHREADS) panel_reduce_kernel(PanelReduceArgs ra) {
  const int z = blockIdx.y, jl = blockIdx.x;
  const long long j = ra.c0[z] + jl, ld = ra.ld;
  const int n = ra.n;
  const double* L = ra.L[z];
  const double* Ba = ra.Ba[z];
  const double* Bn = ra.Bn[z];
  const double* Bm = ra.Bm[z];
  double* out = ra.partials[z] + (size_t)jl * kPanelSums;
  __shared__ double sh[RTHREADS / 32];
  double s[RN];
#pragma unroll
  for (int q = 0; q < RN; ++q) s[q] = 0.0;
  const long long cj = (long long)jl * ld;
  if (j < n) {
    if (threadIdx.x == 0) {
      s[0] = log(L[j + cj]);
      const double y = L[n + cj];
      s[1] = y * y;
      if (Ba != nullptr) {
        const double a = Ba[j + cj], b = Bn[j + cj];
        s[2] = a;
        s[3] = b;
        s[4] = a * a;
        s[5] = a * b;
        s[6] = b * b;
        if (Bm != nullptr) {
          const double c = Bm[j + cj];
          s[7] = c;
          s[8] = a * c;
          s[9] = b * c;
          s[10] = c * c;
        }
      }
    }
    if (Ba != nullptr) {
      for (long long i = j + 1 + threadIdx.x; i < n; i += RTHREADS) {
        const double a = Ba[i + cj], b = Bn[i + cj];
        s[4] += 2.0 * a * a;
        s[5] += 2.0 * a * b;
        s[6] += 2.0 * b * b;
        if (Bm != nullptr) {
          const double c = Bm[i + cj];
          s[8] += 2.0 * a * c;
          s[9] += 2.0 * b * c;
          s[10] += 2.0 * c * c;
        }
      }
    }
  }
  for (int q = 0; q < RN; ++q) {
    const double t = block_sum(s[q], sh);
    if (threadIdx.x == 0) out[q] = t;
  }
  if (threadIdx.x == 0) {
    const bool has_n = (j == n);
    out[RN] = (has_n && Ba) ? Ba[n + cj] : 0.0;
    out[RN + 1] = (has_n && Bn) ? Bn[n + cj] : 0.0;
    out[RN + 2] = (has_n && Bm) ? Bm[n + cj] : 0.0;
  }
}

cudaError_t launch_panel_reduce(const PanelReduceArgs& r, int width, int items, cudaStream_t s) {
  panel_reduce_kernel<<<dim3((unsigned)width, (unsigned)items), RTHREADS, 0, s>>>(r);
  return cudaGetLastError();
}

}  // namespace mle
