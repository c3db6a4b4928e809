// gen.cu — covariance / derivative tile generation (sm_100a).
//
// Replaces build_cov_matrix / build_dcov_matrix (reference matern.py:171-203) and the
// per-distance evaluators _cov_positive / _dalpha_positive / _dnu_positive
// (matern.py:100-125).  Distances are recomputed per element (no pdist + np.unique dedup,
// matern.py:86-97) with the same rounding as scipy's pdist: sqrt((dx*dx) + (dy*dy)).
//
// One CTA owns one 32x32 lower tile (I >= J) of one item's padded, column-major N x N
// matrices (blockIdx.y = item).  It writes tile (I, J) of every requested output with
// coalesced column stores and, for the derivative matrices that are stored in full, the
// mirrored tile (J, I) through a shared-memory transpose.  The item's per-theta scalars
// (ThetaParams, ~1.1 KB) are staged into shared memory once per CTA.
//
// Engine layout: index n is the augmented row carrying z (Sigma[n, j] = z_j,
// Sigma[n, n] = 0), indices > n are padding (identity in Sigma, zero in the derivatives).
#include <cuda_runtime.h>

#include <cstdlib>
#include <type_traits>

#include "pivot_math.cuh"
#include "special.cuh"
#include "kernels.h"

namespace mle {

namespace {

constexpr int kGT = 32;         // generation tile edge
constexpr int kGThreads = 256;  // 8 columns per pass, 4 passes
constexpr int kGenSlots = 24;   // table intervals a tile stages in shared memory (3 binades)
#ifndef MLE_GEN_MINB
#define MLE_GEN_MINB 5
#endif

// b = I (I + 1) / 2 + J, 0 <= J <= I, for a block index b < 2^31 (a grid's x extent): a
// float estimate of I (approximate sqrt, error << 1 for b < 2^24 and a few units at most
// beyond) corrected exactly in integers (the products in 64 bits: (I + 1)(I + 2) passes 2^32
// at the very top of that range).
// The double-precision sqrt with 64-bit corrections this replaces was ~60 instructions of
// every CTA's prologue.
__device__ __forceinline__ void lower_tile_index(unsigned b, int* ti, int* tj) {
  float r;
  asm("sqrt.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(fmaf(8.0f, (float)b, 1.0f)));
  unsigned I = (unsigned)fmaxf((r - 1.0f) * 0.5f, 0.0f);
  while ((unsigned long long)I * (I + 1) / 2 > b) --I;
  while ((unsigned long long)(I + 1) * (I + 2) / 2 <= b) ++I;
  *ti = (int)I;
  *tj = (int)(b - (unsigned)((unsigned long long)I * (I + 1) / 2));
}

// Slot of element (row, col) in a 32 x 32 shared-memory value tile.  The column is XOR-swizzled
// by the row so that all three access patterns of the generation kernel are free of bank
// conflicts on 8-byte words: the 4 x 8 patch writes of a warp (rows R..R+3, R % 4 == 0;
// the 33-double padded rows made these 4-way conflicts), the column reads (32 consecutive
// rows, one column) and the transposed reads of the mirrored tile (one row, 32 columns).
__device__ __forceinline__ int tile_slot(int row, int col) {
  return row * kGT + (col ^ (((row & 3) << 2) | ((row >> 2) & 3)));
}

// A 16-byte coefficient pair from shared memory; MLE_GEN_LDS64 (A/B) splits it into two
// 8-byte loads.
__device__ __forceinline__ double2 lds_pair(const double* p) {
#ifdef MLE_GEN_LDS64
  const unsigned a = (unsigned)__cvta_generic_to_shared(p);
  double2 c;
  asm volatile("ld.shared.f64 %0, [%1];" : "=d"(c.x) : "r"(a));
  asm volatile("ld.shared.f64 %0, [%1+8];" : "=d"(c.y) : "r"(a));
  return c;
#else
  return *reinterpret_cast<const double2*>(p);
#endif
}

// pdist-identical Euclidean distance (no FMA contraction).
__device__ __forceinline__ double pair_distance(const double* lx, const double* ly, int i, int j) {
  const double dx = __dsub_rn(lx[i], lx[j]);
  const double dy = __dsub_rn(ly[i], ly[j]);
  return __dsqrt_rn(__dadd_rn(__dmul_rn(dx, dx), __dmul_rn(dy, dy)));
}

// Stage one ThetaParams (~7 KB) from global memory into shared memory (all threads
// participate; 16-byte words, then the 4-byte tail).
__device__ __forceinline__ void stage_params(ThetaParams* dst, const ThetaParams* src) {
  constexpr int kVec = (int)(sizeof(ThetaParams) / sizeof(int4));
  constexpr int kWords = (int)(sizeof(ThetaParams) / sizeof(int));
  const int4* s4 = reinterpret_cast<const int4*>(src);
  int4* d4 = reinterpret_cast<int4*>(dst);
  for (int w = threadIdx.x; w < kVec; w += blockDim.x) d4[w] = __ldg(s4 + w);
  const int* s = reinterpret_cast<const int*>(src);
  int* d = reinterpret_cast<int*>(dst);
  for (int w = 4 * kVec + threadIdx.x; w < kWords; w += blockDim.x) d[w] = s[w];
  __syncthreads();
}

}  // namespace

// The exact evaluator: inlined everywhere (0), out of line everywhere (1), or out of line in
// the derivative kernel's fast path only (2, default).  Out of line, the fast path's register
// allocation no longer carries the Bessel ladder.  At 48 registers (five CTAs per SM) that
// pays for the derivative kernel (config 4: 1,793 -> 1,845 GB/s; config-2 batch 1,032 ->
// 1,042) and costs the Sigma kernel 5%, hence the split; at 64 registers it measured slower
// everywhere (config-2 batch: 886 / 918 / 892 GB/s at 4 / 5 / 6 CTAs per SM against 920).
#ifndef MLE_GEN_EXACT_NOINLINE
#define MLE_GEN_EXACT_NOINLINE 2
#endif
template <bool kD>
#if MLE_GEN_EXACT_NOINLINE == 1
__device__ __noinline__
#else
__device__ __forceinline__
#endif
MaternVals matern_u_call(const ThetaParams& P, double u) {
  return matern_u<kD>(P, u);
}
#if MLE_GEN_EXACT_NOINLINE == 2  // A/B: out of line in the derivative kernel's fast path only
__device__ __noinline__ MaternVals matern_u_derivs_outofline(const ThetaParams& P, double u) {
  return matern_u<true>(P, u);
}
#endif

// Element (i, j) of the engine's padded matrices (Sigma with the augmented row / column n
// and identity padding; the derivative blocks zero outside [0, n)^2).
__device__ __forceinline__ void engine_element(const GenItem& it, const ThetaParams& P, int i,
                                               int j, int n, bool derivs, double& c, double& da,
                                               double& dn) {
  da = 0.0;
  dn = 0.0;
  if (i >= n || j >= n) {
    // augmented row / padding
    if (i == j) {
      c = (i == n) ? 0.0 : 1.0;
    } else if (i == n && j < n) {
      c = it.z[j];
    } else if (j == n && i < n) {
      c = it.z[i];
    } else {
      c = 0.0;
    }
  } else if (i == j) {
    c = P.sigma2 + P.nugget;  // matern.py:182 fill_diagonal(sigma2)
  } else {
    const double h = pair_distance(it.lx, it.ly, i, j);
    if (h > 0.0) {
      MaternVals v;
      const double u = h / P.alpha;
      if (it.tab != nullptr && u >= P.tab_lo && u < P.tab_hi) {
        if (derivs)
          v = matern_table<true>(P, it.tab, u);
        else
          v = matern_table<false>(P, it.tab, u);
      } else if (derivs) {
        v = matern_u_call<true>(P, u);
      } else {
        v = matern_u_call<false>(P, u);
      }
      c = v.c;
      da = v.dalpha;
      dn = v.dnu;
    } else {
      c = P.sigma2;  // coincident locations: zero-lag limit (matern.py:173-178)
    }
  }
}

// kDerivs = 0: Sigma (lower tiles); 1: both derivative matrices (full storage, mirrored;
// lower tiles only with GenArgs.lower_only -- the two-sided solves read only those).
//
// Interior off-diagonal tiles (every index < n, i != j: nearly all of them) take a fast path.
// Each warp evaluates compact 4 x 8 patches of the tile (4 consecutive rows x 8 consecutive
// columns) rather than one 32-row column: consecutive location indices are spatial
// neighbours, so the 32 pair distances of a patch are close and fall into one to three
// table intervals.  The 16-byte coefficient loads of a warp then touch few distinct lines
// (each distinct interval is one more L1 wavefront: with 32-row columns, ~8 per load, that
// request rate bounded the kernel).  The values go through a shared-memory tile and leave
// with coalesced column stores.
template <int kDerivs>
__global__ void __launch_bounds__(kGThreads, MLE_GEN_MINB) gen_engine_kernel(GenArgs a) {
  const GenItem& it = a.item[blockIdx.y];
  // The item's failure flag is tested after the fast path has issued its parameter loads (no
  // store happens before the test): one global-load latency per CTA instead of two in a row.
  int failed = 0;
  if (it.fail_flag != nullptr) failed = *it.fail_flag;
  __shared__ __align__(16) ThetaParams P;
  __shared__ double s_v0[kGT * kGT];
  __shared__ double s_v1[kDerivs ? kGT * kGT : 1];
  int ti, tj;
  if (a.region == 1) {  // tile columns < jcut: grid (tile rows) x jcut, upper ones skipped
    ti = (int)(blockIdx.x / a.jcut);
    tj = (int)(blockIdx.x % a.jcut);
    if (tj > ti) return;
  } else {
    lower_tile_index(blockIdx.x, &ti, &tj);
    if (a.region == 2) {  // the lower triangle of the trailing block [jcut, T)^2
      ti += a.jcut;
      tj += a.jcut;
    }
  }
  const int lane_row = threadIdx.x & (kGT - 1);
  const int col0 = threadIdx.x >> 5;
  const int i = ti * kGT + lane_row;
  const long long ld = a.ld;
  const int n = a.n;
  if (ti != tj && (ti + 1) * kGT <= n && it.tab != nullptr) {
    // The parameters are read straight from global memory (L1-resident: a few scalars)
    // instead of staging all ~7 KB per CTA.
    const ThetaParams& Pg = *it.P;
    const double lo = Pg.tab_lo, hi = Pg.tab_hi, alpha = Pg.alpha;
    const double ialpha = 1.0 / alpha;  // correctly rounded reciprocal
    const long long key0 = Pg.tab_key0;
    if (failed) return;
    const double* __restrict__ tab = it.tab;
    const double* __restrict__ lx = it.lx;
    const double* __restrict__ ly = it.ly;
    __shared__ unsigned short s_exact[kGT * kGT];
    __shared__ int s_nexact;
    // The tile's table intervals staged in shared memory (a.stage_tab): a warp's coefficient
    // load costs the L1 pipe 3.3 cycles from global memory (LDG.128, any address pattern)
    // and 1.7 from shared memory (LDS.128, up to eight distinct intervals conflict-free at
    // the 84-word interval stride) -- tools/microbench/ld_bcast.cu.  Same coefficients, same
    // Horner order: bit-identical to the global-memory path.
    __shared__ __align__(16) double s_tab[kGenSlots * 3 * MLE_TAB_P];
    __shared__ int s_kmin, s_kmax;
    if (threadIdx.x == 0) {
      s_nexact = 0;
      s_kmin = MLE_TAB_MAX;
      s_kmax = -1;
    }
    __syncthreads();
    const int pr = threadIdx.x & 3, pc = (threadIdx.x >> 2) & 7, warp = threadIdx.x >> 5;
    // This thread's four elements: lane position (pr, pc) of patches warp + 8 e (32 patches:
    // 8 patch rows x 4 patch columns).
    double u[4];
    unsigned kk = 0;     // the four interval indices, one byte each (MLE_TAB_MAX < 256)
    unsigned intab = 0;  // bit e: element e is inside the table range
    int kmin_t = MLE_TAB_MAX, kmax_t = -1;
    // pdist-identical distances (no FMA contraction).  The square root is the branch-free
    // correctly rounded one of the pivot chain (pivot_math.cuh: bit-equal to __dsqrt_rn on
    // normal-range inputs), so the four elements' chains interleave instead of each sitting
    // in its own slow-path basic block; squared distances outside its range (coincident or
    // denormally close points) take the IEEE intrinsic below.
    double s2[4];
    bool odd = false;
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      const int patch = warp + 8 * e;
      const int row = 4 * (patch & 7) + pr, col = 8 * (patch >> 3) + pc;
      const int ii = ti * kGT + row, j = tj * kGT + col;
      const double dx = __dsub_rn(lx[ii], lx[j]);
      const double dy = __dsub_rn(ly[ii], ly[j]);
      s2[e] = __dadd_rn(__dmul_rn(dx, dx), __dmul_rn(dy, dy));
      odd |= !(s2[e] >= 1e-280 && s2[e] <= 1e280);
    }
    double hh[4];
#pragma unroll
    for (int e = 0; e < 4; ++e) hh[e] = pivot_sqrt_rn(s2[e]);
    if (odd) {  // rare: one branch per thread instead of one per element
#pragma unroll
      for (int e = 0; e < 4; ++e) hh[e] = __dsqrt_rn(s2[e]);
    }
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      const double h = hh[e];
      // u = h / alpha (matern.py:103) by Markstein's correction of h * (1 / alpha): the
      // residual h - alpha q is exact (FMA), and q + r / alpha rounds to the correctly
      // rounded quotient, without the division's iteration and slow-path branch
      const double q = h * ialpha;
      u[e] = fma(fma(-alpha, q, h), ialpha, q);
      const bool in = u[e] >= lo && u[e] < hi;
      const double ut = in ? u[e] : lo;  // any valid interval for the others
      const long long b = __double_as_longlong(ut);
      const int key = (int)((b >> 49) - key0);
      const int k = key - (key > kGenMergeKey ? 1 : 0) -
                    (key > kGenMergeKey + 1 && ut < MLE_SMALL_MID_SPLIT ? 1 : 0);
      kk |= (unsigned)k << (8 * e);
      intab |= (in ? 1u : 0u) << e;
      kmin_t = min(kmin_t, k);
      kmax_t = max(kmax_t, k);
    }
    bool staged = false;
    int kbase = 0;
    if (a.stage_tab) {
      kmin_t = __reduce_min_sync(0xffffffffu, kmin_t);
      kmax_t = __reduce_max_sync(0xffffffffu, kmax_t);
      if ((threadIdx.x & 31) == 0) {
        atomicMin(&s_kmin, kmin_t);
        atomicMax(&s_kmax, kmax_t);
      }
      __syncthreads();
      kbase = s_kmin;
      const int nslots = s_kmax - kbase + 1;
      staged = nslots <= kGenSlots;  // CTA-uniform; wider tiles (near neighbours) read global
      if (staged) {
        constexpr int kPer = 3 * MLE_TAB_P / 2;  // 16-byte words per interval
        const double2* src = reinterpret_cast<const double2*>(tab) + (size_t)kbase * kPer;
        double2* dst = reinterpret_cast<double2*>(s_tab);
        for (int w = threadIdx.x; w < nslots * kPer; w += kGThreads) dst[w] = __ldg(src + w);
        __syncthreads();
      }
    }
    // kE elements at a time, their kF Horner chains interleaved (4 independent chains per
    // thread: latency, not issue, bounded the element-serial version), branch-free for the
    // table elements; the rare exact-path / coincident elements are patched afterwards.
    constexpr int kF = kDerivs ? 2 : 1;
#ifndef MLE_GEN_KE_D
#define MLE_GEN_KE_D 2
#endif
#ifndef MLE_GEN_KE_S
#define MLE_GEN_KE_S 4
#endif
    constexpr int kE = kDerivs ? MLE_GEN_KE_D : MLE_GEN_KE_S;  // elements per round
    auto rounds = [&](auto staged_tag) {
      constexpr bool kStaged = decltype(staged_tag)::value;
      const int kofs = kStaged ? kbase : 0;
#pragma unroll
      for (int r0 = 0; r0 < kGT / 8; r0 += kE) {
        double t[kE];
        int cofs[kE];
#pragma unroll
        for (int e = 0; e < kE; ++e) {
          // (an element outside the table range gets some finite t of the first interval's
          // map: its polynomial value is discarded below)
          const int k = (int)((kk >> (8 * (r0 + e))) & 255u);
          t[e] = gen_tab_t(u[r0 + e], k);
          cofs[e] = (k - kofs) * 3 * MLE_TAB_P + (kDerivs ? MLE_TAB_P : 0);
        }
        double p[kE][kF];
#pragma unroll
        for (int e = 0; e < kE; ++e)
#pragma unroll
          for (int f = 0; f < kF; ++f) {
            const int o = cofs[e] + f * MLE_TAB_P + MLE_TAB_P - 2;
            const double2 c = kStaged ? lds_pair(s_tab + o)
                                      : __ldg(reinterpret_cast<const double2*>(tab + o));
            p[e][f] = fma(c.y, t[e], c.x);
          }
#pragma unroll
        for (int i = MLE_TAB_P - 4; i >= 0; i -= 2)
#pragma unroll
          for (int e = 0; e < kE; ++e)
#pragma unroll
            for (int f = 0; f < kF; ++f) {
              const int o = cofs[e] + f * MLE_TAB_P + i;
              const double2 c = kStaged ? lds_pair(s_tab + o)
                                        : __ldg(reinterpret_cast<const double2*>(tab + o));
              p[e][f] = fma(p[e][f], t[e], c.y);
              p[e][f] = fma(p[e][f], t[e], c.x);
            }
#pragma unroll
        for (int e = 0; e < kE; ++e) {
          const int patch = warp + 8 * (r0 + e);
          const int row = 4 * (patch & 7) + pr, col = 8 * (patch >> 3) + pc;
          const double ue = u[r0 + e];
          // below 8.5 the series are of E itself; above, of e^u E (matern_table_at)
          if (ue >= MLE_SMALL_MID_SPLIT) {
            const double eu = exp(-ue);
#pragma unroll
            for (int f = 0; f < kF; ++f) p[e][f] *= eu;
          }
          if ((intab >> (r0 + e)) & 1u) {
            s_v0[tile_slot(row, col)] = p[e][0];
            if (kDerivs) s_v1[tile_slot(row, col)] = p[e][kF - 1];
          } else {  // exact path: queued, evaluated below by the whole CTA
            s_v0[tile_slot(row, col)] = ue;
            s_exact[atomicAdd(&s_nexact, 1)] = (unsigned short)(row * kGT + col);
          }
        }
      }
    };
    if (staged)
      rounds(std::true_type{});
    else
      rounds(std::false_type{});
    __syncthreads();
    // The few pairs outside the table range (u < tab_lo: near neighbours, or coincident)
    // run the exact evaluator compacted onto consecutive threads: one warp pass instead of a
    // mostly idle warp per element (the near-diagonal tiles hold most of them).
    for (int q = threadIdx.x; q < s_nexact; q += kGThreads) {
      const int row = s_exact[q] / kGT, col = s_exact[q] % kGT;
      const double ue = s_v0[tile_slot(row, col)];
      MaternVals v;
      if (ue > 0.0) {
#if MLE_GEN_EXACT_NOINLINE == 2
        if (kDerivs)
          v = matern_u_derivs_outofline(Pg, ue);
        else
          v = matern_u_call<false>(Pg, ue);
#else
        v = matern_u_call<kDerivs != 0>(Pg, ue);
#endif
      } else {  // coincident locations: zero-lag limit (matern.py:173-178)
        v.c = Pg.sigma2;
        v.dalpha = v.dnu = 0.0;
      }
      s_v0[tile_slot(row, col)] = kDerivs ? v.dalpha : v.c;
      if (kDerivs) s_v1[tile_slot(row, col)] = v.dnu;
    }
    __syncthreads();
    const long long j0 = (long long)tj * kGT + col0;
    double* ps = it.sigma + i + j0 * ld;
    double* pa = it.dalpha + i + j0 * ld;
    double* pn = it.dnu + i + j0 * ld;
#pragma unroll
    for (int r = 0; r < kGT / 8; ++r) {
      if (kDerivs) {  // a null block is skipped (sequential-derivative mode: one at a time)
        if (it.dalpha) pa[8 * r * ld] = s_v0[tile_slot(lane_row, col0 + 8 * r)];
        if (it.dnu) pn[8 * r * ld] = s_v1[tile_slot(lane_row, col0 + 8 * r)];
      } else {
        ps[8 * r * ld] = s_v0[tile_slot(lane_row, col0 + 8 * r)];
      }
    }
  } else {
    if (failed) return;
    stage_params(&P, it.P);
#pragma unroll 1
    for (int r = 0; r < kGT / 8; ++r) {
      const int jl = col0 + 8 * r;
      const int j = tj * kGT + jl;
      double c, da, dn;
      engine_element(it, P, i, j, n, kDerivs != 0, c, da, dn);
      const long long off = (long long)i + (long long)j * ld;
      if (kDerivs) {
        if (it.dalpha) it.dalpha[off] = da;
        if (it.dnu) it.dnu[off] = dn;
        s_v0[tile_slot(lane_row, jl)] = da;
        s_v1[tile_slot(lane_row, jl)] = dn;
      } else {
        it.sigma[off] = c;
      }
    }
  }
  if (kDerivs && ti != tj && !a.lower_only) {
    __syncthreads();
    // mirrored tile (J, I): rows from tile J, columns from tile I
    const int i2 = tj * kGT + lane_row;
#pragma unroll 1
    for (int r = 0; r < kGT / 8; ++r) {
      const int jl = col0 + 8 * r;
      const int j2 = ti * kGT + jl;
      const long long off = (long long)i2 + (long long)j2 * ld;
      if (it.dalpha) it.dalpha[off] = s_v0[tile_slot(jl, lane_row)];
      if (it.dnu) it.dnu[off] = s_v1[tile_slot(jl, lane_row)];
    }
  }
}

// Column panels (distributed engine): every element (i, j) of the panel's columns
// [c0, c0 + width), all rows [0, rows), written to panel[i + (j - c0) ld] (no symmetry
// shortcut: derivative panels hold full columns).  GenItem.sigma / dalpha / dnu are the
// panel bases; item b of the launch has its own c0 in a.item[b] via the `z` slot reuse below.
__global__ void __launch_bounds__(kGThreads) gen_panel_kernel(GenArgs a, const int* c0s,
                                                              int width) {
  const GenItem& it = a.item[blockIdx.z];
  if (it.fail_flag != nullptr && *it.fail_flag) return;
  __shared__ __align__(16) ThetaParams P;
  stage_params(&P, it.P);
  const int c0 = c0s[blockIdx.z];
  const int i = blockIdx.x * kGT + (threadIdx.x & (kGT - 1));
  const int jl0 = blockIdx.y * kGT;
  const bool derivs = it.write_derivs != 0;
  const long long ld = a.ld;
  if (i >= a.rows) return;
#pragma unroll 1
  for (int r = 0; r < kGT / 8; ++r) {
    const int jl = jl0 + (threadIdx.x >> 5) + 8 * r;
    if (jl >= width) continue;
    const int j = c0 + jl;
    double c, da, dn;
    engine_element(it, P, i, j, a.n, derivs, c, da, dn);
    const long long off = (long long)i + (long long)jl * ld;
    if (it.write_sigma) it.sigma[off] = c;
    if (derivs) {
      it.dalpha[off] = da;
      it.dnu[off] = dn;
    }
  }
}

// Polynomial pieces of e^u * {c, dalpha, dnu}(u) on every table interval of every item (grid:
// MLE_TAB_MAX x items; one CTA per interval).  Node values come from the exact evaluator
// (matern_u), so the table inherits its accuracy: Chebyshev interpolation at 14 nodes on
// intervals of ratio <= 1.125 (binade eighths; a convergence factor > 30 puts the degree-13
// truncation far below one ulp), expressed in the monomial basis in t in [-1, 1] for a
// one-FMA-per-term Horner evaluation.  Node values -> coefficients is one fixed linear map
// (transform + basis change, built in long double on the host) applied in double-double, so
// each coefficient is rounded once: computing it in plain double cost ~10x in accuracy
// (2.7e-15 vs 1.8e-16 relative on exact node values at u in [0.25, 2.25)), which moved the
// ill-conditioned goldens' log-likelihoods by ~1e-10.  Layout [interval][c, da, dn]
// [power] (16-byte aligned power pairs: the evaluator loads two coefficients per request).
__global__ void __launch_bounds__(64) gen_table_kernel(GenArgs a, int derivs) {
  const GenItem& it = a.item[blockIdx.y];
  if (it.tab == nullptr || (it.fail_flag != nullptr && *it.fail_flag)) return;
  const ThetaParams& P = *it.P;
  const int k = blockIdx.x;
  if (k >= P.tab_n) return;
  __shared__ double f[3][MLE_TAB_P];
  const int t = threadIdx.x;
  if (t < MLE_TAB_P) {
    const double x = cospi((t + 0.5) / MLE_TAB_P);
    const double u = P.tab_ctr[k] + P.tab_hw[k] * x;
    const MaternVals v = derivs ? matern_u<true>(P, u) : matern_u<false>(P, u);
    const double e = u < MLE_SMALL_MID_SPLIT ? 1.0 : exp(u);  // as matern_table
    f[0][t] = e * v.c;
    f[1][t] = e * v.dalpha;
    f[2][t] = e * v.dnu;
  }
  __syncthreads();
  // monomial coefficients a_i = sum_q M[i][q] f_q in double-double (M as hi + lo pairs):
  // the map has entries ~1e4 with alternating signs while high-order a_i are tiny, so a
  // plain double sum would leave ~10 ulps of cancellation error in every coefficient.
  if (t < 3 * MLE_TAB_P) {
    const int fn = t / MLE_TAB_P, i = t % MLE_TAB_P;
    double s_hi = 0.0, s_lo = 0.0;
    for (int q = 0; q < MLE_TAB_P; ++q) {
      const double fq = f[fn][q];
      const double mh = c_tab_map[0][i][q], ml = c_tab_map[1][i][q];
      const double p = mh * fq;
      const double pe = fma(mh, fq, -p) + ml * fq;  // exact product error + low part
      const double sum = s_hi + p;                  // two-sum(s_hi, p)
      const double bv = sum - s_hi;
      const double se = (s_hi - (sum - bv)) + (p - bv);
      s_hi = sum;
      s_lo += se + pe;
    }
    it.tab[((size_t)k * 3 + fn) * MLE_TAB_P + i] = s_hi + s_lo;
  }
}

// Full symmetric n x n matrix of one kind (mle_build), no augmentation / padding.
__global__ void __launch_bounds__(kGThreads) gen_build_kernel(GenArgs a, int which) {
  const GenItem& it = a.item[0];
  __shared__ __align__(16) ThetaParams P;
  __shared__ double s_v[kGT][kGT + 1];
  stage_params(&P, it.P);
  int ti, tj;
  lower_tile_index(blockIdx.x, &ti, &tj);
  const int lane_row = threadIdx.x & (kGT - 1);
  const int col0 = threadIdx.x >> 5;
  const int i = ti * kGT + lane_row;
  const long long ld = a.ld;
  const int n = a.n;
#pragma unroll 1
  for (int r = 0; r < kGT / 8; ++r) {
    const int jl = col0 + 8 * r;
    const int j = tj * kGT + jl;
    double v = 0.0;
    if (i < n && j < n) {
      if (i == j) {
        v = (which == MLE_WHICH_SIGMA) ? P.sigma2 + P.nugget
                                       : (which == MLE_WHICH_SIGMA2 ? 1.0 : 0.0);
      } else {
        const double h = pair_distance(it.lx, it.ly, i, j);
        if (h > 0.0) {
          if (which == MLE_WHICH_SIGMA || which == MLE_WHICH_SIGMA2) {
            const MaternVals m = matern_positive<false>(P, h);
            v = (which == MLE_WHICH_SIGMA) ? m.c : m.c / P.sigma2;  // matern.py:160
          } else {
            const MaternVals m = matern_positive<true>(P, h);
            v = (which == MLE_WHICH_ALPHA) ? m.dalpha : m.dnu;
          }
        } else {
          v = (which == MLE_WHICH_SIGMA) ? P.sigma2 : (which == MLE_WHICH_SIGMA2 ? 1.0 : 0.0);
        }
      }
      it.sigma[(long long)i + (long long)j * ld] = v;
    }
    s_v[lane_row][jl] = v;
  }
  if (ti != tj) {
    __syncthreads();
    const int i2 = tj * kGT + lane_row;
#pragma unroll 1
    for (int r = 0; r < kGT / 8; ++r) {
      const int jl = col0 + 8 * r;
      const int j2 = ti * kGT + jl;
      if (i2 < n && j2 < n) it.sigma[(long long)i2 + (long long)j2 * ld] = s_v[jl][lane_row];
    }
  }
}

// Elementwise evaluators (parity surface for bessel.py / matern.py scalar functions).
__global__ void elem_kernel(const ThetaParams* Pg, int op, int which,
                            const double* __restrict__ x, long long m, double* __restrict__ out) {
  __shared__ __align__(16) ThetaParams P;
  stage_params(&P, Pg);
  for (long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x; t < m;
       t += (long long)gridDim.x * blockDim.x) {
    const double v = x[t];
    double r;
    if (op == 0) {  // bessel_k(nu, x) = K_|nu|(x), x > 0 validated on the host
      double k_nu, k_m1;
      bessel_k_ladder(P.kmain, v, &k_nu, &k_m1);
      r = k_nu;
    } else if (op == 1) {  // dnu_xnu_knu(nu, x), x >= 0
      if (v == 0.0) {
        r = 0.0;  // bessel.py:358 (ZERO_ARG)
      } else {
        double k_nu, k_m1;
        bessel_k_ladder(P.kmain, v, &k_nu, &k_m1);
        const double v_nu = pow(v, P.nu);
        r = dnu_xnu_knu(P, v, v_nu * k_nu, v_nu);
      }
    } else if (op == 3) {  // one d/dnu series by itself (case2/3/4_series), domain checked
      const double v_nu = pow(v, P.nu);
      r = which == 2 ? dnu_case2(P, v, v_nu) : which == 3 ? dnu_case3(P, v, v_nu)
                                                          : dnu_case4(P, v, v_nu);
    } else {  // Matern value / derivative at distance h >= 0
      if (v > 0.0) {
        if (which == MLE_WHICH_SIGMA || which == MLE_WHICH_SIGMA2) {
          const MaternVals mv = matern_positive<false>(P, v);
          r = (which == MLE_WHICH_SIGMA) ? mv.c : mv.c / P.sigma2;
        } else {
          const MaternVals mv = matern_positive<true>(P, v);
          r = (which == MLE_WHICH_ALPHA) ? mv.dalpha : mv.dnu;
        }
      } else {
        r = (which == MLE_WHICH_SIGMA) ? P.sigma2 : (which == MLE_WHICH_SIGMA2 ? 1.0 : 0.0);
      }
    }
    out[t] = r;
  }
}

cudaError_t upload_u_tables(const double* u, const double* du) {
  cudaError_t e = cudaMemcpyToSymbol(c_u_coef, u, sizeof(double) * (MLE_CASE3_NEAR + 1) *
                                                      MLE_U_COEFF_STRIDE);
  if (e != cudaSuccess) return e;
  e = cudaMemcpyToSymbol(c_du_coef, du, sizeof(double) * (MLE_CASE3_NEAR + 1) *
                                            MLE_U_COEFF_STRIDE);
  if (e != cudaSuccess) return e;
  double map[2][MLE_TAB_P * MLE_TAB_P];
  mle_fill_tab_map(map[0], map[1]);
  return cudaMemcpyToSymbol(c_tab_map, map, sizeof(map));
}

static long long lower_tiles(long long rows) {
  const long long t = (rows + kGT - 1) / kGT;
  return t * (t + 1) / 2;
}

// Every item of one launch writes the same kind (Sigma, or the derivative pair).
void launch_gen_engine(const GenArgs& a, int items, cudaStream_t s) {
  const long long T = (a.rows + kGT - 1) / kGT;
  const long long blocks = a.region == 1 ? T * a.jcut
                           : a.region == 2 ? (T - a.jcut) * (T - a.jcut + 1) / 2
                                           : lower_tiles(a.rows);
  if (blocks <= 0) return;
  const dim3 grid((unsigned)blocks, (unsigned)items);
  // The derivative kernel (two functions per element: L1-bound on its coefficient loads)
  // stages the tile's table intervals in shared memory: config 4 1485 -> 1581 GB/s.  The
  // Sigma kernel (one function, issue-bound) loses 4% to the extra barrier, so it reads
  // global memory.  MLE_GEN_STAGE=0 / 2: neither / both (A/B; all bit-identical).
  static const int stage = [] {
    const char* e = std::getenv("MLE_GEN_STAGE");
    return (e != nullptr && e[0] >= '0' && e[0] <= '2') ? e[0] - '0' : 1;
  }();
  GenArgs b = a;
  b.stage_tab = stage == 2 || (stage == 1 && a.item[0].write_derivs);
  if (b.item[0].write_derivs)
    gen_engine_kernel<1><<<grid, kGThreads, 0, s>>>(b);
  else
    gen_engine_kernel<0><<<grid, kGThreads, 0, s>>>(b);
}

void launch_gen_panels(const GenArgs& a, const int* c0s_dev, int width, int items,
                       cudaStream_t s) {
  const dim3 grid((unsigned)((a.rows + kGT - 1) / kGT), (unsigned)((width + kGT - 1) / kGT),
                  (unsigned)items);
  gen_panel_kernel<<<grid, kGThreads, 0, s>>>(a, c0s_dev, width);
}

void launch_gen_table(const GenArgs& a, int items, bool derivs, cudaStream_t s) {
  gen_table_kernel<<<dim3(MLE_TAB_MAX, (unsigned)items), 64, 0, s>>>(a, derivs ? 1 : 0);
}

void launch_gen_build(const GenArgs& a, int which, cudaStream_t s) {
  gen_build_kernel<<<(unsigned)lower_tiles(a.n), kGThreads, 0, s>>>(a, which);
}

void launch_elem(const ThetaParams* P_dev, int op, int which, const double* x, long long m,
                 double* out, cudaStream_t s) {
  long long blocks = (m + 255) / 256;
  if (blocks > 148 * 64) blocks = 148 * 64;
  if (blocks < 1) blocks = 1;
  elem_kernel<<<(unsigned)blocks, 256, 0, s>>>(P_dev, op, which, x, m, out);
}

}  // namespace mle
