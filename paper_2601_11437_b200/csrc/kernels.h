// kernels.h — internal launch interface between the C-ABI engine (engine.cu) and the
// sm_100a kernels (gen.cu, linalg.cu).  Not part of the public ABI.
//
// Every kernel is batched over "items": independent datasets of the same padded size that
// are evaluated together (replicate fits, L9 start points).  Item b of a launch uses the
// b-th pointer of each array below and its own failure flag.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include "../../include/maternfisher.h"
#include "theta.h"

namespace mle {

constexpr int kNB = 128;       // factorization tile (Cholesky / solve block size)
constexpr int kMaxItems = 8;   // datasets per batched launch
constexpr int kMaxGemm = 8 * kMaxItems;  // batch members per GEMM launch (item x block)

struct GenItem {
  const ThetaParams* P;  // device copy of this item's per-theta scalars
  const double* lx;   // x coordinates (n)
  const double* ly;   // y coordinates (n)
  const double* z;    // observed values (n); augmented row
  double* sigma;      // Sigma (engine) or the single output (build)
  double* dalpha;     // dSigma/dalpha (full storage)
  double* dnu;        // dSigma/dnu (full storage)
  const int* fail_flag;
  double* tab;        // generation table ([MLE_TAB_MAX][3][MLE_TAB_P]); null: exact path
  int write_sigma;    // 1: write Sigma (lower tiles + augmented row + padding)
  int write_derivs;   // 1: write both derivative matrices (full storage)
};

struct GenArgs {
  GenItem item[kMaxItems];
  long long ld;       // leading dimension (column-major)
  long long rows;     // padded extent N (engine) / n (build)
  int n;              // number of locations
  int region;         // engine: 0 every lower tile; 1 tile columns < jcut; 2 tile columns >= jcut
  int jcut;           // in 32-wide generation tiles
  int lower_only;     // derivative matrices: lower tiles only (no mirrored upper tiles)
  int stage_tab;      // engine fast path: stage the tile's table intervals in shared memory
};

// Operand layouts of op(B): B(n,k) at b[n + k*ldb] (kBNK) or b[k + n*ldb] (kBKN).
enum BLayout { kBNK = 0, kBKN = 1 };

struct GemmArgs {
  const double* A[kMaxGemm];
  const double* B[kMaxGemm];
  double* C[kMaxGemm];
  const int* fail_flag[kMaxGemm];
  long long lda, ldb, ldc;
  int K;             // multiple of 16
  int tiles_m;       // number of 128-row tiles of C
  int tiles_n;       // number of 128-column tiles of C (full mode)
  int lower;         // 1: only tiles (tm >= tn) of a tiles_m x tiles_m grid
  int trap;          // full mode: 1 skips tiles with tm + trap_off < tn (lower trapezoid)
  int trap_off;      // row-tile offset of C's base above its column-tile offset (0 usually)
  int wide;          // 1: 128-column CTAs (C aliases A across the 128-wide panel)
  double alpha;      // +1 or -1
  double beta;       // 0 (overwrite) or 1 (accumulate into C)
};

struct DiagArgs {
  double* a[kMaxItems];
  double* linv[kMaxItems];      // 128 x 128 inverse of this step's diagonal tile
  int* fail_flag[kMaxItems];
  long long* fail_idx[kMaxItems];
  long long n_aug[kMaxItems];   // augmented index (no pivot check), -1 for none
  long long ld;
  int k0;
};

struct ReduceArgs {
  const double* L[kMaxItems];
  const double* Ba[kMaxItems];  // null for loglik-only items
  const double* Bn[kMaxItems];
  const double* Bm[kMaxItems];  // nugget items: M = L^-1 L^-T (null otherwise)
  double* partials[kMaxItems];
  double* out[kMaxItems];
  const int* fail_flag[kMaxItems];
  long long ld;
  int n;
};

cudaError_t init_kernel_attributes();  // GEMM smem opt-in (per device)
cudaError_t init_diag_attributes();    // diagonal-tile kernel smem opt-in (per device)
cudaError_t upload_u_tables(const double* u, const double* du);
void launch_gen_engine(const GenArgs& a, int items, cudaStream_t s);
// Column panels of the distributed engine: columns [c0s[b], c0s[b] + width) of item b, all
// rows; c0s_dev is a device array (one int per item).
void launch_gen_panels(const GenArgs& a, const int* c0s_dev, int width, int items,
                       cudaStream_t s);
// Coefficients of the items' generation tables (items with tab == null are skipped).
void launch_gen_table(const GenArgs& a, int items, bool derivs, cudaStream_t s);
void launch_gen_build(const GenArgs& a, int which, cudaStream_t s);
void launch_elem(const ThetaParams* P_dev, int op, int which, const double* x, long long m,
                 double* out, cudaStream_t s);

// C = alpha * A * op(B) + beta * C per batch member (gridDim.z = batch).
cudaError_t launch_gemm(const GemmArgs& g, BLayout bl, int batch, cudaStream_t s);
// Small-tile DMMA GEMM for single 128 x 128 tiles on the Cholesky chain (kBNK B, K <= 128):
// rows_only = 1 -> 16 x 128 CTAs (C may alias A), 0 -> 32 x 32 CTAs.
cudaError_t init_small_gemm_attributes();
cudaError_t launch_gemm_small(const GemmArgs& g, int batch, cudaStream_t s, int rows_only);
// Factor the 128x128 diagonal tile at (k0, k0) of every item in place (+ its inverse).
cudaError_t launch_potrf_diag(const DiagArgs& d, int items, cudaStream_t s);
// Reductions: per item kReduceOut results [logdet, quad, trA, trN, <A,A>, <A,N>, <N,N>,
// trM, <A,M>, <N,M>, <M,M>, yBy_A, yBy_N, yBy_M, min L_jj, max L_jj] (the M terms only for
// nugget items; the diagonal extremes give the engine a conditioning estimate).
cudaError_t launch_reduce(const ReduceArgs& r, int items, cudaStream_t s);

// Scatter the diagonal-tile inverses Linv_k into the per-outer-block inverse storage:
// dinv[z] + (k / 4) 512^2 + (k % 4) 128 (1 + 512)  <-  linv[z] + k 128^2   (k < Nt).
cudaError_t launch_linv_to_dinv(double* const* dinv, const double* const* linv, int Nt,
                                int items, cudaStream_t s);

// Per-pass bookkeeping in two launches instead of per-item copies: scatter the staged
// ThetaParams of every item into its context (and clear its failure flag), and gather every
// item's kReduceOut results + failure flag + pivot into one buffer (slots of 8 bytes:
// [0, kReduceOut) results, kReduceOut flag (int), kReduceOut + 1 pivot (long long)).
struct PassIo {
  ThetaParams* theta[kMaxItems];
  int* flag[kMaxItems];
  const double* out[kMaxItems];
  const long long* idx[kMaxItems];
};
cudaError_t launch_scatter_theta(const PassIo& io, const ThetaParams* staged, int items,
                                 cudaStream_t s);
cudaError_t launch_gather_results(const PassIo& io, double* dst, int items, cudaStream_t s);

// Sequential-derivative mode (linalg.cu): park the lower triangle of a finished block in the
// unused upper triangle of an N x (N + 513) array, identity on the lower triangle + diagonal
// band only, and the sums of one block against up to two parked blocks
// (out: [tr W, <W,W>, <W,U1>, <W,U2>, W[n,n]]; partials >= kReduceBlocks * 4 doubles).
constexpr int kParkExtraCols = 513;
cudaError_t launch_park_lower(const double* src, double* park, long long ld, int N,
                              cudaStream_t s);
cudaError_t launch_set_identity_lower(double* S, long long ld, int n, int N, cudaStream_t s);
cudaError_t launch_seq_reduce(const double* W, const double* U1, const double* U2, long long ld,
                              int n, int N, double* partials, double* out, cudaStream_t s);

// S = I_n inside the padded N x N matrix (zero elsewhere), for every item.
cudaError_t launch_set_identity(double* const* S, long long ld, int n, int items,
                                cudaStream_t s);

// z = L w over the leading n x n block of a resident Cholesky factor.
cudaError_t launch_trmv_lower(const double* L, long long ld, int n, const double* w, double* z,
                              cudaStream_t s);

// Ozaki-scheme FP64 GEMM on tcgen05 int8 tensor cores (ozaki.cu).
// Slicing: X is rows x K (rows multiple of 128, K multiple of 32) with X(r,k) at
// X[r + k*ld] (row_contig) or X[k + r*ld]; writes S int8 slices (balanced base-256 digits) in
// UMMA canonical layout [rows/128][K/32][S][128x32] and one power-of-two exponent per row.
struct OzSliceArgs {
  const double* X[kMaxGemm];
  int8_t* slices[kMaxGemm];
  int* e[kMaxGemm];
  const int* fail_flag[kMaxGemm];
  long long ld;
  int K;
  int upper_zero;  // 1: element (r, k) with k > r (same origin) is taken as 0
  int nslices;     // 6 or 7 (0: 7); layout [rows/128][K/32][slices][128 x 32]
  int rows_z[kMaxGemm];  // per-member row count (0: the launch's rows)
};
// C = alpha * A B^T + beta * C from slices (A: M rows, B: N rows, both over the same K).
struct OzGemmArgs {
  const int8_t* As[kMaxGemm];
  const int8_t* Bs[kMaxGemm];
  const int* ea[kMaxGemm];
  const int* eb[kMaxGemm];
  double* C[kMaxGemm];
  const int* fail_flag[kMaxGemm];
  long long ldc;
  int kblocks;   // K / 32
  int tiles_m;   // 128-row tiles
  int tiles_n;   // 128-column tiles (full mode)
  int lower, trap;
  double alpha, beta;
  int beta0_tm, beta0_tn;  // tiles with tm < beta0_tm or tn < beta0_tn overwrite (beta = 0)
  int tiles_m_z[kMaxGemm];  // full/trap mode: per-member row tiles (0: tiles_m)
  int nslices;              // 6 or 7 (0: 7) -- both operands
  int max_ctas;             // persistent grid cap (0: one CTA per SM); look-ahead launches
                            // leave SMs to the latency-bound factorization chain
  int diag_mode;  // developer diagnostics only: 1 skip the MMAs, 2 skip the loads (0: normal)
  long long* diag_out;  // developer diagnostics: MMA-thread timing of CTA 0 (null: off)
};
constexpr int kOzSlices = 7;     // slices of the factor (Cholesky, W_b); also the buffer stride
inline int oz_nslices(int v) { return v == 6 ? 6 : 7; }
inline int oz_products(int v) { const int s = oz_nslices(v); return s * (s + 1) / 2; }
// bytes of slice storage for a rows x K operand (at most kOzSlices slices)
inline size_t oz_slice_bytes(long long rows, int K) { return (size_t)rows * K * kOzSlices; }
cudaError_t init_ozaki_attributes();
cudaError_t launch_oz_slice(const OzSliceArgs& a, int rows, bool row_contig, int batch,
                            cudaStream_t s);
// n_tile: 0 persistent 128x64 in CTA pairs sharing A (default), 1 128x32, 2 128x64 unpaired
cudaError_t launch_ozgemm(const OzGemmArgs& g, int batch, cudaStream_t s, int n_tile = 0);

// ---- distributed engine: column panels (element (i, j) of panel z at p[z][i + (j - c0) ld])
struct PanelArgs {
  double* p[kMaxItems];
  long long c0[kMaxItems];
  long long ld;
  int width;
  int n;
};
constexpr int kPanelSums = 14;  // reduce sums (kReduceSums) + B_alpha / B_nu / M at [n, n]
struct PanelReduceArgs {
  const double* L[kMaxItems];
  const double* Ba[kMaxItems];
  const double* Bn[kMaxItems];
  const double* Bm[kMaxItems];
  double* partials[kMaxItems];  // [width][kPanelSums]
  long long c0[kMaxItems];
  long long ld;
  int n;
};
cudaError_t launch_linv_to_dinv_block(double* const* dinv, const double* const* linv,
                                      int k_begin, int tiles, int items, cudaStream_t s);
cudaError_t launch_panel_identity(const PanelArgs& a, int items, cudaStream_t s);
// developer diagnostics: per-CTA globaltimer trace of potrf_diag_kernel (linalg.cu)
cudaError_t diag_trace_control(long long* buf, unsigned long long cap, unsigned long long* count);
// upper triangle of a size x size block (column-major, ld) from its lower triangle, batched
cudaError_t launch_mirror_lower(double* const* a, int items, long long ld, int size,
                                cudaStream_t s);
cudaError_t launch_panel_reduce(const PanelReduceArgs& r, int width, int items, cudaStream_t s);

constexpr int kReduceBlocks = 148 * 4;
constexpr int kReduceSums = 11;
constexpr int kReducePartials = kReduceSums + 2;  // + per-block min / max of diag(L)
constexpr int kReduceOut = kReduceSums + 5;  // sums, yBy_A/N/M, min diag(L), max diag(L)

}  // namespace mle
