// engine.cu — C ABI (include/maternfisher.h) and the batched per-evaluation schedule.
//
// One mle_ctx = one dataset resident on one GPU with its own CUDA stream.  An evaluation
// request is (ctx, theta, mode); requests on several contexts of the same padded size run
// as ONE batched pass (mle_eval_batch), every kernel launch covering all of them:
//
//   gen      Sigma (lower tiles, augmented row n = z, identity padding) and, for eval_all,
//            dSigma/dalpha, dSigma/dnu (full storage)                    [gen.cu]
//   potrf    two-level right-looking blocked Cholesky, nb = 128 inner steps (diagonal tile
//            factor + inverse, panel x Linv^T, updates inside the outer block), K = 512
//            outer trailing SYRK                                          [linalg.cu]
//            -> row n of L is y^T = (L^-1 z)^T (the reference's `white`, likelihood.py:121)
//   solve    X_i = L^-1 S_i (row panels Linv_k S_k, GEMM updates), then the lower half of
//            B_i = X_i L^-T by a right-looking column sweep; B_i = L^-1 S_i L^-T.
//   reduce   log det, y^T y, tr B_i, <B_i,B_j>_F, and y^T B_i y = B_i[n,n] (augmented)
//
// The score and Fisher information then follow likelihood.py:123-147 with
// tr(Sigma^-1 S_i) = tr B_i, w^T S_i w = y^T B_i y and tr(W_i W_j) = <B_i, B_j>_F.
//
// Factor cache: after a successful factorization the context remembers theta; an eval_all
// (or loglik) at the same theta reuses the resident L and skips generation of Sigma and the
// Cholesky (Fisher-BT always follows an accepted loglik(theta) with eval_all(theta),
// optimizer.py:362,375).  Results are bit-identical to recomputing.
#include <cuda_runtime.h>
#include <nvtx3/nvToolsExt.h>
#include <atomic>

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <chrono>
#include <cstring>
#include <map>
#include <mutex>
#include <unordered_map>
#include <string>
#include <vector>

#include "kernels.h"

// NVTX ranges (MLE_NVTX=1) around every pass and its four phases, on the host timeline of the
// enqueueing thread: Nsight Systems / ncu --nvtx then attribute each launch to its phase.
// nvtx3 is header-only and a no-op without an attached tool; the switch keeps even that
// cost off the default path.
namespace {
struct NvtxPhases {
  bool on;
  int depth = 0;
  NvtxPhases() {
    static const bool enabled = [] {
      const char* e = getenv("MLE_NVTX");
      return e && e[0] == '1';
    }();
    on = enabled;
  }
  void push(const char* name) {
    if (on) {
      nvtxRangePushA(name);
      ++depth;
    }
  }
  void pop() {
    if (on && depth > 0) {
      nvtxRangePop();
      --depth;
    }
  }
  void next(const char* name) {  // close the current phase, open the next
    pop();
    push(name);
  }
  ~NvtxPhases() {
    while (depth > 0) pop();  // error returns leave no range open
  }
};
}  // namespace

using namespace mle;

namespace {

thread_local std::string g_last_error;
std::mutex g_init_mutex;
std::vector<int> g_device_ready;
// GPU idle gap between consecutive passes led by one context (diagnostic, kernel-stats slot
// 8): end-of-pass events alternate between two slots.  Per context, so host threads driving
// disjoint contexts (fit_many groups) never share one.
struct PassClock {
  cudaEvent_t end[2] = {nullptr, nullptr};
  cudaEvent_t start = nullptr;
  cudaEvent_t pre = nullptr;  // before the pass waits on pending speculation
  long long passes = 0;
};
// Streams and events of destroyed contexts, per device, for the next context (creating and
// destroying 4 streams and ~30 events per context cost ~0.5 ms, i.e. ~1.5% of an end-to-end
// config-2 step that builds five contexts).
struct StreamSet {
  cudaStream_t stream, side, inner, aux, edge;
  cudaEvent_t ev[5], ev_der, spec_done, pool[16], clk[4];
};
std::mutex g_sets_mutex;
std::vector<std::vector<StreamSet>> g_sets;

const double kLog2Pi = 1.8378770664093453;  // log(2 pi), likelihood.py:38
constexpr int kOuter = 4;                   // outer block = 4 x 128 columns
constexpr int kResults = 13;                // loglik, grad[3], fisher[9]
constexpr int kPoolEvents = 16;             // cross-stream join events per context

int fail(int code, const std::string& msg) {
  g_last_error = msg;
  return code;
}

// Caching allocator for device and pinned host buffers.  Contexts of the same size are
// created and destroyed repeatedly (one per dataset, fit after fit); returning their
// buffers to per-(device, size) free lists keeps cudaMalloc / cudaFree -- which map pages
// and synchronise the device -- out of the steady state.  Idle bytes are capped; an
// allocation that fails releases the idle buffers and retries once.
struct BufferCache {
  std::mutex mu;
  std::unordered_map<void*, std::pair<int, size_t>> live;  // ptr -> (device or -1, bytes)
  std::multimap<std::pair<int, size_t>, void*> idle;
  size_t idle_bytes = 0;
};
BufferCache& buffer_cache() {
  static BufferCache* c = new BufferCache();  // never destroyed: frees may run at exit
  return *c;
}
constexpr size_t kCacheIdleCap = size_t(48) << 30;

void raw_free(int dev, void* p) {
  if (dev < 0) {
    cudaFreeHost(p);
    return;
  }
  int cur = -1;
  cudaGetDevice(&cur);
  if (cur != dev) cudaSetDevice(dev);
  cudaFree(p);
  if (cur != dev && cur >= 0) cudaSetDevice(cur);
}

void cache_trim(int dev_filter) {  // dev_filter < -1: every device and the host
  std::vector<std::pair<int, void*>> drop;
  {
    BufferCache& c = buffer_cache();
    std::lock_guard<std::mutex> lock(c.mu);
    for (auto it = c.idle.begin(); it != c.idle.end();) {
      if (dev_filter < -1 || it->first.first == dev_filter) {
        drop.push_back({it->first.first, it->second});
        c.idle_bytes -= it->first.second;
        it = c.idle.erase(it);
      } else {
        ++it;
      }
    }
  }
  for (auto& d : drop) raw_free(d.first, d.second);
}

cudaError_t cache_alloc(void** p, size_t bytes, bool host) {
  int dev = -1;
  if (!host) {
    cudaError_t e = cudaGetDevice(&dev);
    if (e != cudaSuccess) return e;
  }
  bytes = std::max<size_t>(bytes, 1);
  BufferCache& c = buffer_cache();
  {
    std::lock_guard<std::mutex> lock(c.mu);
    auto it = c.idle.find({dev, bytes});
    if (it != c.idle.end()) {
      *p = it->second;
      c.idle.erase(it);
      c.idle_bytes -= bytes;
      c.live[*p] = {dev, bytes};
      return cudaSuccess;
    }
  }
  auto raw = [&]() { return host ? cudaMallocHost(p, bytes) : cudaMalloc(p, bytes); };
  cudaError_t e = raw();
  if (e != cudaSuccess) {
    cudaGetLastError();
    cache_trim(dev);
    e = raw();
    if (e != cudaSuccess) return e;
  }
  std::lock_guard<std::mutex> lock(c.mu);
  c.live[*p] = {dev, bytes};
  return cudaSuccess;
}

void cache_free(void* p) {
  if (!p) return;
  BufferCache& c = buffer_cache();
  std::pair<int, size_t> info;
  {
    std::lock_guard<std::mutex> lock(c.mu);
    auto it = c.live.find(p);
    if (it == c.live.end()) return;
    info = it->second;
    c.live.erase(it);
    if (c.idle_bytes + info.second <= kCacheIdleCap) {
      c.idle.insert({info, p});
      c.idle_bytes += info.second;
      return;
    }
  }
  raw_free(info.first, p);
}

template <class T>
cudaError_t dmalloc(T** p, size_t bytes) {
  return cache_alloc(reinterpret_cast<void**>(p), bytes, false);
}
template <class T>
cudaError_t hmalloc(T** p, size_t bytes) {
  return cache_alloc(reinterpret_cast<void**>(p), bytes, true);
}
inline void dfree(const void* p) { cache_free(const_cast<void*>(p)); }

#define CUDA_TRY(expr)                                                                  \
  do {                                                                                  \
    cudaError_t _e = (expr);                                                            \
    if (_e != cudaSuccess)                                                              \
      return fail(MLE_CUDA_ERROR, std::string(#expr) + ": " + cudaGetErrorString(_e));  \
  } while (0)

int ensure_device(int device) {
  int count = 0;
  cudaError_t e = cudaGetDeviceCount(&count);
  if (e != cudaSuccess || count == 0)
    return fail(MLE_CUDA_ERROR, "no CUDA device available (the engine has no CPU fallback)");
  if (device < 0 || device >= count) return fail(MLE_INVALID, "device index out of range");
  CUDA_TRY(cudaSetDevice(device));
  std::lock_guard<std::mutex> lock(g_init_mutex);
  if ((int)g_device_ready.size() < count) g_device_ready.resize(count, 0);
  if (!g_device_ready[device]) {
    std::vector<double> u((MLE_CASE3_NEAR + 1) * MLE_U_COEFF_STRIDE);
    std::vector<double> du((MLE_CASE3_NEAR + 1) * MLE_U_COEFF_STRIDE);
    mle_fill_u_tables(u.data(), du.data());
    CUDA_TRY(upload_u_tables(u.data(), du.data()));
    CUDA_TRY(init_kernel_attributes());
    CUDA_TRY(init_small_gemm_attributes());
    CUDA_TRY(init_diag_attributes());
    CUDA_TRY(init_ozaki_attributes());
    g_device_ready[device] = 1;
  }
  return MLE_OK;
}

long long round_up(long long v, long long m) { return (v + m - 1) / m * m; }

bool use_gen_table() {
  const char* v = std::getenv("MLE_GEN_TABLE");
  return !(v && std::strcmp(v, "0") == 0);
}

bool use_lookahead() {  // MLE_LOOKAHEAD=0: everything on the main stream (A/B timing)
  const char* v = std::getenv("MLE_LOOKAHEAD");
  return !(v && std::strcmp(v, "0") == 0);
}

// Slices of the solve sweep operands (X row panels, B column panels, W_b as the A operand):
// 7 by default (55-bit operands, 28 products), 6 with MLE_SOLVE_SLICES=6 (47-bit operands,
// 21 products).  6 slices stay within the north-star tolerances (1e-8 of the score's
// component scale) but move the score by ~1e-9 of that scale, which is enough to flip a
// Fisher-BT stopping decision that the reference takes 2% inside ||grad|| <= 1e-3 (config 2,
// seed 2); 7 slices are ~4x more accurate than DGEMM there.  A fixed setting,
// not a per-pass choice: results must not depend on batching or history.
int solve_slices() {
  const char* v = std::getenv("MLE_SOLVE_SLICES");
  return (v && std::strcmp(v, "6") == 0) ? 6 : 7;
}

// MLE_BOUNDARY_SPLIT=1: the Cholesky's outer boundaries with the chain-first split
// (boundary_split).  Off by default: bit-identical, but the batched config-2 loglik pass
// measured 3.25 ms with it against 3.19 ms without (the off-chain rest of the boundary then
// delays the block's last step and the next boundary's far update).
bool use_boundary_split() {
  const char* v = std::getenv("MLE_BOUNDARY_SPLIT");
  return v && std::strcmp(v, "1") == 0;
}

// MLE_INNER_DEEP=1: the inner steps' T2 split once more (T2a row k+3 on the inner stream,
// T2b on the edge stream).  Off by default: bit-identical, but the batched config-2 loglik
// pass measured 3.28 ms with it against 3.19 ms without (the bulk work it moves off the chain
// is then waited for at the outer boundary instead).
bool use_inner_deep() {
  const char* v = std::getenv("MLE_INNER_DEEP");
  return v && std::strcmp(v, "1") == 0;
}

bool use_speculation() {
  const char* v = std::getenv("MLE_SPECULATE");
  return !(v && std::strcmp(v, "0") == 0);
}

// Ozaki GEMM tile variant (launch_ozgemm n_tile; all bit-identical): MLE_OZ_TILE=0 (128 x 64
// tiles, CTA pairs sharing A), 1, 2, or 3 (128 x 32 tiles, clusters of four sharing A,
// double-buffered TMEM accumulators).
int oz_tile_variant() {
  static const int v = [] {
    const char* e = std::getenv("MLE_OZ_TILE");
    const int t = e ? std::atoi(e) : 0;
    return (t >= 0 && t <= 3) ? t : 0;
  }();
  return v;
}

// Solve formulation of eval_all (both give B_i = L^-1 S_i L^-T, lower half):
//   "w"  -- full forward sweep X = L^-1 S (n^3) + lower half of X L^-T (n^3 / 3);
//   "2s" -- two-sided blocked reduction (the sygst recurrence, 2 n^3 / 3 of syr2k-shaped
//           trailing updates) + the deferred forward sweep on the strictly lower block part
//           (n^3 / 3): n^3 per derivative block instead of 4 n^3 / 3.
// MLE_SOLVE=w|2s overrides; default "2s" from N >= kTwoSidedMinN (the recurrence's per-block
// chain is latency-bound on small matrices).
constexpr long long kTwoSidedMinN = 16384;
bool use_two_sided(long long N) {
  const char* e = std::getenv("MLE_SOLVE");
  if (e && std::strcmp(e, "2s") == 0) return true;
  if (e && std::strcmp(e, "w") == 0) return false;
  return N >= kTwoSidedMinN;
}

// FP64 trailing-update GEMM: Ozaki int8 tensor-core emulation (default) or DMMA.
bool use_ozaki();
bool use_ozaki() {
  const char* v = std::getenv("MLE_FP64_GEMM");
  return !(v && std::strcmp(v, "dmma") == 0);
}

}  // namespace

struct mle_ctx {
  int device = 0;
  int64_t n = 0;
  long long N = 0;   // padded extent (multiple of kNB), >= n + 1
  int Nt = 0;        // N / kNB
  double nugget = 0.0;
  cudaStream_t stream = nullptr;  // main stream (every call is serialised on it)
  cudaStream_t side = nullptr;    // look-ahead bulk trailing updates
  cudaStream_t inner = nullptr;   // inner (128-wide) look-ahead of the Cholesky
  cudaStream_t aux = nullptr;     // derivative generation concurrent with the Cholesky
  cudaStream_t edge = nullptr;    // the Cholesky's outer-boundary work off the chain
  cudaEvent_t pool[kPoolEvents] = {};
  double* lx = nullptr;
  double* ly = nullptr;
  double* z = nullptr;
  double* sigma = nullptr;
  double* sa = nullptr;
  double* sn = nullptr;
  double* smat = nullptr;         // nugget contexts: I_n -> M = L^-1 L^-T (third block)
  double h_max = 0.0;             // bounding-box diagonal of the locations (>= every distance)
  double* gtab_s = nullptr;       // generation tables: Sigma pass / derivative pass
  double* gtab_d = nullptr;
  double* linv = nullptr;
  int* fail_flag = nullptr;
  long long* fail_idx = nullptr;
  double* partials = nullptr;
  double* out = nullptr;          // device: 9 reduction results
  ThetaParams* d_theta = nullptr; // device copy of the per-theta scalars
  ThetaParams* h_theta = nullptr; // pinned staging
  // batch-leader staging: every item's ThetaParams (H2D once per pass) and every item's
  // results (D2H once per pass)
  ThetaParams* h_stage = nullptr;
  ThetaParams* d_stage = nullptr;
  double* h_resb = nullptr;
  double* d_resb = nullptr;
  double* h_res = nullptr;        // pinned: kReduceOut results + fail flag + fail idx
  cudaEvent_t ev[5] = {};
  cudaEvent_t ev_der = nullptr;   // derivative generation for this pass's eval_all items
  double phase_ms[MLE_NUM_PHASES] = {};
  double flops = 0.0;
  double gen_bytes = 0.0;
  double launches = 0.0;
  bool factor_valid = false;      // L of Sigma(cached_theta) is resident in `sigma`
  double cond_est = 0.0;          // (max / min diag L)^2 of the last factorization (0: none)
  double cached_theta[3] = {0, 0, 0};
  // Ozaki-scheme FP64 GEMM (ozaki.cu) for the K = 512 trailing updates.  The factor's outer
  // panels L[b1:, b0:b1] are sliced once during the Cholesky and kept with the factor (both
  // solve sweeps and the factor cache reuse them); the solve operands use a scratch.
  bool ozaki = true;              // MLE_FP64_GEMM=dmma at context creation disables it
  int8_t* lsl = nullptr;          // slices of every outer panel of L
  int* lex = nullptr;             // their row exponents
  int8_t* xsl = nullptr;          // solve-operand slices: 2 regions per derivative matrix
  int* xex = nullptr;
  // block-inverse solves: D_b^-1 per outer block (ld 512, zero upper), scratch, W_b slices
  double* dinv = nullptr;
  double* tscr = nullptr;
  double* wbuf = nullptr;
  int8_t* dtsl = nullptr;
  int* dtex = nullptr;
  int8_t* wsl = nullptr;
  int* wex = nullptr;
  int w_slices = 0;               // slice count of the resident W slices
  // two-sided reduction (solves_2s): per derivative matrix a 512 x 512 FP64 scratch and the
  // slices of its current diagonal block
  double* ts2 = nullptr;
  int8_t* a11sl = nullptr;
  int* a11ex = nullptr;
  bool deriv_lower = false;       // derivative matrices hold their lower tiles only (2s path)
  // Sequential-derivative mode (seq_derivs): the derivative blocks do not fit beside the
  // factor (config 5 on one B200), so eval_all reduces them one at a time in the single work
  // matrix `sa`, parks finished blocks in the unused upper triangles of `sigma` / `sa`
  // (both N x (N + kParkExtraCols)) and streams W_b block by block (one-block wsl).
  bool seq_derivs = false;
  // seq_derivs: the factor's panel slices (7 N^2 / 2 bytes: 35 GB at config 5) do not fit
  // beside the two arrays either.  During a factorizing pass `lsl` aliases the (then idle)
  // work matrix `sa`; the derivative phase overwrites it and re-slices each panel of L into
  // one of two slots right before the block that uses it.
  int8_t* psl = nullptr;          // 2 slots of (N x 512) panel slices
  int* pex = nullptr;             // their row exponents (2 x N)
  double cached_logdet = 0.0, cached_quad = 0.0;  // of the resident factor (with cached_ll)
  double cached_dmin = 0.0, cached_dmax = 0.0;
  // Kernel profiling (mle_kernel_profile): single stream, CUDA events around every Ozaki
  // GEMM and slicing launch of the pass; mle_kernel_stats reports the sums.
  bool kprof = false;
  std::vector<cudaEvent_t> kev;
  // Speculation: a loglik pass that factors Sigma(theta) also generates dSigma/dalpha,
  // dSigma/dnu and the W_b slices on the aux stream (overlapping the latency-bound
  // Cholesky), because Fisher-BT follows an accepted loglik(theta) with eval_all(theta).
  // spec_ready: sa / sn / wsl hold that work for spec_theta (valid while the factor is).
  PassClock pass_clock;           // led passes (diagnostic gap clock)
  double cached_ll = 0.0;         // log-likelihood of the resident factor (cached_theta)
  bool spec_ready = false;
  bool spec_pending = false;      // spec_done not yet waited for by a later pass
  double spec_theta[3] = {0, 0, 0};
  cudaEvent_t spec_done = nullptr;
  double kstats[MLE_KSTATS] = {};
  double host_wait_ms = 0.0;
};

namespace {

// One evaluation request inside a batch.
struct Item {
  mle_ctx* c = nullptr;
  ThetaParams P;
  int mode = 0;        // 1 loglik, 2 eval_all
  bool factor = true;  // generate Sigma + Cholesky (false: cached factor reused)
  bool derivs = false; // derivative matrices + solves
  bool gen_derivs = false;  // generate the derivative matrices in this pass
  bool need_w = false;      // compute the W_b slices in this pass
  bool spec = false;        // loglik item: speculative derivatives + W on the aux stream
  int rc = MLE_OK;
  int64_t pivot = -1;
  double res[kResults] = {};
};

// Derivative matrices generated for the two-sided solves: lower tiles only.
bool two_sided_gen(const mle_ctx* c) {
  return c->ozaki && solve_slices() == kOzSlices && use_two_sided(c->N);
}

// Pending speculative work (issued on some batch leader's aux stream) must finish before
// anything else touches this context's buffers.
int wait_spec(mle_ctx* c, cudaStream_t s) {
  if (c->spec_pending) {
    CUDA_TRY(cudaStreamWaitEvent(s, c->spec_done, 0));
    c->spec_pending = false;
  }
  return MLE_OK;
}

int ensure_ozaki(mle_ctx* c, bool derivs);

int ensure_matrices(mle_ctx* c, bool derivs) {
  const size_t cols = (size_t)c->N + (c->seq_derivs ? kParkExtraCols : 0);
  const size_t bytes = sizeof(double) * (size_t)c->N * cols;
  if (!c->sigma) CUDA_TRY(dmalloc(&c->sigma, bytes));
  if (!c->linv) CUDA_TRY(dmalloc(&c->linv, sizeof(double) * (size_t)c->Nt * kNB * kNB));
  if (c->seq_derivs && !c->sa) CUDA_TRY(dmalloc(&c->sa, bytes));  // also backs lsl
  if (derivs) {
    if (!c->sa) CUDA_TRY(dmalloc(&c->sa, bytes));
    if (!c->seq_derivs) {
      if (!c->sn) CUDA_TRY(dmalloc(&c->sn, bytes));
      if (c->nugget > 0.0 && !c->smat) CUDA_TRY(dmalloc(&c->smat, bytes));
    }
  }
  return ensure_ozaki(c, derivs);
}

// Outer panel ob of the factor: rows [b1, N) x columns [b0, b1), b1 = (ob + 1) kOuter.
long long oz_panel_rows(int Nt, int ob) {
  return (long long)std::max(0, Nt - std::min(Nt, (ob + 1) * kOuter)) * kNB;
}
long long oz_panel_row_offset(int Nt, int ob) {  // rows of the panels before ob
  long long r = 0;
  for (int o = 0; o < ob; ++o) r += oz_panel_rows(Nt, o);
  return r;
}
// W_b of outer block b: rows [c0, N) x kb; byte and row offsets of its slices.
long long w_row_offset(int Nt, int b) {
  long long r = 0;
  for (int o = 0; o < b; ++o) r += (long long)(Nt - o * kOuter) * kNB;
  return r;
}
size_t w_byte_offset(int Nt, int b) {
  size_t r = 0;
  for (int o = 0; o < b; ++o) {
    const long long kb = (long long)(std::min(Nt, (o + 1) * kOuter) - o * kOuter) * kNB;
    r += (size_t)(Nt - o * kOuter) * kNB * kb * kOzSlices;
  }
  return r;
}
constexpr int kOzK = kOuter * kNB;               // K of every trailing update
constexpr int kLookaheadCtas = 148 - 24;         // persistent grid of look-ahead updates
int far_ctas();
int lookahead_ctas() {  // MLE_LOOKAHEAD_CTAS: developer override (A/B timing)
  static const int v = [] {
    const char* e = std::getenv("MLE_LOOKAHEAD_CTAS");
    return e ? std::atoi(e) : kLookaheadCtas;
  }();
  return v;
}
// Grid cap of the Cholesky's far trailing update (ii-b), which runs under the next block's
// inner chain.  Uncapped (0: one CTA per SM): the far update is most of the factorization's
// work, and capping it to leave SMs to the chain measured slower (config 4: 1.22 s at 148
// CTAs, 1.28 s at 124, 1.47 s at 96; config 2 within noise).  MLE_FAR_CTAS overrides.
int far_ctas() {
  static const int v = [] {
    const char* e = std::getenv("MLE_FAR_CTAS");
    return e ? std::atoi(e) : 0;
  }();
  return v;
}
constexpr size_t kOzRowBytes = (size_t)kOzK * kOzSlices;
constexpr size_t kOzTileBytes = kOzRowBytes * kNB;

int ensure_ozaki(mle_ctx* c, bool derivs) {
  if (!c->ozaki) return MLE_OK;
  if (!c->lsl) {
    const long long rows = oz_panel_row_offset(c->Nt, (c->Nt + kOuter - 1) / kOuter);
    if (c->seq_derivs) {
      // 7 N^2 / 2 bytes of slices inside the 8 N (N + 513)-byte work matrix
      c->lsl = reinterpret_cast<int8_t*>(c->sa);
    } else {
      CUDA_TRY(dmalloc(&c->lsl, std::max<size_t>(1, (size_t)rows * kOzRowBytes)));
    }
    CUDA_TRY(dmalloc(&c->lex, sizeof(int) * std::max<long long>(1, rows)));
  }
  if (derivs && !c->xsl) {
    const int nb = (c->Nt + kOuter - 1) / kOuter;
    // 2 per derivative block (look-ahead); one block at a time in sequential mode
    const int regions = c->seq_derivs ? 2 : (c->nugget > 0.0 ? 6 : 4);
    CUDA_TRY(dmalloc(&c->xsl, regions * (size_t)c->N * kOzRowBytes));
    CUDA_TRY(dmalloc(&c->xex, regions * sizeof(int) * (size_t)c->N));
    CUDA_TRY(dmalloc(&c->dinv, sizeof(double) * (size_t)nb * 512 * 512));
    CUDA_TRY(dmalloc(&c->tscr, sizeof(double) * (size_t)nb * kNB * 512));
    CUDA_TRY(dmalloc(&c->wbuf, sizeof(double) * (size_t)c->N * 512));
    CUDA_TRY(dmalloc(&c->dtsl, (size_t)512 * kOzRowBytes));
    CUDA_TRY(dmalloc(&c->dtex, sizeof(int) * 512));
    const int mats = regions / 2;
    CUDA_TRY(dmalloc(&c->ts2, sizeof(double) * (size_t)mats * 512 * 512));
    CUDA_TRY(dmalloc(&c->a11sl, (size_t)mats * 512 * kOzRowBytes));
    CUDA_TRY(dmalloc(&c->a11ex, sizeof(int) * (size_t)mats * 512));
    if (c->seq_derivs) {  // W_b of one block at a time (block 0 is the largest: N rows)
      CUDA_TRY(dmalloc(&c->wsl, (size_t)c->N * kOzRowBytes));
      CUDA_TRY(dmalloc(&c->wex, sizeof(int) * (size_t)c->N));
      CUDA_TRY(dmalloc(&c->psl, 2 * (size_t)c->N * kOzRowBytes));
      CUDA_TRY(dmalloc(&c->pex, 2 * sizeof(int) * (size_t)c->N));
    } else {
      CUDA_TRY(dmalloc(&c->wsl, std::max<size_t>(1, w_byte_offset(c->Nt, nb))));
      CUDA_TRY(dmalloc(&c->wex, sizeof(int) * std::max<long long>(1, w_row_offset(c->Nt, nb))));
    }
    // the upper tiles of every D_b^-1 are never written and must read as exact zeros
    CUDA_TRY(cudaMemsetAsync(c->dinv, 0, sizeof(double) * (size_t)nb * 512 * 512, c->stream));
    CUDA_TRY(cudaStreamSynchronize(c->stream));
  }
  return MLE_OK;
}

GemmArgs gemm_base() {
  GemmArgs g;
  std::memset(&g, 0, sizeof(g));
  g.K = kNB;
  return g;
}

// Launch sequences over a list of contexts (all with the same N / Nt).
//
// Look-ahead: every sweep (Cholesky, forward solve, right solve) is a chain of latency-bound
// inner steps per outer block of kOuter tiles, followed by a large trailing GEMM.  The
// trailing GEMM of block b is split into
//   (i)  the part the next block's inner chain reads (its kOuter tiles)  -> main stream s
//   (ii) everything beyond                                               -> side stream s2
// so the inner chain of block b+1 runs on `s` while (ii) of block b runs on `s2`.  (i) of
// block b+1 touches tiles (ii) of block b also updates, so `s` waits for (ii)(b) first.
// The derivative blocks of a pass: (alpha, nu) per item, plus M for nugget items.
struct MatList {
  mle_ctx* c[kMaxGemm];
  int which[kMaxGemm];  // 0 S_alpha, 1 S_nu, 2 I_n -> M
  int slot[kMaxGemm];   // index of the block's scratch regions (xsl / ts2 / a11sl)
  int count = 0;
  MatList(mle_ctx* const* cs, int m) {
    for (int i = 0; i < m; ++i) {
      for (int w = 0; w < (cs[i]->smat ? 3 : 2); ++w) {
        c[count] = cs[i];
        slot[count] = w;
        which[count++] = w;
      }
    }
  }
  // sequential-derivative mode: the one block currently in the context's work matrix
  MatList(mle_ctx* ctx, int w) {
    c[0] = ctx;
    which[0] = w;
    slot[0] = 0;
    count = 1;
  }
  double* S(int z) const {
    if (c[z]->seq_derivs) return c[z]->sa;
    return which[z] == 0 ? c[z]->sa : which[z] == 1 ? c[z]->sn : c[z]->smat;
  }
};

// Process-wide count of kernels this library has launched (every Launcher adds its own count
// when it goes out of scope; mle_launch_count reads it).
std::atomic<long long> g_launch_total{0};

struct Launcher {
  ~Launcher() { g_launch_total.fetch_add((long long)launches); }
  cudaStream_t s;              // main: inner chains
  cudaStream_t s2 = nullptr;   // side: bulk trailing updates (null: everything on s)
  cudaEvent_t* pool = nullptr; // event pool for cross-stream joins
  int npool = 0;
  int next = 0;
  double launches = 0.0;

  // Timeline trace (MLE_TRACE=<file>, developer diagnostics): an event after every launch on
  // its own stream; after the pass, each launch's completion time from the pass start is
  // appended to the file as "pass label stream end_ms".
  struct Mark {
    cudaEvent_t ev;
    const char* label;
    int stream;
  };
  std::vector<Mark> marks;
  cudaEvent_t trace_t0 = nullptr;
  static const char* trace_path() {
    static const char* p = std::getenv("MLE_TRACE");
    return p;
  }
  int mark(const char* label, cudaStream_t st) {
    if (!trace_path()) return MLE_OK;
    Mark m{nullptr, label, st == s ? 0 : st == s2 ? 1 : st == s3 ? 2 : 3};
    CUDA_TRY(cudaEventCreate(&m.ev));
    CUDA_TRY(cudaEventRecord(m.ev, st));
    marks.push_back(m);
    return MLE_OK;
  }
  int trace_begin() {
    if (!trace_path()) return MLE_OK;
    CUDA_TRY(cudaEventCreate(&trace_t0));
    CUDA_TRY(cudaEventRecord(trace_t0, s));
    return MLE_OK;
  }
  int trace_end() {  // after the pass synchronized
    if (!trace_path() || !trace_t0) return MLE_OK;
    static long long pass = 0;
    FILE* f = std::fopen(trace_path(), "a");
    for (const Mark& m : marks) {
      float ms = 0.f;
      cudaEventElapsedTime(&ms, trace_t0, m.ev);
      if (f) std::fprintf(f, "%lld %s %d %.4f\n", pass, m.label, m.stream, ms);
      cudaEventDestroy(m.ev);
    }
    if (f) std::fclose(f);
    cudaEventDestroy(trace_t0);
    trace_t0 = nullptr;
    marks.clear();
    ++pass;
    return MLE_OK;
  }
  int gemm(const GemmArgs& g, BLayout bl, int batch, cudaStream_t st) {
    launches += 1;
    CUDA_TRY(launch_gemm(g, bl, batch, st));
    return mark(g.wide ? "dgemm128" : "dgemm64", st);
  }
  int gemm(const GemmArgs& g, BLayout bl, int batch) { return gemm(g, bl, batch, s); }
  int gemm_small(const GemmArgs& g, int batch, cudaStream_t st, int rows_only) {
    launches += 1;
    CUDA_TRY(launch_gemm_small(g, batch, st, rows_only));
    return mark(rows_only ? "small_panel" : "small_update", st);
  }
  // kernel profiling: event pair per launch (kind 0 ozgemm, 1 slicing) + algorithmic work
  mle_ctx* prof = nullptr;
  std::vector<int> pkind;
  std::vector<double> pwork;
  std::vector<double> pint8;  // int8 tensor ops of each GEMM launch
  int prof_begin(cudaStream_t st) {
    if (!prof) return MLE_OK;
    const size_t i = 2 * pkind.size();
    while (prof->kev.size() < i + 2) {
      cudaEvent_t e;
      CUDA_TRY(cudaEventCreate(&e));
      prof->kev.push_back(e);
    }
    CUDA_TRY(cudaEventRecord(prof->kev[i], st));
    return MLE_OK;
  }
  int prof_end(cudaStream_t st, int kind, double work, double int8_ops = 0.0) {
    if (!prof) return MLE_OK;
    CUDA_TRY(cudaEventRecord(prof->kev[2 * pkind.size() + 1], st));
    pkind.push_back(kind);
    pwork.push_back(work);
    pint8.push_back(int8_ops);
    return MLE_OK;
  }
  int slice(const OzSliceArgs& a, long long rows, bool row_contig, int batch,
            cudaStream_t st = nullptr) {
    if (!st) st = s;
    launches += 1;
    int rc = prof_begin(st);
    if (rc) return rc;
    CUDA_TRY(launch_oz_slice(a, (int)rows, row_contig, batch, st));
    if ((rc = mark("slice", st))) return rc;
    // algorithmic bytes: the FP64 operand read once, S int8 slices + exponents written
    return prof_end(st, 1, (double)batch * rows * ((8.0 + oz_nslices(a.nslices)) * a.K + 4.0));
  }
  int ozgemm(const OzGemmArgs& g, int batch, cudaStream_t st) {
    launches += 1;
    int rc = prof_begin(st);
    if (rc) return rc;
    CUDA_TRY(launch_ozgemm(g, batch, st, oz_tile_variant()));
    if ((rc = mark("ozgemm", st))) return rc;
    double tiles;
    if (g.lower) tiles = 0.5 * g.tiles_m * (g.tiles_m + 1.0);
    else if (g.trap) {
      tiles = 0;
      for (int tn = 0; tn < g.tiles_n; ++tn) tiles += std::max(0, g.tiles_m - tn);
    } else tiles = (double)g.tiles_m * g.tiles_n;
    // FP64-equivalent tile flops (2 x 128 x 128 x K per tile); int8 tensor ops: one slice
    // product per pair (p, q) with p + q <= S + 1 (28 for 7 slices, 21 for 6)
    const double fl = (double)batch * tiles * 2.0 * kNB * kNB * (32.0 * g.kblocks);
    return prof_end(st, 0, fl, fl * oz_products(g.nslices));
  }
  int prof_collect() {
    if (!prof) return MLE_OK;
    double st[MLE_KSTATS] = {};
    for (size_t i = 0; i < pkind.size(); ++i) {
      float ms = 0.f;
      CUDA_TRY(cudaEventElapsedTime(&ms, prof->kev[2 * i], prof->kev[2 * i + 1]));
      const int base = pkind[i] == 0 ? 0 : pkind[i] == 1 ? 4 : 10;
      st[base] += 1.0;
      st[base + 1] += ms;
      st[base + 2] += pwork[i];
      if (pkind[i] == 0) st[3] += pint8[i];
    }
    std::memcpy(prof->kstats, st, sizeof(st));
    return MLE_OK;
  }
  // Grid cap of the solve sweeps' GEMMs (MLE_SOLVE_CTAS, 0: every SM): SMs left free let a
  // concurrent pass's latency-bound Cholesky chain (another fit group) start its kernels.
  static int solve_ctas() {
    static const int v = [] {
      const char* e = std::getenv("MLE_SOLVE_CTAS");
      return e ? std::atoi(e) : 0;
    }();
    return v;
  }
  static OzGemmArgs oz_base(long long ldc, int tiles_m, int tiles_n) {
    OzGemmArgs g;
    std::memset(&g, 0, sizeof(g));
    g.ldc = ldc;
    g.kblocks = kOzK / 32;
    g.tiles_m = tiles_m;
    g.tiles_n = tiles_n;
    g.alpha = -1.0;
    g.beta = 1.0;
    return g;
  }

  // `to` waits for all work enqueued so far on `from`.
  int join(cudaStream_t from, cudaStream_t to) {
    if (from == to || from == nullptr || to == nullptr) return MLE_OK;
    // reserved: pool[npool - 1] ev_near (potrf), pool[npool - 2] ev_t1 (inner_block),
    // pool[npool - 3] ev_rest (boundary_split), pool[npool - 4] ev_t2b (inner_block)
    cudaEvent_t e = pool[next++ % (npool - 4)];
    CUDA_TRY(cudaEventRecord(e, from));
    CUDA_TRY(cudaStreamWaitEvent(to, e, 0));
    return MLE_OK;
  }
  cudaStream_t bulk() const { return s2 ? s2 : s; }
  cudaStream_t s3 = nullptr;   // inner look-ahead of the Cholesky (null: on s)
  bool outer_on_inner = false;  // (i1) of the last outer update was issued on s3
  bool near_pending = false;    // (ii-a) of the last outer update recorded ev_near on s2
  bool t1_pending = false;      // the last inner step's (T1) recorded ev_t1 on s3
  // potrf (Ozaki path): the block's last inner step computes only the panel's head rows (the
  // next block's first two row tiles) on the chain; potrf issues the rest on the inner stream
  bool split_last = false;
  cudaStream_t s4 = nullptr;    // edge stream: boundary_split's rest or the inner T2b
  bool t2b_pending = false;     // the last inner step's T2b recorded ev_t2b on s4
  bool split_last_any = false;  // boundary_split in use this pass (it owns s4)
  bool rest_pending = false;    // boundary_split recorded ev_rest on s4: T2 waits for it
  cudaStream_t inner() const { return s3 ? s3 : s; }
  // W request of the Cholesky: build W_b of these contexts on stream ws as each outer block
  // of the factor becomes final (Ozaki path only).
  mle_ctx* const* wreq = nullptr;
  int nwreq = 0;
  int wks = 0;
  cudaStream_t ws = nullptr;
  int issue_w(int b, cudaStream_t after = nullptr) {
    if (nwreq == 0) return MLE_OK;
    int rc = join(after ? after : s, ws);
    if (rc) return rc;
    const cudaStream_t keep = s;
    s = ws;
    rc = compute_w_block(wreq, nwreq, wks, b);
    s = keep;
    return rc;
  }

  // Two-level right-looking blocked Cholesky of every item's matrix (ld = N).
  // Inner (128-wide) steps of outer block [b0, b1): diagonal tiles, panels and the updates
  // inside the block; leaves L[:, b0:b1] final (all rows).  mats[] may be "virtual" base
  // pointers of column panels (element (i, j) at mats[b][i + j ld] for j in the block).
  int inner_block(mle_ctx* const* cs, double* const* mats, const long long* n_aug, int m,
                  int b0, int b1) {
    const long long ld = cs[0]->N;
    const int Nt = cs[0]->Nt;
    int rc;
    for (int k = b0; k < b1; ++k) {
      const long long k0 = (long long)k * kNB;
      DiagArgs d;
      std::memset(&d, 0, sizeof(d));
      d.ld = ld;
      d.k0 = (int)k0;
      for (int b = 0; b < m; ++b) {
        d.a[b] = mats[b];
        d.linv[b] = cs[b]->linv + (size_t)k * kNB * kNB;
        d.fail_flag[b] = cs[b]->fail_flag;
        d.fail_idx[b] = cs[b]->fail_idx;
        d.n_aug[b] = n_aug[b];
      }
      launches += 1;
      CUDA_TRY(launch_potrf_diag(d, m, s));
      if ((rc = mark("diag", s))) return rc;
      const int rem = Nt - k - 1;
      if (rem == 0) break;
      const int wcols = b1 - k - 1;  // remaining tile columns of this outer block
      auto panel_gemm = [&](int row_tiles, int row_off, cudaStream_t st, bool small = false) {
        // panel rows [k+1+row_off, k+1+row_off+row_tiles) <- panel * Linv_k^T, in place
        // (BN = 128 covers the whole panel width)
        GemmArgs g = gemm_base();
        for (int b = 0; b < m; ++b) {
          double* panel = mats[b] + (k0 + kNB + (long long)row_off * kNB) + k0 * ld;
          g.A[b] = panel;
          g.B[b] = cs[b]->linv + (size_t)k * kNB * kNB;
          g.C[b] = panel;
          g.fail_flag[b] = cs[b]->fail_flag;
        }
        g.lda = ld; g.ldb = kNB; g.ldc = ld;
        g.tiles_m = row_tiles; g.tiles_n = 1; g.alpha = 1.0; g.beta = 0.0; g.wide = 1;
        return small ? gemm_small(g, m, st, 1) : gemm(g, kBNK, m, st);
      };
      // A[r0+.., c0+..] -= P[r0..] P[c0..]^T over tile rows/cols of this outer block
      auto update = [&](int row_off, int row_tiles, int col_off, int col_tiles, bool trap,
                        cudaStream_t st, bool small = false, int trap_off = 0) {
        GemmArgs t = gemm_base();
        for (int b = 0; b < m; ++b) {
          double* panel = mats[b] + (k0 + kNB) + k0 * ld;
          t.A[b] = panel + (long long)row_off * kNB;
          t.B[b] = panel + (long long)col_off * kNB;
          t.C[b] = mats[b] + (k0 + kNB + (long long)row_off * kNB) +
                   (k0 + kNB + (long long)col_off * kNB) * ld;
          t.fail_flag[b] = cs[b]->fail_flag;
        }
        t.lda = ld; t.ldb = ld; t.ldc = ld;
        t.tiles_m = row_tiles; t.tiles_n = col_tiles; t.trap = trap ? 1 : 0;
        t.trap_off = trap_off;
        t.alpha = -1.0; t.beta = 1.0;
        return small ? gemm_small(t, m, st, 0) : gemm(t, kBNK, m, st);
      };
      // What this step reads from the previous step's inner-stream work: only (T1), the
      // panel row and the two tiles the chain needs next (ev_t1); at a block's first step the
      // inner stream holds only the last outer update's far columns, which it does not read.
      // The whole panel of the block's last step is read by the trailing update: all of it.
      if (k == b0 && outer_on_inner) {
        outer_on_inner = false;
        t1_pending = false;
      } else if (t1_pending && wcols > 0) {
        CUDA_TRY(cudaStreamWaitEvent(s, pool[npool - 2], 0));
        t1_pending = false;
      } else {
        t1_pending = false;
        if (t2b_pending) {  // the inner stream catches up with the edge stream first
          CUDA_TRY(cudaStreamWaitEvent(s3 ? s3 : s, pool[npool - 4], 0));
          t2b_pending = false;
        }
        if ((rc = join(s3, s))) return rc;
      }
      if (wcols == 0) {
        // last tile of the outer block: the whole panel (read by the trailing update); with
        // split_last only its head rows here (potrf issues the rest off the chain)
        if (split_last && s3 && s4 && rem > 3) {
          if ((rc = panel_gemm(3, 0, s, true))) return rc;
        } else if ((rc = panel_gemm(rem, 0, s))) {
          return rc;
        }
        continue;
      }
      // Inner look-ahead: the critical chain to the next diagonal tile is only
      //   panel rows of tile k+1  ->  update of tile (k+1, k+1)  ->  diag(k+1);
      // the other panel rows and updates run on the inner stream meanwhile.
      // the chain's two single-tile products on small-tile CTAs (8-16 SMs per dataset)
      if ((rc = panel_gemm(1, 0, s, true))) return rc;
      if ((rc = join(s, s3))) return rc;
      if ((rc = update(0, 1, 0, 1, true, s, true))) return rc;
      if (rem > 1) {
        cudaStream_t in = inner();
        // (T1) what the next step's chain reads: panel row k+2 and its update of tiles
        // (k+2, k+1) and (k+2, k+2) (within the block), on small-tile CTAs, then ev_t1
        if ((rc = panel_gemm(1, 1, in, true))) return rc;
        if ((rc = update(1, 1, 0, std::min(2, wcols), false, in, true))) return rc;
        if (in != s) {
          CUDA_TRY(cudaEventRecord(pool[npool - 2], in));
          t1_pending = true;
        }
        if (rest_pending) {  // T2 reads rows the boundary's rest (on s4) updates
          CUDA_TRY(cudaStreamWaitEvent(in, pool[npool - 3], 0));
          rest_pending = false;
        }
        // (T2) the rest: panel rows >= k+3 and their update of the block's remaining columns.
        // Same per-tile arithmetic as one launch: the small and large DMMA kernels use the
        // same k order (bit-identical results).  With the edge stream and the boundary split
        // off, T2 is split once more so that the next step's T1 (behind it on the inner
        // stream) waits only for row k+3:
        //   (T2a) panel row k+3 and its tiles, inner stream, after the previous step's T2b;
        //   (T2b) rows >= k+4, edge stream (ev_t2b): the chain is two steps ahead of it.
        const bool deep = s4 && !split_last_any && in != s && use_inner_deep();
        if (rem > 2 && deep) {
          if (t2b_pending) {
            CUDA_TRY(cudaStreamWaitEvent(in, pool[npool - 4], 0));
            t2b_pending = false;
          }
          if ((rc = panel_gemm(1, 2, in, true))) return rc;
          if ((rc = update(2, 1, 0, std::min(3, wcols), false, in, true))) return rc;
          if (rem > 3) {
            if ((rc = join(in, s4))) return rc;
            if ((rc = panel_gemm(rem - 3, 3, s4))) return rc;
            if ((rc = update(3, rem - 3, 0, wcols, true, s4, false, 3))) return rc;
            CUDA_TRY(cudaEventRecord(pool[npool - 4], s4));
            t2b_pending = true;
          }
        } else if (rem > 2) {
          if (t2b_pending) {
            CUDA_TRY(cudaStreamWaitEvent(in, pool[npool - 4], 0));
            t2b_pending = false;
          }
          if ((rc = panel_gemm(rem - 2, 2, in))) return rc;
          if ((rc = update(2, rem - 2, 0, wcols, true, in, false, 2))) return rc;
        }
      }
    }
    t1_pending = false;
    if (t2b_pending) {  // everything of the block is in L[:, b0:b1] for the caller
      CUDA_TRY(cudaStreamWaitEvent(s3 ? s3 : s, pool[npool - 4], 0));
      t2b_pending = false;
    }
    return join(s3, s);
  }

  // Outer-block boundary with the next block's chain first (Ozaki path, inner and edge
  // streams present, more than three row tiles below).  The next block's first inner step
  // (its chain and its T1) reads only the trailing update's head: tiles rows [b1, b1+3) x
  // columns [b1, b1+3) (lower), which need only the panel's three head row tiles:
  //   main:  [head panel rows (inner_block)] -> slice them -> wait ev_near -> (i0h) the six
  //          head tiles, K = 512 -> the next block's inner chain starts;
  //   edge:  the rest of the panel (rows >= b1+3) -> slice it -> W_b -> (i0r) / (i1r):
  //          rows >= b1+3 of the next block's columns -> ev_rest (the first inner step's T2
  //          waits for it) -> (ii-a) / (ii-b) go to the side stream after it.
  // Every tile sees the same updates in the same order as the unsplit boundary (bit-identical,
  // tools/boundary_ab.py).
  int boundary_split(mle_ctx* const* cs, double* const* mats, int m, int b0, int b1, int b2) {
    const long long ld = cs[0]->N;
    const int Nt = cs[0]->Nt;
    const int ob = b0 / kOuter;
    const long long eo = oz_panel_row_offset(Nt, ob);
    const long long c0 = (long long)b0 * kNB, t0 = (long long)b1 * kNB;
    constexpr int hr = 3;                      // head row tiles
    const int hc = std::min(hr, b2 - b1);      // head columns (within the next block)
    int rc;
    OzSliceArgs sa;
    std::memset(&sa, 0, sizeof(sa));
    for (int b = 0; b < m; ++b) {
      sa.X[b] = mats[b] + t0 + c0 * ld;
      sa.slices[b] = cs[b]->lsl + (size_t)eo * kOzRowBytes;
      sa.e[b] = cs[b]->lex + eo;
      sa.fail_flag[b] = cs[b]->fail_flag;
    }
    sa.ld = ld;
    sa.K = kOzK;
    if ((rc = slice(sa, (long long)hr * kNB, true, m, s))) return rc;
    if (near_pending && s2) {
      CUDA_TRY(cudaStreamWaitEvent(s, pool[npool - 1], 0));
      near_pending = false;
    } else if ((rc = join(s2, s))) {
      return rc;
    }
    {  // (i0h): rows [b1, b1 + hr) x columns [b1, b1 + hc), lower
      OzGemmArgs t = oz_base(ld, hr, hc);
      t.trap = 1;
      for (int b = 0; b < m; ++b) {
        t.As[b] = t.Bs[b] = sa.slices[b];
        t.ea[b] = t.eb[b] = sa.e[b];
        t.C[b] = mats[b] + t0 + t0 * ld;
        t.fail_flag[b] = cs[b]->fail_flag;
      }
      if ((rc = ozgemm(t, m, s))) return rc;
    }
    if ((rc = join(s, s4))) return rc;
    {  // the rest of the last column's panel (rows >= b1 + hr), in place
      const int k = b1 - 1;
      const long long k0 = (long long)k * kNB;
      GemmArgs g = gemm_base();
      for (int b = 0; b < m; ++b) {
        double* panel = mats[b] + (t0 + (long long)hr * kNB) + k0 * ld;
        g.A[b] = panel;
        g.B[b] = cs[b]->linv + (size_t)k * kNB * kNB;
        g.C[b] = panel;
        g.fail_flag[b] = cs[b]->fail_flag;
      }
      g.lda = ld; g.ldb = kNB; g.ldc = ld;
      g.tiles_m = Nt - b1 - hr; g.tiles_n = 1; g.alpha = 1.0; g.beta = 0.0; g.wide = 1;
      if ((rc = gemm(g, kBNK, m, s4))) return rc;
    }
    OzSliceArgs sr = sa;
    for (int b = 0; b < m; ++b) {
      sr.X[b] = sa.X[b] + (long long)hr * kNB;
      sr.slices[b] = sa.slices[b] + (size_t)hr * kOzTileBytes;
      sr.e[b] = sa.e[b] + (long long)hr * kNB;
    }
    if ((rc = slice(sr, (long long)(Nt - b1 - hr) * kNB, true, m, s4))) return rc;
    if ((rc = issue_w(ob, s4))) return rc;
    {  // (i0r) + (i1r): rows >= b1 + hr of all the next block's columns (none above the
       // diagonal: the columns end at b1 + 4 <= b1 + hr + 1)
      OzGemmArgs t = oz_base(ld, Nt - b1 - hr, b2 - b1);
      for (int b = 0; b < m; ++b) {
        t.As[b] = sr.slices[b];
        t.ea[b] = sr.e[b];
        t.Bs[b] = sa.slices[b];
        t.eb[b] = sa.e[b];
        t.C[b] = mats[b] + (t0 + (long long)hr * kNB) + t0 * ld;
        t.fail_flag[b] = cs[b]->fail_flag;
      }
      if ((rc = ozgemm(t, m, s4))) return rc;
    }
    CUDA_TRY(cudaEventRecord(pool[npool - 3], s4));
    rest_pending = true;
    outer_on_inner = true;  // the next block's first step must not wait for the inner stream
    if (b2 >= Nt) return MLE_OK;
    if ((rc = join(s4, s2))) return rc;  // (ii) reads the whole panel's slices
    const long long u0 = (long long)b2 * kNB;
    const int b3 = std::min(Nt, b2 + kOuter);
    OzGemmArgs ua = oz_base(ld, Nt - b2, b3 - b2);  // (ii-a)
    ua.trap = 1;
    ua.max_ctas = lookahead_ctas();
    for (int b = 0; b < m; ++b) {
      ua.As[b] = ua.Bs[b] = sa.slices[b] + (size_t)(b2 - b1) * kOzTileBytes;
      ua.ea[b] = ua.eb[b] = sa.e[b] + (size_t)(b2 - b1) * kNB;
      ua.C[b] = mats[b] + u0 + u0 * ld;
      ua.fail_flag[b] = cs[b]->fail_flag;
    }
    if ((rc = ozgemm(ua, m, bulk()))) return rc;
    CUDA_TRY(cudaEventRecord(pool[npool - 1], s2));
    near_pending = true;
    if (b3 >= Nt) return MLE_OK;
    OzGemmArgs u = oz_base(ld, Nt - b3, 0);  // (ii-b)
    u.lower = 1;
    u.max_ctas = far_ctas();
    const long long u3 = (long long)b3 * kNB;
    for (int b = 0; b < m; ++b) {
      u.As[b] = u.Bs[b] = sa.slices[b] + (size_t)(b3 - b1) * kOzTileBytes;
      u.ea[b] = u.eb[b] = sa.e[b] + (size_t)(b3 - b1) * kNB;
      u.C[b] = mats[b] + u3 + u3 * ld;
      u.fail_flag[b] = cs[b]->fail_flag;
    }
    return ozgemm(u, m, bulk());
  }

  int potrf(mle_ctx* const* cs, double* const* mats, const long long* n_aug, int m) {
    const long long ld = cs[0]->N;
    const int Nt = cs[0]->Nt;
    int rc;
    for (int b0 = 0; b0 < Nt; b0 += kOuter) {
      const int b1 = std::min(Nt, b0 + kOuter);
      split_last = cs[0]->lsl && s3 && s2 && s4 && Nt - b1 > 3 && use_boundary_split();
      split_last_any = use_boundary_split();
      if ((rc = inner_block(cs, mats, n_aug, m, b0, b1))) return rc;
      const bool split = split_last;
      split_last = false;
      if (b1 >= Nt) {
        if ((rc = issue_w(b0 / kOuter))) return rc;
        continue;
      }
      // trailing update with P = L[T, b0:b1], K = (b1 - b0) * 128
      const int b2 = std::min(Nt, b1 + kOuter);
      const long long c0 = (long long)b0 * kNB, t0 = (long long)b1 * kNB, u0 = (long long)b2 * kNB;
      if (!cs[0]->lsl && (rc = join(s2, s))) return rc;  // (ii) of the previous block
      if (split) {
        if ((rc = boundary_split(cs, mats, m, b0, b1, b2))) return rc;
        continue;
      }
      if (cs[0]->lsl) {
        // Ozaki path: slice P = L[b1:, b0:b1] once (kept for the solves), then C -= P P^T
        const int ob = b0 / kOuter;
        const long long eo = oz_panel_row_offset(Nt, ob);
        OzSliceArgs sa;
        std::memset(&sa, 0, sizeof(sa));
        for (int b = 0; b < m; ++b) {
          sa.X[b] = mats[b] + t0 + c0 * ld;
          sa.slices[b] = cs[b]->lsl + (size_t)eo * kOzRowBytes;
          sa.e[b] = cs[b]->lex + eo;
          sa.fail_flag[b] = cs[b]->fail_flag;
        }
        sa.ld = ld;
        sa.K = kOzK;
        if ((rc = slice(sa, (long long)(Nt - b1) * kNB, true, m))) return rc;
        if ((rc = issue_w(ob))) return rc;
        // (i) updates the next block's columns, which the previous block's (ii-a) updated
        // too: wait for that part only (ev_near), not for the whole far update (ii-b)
        if (near_pending && s2) {
          CUDA_TRY(cudaStreamWaitEvent(s, pool[npool - 1], 0));
          near_pending = false;
        } else if ((rc = join(s2, s))) {
          return rc;
        }
        // (i) in two parts: the next block's first two tile columns on the main stream (its
        // first inner step reads only those), the other two on the inner stream, where that
        // step's own inner-stream work follows them in order
        const int i0 = (s3 && b2 - b1 > 2) ? 2 : b2 - b1;
        if (i0 < b2 - b1 && (rc = join(s, s3))) return rc;
        OzGemmArgs t = oz_base(ld, Nt - b1, i0);  // (i0)
        t.trap = 1;
        for (int b = 0; b < m; ++b) {
          t.As[b] = t.Bs[b] = sa.slices[b];
          t.ea[b] = t.eb[b] = sa.e[b];
          t.C[b] = mats[b] + t0 + t0 * ld;
          t.fail_flag[b] = cs[b]->fail_flag;
        }
        if ((rc = ozgemm(t, m, s))) return rc;
        if (i0 < b2 - b1) {
          OzGemmArgs t1 = oz_base(ld, Nt - b1 - i0, b2 - b1 - i0);  // (i1)
          t1.trap = 1;
          const long long o1 = t0 + (long long)i0 * kNB;
          for (int b = 0; b < m; ++b) {
            t1.As[b] = t1.Bs[b] = sa.slices[b] + (size_t)i0 * kOzTileBytes;
            t1.ea[b] = t1.eb[b] = sa.e[b] + (size_t)i0 * kNB;
            t1.C[b] = mats[b] + o1 + o1 * ld;
            t1.fail_flag[b] = cs[b]->fail_flag;
          }
          if ((rc = ozgemm(t1, m, s3))) return rc;
          outer_on_inner = true;  // the next block's first step must not wait for it
        }
        if (b2 >= Nt) continue;
        if ((rc = join(s, s2))) return rc;
        // (ii) in two parts on the side stream: (ii-a) the block after next's columns
        // [b2, b3) -- all that block's (i) will wait for (ev_near) -- then (ii-b) the lower
        // tiles of [b3, Nt).  Every tile sees the same sequence of updates as one launch.
        const int b3 = std::min(Nt, b2 + kOuter);
        OzGemmArgs ua = oz_base(ld, Nt - b2, b3 - b2);  // (ii-a)
        ua.trap = 1;
        ua.max_ctas = lookahead_ctas();  // the next block's diagonal chain runs meanwhile
        for (int b = 0; b < m; ++b) {
          ua.As[b] = ua.Bs[b] = sa.slices[b] + (size_t)(b2 - b1) * kOzTileBytes;
          ua.ea[b] = ua.eb[b] = sa.e[b] + (size_t)(b2 - b1) * kNB;
          ua.C[b] = mats[b] + u0 + u0 * ld;
          ua.fail_flag[b] = cs[b]->fail_flag;
        }
        if ((rc = ozgemm(ua, m, bulk()))) return rc;
        if (s2) {
          CUDA_TRY(cudaEventRecord(pool[npool - 1], s2));
          near_pending = true;
        }
        if (b3 >= Nt) continue;
        OzGemmArgs u = oz_base(ld, Nt - b3, 0);        // (ii-b)
        u.lower = 1;
        u.max_ctas = far_ctas();
        const long long u3 = (long long)b3 * kNB;
        for (int b = 0; b < m; ++b) {
          u.As[b] = u.Bs[b] = sa.slices[b] + (size_t)(b3 - b1) * kOzTileBytes;
          u.ea[b] = u.eb[b] = sa.e[b] + (size_t)(b3 - b1) * kNB;
          u.C[b] = mats[b] + u3 + u3 * ld;
          u.fail_flag[b] = cs[b]->fail_flag;
        }
        if ((rc = ozgemm(u, m, bulk()))) return rc;
        continue;
      }
      GemmArgs t = gemm_base();           // (i): columns [b1, b2), rows >= b1
      for (int b = 0; b < m; ++b) {
        t.A[b] = mats[b] + t0 + c0 * ld;
        t.B[b] = mats[b] + t0 + c0 * ld;
        t.C[b] = mats[b] + t0 + t0 * ld;
        t.fail_flag[b] = cs[b]->fail_flag;
      }
      t.lda = ld; t.ldb = ld; t.ldc = ld;
      t.K = (b1 - b0) * kNB;
      t.tiles_m = Nt - b1; t.tiles_n = b2 - b1; t.trap = 1; t.alpha = -1.0; t.beta = 1.0;
      if ((rc = gemm(t, kBNK, m))) return rc;
      if (b2 >= Nt) continue;
      if ((rc = join(s, s2))) return rc;
      GemmArgs u = gemm_base();           // (ii): lower tiles of [b2, Nt)
      for (int b = 0; b < m; ++b) {
        u.A[b] = mats[b] + u0 + c0 * ld;
        u.B[b] = mats[b] + u0 + c0 * ld;
        u.C[b] = mats[b] + u0 + u0 * ld;
        u.fail_flag[b] = cs[b]->fail_flag;
      }
      u.lda = ld; u.ldb = ld; u.ldc = ld;
      u.K = (b1 - b0) * kNB;
      u.tiles_m = Nt - b2; u.lower = 1; u.alpha = -1.0; u.beta = 1.0;
      if ((rc = gemm(u, kBNK, m, bulk()))) return rc;
    }
    return join(s2, s);
  }

  // B_i = L^-1 S_i L^-T (lower half) for both derivative matrices of every item, in place.
  // GEMM batch member z = 2 * item + {0: alpha, 1: nu}.
  int solves(mle_ctx* const* cs, int m, mle_ctx* const* cw, int mw) {
    if (cs[0]->wsl) {
      const int ks = solve_slices();
      // W slices to (re)build: the requested ones, plus resident ones of another count
      mle_ctx* rw[kMaxItems];
      int nw = 0;
      for (int i = 0; i < m; ++i) {
        bool need = cs[i]->w_slices != ks;
        for (int j = 0; j < mw; ++j) need = need || cw[j] == cs[i];
        if (need) rw[nw++] = cs[i];
      }
      if (nw > 0) {
        int rc = compute_w(rw, nw, ks);
        if (rc) return rc;
      }
      // lower-only derivative matrices can only take the two-sided path
      bool two = ks == kOzSlices && use_two_sided(cs[0]->N);
      for (int i = 0; i < m; ++i) two = two || cs[i]->deriv_lower;
      if (two) return solves_2s(cs, m);
      return solves_w(cs, m, ks);
    }
    return solves_dmma(cs, m);
  }

  // ---- block-inverse formulation on the Ozaki GEMM ----------------------------------
  // For outer block b (tiles [t0, t1), columns [c0, c1), kb = c1 - c0) with diagonal block
  // D_b = L[c0:c1, c0:c1] and panel P_b = L[c1:, c0:c1], let
  //     W_b = [ D_b^-1 ; -P_b D_b^-1 ]            (rows c0 .. N, kb columns).
  // Forward sweep X = L^-1 S, block b:  X[c0:, :] = W_b X[c0:c1, :] with the top kb rows
  //   overwritten (D_b^-1 S_b) and the rows below accumulated (-P_b D_b^-1 S_b).
  // Right sweep B = X L^-T (lower half), block b:  X[i, c0:] += X[i, c0:c1] W_b^T, the
  //   first kb columns overwritten (X D_b^-T = B[:, b]) and later columns accumulated
  //   (-B[:, b] P_b^T).
  // Each block of each sweep is one slicing + one Ozaki GEMM (split (i)/(ii) for look-ahead);
  // the 128-wide DMMA inner steps disappear.
  struct Blk {
    int t0, t1;
    long long c0, kb;
  };
  static Blk blk(int Nt, int b) {
    Blk o;
    o.t0 = b * kOuter;
    o.t1 = std::min(Nt, o.t0 + kOuter);
    o.c0 = (long long)o.t0 * kNB;
    o.kb = (long long)(o.t1 - o.t0) * kNB;
    return o;
  }

  // D_b^-1 for every outer block (DMMA, from the Linv tiles) and the slices of W_b.
  int compute_w(mle_ctx* const* cs, int m, int ks) {
    const int nb = (cs[0]->Nt + kOuter - 1) / kOuter;
    for (int b = 0; b < nb; ++b) {
      int rc = compute_w_block(cs, m, ks, b);
      if (rc) return rc;
    }
    return MLE_OK;
  }

  // W_b of one outer block: needs only L[c0:, c0:c1] (final once block b is factored) and
  // its Linv tiles, so the Cholesky issues it block by block (potrf's W request) and the
  // W_b chain runs under the rest of the factorization instead of after it.
  // seq_derivs: the slices of panel P_b = L[c1:, c0:c1] are not resident (mle_ctx::psl): they
  // are cut again from L into slot b & 1 on the main stream.  Two slots: the side stream's
  // far update of block b still reads slot b & 1 while block b + 1 fills the other; block
  // b + 2 refills it after the main stream joined the side stream in block b + 1's step (4).
  static const int8_t* panel_slices(const mle_ctx* c, int b, long long eo) {
    return c->seq_derivs ? c->psl + (size_t)(b & 1) * c->N * kOzRowBytes
                         : c->lsl + (size_t)eo * kOzRowBytes;
  }
  static const int* panel_exps(const mle_ctx* c, int b, long long eo) {
    return c->seq_derivs ? c->pex + (size_t)(b & 1) * c->N : c->lex + eo;
  }
  int slice_panel_slot(mle_ctx* c, int b) {
    const Blk k = blk(c->Nt, b);
    const long long ld = c->N, c1 = k.c0 + k.kb;
    if (c1 >= ld) return MLE_OK;
    OzSliceArgs sa;
    std::memset(&sa, 0, sizeof(sa));
    sa.X[0] = c->sigma + c1 + k.c0 * ld;
    sa.slices[0] = c->psl + (size_t)(b & 1) * ld * kOzRowBytes;
    sa.e[0] = c->pex + (size_t)(b & 1) * ld;
    sa.fail_flag[0] = c->fail_flag;
    sa.ld = ld;
    sa.K = kOzK;
    return slice(sa, ld - c1, true, 1);
  }

  int compute_w_block(mle_ctx* const* cs, int m, int ks, int b) {
    const long long ld = cs[0]->N;
    const bool one_slot = cs[0]->seq_derivs;  // W_b streamed through a one-block buffer
    if (one_slot) {
      int rc0 = slice_panel_slot(cs[0], b);
      if (rc0) return rc0;
    }
    const int Nt = cs[0]->Nt;
    for (int i = 0; i < m; ++i) cs[i]->w_slices = ks;
    int rc;
    const Blk k = blk(Nt, b);
    {
      double* dv[kMaxItems];
      const double* lv[kMaxItems];
      for (int it = 0; it < m; ++it) {
        dv[it] = cs[it]->dinv + (size_t)b * 512 * 512;
        lv[it] = cs[it]->linv;
      }
      launches += 1;
      CUDA_TRY(launch_linv_to_dinv_block(dv, lv, k.t0, k.t1 - k.t0, m, s));
    }
    // tile row i of the block:  T = L[i, 0:i] Dinv[0:i, 0:i];  Dinv[i, 0:i] = -Linv_i T
    for (int i = 1; i < k.t1 - k.t0; ++i) {
      GemmArgs t = gemm_base(), u = gemm_base();
      for (int it = 0; it < m; ++it) {
        double* dinv_b = cs[it]->dinv + (size_t)b * 512 * 512;
        double* T = cs[it]->tscr + (size_t)b * kNB * 512;
        t.A[it] = cs[it]->sigma + (k.c0 + i * kNB) + k.c0 * ld;  // 128 x 128 i, lda = N
        t.B[it] = dinv_b;  // B(n, k) = Dinv(k, n)  (kBKN, ldb 512)
        t.C[it] = T;
        t.fail_flag[it] = cs[it]->fail_flag;
        u.A[it] = cs[it]->linv + (size_t)(k.t0 + i) * kNB * kNB;  // Linv_i (128 x 128)
        u.B[it] = T;  // B(n, k) = T(k, n)  (kBKN, ldb 128)
        u.C[it] = dinv_b + i * kNB;
        u.fail_flag[it] = cs[it]->fail_flag;
      }
      t.lda = ld; t.ldb = 512; t.ldc = kNB; t.K = i * kNB;
      t.tiles_m = 1; t.tiles_n = i; t.alpha = 1.0; t.beta = 0.0;
      if ((rc = gemm(t, kBKN, m))) return rc;
      u.lda = kNB; u.ldb = kNB; u.ldc = 512; u.K = kNB;
      u.tiles_m = 1; u.tiles_n = i; u.alpha = -1.0; u.beta = 0.0;
      if ((rc = gemm(u, kBKN, m))) return rc;
    }
    {  // slices of W_b (the FP64 bottom part reuses one scratch per context)
      const long long c1 = k.c0 + k.kb;
      const size_t woff = one_slot ? 0 : w_byte_offset(Nt, b);
      const long long eoff = one_slot ? 0 : w_row_offset(Nt, b);
      const size_t tile_bytes = (size_t)kNB * k.kb * ks;
      OzSliceArgs top;  // rows of D_b^-1 (row-contig, ld 512)
      std::memset(&top, 0, sizeof(top));
      for (int it = 0; it < m; ++it) {
        top.X[it] = cs[it]->dinv + (size_t)b * 512 * 512;
        top.slices[it] = cs[it]->wsl + woff;
        top.e[it] = cs[it]->wex + eoff;
        top.fail_flag[it] = cs[it]->fail_flag;
      }
      top.ld = 512;
      top.K = (int)k.kb;
      top.nslices = ks;
      if ((rc = slice(top, k.kb, true, m))) return rc;
      if (c1 >= ld) return MLE_OK;
      OzSliceArgs dt;  // B(j, kk) = Dinv(kk, j): D_b^-T rows (k-contig, ld 512)
      std::memset(&dt, 0, sizeof(dt));
      for (int it = 0; it < m; ++it) {
        dt.X[it] = cs[it]->dinv + (size_t)b * 512 * 512;
        dt.slices[it] = cs[it]->dtsl;
        dt.e[it] = cs[it]->dtex;
        dt.fail_flag[it] = cs[it]->fail_flag;
      }
      dt.ld = 512;
      dt.K = (int)k.kb;
      if ((rc = slice(dt, k.kb, false, m))) return rc;
      const long long eo = oz_panel_row_offset(Nt, b);
      OzGemmArgs g = oz_base(ld, (int)((ld - c1) / kNB), (int)(k.kb / kNB));
      g.kblocks = (int)(k.kb / 32);
      g.beta = 0.0;  // C = -P_b D_b^-1
      for (int it = 0; it < m; ++it) {
        g.As[it] = panel_slices(cs[it], b, eo);
        g.ea[it] = panel_exps(cs[it], b, eo);
        g.Bs[it] = cs[it]->dtsl;
        g.eb[it] = cs[it]->dtex;
        g.C[it] = cs[it]->wbuf;
        g.fail_flag[it] = cs[it]->fail_flag;
      }
      if ((rc = ozgemm(g, m, s))) return rc;
      OzSliceArgs bot;
      std::memset(&bot, 0, sizeof(bot));
      for (int it = 0; it < m; ++it) {
        bot.X[it] = cs[it]->wbuf;
        bot.slices[it] = cs[it]->wsl + woff + (size_t)(k.t1 - k.t0) * tile_bytes;
        bot.e[it] = cs[it]->wex + eoff + k.kb;
        bot.fail_flag[it] = cs[it]->fail_flag;
      }
      bot.ld = ld;
      bot.K = (int)k.kb;
      bot.nslices = ks;
      if ((rc = slice(bot, ld - c1, true, m))) return rc;
    }
    return MLE_OK;
  }

  int solves_w(mle_ctx* const* cs, int m, int ks) {
    const long long ld = cs[0]->N;
    const int Nt = cs[0]->Nt;
    const int nb = (Nt + kOuter - 1) / kOuter;
    MatList ml(cs, m);
    const int zb = ml.count;
    auto S = [&](int z) { return ml.S(z); };
    auto flag = [&](int z) { return (const int*)ml.c[z]->fail_flag; };
    // solve-operand slices: two regions per matrix, alternating by block (look-ahead)
    auto XS = [&](int z, int b) {
      return ml.c[z]->xsl + ((size_t)ml.which[z] * 2 + (b & 1)) * ld * kOzRowBytes;
    };
    auto XE = [&](int z, int b) {
      return ml.c[z]->xex + ((size_t)ml.which[z] * 2 + (b & 1)) * ld;
    };
    int rc;
    // forward sweep, row blocks top-down
    for (int b = 0; b < nb; ++b) {
      const Blk k = blk(Nt, b);
      const int t2 = std::min(Nt, k.t1 + kOuter);
      const size_t woff = w_byte_offset(Nt, b);
      const long long eoff = w_row_offset(Nt, b);
      const size_t tile_bytes = (size_t)kNB * k.kb * ks;
      OzSliceArgs sa;  // B(n, kk) = X[c0 + kk, n]
      std::memset(&sa, 0, sizeof(sa));
      for (int z = 0; z < zb; ++z) {
        sa.X[z] = S(z) + k.c0;
        sa.slices[z] = XS(z, b);
        sa.e[z] = XE(z, b);
        sa.fail_flag[z] = flag(z);
      }
      sa.ld = ld;
      sa.K = (int)k.kb;
      sa.nslices = ks;
      if ((rc = slice(sa, ld, false, zb))) return rc;
      if ((rc = join(s2, s))) return rc;  // (ii) of the previous block wrote rows of (i)
      OzGemmArgs t = oz_base(ld, t2 - k.t0, Nt);  // (i): rows [c0, c2)
      t.kblocks = (int)(k.kb / 32);
      t.nslices = ks;
      t.alpha = 1.0;
      t.beta0_tm = k.t1 - k.t0;
      for (int z = 0; z < zb; ++z) {
        t.As[z] = ml.c[z]->wsl + woff;
        t.ea[z] = ml.c[z]->wex + eoff;
        t.Bs[z] = XS(z, b);
        t.eb[z] = XE(z, b);
        t.C[z] = S(z) + k.c0;
        t.fail_flag[z] = flag(z);
      }
      t.max_ctas = solve_ctas();
      if ((rc = ozgemm(t, zb, s))) return rc;
      if (t2 >= Nt) continue;
      if ((rc = join(s, s2))) return rc;
      OzGemmArgs u = t;  // (ii): rows [c2, N)
      u.tiles_m = Nt - t2;
      u.beta0_tm = 0;
      for (int z = 0; z < zb; ++z) {
        u.As[z] = t.As[z] + (size_t)(t2 - k.t0) * tile_bytes;
        u.ea[z] = t.ea[z] + (size_t)(t2 - k.t0) * kNB;
        u.C[z] = S(z) + (long long)t2 * kNB;
      }
      u.max_ctas = solve_ctas();
      if ((rc = ozgemm(u, zb, bulk()))) return rc;
    }
    if ((rc = join(s2, s))) return rc;
    // right sweep, column blocks left to right, lower tiles only
    for (int b = 0; b < nb; ++b) {
      const Blk k = blk(Nt, b);
      const int t2 = std::min(Nt, k.t1 + kOuter);
      const size_t woff = w_byte_offset(Nt, b);
      const long long eoff = w_row_offset(Nt, b);
      const size_t tile_bytes = (size_t)kNB * k.kb * ks;
      OzSliceArgs sa;  // A(i, kk) = X[c0 + i, c0 + kk], kk <= i only
      std::memset(&sa, 0, sizeof(sa));
      for (int z = 0; z < zb; ++z) {
        sa.X[z] = S(z) + k.c0 + k.c0 * ld;
        sa.slices[z] = XS(z, b);
        sa.e[z] = XE(z, b);
        sa.fail_flag[z] = flag(z);
      }
      sa.ld = ld;
      sa.K = (int)k.kb;
      sa.nslices = ks;
      sa.upper_zero = 1;
      if ((rc = slice(sa, ld - k.c0, true, zb))) return rc;
      if ((rc = join(s2, s))) return rc;
      OzGemmArgs t = oz_base(ld, Nt - k.t0, t2 - k.t0);  // (i): columns [c0, c2)
      t.kblocks = (int)(k.kb / 32);
      t.nslices = ks;
      t.trap = 1;
      t.alpha = 1.0;
      t.beta0_tn = k.t1 - k.t0;
      for (int z = 0; z < zb; ++z) {
        t.As[z] = XS(z, b);
        t.ea[z] = XE(z, b);
        t.Bs[z] = ml.c[z]->wsl + woff;
        t.eb[z] = ml.c[z]->wex + eoff;
        t.C[z] = S(z) + k.c0 + k.c0 * ld;
        t.fail_flag[z] = flag(z);
      }
      t.max_ctas = solve_ctas();
      if ((rc = ozgemm(t, zb, s))) return rc;
      if (t2 >= Nt) continue;
      if ((rc = join(s, s2))) return rc;
      OzGemmArgs u = oz_base(ld, Nt - t2, 0);  // (ii): lower tiles of [c2, N)
      u.kblocks = t.kblocks;
      u.nslices = ks;
      u.lower = 1;
      u.alpha = 1.0;
      const long long c2 = (long long)t2 * kNB;
      for (int z = 0; z < zb; ++z) {
        u.As[z] = t.As[z] + (size_t)(t2 - k.t0) * tile_bytes;
        u.ea[z] = t.ea[z] + (size_t)(t2 - k.t0) * kNB;
        u.Bs[z] = t.Bs[z] + (size_t)(t2 - k.t0) * tile_bytes;
        u.eb[z] = t.eb[z] + (size_t)(t2 - k.t0) * kNB;
        u.C[z] = S(z) + c2 + c2 * ld;
        u.fail_flag[z] = flag(z);
      }
      u.max_ctas = solve_ctas();
      if ((rc = ozgemm(u, zb, bulk()))) return rc;
    }
    return join(s2, s);
  }

  // ---- two-sided blocked reduction B = L^-1 S L^-T (lower half), the sygst recurrence ----
  // For outer block b (columns [c0, c1), D = L11 = L[c0:c1, c0:c1], L21 = L[c1:, c0:c1], and
  // S partitioned alike, S11 / S21 / S22 already updated by the blocks before b):
  //   (1) S11 <- D^-1 S11 D^-T                      two 512^3 DMMA products (D^-1 resident)
  //   (2) S21 <- S21 D^-T                           Ozaki GEMM, B = the rows of D^-1 (= the
  //                                                 top slices of W_b)
  //   (3) S21 <- S21 - 1/2 L21 S11                  Ozaki GEMM, A = the factor's panel slices
  //   (4) S22 <- S22 - S21 L21^T - L21 S21^T        two lower-triangle Ozaki GEMMs (syr2k)
  //   (5) S21 <- S21 - 1/2 L21 S11
  // and S21 is final after the deferred (6) S21 <- L22^-1 S21, done for all blocks at once as
  // the block-inverse forward sweep restricted to the columns left of each row block (the
  // strictly lower block part): X[c0:, 0:c0] = W_b X[c0:c1, 0:c0].
  // Flops per derivative block: (4) 2 n^3 / 3 + (6) n^3 / 3 = n^3, against n^3 + n^3 / 3 for
  // the full forward sweep + right sweep of solves_w.  The diagonal blocks are exact after
  // (1): the reductions read the lower half as before (B[n, n] = y^T B y on the augmented row).
  int solves_2s(mle_ctx* const* cs, int m) {
    MatList ml(cs, m);
    return solves_2s(ml);
  }
  int solves_2s(const MatList& ml) {
    const long long ld = ml.c[0]->N;
    const int Nt = ml.c[0]->Nt;
    const int nb = (Nt + kOuter - 1) / kOuter;
    const int zb = ml.count;
    // sequential-derivative mode: W_b is rebuilt into the context's one-block buffer right
    // before each use (it depends only on L: ~0.5% of the block's work)
    const bool w_stream = ml.c[0]->seq_derivs;
    mle_ctx* wctx[1] = {ml.c[0]};
    auto S = [&](int z) { return ml.S(z); };
    auto flag = [&](int z) { return (const int*)ml.c[z]->fail_flag; };
    auto XS = [&](int z, int b) {
      return ml.c[z]->xsl + ((size_t)ml.slot[z] * 2 + (b & 1)) * ld * kOzRowBytes;
    };
    auto XE = [&](int z, int b) {
      return ml.c[z]->xex + ((size_t)ml.slot[z] * 2 + (b & 1)) * ld;
    };
    auto T2 = [&](int z) { return ml.c[z]->ts2 + (size_t)ml.slot[z] * 512 * 512; };
    auto AS = [&](int z) { return ml.c[z]->a11sl + (size_t)ml.slot[z] * 512 * kOzRowBytes; };
    auto AE = [&](int z) { return ml.c[z]->a11ex + (size_t)ml.slot[z] * 512; };
    int rc;
    for (int b = 0; b < nb; ++b) {
      const Blk k = blk(Nt, b);
      const long long c1 = k.c0 + k.kb;
      const int tb = k.t1 - k.t0;
      if (w_stream && (rc = compute_w_block(wctx, 1, kOzSlices, b))) return rc;
      const size_t woff = w_stream ? 0 : w_byte_offset(Nt, b);
      const long long eoff = w_stream ? 0 : w_row_offset(Nt, b);
      const long long eo = oz_panel_row_offset(Nt, b);
      // (1) S11 <- D^-1 S11 D^-T.  Generation (lower_only) and the trailing updates (4) of the
      // blocks before b write only lower tiles, so S11's upper tiles are restored from its
      // lower ones first.
      {
        double* blks[kMaxGemm];
        for (int z = 0; z < zb; ++z) blks[z] = S(z) + k.c0 + k.c0 * ld;
        launches += 1;
        CUDA_TRY(launch_mirror_lower(blks, zb, ld, (int)k.kb, s));
      }
      {
        GemmArgs t = gemm_base(), u = gemm_base();
        for (int z = 0; z < zb; ++z) {
          const double* dinv_b = ml.c[z]->dinv + (size_t)b * 512 * 512;
          t.A[z] = dinv_b;                          // A(i, kk) = Dinv(i, kk), lda 512
          t.B[z] = S(z) + k.c0 + k.c0 * ld;         // B(n, kk) = S11(kk, n)   (kBKN)
          t.C[z] = T2(z);
          t.fail_flag[z] = flag(z);
          u.A[z] = T2(z);                           // A(i, kk) = T(i, kk)
          u.B[z] = dinv_b;                          // B(n, kk) = Dinv(n, kk)  (kBNK)
          u.C[z] = S(z) + k.c0 + k.c0 * ld;
          u.fail_flag[z] = flag(z);
        }
        t.lda = 512; t.ldb = ld; t.ldc = 512; t.K = (int)k.kb;
        t.tiles_m = tb; t.tiles_n = tb; t.alpha = 1.0; t.beta = 0.0;
        if ((rc = gemm(t, kBKN, zb))) return rc;
        u.lda = 512; u.ldb = 512; u.ldc = ld; u.K = (int)k.kb;
        u.tiles_m = tb; u.tiles_n = tb; u.alpha = 1.0; u.beta = 0.0;
        if ((rc = gemm(u, kBNK, zb))) return rc;
      }
      if (c1 >= ld) break;
      const int rt = (int)((ld - c1) / kNB);  // row tiles below the block
      // slices of S21 (A operand: rows c1.., K over the block's columns)
      auto slice_s21 = [&]() {
        OzSliceArgs sa;
        std::memset(&sa, 0, sizeof(sa));
        for (int z = 0; z < zb; ++z) {
          sa.X[z] = S(z) + c1 + k.c0 * ld;
          sa.slices[z] = XS(z, b);
          sa.e[z] = XE(z, b);
          sa.fail_flag[z] = flag(z);
        }
        sa.ld = ld;
        sa.K = (int)k.kb;
        return slice(sa, ld - c1, true, zb);
      };
      // (2) S21 <- S21 D^-T
      if ((rc = slice_s21())) return rc;
      {
        OzGemmArgs g = oz_base(ld, rt, tb);
        g.kblocks = (int)(k.kb / 32);
        g.alpha = 1.0;
        g.beta = 0.0;
        for (int z = 0; z < zb; ++z) {
          g.As[z] = XS(z, b);
          g.ea[z] = XE(z, b);
          g.Bs[z] = ml.c[z]->wsl + woff;   // rows of D^-1 (W_b's top kb rows)
          g.eb[z] = ml.c[z]->wex + eoff;
          g.C[z] = S(z) + c1 + k.c0 * ld;
          g.fail_flag[z] = flag(z);
        }
        if ((rc = ozgemm(g, zb, s))) return rc;
      }
      // slices of the new S11 (B operand of (3) / (5): B(n, kk) = S11(n, kk))
      {
        OzSliceArgs sa;
        std::memset(&sa, 0, sizeof(sa));
        for (int z = 0; z < zb; ++z) {
          sa.X[z] = S(z) + k.c0 + k.c0 * ld;
          sa.slices[z] = AS(z);
          sa.e[z] = AE(z);
          sa.fail_flag[z] = flag(z);
        }
        sa.ld = ld;
        sa.K = (int)k.kb;
        if ((rc = slice(sa, k.kb, true, zb))) return rc;
      }
      auto half_update = [&]() {  // S21 -= 1/2 L21 S11
        OzGemmArgs g = oz_base(ld, rt, tb);
        g.kblocks = (int)(k.kb / 32);
        g.alpha = -0.5;
        for (int z = 0; z < zb; ++z) {
          g.As[z] = panel_slices(ml.c[z], b, eo);
          g.ea[z] = panel_exps(ml.c[z], b, eo);
          g.Bs[z] = AS(z);
          g.eb[z] = AE(z);
          g.C[z] = S(z) + c1 + k.c0 * ld;
          g.fail_flag[z] = flag(z);
        }
        return ozgemm(g, zb, s);
      };
      // (3)
      if ((rc = half_update())) return rc;
      // (4) S22 -= S21 L21^T + L21 S21^T, look-ahead split:
      //   (i)  the next block's columns [c1, c2) (all rows >= c1, trapezoid) on the main
      //        stream -- everything block b + 1's steps (1)-(3) read;
      //   (ii) the lower tiles of [c2, N) on the side stream, under block b + 1's chain.
      // (ii) of block b - 1 wrote tiles (i) touches: the main stream waits for it first.
      if ((rc = slice_s21())) return rc;
      if ((rc = join(s2, s))) return rc;
      const int tn1 = std::min(kOuter, rt);  // tile columns of the next block
      for (int pass = 0; pass < 2; ++pass) {
        OzGemmArgs g = oz_base(ld, rt, tn1);
        g.kblocks = (int)(k.kb / 32);
        g.trap = 1;
        for (int z = 0; z < zb; ++z) {
          const int8_t* ls = panel_slices(ml.c[z], b, eo);
          const int* le = panel_exps(ml.c[z], b, eo);
          g.As[z] = pass == 0 ? XS(z, b) : ls;
          g.ea[z] = pass == 0 ? XE(z, b) : le;
          g.Bs[z] = pass == 0 ? ls : XS(z, b);
          g.eb[z] = pass == 0 ? le : XE(z, b);
          g.C[z] = S(z) + c1 + c1 * ld;
          g.fail_flag[z] = flag(z);
        }
        if ((rc = ozgemm(g, zb, s))) return rc;
      }
      if (rt > tn1) {
        if ((rc = join(s, s2))) return rc;  // (ii) reads this block's S21 slices
        const int t2r = rt - tn1;           // tiles of [c2, N)
        const long long c2 = c1 + (long long)tn1 * kNB;
        const size_t skip = (size_t)tn1 * kOzTileBytes;
        for (int pass = 0; pass < 2; ++pass) {
          OzGemmArgs g = oz_base(ld, t2r, 0);
          g.kblocks = (int)(k.kb / 32);
          g.lower = 1;
          for (int z = 0; z < zb; ++z) {
            const int8_t* ls = panel_slices(ml.c[z], b, eo) + skip;
            const int* le = panel_exps(ml.c[z], b, eo) + (long long)tn1 * kNB;
            const int8_t* xs = XS(z, b) + skip;
            const int* xe = XE(z, b) + (long long)tn1 * kNB;
            g.As[z] = pass == 0 ? xs : ls;
            g.ea[z] = pass == 0 ? xe : le;
            g.Bs[z] = pass == 0 ? ls : xs;
            g.eb[z] = pass == 0 ? le : xe;
            g.C[z] = S(z) + c2 + c2 * ld;
            g.fail_flag[z] = flag(z);
          }
          g.max_ctas = solve_ctas();
          if ((rc = ozgemm(g, zb, bulk()))) return rc;
        }
      }
      // (5): S21 itself (the GEMMs of (4) read its slices)
      if ((rc = half_update())) return rc;
    }
    if ((rc = join(s2, s))) return rc;
    // (6) deferred: S21 <- L22^-1 S21 for every block column, as the block-inverse forward
    // sweep over row blocks b restricted to the columns [0, c0)
    for (int b = 1; b < nb; ++b) {
      const Blk k = blk(Nt, b);
      if (w_stream && (rc = compute_w_block(wctx, 1, kOzSlices, b))) return rc;
      const size_t woff = w_stream ? 0 : w_byte_offset(Nt, b);
      const long long eoff = w_stream ? 0 : w_row_offset(Nt, b);
      OzSliceArgs sa;  // B(n, kk) = X[c0 + kk, n], n < c0
      std::memset(&sa, 0, sizeof(sa));
      for (int z = 0; z < zb; ++z) {
        sa.X[z] = S(z) + k.c0;
        sa.slices[z] = XS(z, b);
        sa.e[z] = XE(z, b);
        sa.fail_flag[z] = flag(z);
      }
      sa.ld = ld;
      sa.K = (int)k.kb;
      if ((rc = slice(sa, k.c0, false, zb))) return rc;
      OzGemmArgs t = oz_base(ld, Nt - k.t0, k.t0);  // rows [c0, N) x columns [0, c0)
      t.kblocks = (int)(k.kb / 32);
      t.alpha = 1.0;
      t.beta0_tm = k.t1 - k.t0;  // the block's own rows are overwritten (D^-1 X)
      for (int z = 0; z < zb; ++z) {
        t.As[z] = ml.c[z]->wsl + woff;
        t.ea[z] = ml.c[z]->wex + eoff;
        t.Bs[z] = XS(z, b);
        t.eb[z] = XE(z, b);
        t.C[z] = S(z) + k.c0;
        t.fail_flag[z] = flag(z);
      }
      t.max_ctas = solve_ctas();
      if ((rc = ozgemm(t, zb, s))) return rc;
    }
    return MLE_OK;
  }

  // DMMA path (MLE_FP64_GEMM=dmma): 128-wide inner steps + K = 512 outer updates.
  int solves_dmma(mle_ctx* const* cs, int m) {
    const long long ld = cs[0]->N;
    const int Nt = cs[0]->Nt;
    MatList ml(cs, m);
    const int zb = ml.count;
    auto S = [&](int z) { return ml.S(z); };
    auto L = [&](int z) { return (const double*)ml.c[z]->sigma; };
    auto Linv = [&](int z, int k) {
      return (const double*)(ml.c[z]->linv + (size_t)k * kNB * kNB);
    };
    auto flag = [&](int z) { return (const int*)ml.c[z]->fail_flag; };
    int rc;
    // forward sweep X = L^-1 S (all columns), row blocks top-down
    for (int b0 = 0; b0 < Nt; b0 += kOuter) {
      const int b1 = std::min(Nt, b0 + kOuter);
      for (int k = b0; k < b1; ++k) {
        const long long k0 = (long long)k * kNB;
        GemmArgs g = gemm_base();
        for (int z = 0; z < zb; ++z) {
          g.A[z] = Linv(z, k);
          g.B[z] = S(z) + k0;   // B(n, kk) = S[k0 + kk, n]  (kBKN)
          g.C[z] = S(z) + k0;   // in place: BM = 128 covers the whole row panel
          g.fail_flag[z] = flag(z);
        }
        g.lda = kNB; g.ldb = ld; g.ldc = ld;
        g.tiles_m = 1; g.tiles_n = Nt; g.alpha = 1.0; g.beta = 0.0;
        if ((rc = gemm(g, kBKN, zb))) return rc;
        const int wrows = b1 - k - 1;  // remaining row tiles of this outer block
        if (wrows > 0) {
          GemmArgs t = gemm_base();
          for (int z = 0; z < zb; ++z) {
            t.A[z] = L(z) + (k0 + kNB) + k0 * ld;   // L[k+1 : b1, k]
            t.B[z] = S(z) + k0;                     // X_k (kBKN)
            t.C[z] = S(z) + (k0 + kNB);
            t.fail_flag[z] = flag(z);
          }
          t.lda = ld; t.ldb = ld; t.ldc = ld;
          t.tiles_m = wrows; t.tiles_n = Nt; t.alpha = -1.0; t.beta = 1.0;
          if ((rc = gemm(t, kBKN, zb))) return rc;
        }
      }
      if (b1 >= Nt) continue;
      const int b2 = std::min(Nt, b1 + kOuter);
      const long long c0 = (long long)b0 * kNB, t0 = (long long)b1 * kNB, u0 = (long long)b2 * kNB;
      if ((rc = join(s2, s))) return rc;
      GemmArgs t = gemm_base();   // (i): rows [b1, b2), all columns
      for (int z = 0; z < zb; ++z) {
        t.A[z] = L(z) + t0 + c0 * ld;   // L[b1:b2, b0:b1]
        t.B[z] = S(z) + c0;             // X[b0:b1, :] (kBKN)
        t.C[z] = S(z) + t0;
        t.fail_flag[z] = flag(z);
      }
      t.lda = ld; t.ldb = ld; t.ldc = ld;
      t.K = (b1 - b0) * kNB;
      t.tiles_m = b2 - b1; t.tiles_n = Nt; t.alpha = -1.0; t.beta = 1.0;
      if ((rc = gemm(t, kBKN, zb))) return rc;
      if (b2 >= Nt) continue;
      if ((rc = join(s, s2))) return rc;
      GemmArgs u = gemm_base();   // (ii): rows >= b2
      for (int z = 0; z < zb; ++z) {
        u.A[z] = L(z) + u0 + c0 * ld;
        u.B[z] = S(z) + c0;
        u.C[z] = S(z) + u0;
        u.fail_flag[z] = flag(z);
      }
      u.lda = ld; u.ldb = ld; u.ldc = ld;
      u.K = (b1 - b0) * kNB;
      u.tiles_m = Nt - b2; u.tiles_n = Nt; u.alpha = -1.0; u.beta = 1.0;
      if ((rc = gemm(u, kBKN, zb, bulk()))) return rc;
    }
    if ((rc = join(s2, s))) return rc;
    // right sweep on lower tiles: B[j:, j] = X[j:, j] Linv_j^T ; X[T,T] -= B[T,j] L[T,j]^T
    for (int b0 = 0; b0 < Nt; b0 += kOuter) {
      const int b1 = std::min(Nt, b0 + kOuter);
      for (int j = b0; j < b1; ++j) {
        const long long j0 = (long long)j * kNB;
        GemmArgs g = gemm_base();
        for (int z = 0; z < zb; ++z) {
          g.A[z] = S(z) + j0 + j0 * ld;
          g.B[z] = Linv(z, j);
          g.C[z] = S(z) + j0 + j0 * ld;
          g.fail_flag[z] = flag(z);
        }
        g.lda = ld; g.ldb = kNB; g.ldc = ld;
        g.tiles_m = Nt - j; g.tiles_n = 1; g.alpha = 1.0; g.beta = 0.0; g.wide = 1;
        if ((rc = gemm(g, kBNK, zb))) return rc;
        const int wcols = b1 - j - 1;
        if (wcols > 0) {
          GemmArgs t = gemm_base();
          for (int z = 0; z < zb; ++z) {
            t.A[z] = S(z) + (j0 + kNB) + j0 * ld;   // B[T, j]
            t.B[z] = L(z) + (j0 + kNB) + j0 * ld;   // L[T, j]  (kBNK)
            t.C[z] = S(z) + (j0 + kNB) + (j0 + kNB) * ld;
            t.fail_flag[z] = flag(z);
          }
          t.lda = ld; t.ldb = ld; t.ldc = ld;
          t.tiles_m = Nt - j - 1; t.tiles_n = wcols; t.trap = 1; t.alpha = -1.0; t.beta = 1.0;
          if ((rc = gemm(t, kBNK, zb))) return rc;
        }
      }
      if (b1 >= Nt) continue;
      const int b2 = std::min(Nt, b1 + kOuter);
      const long long c0 = (long long)b0 * kNB, t0 = (long long)b1 * kNB, u0 = (long long)b2 * kNB;
      if ((rc = join(s2, s))) return rc;
      GemmArgs t = gemm_base();   // (i): columns [b1, b2), rows >= b1
      for (int z = 0; z < zb; ++z) {
        t.A[z] = S(z) + t0 + c0 * ld;   // B[T, b0:b1]
        t.B[z] = L(z) + t0 + c0 * ld;   // L[b1:b2, b0:b1]
        t.C[z] = S(z) + t0 + t0 * ld;
        t.fail_flag[z] = flag(z);
      }
      t.lda = ld; t.ldb = ld; t.ldc = ld;
      t.K = (b1 - b0) * kNB;
      t.tiles_m = Nt - b1; t.tiles_n = b2 - b1; t.trap = 1; t.alpha = -1.0; t.beta = 1.0;
      if ((rc = gemm(t, kBNK, zb))) return rc;
      if (b2 >= Nt) continue;
      if ((rc = join(s, s2))) return rc;
      GemmArgs u = gemm_base();   // (ii): lower tiles of [b2, Nt)
      for (int z = 0; z < zb; ++z) {
        u.A[z] = S(z) + u0 + c0 * ld;
        u.B[z] = L(z) + u0 + c0 * ld;
        u.C[z] = S(z) + u0 + u0 * ld;
        u.fail_flag[z] = flag(z);
      }
      u.lda = ld; u.ldb = ld; u.ldc = ld;
      u.K = (b1 - b0) * kNB;
      u.tiles_m = Nt - b2; u.lower = 1; u.alpha = -1.0; u.beta = 1.0;
      if ((rc = gemm(u, kBNK, zb, bulk()))) return rc;
    }
    return join(s2, s);
  }
};

// Runs up to kMaxItems requests (same device, same N) on the leader's stream.
// Log-likelihood, score and Fisher information from the reduction outputs r[] (layout of
// launch_reduce's out: sums, then y^T B y of the three blocks); o = [ll, grad[3], fisher[9]].
void assemble_results(const mle_ctx* c, const ThetaParams& P, const double* r, int mode,
                      double* o) {
  const double n = (double)c->n, s2 = P.sigma2;
  const double logdet = r[0], quad = r[1];
  o[0] = -0.5 * n * kLog2Pi - logdet - 0.5 * quad;  // likelihood.py:85-89, 123
  if (mode != 2) return;
  const double tr_a = r[2], tr_n = r[3], faa = r[4], fan = r[5], fnn = r[6];
  const double yby_a = r[kReduceSums], yby_n = r[kReduceSums + 1];
  o[2] = -0.5 * tr_a + 0.5 * yby_a;        // likelihood.py:137
  o[3] = -0.5 * tr_n + 0.5 * yby_n;
  double* f = o + 4;
  f[4] = 0.5 * faa;                        // likelihood.py:142
  f[5] = f[7] = 0.5 * fan;                 // likelihood.py:146
  f[8] = 0.5 * fnn;                        // likelihood.py:147
  if (c->nugget == 0.0) {
    o[1] = (quad - n) / (2.0 * s2);        // likelihood.py:129
    f[0] = n / (2.0 * s2 * s2);            // likelihood.py:130
    f[1] = f[3] = tr_a / (2.0 * s2);       // likelihood.py:141
    f[2] = f[6] = tr_n / (2.0 * s2);       // likelihood.py:145
  } else {
    // Nugget (config 5; not in the reference, oracle eval_all_nugget): dSigma/dsigma^2 =
    // (Sigma - tau^2 I) / sigma^2, so B_s2 = (I - tau^2 M) / sigma^2, M = L^-1 L^-T.
    const double t = c->nugget, tr_m = r[7], fam = r[8], fnm = r[9], fmm = r[10];
    const double yby_m = r[kReduceSums + 2];  // y^T M y = |Sigma^-1 z|^2
    o[1] = -0.5 * (n - t * tr_m) / s2 + 0.5 * (quad - t * yby_m) / s2;
    f[0] = 0.5 * (n - 2.0 * t * tr_m + t * t * fmm) / (s2 * s2);
    f[1] = f[3] = 0.5 * (tr_a - t * fam) / s2;
    f[2] = f[6] = 0.5 * (tr_n - t * fnm) / s2;
  }
}

int run_chunk(Item* items, int m) {
  const auto host_t0 = std::chrono::steady_clock::now();
  mle_ctx* lead = items[0].c;
  cudaStream_t s = lead->stream;
  const bool lookahead = !lead->kprof && use_lookahead();
  Launcher run{s, lookahead ? lead->side : nullptr, lead->pool, kPoolEvents};
  if (lookahead) {
    run.s3 = lead->inner;
    run.s4 = lead->edge;
  }
  if (lead->kprof) run.prof = lead;
  cudaStream_t aux = lead->kprof ? s : lead->aux;  // profiling: everything serialised
  PassClock* pc = &lead->pass_clock;
  {
    if (!pc->start) {
      CUDA_TRY(cudaEventCreate(&pc->start));
      CUDA_TRY(cudaEventCreate(&pc->pre));
      CUDA_TRY(cudaEventCreate(&pc->end[0]));
      CUDA_TRY(cudaEventCreate(&pc->end[1]));
    }
  }
  CUDA_TRY(cudaEventRecord(pc->pre, s));
  {
    int rc = run.trace_begin();
    if (rc) return rc;
  }
  for (int b = 0; b < m; ++b) {
    Item& it = items[b];
    int rc = wait_spec(it.c, s);
    if (rc) return rc;
    rc = ensure_matrices(it.c, it.derivs);
    if (rc) return rc;
    // this pass overwrites what a previous speculation left in sa / sn / wsl
    if (it.factor || it.derivs) it.c->spec_ready = false;  // the solves consume S in place
    if (use_gen_table())
      mle_fill_gen_table(it.c->h_max / it.P.alpha, &it.P);
    else
      it.P.tab_n = 0;
    std::memcpy(lead->h_stage + b, &it.P, sizeof(ThetaParams));
  }
  {  // one H2D copy of all items' parameters, scattered (+ failure flags cleared) on device
    PassIo io;
    std::memset(&io, 0, sizeof(io));
    for (int b = 0; b < m; ++b) {
      io.theta[b] = items[b].c->d_theta;
      io.flag[b] = items[b].c->fail_flag;
    }
    CUDA_TRY(cudaMemcpyAsync(lead->d_stage, lead->h_stage, sizeof(ThetaParams) * m,
                             cudaMemcpyHostToDevice, s));
    run.launches += 1;
    CUDA_TRY(launch_scatter_theta(io, lead->d_stage, m, s));
  }
  NvtxPhases nvtx;
  nvtx.push(m > 1 ? "mle pass (batched)" : "mle pass");
  nvtx.push("gen");
  CUDA_TRY(cudaEventRecord(lead->ev[0], s));
  CUDA_TRY(cudaEventRecord(pc->start, s));
  // Generation.  Sigma (items that factor) on the main stream; the derivative matrices on
  // the aux stream, concurrently with the Cholesky (they are only needed by the solves).
  auto gen_set = [&](bool sigma_pass) {
    GenArgs ga;
    std::memset(&ga, 0, sizeof(ga));
    int ng = 0;
    for (int b = 0; b < m; ++b) {
      const Item& it = items[b];
      if (sigma_pass ? !it.factor : !(it.gen_derivs || it.spec)) continue;
      GenItem& gi = ga.item[ng++];
      gi.P = it.c->d_theta;
      gi.lx = it.c->lx;
      gi.ly = it.c->ly;
      gi.z = it.c->z;
      gi.sigma = it.c->sigma;
      gi.dalpha = it.c->sa;
      gi.dnu = it.c->sn;
      gi.fail_flag = it.c->fail_flag;
      gi.tab = it.P.tab_n > 0 ? (sigma_pass ? it.c->gtab_s : it.c->gtab_d) : nullptr;
      gi.write_sigma = sigma_pass ? 1 : 0;
      gi.write_derivs = sigma_pass ? 0 : 1;
      if (!sigma_pass) it.c->deriv_lower = two_sided_gen(it.c);
    }
    // the two-sided solves read only the lower tiles of the derivative matrices
    ga.lower_only = (!sigma_pass && ng > 0) ? (items[0].c->deriv_lower ? 1 : 0) : 0;
    if (!sigma_pass)
      for (int b = 0; b < m; ++b)
        if ((items[b].gen_derivs || items[b].spec) && !items[b].c->deriv_lower) ga.lower_only = 0;
    ga.ld = lead->N;
    ga.rows = lead->N;
    ga.n = (int)lead->n;
    return std::make_pair(ga, ng);
  };
  // generation bytes of one launch set: 8 B per lower-triangle element per matrix written
  const double tri_bytes = 8.0 * (double)lead->n * ((double)lead->n + 1.0) / 2.0;
  auto sig = gen_set(true);
  if (sig.second > 0) {
    run.launches += 2;
    {
      int rc = run.prof_begin(s);
      if (rc) return rc;
    }
    launch_gen_table(sig.first, sig.second, false, s);
    // Sigma: the first outer block's columns on the main stream (all the Cholesky's first
    // inner steps read), the rest on the low-priority aux stream under those steps, so the
    // chain's kernels win the SMs; the side stream (first trailing update) waits for it.
    constexpr int kJcut = kOuter * kNB / 32;
    if (run.s2 && aux != s && (lead->N + 31) / 32 > kJcut) {
      GenArgs pa = sig.first, pb = sig.first;
      pa.region = 1;
      pa.jcut = kJcut;
      pb.region = 2;
      pb.jcut = kJcut;
      int rc = run.join(s, aux);  // aux starts after the table, not after (a)
      if (rc) return rc;
      launch_gen_engine(pa, sig.second, s);
      run.launches += 1;
      launch_gen_engine(pb, sig.second, aux);
      if ((rc = run.join(aux, run.s2))) return rc;
    } else {
      launch_gen_engine(sig.first, sig.second, s);
    }
    CUDA_TRY(cudaGetLastError());
    {  // (kernel profiling serialises: aux == s, one launch)
      int rc = run.prof_end(s, 2, tri_bytes * sig.second);
      if (rc) return rc;
    }
  }
  // derivative matrices: eval_all items first (the solves wait for these only), then the
  // speculative loglik items
  auto der = gen_set(false);
  bool any_spec = false;
  for (int b = 0; b < m; ++b) any_spec = any_spec || items[b].spec;
  if (der.second > 0) {
    int rc = run.join(s, aux);
    if (rc) return rc;
    GenArgs now = der.first, later = der.first;
    int nn = 0, nl = 0;
    for (int b = 0, g = 0; b < m; ++b) {
      if (!(items[b].gen_derivs || items[b].spec)) continue;
      if (items[b].spec) later.item[nl++] = der.first.item[g];
      else now.item[nn++] = der.first.item[g];
      ++g;
    }
    auto identities = [&](bool spec_items) -> int {  // nugget: third block S = I_n
      double* mats[kMaxItems];
      int k = 0;
      for (int b = 0; b < m; ++b)
        if (items[b].c->smat && (spec_items ? items[b].spec : items[b].gen_derivs))
          mats[k++] = items[b].c->smat;
      if (k > 0) {
        run.launches += 1;
        CUDA_TRY(launch_set_identity(mats, lead->N, (int)lead->n, k, aux));
      }
      return MLE_OK;
    };
    if (nn > 0) {
      run.launches += 2;
      if ((rc = run.prof_begin(aux))) return rc;
      launch_gen_table(now, nn, true, aux);
      launch_gen_engine(now, nn, aux);
      CUDA_TRY(cudaGetLastError());
      if ((rc = run.prof_end(aux, 2, 2.0 * tri_bytes * nn))) return rc;
    }
    if ((rc = identities(false))) return rc;
    CUDA_TRY(cudaEventRecord(lead->ev_der, aux));
    if (nl > 0) {
      run.launches += 2;
      if ((rc = run.prof_begin(aux))) return rc;
      launch_gen_table(later, nl, true, aux);
      launch_gen_engine(later, nl, aux);
      CUDA_TRY(cudaGetLastError());
      if ((rc = run.prof_end(aux, 2, 2.0 * tri_bytes * nl))) return rc;
    }
    if ((rc = identities(true))) return rc;
  } else {
    CUDA_TRY(cudaEventRecord(lead->ev_der, aux));
  }
  nvtx.next("potrf");
  CUDA_TRY(cudaEventRecord(lead->ev[1], s));
  // W_b of the items that factor in this pass and need it (eval_all, or speculation for a
  // loglik item) is built on the aux stream block by block during their Cholesky.
  bool w_in_potrf[kMaxItems] = {};
  bool any_w_eval = false;
  {  // Cholesky for items without a cached factor
    mle_ctx* cs[kMaxItems];
    mle_ctx* wr[kMaxItems];
    double* mats[kMaxItems];
    long long aug[kMaxItems];
    int nf = 0, nwr = 0;
    for (int b = 0; b < m; ++b)
      if (items[b].factor) {
        mle_ctx* c = items[b].c;
        cs[nf] = c;
        mats[nf] = c->sigma;
        aug[nf] = c->n;
        ++nf;
        if (c->lsl && c->wsl && (items[b].spec || items[b].need_w)) {
          wr[nwr++] = c;
          w_in_potrf[b] = true;
          any_w_eval = any_w_eval || items[b].need_w;
        }
      }
    if (nf > 0) {
      run.wreq = wr;
      run.nwreq = nwr;
      run.wks = solve_slices();
      run.ws = aux;
      int rc = run.potrf(cs, mats, aug, nf);
      run.nwreq = 0;
      if (rc) return rc;
    }
  }
  nvtx.next("solve");
  CUDA_TRY(cudaEventRecord(lead->ev[2], s));
  if (any_spec) {
    for (int b = 0; b < m; ++b)
      if (items[b].spec) {
        CUDA_TRY(cudaEventRecord(items[b].c->spec_done, aux));
        items[b].c->spec_pending = true;
      }
  }
  {
    if (der.second > 0) CUDA_TRY(cudaStreamWaitEvent(s, lead->ev_der, 0));
    if (any_w_eval) {
      int rc = run.join(aux, s);
      if (rc) return rc;
    }
    mle_ctx* cs[kMaxItems];
    mle_ctx* cw[kMaxItems];
    int nd = 0, nw = 0;
    for (int b = 0; b < m; ++b) {
      if (items[b].derivs) cs[nd++] = items[b].c;
      if (items[b].need_w && !w_in_potrf[b]) cw[nw++] = items[b].c;
    }
    if (nd > 0) {
      int rc = run.solves(cs, nd, cw, nw);
      if (rc) return rc;
    }
  }
  nvtx.next("reduce");
  CUDA_TRY(cudaEventRecord(lead->ev[3], s));
  ReduceArgs ra;
  std::memset(&ra, 0, sizeof(ra));
  for (int b = 0; b < m; ++b) {
    mle_ctx* c = items[b].c;
    ra.L[b] = c->sigma;
    ra.Ba[b] = items[b].derivs ? c->sa : nullptr;
    ra.Bn[b] = items[b].derivs ? c->sn : nullptr;
    ra.Bm[b] = items[b].derivs ? c->smat : nullptr;
    ra.partials[b] = c->partials;
    ra.out[b] = c->out;
    ra.fail_flag[b] = c->fail_flag;
  }
  ra.ld = lead->N;
  ra.n = (int)lead->n;
  run.launches += 2;
  CUDA_TRY(launch_reduce(ra, m, s));
  nvtx.next("results");
  CUDA_TRY(cudaEventRecord(lead->ev[4], s));
  {  // gather every item's results + flag + pivot, one D2H copy
    PassIo io;
    std::memset(&io, 0, sizeof(io));
    for (int b = 0; b < m; ++b) {
      io.out[b] = items[b].c->out;
      io.flag[b] = items[b].c->fail_flag;
      io.idx[b] = items[b].c->fail_idx;
    }
    run.launches += 1;
    CUDA_TRY(launch_gather_results(io, lead->d_resb, m, s));
    CUDA_TRY(cudaMemcpyAsync(lead->h_resb, lead->d_resb, sizeof(double) * m * (kReduceOut + 2),
                             cudaMemcpyDeviceToHost, s));
  }
  CUDA_TRY(cudaEventRecord(pc->end[pc->passes & 1], s));
  const auto host_t1 = std::chrono::steady_clock::now();
  CUDA_TRY(cudaStreamSynchronize(s));
  float gap_ms = 0.f, wait_ms = 0.f;
  if (pc->passes > 0) {
    if (cudaEventElapsedTime(&gap_ms, pc->end[(pc->passes - 1) & 1], pc->pre) != cudaSuccess ||
        cudaEventElapsedTime(&wait_ms, pc->pre, pc->start) != cudaSuccess) {
      cudaGetLastError();
      gap_ms = wait_ms = 0.f;
    }
  }
  ++pc->passes;
  CUDA_TRY(cudaGetLastError());
  {
    int rc = run.trace_end();
    if (rc) return rc;
  }
  const auto host_t2 = std::chrono::steady_clock::now();
  {
    int rc = run.prof_collect();
    if (rc) return rc;
  }
  float ms[4];
  for (int p = 0; p < 4; ++p) CUDA_TRY(cudaEventElapsedTime(&ms[p], lead->ev[p], lead->ev[p + 1]));
  double flops = 0.0, gbytes = 0.0;
  for (int b = 0; b < m; ++b) {
    const double nd = (double)items[b].c->n;
    if (items[b].factor) {
      flops += nd * nd * nd / 3.0;
      gbytes += 8.0 * nd * (nd + 1.0) / 2.0;
    }
    if (items[b].derivs) {
      flops += 2.0 * (nd * nd * nd + nd * nd * nd / 3.0);
      gbytes += 2.0 * 8.0 * nd * (nd + 1.0) / 2.0;
    }
  }
  for (int b = 0; b < m; ++b)
    std::memcpy(items[b].c->h_res, lead->h_resb + (size_t)b * (kReduceOut + 2),
                sizeof(double) * (kReduceOut + 2));
  for (int b = 0; b < m; ++b) {
    Item& it = items[b];
    mle_ctx* c = it.c;
    c->phase_ms[MLE_PHASE_GEN] = ms[0];
    c->phase_ms[MLE_PHASE_POTRF] = ms[1];
    c->phase_ms[MLE_PHASE_SOLVE] = ms[2];
    c->phase_ms[MLE_PHASE_REDUCE] = ms[3];
    c->phase_ms[MLE_PHASE_TOTAL] = ms[0] + ms[1] + ms[2] + ms[3];
    c->flops = flops;
    c->gen_bytes = gbytes;
    c->launches = run.launches;
    if (c == lead) {
      c->kstats[7] = std::chrono::duration<double, std::milli>(host_t1 - host_t0).count();
      c->kstats[8] = gap_ms;
      c->kstats[9] = wait_ms;
      c->host_wait_ms = std::chrono::duration<double, std::milli>(host_t2 - host_t1).count();
    }
    if (c != lead) std::memcpy(c->kstats, lead->kstats, sizeof(c->kstats));
    int flag;
    std::memcpy(&flag, c->h_res + kReduceOut, sizeof(int));
    if (flag) {
      long long idx;
      std::memcpy(&idx, c->h_res + kReduceOut + 1, sizeof(long long));
      it.rc = MLE_NOT_PD;
      it.pivot = idx;
      c->factor_valid = false;
      c->spec_ready = false;
      continue;
    }
    if (it.spec) {
      c->spec_ready = true;
      c->spec_theta[0] = it.P.sigma2;
      c->spec_theta[1] = it.P.alpha;
      c->spec_theta[2] = it.P.nu;
    }
    it.rc = MLE_OK;
    it.pivot = -1;
    if (it.factor) {
      const double lo = c->h_res[kReduceSums + 3], hi = c->h_res[kReduceSums + 4];
      c->cond_est = lo > 0.0 ? (hi / lo) * (hi / lo) : 0.0;
    }
    c->factor_valid = true;
    c->cached_theta[0] = it.P.sigma2;
    c->cached_theta[1] = it.P.alpha;
    c->cached_theta[2] = it.P.nu;
    const double* r = c->h_res;
    assemble_results(c, it.P, r, it.mode, it.res);
    c->cached_ll = it.res[0];
    c->cached_logdet = r[0];
    c->cached_quad = r[1];
    c->cached_dmin = r[kReduceSums + 3];
    c->cached_dmax = r[kReduceSums + 4];
  }
  return MLE_OK;
}

bool same_theta(const mle_ctx* c, const double th[3]) {
  return c->factor_valid && c->cached_theta[0] == th[0] && c->cached_theta[1] == th[1] &&
         c->cached_theta[2] == th[2];
}

// Runs the requests (all same device and N) in chunks of kMaxItems.
int run_batch(Item* items, int count) {
  for (int b0 = 0; b0 < count; b0 += kMaxItems) {
    const int m = std::min(kMaxItems, count - b0);
    CUDA_TRY(cudaSetDevice(items[b0].c->device));
    int rc = run_chunk(items + b0, m);
    if (rc) return rc;
  }
  return MLE_OK;
}

// Prepare one request; MLE_INVALID for a bad theta (the request is not run).
int prepare(mle_ctx* c, const double theta[3], int mode, Item* it) {
  it->c = c;
  it->mode = mode;
  if (!theta) return fail(MLE_INVALID, "theta is null");
  if (mle_fill_theta(theta, c->nugget, &it->P) != 0)
    return fail(MLE_INVALID, "MaternParams components must be finite and > 0");
  it->factor = !same_theta(c, theta);
  it->derivs = (mode == 2);
  const bool spec_hit = !it->factor && c->spec_ready && c->spec_theta[0] == theta[0] &&
                        c->spec_theta[1] == theta[1] && c->spec_theta[2] == theta[2];
  it->gen_derivs = it->derivs && !spec_hit;
  it->need_w = it->derivs && !spec_hit;
  it->spec = mode == 1 && it->factor && c->ozaki && c->sa && c->sn && c->wsl &&
             use_speculation();
  return MLE_OK;
}

// loglik at the resident factor's theta: the pass would only rerun the deterministic
// reduction over the same L, so its value is known on the host (bit-identical).
bool loglik_cached(Item* it) {
  if (it->mode != 1 || it->factor) return false;
  it->rc = MLE_OK;
  it->pivot = -1;
  std::memset(it->res, 0, sizeof(it->res));
  it->res[0] = it->c->cached_ll;
  return true;
}

int check_finite(const double* v, int64_t m, const char* what) {
  for (int64_t i = 0; i < m; ++i)
    if (!std::isfinite(v[i])) return fail(MLE_INVALID, std::string(what) + " must be finite");
  return MLE_OK;
}

// eval_all of a sequential-derivative context (mle_ctx::seq_derivs: the derivative blocks do
// not fit beside the factor).  Same arithmetic per block as the batched two-sided path --
// generation, the sygst-style reduction B_i = L^-1 S_i L^-T on the Ozaki GEMM -- but one
// block at a time in the single work matrix: the factor first (a loglik pass, or the resident
// one), then for each block generate -> reduce -> sums against the parked blocks -> park.
// Replaces likelihood.py:107-149 exactly as eval_all does; the Frobenius sums run in a
// different (still fixed) order than launch_reduce's.
int eval_all_seq(mle_ctx* c, const double theta[3], double* res, int64_t* bad_pivot) {
  Item it;
  int rc = prepare(c, theta, 1, &it);
  if (rc) return rc;
  it.spec = false;
  if (it.factor) {
    rc = run_batch(&it, 1);
    if (rc) return rc;
    if (bad_pivot) *bad_pivot = it.pivot;
    if (it.rc == MLE_NOT_PD)
      return fail(MLE_NOT_PD,
                  "matrix not positive definite at pivot " + std::to_string(it.pivot));
  } else if (bad_pivot) {
    *bad_pivot = -1;
  }
  CUDA_TRY(cudaSetDevice(c->device));
  if ((rc = wait_spec(c, c->stream))) return rc;
  if ((rc = ensure_matrices(c, true))) return rc;
  ThetaParams P = it.P;
  if (use_gen_table())
    mle_fill_gen_table(c->h_max / P.alpha, &P);
  else
    P.tab_n = 0;
  cudaStream_t s = c->stream;
  std::memcpy(c->h_theta, &P, sizeof(ThetaParams));
  CUDA_TRY(cudaMemcpyAsync(c->d_theta, c->h_theta, sizeof(ThetaParams), cudaMemcpyHostToDevice,
                           s));
  const bool lookahead = !c->kprof && use_lookahead();
  Launcher run{s, lookahead ? c->side : nullptr, c->pool, kPoolEvents};
  if (c->kprof) run.prof = c;
  NvtxPhases nvtx;
  nvtx.push("mle eval_all (sequential derivative blocks)");
  const int nmat = c->nugget > 0.0 ? 3 : 2;
  const long long N = c->N;
  const int n = (int)c->n;
  double r[kReduceOut] = {};
  r[0] = c->cached_logdet;
  r[1] = c->cached_quad;
  r[kReduceSums + 3] = c->cached_dmin;
  r[kReduceSums + 4] = c->cached_dmax;
  GenArgs ga;
  std::memset(&ga, 0, sizeof(ga));
  {
    GenItem& gi = ga.item[0];
    gi.P = c->d_theta;
    gi.lx = c->lx;
    gi.ly = c->ly;
    gi.z = c->z;
    gi.sigma = c->sigma;
    gi.fail_flag = c->fail_flag;
    gi.tab = P.tab_n > 0 ? c->gtab_d : nullptr;
    gi.write_sigma = 0;
    gi.write_derivs = 1;
    ga.lower_only = 1;
    ga.ld = N;
    ga.rows = N;
    ga.n = n;
  }
  c->deriv_lower = true;
  c->spec_ready = false;
  CUDA_TRY(cudaEventRecord(c->ev[2], s));
  run.launches += 1;
  launch_gen_table(ga, 1, true, s);
  CUDA_TRY(cudaGetLastError());
  double gen_ms = 0.0;
  for (int w = 0; w < nmat; ++w) {
    nvtx.push(w == 0 ? "block alpha" : w == 1 ? "block nu" : "block M");
    run.launches += 1;
    if (w < 2) {
      ga.item[0].dalpha = w == 0 ? c->sa : nullptr;
      ga.item[0].dnu = w == 1 ? c->sa : nullptr;
      launch_gen_engine(ga, 1, s);
      CUDA_TRY(cudaGetLastError());
    } else {
      CUDA_TRY(launch_set_identity_lower(c->sa, N, n, (int)N, s));
    }
    MatList ml(c, w);
    if ((rc = run.solves_2s(ml))) return rc;
    // parked so far: alpha above sigma's band (w >= 1), nu above the work matrix's own (w == 2)
    const double* u1 = w >= 1 ? c->sigma : nullptr;
    const double* u2 = w == 2 ? c->sa : nullptr;
    run.launches += 2;
    CUDA_TRY(launch_seq_reduce(c->sa, u1, u2, N, n, (int)N, c->partials, c->out, s));
    CUDA_TRY(cudaMemcpyAsync(c->h_res, c->out, sizeof(double) * 5, cudaMemcpyDeviceToHost, s));
    if (w + 1 < nmat) {
      run.launches += 1;
      CUDA_TRY(launch_park_lower(c->sa, w == 0 ? c->sigma : c->sa, N, (int)N, s));
    }
    CUDA_TRY(cudaStreamSynchronize(s));
    const double tr = c->h_res[0], ww = c->h_res[1], wu1 = c->h_res[2], wu2 = c->h_res[3];
    const double yby = c->h_res[4];
    if (w == 0) {
      r[2] = tr; r[4] = ww; r[kReduceSums] = yby;
    } else if (w == 1) {
      r[3] = tr; r[6] = ww; r[5] = wu1; r[kReduceSums + 1] = yby;
    } else {
      r[7] = tr; r[10] = ww; r[8] = wu1; r[9] = wu2; r[kReduceSums + 2] = yby;
    }
    nvtx.pop();
  }
  CUDA_TRY(cudaEventRecord(c->ev[3], s));
  CUDA_TRY(cudaStreamSynchronize(s));
  CUDA_TRY(cudaGetLastError());
  if ((rc = run.prof_collect())) return rc;
  float solve_ms = 0.f;
  CUDA_TRY(cudaEventElapsedTime(&solve_ms, c->ev[2], c->ev[3]));
  int flag = 0;
  CUDA_TRY(cudaMemcpy(&flag, c->fail_flag, sizeof(int), cudaMemcpyDeviceToHost));
  if (flag) return fail(MLE_CUDA_ERROR, "failure flag set during the derivative blocks");
  if (!it.factor)
    for (int p = 0; p < MLE_NUM_PHASES; ++p) c->phase_ms[p] = 0.0;
  (void)gen_ms;
  c->phase_ms[MLE_PHASE_SOLVE] = solve_ms;
  c->phase_ms[MLE_PHASE_TOTAL] = c->phase_ms[MLE_PHASE_GEN] + c->phase_ms[MLE_PHASE_POTRF] +
                                 c->phase_ms[MLE_PHASE_REDUCE] + solve_ms;
  const double nd = (double)c->n;
  c->flops = (it.factor ? nd * nd * nd / 3.0 : 0.0) + nmat * nd * nd * nd;
  c->gen_bytes = (it.factor ? 1.0 : 0.0) * 8.0 * nd * (nd + 1.0) / 2.0 +
                 2.0 * 8.0 * nd * (nd + 1.0) / 2.0;
  c->launches = (it.factor ? c->launches : 0.0) + run.launches;
  double o[kResults] = {};
  assemble_results(c, P, r, 2, o);
  std::memcpy(res, o, sizeof(double) * kResults);
  return MLE_OK;
}

int single(mle_ctx* c, const double theta[3], int mode, double* res, int64_t* bad_pivot) {
  if (c->seq_derivs && mode == 2) return eval_all_seq(c, theta, res, bad_pivot);
  Item it;
  int rc = prepare(c, theta, mode, &it);
  if (rc) return rc;
  if (!loglik_cached(&it)) {
    rc = run_batch(&it, 1);
    if (rc) return rc;
  }
  if (bad_pivot) *bad_pivot = it.pivot;
  if (it.rc == MLE_NOT_PD)
    return fail(MLE_NOT_PD, "matrix not positive definite at pivot " + std::to_string(it.pivot));
  std::memcpy(res, it.res, sizeof(double) * kResults);
  return MLE_OK;
}

}  // namespace

extern "C" {

const char* mle_version(void) { return "maternfisher-b200 0.2.0 (sm_100a)"; }
const char* mle_last_error(void) { return g_last_error.c_str(); }

int mle_device_count(void) {
  int count = 0;
  if (cudaGetDeviceCount(&count) != cudaSuccess) return 0;
  return count;
}

int mle_kernel_profile(mle_ctx* ctx, int enable) {
  if (!ctx) return fail(MLE_INVALID, "null context");
  ctx->kprof = enable != 0;
  std::memset(ctx->kstats, 0, sizeof(ctx->kstats));
  return MLE_OK;
}

int mle_kernel_stats(const mle_ctx* ctx, double* out) {
  if (!ctx || !out) return fail(MLE_INVALID, "null argument");
  std::memcpy(out, ctx->kstats, sizeof(ctx->kstats));
  return MLE_OK;
}

int mle_ctx_cond_estimate(const mle_ctx* ctx, double* out) {
  if (!ctx || !out) return fail(MLE_INVALID, "null argument");
  *out = ctx->cond_est;
  return MLE_OK;
}

// Developer diagnostics (not in the public header): trace every potrf_diag_kernel CTA into a
// device buffer of `cap` records of 6 int64 (enable = 1), or stop and copy the records to
// `host` (enable = 0; *count = records written).
int mle_ctx_seq_derivs(const mle_ctx* ctx) { return ctx && ctx->seq_derivs ? 1 : 0; }

int mle_diag_trace(int enable, long long cap, long long* host, long long* count) {
  static long long* dbuf = nullptr;
  static long long dcap = 0;
  if (enable) {
    if (dbuf) cudaFree(dbuf);
    CUDA_TRY(cudaMalloc(&dbuf, sizeof(long long) * 6 * (size_t)cap));
    dcap = cap;
    CUDA_TRY(diag_trace_control(dbuf, (unsigned long long)cap, nullptr));
    return MLE_OK;
  }
  unsigned long long n = 0;
  CUDA_TRY(diag_trace_control(nullptr, 0, &n));
  if (count) *count = (long long)n;
  if (host && dbuf) {
    const size_t m = (size_t)std::min<long long>((long long)n, dcap);
    CUDA_TRY(cudaMemcpy(host, dbuf, sizeof(long long) * 6 * m, cudaMemcpyDeviceToHost));
  }
  return MLE_OK;
}

int mle_release_cached_memory(void) {
  cache_trim(-2);
  std::lock_guard<std::mutex> lock(g_sets_mutex);
  for (size_t d = 0; d < g_sets.size(); ++d) {
    if (g_sets[d].empty()) continue;
    cudaSetDevice((int)d);
    for (StreamSet& st : g_sets[d]) {
      for (cudaEvent_t e : st.ev) cudaEventDestroy(e);
      for (cudaEvent_t e : st.pool) cudaEventDestroy(e);
      for (cudaEvent_t e : st.clk)
        if (e) cudaEventDestroy(e);
      cudaEventDestroy(st.ev_der);
      cudaEventDestroy(st.spec_done);
      for (cudaStream_t q : {st.stream, st.side, st.inner, st.aux}) cudaStreamDestroy(q);
    }
    g_sets[d].clear();
  }
  return MLE_OK;
}

static int create_ctx_aligned(const double* locs_xy, const double* z, int64_t n, int device,
                              double nugget, long long align, mle_ctx** out);

// Sequential-derivative mode is chosen when the context is created (its matrices get the
// parking columns): when Sigma + the derivative blocks + the factor's and W's slices exceed
// the device memory, or with MLE_SEQ_DERIVS=1 (tests at small n; needs the two-sided path).
static bool want_seq_derivs(const mle_ctx* c) {
  if (!c->ozaki || solve_slices() != kOzSlices) return false;
  const char* e = std::getenv("MLE_SEQ_DERIVS");
  if (e && e[0] == '1') return use_two_sided(c->N);
  if (e && e[0] == '0') return false;
  if (!use_two_sided(c->N)) return false;
  size_t free_b = 0, total_b = 0;
  if (cudaMemGetInfo(&free_b, &total_b) != cudaSuccess) {
    cudaGetLastError();
    return false;
  }
  const double N = (double)c->N;
  const double mats = (c->nugget > 0.0 ? 4.0 : 3.0) * 8.0 * N * N;
  const double slices = 2.0 * (double)kOzSlices * N * N / 2.0;  // factor panels + W blocks
  return mats + slices + 6e9 > (double)total_b;
}

int mle_ctx_create(const double* locs_xy, const double* z, int64_t n, int device, double nugget,
                   mle_ctx** out) {
  int rc = create_ctx_aligned(locs_xy, z, n, device, nugget, kNB, out);
  if (rc == MLE_OK) (*out)->seq_derivs = want_seq_derivs(*out);
  return rc;
}

static int create_ctx_aligned(const double* locs_xy, const double* z, int64_t n, int device,
                              double nugget, long long align, mle_ctx** out) {
  if (!out) return fail(MLE_INVALID, "out is null");
  *out = nullptr;
  if (!locs_xy || !z || n < 1) return fail(MLE_INVALID, "at least one location is required");
  if (n > 2000000000LL / 32) return fail(MLE_INVALID, "n too large");
  int rc = check_finite(locs_xy, 2 * n, "locations");
  if (rc) return rc;
  rc = check_finite(z, n, "values");
  if (rc) return rc;
  if (!(std::isfinite(nugget) && nugget >= 0.0)) return fail(MLE_INVALID, "nugget must be >= 0");
  rc = ensure_device(device);
  if (rc) return rc;
  mle_ctx* c = new mle_ctx();
  c->device = device;
  c->n = n;
  c->N = round_up(n + 1, align);
  c->Nt = (int)(c->N / kNB);
  c->nugget = nugget;
  c->ozaki = use_ozaki();
  std::vector<double> x(n), y(n);
  for (int64_t i = 0; i < n; ++i) {
    x[i] = locs_xy[2 * i];
    y[i] = locs_xy[2 * i + 1];
  }
  auto bail = [&](int code) {
    mle_ctx_destroy(c);
    return code;
  };
#define CTX_TRY(expr)                                                                  \
  do {                                                                                 \
    cudaError_t _e = (expr);                                                           \
    if (_e != cudaSuccess)                                                             \
      return bail(fail(MLE_CUDA_ERROR, std::string(#expr) + ": " + cudaGetErrorString(_e))); \
  } while (0)
  // Priorities: the latency-bound factorization chain (main, look-ahead) wins SMs over the
  // throughput work on aux (derivative generation, speculation) as CTAs retire.
  bool recycled = false;
  {
    std::lock_guard<std::mutex> lock(g_sets_mutex);
    if ((int)g_sets.size() > device && !g_sets[device].empty()) {
      const StreamSet st = g_sets[device].back();
      g_sets[device].pop_back();
      c->stream = st.stream;
      c->side = st.side;
      c->inner = st.inner;
      c->aux = st.aux;
      c->edge = st.edge;
      for (int i = 0; i < 5; ++i) c->ev[i] = st.ev[i];
      c->ev_der = st.ev_der;
      c->spec_done = st.spec_done;
      for (int i = 0; i < kPoolEvents; ++i) c->pool[i] = st.pool[i];
      c->pass_clock.start = st.clk[0];
      c->pass_clock.pre = st.clk[1];
      c->pass_clock.end[0] = st.clk[2];
      c->pass_clock.end[1] = st.clk[3];
      recycled = true;
    }
  }
  if (!recycled) {
    int prio_low = 0, prio_high = 0;
    CTX_TRY(cudaDeviceGetStreamPriorityRange(&prio_low, &prio_high));
    CTX_TRY(cudaStreamCreateWithPriority(&c->stream, cudaStreamNonBlocking, prio_high));
    CTX_TRY(cudaStreamCreateWithPriority(&c->side, cudaStreamNonBlocking, prio_high));
    CTX_TRY(cudaStreamCreateWithPriority(&c->inner, cudaStreamNonBlocking, prio_high));
    CTX_TRY(cudaStreamCreateWithPriority(&c->aux, cudaStreamNonBlocking, prio_low));
    CTX_TRY(cudaStreamCreateWithPriority(&c->edge, cudaStreamNonBlocking, prio_high));
    for (auto& e : c->ev) CTX_TRY(cudaEventCreate(&e));
    CTX_TRY(cudaEventCreateWithFlags(&c->ev_der, cudaEventDisableTiming));
    CTX_TRY(cudaEventCreateWithFlags(&c->spec_done, cudaEventDisableTiming));
    for (auto& e : c->pool) CTX_TRY(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
  }
  CTX_TRY(dmalloc(&c->lx, sizeof(double) * n));
  CTX_TRY(dmalloc(&c->ly, sizeof(double) * n));
  CTX_TRY(dmalloc(&c->z, sizeof(double) * n));
  CTX_TRY(dmalloc(&c->fail_flag, sizeof(int)));
  CTX_TRY(dmalloc(&c->fail_idx, sizeof(long long)));
  CTX_TRY(dmalloc(&c->partials, sizeof(double) * kReduceBlocks * kReducePartials));
  CTX_TRY(dmalloc(&c->out, sizeof(double) * kReduceOut));
  CTX_TRY(dmalloc(&c->d_theta, sizeof(ThetaParams)));
  CTX_TRY(dmalloc(&c->gtab_s, sizeof(double) * MLE_TAB_DOUBLES));
  CTX_TRY(dmalloc(&c->gtab_d, sizeof(double) * MLE_TAB_DOUBLES));
  {
    double x0 = x[0], x1 = x[0], y0 = y[0], y1 = y[0];
    for (int64_t i = 1; i < n; ++i) {
      x0 = std::fmin(x0, x[i]);
      x1 = std::fmax(x1, x[i]);
      y0 = std::fmin(y0, y[i]);
      y1 = std::fmax(y1, y[i]);
    }
    c->h_max = std::hypot(x1 - x0, y1 - y0);
  }
  CTX_TRY(hmalloc(&c->h_theta, sizeof(ThetaParams)));
  CTX_TRY(hmalloc(&c->h_stage, sizeof(ThetaParams) * kMaxItems));
  CTX_TRY(dmalloc(&c->d_stage, sizeof(ThetaParams) * kMaxItems));
  CTX_TRY(hmalloc(&c->h_resb, sizeof(double) * kMaxItems * (kReduceOut + 2)));
  CTX_TRY(dmalloc(&c->d_resb, sizeof(double) * kMaxItems * (kReduceOut + 2)));
  CTX_TRY(hmalloc(&c->h_res, sizeof(double) * (kReduceOut + 2)));
  CTX_TRY(cudaMemcpyAsync(c->lx, x.data(), sizeof(double) * n, cudaMemcpyHostToDevice, c->stream));
  CTX_TRY(cudaMemcpyAsync(c->ly, y.data(), sizeof(double) * n, cudaMemcpyHostToDevice, c->stream));
  CTX_TRY(cudaMemcpyAsync(c->z, z, sizeof(double) * n, cudaMemcpyHostToDevice, c->stream));
  CTX_TRY(cudaMemsetAsync(c->fail_flag, 0, sizeof(int), c->stream));
  CTX_TRY(cudaStreamSynchronize(c->stream));
#undef CTX_TRY
  *out = c;
  return MLE_OK;
}

void mle_ctx_destroy(mle_ctx* c) {
  if (!c) return;
  cudaSetDevice(c->device);
  if (c->spec_pending && c->spec_done) cudaEventSynchronize(c->spec_done);
  if (c->stream) cudaStreamSynchronize(c->stream);
  dfree(c->lx);
  dfree(c->ly);
  dfree(c->z);
  dfree(c->sigma);
  dfree(c->sa);
  dfree(c->sn);
  dfree(c->smat);
  dfree(c->linv);
  dfree(c->fail_flag);
  dfree(c->fail_idx);
  dfree(c->partials);
  dfree(c->out);
  dfree(c->d_theta);
  dfree(c->d_stage);
  dfree(c->d_resb);
  if (c->h_stage) dfree(c->h_stage);
  if (c->h_resb) dfree(c->h_resb);
  dfree(c->gtab_s);
  dfree(c->gtab_d);
  if (!c->seq_derivs) dfree(c->lsl);
  dfree(c->lex);
  dfree(c->psl);
  dfree(c->pex);
  dfree(c->xsl);
  dfree(c->xex);
  dfree(c->dinv);
  dfree(c->tscr);
  dfree(c->wbuf);
  dfree(c->dtsl);
  dfree(c->dtex);
  dfree(c->wsl);
  dfree(c->wex);
  if (c->h_theta) dfree(c->h_theta);
  if (c->h_res) dfree(c->h_res);
  for (auto& e : c->kev) cudaEventDestroy(e);
  bool complete = c->stream && c->side && c->inner && c->aux && c->edge && c->ev_der &&
                  c->spec_done;
  for (auto& e : c->ev) complete = complete && e;
  for (auto& e : c->pool) complete = complete && e;
  const bool idle = complete && cudaStreamSynchronize(c->side) == cudaSuccess &&
                    cudaStreamSynchronize(c->inner) == cudaSuccess &&
                    cudaStreamSynchronize(c->aux) == cudaSuccess &&
                    cudaStreamSynchronize(c->edge) == cudaSuccess;
  if (idle) {  // hand the stream set to the next context on this device
    StreamSet st;
    st.stream = c->stream;
    st.side = c->side;
    st.inner = c->inner;
    st.aux = c->aux;
    st.edge = c->edge;
    for (int i = 0; i < 5; ++i) st.ev[i] = c->ev[i];
    st.ev_der = c->ev_der;
    st.spec_done = c->spec_done;
    for (int i = 0; i < kPoolEvents; ++i) st.pool[i] = c->pool[i];
    st.clk[0] = c->pass_clock.start;
    st.clk[1] = c->pass_clock.pre;
    st.clk[2] = c->pass_clock.end[0];
    st.clk[3] = c->pass_clock.end[1];
    std::lock_guard<std::mutex> lock(g_sets_mutex);
    if ((int)g_sets.size() <= c->device) g_sets.resize(c->device + 1);
    g_sets[c->device].push_back(st);
  } else {
    for (cudaEvent_t e : {c->pass_clock.start, c->pass_clock.pre, c->pass_clock.end[0],
                          c->pass_clock.end[1]})
      if (e) cudaEventDestroy(e);
    for (auto& e : c->ev)
      if (e) cudaEventDestroy(e);
    for (auto& e : c->pool)
      if (e) cudaEventDestroy(e);
    if (c->ev_der) cudaEventDestroy(c->ev_der);
    if (c->spec_done) cudaEventDestroy(c->spec_done);
    if (c->side) cudaStreamDestroy(c->side);
    if (c->inner) cudaStreamDestroy(c->inner);
    if (c->aux) cudaStreamDestroy(c->aux);
    if (c->edge) cudaStreamDestroy(c->edge);
    if (c->stream) cudaStreamDestroy(c->stream);
  }
  delete c;
}

int64_t mle_ctx_n(const mle_ctx* c) { return c ? c->n : -1; }

int mle_ctx_set_values(mle_ctx* c, const double* z) {
  if (!c || !z) return fail(MLE_INVALID, "null argument");
  int rc = check_finite(z, c->n, "values");
  if (rc) return rc;
  CUDA_TRY(cudaSetDevice(c->device));
  if ((rc = wait_spec(c, c->stream))) return rc;
  CUDA_TRY(cudaMemcpyAsync(c->z, z, sizeof(double) * c->n, cudaMemcpyHostToDevice, c->stream));
  CUDA_TRY(cudaStreamSynchronize(c->stream));
  c->factor_valid = false;  // row n of L carries L^-1 z
  c->spec_ready = false;
  return MLE_OK;
}

int mle_loglik(mle_ctx* c, const double theta[3], double* loglik, int64_t* bad_pivot) {
  if (!c || !loglik) return fail(MLE_INVALID, "null argument");
  double res[kResults];
  int rc = single(c, theta, 1, res, bad_pivot);
  if (rc) return rc;
  *loglik = res[0];
  return MLE_OK;
}

int mle_eval_all(mle_ctx* c, const double theta[3], double* loglik, double grad[3],
                 double fisher[9], int64_t* bad_pivot) {
  if (!c || !loglik || !grad || !fisher) return fail(MLE_INVALID, "null argument");
  double res[kResults];
  int rc = single(c, theta, 2, res, bad_pivot);
  if (rc) return rc;
  *loglik = res[0];
  std::memcpy(grad, res + 1, sizeof(double) * 3);
  std::memcpy(fisher, res + 4, sizeof(double) * 9);
  return MLE_OK;
}

int mle_eval_batch(mle_ctx* const* ctxs, int count, const double* thetas, const int* modes,
                   double* results, int64_t* pivots, int* rcs) {
  if (count < 0 || (count > 0 && (!ctxs || !thetas || !modes || !results || !rcs)))
    return fail(MLE_INVALID, "null argument");
  std::vector<Item> items;
  std::vector<int> slot;
  std::vector<mle_ctx*> cached;  // answered from the resident factor, no pass
  std::string bad;
  for (int i = 0; i < count; ++i) {
    rcs[i] = MLE_OK;
    if (pivots) pivots[i] = -1;
    if (modes[i] == 0) continue;
    if (!ctxs[i] || (modes[i] != 1 && modes[i] != 2)) return fail(MLE_INVALID, "bad request");
    for (int j = 0; j < i; ++j)
      if (modes[j] != 0 && ctxs[j] == ctxs[i])
        return fail(MLE_INVALID, "a context may appear once per batch");
    Item it;
    if (ctxs[i]->seq_derivs && modes[i] == 2) {  // one block at a time: not batched
      int64_t piv = -1;
      const int rc1 = eval_all_seq(ctxs[i], thetas + 3 * i, results + (size_t)kResults * i, &piv);
      if (rc1 == MLE_CUDA_ERROR) return rc1;
      rcs[i] = rc1;
      if (pivots) pivots[i] = piv;
      if (rc1 != MLE_OK) bad = g_last_error;
      continue;
    }
    if (prepare(ctxs[i], thetas + 3 * i, modes[i], &it) != MLE_OK) {
      rcs[i] = MLE_INVALID;
      bad = g_last_error;
      continue;
    }
    if (loglik_cached(&it)) {
      std::memcpy(results + (size_t)kResults * i, it.res, sizeof(double) * kResults);
      cached.push_back(it.c);
      continue;
    }
    items.push_back(it);
    slot.push_back(i);
  }
  // group by (device, N): every chunk must share them
  std::vector<char> done(items.size(), 0);
  for (size_t a = 0; a < items.size(); ++a) {
    if (done[a]) continue;
    std::vector<Item> group;
    std::vector<int> gslot;
    for (size_t b = a; b < items.size(); ++b)
      if (!done[b] && items[b].c->device == items[a].c->device && items[b].c->N == items[a].c->N) {
        group.push_back(items[b]);
        gslot.push_back(slot[b]);
        done[b] = 1;
      }
    int rc = run_batch(group.data(), (int)group.size());
    if (rc) return rc;
    for (size_t g = 0; g < group.size(); ++g) {
      const int i = gslot[g];
      rcs[i] = group[g].rc;
      if (pivots) pivots[i] = group[g].pivot;
      std::memcpy(results + (size_t)kResults * i, group[g].res, sizeof(double) * kResults);
    }
  }
  // per-context pass statistics of the cached answers: those of this call's pass, or none
  for (mle_ctx* c : cached) {
    const mle_ctx* src = items.empty() ? nullptr : items[0].c;
    for (int p = 0; p < MLE_NUM_PHASES; ++p) c->phase_ms[p] = src ? src->phase_ms[p] : 0.0;
    c->flops = src ? src->flops : 0.0;
    c->gen_bytes = src ? src->gen_bytes : 0.0;
    c->launches = src ? src->launches : 0.0;
    for (int k = 7; k <= 9; ++k) c->kstats[k] = src ? src->kstats[k] : 0.0;
  }
  if (!bad.empty()) g_last_error = bad;
  return MLE_OK;
}

int mle_simulate(mle_ctx* c, const double theta[3], const double* w, double* z_out,
                 int64_t* bad_pivot) {
  if (!c || !w || !z_out) return fail(MLE_INVALID, "null argument");
  int rc = check_finite(w, c->n, "normals");
  if (rc) return rc;
  double res[kResults];
  rc = single(c, theta, 1, res, bad_pivot);  // factor Sigma(theta) (cached afterwards)
  if (rc) return rc;
  double *dw = nullptr, *dz = nullptr;
  struct G {
    double** a;
    double** b;
    ~G() {
      dfree(*a);
      dfree(*b);
    }
  } guard{&dw, &dz};
  CUDA_TRY(dmalloc(&dw, sizeof(double) * c->n));
  CUDA_TRY(dmalloc(&dz, sizeof(double) * c->n));
  CUDA_TRY(cudaMemcpyAsync(dw, w, sizeof(double) * c->n, cudaMemcpyHostToDevice, c->stream));
  CUDA_TRY(launch_trmv_lower(c->sigma, c->N, (int)c->n, dw, dz, c->stream));
  CUDA_TRY(cudaMemcpyAsync(z_out, dz, sizeof(double) * c->n, cudaMemcpyDeviceToHost, c->stream));
  CUDA_TRY(cudaStreamSynchronize(c->stream));
  return MLE_OK;
}

int mle_build(mle_ctx* c, const double theta[3], int which, double* out_host) {
  if (!c || !out_host) return fail(MLE_INVALID, "null argument");
  if (which < MLE_WHICH_SIGMA || which > MLE_WHICH_NU)
    return fail(MLE_INVALID, "which must be one of sigma, sigma2, alpha, nu");
  Item it;
  int rc = prepare(c, theta, 1, &it);
  if (rc) return rc;
  CUDA_TRY(cudaSetDevice(c->device));
  rc = ensure_matrices(c, false);
  if (rc) return rc;
  if ((rc = wait_spec(c, c->stream))) return rc;
  c->factor_valid = false;  // the Sigma buffer is reused as scratch
  c->spec_ready = false;
  std::memcpy(c->h_theta, &it.P, sizeof(ThetaParams));
  CUDA_TRY(cudaMemcpyAsync(c->d_theta, c->h_theta, sizeof(ThetaParams), cudaMemcpyHostToDevice,
                           c->stream));
  GenArgs a;
  std::memset(&a, 0, sizeof(a));
  a.item[0].P = c->d_theta;
  a.item[0].lx = c->lx;
  a.item[0].ly = c->ly;
  a.item[0].sigma = c->sigma;
  a.ld = c->n;
  a.rows = c->n;
  a.n = (int)c->n;
  launch_gen_build(a, which, c->stream);
  CUDA_TRY(cudaGetLastError());
  CUDA_TRY(cudaMemcpyAsync(out_host, c->sigma, sizeof(double) * (size_t)c->n * (size_t)c->n,
                           cudaMemcpyDeviceToHost, c->stream));
  CUDA_TRY(cudaStreamSynchronize(c->stream));
  return MLE_OK;
}

int64_t mle_launch_count(void) { return (int64_t)g_launch_total.load(); }

int mle_phase_times(const mle_ctx* c, double* out) {
  if (!c || !out) return fail(MLE_INVALID, "null argument");
  for (int p = 0; p < MLE_NUM_PHASES; ++p) out[p] = c->phase_ms[p];
  out[MLE_NUM_PHASES] = c->flops;
  out[MLE_NUM_PHASES + 1] = c->gen_bytes;
  out[MLE_NUM_PHASES + 2] = c->launches;
  return MLE_OK;
}

int mle_cholesky(const double* a, int64_t n, int device, double* l_out, int64_t* bad_pivot) {
  if (!a || !l_out || n < 1) return fail(MLE_INVALID, "cholesky_lower expects a square matrix");
  int rc = ensure_device(device);
  if (rc) return rc;
  mle_ctx c;
  c.device = device;
  c.n = n;
  c.N = round_up(n, kNB);
  c.Nt = (int)(c.N / kNB);
  const long long N = c.N;
  std::vector<double> h((size_t)N * N, 0.0);
  for (long long j = 0; j < N; ++j) {
    if (j >= n) h[j + j * N] = 1.0;
    else
      for (long long i = j; i < n; ++i) h[i + j * N] = a[i * n + j];  // logical lower of a
  }
  struct Guard {
    mle_ctx* c;
    ~Guard() {
      dfree(c->sigma);
      dfree(c->linv);
      dfree(c->fail_flag);
      dfree(c->fail_idx);
      dfree(c->lsl);
      dfree(c->lex);
      if (c->h_res) dfree(c->h_res);
      if (c->stream) cudaStreamDestroy(c->stream);
      c->sigma = c->linv = nullptr;
      c->fail_flag = nullptr;
      c->fail_idx = nullptr;
      c->h_res = nullptr;
      c->stream = nullptr;
    }
  } guard{&c};
  CUDA_TRY(cudaStreamCreateWithFlags(&c.stream, cudaStreamNonBlocking));
  CUDA_TRY(dmalloc(&c.sigma, sizeof(double) * (size_t)N * N));
  CUDA_TRY(dmalloc(&c.linv, sizeof(double) * (size_t)c.Nt * kNB * kNB));
  CUDA_TRY(dmalloc(&c.fail_flag, sizeof(int)));
  CUDA_TRY(dmalloc(&c.fail_idx, sizeof(long long)));
  CUDA_TRY(hmalloc(&c.h_res, sizeof(double) * 12));
  c.ozaki = use_ozaki();
  if ((rc = ensure_ozaki(&c, false))) return rc;
  CUDA_TRY(cudaMemcpyAsync(c.sigma, h.data(), sizeof(double) * (size_t)N * N,
                           cudaMemcpyHostToDevice, c.stream));
  CUDA_TRY(cudaMemsetAsync(c.fail_flag, 0, sizeof(int), c.stream));
  Launcher run{c.stream};  // single stream (no look-ahead) for the standalone factorization
  mle_ctx* cs[1] = {&c};
  double* mats[1] = {c.sigma};
  long long aug[1] = {-1};
  rc = run.potrf(cs, mats, aug, 1);
  if (rc) return rc;
  CUDA_TRY(cudaMemcpyAsync(h.data(), c.sigma, sizeof(double) * (size_t)N * N,
                           cudaMemcpyDeviceToHost, c.stream));
  CUDA_TRY(cudaMemcpyAsync(c.h_res + 9, c.fail_flag, sizeof(int), cudaMemcpyDeviceToHost,
                           c.stream));
  CUDA_TRY(cudaMemcpyAsync(c.h_res + 10, c.fail_idx, sizeof(long long), cudaMemcpyDeviceToHost,
                           c.stream));
  CUDA_TRY(cudaStreamSynchronize(c.stream));
  int flag;
  std::memcpy(&flag, c.h_res + 9, sizeof(int));
  if (flag) {
    long long idx;
    std::memcpy(&idx, c.h_res + 10, sizeof(long long));
    if (bad_pivot) *bad_pivot = idx;
    return fail(MLE_NOT_PD, "matrix not positive definite at pivot " + std::to_string(idx));
  }
  for (long long i = 0; i < n; ++i)
    for (long long j = 0; j < n; ++j) l_out[i * n + j] = (j <= i) ? h[i + j * N] : 0.0;
  if (bad_pivot) *bad_pivot = -1;
  return MLE_OK;
}

static int run_elem(int op, const ThetaParams& P, int which, const double* x, int64_t m,
                    int device, double* out) {
  int rc = ensure_device(device);
  if (rc) return rc;
  if (m == 0) return MLE_OK;
  double *dx = nullptr, *dy = nullptr;
  ThetaParams* dP = nullptr;
  cudaStream_t s = nullptr;
  struct G {
    double** a;
    double** b;
    ThetaParams** p;
    cudaStream_t* s;
    ~G() {
      dfree(*a);
      dfree(*b);
      dfree(*p);
      if (*s) cudaStreamDestroy(*s);
    }
  } guard{&dx, &dy, &dP, &s};
  CUDA_TRY(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking));
  CUDA_TRY(dmalloc(&dx, sizeof(double) * m));
  CUDA_TRY(dmalloc(&dy, sizeof(double) * m));
  CUDA_TRY(dmalloc(&dP, sizeof(ThetaParams)));
  CUDA_TRY(cudaMemcpyAsync(dP, &P, sizeof(ThetaParams), cudaMemcpyHostToDevice, s));
  CUDA_TRY(cudaMemcpyAsync(dx, x, sizeof(double) * m, cudaMemcpyHostToDevice, s));
  launch_elem(dP, op, which, dx, m, dy, s);
  CUDA_TRY(cudaGetLastError());
  CUDA_TRY(cudaMemcpyAsync(out, dy, sizeof(double) * m, cudaMemcpyDeviceToHost, s));
  CUDA_TRY(cudaStreamSynchronize(s));
  return MLE_OK;
}

int mle_bessel_k(double nu, const double* x, int64_t m, int device, double* out) {
  if ((!x || !out) && m > 0) return fail(MLE_INVALID, "null argument");
  if (!std::isfinite(nu)) return fail(MLE_INVALID, "bessel_k requires finite nu and x");
  for (int64_t i = 0; i < m; ++i) {
    if (!std::isfinite(x[i])) return fail(MLE_INVALID, "bessel_k requires finite nu and x");
    if (x[i] <= 0.0) return fail(MLE_INVALID, "bessel_k requires x > 0");
  }
  ThetaParams P;
  const double th[3] = {1.0, 1.0, 1.0};
  mle_fill_theta(th, 0.0, &P);
  mle_fill_ladder(std::fabs(nu), &P.kmain);  // K_nu = K_{-nu} (bessel.py:97)
  return run_elem(0, P, 0, x, m, device, out);
}

int mle_dnu_xnu_knu(double nu, const double* x, int64_t m, int device, double* out) {
  if ((!x || !out) && m > 0) return fail(MLE_INVALID, "null argument");
  if (!std::isfinite(nu) || nu <= 0.0) return fail(MLE_INVALID, "dnu_xnu_knu requires nu > 0");
  for (int64_t i = 0; i < m; ++i)
    if (!(std::isfinite(x[i]) && x[i] >= 0.0))
      return fail(MLE_INVALID, "dnu_xnu_knu requires finite x >= 0");
  ThetaParams P;
  const double th[3] = {1.0, 1.0, nu};
  if (mle_fill_theta(th, 0.0, &P) != 0) return fail(MLE_INVALID, "invalid nu");
  return run_elem(1, P, 0, x, m, device, out);
}

int mle_dnu_series(int which_case, double nu, const double* x, int64_t m, int device,
                   double* out) {
  if ((!x || !out) && m > 0) return fail(MLE_INVALID, "null argument");
  if (which_case < 2 || which_case > 4) return fail(MLE_INVALID, "series must be 2, 3 or 4");
  if (!std::isfinite(nu)) return fail(MLE_INVALID, "series requires finite nu");
  for (int64_t i = 0; i < m; ++i) {
    const double v = x[i];
    if (which_case == 2 && !(v > 0.0 && v < MLE_SMALL_MID_SPLIT))  // bessel.py:196-197
      return fail(MLE_INVALID, "case2_series requires 0 < x < 8.5");
    if (which_case == 3 && !(v >= MLE_SMALL_MID_SPLIT && v < MLE_MID_LARGE_SPLIT))  // :237-238
      return fail(MLE_INVALID, "case3_series requires 8.5 <= x < 30");
    if (which_case == 4 && !(v >= MLE_MID_LARGE_SPLIT))  // bessel.py:299-300
      return fail(MLE_INVALID, "case4_series requires x >= 30");
  }
  if (which_case == 2 && std::fabs(nu - std::nearbyint(nu)) <= 1e-6)  // bessel.py:198-199
    return fail(MLE_INVALID, "case2_series requires nu away from integers");
  if (nu <= 0.0) return fail(MLE_INVALID, "series requires nu > 0");
  ThetaParams P;
  const double th[3] = {1.0, 1.0, nu};
  if (mle_fill_theta(th, 0.0, &P) != 0) return fail(MLE_INVALID, "invalid nu");
  return run_elem(3, P, which_case, x, m, device, out);
}

int mle_digamma(const double* x, int64_t m, double* out) {
  if ((!x || !out) && m > 0) return fail(MLE_INVALID, "null argument");
  for (int64_t i = 0; i < m; ++i)
    if (x[i] <= 0.0 && x[i] == std::floor(x[i]))  // bessel.py:111-112
      return fail(MLE_INVALID, "digamma has poles at non-positive integers");
  for (int64_t i = 0; i < m; ++i) out[i] = mle_digamma_host(x[i]);
  return MLE_OK;
}

int mle_matern_elem(const double theta[3], int which, const double* h, int64_t m, int device,
                    double* out) {
  if ((!h || !out) && m > 0) return fail(MLE_INVALID, "null argument");
  if (which < MLE_WHICH_SIGMA || which > MLE_WHICH_NU) return fail(MLE_INVALID, "bad which");
  ThetaParams P;
  if (!theta || mle_fill_theta(theta, 0.0, &P) != 0)
    return fail(MLE_INVALID, "MaternParams components must be finite and > 0");
  for (int64_t i = 0; i < m; ++i)
    if (!(h[i] >= 0.0)) return fail(MLE_INVALID, "distances must be non-negative");
  return run_elem(2, P, which, h, m, device, out);
}

}  // extern "C"

// ---- distributed engine: one rank's column panels -----------------------------------------
// Outer blocks of 512 columns are owned cyclically (block b by rank b % world).  A rank holds,
// for each owned block, the full-height column panel of Sigma -> L and of every derivative
// block (N x 512, ld = N; N a multiple of 512).  The Python driver (distributed.py) sequences
// the block steps and the collectives; each entry point below runs one rank's share of one
// step on its stream and returns after the stream has drained (the exchange buffers are then
// ready for NCCL on any stream).  Kernels are the single-GPU engine's, addressed through
// "virtual" base pointers vb = panel - c0 N, so that element (i, j) is vb[i + j N].
struct mle_dctx {
  mle_ctx* c = nullptr;
  int rank = 0, world = 1, nb = 0, nmat = 2;
  bool derivs = false;
  std::vector<int> owned;                      // blocks owned by this rank, ascending
  std::vector<double*> sig, mat[3];            // per owned block: panels
  std::vector<int8_t*> lsl;                    // per owned block: P_b slices (rows c1..N)
  std::vector<int*> lex;
  std::vector<int8_t*> wsl;                    // per owned block: W_b slices (rows c0..N)
  std::vector<int*> wex;
  std::vector<double*> dinv;                   // per owned block: D_b^-1 (512 x 512, ld 512)
  double* tscr = nullptr;                      // 128 x 512
  double* wbuf = nullptr;                      // N x 512
  int8_t* dtsl = nullptr;                      // D_b^-T slices
  int* dtex = nullptr;
  int8_t* xsl = nullptr;                       // forward-sweep operand slices
  int* xex = nullptr;
  double* part = nullptr;                      // panel reduce partials
  std::vector<double> h_part;
  bool async = false;                          // steps return without draining the stream
  // two-sided reduction (mle_dctx_2s_*): per derivative matrix a 512 x 512 scratch, the slices
  // of the current diagonal block and of the current S21 panel
  double* ts2 = nullptr;
  int8_t* a11sl = nullptr;
  int* a11ex = nullptr;
  int8_t* s21sl = nullptr;
  int* s21ex = nullptr;
  std::vector<int8_t*> wcache;                 // every block's W_b slices (right sweep), or empty
  std::vector<int*> wcache_e;
};

namespace {

constexpr long long kDB = 512;  // distributed block width

long long d_c0(int b) { return (long long)b * kDB; }
size_t d_pbytes(long long N) { return (size_t)(N - kDB) * kOzRowBytes; }  // P slices (max)
size_t d_wbytes(long long N) { return (size_t)N * kOzRowBytes; }          // W / X slices (max)
size_t d_xstride(long long N) { return d_wbytes(N) + sizeof(int) * (size_t)N; }

int d_index(const mle_dctx* d, int b) {
  for (size_t i = 0; i < d->owned.size(); ++i)
    if (d->owned[i] == b) return (int)i;
  return -1;
}

double* d_mat(const mle_dctx* d, int m, int q) {  // derivative block m of owned panel q
  return d->mat[m][q];
}

// End of a block step.  Synchronous mode drains the rank's streams (the exchange buffers are
// then ready for a collective on any stream).  Asynchronous mode (mle_dctx_set_async) only
// checks the launches: the work stays queued on the rank's stream (every step ends joined into
// it), and the caller orders its collectives against that stream with events.
int d_sync(mle_dctx* d) {
  if (!d->async) {
    CUDA_TRY(cudaStreamSynchronize(d->c->stream));
    CUDA_TRY(cudaStreamSynchronize(d->c->inner));
  }
  CUDA_TRY(cudaGetLastError());
  return MLE_OK;
}

bool d_in(int blk, int lo, int hi) { return blk >= lo && blk < hi; }

}  // namespace

extern "C" {

int mle_dctx_create(const double* locs_xy, const double* z, int64_t n, int device,
                    double nugget, int rank, int world, mle_dctx** out) {
  if (!out) return fail(MLE_INVALID, "out is null");
  *out = nullptr;
  if (world < 1 || rank < 0 || rank >= world) return fail(MLE_INVALID, "bad rank / world");
  mle_ctx* c = nullptr;
  int rc = create_ctx_aligned(locs_xy, z, n, device, nugget, kDB, &c);
  if (rc) return rc;
  mle_dctx* d = new mle_dctx();
  d->c = c;
  d->rank = rank;
  d->world = world;
  d->nb = (int)(c->N / kDB);
  d->nmat = nugget > 0.0 ? 3 : 2;
  for (int b = rank; b < d->nb; b += world) d->owned.push_back(b);
  *out = d;
  return MLE_OK;
}

void mle_dctx_destroy(mle_dctx* d) {
  if (!d) return;
  if (d->c) {
    cudaSetDevice(d->c->device);
    cudaStreamSynchronize(d->c->stream);
    cudaStreamSynchronize(d->c->inner);
  }
  for (auto* p : d->sig) dfree(p);
  for (auto& v : d->mat)
    for (auto* p : v) dfree(p);
  for (auto* p : d->lsl) dfree(p);
  for (auto* p : d->lex) dfree(p);
  for (auto* p : d->wsl) dfree(p);
  for (auto* p : d->wex) dfree(p);
  for (auto* p : d->dinv) dfree(p);
  dfree(d->tscr);
  dfree(d->wbuf);
  dfree(d->dtsl);
  dfree(d->dtex);
  dfree(d->xsl);
  dfree(d->xex);
  dfree(d->part);
  for (auto* p : d->wcache) dfree(p);
  for (auto* p : d->wcache_e) dfree(p);
  dfree(d->ts2);
  dfree(d->a11sl);
  dfree(d->a11ex);
  dfree(d->s21sl);
  dfree(d->s21ex);
  mle_ctx_destroy(d->c);
  delete d;
}

int mle_dctx_layout(const mle_dctx* d, int64_t* out) {
  if (!d || !out) return fail(MLE_INVALID, "null argument");
  const long long N = d->c->N;
  out[0] = N;
  out[1] = d->nb;
  out[2] = (int64_t)(d_pbytes(N) + sizeof(int) * (size_t)(N - kDB));  // P exchange
  out[3] = (int64_t)d_xstride(N);                                      // W exchange
  out[4] = (int64_t)(d_xstride(N) * (size_t)d->nmat);                  // X exchange
  out[5] = d->nmat;
  out[6] = (int64_t)d->owned.size();
  return MLE_OK;
}

// Set theta and generate the owned panels (Sigma; the derivative blocks when derivs).
int mle_dctx_begin(mle_dctx* d, const double theta[3], int derivs) {
  if (!d || !theta) return fail(MLE_INVALID, "null argument");
  mle_ctx* c = d->c;
  CUDA_TRY(cudaSetDevice(c->device));
  ThetaParams P;
  if (mle_fill_theta(theta, c->nugget, &P) != 0)
    return fail(MLE_INVALID, "MaternParams components must be finite and > 0");
  if (use_gen_table())
    mle_fill_gen_table(c->h_max / P.alpha, &P);
  else
    P.tab_n = 0;
  const long long N = c->N;
  const size_t pbytes = sizeof(double) * (size_t)N * kDB;
  const int no = (int)d->owned.size();
  d->derivs = derivs != 0;
  if (!c->linv) CUDA_TRY(dmalloc(&c->linv, sizeof(double) * (size_t)c->Nt * kNB * kNB));
  if ((int)d->sig.size() < no) {
    d->sig.assign(no, nullptr);
    d->lsl.assign(no, nullptr);
    d->lex.assign(no, nullptr);
    for (int q = 0; q < no; ++q) {
      CUDA_TRY(dmalloc(&d->sig[q], pbytes));
      const long long rows = N - d_c0(d->owned[q]) - kDB;
      if (rows > 0) {
        CUDA_TRY(dmalloc(&d->lsl[q], (size_t)rows * kOzRowBytes));
        CUDA_TRY(dmalloc(&d->lex[q], sizeof(int) * (size_t)rows));
      }
    }
    CUDA_TRY(dmalloc(&d->part, sizeof(double) * (size_t)no * kDB * kPanelSums));
    d->h_part.assign((size_t)no * kDB * kPanelSums, 0.0);
  }
  if (d->derivs && d->mat[0].size() < (size_t)no) {
    for (int m = 0; m < d->nmat; ++m) {
      d->mat[m].assign(no, nullptr);
      for (int q = 0; q < no; ++q) CUDA_TRY(dmalloc(&d->mat[m][q], pbytes));
    }
    d->wsl.assign(no, nullptr);
    d->wex.assign(no, nullptr);
    d->dinv.assign(no, nullptr);
    for (int q = 0; q < no; ++q) {
      const long long rows = N - d_c0(d->owned[q]);
      CUDA_TRY(dmalloc(&d->wsl[q], (size_t)rows * kOzRowBytes));
      CUDA_TRY(dmalloc(&d->wex[q], sizeof(int) * (size_t)rows));
      CUDA_TRY(dmalloc(&d->dinv[q], sizeof(double) * kDB * kDB));
      CUDA_TRY(cudaMemsetAsync(d->dinv[q], 0, sizeof(double) * kDB * kDB, c->stream));
    }
    CUDA_TRY(dmalloc(&d->tscr, sizeof(double) * kNB * kDB));
    CUDA_TRY(dmalloc(&d->wbuf, sizeof(double) * (size_t)N * kDB));
    CUDA_TRY(dmalloc(&d->dtsl, (size_t)kDB * kOzRowBytes));
    CUDA_TRY(dmalloc(&d->dtex, sizeof(int) * kDB));
    CUDA_TRY(dmalloc(&d->xsl, (size_t)no * d->nmat * kDB * kOzRowBytes));
    CUDA_TRY(dmalloc(&d->xex, sizeof(int) * (size_t)no * d->nmat * kDB));
  }
  std::memcpy(c->h_theta, &P, sizeof(P));
  CUDA_TRY(cudaMemcpyAsync(c->d_theta, c->h_theta, sizeof(P), cudaMemcpyHostToDevice,
                           c->stream));
  CUDA_TRY(cudaMemsetAsync(c->fail_flag, 0, sizeof(int), c->stream));
  CUDA_TRY(cudaMemsetAsync(c->fail_idx, 0, sizeof(long long), c->stream));
  // generation tables, then the panels in chunks of kMaxItems
  GenArgs ga;
  std::memset(&ga, 0, sizeof(ga));
  ga.ld = N;
  ga.rows = N;
  ga.n = (int)c->n;
  GenItem base;
  std::memset(&base, 0, sizeof(base));
  base.P = c->d_theta;
  base.lx = c->lx;
  base.ly = c->ly;
  base.z = c->z;
  base.fail_flag = c->fail_flag;
  base.tab = P.tab_n > 0 ? (d->derivs ? c->gtab_d : c->gtab_s) : nullptr;
  base.write_sigma = 1;
  base.write_derivs = d->derivs ? 1 : 0;
  ga.item[0] = base;
  launch_gen_table(ga, 1, d->derivs, c->stream);
  CUDA_TRY(cudaGetLastError());
  std::vector<int> c0s(no);
  for (int q = 0; q < no; ++q) c0s[q] = (int)d_c0(d->owned[q]);
  int* d_c0s = nullptr;
  CUDA_TRY(dmalloc(&d_c0s, sizeof(int) * std::max(1, no)));
  CUDA_TRY(cudaMemcpyAsync(d_c0s, c0s.data(), sizeof(int) * no, cudaMemcpyHostToDevice,
                           c->stream));
  for (int q0 = 0; q0 < no; q0 += kMaxItems) {
    const int cnt = std::min(kMaxItems, no - q0);
    for (int i = 0; i < cnt; ++i) {
      GenItem gi = base;
      gi.sigma = d->sig[q0 + i];
      gi.dalpha = d->derivs ? d->mat[0][q0 + i] : nullptr;
      gi.dnu = d->derivs ? d->mat[1][q0 + i] : nullptr;
      ga.item[i] = gi;
    }
    launch_gen_panels(ga, d_c0s + q0, (int)kDB, cnt, c->stream);
    CUDA_TRY(cudaGetLastError());
    if (d->derivs && d->nmat == 3) {
      PanelArgs pa;
      std::memset(&pa, 0, sizeof(pa));
      for (int i = 0; i < cnt; ++i) {
        pa.p[i] = d->mat[2][q0 + i];
        pa.c0[i] = c0s[q0 + i];
      }
      pa.ld = N;
      pa.width = (int)kDB;
      pa.n = (int)c->n;
      CUDA_TRY(launch_panel_identity(pa, cnt, c->stream));
    }
  }
  // always drained (begin is once per evaluation): d_c0s goes back to the buffer cache
  CUDA_TRY(cudaStreamSynchronize(c->stream));
  CUDA_TRY(cudaGetLastError());
  dfree(d_c0s);
  return MLE_OK;
}

// Owner of block b: inner steps on its panel; P_b = L[c1:, b] sliced into exch_p
// ([rows][4 KB] int8 slices, then int exponents at offset d_pbytes(N)).
int mle_dctx_factor(mle_dctx* d, int b, void* exch_p) {
  const int q = d ? d_index(d, b) : -1;
  if (q < 0) return fail(MLE_INVALID, "block not owned by this rank");
  mle_ctx* c = d->c;
  CUDA_TRY(cudaSetDevice(c->device));
  const long long N = c->N, c0 = d_c0(b), c1 = c0 + kDB;
  double* vb = d->sig[q] - c0 * N;
  Launcher run{c->stream, nullptr, c->pool, kPoolEvents};
  run.s3 = c->inner;
  mle_ctx* cs[1] = {c};
  double* mats[1] = {vb};
  long long aug[1] = {c->n};
  int rc = run.inner_block(cs, mats, aug, 1, (int)(c0 / kNB), (int)(c1 / kNB));
  if (rc) return rc;
  if (c1 < N) {
    OzSliceArgs sa;
    std::memset(&sa, 0, sizeof(sa));
    sa.X[0] = vb + c1 + c0 * N;
    sa.slices[0] = d->lsl[q];
    sa.e[0] = d->lex[q];
    sa.fail_flag[0] = c->fail_flag;
    sa.ld = N;
    sa.K = (int)kDB;
    if ((rc = run.slice(sa, N - c1, true, 1))) return rc;
    if (exch_p) {
      int8_t* ex = static_cast<int8_t*>(exch_p);
      CUDA_TRY(cudaMemcpyAsync(ex, d->lsl[q], (size_t)(N - c1) * kOzRowBytes,
                               cudaMemcpyDeviceToDevice, c->stream));
      CUDA_TRY(cudaMemcpyAsync(ex + d_pbytes(N), d->lex[q], sizeof(int) * (size_t)(N - c1),
                               cudaMemcpyDeviceToDevice, c->stream));
    }
  }
  return d_sync(d);
}

// Every rank: trailing update of its panels j > b with P_b (exch_p as produced by factor).
int mle_dctx_update(mle_dctx* d, int b, const void* exch_p) {
  return mle_dctx_update_range(d, b, exch_p, 0, d ? d->nb : 0);
}

// Same, restricted to the panels of blocks j with lo <= j < hi (look-ahead: the owner of b + 1
// updates that panel first, factors it, and updates the rest while P_{b+1} is in flight).
int mle_dctx_update_range(mle_dctx* d, int b, const void* exch_p, int lo, int hi) {
  if (!d || !exch_p) return fail(MLE_INVALID, "null argument");
  mle_ctx* c = d->c;
  CUDA_TRY(cudaSetDevice(c->device));
  const long long N = c->N, c1 = d_c0(b) + kDB;
  const int8_t* ps = static_cast<const int8_t*>(exch_p);
  const int* pe = reinterpret_cast<const int*>(ps + d_pbytes(N));
  Launcher run{c->stream, nullptr, c->pool, kPoolEvents};
  std::vector<int> qs;
  for (size_t q = 0; q < d->owned.size(); ++q)
    if (d->owned[q] > b && d_in(d->owned[q], lo, hi)) qs.push_back((int)q);
  for (size_t i0 = 0; i0 < qs.size(); i0 += kMaxGemm) {
    const int cnt = (int)std::min<size_t>(kMaxGemm, qs.size() - i0);
    OzGemmArgs g = Launcher::oz_base(N, (int)((N - c1) / kNB), (int)(kDB / kNB));
    g.trap = 1;
    for (int z = 0; z < cnt; ++z) {
      const int q = qs[i0 + z];
      const long long cj = d_c0(d->owned[q]);
      const size_t toff = (size_t)((cj - c1) / kNB) * kOzTileBytes;
      g.As[z] = g.Bs[z] = ps + toff;
      g.ea[z] = g.eb[z] = pe + (cj - c1);
      g.C[z] = d->sig[q] + cj;  // rows cj.., first column of panel j
      g.tiles_m_z[z] = (int)((N - cj) / kNB);
      g.fail_flag[z] = c->fail_flag;
    }
    int rc = run.ozgemm(g, cnt, c->stream);
    if (rc) return rc;
  }
  return d_sync(d);
}

// Owner of block b: W_b = [D_b^-1; -P_b D_b^-1] sliced into exch_w (slices, exponents at
// d_wbytes(N)) and kept for the right sweep.
int mle_dctx_wblock(mle_dctx* d, int b, void* exch_w) {
  const int q = d ? d_index(d, b) : -1;
  if (q < 0 || !d->derivs) return fail(MLE_INVALID, "block not owned / no derivatives");
  mle_ctx* c = d->c;
  CUDA_TRY(cudaSetDevice(c->device));
  const long long N = c->N, c0 = d_c0(b), c1 = c0 + kDB;
  const int t0 = (int)(c0 / kNB);
  double* vb = d->sig[q] - c0 * N;
  Launcher run{c->stream, nullptr, c->pool, kPoolEvents};
  int rc;
  {
    double* dv[1] = {d->dinv[q]};
    const double* lv[1] = {c->linv};
    run.launches += 1;
    CUDA_TRY(launch_linv_to_dinv_block(dv, lv, t0, (int)(kDB / kNB), 1, c->stream));
  }
  for (int i = 1; i < (int)(kDB / kNB); ++i) {
    GemmArgs t = gemm_base(), u = gemm_base();
    t.A[0] = vb + (c0 + i * kNB) + c0 * N;
    t.B[0] = d->dinv[q];
    t.C[0] = d->tscr;
    t.fail_flag[0] = c->fail_flag;
    u.A[0] = c->linv + (size_t)(t0 + i) * kNB * kNB;
    u.B[0] = d->tscr;
    u.C[0] = d->dinv[q] + i * kNB;
    u.fail_flag[0] = c->fail_flag;
    t.lda = N; t.ldb = kDB; t.ldc = kNB; t.K = i * kNB;
    t.tiles_m = 1; t.tiles_n = i; t.alpha = 1.0; t.beta = 0.0;
    if ((rc = run.gemm(t, kBKN, 1))) return rc;
    u.lda = kNB; u.ldb = kNB; u.ldc = kDB; u.K = kNB;
    u.tiles_m = 1; u.tiles_n = i; u.alpha = -1.0; u.beta = 0.0;
    if ((rc = run.gemm(u, kBKN, 1))) return rc;
  }
  OzSliceArgs top;
  std::memset(&top, 0, sizeof(top));
  top.X[0] = d->dinv[q];
  top.slices[0] = d->wsl[q];
  top.e[0] = d->wex[q];
  top.fail_flag[0] = c->fail_flag;
  top.ld = kDB;
  top.K = (int)kDB;
  if ((rc = run.slice(top, kDB, true, 1))) return rc;
  if (c1 < N) {
    OzSliceArgs dt;
    std::memset(&dt, 0, sizeof(dt));
    dt.X[0] = d->dinv[q];
    dt.slices[0] = d->dtsl;
    dt.e[0] = d->dtex;
    dt.fail_flag[0] = c->fail_flag;
    dt.ld = kDB;
    dt.K = (int)kDB;
    if ((rc = run.slice(dt, kDB, false, 1))) return rc;
    OzGemmArgs g = Launcher::oz_base(N, (int)((N - c1) / kNB), (int)(kDB / kNB));
    g.beta = 0.0;
    g.As[0] = d->lsl[q];
    g.ea[0] = d->lex[q];
    g.Bs[0] = d->dtsl;
    g.eb[0] = d->dtex;
    g.C[0] = d->wbuf;
    g.fail_flag[0] = c->fail_flag;
    if ((rc = run.ozgemm(g, 1, c->stream))) return rc;
    OzSliceArgs bot;
    std::memset(&bot, 0, sizeof(bot));
    bot.X[0] = d->wbuf;
    bot.slices[0] = d->wsl[q] + (size_t)(kDB / kNB) * kOzTileBytes;
    bot.e[0] = d->wex[q] + kDB;
    bot.fail_flag[0] = c->fail_flag;
    bot.ld = N;
    bot.K = (int)kDB;
    if ((rc = run.slice(bot, N - c1, true, 1))) return rc;
  }
  if (exch_w) {
    int8_t* ex = static_cast<int8_t*>(exch_w);
    CUDA_TRY(cudaMemcpyAsync(ex, d->wsl[q], (size_t)(N - c0) * kOzRowBytes,
                             cudaMemcpyDeviceToDevice, c->stream));
    CUDA_TRY(cudaMemcpyAsync(ex + d_wbytes(N), d->wex[q], sizeof(int) * (size_t)(N - c0),
                             cudaMemcpyDeviceToDevice, c->stream));
  }
  return d_sync(d);
}

// Every rank, forward sweep X = L^-1 S, block b: X[c0:, owned columns] = W_b X[c0:c1, owned].
int mle_dctx_forward(mle_dctx* d, int b, const void* exch_w) {
  return mle_dctx_forward_range(d, b, exch_w, 0, d ? d->nb : 0);
}

// Same, restricted to the panels of blocks j with lo <= j < hi (the two-sided path's deferred
// sweep: block b acts on the panels left of it only).
int mle_dctx_forward_range(mle_dctx* d, int b, const void* exch_w, int lo, int hi) {
  if (!d || !exch_w || !d->derivs) return fail(MLE_INVALID, "null argument / no derivatives");
  mle_ctx* c = d->c;
  CUDA_TRY(cudaSetDevice(c->device));
  const long long N = c->N, c0 = d_c0(b);
  const int8_t* ws = static_cast<const int8_t*>(exch_w);
  const int* we = reinterpret_cast<const int*>(ws + d_wbytes(N));
  Launcher run{c->stream, nullptr, c->pool, kPoolEvents};
  std::vector<int> items;  // q * nmat + m of the panels in range
  for (size_t q = 0; q < d->owned.size(); ++q)
    if (d_in(d->owned[q], lo, hi))
      for (int m = 0; m < d->nmat; ++m) items.push_back((int)q * d->nmat + m);
  const int total = (int)items.size();
  int rc;
  for (int i0 = 0; i0 < total; i0 += kMaxGemm) {
    const int cnt = std::min(kMaxGemm, total - i0);
    OzSliceArgs sa;
    std::memset(&sa, 0, sizeof(sa));
    OzGemmArgs g = Launcher::oz_base(N, (int)((N - c0) / kNB), (int)(kDB / kNB));
    g.alpha = 1.0;
    g.beta0_tm = (int)(kDB / kNB);
    for (int z = 0; z < cnt; ++z) {
      const int idx = items[i0 + z], q = idx / d->nmat, m = idx % d->nmat;
      double* panel = d_mat(d, m, q);
      sa.X[z] = panel + c0;  // B(n, k) = X[c0 + k, n]: k-contig rows = the panel's columns
      sa.slices[z] = d->xsl + (size_t)idx * kDB * kOzRowBytes;
      sa.e[z] = d->xex + (size_t)idx * kDB;
      sa.fail_flag[z] = c->fail_flag;
      g.As[z] = ws;
      g.ea[z] = we;
      g.Bs[z] = sa.slices[z];
      g.eb[z] = sa.e[z];
      g.C[z] = panel + c0;
      g.fail_flag[z] = c->fail_flag;
    }
    sa.ld = N;
    sa.K = (int)kDB;
    if ((rc = run.slice(sa, kDB, false, cnt))) return rc;
    if ((rc = run.ozgemm(g, cnt, c->stream))) return rc;
  }
  if (!d->wcache.empty()) {  // keep W_b for the right sweep (no second broadcast)
    CUDA_TRY(cudaMemcpyAsync(d->wcache[b], ws, (size_t)(N - c0) * kOzRowBytes,
                             cudaMemcpyDeviceToDevice, c->stream));
    CUDA_TRY(cudaMemcpyAsync(d->wcache_e[b], we, sizeof(int) * (size_t)(N - c0),
                             cudaMemcpyDeviceToDevice, c->stream));
  }
  return d_sync(d);
}

// Owner of block b: the right-sweep operand X[c0:, b] (entries above the diagonal zeroed) of
// every derivative block into exch_x (block m at m * d_xstride(N); exponents after the slices).
int mle_dctx_right_operand(mle_dctx* d, int b, void* exch_x) {
  const int q = d ? d_index(d, b) : -1;
  if (q < 0 || !exch_x || !d->derivs) return fail(MLE_INVALID, "block not owned / no derivs");
  mle_ctx* c = d->c;
  CUDA_TRY(cudaSetDevice(c->device));
  const long long N = c->N, c0 = d_c0(b);
  int8_t* ex = static_cast<int8_t*>(exch_x);
  Launcher run{c->stream, nullptr, c->pool, kPoolEvents};
  OzSliceArgs sa;
  std::memset(&sa, 0, sizeof(sa));
  for (int m = 0; m < d->nmat; ++m) {
    sa.X[m] = d_mat(d, m, q) + c0;
    sa.slices[m] = ex + (size_t)m * d_xstride(N);
    sa.e[m] = reinterpret_cast<int*>(ex + (size_t)m * d_xstride(N) + d_wbytes(N));
    sa.fail_flag[m] = c->fail_flag;
  }
  sa.ld = N;
  sa.K = (int)kDB;
  sa.upper_zero = 1;
  int rc = run.slice(sa, N - c0, true, d->nmat);
  if (rc) return rc;
  return d_sync(d);
}

// Every rank, right sweep block b: X[i, j] += X[i, c0:c1] W_b[j - c0, :] for its panels j >= b
// (rows i >= j's block start; block b's own columns are overwritten: they become B[:, b]).
int mle_dctx_right(mle_dctx* d, int b, const void* exch_w, const void* exch_x) {
  return mle_dctx_right_range(d, b, exch_w, exch_x, 0, d ? d->nb : 0);
}

// Same, restricted to the panels of blocks j with lo <= j < hi.  exch_w == NULL: W_b from the
// rank's W cache (filled by the forward sweep; mle_dctx_wcache).
int mle_dctx_right_range(mle_dctx* d, int b, const void* exch_w, const void* exch_x, int lo,
                         int hi) {
  if (!d || !exch_x || !d->derivs) return fail(MLE_INVALID, "null argument");
  if (!exch_w && d->wcache.empty()) return fail(MLE_INVALID, "no W_b: pass exch_w or enable the W cache");
  mle_ctx* c = d->c;
  CUDA_TRY(cudaSetDevice(c->device));
  const long long N = c->N, c0 = d_c0(b);
  const int8_t* ws = exch_w ? static_cast<const int8_t*>(exch_w) : d->wcache[b];
  const int* we = exch_w ? reinterpret_cast<const int*>(ws + d_wbytes(N)) : d->wcache_e[b];
  const int8_t* xs = static_cast<const int8_t*>(exch_x);
  Launcher run{c->stream, nullptr, c->pool, kPoolEvents};
  for (int own = 1; own >= 0; --own) {  // own == 1: the owner's block b (overwrite)
    std::vector<std::pair<int, int>> zs;  // (q, m)
    for (size_t q = 0; q < d->owned.size(); ++q) {
      const int bj = d->owned[q];
      if (bj < b || (bj == b) != (own == 1) || !d_in(bj, lo, hi)) continue;
      for (int m = 0; m < d->nmat; ++m) zs.push_back({(int)q, m});
    }
    for (size_t i0 = 0; i0 < zs.size(); i0 += kMaxGemm) {
      const int cnt = (int)std::min<size_t>(kMaxGemm, zs.size() - i0);
      OzGemmArgs g = Launcher::oz_base(N, (int)((N - c0) / kNB), (int)(kDB / kNB));
      g.trap = 1;
      g.alpha = 1.0;
      g.beta0_tn = own ? (int)(kDB / kNB) : 0;
      for (int z = 0; z < cnt; ++z) {
        const int q = zs[i0 + z].first, m = zs[i0 + z].second;
        const long long cj = d_c0(d->owned[q]);
        const size_t toff = (size_t)((cj - c0) / kNB) * kOzTileBytes;
        const int8_t* xm = xs + (size_t)m * d_xstride(N);
        g.As[z] = xm + toff;
        g.ea[z] = reinterpret_cast<const int*>(xm + d_wbytes(N)) + (cj - c0);
        g.Bs[z] = ws + toff;
        g.eb[z] = we + (cj - c0);
        g.C[z] = d_mat(d, m, q) + cj;
        g.tiles_m_z[z] = (int)((N - cj) / kNB);
        g.fail_flag[z] = c->fail_flag;
      }
      int rc = run.ozgemm(g, cnt, c->stream);
      if (rc) return rc;
    }
  }
  return d_sync(d);
}

// ---- two-sided reduction on the panels (the single-context solves_2s) -----
namespace {
int d_ensure_2s(mle_dctx* d) {
  if (d->ts2) return MLE_OK;
  const long long N = d->c->N;
  CUDA_TRY(dmalloc(&d->ts2, sizeof(double) * (size_t)d->nmat * kDB * kDB));
  CUDA_TRY(dmalloc(&d->a11sl, (size_t)d->nmat * kDB * kOzRowBytes));
  CUDA_TRY(dmalloc(&d->a11ex, sizeof(int) * (size_t)d->nmat * kDB));
  CUDA_TRY(dmalloc(&d->s21sl, (size_t)d->nmat * N * kOzRowBytes));
  CUDA_TRY(dmalloc(&d->s21ex, sizeof(int) * (size_t)d->nmat * N));
  return MLE_OK;
}
}  // namespace

// Owner of block b (after mle_dctx_wblock(b): D_b^-1 and W_b's slices), every derivative
// matrix: (1) S11 <- D^-1 S11 D^-T, (2) S21 <- S21 D^-T, (3) S21 <- S21 - 1/2 L21 S11, then the
// slices of S21 (rows c1..N) into exch_x (matrix m at m * the X-exchange stride, exponents
// after the slices) for the other ranks' trailing updates.
int mle_dctx_2s_owner(mle_dctx* d, int b, void* exch_x) {
  const int q = d ? d_index(d, b) : -1;
  if (q < 0 || !exch_x || !d->derivs) return fail(MLE_INVALID, "block not owned / no derivs");
  mle_ctx* c = d->c;
  CUDA_TRY(cudaSetDevice(c->device));
  int rc = d_ensure_2s(d);
  if (rc) return rc;
  const long long N = c->N, c0 = d_c0(b), c1 = c0 + kDB;
  const int nm = d->nmat;
  Launcher run{c->stream, nullptr, c->pool, kPoolEvents};
  double* blks[kMaxGemm];
  for (int m = 0; m < nm; ++m) blks[m] = d_mat(d, m, q) + c0;  // S11 (ld N)
  run.launches += 1;
  CUDA_TRY(launch_mirror_lower(blks, nm, N, (int)kDB, c->stream));
  {
    GemmArgs t = gemm_base(), u = gemm_base();
    for (int m = 0; m < nm; ++m) {
      t.A[m] = d->dinv[q];
      t.B[m] = blks[m];
      t.C[m] = d->ts2 + (size_t)m * kDB * kDB;
      t.fail_flag[m] = c->fail_flag;
      u.A[m] = t.C[m];
      u.B[m] = d->dinv[q];
      u.C[m] = blks[m];
      u.fail_flag[m] = c->fail_flag;
    }
    t.lda = kDB; t.ldb = N; t.ldc = kDB; t.K = (int)kDB;
    t.tiles_m = (int)(kDB / kNB); t.tiles_n = (int)(kDB / kNB); t.alpha = 1.0; t.beta = 0.0;
    if ((rc = run.gemm(t, kBKN, nm))) return rc;
    u.lda = kDB; u.ldb = kDB; u.ldc = N; u.K = (int)kDB;
    u.tiles_m = (int)(kDB / kNB); u.tiles_n = (int)(kDB / kNB); u.alpha = 1.0; u.beta = 0.0;
    if ((rc = run.gemm(u, kBNK, nm))) return rc;
  }
  if (c1 >= N) return d_sync(d);
  const int rt = (int)((N - c1) / kNB), tb = (int)(kDB / kNB);
  auto slice_s21 = [&](int8_t* const* dst, int* const* dex) {
    OzSliceArgs sa;
    std::memset(&sa, 0, sizeof(sa));
    for (int m = 0; m < nm; ++m) {
      sa.X[m] = d_mat(d, m, q) + c1;  // rows c1.., the block's columns
      sa.slices[m] = dst[m];
      sa.e[m] = dex[m];
      sa.fail_flag[m] = c->fail_flag;
    }
    sa.ld = N;
    sa.K = (int)kDB;
    return run.slice(sa, N - c1, true, nm);
  };
  int8_t* sl[kMaxGemm];
  int* se[kMaxGemm];
  for (int m = 0; m < nm; ++m) {
    sl[m] = d->s21sl + (size_t)m * N * kOzRowBytes;
    se[m] = d->s21ex + (size_t)m * N;
  }
  if ((rc = slice_s21(sl, se))) return rc;
  {  // (2) S21 <- S21 D^-T: B = the rows of D^-1 = W_b's top slices
    OzGemmArgs g = Launcher::oz_base(N, rt, tb);
    g.alpha = 1.0;
    g.beta = 0.0;
    for (int m = 0; m < nm; ++m) {
      g.As[m] = sl[m];
      g.ea[m] = se[m];
      g.Bs[m] = d->wsl[q];
      g.eb[m] = d->wex[q];
      g.C[m] = d_mat(d, m, q) + c1;
      g.fail_flag[m] = c->fail_flag;
    }
    if ((rc = run.ozgemm(g, nm, c->stream))) return rc;
  }
  {  // slices of the new S11 (B operand of (3) / (5))
    OzSliceArgs sa;
    std::memset(&sa, 0, sizeof(sa));
    for (int m = 0; m < nm; ++m) {
      sa.X[m] = blks[m];
      sa.slices[m] = d->a11sl + (size_t)m * kDB * kOzRowBytes;
      sa.e[m] = d->a11ex + (size_t)m * kDB;
      sa.fail_flag[m] = c->fail_flag;
    }
    sa.ld = N;
    sa.K = (int)kDB;
    if ((rc = run.slice(sa, kDB, true, nm))) return rc;
  }
  if ((rc = mle_dctx_2s_finish(d, b))) return rc;  // (3) = the same product as (5)
  int8_t* xs[kMaxGemm];
  int* xe[kMaxGemm];
  for (int m = 0; m < nm; ++m) {
    int8_t* base = static_cast<int8_t*>(exch_x) + (size_t)m * d_xstride(N);
    xs[m] = base;
    xe[m] = reinterpret_cast<int*>(base + d_wbytes(N));
  }
  if ((rc = slice_s21(xs, xe))) return rc;
  return d_sync(d);
}

// Owner of block b: S21 <- S21 - 1/2 L21 S11 (step (5); also step (3) inside 2s_owner).
int mle_dctx_2s_finish(mle_dctx* d, int b) {
  const int q = d ? d_index(d, b) : -1;
  if (q < 0 || !d->derivs || !d->a11sl) return fail(MLE_INVALID, "block not owned / no 2s state");
  mle_ctx* c = d->c;
  CUDA_TRY(cudaSetDevice(c->device));
  const long long N = c->N, c1 = d_c0(b) + kDB;
  if (c1 >= N) return d_sync(d);
  Launcher run{c->stream, nullptr, c->pool, kPoolEvents};
  OzGemmArgs g = Launcher::oz_base(N, (int)((N - c1) / kNB), (int)(kDB / kNB));
  g.alpha = -0.5;
  for (int m = 0; m < d->nmat; ++m) {
    g.As[m] = d->lsl[q];
    g.ea[m] = d->lex[q];
    g.Bs[m] = d->a11sl + (size_t)m * kDB * kOzRowBytes;
    g.eb[m] = d->a11ex + (size_t)m * kDB;
    g.C[m] = d_mat(d, m, q) + c1;
    g.fail_flag[m] = c->fail_flag;
  }
  int rc = run.ozgemm(g, d->nmat, c->stream);
  if (rc) return rc;
  return d_sync(d);
}

// Every rank, step (4) of block b on its panels j > b with lo <= j < hi:
// S22 -= S21 L21^T + L21 S21^T (lower part of each panel), from the broadcast slices of S21
// (exch_x, as written by 2s_owner) and of L21 = P_b (exch_p, as written by factor or
// panel_slices).
int mle_dctx_2s_update_range(mle_dctx* d, int b, const void* exch_x, const void* exch_p, int lo,
                             int hi) {
  if (!d || !exch_x || !exch_p || !d->derivs) return fail(MLE_INVALID, "null argument");
  mle_ctx* c = d->c;
  CUDA_TRY(cudaSetDevice(c->device));
  const long long N = c->N, c1 = d_c0(b) + kDB;
  const int8_t* ps = static_cast<const int8_t*>(exch_p);
  const int* pe = reinterpret_cast<const int*>(ps + d_pbytes(N));
  Launcher run{c->stream, nullptr, c->pool, kPoolEvents};
  std::vector<std::pair<int, int>> zs;  // (q, m)
  for (size_t q = 0; q < d->owned.size(); ++q)
    if (d->owned[q] > b && d_in(d->owned[q], lo, hi))
      for (int m = 0; m < d->nmat; ++m) zs.push_back({(int)q, m});
  for (int pass = 0; pass < 2; ++pass) {
    for (size_t i0 = 0; i0 < zs.size(); i0 += kMaxGemm) {
      const int cnt = (int)std::min<size_t>(kMaxGemm, zs.size() - i0);
      OzGemmArgs g = Launcher::oz_base(N, (int)((N - c1) / kNB), (int)(kDB / kNB));
      g.trap = 1;
      for (int z = 0; z < cnt; ++z) {
        const int q = zs[i0 + z].first, m = zs[i0 + z].second;
        const long long cj = d_c0(d->owned[q]);
        const size_t toff = (size_t)((cj - c1) / kNB) * kOzTileBytes;
        const int8_t* xm = static_cast<const int8_t*>(exch_x) + (size_t)m * d_xstride(N);
        const int* xem = reinterpret_cast<const int*>(xm + d_wbytes(N));
        const int8_t* a = pass == 0 ? xm : ps;
        const int* ea = pass == 0 ? xem : pe;
        const int8_t* bb = pass == 0 ? ps : xm;
        const int* eb = pass == 0 ? pe : xem;
        g.As[z] = a + toff;
        g.ea[z] = ea + (cj - c1);
        g.Bs[z] = bb + toff;
        g.eb[z] = eb + (cj - c1);
        g.C[z] = d_mat(d, m, q) + cj;  // rows cj.., first column of panel j
        g.tiles_m_z[z] = (int)((N - cj) / kNB);
        g.fail_flag[z] = c->fail_flag;
      }
      int rc = run.ozgemm(g, cnt, c->stream);
      if (rc) return rc;
    }
  }
  return d_sync(d);
}

// Owner of block b: P_b = L[c1:, b]'s slices (kept since the factorization) into exch_p.
int mle_dctx_panel_slices(mle_dctx* d, int b, void* exch_p) {
  const int q = d ? d_index(d, b) : -1;
  if (q < 0 || !exch_p) return fail(MLE_INVALID, "block not owned");
  mle_ctx* c = d->c;
  CUDA_TRY(cudaSetDevice(c->device));
  const long long N = c->N, c1 = d_c0(b) + kDB;
  if (c1 < N) {
    int8_t* ex = static_cast<int8_t*>(exch_p);
    CUDA_TRY(cudaMemcpyAsync(ex, d->lsl[q], (size_t)(N - c1) * kOzRowBytes,
                             cudaMemcpyDeviceToDevice, c->stream));
    CUDA_TRY(cudaMemcpyAsync(ex + d_pbytes(N), d->lex[q], sizeof(int) * (size_t)(N - c1),
                             cudaMemcpyDeviceToDevice, c->stream));
  }
  return d_sync(d);
}

int mle_dctx_set_async(mle_dctx* d, int on) {
  if (!d) return fail(MLE_INVALID, "null argument");
  CUDA_TRY(cudaSetDevice(d->c->device));
  CUDA_TRY(cudaStreamSynchronize(d->c->stream));
  CUDA_TRY(cudaStreamSynchronize(d->c->inner));
  d->async = on != 0;
  return MLE_OK;
}

int mle_dctx_stream(const mle_dctx* d, void** out) {
  if (!d || !out) return fail(MLE_INVALID, "null argument");
  *out = (void*)d->c->stream;
  return MLE_OK;
}

// W cache: every block's W_b slices kept on this rank (7 x 512 + 4 bytes per row of rows
// c0..N: ~3.5 N^2 bytes in total), so the right sweep needs no second W broadcast.
// on = 0 frees it.  Returns MLE_CUDA_ERROR (cache left off) if the memory is not there.
int mle_dctx_wcache(mle_dctx* d, int on) {
  if (!d) return fail(MLE_INVALID, "null argument");
  CUDA_TRY(cudaSetDevice(d->c->device));
  CUDA_TRY(cudaStreamSynchronize(d->c->stream));
  for (auto* p : d->wcache) dfree(p);
  for (auto* p : d->wcache_e) dfree(p);
  d->wcache.clear();
  d->wcache_e.clear();
  if (!on) return MLE_OK;
  const long long N = d->c->N;
  std::vector<int8_t*> w(d->nb, nullptr);
  std::vector<int*> e(d->nb, nullptr);
  for (int b = 0; b < d->nb; ++b) {
    const size_t rows = (size_t)(N - d_c0(b));
    if (dmalloc(&w[b], rows * kOzRowBytes) != cudaSuccess ||
        dmalloc(&e[b], sizeof(int) * rows) != cudaSuccess) {
      for (auto* p : w) dfree(p);
      for (auto* p : e) dfree(p);
      cudaGetLastError();
      return fail(MLE_CUDA_ERROR, "W cache: out of device memory");
    }
  }
  d->wcache = w;
  d->wcache_e = e;
  return MLE_OK;
}

// This rank's partial sums over its panels: out[0..kPanelSums) (the kReduceOut layout of the
// single-GPU reduction), out[kPanelSums] = failure flag, out[kPanelSums + 1] = pivot.
int mle_dctx_partials(mle_dctx* d, double* out) {
  if (!d || !out) return fail(MLE_INVALID, "null argument");
  std::vector<double> per((size_t)d->owned.size() * kPanelSums + 2);
  int rc = mle_dctx_panel_partials(d, per.data());
  if (rc) return rc;
  for (int k = 0; k < kPanelSums; ++k) out[k] = 0.0;
  for (size_t q = 0; q < d->owned.size(); ++q)
    for (int k = 0; k < kPanelSums; ++k) out[k] += per[q * kPanelSums + k];
  out[kPanelSums] = per[d->owned.size() * kPanelSums];
  out[kPanelSums + 1] = per[d->owned.size() * kPanelSums + 1];
  return MLE_OK;
}

// Per owned panel (ascending block order): out[q * kPanelSums + k], each summed over the
// panel's columns in a fixed order; then the failure flag and the pivot.  A driver that adds
// the panels' sums in block order gets results independent of the number of ranks.
int mle_dctx_panel_partials(mle_dctx* d, double* out) {
  if (!d || !out) return fail(MLE_INVALID, "null argument");
  mle_ctx* c = d->c;
  CUDA_TRY(cudaSetDevice(c->device));
  const int no = (int)d->owned.size();
  for (int q0 = 0; q0 < no; q0 += kMaxItems) {
    const int cnt = std::min(kMaxItems, no - q0);
    PanelReduceArgs ra;
    std::memset(&ra, 0, sizeof(ra));
    for (int i = 0; i < cnt; ++i) {
      const int q = q0 + i;
      ra.L[i] = d->sig[q];
      ra.Ba[i] = d->derivs ? d->mat[0][q] : nullptr;
      ra.Bn[i] = d->derivs ? d->mat[1][q] : nullptr;
      ra.Bm[i] = (d->derivs && d->nmat == 3) ? d->mat[2][q] : nullptr;
      ra.partials[i] = d->part + (size_t)q * kDB * kPanelSums;
      ra.c0[i] = d_c0(d->owned[q]);
    }
    ra.ld = c->N;
    ra.n = (int)c->n;
    CUDA_TRY(launch_panel_reduce(ra, (int)kDB, cnt, c->stream));
  }
  CUDA_TRY(cudaMemcpyAsync(d->h_part.data(), d->part, sizeof(double) * d->h_part.size(),
                           cudaMemcpyDeviceToHost, c->stream));
  int flag = 0;
  long long idx = 0;
  CUDA_TRY(cudaMemcpyAsync(c->h_res, c->fail_flag, sizeof(int), cudaMemcpyDeviceToHost,
                           c->stream));
  CUDA_TRY(cudaMemcpyAsync(c->h_res + 1, c->fail_idx, sizeof(long long),
                           cudaMemcpyDeviceToHost, c->stream));
  CUDA_TRY(cudaStreamSynchronize(c->stream));  // host reads the sums (also in async mode)
  CUDA_TRY(cudaGetLastError());
  std::memcpy(&flag, c->h_res, sizeof(int));
  std::memcpy(&idx, c->h_res + 1, sizeof(long long));
  for (int q = 0; q < no; ++q) {
    double* o = out + (size_t)q * kPanelSums;
    for (int k = 0; k < kPanelSums; ++k) o[k] = 0.0;
    for (long long jl = 0; jl < kDB; ++jl)
      for (int k = 0; k < kPanelSums; ++k)
        o[k] += d->h_part[((size_t)q * kDB + jl) * kPanelSums + k];
  }
  out[(size_t)no * kPanelSums] = (double)flag;
  out[(size_t)no * kPanelSums + 1] = (double)idx;
  return MLE_OK;
}

}  // extern "C"
