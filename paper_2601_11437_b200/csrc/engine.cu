// engine.cu — C ABI (include/maternfisher.h) and the per-evaluation schedule.
//
// One mle_ctx = one dataset resident on one GPU with its own CUDA stream.  Per evaluation:
//
//   gen      Sigma (lower tiles, augmented row n = z, identity padding) and, for eval_all,
//            dSigma/dalpha, dSigma/dnu (full storage)                    [gen.cu]
//   potrf    right-looking blocked Cholesky, nb = 128: diag tile factor + inverse,
//            panel = A_T,K Linv_k^T, trailing lower SYRK                 [linalg.cu]
//            -> row n of L is y^T = (L^-1 z)^T (the reference's `white`, likelihood.py:121)
//   solve    X_i = L^-1 S_i (row panel Linv_k S_k, full trailing GEMM), then the lower half
//            of B_i = X_i L^-T by a right-looking column sweep; B_i = L^-1 S_i L^-T.
//   reduce   log det, y^T y, tr B_i, <B_i,B_j>_F, and y^T B_i y = B_i[n,n] (augmented)
//
// The score and Fisher information then follow likelihood.py:123-147 with
// tr(Sigma^-1 S_i) = tr B_i, w^T S_i w = y^T B_i y and tr(W_i W_j) = <B_i, B_j>_F.
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <mutex>
#include <string>
#include <vector>

#include "kernels.h"

using namespace mle;

namespace {

thread_local std::string g_last_error;
std::mutex g_init_mutex;
std::vector<int> g_device_ready;
const double kLog2Pi = 1.8378770664093453;  // log(2 pi), likelihood.py:38

int fail(int code, const std::string& msg) {
  g_last_error = msg;
  return code;
}

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
    CUDA_TRY(init_diag_attributes());
    g_device_ready[device] = 1;
  }
  return MLE_OK;
}

long long round_up(long long v, long long m) { return (v + m - 1) / m * m; }

}  // namespace

struct mle_ctx {
  int device = 0;
  int64_t n = 0;
  long long N = 0;   // padded extent (multiple of kNB), >= n + 1
  int Nt = 0;        // N / kNB
  double nugget = 0.0;
  cudaStream_t stream = nullptr;
  double* lx = nullptr;
  double* ly = nullptr;
  double* z = nullptr;
  double* sigma = nullptr;
  double* sa = nullptr;
  double* sn = nullptr;
  double* linv = nullptr;
  int* fail_flag = nullptr;
  long long* fail_idx = nullptr;
  double* partials = nullptr;
  double* out = nullptr;     // device: 9 reduction results
  double* h_res = nullptr;   // pinned: 9 results + fail flag + fail idx
  cudaEvent_t ev[5] = {};
  double phase_ms[MLE_NUM_PHASES] = {};
  double flops = 0.0;
  double gen_bytes = 0.0;
  double launches = 0.0;  // kernels launched by the last evaluation
};

namespace {

int ensure_matrices(mle_ctx* c, bool derivs) {
  const size_t bytes = sizeof(double) * (size_t)c->N * (size_t)c->N;
  if (!c->sigma) CUDA_TRY(cudaMalloc(&c->sigma, bytes));
  if (!c->linv) CUDA_TRY(cudaMalloc(&c->linv, sizeof(double) * (size_t)c->Nt * kNB * kNB));
  if (derivs) {
    if (!c->sa) CUDA_TRY(cudaMalloc(&c->sa, bytes));
    if (!c->sn) CUDA_TRY(cudaMalloc(&c->sn, bytes));
  }
  return MLE_OK;
}

GemmArgs gemm_base(const mle_ctx* c) {
  GemmArgs g;
  std::memset(&g, 0, sizeof(g));
  g.K = kNB;
  g.fail_flag = c->fail_flag;
  return g;
}

// Two-level blocking: inner steps of kNB = 128 (diagonal tile factor/inverse, panel
// products, updates confined to the current outer block), then one trailing update per
// outer block of kOuter tiles with K = kOuter * 128, which amortises the GEMM pipeline
// fill / C traffic over 4x more k-steps than a single-level right-looking sweep.
constexpr int kOuter = 4;

int gemm(mle_ctx* c, const GemmArgs& g, BLayout bl, int batch) {
  ++c->launches;
  CUDA_TRY(launch_gemm(g, bl, batch, c->stream));
  return MLE_OK;
}

// Right-looking blocked Cholesky of the padded, augmented matrix `a` (ld = N).
int run_potrf(mle_ctx* c, double* a, long long N, int Nt, long long n_aug) {
  const long long ld = N;
  int rc;
  for (int b0 = 0; b0 < Nt; b0 += kOuter) {
    const int b1 = std::min(Nt, b0 + kOuter);
    for (int k = b0; k < b1; ++k) {
      const long long k0 = (long long)k * kNB;
      double* linv_k = c->linv + (size_t)k * kNB * kNB;
      ++c->launches;
      CUDA_TRY(launch_potrf_diag(a, ld, (int)k0, n_aug, linv_k, c->fail_flag, c->fail_idx,
                                 c->stream));
      const int rem = Nt - k - 1;
      if (rem == 0) break;
      double* panel = a + (k0 + kNB) + k0 * ld;
      // panel <- panel * Linv_k^T   (in place: BN = 128 covers the whole panel width)
      GemmArgs g = gemm_base(c);
      g.A[0] = panel; g.lda = ld;
      g.B[0] = linv_k; g.ldb = kNB;
      g.C[0] = panel; g.ldc = ld;
      g.tiles_m = rem; g.tiles_n = 1; g.alpha = 1.0; g.beta = 0.0;
      if ((rc = gemm(c, g, kBNK, 1))) return rc;
      // inner update of the remaining columns of this outer block (lower trapezoid)
      const int wcols = b1 - k - 1;
      if (wcols > 0) {
        GemmArgs t = gemm_base(c);
        t.A[0] = panel; t.lda = ld;
        t.B[0] = panel; t.ldb = ld;
        t.C[0] = a + (k0 + kNB) + (k0 + kNB) * ld; t.ldc = ld;
        t.tiles_m = rem; t.tiles_n = wcols; t.trap = 1; t.alpha = -1.0; t.beta = 1.0;
        if ((rc = gemm(c, t, kBNK, 1))) return rc;
      }
    }
    const int rem = Nt - b1;
    if (rem <= 0) continue;
    // outer trailing update: A_TT -= P P^T with P = L[T, b0:b1], K = (b1 - b0) * 128
    const long long c0 = (long long)b0 * kNB, t0 = (long long)b1 * kNB;
    GemmArgs t = gemm_base(c);
    t.A[0] = a + t0 + c0 * ld; t.lda = ld;
    t.B[0] = a + t0 + c0 * ld; t.ldb = ld;
    t.C[0] = a + t0 + t0 * ld; t.ldc = ld;
    t.K = (b1 - b0) * kNB;
    t.tiles_m = rem; t.lower = 1; t.alpha = -1.0; t.beta = 1.0;
    if ((rc = gemm(c, t, kBNK, 1))) return rc;
  }
  return MLE_OK;
}

// B_i = L^-1 S_i L^-T (lower half) for both derivative matrices, in place.
int run_solves(mle_ctx* c) {
  const long long N = c->N, ld = N;
  const int Nt = c->Nt;
  double* S[2] = {c->sa, c->sn};
  const double* L = c->sigma;
  int rc;
  // forward sweep X = L^-1 S (all columns), row blocks top-down
  for (int b0 = 0; b0 < Nt; b0 += kOuter) {
    const int b1 = std::min(Nt, b0 + kOuter);
    for (int k = b0; k < b1; ++k) {
      const long long k0 = (long long)k * kNB;
      const double* linv_k = c->linv + (size_t)k * kNB * kNB;
      GemmArgs g = gemm_base(c);
      for (int b = 0; b < 2; ++b) {
        g.A[b] = linv_k;
        g.B[b] = S[b] + k0;   // B(n, kk) = S[k0 + kk, n]  (kBKN)
        g.C[b] = S[b] + k0;   // in place: BM = 128 covers the whole row panel
      }
      g.lda = kNB; g.ldb = ld; g.ldc = ld;
      g.tiles_m = 1; g.tiles_n = Nt; g.alpha = 1.0; g.beta = 0.0;
      if ((rc = gemm(c, g, kBKN, 2))) return rc;
      const int wrows = b1 - k - 1;  // remaining row tiles of this outer block
      if (wrows > 0) {
        GemmArgs t = gemm_base(c);
        for (int b = 0; b < 2; ++b) {
          t.A[b] = L + (k0 + kNB) + k0 * ld;   // L[k+1 : b1, k]
          t.B[b] = S[b] + k0;                  // X_k (kBKN)
          t.C[b] = S[b] + (k0 + kNB);
        }
        t.lda = ld; t.ldb = ld; t.ldc = ld;
        t.tiles_m = wrows; t.tiles_n = Nt; t.alpha = -1.0; t.beta = 1.0;
        if ((rc = gemm(c, t, kBKN, 2))) return rc;
      }
    }
    const int rem = Nt - b1;
    if (rem <= 0) continue;
    const long long c0 = (long long)b0 * kNB, t0 = (long long)b1 * kNB;
    GemmArgs t = gemm_base(c);
    for (int b = 0; b < 2; ++b) {
      t.A[b] = L + t0 + c0 * ld;   // L[T, b0:b1]
      t.B[b] = S[b] + c0;          // X[b0:b1, :] (kBKN)
      t.C[b] = S[b] + t0;
    }
    t.lda = ld; t.ldb = ld; t.ldc = ld;
    t.K = (b1 - b0) * kNB;
    t.tiles_m = rem; t.tiles_n = Nt; t.alpha = -1.0; t.beta = 1.0;
    if ((rc = gemm(c, t, kBKN, 2))) return rc;
  }
  // right sweep on lower tiles: B[j:, j] = X[j:, j] Linv_j^T ; X[T,T] -= B[T,j] L[T,j]^T
  for (int b0 = 0; b0 < Nt; b0 += kOuter) {
    const int b1 = std::min(Nt, b0 + kOuter);
    for (int j = b0; j < b1; ++j) {
      const long long j0 = (long long)j * kNB;
      const double* linv_j = c->linv + (size_t)j * kNB * kNB;
      GemmArgs g = gemm_base(c);
      for (int b = 0; b < 2; ++b) {
        g.A[b] = S[b] + j0 + j0 * ld;
        g.B[b] = linv_j;
        g.C[b] = S[b] + j0 + j0 * ld;
      }
      g.lda = ld; g.ldb = kNB; g.ldc = ld;
      g.tiles_m = Nt - j; g.tiles_n = 1; g.alpha = 1.0; g.beta = 0.0;
      if ((rc = gemm(c, g, kBNK, 2))) return rc;
      const int wcols = b1 - j - 1;
      if (wcols > 0) {
        GemmArgs t = gemm_base(c);
        for (int b = 0; b < 2; ++b) {
          t.A[b] = S[b] + (j0 + kNB) + j0 * ld;   // B[T, j]
          t.B[b] = L + (j0 + kNB) + j0 * ld;      // L[T, j]  (kBNK)
          t.C[b] = S[b] + (j0 + kNB) + (j0 + kNB) * ld;
        }
        t.lda = ld; t.ldb = ld; t.ldc = ld;
        t.tiles_m = Nt - j - 1; t.tiles_n = wcols; t.trap = 1; t.alpha = -1.0; t.beta = 1.0;
        if ((rc = gemm(c, t, kBNK, 2))) return rc;
      }
    }
    const int rem = Nt - b1;
    if (rem <= 0) continue;
    const long long c0 = (long long)b0 * kNB, t0 = (long long)b1 * kNB;
    GemmArgs t = gemm_base(c);
    for (int b = 0; b < 2; ++b) {
      t.A[b] = S[b] + t0 + c0 * ld;   // B[T, b0:b1]
      t.B[b] = L + t0 + c0 * ld;      // L[T, b0:b1]
      t.C[b] = S[b] + t0 + t0 * ld;
    }
    t.lda = ld; t.ldb = ld; t.ldc = ld;
    t.K = (b1 - b0) * kNB;
    t.tiles_m = rem; t.lower = 1; t.alpha = -1.0; t.beta = 1.0;
    if ((rc = gemm(c, t, kBNK, 2))) return rc;
  }
  return MLE_OK;
}

int begin_eval(mle_ctx* c, const double theta[3], ThetaParams* P) {
  if (!theta) return fail(MLE_INVALID, "theta is null");
  if (mle_fill_theta(theta, c->nugget, P) != 0)
    return fail(MLE_INVALID, "MaternParams components must be finite and > 0");
  CUDA_TRY(cudaSetDevice(c->device));
  CUDA_TRY(cudaMemsetAsync(c->fail_flag, 0, sizeof(int), c->stream));
  c->launches = 0.0;
  return MLE_OK;
}

int finish_eval(mle_ctx* c, int64_t* bad_pivot, bool derivs) {
  CUDA_TRY(cudaMemcpyAsync(c->h_res, c->out, sizeof(double) * 9, cudaMemcpyDeviceToHost,
                           c->stream));
  CUDA_TRY(cudaMemcpyAsync(c->h_res + 9, c->fail_flag, sizeof(int), cudaMemcpyDeviceToHost,
                           c->stream));
  CUDA_TRY(cudaMemcpyAsync(c->h_res + 10, c->fail_idx, sizeof(long long),
                           cudaMemcpyDeviceToHost, c->stream));
  CUDA_TRY(cudaStreamSynchronize(c->stream));
  CUDA_TRY(cudaGetLastError());
  float ms[4];
  for (int p = 0; p < 4; ++p) CUDA_TRY(cudaEventElapsedTime(&ms[p], c->ev[p], c->ev[p + 1]));
  c->phase_ms[MLE_PHASE_GEN] = ms[0];
  c->phase_ms[MLE_PHASE_POTRF] = ms[1];
  c->phase_ms[MLE_PHASE_SOLVE] = ms[2];
  c->phase_ms[MLE_PHASE_REDUCE] = ms[3];
  c->phase_ms[MLE_PHASE_TOTAL] = ms[0] + ms[1] + ms[2] + ms[3];
  const double nd = (double)c->n;
  c->flops = nd * nd * nd / 3.0 + (derivs ? 2.0 * (nd * nd * nd + nd * nd * nd / 3.0) : 0.0);
  c->gen_bytes = 8.0 * nd * (nd + 1.0) / 2.0 * (derivs ? 3.0 : 1.0);
  int flag;
  std::memcpy(&flag, c->h_res + 9, sizeof(int));
  if (flag) {
    long long idx;
    std::memcpy(&idx, c->h_res + 10, sizeof(long long));
    if (bad_pivot) *bad_pivot = idx;
    return fail(MLE_NOT_PD, "matrix not positive definite at pivot " + std::to_string(idx));
  }
  if (bad_pivot) *bad_pivot = -1;
  return MLE_OK;
}

GenArgs gen_args(const mle_ctx* c, const ThetaParams& P) {
  GenArgs a;
  std::memset(&a, 0, sizeof(a));
  a.P = P;
  a.lx = c->lx;
  a.ly = c->ly;
  a.z = c->z;
  a.sigma = c->sigma;
  a.dalpha = c->sa;
  a.dnu = c->sn;
  a.ld = c->N;
  a.rows = c->N;
  a.n = (int)c->n;
  a.fail_flag = c->fail_flag;
  return a;
}

int check_finite(const double* v, int64_t m, const char* what) {
  for (int64_t i = 0; i < m; ++i)
    if (!std::isfinite(v[i])) return fail(MLE_INVALID, std::string(what) + " must be finite");
  return MLE_OK;
}

}  // namespace

extern "C" {

const char* mle_version(void) { return "maternfisher-b200 0.1.0 (sm_100a)"; }
const char* mle_last_error(void) { return g_last_error.c_str(); }

int mle_device_count(void) {
  int count = 0;
  if (cudaGetDeviceCount(&count) != cudaSuccess) return 0;
  return count;
}

int mle_ctx_create(const double* locs_xy, const double* z, int64_t n, int device, double nugget,
                   mle_ctx** out) {
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
  c->N = round_up(n + 1, kNB);
  c->Nt = (int)(c->N / kNB);
  c->nugget = nugget;
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
  CTX_TRY(cudaStreamCreateWithFlags(&c->stream, cudaStreamNonBlocking));
  for (auto& e : c->ev) CTX_TRY(cudaEventCreate(&e));
  CTX_TRY(cudaMalloc(&c->lx, sizeof(double) * n));
  CTX_TRY(cudaMalloc(&c->ly, sizeof(double) * n));
  CTX_TRY(cudaMalloc(&c->z, sizeof(double) * n));
  CTX_TRY(cudaMalloc(&c->fail_flag, sizeof(int)));
  CTX_TRY(cudaMalloc(&c->fail_idx, sizeof(long long)));
  CTX_TRY(cudaMalloc(&c->partials, sizeof(double) * 148 * 4 * 7));
  CTX_TRY(cudaMalloc(&c->out, sizeof(double) * 9));
  CTX_TRY(cudaMallocHost(&c->h_res, sizeof(double) * 12));
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
  if (c->stream) cudaStreamSynchronize(c->stream);
  cudaFree(c->lx);
  cudaFree(c->ly);
  cudaFree(c->z);
  cudaFree(c->sigma);
  cudaFree(c->sa);
  cudaFree(c->sn);
  cudaFree(c->linv);
  cudaFree(c->fail_flag);
  cudaFree(c->fail_idx);
  cudaFree(c->partials);
  cudaFree(c->out);
  if (c->h_res) cudaFreeHost(c->h_res);
  for (auto& e : c->ev)
    if (e) cudaEventDestroy(e);
  if (c->stream) cudaStreamDestroy(c->stream);
  delete c;
}

int64_t mle_ctx_n(const mle_ctx* c) { return c ? c->n : -1; }

int mle_ctx_set_values(mle_ctx* c, const double* z) {
  if (!c || !z) return fail(MLE_INVALID, "null argument");
  int rc = check_finite(z, c->n, "values");
  if (rc) return rc;
  CUDA_TRY(cudaSetDevice(c->device));
  CUDA_TRY(cudaMemcpyAsync(c->z, z, sizeof(double) * c->n, cudaMemcpyHostToDevice, c->stream));
  CUDA_TRY(cudaStreamSynchronize(c->stream));
  return MLE_OK;
}

int mle_loglik(mle_ctx* c, const double theta[3], double* loglik, int64_t* bad_pivot) {
  if (!c || !loglik) return fail(MLE_INVALID, "null argument");
  ThetaParams P;
  int rc = begin_eval(c, theta, &P);
  if (rc) return rc;
  rc = ensure_matrices(c, false);
  if (rc) return rc;
  CUDA_TRY(cudaEventRecord(c->ev[0], c->stream));
  ++c->launches;
  launch_gen_engine(gen_args(c, P), false, c->stream);
  CUDA_TRY(cudaGetLastError());
  CUDA_TRY(cudaEventRecord(c->ev[1], c->stream));
  rc = run_potrf(c, c->sigma, c->N, c->Nt, c->n);
  if (rc) return rc;
  CUDA_TRY(cudaEventRecord(c->ev[2], c->stream));
  CUDA_TRY(cudaEventRecord(c->ev[3], c->stream));
  c->launches += 2;
  CUDA_TRY(launch_reduce_loglik(c->sigma, c->N, (int)c->n, c->partials, c->out, c->fail_flag,
                                c->stream));
  CUDA_TRY(cudaEventRecord(c->ev[4], c->stream));
  rc = finish_eval(c, bad_pivot, false);
  if (rc) return rc;
  const double logdet = c->h_res[0], quad = c->h_res[1];
  *loglik = -0.5 * (double)c->n * kLog2Pi - logdet - 0.5 * quad;  // likelihood.py:85-89
  return MLE_OK;
}

int mle_eval_all(mle_ctx* c, const double theta[3], double* loglik, double grad[3],
                 double fisher[9], int64_t* bad_pivot) {
  if (!c || !loglik || !grad || !fisher) return fail(MLE_INVALID, "null argument");
  if (c->nugget != 0.0)
    return fail(MLE_INVALID, "eval_all with a nugget is not implemented yet (loglik only)");
  ThetaParams P;
  int rc = begin_eval(c, theta, &P);
  if (rc) return rc;
  rc = ensure_matrices(c, true);
  if (rc) return rc;
  CUDA_TRY(cudaEventRecord(c->ev[0], c->stream));
  ++c->launches;
  launch_gen_engine(gen_args(c, P), true, c->stream);
  CUDA_TRY(cudaGetLastError());
  CUDA_TRY(cudaEventRecord(c->ev[1], c->stream));
  rc = run_potrf(c, c->sigma, c->N, c->Nt, c->n);
  if (rc) return rc;
  CUDA_TRY(cudaEventRecord(c->ev[2], c->stream));
  rc = run_solves(c);
  if (rc) return rc;
  CUDA_TRY(cudaEventRecord(c->ev[3], c->stream));
  c->launches += 2;
  CUDA_TRY(launch_reduce_eval(c->sigma, c->sa, c->sn, c->N, (int)c->n, c->partials, c->out,
                              c->fail_flag, c->stream));
  CUDA_TRY(cudaEventRecord(c->ev[4], c->stream));
  rc = finish_eval(c, bad_pivot, true);
  if (rc) return rc;
  const double* r = c->h_res;
  const double n = (double)c->n, s2 = P.sigma2;
  const double logdet = r[0], quad = r[1], tr_a = r[2], tr_n = r[3];
  const double faa = r[4], fan = r[5], fnn = r[6], yby_a = r[7], yby_n = r[8];
  *loglik = -0.5 * n * kLog2Pi - logdet - 0.5 * quad;            // likelihood.py:123
  grad[0] = (quad - n) / (2.0 * s2);                              // likelihood.py:129
  grad[1] = -0.5 * tr_a + 0.5 * yby_a;                            // likelihood.py:137
  grad[2] = -0.5 * tr_n + 0.5 * yby_n;
  fisher[0] = n / (2.0 * s2 * s2);                                // likelihood.py:130
  fisher[1] = fisher[3] = tr_a / (2.0 * s2);                      // likelihood.py:141
  fisher[2] = fisher[6] = tr_n / (2.0 * s2);                      // likelihood.py:145
  fisher[4] = 0.5 * faa;                                          // likelihood.py:142
  fisher[5] = fisher[7] = 0.5 * fan;                              // likelihood.py:146
  fisher[8] = 0.5 * fnn;                                          // likelihood.py:147
  return MLE_OK;
}

int mle_build(mle_ctx* c, const double theta[3], int which, double* out_host) {
  if (!c || !out_host) return fail(MLE_INVALID, "null argument");
  if (which < MLE_WHICH_SIGMA || which > MLE_WHICH_NU)
    return fail(MLE_INVALID, "which must be one of sigma, sigma2, alpha, nu");
  ThetaParams P;
  int rc = begin_eval(c, theta, &P);
  if (rc) return rc;
  rc = ensure_matrices(c, false);
  if (rc) return rc;
  GenArgs a = gen_args(c, P);
  a.ld = c->n;
  a.rows = c->n;
  launch_gen_build(a, which, c->stream);
  CUDA_TRY(cudaGetLastError());
  CUDA_TRY(cudaMemcpyAsync(out_host, c->sigma, sizeof(double) * (size_t)c->n * (size_t)c->n,
                           cudaMemcpyDeviceToHost, c->stream));
  CUDA_TRY(cudaStreamSynchronize(c->stream));
  return MLE_OK;
}

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
    double* dA = nullptr;
    ~Guard() {
      cudaFree(dA);
      cudaFree(c->linv);
      cudaFree(c->fail_flag);
      cudaFree(c->fail_idx);
      if (c->h_res) cudaFreeHost(c->h_res);
      if (c->stream) cudaStreamDestroy(c->stream);
      c->linv = nullptr;
      c->fail_flag = nullptr;
      c->fail_idx = nullptr;
      c->h_res = nullptr;
      c->stream = nullptr;
    }
  } guard{&c};
  CUDA_TRY(cudaStreamCreateWithFlags(&c.stream, cudaStreamNonBlocking));
  CUDA_TRY(cudaMalloc(&guard.dA, sizeof(double) * (size_t)N * N));
  CUDA_TRY(cudaMalloc(&c.linv, sizeof(double) * (size_t)c.Nt * kNB * kNB));
  CUDA_TRY(cudaMalloc(&c.fail_flag, sizeof(int)));
  CUDA_TRY(cudaMalloc(&c.fail_idx, sizeof(long long)));
  CUDA_TRY(cudaMallocHost(&c.h_res, sizeof(double) * 12));
  CUDA_TRY(cudaMemcpyAsync(guard.dA, h.data(), sizeof(double) * (size_t)N * N,
                           cudaMemcpyHostToDevice, c.stream));
  CUDA_TRY(cudaMemsetAsync(c.fail_flag, 0, sizeof(int), c.stream));
  rc = run_potrf(&c, guard.dA, N, c.Nt, -1);
  if (rc) return rc;
  CUDA_TRY(cudaMemcpyAsync(h.data(), guard.dA, sizeof(double) * (size_t)N * N,
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
  cudaStream_t s = nullptr;
  struct G {
    double** a;
    double** b;
    cudaStream_t* s;
    ~G() {
      cudaFree(*a);
      cudaFree(*b);
      if (*s) cudaStreamDestroy(*s);
    }
  } guard{&dx, &dy, &s};
  CUDA_TRY(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking));
  CUDA_TRY(cudaMalloc(&dx, sizeof(double) * m));
  CUDA_TRY(cudaMalloc(&dy, sizeof(double) * m));
  CUDA_TRY(cudaMemcpyAsync(dx, x, sizeof(double) * m, cudaMemcpyHostToDevice, s));
  launch_elem(P, op, which, dx, m, dy, s);
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
