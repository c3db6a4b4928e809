// kernels.h — internal launch interface between the C-ABI engine (engine.cu) and the
// sm_100a kernels (gen.cu, linalg.cu).  Not part of the public ABI.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include "../../include/maternfisher.h"
#include "theta.h"

namespace mle {

constexpr int kNB = 128;  // factorization tile (Cholesky / solve block size)

struct GenArgs {
  ThetaParams P;
  const double* lx;   // x coordinates (n)
  const double* ly;   // y coordinates (n)
  const double* z;    // observed values (n); augmented row
  double* sigma;      // Sigma (engine) or the single output (build)
  double* dalpha;     // dSigma/dalpha (full storage)
  double* dnu;        // dSigma/dnu (full storage)
  long long ld;       // leading dimension (column-major)
  long long rows;     // padded extent N (engine) / n (build)
  int n;              // number of locations
  const int* fail_flag;
};

// Operand layouts of op(B): B(n,k) at b[n + k*ldb] (kBNK) or b[k + n*ldb] (kBKN).
enum BLayout { kBNK = 0, kBKN = 1 };

struct GemmArgs {
  const double* A[2];
  const double* B[2];
  double* C[2];
  long long lda, ldb, ldc;
  int K;             // multiple of 16
  int tiles_m;       // number of 128-row tiles of C
  int tiles_n;       // number of 128-column tiles of C (full mode)
  int lower;         // 1: only tiles (tm >= tn) of a tiles_m x tiles_m grid
  int trap;          // full mode: 1 skips tiles with tm < tn (lower trapezoid)
  double alpha;      // +1 or -1
  double beta;       // 0 (overwrite) or 1 (accumulate into C)
  const int* fail_flag;
};

cudaError_t init_kernel_attributes();  // GEMM smem opt-in (per device)
cudaError_t init_diag_attributes();    // diagonal-tile kernel smem opt-in (per device)
cudaError_t upload_u_tables(const double* u, const double* du);
void launch_gen_engine(const GenArgs& a, bool derivs, cudaStream_t s);
void launch_gen_build(const GenArgs& a, int which, cudaStream_t s);
void launch_elem(const ThetaParams& P, int op, int which, const double* x, long long m,
                 double* out, cudaStream_t s);

// C = alpha * A * op(B)^T-style product (see linalg.cu) + beta * C, batched over gridDim.z.
cudaError_t launch_gemm(const GemmArgs& g, BLayout bl, int batch, cudaStream_t s);
// Factor the 128x128 diagonal tile at (k0, k0) in place and write its inverse to linv.
cudaError_t launch_potrf_diag(double* a, long long ld, int k0, long long n_aug, double* linv,
                              int* fail_flag, long long* fail_idx, cudaStream_t s);
// Reductions: 7 partial sums per block over the first n indices.
cudaError_t launch_reduce_eval(const double* L, const double* Ba, const double* Bn,
                               long long ld, int n, double* partials, double* out,
                               const int* fail_flag, cudaStream_t s);
cudaError_t launch_reduce_loglik(const double* L, long long ld, int n, double* partials,
                                 double* out, const int* fail_flag, cudaStream_t s);
cudaError_t launch_clear_upper(double* a, long long ld, int n, cudaStream_t s);

}  // namespace mle
