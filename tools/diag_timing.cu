// Developer harness: phase timestamps (clock64) inside potrf_diag_kernel, plus the accuracy
// of the factor and inverse of one 128x128 tile (L L^T - A and Linv L - I).
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -DMLE_DIAG_TIMING \
//      -o tools/diag_timing tools/diag_timing.cu
#include <cmath>
#include <cstdio>
#include <random>
#include <vector>

#include "../paper_2601_11437_b200/csrc/linalg.cu"

int main() {
  const int n = 128 * 4;
  std::vector<double> h((size_t)n * n);
  std::mt19937_64 rng(7);
  std::uniform_real_distribution<double> U(0.0, 1.0);
  std::vector<double> px(n), py(n);
  for (int i = 0; i < n; ++i) px[i] = U(rng), py[i] = U(rng);
  // exponential covariance (nu = 1/2, range 0.2) + small nugget: a realistic tile
  for (int j = 0; j < n; ++j)
    for (int i = 0; i < n; ++i) {
      const double r = std::hypot(px[i] - px[j], py[i] - py[j]);
      h[(size_t)j * n + i] = std::exp(-r / 0.2) + (i == j ? 1e-3 : 0.0);
    }
  double *a, *linv;
  int* flag;
  long long* idx;
  cudaMalloc(&a, sizeof(double) * n * n);
  cudaMalloc(&linv, sizeof(double) * 128 * 128);
  cudaMalloc(&flag, 4);
  cudaMalloc(&idx, 8);
  cudaMemset(flag, 0, 4);
  mle::init_diag_attributes();
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  for (int rep = 0; rep < 3; ++rep) {
    cudaMemcpy(a, h.data(), sizeof(double) * n * n, cudaMemcpyHostToDevice);
    cudaMemset(flag, 0, 4);
    cudaEventRecord(e0);
    mle::DiagArgs d = {};
    d.a[0] = a; d.linv[0] = linv; d.fail_flag[0] = flag; d.fail_idx[0] = idx;
    d.n_aug[0] = -1; d.ld = n; d.k0 = 0;
    mle::launch_potrf_diag(d, 1, 0);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    long long c[32];
    cudaMemcpyFromSymbol(c, mle::g_diag_clock, sizeof(c));
    printf("kernel %.1f us; err=%s\n", ms * 1e3, cudaGetErrorString(cudaGetLastError()));
    long long tot = 0;
    for (int J = 0; J < 8; ++J) {
      printf("  J=%d  chol16 %6lld  panel %6lld  trailing %6lld cycles\n", J,
             c[1 + 3 * J] - (J ? c[3 * J] : c[0]), c[2 + 3 * J] - c[1 + 3 * J],
             c[3 + 3 * J] - c[2 + 3 * J]);
    }
    tot = c[26] - c[0];
    printf("  inverse: diag blocks %lld, block rows %lld cycles | total %lld cycles\n",
           c[25] - c[24], c[26] - c[25], tot);
  }
  std::vector<double> L((size_t)n * n), X(128 * 128);
  cudaMemcpy(L.data(), a, sizeof(double) * n * n, cudaMemcpyDeviceToHost);
  cudaMemcpy(X.data(), linv, sizeof(double) * 128 * 128, cudaMemcpyDeviceToHost);
  double ef = 0, ei = 0;
  for (int i = 0; i < 128; ++i)
    for (int j = 0; j <= i; ++j) {
      double s = 0;
      for (int k = 0; k <= j; ++k) s += L[(size_t)k * n + i] * L[(size_t)k * n + j];
      ef = std::fmax(ef, std::fabs(s - h[(size_t)j * n + i]));
    }
  for (int i = 0; i < 128; ++i)
    for (int j = 0; j < 128; ++j) {
      double s = 0;  // (Linv L)(i, j), Linv row-major? linv[idx], idx = i + 128 j (column-major)
      for (int k = 0; k < 128; ++k) s += X[i + 128 * k] * (k >= j ? L[(size_t)j * n + k] : 0.0);
      ei = std::fmax(ei, std::fabs(s - (i == j ? 1.0 : 0.0)));
    }
  printf("max |L L^T - A| = %.3e   max |Linv L - I| = %.3e\n", ef, ei);
  return 0;
}
