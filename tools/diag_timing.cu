// Developer harness: phase timestamps (clock64) inside potrf_diag_kernel.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -DMLE_DIAG_TIMING \
//      -o tools/diag_timing tools/diag_timing.cu
#include <cstdio>
#include <vector>

#include "../paper_2601_11437_b200/csrc/linalg.cu"

int main() {
  const int n = 128 * 4;
  std::vector<double> h((size_t)n * n);
  for (int j = 0; j < n; ++j)
    for (int i = 0; i < n; ++i) h[(size_t)j * n + i] = (i == j) ? n : 1.0 / (1.0 + (i - j) * (i - j));
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
    for (int J = 0; J < 8; ++J)
      printf("  J=%d  chol16 %6lld  panel %6lld  trailing %6lld cycles\n", J,
             c[1 + 3 * J] - (J ? c[3 * J] : c[0]), c[2 + 3 * J] - c[1 + 3 * J],
             c[3 + 3 * J] - c[2 + 3 * J]);
    printf("  inverse: diag blocks %lld, block rows %lld cycles\n", c[25] - c[24], c[26] - c[25]);
  }
  return 0;
}
