// Developer harness: Ozaki int8-tcgen05 FP64 GEMM vs the DMMA GEMM vs a long-double CPU
// reference, on Cholesky-like operands; prints max |err| / (|A||B| scale) and TF/s.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o tools/oz_gemm_test \
//   tools/oz_gemm_test.cu paper_2601_11437_b200/csrc/linalg.cu paper_2601_11437_b200/csrc/ozaki.cu
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <random>
#include <vector>

#include "../paper_2601_11437_b200/csrc/kernels.h"

#define CK(x) do { cudaError_t e_ = (x); if (e_ != cudaSuccess) { printf("CUDA %s @%d\n", cudaGetErrorString(e_), __LINE__); exit(1);} } while (0)

using namespace mle;
static int g_ntile = 0;
static int g_slices = 7;

struct Case {
  const char* name;
  int M, N, K;
  bool lower;      // C lower (M == N), B = A (potrf outer update)
  bool b_kcontig;  // B(n,k) at X[k + n*ld] (solve-1 operand)
};

static double run_case(const Case& cs, int batch, int reps) {
  const int M = cs.M, N = cs.N, K = cs.K;
  std::mt19937_64 rng(42);
  std::normal_distribution<double> nd;
  // A: M x K column-major (ld = M); rows scaled over a few decades like a factor panel
  std::vector<double> A((size_t)M * K), Bm, C((size_t)M * N);
  for (int i = 0; i < M; ++i) {
    const double sc = std::pow(10.0, -3.0 * (double)(i % 7) / 7.0);
    for (int k = 0; k < K; ++k) A[i + (size_t)k * M] = sc * nd(rng) / std::sqrt((double)K);
  }
  const long long ldb = cs.b_kcontig ? K : N;
  if (!cs.lower) {
    Bm.resize((size_t)N * K);
    for (int j = 0; j < N; ++j)
      for (int k = 0; k < K; ++k) {
        const double v = nd(rng) * (1.0 + 0.1 * (k % 5));
        if (cs.b_kcontig) Bm[k + (size_t)j * ldb] = v; else Bm[j + (size_t)k * ldb] = v;
      }
  }
  for (auto& c : C) c = nd(rng);
  auto bval = [&](int j, int k) {
    if (cs.lower) return A[j + (size_t)k * M];
    return cs.b_kcontig ? Bm[k + (size_t)j * ldb] : Bm[j + (size_t)k * ldb];
  };

  double *dA, *dB = nullptr, *dC1, *dC2;
  int8_t *sA, *sB;
  int *eA, *eB, *flag;
  CK(cudaMalloc(&dA, A.size() * 8));
  CK(cudaMemcpy(dA, A.data(), A.size() * 8, cudaMemcpyHostToDevice));
  if (!cs.lower) {
    CK(cudaMalloc(&dB, Bm.size() * 8));
    CK(cudaMemcpy(dB, Bm.data(), Bm.size() * 8, cudaMemcpyHostToDevice));
  }
  CK(cudaMalloc(&dC1, C.size() * 8));
  CK(cudaMalloc(&dC2, C.size() * 8));
  CK(cudaMalloc(&sA, oz_slice_bytes(M, K)));
  CK(cudaMalloc(&sB, oz_slice_bytes(N, K)));
  CK(cudaMalloc(&eA, M * 4));
  CK(cudaMalloc(&eB, N * 4));
  CK(cudaMalloc(&flag, 4));
  CK(cudaMemset(flag, 0, 4));
  CK(cudaMemcpy(dC1, C.data(), C.size() * 8, cudaMemcpyHostToDevice));
  CK(cudaMemcpy(dC2, C.data(), C.size() * 8, cudaMemcpyHostToDevice));

  GemmArgs g{};
  OzSliceArgs sa{}, sb{};
  OzGemmArgs o{};
  for (int z = 0; z < batch; ++z) {  // batch members alias (timing only; z=0 checked)
    g.A[z] = dA; g.B[z] = cs.lower ? dA : dB; g.C[z] = dC1; g.fail_flag[z] = flag;
    sa.X[z] = dA; sa.slices[z] = sA; sa.e[z] = eA; sa.fail_flag[z] = flag;
    sb.X[z] = dB; sb.slices[z] = sB; sb.e[z] = eB; sb.fail_flag[z] = flag;
    o.As[z] = sA; o.Bs[z] = cs.lower ? sA : sB; o.ea[z] = eA; o.eb[z] = cs.lower ? eA : eB;
    o.C[z] = dC2; o.fail_flag[z] = flag;
  }
  g.lda = M; g.ldb = cs.lower ? M : ldb; g.ldc = M; g.K = K; g.tiles_m = M / 128;
  g.tiles_n = N / 128; g.lower = cs.lower; g.trap = 0; g.wide = 0; g.alpha = -1; g.beta = 1;
  sa.ld = M; sa.K = K; sb.ld = ldb; sb.K = K;
  o.ldc = M; o.kblocks = K / 32; o.tiles_m = M / 128; o.tiles_n = N / 128; o.lower = cs.lower;
  o.trap = 0; o.alpha = -1; o.beta = 1;
  o.nslices = g_slices; sa.nslices = g_slices; sb.nslices = g_slices;
  const BLayout bl = (cs.lower || !cs.b_kcontig) ? kBNK : kBKN;

  // one checked application each
  CK(launch_gemm(g, bl, 1, 0));
  CK(launch_oz_slice(sa, M, true, 1, 0));
  if (!cs.lower) CK(launch_oz_slice(sb, N, !cs.b_kcontig, 1, 0));
  CK(launch_ozgemm(o, 1, 0, g_ntile));
  CK(cudaDeviceSynchronize());
  std::vector<double> C1(C.size()), C2(C.size());
  CK(cudaMemcpy(C1.data(), dC1, C.size() * 8, cudaMemcpyDeviceToHost));
  CK(cudaMemcpy(C2.data(), dC2, C.size() * 8, cudaMemcpyDeviceToHost));
  for (int other : {0, 1, 2, 3}) {  // every kernel variant must give bit-identical results
    if (other == g_ntile) continue;
    CK(cudaMemcpy(dC2, C.data(), C.size() * 8, cudaMemcpyHostToDevice));
    CK(launch_ozgemm(o, 1, 0, other));
    CK(cudaDeviceSynchronize());
    std::vector<double> C3(C.size());
    CK(cudaMemcpy(C3.data(), dC2, C.size() * 8, cudaMemcpyDeviceToHost));
    long diff = 0;
    for (int j = 0; j < N; ++j)
      for (int i = cs.lower ? j : 0; i < M; ++i) diff += C3[i + (size_t)j * M] != C2[i + (size_t)j * M];
    if (diff) printf("  !! n_tile %d vs %d: %ld differing entries\n", g_ntile, other, diff);
  }
  CK(cudaMemcpy(dC2, C.data(), C.size() * 8, cudaMemcpyHostToDevice));
  double e1 = 0, e2 = 0, e12 = 0;
  std::uniform_int_distribution<int> ri(0, M - 1), rj(0, N - 1);
  for (int t = 0; t < 20000; ++t) {
    int i = ri(rng), j = rj(rng);
    if (cs.lower && j > i) std::swap(i, j);
    long double acc = C[i + (size_t)j * M], sc = fabsl(acc);
    for (int k = 0; k < K; ++k) {
      const long double p = (long double)A[i + (size_t)k * M] * bval(j, k);
      acc -= p;
      sc += fabsl(p);
    }
    const size_t idx = i + (size_t)j * M;
    e1 = std::max(e1, (double)(fabsl(C1[idx] - acc) / sc));
    e2 = std::max(e2, (double)(fabsl(C2[idx] - acc) / sc));
    e12 = std::max(e12, std::fabs(C1[idx] - C2[idx]) / (double)sc);
  }
  // timing (C keeps accumulating; values irrelevant)
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  const double area = cs.lower ? (double)M * (M + 128) / 2 : (double)M * N;
  const double flops = 2.0 * area * K * batch;
  float t_d = 0, t_s = 0, t_o = 0;
  for (int pass = 0; pass < 2; ++pass) {
    cudaEventRecord(a);
    for (int r = 0; r < reps; ++r) launch_gemm(g, bl, batch, 0);
    cudaEventRecord(b);
    CK(cudaEventSynchronize(b));
    cudaEventElapsedTime(&t_d, a, b);
    cudaEventRecord(a);
    for (int r = 0; r < reps; ++r) {
      launch_oz_slice(sa, M, true, batch, 0);
      if (!cs.lower) launch_oz_slice(sb, N, !cs.b_kcontig, batch, 0);
    }
    cudaEventRecord(b);
    CK(cudaEventSynchronize(b));
    cudaEventElapsedTime(&t_s, a, b);
    cudaEventRecord(a);
    for (int r = 0; r < reps; ++r) launch_ozgemm(o, batch, 0, g_ntile);
    cudaEventRecord(b);
    CK(cudaEventSynchronize(b));
    cudaEventElapsedTime(&t_o, a, b);
  }
  if (getenv("OZ_DIAG")) {  // diagnostics: loads only / MMAs only
    float t1, t2;
    o.diag_mode = 1;
    cudaEventRecord(a);
    for (int r = 0; r < reps; ++r) launch_ozgemm(o, batch, 0, g_ntile);
    cudaEventRecord(b);
    CK(cudaEventSynchronize(b));
    cudaEventElapsedTime(&t1, a, b);
    o.diag_mode = 2;
    cudaEventRecord(a);
    for (int r = 0; r < reps; ++r) launch_ozgemm(o, batch, 0, g_ntile);
    cudaEventRecord(b);
    CK(cudaEventSynchronize(b));
    cudaEventElapsedTime(&t2, a, b);
    float t3;
    o.diag_mode = 3;
    cudaEventRecord(a);
    for (int r = 0; r < reps; ++r) launch_ozgemm(o, batch, 0, g_ntile);
    cudaEventRecord(b);
    CK(cudaEventSynchronize(b));
    cudaEventElapsedTime(&t3, a, b);
    float t5;
    o.diag_mode = 5;
    cudaEventRecord(a);
    for (int r = 0; r < reps; ++r) launch_ozgemm(o, batch, 0, g_ntile);
    cudaEventRecord(b);
    CK(cudaEventSynchronize(b));
    cudaEventElapsedTime(&t5, a, b);
    long long* dd;
    CK(cudaMalloc(&dd, 8 * sizeof(long long)));
    o.diag_out = dd;
    for (int mode : {0, 5, 6, 7, 8, 9}) {
      o.diag_mode = mode;
      launch_ozgemm(o, batch, 0, g_ntile);
      long long h[8];
      CK(cudaMemcpy(h, dd, sizeof(h), cudaMemcpyDeviceToHost));
      printf("  mma thread (mode %d): %lld cycles, %.3f ms -> %.0f MHz | full-wait %.1f%% | "
             "acc-wait %.1f%% | %lld tiles, %lld k blocks -> %.0f cycles/k block\n", mode, h[0],
             h[3] * 1e-6, (double)h[0] / (h[3] * 1e-3), 100.0 * h[1] / h[0], 100.0 * h[2] / h[0],
             h[4], h[5], (double)h[0] / h[5]);
    }
    o.diag_out = nullptr;
    cudaFree(dd);
    o.diag_mode = 0;
    printf("  diag: full %.3f ms | loads+epilogue only %.3f ms | MMAs+epilogue only %.3f ms | "
           "no TMEM epilogue %.3f ms | MMAs only %.3f ms\n", t_o / reps, t1 / reps, t2 / reps,
           t3 / reps, t5 / reps);
  }
  CK(cudaGetLastError());
  printf("%-10s M=%5d N=%5d K=%d batch=%d | err/scale dmma %.2e ozaki %.2e diff %.2e | "
         "dmma %.3f ms %.1f TF/s | slice %.3f ms | ozgemm %.3f ms %.1f TF/s | oz total %.1f TF/s\n",
         cs.name, M, N, K, batch, e1, e2, e12, t_d / reps, flops / (t_d / reps) * 1e-9,
         t_s / reps, t_o / reps, flops / (t_o / reps) * 1e-9,
         flops / ((t_o + t_s) / reps) * 1e-9);
  cudaFree(dA); if (dB) cudaFree(dB); cudaFree(dC1); cudaFree(dC2); cudaFree(sA); cudaFree(sB);
  cudaFree(eA); cudaFree(eB); cudaFree(flag);
  return e2;
}

int main(int argc, char** argv) {
  CK(init_kernel_attributes());
  CK(init_ozaki_attributes());
  const Case cases[] = {
      {"potrf", 3328, 3328, 512, true, false},
      {"potrf", 16384, 16384, 512, true, false},
      {"solve1", 3328, 6656, 512, false, true},
      {"solve2", 3328, 3328, 512, false, false},
      {"solve1", 16384, 32768, 512, false, true},
  };
  if (getenv("OZ_NTILE")) g_ntile = atoi(getenv("OZ_NTILE"));
  if (getenv("OZ_SLICES")) g_slices = atoi(getenv("OZ_SLICES"));
  printf("slices %d\n", g_slices);
  printf("n_tile %d\n", g_ntile);
  if (argc > 1) {  // profiling: one case, batch, reps
    run_case(cases[atoi(argv[1])], argc > 2 ? atoi(argv[2]) : 1, argc > 3 ? atoi(argv[3]) : 1);
    return 0;
  }
  double worst = 0;
  for (const auto& c : cases) worst = std::max(worst, run_case(c, 1, 10));
  run_case(cases[0], 5, 10);
  run_case(cases[2], 5, 10);
  printf("worst ozaki err/scale %.2e\n", worst);
  return worst < (g_slices == 7 ? 1e-14 : 1e-13) ? 0 : 1;
}
