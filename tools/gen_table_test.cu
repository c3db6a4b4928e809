// Developer harness: generation tables (Chebyshev pieces of e^u * {c, dalpha, dnu}) vs the exact
// evaluator, elementwise, over a dense sweep of u for many theta (incl. the FD bands).
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o tools/gen_table_test \
//   tools/gen_table_test.cu paper_2601_11437_b200/csrc/prologue.cpp
#include <cmath>
#include <cstdio>
#include <vector>

#include "../paper_2601_11437_b200/csrc/gen.cu"

using namespace mle;

__global__ void eval_kernel(const ThetaParams* P, const double* tab, const double* u, int m,
                            double* out) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= m) return;
  const MaternVals e = matern_u<true>(*P, u[i]);
  const MaternVals t = matern_table<true>(*P, tab, u[i]);
  out[6 * i + 0] = e.c;
  out[6 * i + 1] = e.dalpha;
  out[6 * i + 2] = e.dnu;
  out[6 * i + 3] = t.c;
  out[6 * i + 4] = t.dalpha;
  out[6 * i + 5] = t.dnu;
}

int main() {
  std::vector<double> uu((MLE_CASE3_NEAR + 1) * MLE_U_COEFF_STRIDE),
      du((MLE_CASE3_NEAR + 1) * MLE_U_COEFF_STRIDE);
  mle_fill_u_tables(uu.data(), du.data());
  upload_u_tables(uu.data(), du.data());
  const double thetas[][3] = {{1.0, 0.2, 1.5},  {0.8, 0.1, 1.0},   {1.0, 0.1, 0.5},
                              {1.5, 0.05, 0.8}, {0.9, 0.08, 1.013}, {2.0, 1.0, 2.7},
                              {1.0, 0.01, 1.2}, {0.5, 3.0, 0.3},    {1.0, 0.002, 0.5000001}};
  const int m = 200000;
  double worst[3] = {0, 0, 0};
  for (const auto& th : thetas) {
    ThetaParams P;
    if (mle_fill_theta(th, 0.0, &P) != 0) {
      printf("bad theta\n");
      return 1;
    }
    const double h_max = 1.8;
    mle_fill_gen_table(h_max / th[1], &P);
    ThetaParams* dP;
    double *dtab, *du_, *dout;
    cudaMalloc(&dP, sizeof(P));
    cudaMemcpy(dP, &P, sizeof(P), cudaMemcpyHostToDevice);
    cudaMalloc(&dtab, sizeof(double) * MLE_TAB_DOUBLES);
    GenArgs a{};
    a.item[0].P = dP;
    a.item[0].tab = dtab;
    launch_gen_table(a, 1, true, 0);
    std::vector<double> u(m);
    const double lo = P.tab_lo, hi = P.tab_hi;
    for (int i = 0; i < m; ++i) u[i] = lo * std::pow(hi / lo, (i + 0.5) / m);
    cudaMalloc(&du_, sizeof(double) * m);
    cudaMalloc(&dout, sizeof(double) * 6 * m);
    cudaMemcpy(du_, u.data(), sizeof(double) * m, cudaMemcpyHostToDevice);
    eval_kernel<<<(m + 255) / 256, 256>>>(dP, dtab, du_, m, dout);
    std::vector<double> o(6 * (size_t)m);
    cudaMemcpy(o.data(), dout, sizeof(double) * 6 * m, cudaMemcpyDeviceToHost);
    double e[3] = {0, 0, 0}, scale[3] = {0, 0, 0}, eabs[3] = {0, 0, 0};
    int wi[3] = {0, 0, 0};
    for (int i = 0; i < m; ++i)
      for (int f = 0; f < 3; ++f) scale[f] = std::fmax(scale[f], std::fabs(o[6 * i + f]));
    for (int i = 0; i < m; ++i)
      for (int f = 0; f < 3; ++f) {
        const double ex = o[6 * i + f], tb = o[6 * i + 3 + f];
        // relative to the element, floored at 1e-12 of the function's scale
        const double d = std::fabs(tb - ex) / std::fmax(std::fabs(ex), 1e-12 * scale[f]);
        if (d > e[f]) { e[f] = d; wi[f] = i; }
        eabs[f] = std::fmax(eabs[f], std::fabs(tb - ex) / scale[f]);
      }
    {
      const int i = wi[2];
      printf("   worst dnu at u=%.6f exact %.17g table %.17g | max |err|/max|f|: c %.1e da %.1e dnu %.1e\n",
             u[i], o[6 * i + 2], o[6 * i + 5], eabs[0], eabs[1], eabs[2]);
      // local noise of the exact evaluator: neighbours
      for (int d = -2; d <= 2; ++d) {
        const int q = i + d;
        if (q >= 0 && q < m) printf("     u=%.9f exact %.17g table %.17g\n", u[q], o[6*q+2], o[6*q+5]);
      }
    }
    printf("theta (%g, %g, %.7g): intervals %d, u in [%g, %g) | max rel err c %.2e  dalpha %.2e"
           "  dnu %.2e  (%s)\n", th[0], th[1], th[2], P.tab_n, lo, hi, e[0], e[1], e[2],
           cudaGetErrorString(cudaGetLastError()));
    for (int f = 0; f < 3; ++f) worst[f] = std::fmax(worst[f], e[f]);
    cudaFree(dP);
    cudaFree(dtab);
    cudaFree(du_);
    cudaFree(dout);
  }
  printf("worst: c %.2e dalpha %.2e dnu %.2e\n", worst[0], worst[1], worst[2]);
  return 0;
}
