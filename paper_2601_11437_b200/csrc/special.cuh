// special.cuh — per-thread FP64 special functions for the Matern generation kernel.
//
//  * K_mu / K_{mu+1} for |mu| <= 1/2: Temme's small-argument expansion (unrolled into
//    per-theta power series) for x < 1, the trapezoidal rule on K_v's cosh integral for
//    x >= 1; then upward recurrence to K_nu and K_{nu-1}.
//    This replaces scipy.special.kv (reference call sites bessel.py:97, matern.py:104, 111,
//    123, bessel.py:322-323).
//  * d/dnu [x^nu K_nu(x)] by the reference's four-regime dispatch (bessel.py:327-370):
//    case 2 ascending series (bessel.py:184-223), case 3 uniform asymptotics
//    (bessel.py:226-283), case 4 large-x (bessel.py:286-318), forward difference
//    (bessel.py:321-324).  nu-only factors come precomputed in ThetaParams.
#pragma once
#include <cuda_runtime.h>

#include "theta.h"

namespace mle {

// Debye U_k and U_k' coefficient tables (theta independent), uploaded once per device.
// Defined here: gen.cu is the only translation unit that includes this header.
__constant__ double c_u_coef[(MLE_CASE3_NEAR + 1) * MLE_U_COEFF_STRIDE];
__constant__ double c_du_coef[(MLE_CASE3_NEAR + 1) * MLE_U_COEFF_STRIDE];
// Node values -> monomial coefficients of the generation tables' interpolants (prologue.cpp,
// mle_fill_tab_map): [hi/lo][power i][node q], a double-double pair per entry.
__constant__ double c_tab_map[2][MLE_TAB_P][MLE_TAB_P];

#define MLE_PI 3.141592653589793
#define MLE_SQRT_HALF_PI 1.2533141373155003  // sqrt(pi/2), bessel.py:58

// K_mu(x) and K_{mu+1}(x) for |mu| <= 1/2, x > 0, written from the mathematics:
//
//  * x < MLE_KSER_XMAX: Temme's small-argument expansion (N. M. Temme, J. Comput. Phys. 19
//    (1975) 324-337) in the unrolled form of prologue.cpp (fill_ladder): the series' mu-only
//    recurrences are folded into six power series in d = x^2/4 whose coefficients are fixed
//    per theta, so an element costs three x-dependent seeds (f0, p0, q0) and six Horner
//    chains of fixed length -- no data-dependent loop, warps stay converged;
//  * x >= MLE_KSER_XMAX: the integral K_v(x) = int_0^inf exp(-x cosh t) cosh(v t) dt
//    (DLMF 10.32.9) by the trapezoidal rule.  The integrand is entire and even in t, so the
//    rule converges geometrically in 1/step: with the scaled integrand exp(-x (cosh t - 1))
//    bounded by e^x on the strip |Im t| < pi/2 and by a Gaussian of variance 1/x near the
//    real axis, the step min(pi^2 / (x + 45), 0.75 / sqrt(x)) keeps the discretisation error
//    below ~e^-40 of the integral; the positive terms are summed until they no longer
//    register.  Measured against 40-digit mpmath on mu in [-1/2, 1/2]: <= 1e-15 relative for
//    x in [1/2, 700] (tests/test_gpu_special.py pins the ladder at 5e-15).
// Used by the exact evaluator only (table nodes, u < MLE_TAB_LO, u >= MLE_TAB_HI, and
// MLE_GEN_TABLE=0), never on the table fast path.
__device__ __forceinline__ void bessel_k_pair(const KLadder& L, double x, double* k_mu,
                                              double* k_mu1) {
  if (x < MLE_KSER_XMAX) {
    const double log_2_over_x = -log(0.5 * x);
    const double sig = L.mu * log_2_over_x;
    double sinhc;  // sinh(sig) / sig
    if (fabs(sig) < 1e-3) {
      const double s2 = sig * sig;
      sinhc = 1.0 + s2 * (1.0 / 6.0) * (1.0 + s2 * (1.0 / 20.0) * (1.0 + s2 * (1.0 / 42.0)));
    } else {
      sinhc = sinh(sig) / sig;
    }
    const double half_x_pow_neg_mu = exp(sig);  // (x/2)^-mu
    const double seed_f = L.f0_cosh * cosh(sig) + L.f0_sinh * sinhc * log_2_over_x;
    const double seed_p = L.p0 * half_x_pow_neg_mu;
    const double seed_q = L.q0 / half_x_pow_neg_mu;
    const double d = 0.25 * x * x;
    double acc[6];
#pragma unroll
    for (int j = 0; j < 6; ++j) acc[j] = L.ser[MLE_KSER_TERMS - 1][j];
#pragma unroll 1
    for (int k = MLE_KSER_TERMS - 2; k >= 0; --k) {
#pragma unroll
      for (int j = 0; j < 6; ++j) acc[j] = fma(acc[j], d, L.ser[k][j]);
    }
    *k_mu = seed_f * acc[0] + seed_p * acc[1] + seed_q * acc[2];
    *k_mu1 = (seed_f * acc[3] + seed_p * acc[4] + seed_q * acc[5]) * (2.0 / x);
  } else {
    const double step = fmin(MLE_PI * MLE_PI / (x + 45.0), 0.75 * rsqrt(x));
    double sum_lo = 0.5, sum_hi = 0.5;  // t = 0 node, half weight
#pragma unroll 1
    for (int node = 1; node <= MLE_KTRAP_MAX; ++node) {
      const double t = node * step;
      const double sh = sinh(0.5 * t);
      const double sh2 = sh * sh;                 // (cosh t - 1) / 2
      const double decay = exp(-2.0 * x * sh2);   // exp(-x (cosh t - 1))
      const double e_mu = exp(L.mu * t);
      const double r_mu = 1.0 / e_mu;
      const double cosh_mu = 0.5 * (e_mu + r_mu), sinh_mu = 0.5 * (e_mu - r_mu);
      const double cosh_t = 1.0 + 2.0 * sh2, sinh_t = 2.0 * sh * sqrt(1.0 + sh2);
      const double term_lo = decay * cosh_mu;
      const double term_hi = decay * (cosh_mu * cosh_t + sinh_mu * sinh_t);  // cosh((mu+1)t)
      sum_lo += term_lo;
      sum_hi += term_hi;
      if (term_hi < 1e-18 * sum_hi && x * sh2 > 1.0) break;  // past the peak, negligible
    }
    const double scale = step * exp(-x);
    *k_mu = scale * sum_lo;
    *k_mu1 = scale * sum_hi;
  }
}

// Runs the ladder: returns K_order (and K_{order-1} if wanted) for the ladder's order, by
// the upward recurrence K_{v+1} = K_{v-1} + (2v/x) K_v (stable for K).
__device__ __forceinline__ void bessel_k_ladder(const KLadder& L, double x, double* k_nu,
                                                double* k_num1) {
  double k0, k1;
  bessel_k_pair(L, x, &k0, &k1);
  const double two_over_x = 2.0 / x;
#pragma unroll 1
  for (int j = 1; j <= L.nsteps; ++j) {
    const double kn = k0 + (L.mu + (double)j) * two_over_x * k1;
    k0 = k1;
    k1 = kn;
  }
  if (L.order_is_low) {
    *k_nu = k0;
    *k_num1 = k1;
  } else {
    *k_nu = k1;
    *k_num1 = k0;
  }
}

// numpy.polynomial.polynomial.polyval order (Horner from the top coefficient).
__device__ __forceinline__ double polyval_const(const double* c, int ncoef, double p) {
  double acc = c[ncoef - 1];
#pragma unroll 1
  for (int i = ncoef - 2; i >= 0; --i) acc = c[i] + acc * p;
  return acc;
}

// Case 2: 0 < x < 8.5, nu away from integers (bessel.py:184-223).
__device__ __forceinline__ double dnu_case2(const ThetaParams& P, double x, double x_nu) {
  const double two_log_x = 2.0 * log(x);
  const double x_two_nu = x_nu * x_nu;  // x^(2 nu)
  const double quarter_x2 = 0.25 * x * x;
  const double lead = P.c2_two_m_nu * x_two_nu;
  const double log2 = 0.6931471805599453;
  double prefactor = 0.5;
  double total = 0.0;
#pragma unroll 1
  for (int k = 0; k <= MLE_CASE2_TERMS; ++k) {
    if (k > 0) prefactor = prefactor * quarter_x2 * P.recip_int[k];
    const double term_neg =
        lead * (-log2 + two_log_x - P.c2_psi_neg + P.c2_d_pos[k]) * P.c2_gam_neg * P.c2_g_pos[k];
    total = total + prefactor * (P.c2_term_pos[k] + term_neg);
  }
  return total;
}

// Case 3: 8.5 <= x < 30 (bessel.py:226-283).
__device__ __forceinline__ double dnu_case3(const ThetaParams& P, double x, double x_nu) {
  const double nu = P.nu;
  const int kterms = (x < MLE_MID_TRUNC_SPLIT) ? MLE_CASE3_NEAR : MLE_CASE3_FAR;
  const double z = x / nu;
  const double zz1 = 1.0 + z * z;
  const double root = sqrt(zz1);
  const double p = 1.0 / root;
  const double eta = root + log(z / (1.0 + root));
  const double prefactor = x_nu * P.c3_sqrt_pi_2nu * exp(-nu * eta) / sqrt(root);
  double sum_u = 0.0, sum_ku = 0.0, sum_du = 0.0;
#pragma unroll 1
  for (int k = 0; k <= kterms; ++k) {
    const double u_val = polyval_const(c_u_coef + k * MLE_U_COEFF_STRIDE, 3 * k + 1, p);
    const double du_val =
        k == 0 ? 0.0 : polyval_const(c_du_coef + k * MLE_U_COEFF_STRIDE, 3 * k, p);
    sum_u += P.c3_w[k] * u_val;
    sum_ku += P.c3_wk[k] * u_val;
    sum_du += P.c3_w[k] * du_val;
  }
  const double bracket = P.c3_log_nu + log(1.0 + root) - 1.0 / (2.0 * nu * zz1);
  return bracket * prefactor * sum_u - prefactor * sum_ku +
         (x * x / P.c3_nu3) / (zz1 * root) * prefactor * sum_du;  // (1+z^2)^-1.5
}

// Case 4: x >= 30 (bessel.py:286-318).
__device__ __forceinline__ double dnu_case4(const ThetaParams& P, double x, double x_nu) {
  const double log_x = log(x);
  double total = log_x;
  double x_pow = 1.0;
#pragma unroll 1
  for (int k = 1; k <= P.c4_kmax; ++k) {
    x_pow = x_pow / x;
    total = total + x_pow * (log_x + P.c4_b[k]) * P.c4_a[k];
  }
  return MLE_SQRT_HALF_PI * (x_nu / sqrt(x)) * exp(-x) * total;  // x^(nu - 1/2)
}

// Forward difference (bessel.py:321-324); f_lo = x^nu K_nu(x) is shared with the caller.
__device__ __forceinline__ double dnu_fd(const ThetaParams& P, double x, double f_lo) {
  double k_hi, unused;
  bessel_k_ladder(P.kfd, x, &k_hi, &unused);
  const double f_hi = pow(x, P.nu_fd) * k_hi;
  return (f_hi - f_lo) / MLE_FD_LAG;
}

// d/dnu [x^nu K_nu(x)] for x > 0 with the regime dispatch of bessel.py:327-370.
// f = x^nu K_nu(x) and x_nu = x^nu are shared with the caller.
__device__ __forceinline__ double dnu_xnu_knu(const ThetaParams& P, double x, double f,
                                              double x_nu) {
  if (x < MLE_SMALL_MID_SPLIT) {
    return P.fd_small ? dnu_fd(P, x, f) : dnu_case2(P, x, x_nu);
  } else if (x < MLE_MID_LARGE_SPLIT) {
    return dnu_case3(P, x, x_nu);
  } else {
    return P.fd_large ? dnu_fd(P, x, f) : dnu_case4(P, x, x_nu);
  }
}

// Matern covariance and its alpha / nu derivatives at distance h > 0 (matern.py:100-125).
struct MaternVals {
  double c, dalpha, dnu;
};

// Element values as functions of the scaled distance u = h / alpha > 0.
template <bool kDerivs>
__device__ __forceinline__ MaternVals matern_u(const ThetaParams& P, double u) {
  MaternVals out;
  double k_nu, k_num1;
  bessel_k_ladder(P.kmain, u, &k_nu, &k_num1);
  const double u_nu = pow(u, P.nu);
  out.c = P.scale_c * u_nu * k_nu;                                  // matern.py:104
  if (kDerivs) {
    out.dalpha = P.scale_a * (u_nu * u) * k_num1;                   // matern.py:111
    const double f = u_nu * k_nu;                                   // matern.py:122
    out.dnu = P.sigma2 * P.q * (P.dlog_q * f + dnu_xnu_knu(P, u, f, u_nu));  // matern.py:125
  } else {
    out.dalpha = 0.0;
    out.dnu = 0.0;
  }
  return out;
}

template <bool kDerivs>
__device__ __forceinline__ MaternVals matern_positive(const ThetaParams& P, double h) {
  return matern_u<kDerivs>(P, h / P.alpha);  // u = h / alpha (matern.py:103)
}

// ---- table path ------------------------------------------------------------------------
// Interval of u in [tab_lo, tab_hi): the bin from the bits of u (exponent and the top three
// mantissa bits: eight bins per binade), integer ALU only (a float log2 and its conversions
// made the XU pipe a generation bottleneck).  Bins are table intervals one to one, except
// around the reference's regime switch 8.5 (bessel.py:46): [7, 7.5), [7.5, 8) and [8, 8.5)
// form one interval [7, 8.5) and [8.5, 9) is its own.  (Below 8.5 the reference's case-2
// series cancels catastrophically, bessel.py:213-222; interpolation nodes crowded into
// [8, 8.5) fitted its noise into a coherent bias of the nu score.)
constexpr int kGenMergeKey = (2 - MLE_TAB_LO_EXP) * 8 + 6;  // bin [7, 7.5) (binade [4, 8), j = 6)
__device__ __forceinline__ int gen_tab_index(const ThetaParams& P, double u) {
  const int key = (int)((__double_as_longlong(u) >> 49) - P.tab_key0);
  return key - (key > kGenMergeKey ? 1 : 0) -
         (key > kGenMergeKey + 1 && u < MLE_SMALL_MID_SPLIT ? 1 : 0);
}

// tab: [MLE_TAB_MAX][3][MLE_TAB_P] monomial coefficients (powers of t in [-1, 1]) of
// e^u * {c, dalpha, dnu}; Horner, one FMA per term, coefficients loaded in 16-byte pairs
// (the L1 request count, not the arithmetic, bounds the generation kernels).
__device__ __forceinline__ double horner_pairs(const double* __restrict__ c, double t) {
  static_assert(MLE_TAB_P % 2 == 0, "pairs");
  double2 q = __ldg(reinterpret_cast<const double2*>(c + MLE_TAB_P - 2));
  double p = fma(q.y, t, q.x);
#pragma unroll
  for (int i = MLE_TAB_P - 4; i >= 0; i -= 2) {
    q = __ldg(reinterpret_cast<const double2*>(c + i));
    p = fma(p, t, q.y);
    p = fma(p, t, q.x);
  }
  return p;
}

// Position of u in its interval k, t in [-1, 1].  On a bin (u = 2^e m, m in [1, 2), bin j =
// the top three mantissa bits; centre 2^e (1 + (2j + 1)/16), half-width 2^e / 16) it is
// t = 16 m' - 17 exactly, m' = 1 + (the mantissa below those three bits): no table loads,
// no conversion.  [8.5, 9) gives 4 u - 35 exactly and the merged [7, 8.5) (u - 7.75) / 0.75.
// Branch-free (selects), so a warp's elements evaluate in lock step.
__device__ __forceinline__ double gen_tab_t(double u, int k) {
  const long long b = __double_as_longlong(u);
  const double m = __longlong_as_double((b & 0x0001FFFFFFFFFFFFLL) | 0x3FF0000000000000LL);
  double t = 16.0 * m - 17.0;
  t = k == kGenMergeKey ? (u - 7.75) * (4.0 / 3.0) : t;
  t = k == kGenMergeKey + 1 ? 4.0 * u - 35.0 : t;
  return t;
}

// Table evaluation on a known interval k (= gen_tab_index(P, u)).
template <bool kDerivs>
__device__ __forceinline__ MaternVals matern_table_at(const ThetaParams& P,
                                                      const double* __restrict__ tab, double u,
                                                      int k) {
  const double t = gen_tab_t(u, k);
  // below 8.5 the series are of E itself (no e^u scaling error); above, of e^u E
  const double eu = u < MLE_SMALL_MID_SPLIT ? 1.0 : exp(-u);
  const double* c = tab + (size_t)k * 3 * MLE_TAB_P;
  MaternVals out;
  out.c = eu * horner_pairs(c, t);
  if (kDerivs) {
    out.dalpha = eu * horner_pairs(c + MLE_TAB_P, t);
    out.dnu = eu * horner_pairs(c + 2 * MLE_TAB_P, t);
  } else {
    out.dalpha = 0.0;
    out.dnu = 0.0;
  }
  return out;
}

template <bool kDerivs>
__device__ __forceinline__ MaternVals matern_table(const ThetaParams& P,
                                                   const double* __restrict__ tab, double u) {
  return matern_table_at<kDerivs>(P, tab, u, gen_tab_index(P, u));
}

}  // namespace mle
