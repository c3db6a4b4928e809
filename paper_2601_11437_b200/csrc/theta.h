// theta.h — per-theta scalar prologue shared by the host (prologue.cpp) and the device
// kernels.  Everything that depends on nu alone is hoisted here once per evaluation so the
// per-pair work in the generation kernel is only the x-dependent part of each series.
//
// Sources of every quantity (reference tree, path:line):
//   scale_c, scale_a, q, dlog_q       pkg/src/maternmle/matern.py:100-125
//   case-2 constants (g_k, d_k, ...)   pkg/src/maternmle/bessel.py:184-223
//   case-3 weights (sign * nu^-k ...)  pkg/src/maternmle/bessel.py:226-283
//   case-4 a_k, b_k                    pkg/src/maternmle/bessel.py:286-318
//   FD band and lag                    pkg/src/maternmle/bessel.py:117-141, 321-324
// The K_nu ladder parameters (Temme expansion / trapezoidal integral) replace scipy.special.kv.
#pragma once

#define MLE_CASE2_TERMS 20       // bessel.py:52  (k = 0..20)
#define MLE_CASE3_NEAR 12        // bessel.py:53
#define MLE_CASE3_FAR 8          // bessel.py:54
#define MLE_CASE4_TERMS 5        // bessel.py:55
#define MLE_U_COEFF_STRIDE 40    // >= 3*12+1 coefficients per Debye polynomial
#define MLE_TAB_P 14              // interpolation points per interval (degree 13, even)
#define MLE_TAB_MAX 96            // intervals per table (8 per binade of u in [0.25, 1024))
#define MLE_TAB_DOUBLES (MLE_TAB_MAX * 3 * MLE_TAB_P)  // [interval][c, da, dn][power]
#define MLE_TAB_LO_EXP (-2)       // tables from u = 2^-2 up; below, the exact evaluator: near
                                  // u = 0, C ~ sigma^2 and the ill-conditioned goldens need its
                                  // few-ulp accuracy (tables from 2^-16 moved one by 1.6e-10)
#define MLE_TAB_LO 0.25           // 2^MLE_TAB_LO_EXP
#define MLE_TAB_HI 640.0          // above: exact evaluation (elements ~1e-280 sigma^2 or zero).  A
                                  // bin edge well below 709.78: the tables hold e^u E(u), and
                                  // exp(u) overflows there (at 800 the bins from 704 up were
                                  // inf x 0 = NaN: a very short range, u > 709 for some pair,
                                  // made Sigma NaN -- found by a theta probe, pinned by
                                  // tests/test_gpu_likelihood.py::test_very_short_range)
#define MLE_SMALL_MID_SPLIT 8.5  // bessel.py:46
#define MLE_MID_LARGE_SPLIT 30.0 // bessel.py:47
#define MLE_MID_TRUNC_SPLIT 15.0 // bessel.py:48
#define MLE_FD_LAG 1e-9          // bessel.py:50

#define MLE_KSER_XMAX 1.0  // x below: small-argument series; at and above: trapezoidal rule
#define MLE_KSER_TERMS 14  // power-series terms in d = x^2/4 <= 1/4 (d^13 / 13!^2 < 1e-27)
#define MLE_KTRAP_MAX 64   // trapezoid nodes cap (x >= 1 needs <= ~30)
#define MLE_RECIP_INT_MAX 40

// Parameters of one K-ladder: K_mu and K_{mu+1} for |mu| <= 1/2 (special.cuh,
// bessel_k_pair), then `nsteps` upward recurrences.
//
// Small-argument data (x < MLE_KSER_XMAX).  Temme's expansion writes K_mu and K_{mu+1}
// through three sequences f_k, p_k, q_k that obey mu-only linear recurrences from seeds
// f0(x), p0(x), q0(x); unrolled, each of K_mu, (x/2) K_{mu+1} is f0, p0, q0 times a power
// series in d = x^2/4 whose coefficients depend on mu alone (prologue.cpp, fill_ladder):
//   ser[k][0..2]: d^k coefficient multiplying f0, p0, q0 in K_mu,
//   ser[k][3..5]: the same for (x/2) K_{mu+1}.
// Seeds: f0 = f0_cosh cosh(s) + f0_sinh ln(2/x) sinh(s)/s with s = mu ln(2/x);
//        p0 = p0c (x/2)^-mu,  q0 = q0c (x/2)^mu.
struct KLadder {
  double mu;
  int nsteps;            // upward recurrence steps applied to (K_mu, K_{mu+1})
  int order_is_low;      // 1: K_nu is the lower member of the final pair (nu < 1/2 case)
  double f0_cosh;        // (pi mu / sin pi mu) * (1/G(1-mu) - 1/G(1+mu)) / (2 mu)
  double f0_sinh;        // (pi mu / sin pi mu) * (1/G(1-mu) + 1/G(1+mu)) / 2
  double p0, q0;         // G(1+mu) / 2, G(1-mu) / 2
  double ser[MLE_KSER_TERMS][6];
};

struct ThetaParams {
  double sigma2, alpha, nu, nugget;
  double scale_c;   // sigma2 * 2^(1-nu) / Gamma(nu)               matern.py:102
  double scale_a;   // 2^(1-nu)/Gamma(nu) * sigma2 / alpha          matern.py:109
  double q;         // 2^(1-nu) / Gamma(nu)                         matern.py:121
  double dlog_q;    // -log 2 - psi(nu)                             matern.py:123
  double nu_fd;     // fl(nu + 1e-9)                                bessel.py:322
  int fd_small;     // nu within 1e-6 of an integer: x in (0, 8.5) uses the FD fallback
  int fd_large;     // nu within 1e-6 of a half-integer: x >= 30 uses the FD fallback
  KLadder kmain;    // ladder for K_nu and K_{nu-1}
  KLadder kfd;      // ladder for K_{nu_fd} (only used in FD bands)
  double recip_int[MLE_RECIP_INT_MAX + 1];  // 1 / i (case-2 prefactor recursion)
  // ---- case 2 (0 < x < 8.5) ----
  double c2_term_pos[MLE_CASE2_TERMS + 1];  // 2^nu (log2 + psi(nu) - d_k(-nu)) G(nu) g_k(-nu)
  double c2_d_pos[MLE_CASE2_TERMS + 1];     // d_k(nu)
  double c2_g_pos[MLE_CASE2_TERMS + 1];     // g_k(nu)
  double c2_two_m_nu;                       // 2^-nu
  double c2_psi_neg;                        // psi(-nu)
  double c2_gam_neg;                        // Gamma(-nu) by reflection
  double two_nu;                            // 2 nu
  // ---- case 3 (8.5 <= x < 30) ----
  double c3_w[MLE_CASE3_NEAR + 1];          // sign * nu^-k
  double c3_wk[MLE_CASE3_NEAR + 1];         // sign * (k nu^-k / nu)
  double c3_log_nu;                         // log(nu)
  double c3_sqrt_pi_2nu;                    // sqrt(pi / (2 nu))
  double c3_nu3;                            // nu^3
  // ---- case 4 (x >= 30) ----
  double c4_a[MLE_CASE4_TERMS + 1];
  double c4_b[MLE_CASE4_TERMS + 1];
  int c4_kmax;                              // last k with a_k != 0
  double nu_m_half;                         // nu - 0.5
  // ---- engine generation tables (filled per pass by the engine, mle_fill_gen_table) ----
  // For u = h / alpha in [tab_lo, tab_hi): e^u * {Sigma, dalpha, dnu element} as Chebyshev
  // series of degree MLE_TAB_P - 1 on log-spaced intervals, in three segments split exactly
  // at the reference's dnu regime boundaries 8.5 and 30 (bessel.py:46-47).
  // Intervals are the binades of u cut into 8 equal bins (ratio <= 1.125), found from the
  // bits of u by one shift (bin = (bits(u) >> 49) - tab_key0); the bin [8, 9) is split at 8.5.
  int tab_n;                                // intervals (0: exact evaluation everywhere)
  long long tab_key0;                       // bits(MLE_TAB_LO) >> 49
  double tab_lo, tab_hi;
  double tab_ctr[MLE_TAB_MAX], tab_hw[MLE_TAB_MAX];  // interval centre, half-width
};

#ifdef __cplusplus
extern "C++" {
// Host prologue: fills P from theta (+ nugget).  Returns 0, or 2 for invalid theta
// (non-finite or <= 0 components: MaternParams.__post_init__, matern.py:44-48).
int mle_fill_theta(const double theta[3], double nugget, ThetaParams* P);
// Ladder for a single order >= 0 (bessel_k of any non-negative order, including 0).
void mle_fill_ladder(double order, KLadder* L);
// Debye U_k coefficient tables (bessel.py:144-176), flattened [k][j] with stride
// MLE_U_COEFF_STRIDE, for U and U'.  Filled once.
void mle_fill_u_tables(double* u, double* du);
// Interval layout of the generation tables for scaled distances up to u_max (tab_n = 0
// when u_max < MLE_TAB_LO).
void mle_fill_gen_table(double u_max, ThetaParams* P);
// The linear map from the MLE_TAB_P Chebyshev-node values of an interval to the monomial
// coefficients (powers of t in [-1, 1]) of their interpolant, as double-double pairs
// hi[i * MLE_TAB_P + q] + lo[...] (long-double construction).  The table kernel applies it in
// double-double arithmetic so the coefficients carry one rounding each.
void mle_fill_tab_map(double* hi, double* lo);
// digamma of a double off the poles (host; the prologue's psi(nu) uses the same series).
double mle_digamma_host(double x);
}
#endif
