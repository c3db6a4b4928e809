// prologue.cpp — host-side per-theta scalars for the generation kernel.
//
// The per-pair series of the reference (bessel.py / matern.py) mix x-dependent and
// nu-only factors.  The nu-only factors are evaluated here once per theta, in the same
// double-precision order the reference uses for its scalar arithmetic (so that they
// agree with it bit for bit where the reference itself works in doubles), while the
// special functions the reference takes from scipy (Gamma, digamma) are evaluated in
// 80-bit long double and rounded once.
#include <cmath>
#include <cstdlib>
#include <cstring>

#include "theta.h"

namespace {

const long double kPiL = 3.141592653589793238462643383279502884L;

// Taylor coefficients of 1/Gamma(1+x) about 0 (c_0 = 1, c_1 = Euler's gamma, ...),
// derived with mpmath at 40 digits; 31 terms reach < 1e-22 at |x| = 1/2.
const long double kRecipGammaTaylor[31] = {
    1.0L,
    0.577215664901532860606512090082L,
    -0.655878071520253881077019515145L,
    -0.0420026350340952355290039348754L,
    0.166538611382291489501700795102L,
    -0.0421977345555443367482083012892L,
    -0.00962197152787697356211492167235L,
    0.00721894324666309954239501034045L,
    -0.00116516759185906511211397108402L,
    -0.000215241674114950972815729963054L,
    0.000128050282388116186153198626328L,
    -0.000020134854780788238655689391421L,
    -0.00000125049348214267065734535947383L,
    0.00000113302723198169588237412962033L,
    -0.000000205633841697760710345015413002L,
    0.00000000611609510448141581786249868286L,
    0.00000000500200764446922293005566504806L,
    -0.00000000118127457048702014458812656544L,
    1.04342671169110051049154033231e-10L,
    7.78226343990507125404993731136e-12L,
    -3.69680561864220570818781587809e-12L,
    5.10037028745447597901548132286e-13L,
    -2.05832605356650678322242954486e-14L,
    -5.34812253942301798237001731873e-15L,
    1.22677862823826079015889384662e-15L,
    -1.18125930169745876951376458684e-16L,
    1.18669225475160033257977724293e-18L,
    1.41238065531803178155580394757e-18L,
    -2.29874568443537020659247858063e-19L,
    1.71440632192733743338396337027e-20L,
    1.33735173049369311486478139512e-22L,
};

// 1/Gamma(1+x) for |x| <= 1/2 by the Taylor series (Horner, long double).
long double recip_gamma_1p(long double x) {
  long double s = 0.0L;
  for (int k = 30; k >= 0; --k) s = s * x + kRecipGammaTaylor[k];
  return s;
}

// (1/G(1-mu) - 1/G(1+mu)) / (2 mu) = -sum_{k odd} c_k mu^{k-1}: the odd part of the Taylor
// series divided by mu, so it has no cancellation and a finite limit (-Euler gamma) at mu = 0.
long double recip_gamma_odd_over_mu(long double mu) {
  long double s = 0.0L;
  const long double m2 = mu * mu;
  for (int k = 29; k >= 1; k -= 2) s = s * m2 + kRecipGammaTaylor[k];
  return -s;
}

// digamma for x > 0: upward shift to x >= 20, then the Stirling-type asymptotic series.
long double digamma_pos(long double x) {
  long double acc = 0.0L;
  while (x < 20.0L) {
    acc -= 1.0L / x;
    x += 1.0L;
  }
  const long double r = 1.0L / (x * x);
  // sum_k B_{2k} / (2k x^{2k}), k = 1..8
  const long double series =
      r * (1.0L / 12 - r * (1.0L / 120 - r * (1.0L / 252 - r * (1.0L / 240 -
      r * (1.0L / 132 - r * (691.0L / 32760 - r * (1.0L / 12 - r * (3617.0L / 8160))))))));
  return acc + logl(x) - 0.5L / x - series;
}

// digamma(-nu) for nu > 0 non-integer: psi(-nu) = psi(nu) + 1/nu + pi cot(pi nu), with the
// cotangent argument reduced to the fractional part so it stays accurate near integers.
long double digamma_neg(long double nu) {
  const long double fl = floorl(nu);
  const long double frac = nu - fl;  // exact
  const long double cot = cosl(kPiL * frac) / sinl(kPiL * frac);
  return digamma_pos(nu) + 1.0L / nu + kPiL * cot;
}

// pi mu / sin(pi mu), series near 0.
long double pi_mu_over_sin(long double mu) {
  const long double pm = kPiL * mu;
  if (fabsl(pm) < 1e-4L) return 1.0L + pm * pm / 6.0L + 7.0L * pm * pm * pm * pm / 360.0L;
  return pm / sinl(pm);
}

// Build the ladder that ends at order `order` (>= 0).  If `want_low` is set we also need
// K_{order-1}: for order >= 1/2 the pair (K_{order-1}, K_order) is reached from mu =
// order - N; for order < 1/2 we start from mu = -order so that the pair is
// (K_{-order} = K_order, K_{1-order} = K_{order-1}).
//
// Small-argument coefficients.  Temme's expansion of the pair (|mu| <= 1/2):
//   K_mu(x)         = sum_k (d^k / k!) f_k,
//   (x/2) K_{mu+1}  = sum_k (d^k / k!) (p_k - k f_k),          d = x^2 / 4,
//   f_k = (k f_{k-1} + p_{k-1} + q_{k-1}) / (k^2 - mu^2),  p_k = p_{k-1} / (k - mu),
//   q_k = q_{k-1} / (k + mu),
// with seeds f_0, p_0, q_0 that carry all the x dependence (theta.h).  Every step is linear
// with mu-only coefficients, so f_k = a_k f_0 + b_k p_0 + c_k q_0 and p_k = P_k p_0,
// q_k = Q_k q_0, where
//   a_0 = 1, b_0 = c_0 = 0, P_0 = Q_0 = 1,
//   a_k = k a_{k-1} / (k^2 - mu^2),  b_k = (k b_{k-1} + P_{k-1}) / (k^2 - mu^2),
//   c_k = (k c_{k-1} + Q_{k-1}) / (k^2 - mu^2),  P_k = P_{k-1} / (k - mu),  Q_k = Q_{k-1} / (k + mu).
// The d^k coefficients (a_k, b_k, c_k) / k! and (-k a_k, P_k - k b_k, -k c_k) / k! are formed in
// long double and rounded once; a_k, b_k, c_k, P_k, Q_k are all positive for |mu| <= 1/2.
void fill_ladder(double order, KLadder* L) {
  const double N = std::floor(order + 0.5);
  double mu;
  if (N >= 1.0) {
    mu = order - N;  // exact (Sterbenz)
    L->nsteps = (int)N - 1;
    L->order_is_low = 0;
  } else {
    mu = -order;
    L->nsteps = 0;
    L->order_is_low = 1;
  }
  const long double m = mu;
  L->mu = mu;
  const long double rg_plus = recip_gamma_1p(m);    // 1 / G(1 + mu)
  const long double rg_minus = recip_gamma_1p(-m);  // 1 / G(1 - mu)
  const long double pms = pi_mu_over_sin(m);
  L->f0_cosh = (double)(pms * recip_gamma_odd_over_mu(m));
  L->f0_sinh = (double)(pms * 0.5L * (rg_plus + rg_minus));
  L->p0 = (double)(0.5L / rg_plus);
  L->q0 = (double)(0.5L / rg_minus);
  long double a = 1.0L, b = 0.0L, c = 0.0L, pk = 1.0L, qk = 1.0L, fact = 1.0L;
  for (int k = 0; k < MLE_KSER_TERMS; ++k) {
    const long double kl = (long double)k;
    if (k > 0) {
      const long double den = kl * kl - m * m;
      a = kl * a / den;
      b = (kl * b + pk) / den;
      c = (kl * c + qk) / den;
      pk /= kl - m;
      qk /= kl + m;
      fact *= kl;
    }
    L->ser[k][0] = (double)(a / fact);
    L->ser[k][1] = (double)(b / fact);
    L->ser[k][2] = (double)(c / fact);
    L->ser[k][3] = (double)(-kl * a / fact);
    L->ser[k][4] = (double)((pk - kl * b) / fact);
    L->ser[k][5] = (double)(-kl * c / fact);
  }
}

bool near_integer(double v) {  // bessel.py:117-118  (|nu - round(nu)| <= 1e-6)
  return std::fabs(v - std::nearbyint(v)) <= 1e-6;
}
bool near_half_integer(double v) {  // bessel.py:121-122
  return std::fabs((v + 0.5) - std::nearbyint(v + 0.5)) <= 1e-6;
}

}  // namespace

int mle_fill_theta(const double theta[3], double nugget, ThetaParams* P) {
  const double s2 = theta[0], al = theta[1], nu = theta[2];
  if (!(std::isfinite(s2) && s2 > 0.0 && std::isfinite(al) && al > 0.0 && std::isfinite(nu) &&
        nu > 0.0))
    return 2;
  if (!(std::isfinite(nugget) && nugget >= 0.0)) return 2;
  std::memset(P, 0, sizeof(*P));
  P->sigma2 = s2;
  P->alpha = al;
  P->nu = nu;
  P->nugget = nugget;

  const double gam = (double)tgammal((long double)nu);          // scipy gamma(nu)
  const double psi = (double)digamma_pos((long double)nu);      // scipy digamma(nu)
  const double two_1mnu = std::pow(2.0, 1.0 - nu);               // 2.0 ** (1.0 - nu)
  P->scale_c = s2 * two_1mnu / gam;                              // matern.py:102
  P->scale_a = two_1mnu / gam * s2 / al;                         // matern.py:109
  P->q = two_1mnu / gam;                                         // matern.py:121
  P->dlog_q = -std::log(2.0) - psi;                              // matern.py:123

  fill_ladder(nu, &P->kmain);
  P->nu_fd = nu + MLE_FD_LAG;                                    // bessel.py:322
  fill_ladder(P->nu_fd, &P->kfd);
  P->recip_int[0] = 0.0;
  for (int i = 1; i <= MLE_RECIP_INT_MAX; ++i) P->recip_int[i] = 1.0 / (double)i;
  P->fd_small = near_integer(nu) ? 1 : 0;                        // bessel.py:361-363
  P->fd_large = near_half_integer(nu) ? 1 : 0;                   // bessel.py:364-366
  P->two_nu = 2.0 * nu;

  // ---- case 2 constants, in the reference's order (bessel.py:201-222) ----
  {
    const double gam_pos = gam;
    const double gam_neg = -M_PI / (std::sin(M_PI * nu) * nu * gam_pos);  // bessel.py:202
    const double psi_pos = psi;
    const double psi_neg = P->fd_small ? 0.0 : (double)digamma_neg((long double)nu);
    const double two_pow_nu = std::pow(2.0, nu);
    const double log2 = std::log(2.0);
    double g_pos = 1.0, g_neg = 1.0, d_pos = 0.0, d_neg = 0.0;
    for (int k = 0; k <= MLE_CASE2_TERMS; ++k) {
      if (k > 0) {
        g_pos /= nu + k;
        g_neg /= -nu + k;
        d_pos -= 1.0 / (nu + k);
        d_neg -= 1.0 / (-nu + k);
      }
      P->c2_term_pos[k] = two_pow_nu * (log2 + psi_pos - d_neg) * gam_pos * g_neg;
      P->c2_d_pos[k] = d_pos;
      P->c2_g_pos[k] = g_pos;
    }
    P->c2_two_m_nu = std::pow(2.0, -nu);
    P->c2_psi_neg = psi_neg;
    P->c2_gam_neg = gam_neg;
  }
  // ---- case 3 weights (bessel.py:258-276) ----
  {
    double sign = 1.0, nu_pow = 1.0;
    for (int k = 0; k <= MLE_CASE3_NEAR; ++k) {
      P->c3_w[k] = sign * nu_pow;
      P->c3_wk[k] = sign * (k * nu_pow / nu);
      sign = -sign;
      nu_pow /= nu;
    }
    P->c3_log_nu = std::log(nu);
    P->c3_sqrt_pi_2nu = std::sqrt(M_PI / (2.0 * nu));
    P->c3_nu3 = std::pow(nu, 3.0);
  }
  // ---- case 4 coefficients (bessel.py:303-316) ----
  {
    double a_k = 1.0, b_k = 0.0;
    const double four_nu2 = 4.0 * nu * nu;
    P->c4_a[0] = 1.0;
    P->c4_b[0] = 0.0;
    P->c4_kmax = MLE_CASE4_TERMS;
    for (int k = 1; k <= MLE_CASE4_TERMS; ++k) {
      const double factor = four_nu2 - (double)((2 * k - 1) * (2 * k - 1));
      a_k *= factor / (8.0 * k);
      if (a_k == 0.0) {
        P->c4_kmax = k - 1;
        break;
      }
      b_k += 8.0 * nu / factor;
      P->c4_a[k] = a_k;
      P->c4_b[k] = b_k;
    }
    P->nu_m_half = nu - 0.5;
  }
  return 0;
}

void mle_fill_ladder(double order, KLadder* L) { fill_ladder(order, L); }

// Debye polynomials U_0..U_12 by the coefficient recursion of bessel.py:144-170 and
// their derivatives (bessel.py:173-176).
void mle_fill_u_tables(double* u, double* du) {
  std::memset(u, 0, sizeof(double) * (MLE_CASE3_NEAR + 1) * MLE_U_COEFF_STRIDE);
  std::memset(du, 0, sizeof(double) * (MLE_CASE3_NEAR + 1) * MLE_U_COEFF_STRIDE);
  u[0] = 1.0;
  for (int k = 0; k < MLE_CASE3_NEAR; ++k) {
    const double* prev = u + k * MLE_U_COEFF_STRIDE;
    double* nxt = u + (k + 1) * MLE_U_COEFF_STRIDE;
    const int prev_size = 3 * k + 1;
    for (int j = 1; j <= 3 * (k + 1); ++j) {
      double cj = 0.0;
      if (j - 1 >= 0 && j - 1 < prev_size) cj += 0.5 * (j - 1 + 1.0 / (4.0 * j)) * prev[j - 1];
      if (j - 3 >= 0 && j - 3 < prev_size) cj -= 0.5 * (j - 3 + 5.0 / (4.0 * j)) * prev[j - 3];
      nxt[j] = cj;
    }
  }
  for (int k = 0; k <= MLE_CASE3_NEAR; ++k) {
    const double* c = u + k * MLE_U_COEFF_STRIDE;
    double* d = du + k * MLE_U_COEFF_STRIDE;
    const int size = 3 * k + 1;
    for (int j = 1; j < size; ++j) d[j - 1] = c[j] * (double)j;
  }
}

void mle_fill_gen_table(double u_max, ThetaParams* P) {
  P->tab_n = 0;
  const double lo = MLE_TAB_LO;
  const double hi = std::fmin(u_max * (1.0 + 1e-9), MLE_TAB_HI);
  P->tab_lo = lo;
  P->tab_hi = hi;
  long long bits_lo;
  std::memcpy(&bits_lo, &lo, sizeof(lo));
  P->tab_key0 = bits_lo >> 49;
  if (!(hi > lo)) return;
  // Interval bins: each binade [2^e, 2^(e+1)) of u in 8 equal pieces (ratio <= 1.125; the
  // Chebyshev convergence factor of the degree-13 pieces is then > 30 per degree), so the
  // device finds the bin with one shift of the bits of u and no transcendental.  Around the
  // reference's regime switch 8.5 (bessel.py:46) the pieces are [7, 8.5) (the bins [7, 7.5),
  // [7.5, 8) and the lower half of [8, 9)) and [8.5, 9); 30 = 16 * 15/8 is a bin edge (bessel.py:47),
  // so no piece straddles a switch (gen_tab_index / gen_tab_t in special.cuh).
  constexpr int kMerge = (2 - MLE_TAB_LO_EXP) * 8 + 6;  // = kGenMergeKey (special.cuh)
  int k = 0;
  for (int key = 0; k < MLE_TAB_MAX; ++key) {
    const int e = MLE_TAB_LO_EXP + key / 8, j = key % 8;
    double a = std::ldexp(1.0 + j / 8.0, e), b = std::ldexp(1.0 + (j + 1) / 8.0, e);
    if (!(a < hi)) break;
    if (key == kMerge + 1) continue;
    if (key == kMerge) b = MLE_SMALL_MID_SPLIT;
    if (key == kMerge + 2) a = MLE_SMALL_MID_SPLIT;
    P->tab_ctr[k] = 0.5 * (a + b);
    P->tab_hw[k] = 0.5 * (b - a);
    ++k;
  }
  if (k >= MLE_TAB_MAX && P->tab_ctr[k - 1] + P->tab_hw[k - 1] < hi)
    P->tab_hi = P->tab_ctr[k - 1] + P->tab_hw[k - 1];  // (MLE_TAB_HI keeps this unreachable)
  P->tab_n = k;
}

// M = (monomial coefficients of T_j) x (discrete Chebyshev transform at the nodes
// t_q = cos(pi (q + 1/2) / P)): a_i = sum_q M[i][q] f(t_q).  Transform: c_j = (2 / P) sum_q
// f_q cos(pi j (q + 1/2) / P), halved for j = 0; T_j from T_j = 2 t T_{j-1} - T_{j-2} (integer
// coefficients, exact).  Built in long double and split into a double-double pair.
void mle_fill_tab_map(double* hi, double* lo) {
  constexpr int P = MLE_TAB_P;
  long double mono[P][P] = {};  // mono[j][i] = [t^i] T_j(t)
  mono[0][0] = 1.0L;
  mono[1][1] = 1.0L;
  for (int j = 2; j < P; ++j)
    for (int i = 0; i < P; ++i)
      mono[j][i] = (i > 0 ? 2.0L * mono[j - 1][i - 1] : 0.0L) - mono[j - 2][i];
  for (int i = 0; i < P; ++i) {
    for (int q = 0; q < P; ++q) {
      long double m = 0.0L;
      for (int j = i; j < P; ++j) {
        long double w = (2.0L / P) * cosl(kPiL * j * (q + 0.5L) / P);
        if (j == 0) w *= 0.5L;
        m += mono[j][i] * w;
      }
      const double h = (double)m;
      hi[i * P + q] = h;
      lo[i * P + q] = (double)(m - (long double)h);
    }
  }
}

// psi(x) for any x off the poles: the upward-shift asymptotic series for x > 0, reflection
// psi(1 - x) - psi(x) = pi cot(pi x) below (the cotangent on the reduced argument).
double mle_digamma_host(double x) {
  if (std::isnan(x)) return x;
  if (x > 0.0) return (double)digamma_pos((long double)x);
  const long double xl = x;
  const long double fl = floorl(xl);
  const long double frac = xl - fl;  // in (0, 1): x is not a pole here
  const long double cot = cosl(kPiL * frac) / sinl(kPiL * frac);
  return (double)(digamma_pos(1.0L - xl) - kPiL * cot);
}
