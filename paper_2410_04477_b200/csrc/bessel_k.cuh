// bessel_k.cuh — device x^ν K_ν(x) for the general-ν Matérn of Eq. (7)
// (ν is estimated by the paper's MLE, so the
// general path is on the hot path of the c2 fit).
//
// Method, ν > 0:
//   x ≤ 2: write ν = μ + n with n = ⌊ν + ½⌋, |μ| ≤ ½; Temme's series (Temme
//     1975) for K_μ(x), K_{μ+1}(x), then the stable forward recurrence
//     K_{μ+i+1} = 2(μ+i)/x K_{μ+i} + K_{μ+i−1};
//   2 < x ≤ 22: K_ν(x) = e^{−x} ∫_0^∞ e^{−x(cosh t − 1)} cosh(νt) dt by the
//     trapezoidal rule, h = 0.15, 28 nodes (exponentially convergent for this
//     entire integrand; ≤ 7e-16 relative vs mpmath over x ∈ [2, 22],
//     ν ∈ [0.2, 3] — matern.cuh: xnu_bessel_k);
//   x > 22: the asymptotic series √(π/2x) e^{−x} Σ_j a_j x^{−j}, 20 terms
//     (≤ 5e-16 relative there).
// (Steed's CF2, used for x > 2 before, needs 40-90 iterations with three
// divisions each for x ∈ (2, 6), where most Matérn entries fall.)
// The trapezoid nodes cosh(t_k) − 1, cosh(ν t_k) and the series coefficients
// a_j depend on ν alone: computed on the host in long double once per
// evaluation (bv_host.cpp fill_nu_table), read through Theta::nutab.
// Every constant that depends on ν alone (μ, n, Γ-function combinations) is
// computed on the host once per evaluation (bv_host.cpp: fill_general_nu)
// and read from Theta::gen:
//   gen[0] = μ, gen[1] = n, gen[2] = γ1(μ) = (1/Γ(1−μ) − 1/Γ(1+μ))/(2μ),
//   gen[3] = γ2(μ) = (1/Γ(1−μ) + 1/Γ(1+μ))/2, gen[4] = 1/Γ(1+μ),
//   gen[5] = 1/Γ(1−μ), gen[6] = πμ / sin(πμ).
#pragma once
#include "bv_common.cuh"

namespace bv {

// x ≤ 2: x^ν K_ν(x) by Temme's series + forward recurrence
__device__ __forceinline__ double xnu_bessel_k_small(double x, const Theta& th) {
  const double mu = th.gen[0];
  const int nl = (int)th.gen[1];
  const double mu2 = mu * mu;
  const double xi = 1.0 / x, xi2 = 2.0 * xi;
  // Temme's series (K_μ and K_{μ+1}); terms decay like (x²/4)^i / (i!)².
  const double x2 = 0.5 * x;
  const double dlog = -log(x2);
  double e = mu * dlog;
  const double fact2 = (fabs(e) < 1e-16) ? 1.0 : sinh(e) / e;
  double ff = th.gen[6] * (th.gen[2] * cosh(e) + th.gen[3] * fact2 * dlog);
  double sum = ff;
  e = exp(e);
  double p = 0.5 * e / th.gen[4];
  double q = 0.5 / (e * th.gen[5]);
  double c = 1.0;
  const double dd = x2 * x2;
  double sum1 = p;
  for (int i = 1; i < 60; ++i) {
    const double di = (double)i;
    ff = (di * ff + p + q) / (di * di - mu2);
    c *= dd / di;
    p /= (di - mu);
    q /= (di + mu);
    const double del = c * ff;
    sum += del;
    sum1 += c * (p - di * ff);
    if (fabs(del) < fabs(sum) * 1.0e-17) break;
  }
  double rkmu = sum;
  double rk1 = sum1 * xi2;
  for (int i = 1; i <= nl; ++i) {
    const double t = (mu + (double)i) * xi2 * rk1 + rkmu;
    rkmu = rk1;
    rk1 = t;
  }
  return pow(x, th.nu) * rkmu;
}

}  // namespace bv
