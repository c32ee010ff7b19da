// bessel_k.cuh — device x^ν K_ν(x) for the general-ν Matérn of Eq. (7)
// (ν is estimated by the paper's MLE, so the
// general path is on the hot path of the c2 fit).
//
// Method (Temme 1975; Steed's continued fraction), ν ≥ 0:
//   write ν = μ + n with n = ⌊ν + ½⌋, |μ| ≤ ½;
//   x ≤ 2: Temme's series for K_μ(x), K_{μ+1}(x);
//   x > 2: Steed's continued fraction CF2 for K_μ, K_{μ+1};
//   then the stable forward recurrence K_{μ+i+1} = 2(μ+i)/x K_{μ+i} + K_{μ+i−1}.
// Every constant that depends on ν alone (μ, n, Γ-function combinations) is
// computed on the host once per evaluation (bv_host.cpp: fill_general_nu)
// and read from Theta::gen:
//   gen[0] = μ, gen[1] = n, gen[2] = γ1(μ) = (1/Γ(1−μ) − 1/Γ(1+μ))/(2μ),
//   gen[3] = γ2(μ) = (1/Γ(1−μ) + 1/Γ(1+μ))/2, gen[4] = 1/Γ(1+μ),
//   gen[5] = 1/Γ(1−μ), gen[6] = πμ / sin(πμ).
#pragma once
#include "bv_common.cuh"

namespace bv {

__device__ __forceinline__ double xnu_bessel_k(double x, const Theta& th) {
  const double mu = th.gen[0];
  const int nl = (int)th.gen[1];
  const double mu2 = mu * mu;
  const double xi = 1.0 / x, xi2 = 2.0 * xi;
  double rkmu, rk1;
  if (x <= 2.0) {
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
    for (int i = 1; i < 200; ++i) {
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
    rkmu = sum;
    rk1 = sum1 * xi2;
  } else {
    // Steed's algorithm for CF2 with Temme's normalisation.
    double b = 2.0 * (1.0 + x);
    double d = 1.0 / b;
    double h = d, delh = d;
    double q1 = 0.0, q2 = 1.0;
    const double a1 = 0.25 - mu2;
    double q = a1, c = a1;
    double a = -a1;
    double s = 1.0 + q * delh;
    for (int i = 2; i < 400; ++i) {
      a -= 2.0 * (double)(i - 1);
      c = -a * c / (double)i;
      const double qnew = (q1 - b * q2) / a;
      q1 = q2;
      q2 = qnew;
      q += c * qnew;
      b += 2.0;
      d = 1.0 / (b + a * d);
      delh = (b * d - 1.0) * delh;
      h += delh;
      const double dels = q * delh;
      s += dels;
      if (fabs(dels) < fabs(s) * 1.0e-17) break;
    }
    h = a1 * h;
    // K_μ(x) = sqrt(π/(2x)) e^{−x} / s
    rkmu = sqrt(1.5707963267948966 * xi) * exp(-x) / s;
    rk1 = rkmu * (mu + x + 0.5 - h) * xi;
  }
  for (int i = 1; i <= nl; ++i) {
    const double t = (mu + (double)i) * xi2 * rk1 + rkmu;
    rkmu = rk1;
    rk1 = t;
  }
  if (rkmu == 0.0) return 0.0;
  return pow(x, th.nu) * rkmu;
}

}  // namespace bv
