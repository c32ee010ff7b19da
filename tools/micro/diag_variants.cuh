// Candidate diagonal-tile factorisations for tools/micro/diag_bench.cu.
#pragma once
namespace bv {
// rsqrt with a single third-order refinement of the MUFU.RSQ64H seed.
__device__ __forceinline__ double rsqrt_pos1(double x) {
  double y;
  asm("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(x));
  const double e = fma(-x, y * y, 1.0);
  return fma(fma(0.375, e, 0.5), y * e, y);
}

// Full in-lane 8x8, minimal chain; log deferred (returns prod and nbad, qd).
template <bool ONE_STEP>
__device__ __forceinline__ void diag_inlane_fast(const double* tile, double* diagL, double* rinv, int J, int m, int N,
                                                 int lane, double& prod, int& nbad, double& qd) {
  const int nreal = N - 8 * J, jm = m - 8 * J, yr = N - 8 * J;
  double a[8][8];
#pragma unroll
  for (int i = 0; i < 8; ++i)
#pragma unroll
    for (int k = 0; k <= i; ++k) a[i][k] = tile[8 * i + k];
  double rv[8];
#pragma unroll
  for (int j = 0; j < 8; ++j) {
    double p = a[j][j];
    const bool ok = (p > 0.0) & (p <= 1.7976931348623157e308);
    const bool real = j < nreal;
    nbad += (real & !ok) ? 1 : 0;
    p = (real & ok) ? p : 1.0;
    prod *= (j >= jm) ? p : 1.0;
    const double r = ONE_STEP ? rsqrt_pos1(p) : rsqrt_pos(p);
    rv[j] = real ? r : 0.0;
#pragma unroll
    for (int i = j + 1; i < 8; ++i) a[i][j] *= rv[j];
#pragma unroll
    for (int i = j + 1; i < 8; ++i)
#pragma unroll
      for (int k = j + 1; k <= i; ++k) a[i][k] = fma(-a[i][j], a[k][j], a[i][k]);
  }
#pragma unroll
  for (int i = 1; i < 8; ++i)
    if (i == yr) {
#pragma unroll
      for (int k = 0; k < i; ++k)
        if (k >= jm) qd = fma(a[i][k], a[i][k], qd);
    }
  if (lane == 0) {
#pragma unroll
    for (int i = 1; i < 8; ++i)
#pragma unroll
      for (int k = 0; k < i; ++k) diagL[8 * i + k] = a[i][k];
#pragma unroll
    for (int k = 0; k < 8; ++k) rinv[k] = rv[k];
  }
}
}  // namespace bv
