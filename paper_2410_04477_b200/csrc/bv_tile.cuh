// bv_tile.cuh — 8×8 FP64 tile primitives of the joint Cholesky (Alg. 1 l.16-27,
// PAPER.md:602-629, fused as in DESIGN.md §4), shared by the block kernels.
//
// Tiles are kept in the FP64 MMA accumulator layout (lane (g,t) = (lane/4, lane%4)
// holds row g, columns 2t and 2t+1), which in memory is simply row-major.  The
// same layout serves as the A and B operands of mma.m8n8k4 when the k index is
// permuted (step one sums k = 2t, step two k = 2t+1), so no tile is ever
// transposed.  Tiles of the matrix being factored are stored NEGATED (Ĉ = −C),
// which makes every Schur update a plain D = A·B + D.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include "bv_common.cuh"
#include "matern.cuh"

namespace bv {
namespace tile {

constexpr int kPre = 4;  // KIND: Σ entries read from the pre-generation buffer

__device__ __forceinline__ void dmma(double& d0, double& d1, double a, double b) {
  asm("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
      : "+d"(d0), "+d"(d1)
      : "d"(a), "d"(b));
}
__device__ __forceinline__ double2 lds2(const double* p) { return *reinterpret_cast<const double2*>(p); }
__device__ __forceinline__ void sts2(double* p, double a, double b) {
  *reinterpret_cast<double2*>(p) = make_double2(a, b);
}
__device__ __forceinline__ double neg(double x) {
  return __longlong_as_double(__double_as_longlong(x) ^ (long long)0x8000000000000000ULL);
}

// Joint-matrix entry (r, c), r ≥ c: Eq. (7) between the gathered points, the y row
// (r == N) holds the column point's observation.  Padding points are far apart, so
// every padding entry off the diagonal is exactly 0 and the padding diagonal is σ².
template <int KIND>
__device__ __forceinline__ double entry(const PointRec& pr, const PointRec& pc, int r, int c, int N,
                                        const Theta& th, const double* etab, const double* pre) {
  double v;
  if constexpr (KIND == kPre) {
    const int rr = r > c ? r : c, cc = r > c ? c : r;
    v = rr < N ? pre[(rr * (rr + 1) >> 1) + cc] : (rr == cc ? th.sigma2 : 0.0);
  } else {
    v = matern_kind<KIND>(sqdist(pr, pc), th, etab);
  }
  return (r == N) ? pc.v : v;
}

// Ĉ tile (I,K) in the accumulator layout (negated).
template <int KIND>
__device__ __forceinline__ double2 gen_tile(const PointRec* P, int I, int K, int g, int t, int N, const Theta& th,
                                            const double* etab, const double* pre) {
  const int r = 8 * I + g, c = 8 * K + 2 * t;
  const PointRec pr = P[r], p0 = P[c], p1 = P[c + 1];
  const double v0 = entry<KIND>(pr, p0, r, c, N, th, etab, pre);
  const double v1 = entry<KIND>(pr, p1, r, c + 1, N, th, etab, pre);
  return make_double2(neg(v0), neg(v1));
}

// L(I,J) = C(I,J) L_JJ⁻ᵀ from Ĉ = −C, in registers: X₁ = Ĉ Zₙᵀ (Zₙ = −L_JJ⁻¹),
// R̂ = Ĉ + X₁ L_JJᵀ (= −residual), X = X₁ + R̂ Zₙᵀ — one FP64 refinement step,
// which restores the accuracy of substitution that a bare product with an
// explicit inverse loses on ill-conditioned L_JJ.  zn, lj: this lane's
// (row g, columns 2t, 2t+1) of Zₙ and L_JJ — the B fragments of the k-permuted
// products.  c is consumed.
__device__ __forceinline__ double2 trsm(double2 c, double2 zn, double2 lj) {
  double x0 = 0.0, x1 = 0.0;
  dmma(x0, x1, c.x, zn.x);
  dmma(x0, x1, c.y, zn.y);
  dmma(c.x, c.y, x0, lj.x);
  dmma(c.x, c.y, x1, lj.y);
  dmma(x0, x1, c.x, zn.x);
  dmma(x0, x1, c.y, zn.y);
  return make_double2(x0, x1);
}

// y-row term of one solved tile: u += Σ_{j ≥ m, j < N} L_Nj² over this lane's two columns
__device__ __forceinline__ double yrow_sq(double2 x, int J, int t, int m, int N) {
  const int k0 = 8 * J + 2 * t, k1 = k0 + 1;
  double q = (k0 >= m && k0 < N) ? x.x * x.x : 0.0;
  return (k1 >= m && k1 < N) ? fma(x.y, x.y, q) : q;
}

// In-lane Cholesky of the diagonal tile (row-major at dg, negated storage when
// NEGIN; every lane holds all of it), then L_JJ⁻¹ by columns (lane j&7 solves
// L x = e_j).  Lane 0 publishes L_JJ row-major (lb), lanes 0..7 column j of
// −L_JJ⁻¹ (zb).  The pivot chain carries no selects: padding rows are far
// points (pivot σ², zero coupling) and the y row's "pivot" (it is eliminated,
// never pivoted) only poisons rows below it in the LAST tile, which nothing
// reads.  Pivot checks (reading G15: a real pivot must exceed pfloor) and the d
// product over real rows j ≥ m run on the recorded pivots, off the chain.  The
// y row's in-tile entries give u's last terms (qd).  jit (optional jitter mode,
// reading G15b) is added to the diagonal (harmless on padding and the y row).
template <bool NEGIN>
__device__ __forceinline__ void factor_tile(const double* dg, double* lb, double* zb, int J, int m, int N, int lane,
                                            double pfloor, double jit, double& prod, int& nbad, double& qd) {
  const int nreal = N - 8 * J, jm = m - 8 * J, yr = N - 8 * J;
  double a[8][8], rr[8];
#pragma unroll
  for (int i = 0; i < 8; ++i)
#pragma unroll
    for (int k = 0; k <= i; ++k) a[i][k] = NEGIN ? neg(dg[8 * i + k]) : dg[8 * i + k];
#pragma unroll
  for (int i = 0; i < 8; ++i) a[i][i] += jit;
#pragma unroll
  for (int j = 0; j < 8; ++j) {
    const double p = a[j][j];
    const double r = rsqrt_pos(p);
    const double lv = p * r;
    {  // off the chain: pivot check (reading G15) and the d product over real rows ≥ m
      const bool real = j < nreal, ok = (p > pfloor) & (p <= 1.7976931348623157e308);
      nbad += (real & !ok) ? 1 : 0;
      prod *= (real & (j >= jm)) ? p : 1.0;
    }
    a[j][j] = lv;
#pragma unroll
    for (int i = j + 1; i < 8; ++i) {
      const double x = a[i][j] * r;
      a[i][j] = fma(fma(-x, lv, a[i][j]), r, x);
    }
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
  // column j = lane & 7 of L⁻¹: x_i = (δ_ij − Σ_{k<i} L_ik x_k) / L_ii
  const int j = lane & 7;
  double x[8];
#pragma unroll
  for (int i = 0; i < 8; ++i) {
    double s = (i == j) ? 1.0 : 0.0;
#pragma unroll
    for (int k = 0; k < i; ++k) s = fma(-a[i][k], x[k], s);
    x[i] = s * rr[i];
  }
  if (lane < 8) {
#pragma unroll
    for (int i = 0; i < 8; ++i) zb[8 * i + j] = neg(x[i]);
  }
  if (lane == 0) {
#pragma unroll
    for (int i = 0; i < 8; ++i)
#pragma unroll
      for (int k = 0; k < 8; k += 2) sts2(lb + 8 * i + k, k <= i ? a[i][k] : 0.0, k + 1 <= i ? a[i][k + 1] : 0.0);
  }
}

__device__ __forceinline__ double shfl(double v, int src) { return __shfl_sync(0xffffffffu, v, src); }

// Cholesky of one 8×8 tile spread over the warp (c0, c1 = this lane's C[g][2t], C[g][2t+1],
// positive, lower part meaningful) → c0, c1 = L[g][2t], L[g][2t+1] (0 above the diagonal) and
// z0, z1 = −(L⁻¹)[g][2t], −(L⁻¹)[g][2t+1].  Pivot j: the pivot is broadcast from lane
// (j, j/2); every lane forms 1/L_jj by the same rsqrt steps as the other kernels; column j is
// scaled with one residual correction per entry (each L_gj consistent with L_jj to an ulp);
// the trailing entries get C[g][c] −= L_gj L_cj with L_gj, L_cj shuffled from column j's lanes.
// The inverse is the same elimination applied to the identity, one step behind.  Rows j ≥ N − 8J (the y row,
// eliminated but never pivoted, and padding) only occur in the LAST tile, whose L and L⁻¹ no
// solve reads; pivot checks (reading G15) and the d product over real rows j ≥ m run off the
// chain; the y row's in-tile entries give u's last terms (qd, this lane's share).  jit: the
// optional jitter mode's ε·σ² on the diagonal (reading G15b).  UNROLL: the pivot loop
// unrolled (the block kernel's single chain copy: latency) or rolled (the warp kernel, one
// copy per panel: code size).
template <int UNROLL = 8>
__device__ __forceinline__ void factor_dist(double& c0, double& c1, double& z0, double& z1, int lane, int J, int m,
                                            int N, double pfloor, double jit, double& prod, int& nbad, double& qd) {
  const int g = lane >> 2, t = lane & 3, nreal = N - 8 * J, jm = m - 8 * J, yr = N - 8 * J;
  if (g == 2 * t) c0 += jit;
  if (g == 2 * t + 1) c1 += jit;
  // Z = L⁻¹ by the same elimination on the identity, one step behind the factorisation
  // (step j needs column j of L and rows < j of Z): row j scaled by 1/L_jj, then
  // Z[g][·] −= L[g][j] Z[j][·] for g > j — the two dependency chains overlap
  z0 = (g == 2 * t) ? 1.0 : 0.0;
  z1 = (g == 2 * t + 1) ? 1.0 : 0.0;
#pragma unroll UNROLL
  for (int j = 0; j < 8; ++j) {
    const int tj = j >> 1;
    const double vj = (j & 1) ? c1 : c0;  // this lane's entry in column j (if t == tj)
    const double p = shfl(vj, 4 * j + tj);
    const double r = rsqrt_pos(p);
    const double lv = p * r;
    {  // off the chain: pivot check and d (every lane holds the same p)
      const bool real = j < nreal, ok = (p > pfloor) & (p <= 1.7976931348623157e308);
      nbad += (real & !ok) ? 1 : 0;
      prod *= (real & (j >= jm)) ? p : 1.0;
    }
    const double x = vj * r;
    const double lval = (g > j) ? fma(fma(-x, lv, vj), r, x) : ((g == j) ? lv : 0.0);
    if (t == tj) {
      if (j & 1) c1 = lval;
      else c0 = lval;
    }
    const double lgj = shfl(lval, 4 * g + tj);        // L[g][j]
    const double lc0 = shfl(lval, 8 * t + tj);        // L[2t][j]
    const double lc1 = shfl(lval, 8 * t + 4 + tj);    // L[2t+1][j]
    if (g > j) {
      if (2 * t > j) c0 = fma(-lgj, lc0, c0);
      if (2 * t + 1 > j) c1 = fma(-lgj, lc1, c1);
    }
    if (g == j) {
      z0 *= r;
      z1 *= r;
    }
    const double zj0 = shfl(z0, 4 * j + t), zj1 = shfl(z1, 4 * j + t);
    if (g > j) {
      z0 = fma(-lgj, zj0, z0);
      z1 = fma(-lgj, zj1, z1);
    }
  }
  if (2 * t > g) c0 = 0.0;  // upper part of L_JJ: zero (the panel solves read all 64 entries)
  if (2 * t + 1 > g) c1 = 0.0;
  if (g == yr) {            // the y row's entries in this tile: u's last terms (columns ≥ m)
    if (2 * t < g && 2 * t >= jm) qd = fma(c0, c0, qd);
    if (2 * t + 1 < g && 2 * t + 1 >= jm) qd = fma(c1, c1, qd);
  }
  z0 = neg(z0);
  z1 = neg(z1);
}

}  // namespace tile
}  // namespace bv
