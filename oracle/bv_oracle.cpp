/* =============================================================================
 * oracle/bv_oracle.cpp — CPU ORACLE for the block-Vecchia log-likelihood.
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke(), bench.py's
 * cpu_baseline / --impl reference legs and the offline diagnostics under tools/
 * (parity_diag, pivot_floor_audit, accuracy_c5) may load this library.
 * It shares no code, header, table or constant with the CUDA product path
 * (paper_2410_04477_b200/), and it never includes anything from there.
 *
 * What it computes, each function citing the passage it follows
 * (PAPER.md = arXiv 2410.04477 LaTeX source):
 *   or_matern            Eq. (7), PAPER.md:304-311 (§3.1) — isotropic Matérn,
 *                        x = r/β (reading G2/G3), closed forms at ν ∈ {½,3/2,5/2}.
 *   or_bv_loglik         Alg. 1 l.10-30, PAPER.md:593-633 (§S1), taken
 *                        literally: POTRF, TRSM, TRSV, GEMM, GEMV, subtract,
 *                        POTRF, TRSV, dot, logdet, accumulate — nine separate
 *                        steps, NOT the fused joint Cholesky the GPU uses.
 *   or_bv_loglik_jitter  the same with the optional jitter retry schedule
 *                        (reading G15b).
 *   or_bv_loglik_joint   DIAGNOSTIC ONLY, never a parity reference: the same
 *                        block terms through the other exact formulation (one
 *                        joint Cholesky), to measure how two FP64 formulations
 *                        differ on ill-conditioned blocks (reading G22).
 *   or_set_pivot_floor   the non-PD floor of reading G15 (floor audit only).
 *   or_exact_loglik      Eq. (1), PAPER.md:62-67 (§1) — dense Cholesky.
 *   or_classic_vecchia   classic Vecchia = block size 1, PAPER.md:76-78, :83;
 *                        univariate conditionals solved by Gaussian
 *                        elimination with partial pivoting (a different
 *                        algorithm from Alg. 1 on purpose).
 *   or_simulate_bv       block-Vecchia sequential simulation:
 *                        y_B = E[y_B | y_NN] + chol(Var[y_B | y_NN]) ε, formed
 *                        from ONE joint dense Cholesky of [NN; B] (a different
 *                        formulation from or_bv_loglik, so the generating-model
 *                        pin u_i ≈ ‖ε_i‖² cross-checks two formulations).
 *   or_simulate_exact    y = chol(Σθ) ε, for exact GRFs at small n (pinned:
 *                        Eq. (1) at y plus ½‖ε‖² is ε-independent).
 *   or_bv_predict        Alg. 2 l.8-13, PAPER.md:651-662 (§S1; §2.3
 *                        PAPER.md:194-240) taken literally per prediction block:
 *                        Σcon, Σcross, Σlk → L = POTRF(Σcon), W = L⁻¹Σcross,
 *                        z = L⁻¹y_NN, μ = Wᵀz, Σ_B* = Σlk − WᵀW (Σcross read as
 *                        K(s_NN, s_B*), m×l, as in Alg. 1 — reading G8).
 *   or_block_nn_bruteforce  Alg. 1 l.7-9 mNearestNeighborsForBlock,
 *                        PAPER.md:589-591, :104 (centroid), :165 (earlier blocks
 *                        only); O(n²) brute force used to pin the planner.
 *   or_kmeans_assign_bruteforce  Lloyd assignment step.
 *
 * Readings of the paper (DESIGN.md §3 lists them all): FP64 (G1); modified
 * Bessel K_ν with x = r/β (G2); m_1 = 0 → Σnew = Σlk, μ = 0 (G7); Σcross is
 * m×l = K(s_NN, s_B) (G8); d = 2 Σ log L'_jj (G10); −½ l log 2π per block
 * (G11); block points in ascending global id, neighbours in the order given
 * (G13); per-block terms summed in position order (G14); no jitter (G15).
 *
 * Build: g++ -O2 -std=c++17 -ffp-contract=off -fopenmp -shared -fPIC
 * (-ffp-contract=off: no FMA contraction, so results do not depend on the
 * host's FMA support — reading G23).
 *
 * Templated on Real ∈ {double, long double}; the long-double instance gives
 * FP64's own error δ for the κ-aware parity rule.
 * ========================================================================== */
#include <algorithm>
#include <cmath>
#include <cstdint>
#include <cstring>
#include <numeric>
#include <vector>
#ifdef _OPENMP
#include <omp.h>
#endif

namespace {

/* ln(2π) rounded to nearest double: 0x3FFD67F1C864BEB5 (reading G23).  The
 * long-double value is the 64-bit-mantissa rounding of 1.837877066409345483560659472811... */
template <class R> inline R ln_2pi();
template <> inline double ln_2pi<double>() { return 0x1.d67f1c864beb5p+0; }
template <> inline long double ln_2pi<long double>() { return 1.8378770664093454835606594728112353L; }

inline double m_exp(double x) { return std::exp(x); }
inline long double m_exp(long double x) { return std::exp(x); }

/* Eq. (7): C(r) = σ² 2^{1−ν}/Γ(ν) (r/β)^ν K_ν(r/β), general ν.
 * Evaluated literally with std::tgamma, std::pow and std::cyl_bessel_k. */
template <class R> R matern_general(R r, R sigma2, R beta, R nu) {
  if (r == R(0)) return sigma2;  // continuous limit C(0) = σ²
  R x = r / beta;
  R c = std::pow(R(2), R(1) - nu) / std::tgamma(nu);
  R k = std::cyl_bessel_k(nu, x);
  if (k == R(0)) return R(0);  // K_ν underflowed; avoid 0·inf
  return sigma2 * c * std::pow(x, nu) * k;
}

/* Eq. (7) with the half-integer closed forms (K_{1/2}, K_{3/2}, K_{5/2} are
 * elementary): ν=½: σ²e^{−x}; ν=3/2: σ²(1+x)e^{−x}; ν=5/2: σ²(1+x+x²/3)e^{−x}.
 * Dispatch rule (shared contract with the GPU): closed forms iff ν
 * is exactly 0.5, 1.5 or 2.5, else the general path. */
template <class R> R matern(R r, R sigma2, R beta, R nu) {
  if (r == R(0)) return sigma2;
  R x = r / beta;
  if (nu == R(0.5)) return sigma2 * m_exp(-x);
  if (nu == R(1.5)) return sigma2 * (R(1) + x) * m_exp(-x);
  if (nu == R(2.5)) return sigma2 * (R(1) + x + x * x / R(3)) * m_exp(-x);
  return matern_general<R>(r, sigma2, beta, nu);
}

/* Euclidean distance, dimensions summed in x, y, z order. */
template <class R> inline R dist(const double* a, const double* b, int d) {
  R s = 0;
  for (int k = 0; k < d; ++k) {
    R t = R(a[k]) - R(b[k]);
    s += t * t;
  }
  return std::sqrt(s);
}

/* Optional ±1-ulp perturbation of a covariance entry (parity reading G22,
 * DESIGN.md §3): FP64 cannot distinguish Σ from Σ with every entry moved by
 * one ulp, so the spread of FP64 results over a few such perturbations
 * estimates FP64's own error at ill-conditioned blocks.  The perturbation of
 * the pair {a, b} is a fixed function of (min id, max id, seed), so Σcon,
 * Σcross and Σlk see one consistent symmetric matrix; the diagonal (a == b)
 * is never perturbed.  seed == 0 → no perturbation (the default oracle). */
inline double perturb_entry(double v, int32_t a, int32_t b, uint32_t seed) {
  if (seed == 0 || a == b) return v;
  uint64_t lo = (uint64_t)(a < b ? a : b), hi = (uint64_t)(a < b ? b : a);
  uint64_t z = (lo << 32 | hi) + 0x9E3779B97F4A7C15ull * (uint64_t)seed;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  z ^= z >> 31;
  // seed s ≥ 1: a move of −s..+s ulp, uniform (the magnitude models an FP64
  // Eq. (7) evaluation — sqrt, division, exp, products — a few ulp off)
  const int span = 2 * (int)(seed >= 1000 ? seed / 1000 : 1) + 1;
  const int r = (int)(z % (uint64_t)span) - (span - 1) / 2;
  for (int i = 0; i < r; ++i) v = std::nextafter(v, INFINITY);
  for (int i = 0; i > r; --i) v = std::nextafter(v, -INFINITY);
  return v;
}
inline long double perturb_entry(long double v, int32_t, int32_t, uint32_t) { return v; }

/* Textbook unblocked Cholesky (Cholesky–Crout, column by column), row-major
 * lower factor in L (n×n, only j ≤ i used).  Returns false on a pivot that is
 * not > floor or not finite (reading G15: non-PD → failure; a covariance's
 * pivots are compared with kPivotFloor·σ², σ² being every diagonal entry of
 * Σθ, so an FP64-singular matrix — e.g. a repeated location, whose pivot is
 * rounding noise of either sign — fails whatever the rounding order). */
double kPivotFloor = 1e-14;  // reading G15; or_set_pivot_floor changes it (the floor audit only)
template <class R> bool potrf(const std::vector<R>& A, std::vector<R>& L, int n, R floor = R(0)) {
  L.assign((size_t)n * n, R(0));
  for (int j = 0; j < n; ++j) {
    R s = A[(size_t)j * n + j];
    for (int k = 0; k < j; ++k) s -= L[(size_t)j * n + k] * L[(size_t)j * n + k];
    if (!(s > floor) || !std::isfinite((double)s)) return false;
    R ljj = std::sqrt(s);
    L[(size_t)j * n + j] = ljj;
    for (int i = j + 1; i < n; ++i) {
      R t = A[(size_t)i * n + j];
      for (int k = 0; k < j; ++k) t -= L[(size_t)i * n + k] * L[(size_t)j * n + k];
      L[(size_t)i * n + j] = t / ljj;
    }
  }
  return true;
}

/* Forward substitution L x = b (TRSV), in place on x (= b on entry). */
template <class R> void trsv(const std::vector<R>& L, int n, R* x, size_t stride) {
  for (int i = 0; i < n; ++i) {
    R t = x[(size_t)i * stride];
    for (int k = 0; k < i; ++k) t -= L[(size_t)i * n + k] * x[(size_t)k * stride];
    x[(size_t)i * stride] = t / L[(size_t)i * n + i];
  }
}

struct PlanView {
  int64_t n;
  int d;
  const double* locs;
  const double* y;
  int32_t bc;
  const int32_t* order;
  const int64_t* nbr_ptr;
  const int32_t* nbr_idx;
  std::vector<int64_t> bptr;  // CSR of block members by block id, ascending id
  std::vector<int32_t> bidx;
};

void build_block_lists(PlanView& P, const int32_t* block_id) {
  P.bptr.assign((size_t)P.bc + 1, 0);
  for (int64_t i = 0; i < P.n; ++i) P.bptr[(size_t)block_id[i] + 1]++;
  for (int32_t b = 0; b < P.bc; ++b) P.bptr[(size_t)b + 1] += P.bptr[b];
  P.bidx.assign((size_t)P.n, 0);
  std::vector<int64_t> fill(P.bptr.begin(), P.bptr.end() - 1);
  for (int64_t i = 0; i < P.n; ++i) P.bidx[(size_t)fill[block_id[i]]++] = (int32_t)i;  // ascending id
}

/* One block of Alg. 1, literally, at permuted position k.
 * Returns 0, or 3 if a POTRF failed (non-PD). */
template <class R>
int alg1_block(const PlanView& P, int32_t k, R sigma2, R beta, R nu, R* u_out, R* d_out, uint32_t seed,
               R jit = R(0)) {
  const int32_t b = P.order[k];
  const int l = (int)(P.bptr[(size_t)b + 1] - P.bptr[b]);
  const int32_t* B = P.bidx.data() + P.bptr[b];
  const int m = (int)(P.nbr_ptr[(size_t)k + 1] - P.nbr_ptr[k]);
  const int32_t* NN = P.nbr_idx + P.nbr_ptr[k];
  const int d = P.d;
  auto loc = [&](int32_t i) { return P.locs + (size_t)i * d; };

  // l.11  Σlk ← K(s_B, s_B)          (l×l)
  std::vector<R> Slk((size_t)l * l);
  for (int a = 0; a < l; ++a)
    for (int c = 0; c < l; ++c)
      Slk[(size_t)a * l + c] = perturb_entry(matern<R>(dist<R>(loc(B[a]), loc(B[c]), d), sigma2, beta, nu), B[a], B[c], seed);
  for (int a = 0; a < l; ++a) Slk[(size_t)a * l + a] += jit;  // optional jitter mode (reading G15b)
  // l.14  y_B, y_NN
  std::vector<R> yB(l), yN(m);
  for (int a = 0; a < l; ++a) yB[a] = R(P.y[B[a]]);
  for (int a = 0; a < m; ++a) yN[a] = R(P.y[NN[a]]);

  std::vector<R> Snew = Slk;        // l.22 (m = 0: Σnew = Σlk, reading G7)
  std::vector<R> munew(l, R(0));    // l.23 (m = 0: μnew = 0)
  if (m > 0) {
    // l.12  Σcon ← K(s_NN, s_NN)    (m×m)
    std::vector<R> Scon((size_t)m * m);
    for (int a = 0; a < m; ++a)
      for (int c = 0; c < m; ++c)
        Scon[(size_t)a * m + c] = perturb_entry(matern<R>(dist<R>(loc(NN[a]), loc(NN[c]), d), sigma2, beta, nu), NN[a], NN[c], seed);
    for (int a = 0; a < m; ++a) Scon[(size_t)a * m + a] += jit;  // reading G15b
    // l.13  Σcross ← K(s_NN, s_B)   (m×l, reading G8)
    std::vector<R> Scross((size_t)m * l);
    for (int a = 0; a < m; ++a)
      for (int c = 0; c < l; ++c)
        Scross[(size_t)a * l + c] = perturb_entry(matern<R>(dist<R>(loc(NN[a]), loc(B[c]), d), sigma2, beta, nu), NN[a], B[c], seed);
    // l.17  L ← POTRF(Σcon)
    std::vector<R> L;
    if (!potrf<R>(Scon, L, m, R(kPivotFloor) * sigma2)) return 3;
    // l.18  Σ'cross ← TRSM(L, Σcross): column by column forward substitution
    std::vector<R> W = Scross;
    for (int c = 0; c < l; ++c) trsv<R>(L, m, W.data() + c, (size_t)l);
    // l.19  y' ← TRSV(L, y_NN)     (garbled "y'^τ", reading G9)
    std::vector<R> z = yN;
    trsv<R>(L, m, z.data(), 1);
    // l.20  Σcor ← GEMM(Σ'crossᵀ, Σ'cross)  (l×l)
    std::vector<R> Scor((size_t)l * l, R(0));
    for (int a = 0; a < l; ++a)
      for (int c = 0; c < l; ++c) {
        R s = 0;
        for (int q = 0; q < m; ++q) s += W[(size_t)q * l + a] * W[(size_t)q * l + c];
        Scor[(size_t)a * l + c] = s;
      }
    // l.21  μcor ← GEMV(Σ'crossᵀ, y')
    std::vector<R> mucor(l, R(0));
    for (int a = 0; a < l; ++a) {
      R s = 0;
      for (int q = 0; q < m; ++q) s += W[(size_t)q * l + a] * z[q];
      mucor[a] = s;
    }
    // l.22  Σnew ← Σold − Σcor ;  l.23  μnew ← μcor
    for (size_t e = 0; e < Snew.size(); ++e) Snew[e] = Slk[e] - Scor[e];
    munew = mucor;
  }
  // l.24  L' ← POTRF(Σnew)
  std::vector<R> Lp;
  if (!potrf<R>(Snew, Lp, l, R(kPivotFloor) * sigma2)) return 3;
  // l.25  v ← TRSV(L', y_B − μnew)
  std::vector<R> v(l);
  for (int a = 0; a < l; ++a) v[a] = yB[a] - munew[a];
  trsv<R>(Lp, l, v.data(), 1);
  // l.26  u ← vᵀv ;  l.27  d ← 2 log det L' = 2 Σ log L'_jj (reading G10)
  R u = 0, ld = 0;
  for (int a = 0; a < l; ++a) u += v[a] * v[a];
  for (int a = 0; a < l; ++a) ld += std::log(Lp[(size_t)a * l + a]);
  *u_out = u;
  *d_out = R(2) * ld;
  return 0;
}

/* DIAGNOSTIC ONLY (not a parity reference): the same block term through the
 * other exact formulation — ONE unblocked right-looking Cholesky of the joint
 * (N+1)×(N+1) matrix [[Σcon, Σcross, ·],[Σcrossᵀ, Σlk, ·],[y_NNᵀ, y_Bᵀ, ·]]
 * (neighbours first, the y row appended and eliminated but never pivoted):
 * d = Σ_{j≥m} log p_j, u = Σ_{j≥m} L_Nj² (identical to l.17-27 in exact
 * arithmetic).  Lets tools/parity_diag.py measure how far two
 * FP64 formulations of Alg. 1 differ on ill-conditioned blocks (reading G22). */
template <class R>
int joint_block(const PlanView& P, int32_t k, R sigma2, R beta, R nu, R* u_out, R* d_out) {
  const int32_t b = P.order[k];
  const int l = (int)(P.bptr[(size_t)b + 1] - P.bptr[b]);
  const int32_t* B = P.bidx.data() + P.bptr[b];
  const int m = (int)(P.nbr_ptr[(size_t)k + 1] - P.nbr_ptr[k]);
  const int32_t* NN = P.nbr_idx + P.nbr_ptr[k];
  const int N = m + l, d = P.d;
  std::vector<int32_t> id((size_t)N);
  for (int a = 0; a < m; ++a) id[a] = NN[a];
  for (int a = 0; a < l; ++a) id[(size_t)m + a] = B[a];
  auto loc = [&](int32_t i) { return P.locs + (size_t)i * d; };
  const int Na = N + 1;
  std::vector<R> A((size_t)Na * Na, R(0));  // lower triangle, row-major
  for (int r = 0; r < N; ++r)
    for (int c = 0; c <= r; ++c) A[(size_t)r * Na + c] = matern<R>(dist<R>(loc(id[r]), loc(id[c]), d), sigma2, beta, nu);
  for (int c = 0; c < N; ++c) A[(size_t)N * Na + c] = R(P.y[id[c]]);
  R u = 0, ld = 0;
  for (int j = 0; j < N; ++j) {
    const R p = A[(size_t)j * Na + j];
    if (!(p > R(kPivotFloor) * sigma2) || !std::isfinite((double)p)) return 3;
    const R Ljj = std::sqrt(p);
    if (j >= m) ld += std::log(p);
    for (int i = j + 1; i <= N; ++i) A[(size_t)i * Na + j] /= Ljj;
    for (int i = j + 1; i <= N; ++i)
      for (int c = j + 1; c <= i && c < N; ++c) A[(size_t)i * Na + c] -= A[(size_t)i * Na + j] * A[(size_t)c * Na + j];
    if (j >= m) u += A[(size_t)N * Na + j] * A[(size_t)N * Na + j];
  }
  *u_out = u;
  *d_out = ld;
  return 0;
}

template <class R>
int bv_loglik_impl(PlanView& P, const int32_t* block_id, const double* theta, double* out_u, double* out_d,
                   double* out_t, double* out_loglik, int32_t* failed_pos, int nthreads, int k_begin, int k_end,
                   double* out_loglik_ld_sum, uint32_t seed, int jitter_mode = 0, double* out_eps = nullptr,
                   int32_t* out_events = nullptr, int joint = 0) {
  build_block_lists(P, block_id);
  const R sigma2 = R(theta[0]), beta = R(theta[1]), nu = R(theta[2]);
  const int nk = k_end - k_begin;
  std::vector<R> t(nk), uu(nk), dd(nk);
  std::vector<int> st(nk, 0);
#ifdef _OPENMP
  if (nthreads > 0) omp_set_num_threads(nthreads);
#pragma omp parallel for schedule(dynamic, 4)
#endif
  for (int q = 0; q < nk; ++q) {
    const int32_t k = k_begin + q;
    R u = 0, d = 0;
    st[q] = joint ? joint_block<R>(P, k, sigma2, beta, nu, &u, &d) : alg1_block<R>(P, k, sigma2, beta, nu, &u, &d, seed);
    // Optional jitter mode (reading G15b; SPEC.md:197 schedule with base_scale = σ²,
    // SPEC.md:238): a block whose POTRF failed is re-run from scratch with
    // ε·σ² added to every diagonal entry of Σcon and Σlk, ε = 1e-10, 1e-8, 1e-6
    // in turn; the first ε that succeeds is kept.
    double eps_used = 0.0;
    if (jitter_mode && st[q] != 0) {
      static const double kSched[3] = {1e-10, 1e-8, 1e-6};
      for (int e = 0; e < 3 && st[q] != 0; ++e) {
        st[q] = alg1_block<R>(P, k, sigma2, beta, nu, &u, &d, seed, R(kSched[e]) * sigma2);
        eps_used = kSched[e];
      }
      if (st[q] != 0) eps_used = 0.0;
    }
    if (out_eps) out_eps[q] = eps_used;
    const int l = (int)(P.bptr[(size_t)P.order[k] + 1] - P.bptr[P.order[k]]);
    uu[q] = u;
    dd[q] = d;
    // l.29  ℓ ← ℓ − ½(u_i + d_i + l_i log 2π)
    t[q] = -R(0.5) * (u + d + R(l) * ln_2pi<R>());
  }
  int32_t fail = -1;
  for (int q = 0; q < nk; ++q)
    if (st[q] != 0) { fail = k_begin + q; break; }
  if (out_events) {
    int32_t ev = 0;
    if (out_eps)
      for (int q = 0; q < nk; ++q) ev += (st[q] == 0 && out_eps[q] > 0.0) ? 1 : 0;
    *out_events = ev;
  }
  if (failed_pos) *failed_pos = fail;
  if (fail >= 0) {
    if (out_loglik) *out_loglik = -INFINITY;
    return 3;
  }
  // l.28-30: accumulate in position order (reading G14)
  R acc = 0;
  long double acc_ld = 0;
  for (int q = 0; q < nk; ++q) {
    acc += t[q];
    acc_ld += (long double)t[q];
    if (out_u) out_u[q] = (double)uu[q];
    if (out_d) out_d[q] = (double)dd[q];
    if (out_t) out_t[q] = (double)t[q];
  }
  if (out_loglik) *out_loglik = (double)acc;
  if (out_loglik_ld_sum) *out_loglik_ld_sum = (double)acc_ld;
  return 0;
}

/* Gaussian elimination with partial pivoting, solving A x = b in place (A n×n
 * row-major, destroyed).  Used by the classic-Vecchia oracle only. */
bool gepp_solve(std::vector<double>& A, std::vector<double>& b, int n) {
  for (int c = 0; c < n; ++c) {
    int p = c;
    for (int r = c + 1; r < n; ++r)
      if (std::fabs(A[(size_t)r * n + c]) > std::fabs(A[(size_t)p * n + c])) p = r;
    if (A[(size_t)p * n + c] == 0.0) return false;
    if (p != c) {
      for (int q = 0; q < n; ++q) std::swap(A[(size_t)p * n + q], A[(size_t)c * n + q]);
      std::swap(b[p], b[c]);
    }
    for (int r = c + 1; r < n; ++r) {
      double f = A[(size_t)r * n + c] / A[(size_t)c * n + c];
      for (int q = c; q < n; ++q) A[(size_t)r * n + q] -= f * A[(size_t)c * n + q];
      b[r] -= f * b[c];
    }
  }
  for (int r = n - 1; r >= 0; --r) {
    double s = b[r];
    for (int q = r + 1; q < n; ++q) s -= A[(size_t)r * n + q] * b[q];
    b[r] = s / A[(size_t)r * n + r];
  }
  return true;
}

bool theta_ok(const double* th) {
  for (int i = 0; i < 3; ++i)
    if (!(th[i] > 0) || !std::isfinite(th[i])) return false;
  return true;
}

}  // namespace

extern "C" {

/* The non-PD floor of reading G15 (default 1e-14, i.e. a pivot must exceed 1e-14·σ²);
 * 0 = SURVEY §8b's plain "pivot ≤ 0" rule.  Process-global; for the floor audit
 * (tools/pivot_floor_audit.py) only. */
void or_set_pivot_floor(double f) { kPivotFloor = f; }

/* Eq. (7).  mode 0: dispatching (closed forms at ν ∈ {½,3/2,5/2});
 * mode 1: always the general K_ν path; mode 2: long-double dispatching. */
double or_matern(double r, double sigma2, double beta, double nu, int mode) {
  if (mode == 1) return matern_general<double>(r, sigma2, beta, nu);
  if (mode == 2) return (double)matern<long double>(r, sigma2, beta, nu);
  return matern<double>(r, sigma2, beta, nu);
}

double or_ln_2pi(int long_double_mode) { return long_double_mode ? (double)ln_2pi<long double>() : ln_2pi<double>(); }

/* Unblocked Cholesky of a row-major n×n SPD matrix (Alg. 1 POTRF building block).
 * Returns 0 or 3 (non-PD).  L is n×n row-major, upper part zero. */
int or_potrf(const double* A, int n, double* L) {
  std::vector<double> a(A, A + (size_t)n * n), l;
  if (!potrf<double>(a, l, n)) return 3;
  std::memcpy(L, l.data(), sizeof(double) * (size_t)n * n);
  return 0;
}

/* Forward substitution L x = b (Alg. 1 TRSV building block). */
void or_trsv(const double* L, int n, double* x) {
  std::vector<double> l(L, L + (size_t)n * n);
  trsv<double>(l, n, x, 1);
}

/* Alg. 1: block-Vecchia log-likelihood for a frozen plan.
 *   locs n×d row-major; y n; block_id n in [0,bc); order bc (order[k] = block at
 *   position k); nbr_ptr bc+1 (CSR by position); nbr_idx global point ids.
 *   theta = (σ², β, ν).  long_double != 0 runs the whole algorithm in 80-bit.
 *   Per-block outputs (u_k, d_k, t_k) for positions [k_begin, k_end) are
 *   written to out_* (each may be NULL); out_loglik = Σ t_k over that range.
 *   perturb_seed != 0 (FP64 only): every off-diagonal covariance entry moved
 *   by −1, 0 or +1 ulp (perturb_entry; parity reading G22).
 * Returns 0, 2 (invalid θ) or 3 (non-PD; *failed_pos = smallest failing k). */
int or_bv_loglik(int64_t n, int d, const double* locs, const double* y, int32_t bc, const int32_t* block_id,
                 const int32_t* order, const int64_t* nbr_ptr, const int32_t* nbr_idx, const double* theta,
                 int long_double, int nthreads, int32_t k_begin, int32_t k_end, double* out_u, double* out_d,
                 double* out_t, double* out_loglik, int32_t* failed_pos, uint32_t perturb_seed) {
  if (!theta_ok(theta) || n < 1 || (d != 2 && d != 3) || bc < 1 || k_begin < 0 || k_end > bc || k_begin > k_end)
    return 2;
  PlanView P{n, d, locs, y, bc, order, nbr_ptr, nbr_idx, {}, {}};
  if (long_double)
    return bv_loglik_impl<long double>(P, block_id, theta, out_u, out_d, out_t, out_loglik, failed_pos, nthreads,
                                       k_begin, k_end, nullptr, 0u);
  return bv_loglik_impl<double>(P, block_id, theta, out_u, out_d, out_t, out_loglik, failed_pos, nthreads, k_begin,
                                k_end, nullptr, perturb_seed);
}

/* DIAGNOSTIC ONLY: or_bv_loglik through the joint formulation (joint_block above);
 * same arguments minus perturb_seed.  Not used for parity. */
int or_bv_loglik_joint(int64_t n, int d, const double* locs, const double* y, int32_t bc, const int32_t* block_id,
                       const int32_t* order, const int64_t* nbr_ptr, const int32_t* nbr_idx, const double* theta,
                       int long_double, int nthreads, int32_t k_begin, int32_t k_end, double* out_u, double* out_d,
                       double* out_t, double* out_loglik, int32_t* failed_pos) {
  if (!theta_ok(theta) || n < 1 || (d != 2 && d != 3) || bc < 1 || k_begin < 0 || k_end > bc || k_begin > k_end)
    return 2;
  PlanView P{n, d, locs, y, bc, order, nbr_ptr, nbr_idx, {}, {}};
  if (long_double)
    return bv_loglik_impl<long double>(P, block_id, theta, out_u, out_d, out_t, out_loglik, failed_pos, nthreads,
                                       k_begin, k_end, nullptr, 0u, 0, nullptr, nullptr, 1);
  return bv_loglik_impl<double>(P, block_id, theta, out_u, out_d, out_t, out_loglik, failed_pos, nthreads, k_begin,
                                k_end, nullptr, 0u, 0, nullptr, nullptr, 1);
}

/* Alg. 1 with the optional jitter mode (reading G15b): per block, the
 * failed-POTRF retry schedule ε ∈ {1e-10, 1e-8, 1e-6}·σ² on the diagonal of
 * Σcon and Σlk.  out_eps[q] = the ε used (0 = none); *events = blocks that
 * needed one (SPEC.md:269 jitter_events).  FP64 only. */
int or_bv_loglik_jitter(int64_t n, int d, const double* locs, const double* y, int32_t bc, const int32_t* block_id,
                        const int32_t* order, const int64_t* nbr_ptr, const int32_t* nbr_idx, const double* theta,
                        int nthreads, int32_t k_begin, int32_t k_end, double* out_u, double* out_d, double* out_t,
                        double* out_eps, double* out_loglik, int32_t* failed_pos, int32_t* events) {
  if (!theta_ok(theta) || n < 1 || (d != 2 && d != 3) || bc < 1 || k_begin < 0 || k_end > bc || k_begin > k_end ||
      !out_eps || !events)
    return 2;
  PlanView P{n, d, locs, y, bc, order, nbr_ptr, nbr_idx, {}, {}};
  return bv_loglik_impl<double>(P, block_id, theta, out_u, out_d, out_t, out_loglik, failed_pos, nthreads, k_begin,
                                k_end, nullptr, 0u, 1, out_eps, events);
}

/* Alg. 2: block-Vecchia prediction at n_new new locations.
 *   locs (n×d) / y (n): the training data; locs_new (n_new×d); block_new
 *   (n_new, in [0, bc_new)): the clustering g of l.4; nbr_ptr/nbr_idx (CSR by
 *   prediction block, training ids): the NN sets of l.6 (m nearest training
 *   points, any training point — PAPER.md:203 "from y").  Block points in
 *   ascending new-point id (reading G13).  Outputs: mean[n_new] = μ (l.9,
 *   l.12), var[n_new] = diag Σ_B* (PAPER.md:242), cov (may be NULL): block b's
 *   l_b×l_b Σ_B* row-major at offset Σ_{b'<b} l_b'² (l.10-11, "for conditional
 *   simulations", l.15).  Returns 0, 2 or 3 (non-PD; *failed_block).  FP64. */
int or_bv_predict(int64_t n, int d, const double* locs, const double* y, const double* theta, int64_t n_new,
                  const double* locs_new, int32_t bc_new, const int32_t* block_new, const int64_t* nbr_ptr,
                  const int32_t* nbr_idx, double* mean, double* var, double* cov, int32_t* failed_block) {
  if (!theta_ok(theta) || n < 1 || (d != 2 && d != 3) || n_new < 1 || bc_new < 1) return 2;
  std::vector<int64_t> bptr((size_t)bc_new + 1, 0);
  for (int64_t i = 0; i < n_new; ++i) {
    if (block_new[i] < 0 || block_new[i] >= bc_new) return 2;
    bptr[(size_t)block_new[i] + 1]++;
  }
  for (int32_t b = 0; b < bc_new; ++b) bptr[(size_t)b + 1] += bptr[b];
  std::vector<int32_t> bidx((size_t)n_new);
  {
    std::vector<int64_t> fill(bptr.begin(), bptr.end() - 1);
    for (int64_t i = 0; i < n_new; ++i) bidx[(size_t)fill[block_new[i]]++] = (int32_t)i;
  }
  std::vector<int64_t> coff((size_t)bc_new + 1, 0);
  for (int32_t b = 0; b < bc_new; ++b) {
    const int64_t l = bptr[(size_t)b + 1] - bptr[b];
    coff[(size_t)b + 1] = coff[b] + l * l;
  }
  const double s2 = theta[0], beta = theta[1], nu = theta[2];
  int32_t fail = -1;
  for (int32_t b = 0; b < bc_new; ++b) {
    const int l = (int)(bptr[(size_t)b + 1] - bptr[b]);
    const int32_t* B = bidx.data() + bptr[b];
    const int m = (int)(nbr_ptr[(size_t)b + 1] - nbr_ptr[b]);
    const int32_t* NN = nbr_idx + nbr_ptr[b];
    auto lt = [&](int32_t i) { return locs + (size_t)i * d; };
    auto ln = [&](int32_t i) { return locs_new + (size_t)i * d; };
    // l.8  Σlk ← cov(S_B*, S_B*)   (l×l)
    std::vector<double> Slk((size_t)l * l);
    for (int a = 0; a < l; ++a)
      for (int c = 0; c < l; ++c) Slk[(size_t)a * l + c] = matern<double>(dist<double>(ln(B[a]), ln(B[c]), d), s2, beta, nu);
    std::vector<double> mu(l, 0.0), Sb = Slk;
    if (m > 0) {
      // l.6  Σcon ← cov(S_NN, S_NN) (m×m);  l.7  Σcross ← cov(S_NN, S_B*) (m×l)
      std::vector<double> Scon((size_t)m * m), W((size_t)m * l), z(m);
      for (int a = 0; a < m; ++a)
        for (int c = 0; c < m; ++c) Scon[(size_t)a * m + c] = matern<double>(dist<double>(lt(NN[a]), lt(NN[c]), d), s2, beta, nu);
      for (int a = 0; a < m; ++a)
        for (int c = 0; c < l; ++c) W[(size_t)a * l + c] = matern<double>(dist<double>(lt(NN[a]), ln(B[c]), d), s2, beta, nu);
      for (int a = 0; a < m; ++a) z[a] = y[NN[a]];
      // (Σcon)⁻¹ applied through its Cholesky factor: L = POTRF(Σcon), W = L⁻¹Σcross, z = L⁻¹y_NN
      std::vector<double> L;
      if (!potrf<double>(Scon, L, m, kPivotFloor * s2)) {
        fail = b;
        break;
      }
      for (int c = 0; c < l; ++c) trsv<double>(L, m, W.data() + c, (size_t)l);
      trsv<double>(L, m, z.data(), 1);
      // l.9  μ_B* = Σcrossᵀ (Σcon)⁻¹ y_NN = Wᵀz
      for (int a = 0; a < l; ++a) {
        double t = 0;
        for (int q = 0; q < m; ++q) t += W[(size_t)q * l + a] * z[q];
        mu[a] = t;
      }
      // l.10-11  Σ_B* = Σlk − Σcrossᵀ (Σcon)⁻¹ Σcross = Σlk − WᵀW
      for (int a = 0; a < l; ++a)
        for (int c = 0; c < l; ++c) {
          double t = 0;
          for (int q = 0; q < m; ++q) t += W[(size_t)q * l + a] * W[(size_t)q * l + c];
          Sb[(size_t)a * l + c] = Slk[(size_t)a * l + c] - t;
        }
    }
    // l.12  y_B* = μ_B*; variances = diag Σ_B*
    for (int a = 0; a < l; ++a) {
      mean[B[a]] = mu[a];
      if (var) var[B[a]] = Sb[(size_t)a * l + a];
    }
    if (cov) std::copy(Sb.begin(), Sb.end(), cov + coff[b]);
  }
  if (fail >= 0) {
    if (failed_block) *failed_block = fail;
    return 3;
  }
  return 0;
}

/* Eq. (1): ℓ = −n/2 log 2π − ½ log|Σθ| − ½ yᵀΣθ⁻¹y, dense
 * Cholesky, n ≤ 6000 guard.  Returns 0, 2, or 3 (non-PD). */
int or_exact_loglik(int64_t n, int d, const double* locs, const double* y, const double* theta, int long_double,
                    double* out) {
  if (!theta_ok(theta) || n < 1 || n > 6000 || (d != 2 && d != 3)) return 2;
  auto run = [&](auto zero) -> int {
    using R = decltype(zero);
    const R s2 = R(theta[0]), be = R(theta[1]), nu = R(theta[2]);
    std::vector<R> S((size_t)n * n), L;
    for (int64_t i = 0; i < n; ++i)
      for (int64_t j = 0; j < n; ++j)
        S[(size_t)i * n + j] = matern<R>(dist<R>(locs + i * d, locs + j * d, d), s2, be, nu);
    if (!potrf<R>(S, L, (int)n, R(kPivotFloor) * s2)) return 3;
    std::vector<R> z(n);
    for (int64_t i = 0; i < n; ++i) z[i] = R(y[i]);
    trsv<R>(L, (int)n, z.data(), 1);
    R quad = 0, ld = 0;
    for (int64_t i = 0; i < n; ++i) {
      quad += z[i] * z[i];
      ld += std::log(L[(size_t)i * n + i]);
    }
    *out = (double)(-R(n) / R(2) * ln_2pi<R>() - ld - R(0.5) * quad);  // ½ log|Σ| = Σ log L_ii
    return 0;
  };
  return long_double ? run((long double)0) : run(0.0);
}

/* Classic Vecchia ("special case when each block size is 1",
 * PAPER.md:83): ℓ = Σ_i log N(y_i; μ_i, σ_i²) with μ_i = cᵀΣ_N⁻¹y_N,
 * σ_i² = σ² − cᵀΣ_N⁻¹c, over points in the order point_order[0..n), each
 * conditioned on nbr_idx[nbr_ptr[p]..nbr_ptr[p+1]) (point ids, all earlier).
 * Solves with Gaussian elimination with partial pivoting, not Cholesky. */
int or_classic_vecchia(int64_t n, int d, const double* locs, const double* y, const int32_t* point_order,
                       const int64_t* nbr_ptr, const int32_t* nbr_idx, const double* theta, double* out) {
  if (!theta_ok(theta)) return 2;
  const double s2 = theta[0], be = theta[1], nu = theta[2];
  double total = 0;
  for (int64_t p = 0; p < n; ++p) {
    const int32_t i = point_order[p];
    const int m = (int)(nbr_ptr[p + 1] - nbr_ptr[p]);
    const int32_t* N = nbr_idx + nbr_ptr[p];
    double mu = 0, var = s2;
    if (m > 0) {
      std::vector<double> A((size_t)m * m), c(m), w(m);
      for (int a = 0; a < m; ++a) {
        for (int b = 0; b < m; ++b) A[(size_t)a * m + b] = matern<double>(dist<double>(locs + (size_t)N[a] * d, locs + (size_t)N[b] * d, d), s2, be, nu);
        c[a] = matern<double>(dist<double>(locs + (size_t)N[a] * d, locs + (size_t)i * d, d), s2, be, nu);
      }
      w = c;
      if (!gepp_solve(A, w, m)) return 3;  // w = Σ_N⁻¹ c
      for (int a = 0; a < m; ++a) {
        mu += w[a] * y[N[a]];
        var -= w[a] * c[a];
      }
    }
    if (!(var > 0)) return 3;
    const double r = y[i] - mu;
    total += -0.5 * (std::log(var) + ln_2pi<double>() + r * r / var);
  }
  *out = total;
  return 0;
}

/* Block-Vecchia sequential simulation: positions are visited so
 * that every block's neighbours are simulated first (level schedule over the
 * neighbour DAG; each block depends only on its own inputs, so the result is
 * independent of thread count).  For position k with joint points J = [NN; B]:
 * chol(Σ_J) = [[L11,0],[L21,L22]], y_B = L21 L11⁻¹ y_NN + L22 ε_B, where
 * ε_B = eps[B] (one standard normal per global point id). */
int or_simulate_bv(int64_t n, int d, const double* locs, int32_t bc, const int32_t* block_id, const int32_t* order,
                   const int64_t* nbr_ptr, const int32_t* nbr_idx, const double* theta, const double* eps,
                   double* y_out, int nthreads) {
  if (!theta_ok(theta)) return 2;
  PlanView P{n, d, locs, y_out, bc, order, nbr_ptr, nbr_idx, {}, {}};
  build_block_lists(P, block_id);
  const double s2 = theta[0], be = theta[1], nu = theta[2];
  // level of each position: 1 + max level of the positions owning its neighbours
  std::vector<int32_t> pos_of_block(bc);
  for (int32_t k = 0; k < bc; ++k) pos_of_block[order[k]] = k;
  std::vector<int32_t> level(bc, 0);
  int32_t maxlev = 0;
  for (int32_t k = 0; k < bc; ++k) {
    int32_t lv = 0;
    for (int64_t q = nbr_ptr[k]; q < nbr_ptr[k + 1]; ++q) lv = std::max(lv, level[pos_of_block[block_id[nbr_idx[q]]]] + 1);
    level[k] = lv;
    maxlev = std::max(maxlev, lv);
  }
  std::vector<std::vector<int32_t>> bylev(maxlev + 1);
  for (int32_t k = 0; k < bc; ++k) bylev[level[k]].push_back(k);
  int status = 0;
#ifdef _OPENMP
  if (nthreads > 0) omp_set_num_threads(nthreads);
#endif
  for (int32_t lv = 0; lv <= maxlev && status == 0; ++lv) {
    const auto& ks = bylev[lv];
#ifdef _OPENMP
#pragma omp parallel for schedule(dynamic, 1)
#endif
    for (size_t q = 0; q < ks.size(); ++q) {
      const int32_t k = ks[q];
      const int32_t b = order[k];
      const int l = (int)(P.bptr[(size_t)b + 1] - P.bptr[b]);
      const int32_t* B = P.bidx.data() + P.bptr[b];
      const int m = (int)(nbr_ptr[k + 1] - nbr_ptr[k]);
      const int32_t* NN = nbr_idx + nbr_ptr[k];
      const int N = m + l;
      std::vector<int32_t> J(N);
      for (int a = 0; a < m; ++a) J[a] = NN[a];
      for (int a = 0; a < l; ++a) J[m + a] = B[a];
      std::vector<double> S((size_t)N * N), L;
      for (int a = 0; a < N; ++a)
        for (int c = 0; c < N; ++c)
          S[(size_t)a * N + c] = matern<double>(dist<double>(locs + (size_t)J[a] * d, locs + (size_t)J[c] * d, d), s2, be, nu);
      if (!potrf<double>(S, L, N, kPivotFloor * s2)) {
#ifdef _OPENMP
#pragma omp critical
#endif
        status = 3;
        continue;
      }
      std::vector<double> e(m);
      for (int a = 0; a < m; ++a) e[a] = y_out[NN[a]];
      for (int a = 0; a < m; ++a) {  // L11 e = y_NN (L11 = leading m×m block of L, leading dim N)
        double t = e[a];
        for (int c = 0; c < a; ++c) t -= L[(size_t)a * N + c] * e[c];
        e[a] = t / L[(size_t)a * N + a];
      }
      for (int a = 0; a < l; ++a) {
        double s = 0;
        for (int c = 0; c < m; ++c) s += L[(size_t)(m + a) * N + c] * e[c];
        for (int c = 0; c <= a; ++c) s += L[(size_t)(m + a) * N + m + c] * eps[B[c]];
        y_out[B[a]] = s;
      }
    }
  }
  return status;
}

/* Exact GRF: y = chol(Σθ) ε (dense; n ≤ 6000). */
int or_simulate_exact(int64_t n, int d, const double* locs, const double* theta, const double* eps, double* y_out) {
  if (!theta_ok(theta) || n > 6000) return 2;
  std::vector<double> S((size_t)n * n), L;
  for (int64_t i = 0; i < n; ++i)
    for (int64_t j = 0; j < n; ++j)
      S[(size_t)i * n + j] = matern<double>(dist<double>(locs + i * d, locs + j * d, d), theta[0], theta[1], theta[2]);
  if (!potrf<double>(S, L, (int)n, kPivotFloor * theta[0])) return 3;
  for (int64_t i = 0; i < n; ++i) {
    double s = 0;
    for (int64_t j = 0; j <= i; ++j) s += L[(size_t)i * n + j] * eps[j];
    y_out[i] = s;
  }
  return 0;
}

/* mNearestNeighborsForBlock (Alg. 1 l.7-9), brute force
 * O(n²): for each position k, centroid c_k = mean of block order[k]'s points
 * (summed in ascending id, each dimension, then divided by l); candidates are
 * all points of blocks order[0..k-1]; key = (‖s − c_k‖², id)
 * with the squared distance summed in x, y, z order; the m_k = min(m, #cand)
 * smallest keys, ascending.  nbr_ptr must have bc+1 entries; nbr_idx room for
 * Σ m_k ≤ bc·m ids. */
int or_block_nn_bruteforce(int64_t n, int d, const double* locs, int32_t bc, const int32_t* block_id,
                           const int32_t* order, int32_t m, int64_t* nbr_ptr, int32_t* nbr_idx) {
  std::vector<int32_t> pos_of_block(bc);
  for (int32_t k = 0; k < bc; ++k) pos_of_block[order[k]] = k;
  nbr_ptr[0] = 0;
  std::vector<std::pair<double, int32_t>> cand;
  for (int32_t k = 0; k < bc; ++k) {
    double c[3] = {0, 0, 0};
    int64_t cnt = 0;
    for (int64_t i = 0; i < n; ++i)
      if (block_id[i] == order[k]) {
        for (int q = 0; q < d; ++q) c[q] += locs[i * d + q];
        ++cnt;
      }
    for (int q = 0; q < d; ++q) c[q] /= (double)cnt;
    cand.clear();
    for (int64_t i = 0; i < n; ++i)
      if (pos_of_block[block_id[i]] < k) {
        double s = 0;
        for (int q = 0; q < d; ++q) {
          double t = locs[i * d + q] - c[q];
          s += t * t;
        }
        cand.emplace_back(s, (int32_t)i);
      }
    std::sort(cand.begin(), cand.end());
    const int64_t mk = std::min<int64_t>(m, (int64_t)cand.size());
    for (int64_t q = 0; q < mk; ++q) nbr_idx[nbr_ptr[k] + q] = cand[q].second;
    nbr_ptr[k + 1] = nbr_ptr[k] + mk;
  }
  return 0;
}

/* Lloyd assignment step: nearest centroid by squared
 * distance (x, y, z order), ties → lower centroid id. */
void or_kmeans_assign_bruteforce(int64_t n, int d, const double* locs, int32_t k, const double* cent, int32_t* assign) {
  for (int64_t i = 0; i < n; ++i) {
    double best = INFINITY;
    int32_t bi = -1;
    for (int32_t c = 0; c < k; ++c) {
      double s = 0;
      for (int q = 0; q < d; ++q) {
        double t = locs[i * d + q] - cent[(size_t)c * d + q];
        s += t * t;
      }
      if (s < best) {
        best = s;
        bi = c;
      }
    }
    assign[i] = bi;
  }
}

}  // extern "C"
