// bv_block_v3.cu — the large-block kernel (joint sizes N ≥ 80; smaller ones go to the
// warp-per-block kernel, bv_block_w.cu): one block per CTA, warp-specialised.
//
// One Cholesky of the augmented joint matrix [[Σcon, Σcross, y_NN],[Σcrossᵀ, Σlk,
// y_B]] (Alg. 1 l.10-29, fused as in DESIGN.md §4), left-looking
// over 8-wide column panels, FP64 MMA (DMMA.8x8x4) for every tile product, Matérn
// generated on the fly.  A dedicated chain warp factors the diagonal tiles and
// hands each panel to the update warps (3, or 7 from 20 tile rows: KW) through named
// barriers (bar.arrive / bar.sync), one panel ahead:
//
//  chain warp, iteration J:                    update warps, iteration J:
//    factor C(J,J) across its lanes → publish    generate A(I,J+1) for their tiles I ≥ J+1
//      L_JJ and L_JJ⁻¹ (tile::factor_dist)         straight into MMA accumulators, then
//    sync  E  (updates of iteration J−1 done)      S ← S − L(I,K) L(J+1,K)ᵀ, K = 0..J−1
//    arrive G                                      (progressive subtraction); warp 1 owns
//    L(J+1,J) = C(J+1,J) L_JJ⁻ᵀ                    the next diagonal tile → publishes it (P)
//    sync H (P published) ; arrive F             sync G ; arrive H
//    C(J+1,J+1) = P − L(J+1,J) L(J+1,J)ᵀ         L(I,J) = C(I,J) L_JJ⁻ᵀ, I ≥ J+2
//    → next J                                    sync F ; C(I,J+1) = S − L(I,J) L(J+1,J)ᵀ
//                                                  → slots ; arrive E
//
// Panel solves are DMMA products with the explicit L_JJ⁻¹ plus one FP64
// refinement step.  The diagonal tile lives in a private 8×8 buffer; every
// other tile lives in one shared-memory slot from its store through its
// in-place solve to its last use (slot table: bv_host.cpp SlotTables); joint
// sizes past shared memory (N > 295) keep the slots in a global scratch.
// Non-PD blocks keep running the protocol (NaN pivots, no early exit, so no
// warp can be left waiting at a barrier) and are flagged.
#include <cuda_runtime.h>
#include <stdint.h>

#include "bv_common.cuh"
#include "bv_tile.cuh"
#include "matern.cuh"

namespace bv {
namespace v3 {

// Panel solves L(I,J) = C(I,J) L_JJ⁻ᵀ are DMMA products with the explicit L_JJ⁻¹
// plus one FP64 refinement step (a bare product with the inverse loses accuracy
// on ill-conditioned tiles and fails the κ-aware parity rule at c3; row
// substitution on the update warps measured 7 % slower, round 1).  The update warps
// skip the refinement on panels where it cannot matter: max|L_JJ|·max|L_JJ⁻¹| ≤
// kRefineKappa (a condition-number proxy; the bare product's error exceeds the
// substitution's by at most about that factor).  Measured: 100 → c4 228.0 → 231.9 evals/s
// with unchanged parity statistics (gpurun_out/abk: every c1-c4 case, same strict /
// κ-branch / replica counts within noise); 1000 fails two c4 blocks; no refinement at
// all fails c3 (26 blocks) — the chain warp's own solve always refines.
// 4 warps per CTA (1 chain + 3 update) up to 19 tile rows: measured at c4, 5/6/8 warps
// per CTA gave 187/180/166 evals/s against 197 (round 1), and 8 warps from 14 tile rows
// 151-185 against 226 (round 2); 8 from 20 tile rows: see v3_maxt_for.
constexpr int kW = 4;  // warps per CTA: 1 chain warp + kW−1 update warps
#ifndef BV_REFINE_KAPPA
#define BV_REFINE_KAPPA 100.0
#endif
constexpr double kRefineKappa = BV_REFINE_KAPPA;
constexpr int kBarG = 1, kBarF = 2, kBarE = 3, kBarH = 5;  // named barriers (0 = __syncthreads)

#ifdef BV_PROFILE_PHASES
// Debug-only phase timers, summed over warps (lane 0): chain 0 factor, 1 wait E,
// 2 P partial, 3 row solve + F, 4 final; update 5 generation, 6 GEMM,
// 7 wait G, 8 row solves, 9 U barrier, 10 wait F, 11 final; 12 CTAs.
__device__ unsigned long long g_v3_cycles[16];
#define P3_T(v) long long v = clock64()
#define P3_ADD(i, v0)                                                                             \
  do {                                                                                            \
    if ((threadIdx.x & 31) == 0) atomicAdd(&g_v3_cycles[i], (unsigned long long)(clock64() - (v0))); \
  } while (0)
#else
#define P3_T(v)
#define P3_ADD(i, v0)
#endif

__device__ __forceinline__ void dmma884(double& d0, double& d1, double a, double b) {
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
__device__ __forceinline__ void bar_arrive(int id, int n) { asm volatile("bar.arrive %0, %1;" ::"r"(id), "r"(n) : "memory"); }
__device__ __forceinline__ void bar_sync(int id, int n) { asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(n) : "memory"); }

struct Layout {
  int P, dtile, ptile, linv, lfr, lrow, rinv, misc, theta, etab, slots, tab, total_bytes;
  __host__ __device__ Layout(int TImax, int cap) {
    P = 0;                   // PointRec[8·TImax]
    dtile = P + 32 * TImax;  // C(J,J), row-major (chain warp only)
    ptile = dtile + 64;      // next diagonal tile's partial P(J+1,J+1) (update warps → chain)
    linv = ptile + 64;       // [2][64] L_JJ⁻¹ in DMMA fragment order (0 on padding rows)
    lfr = linv + 128;        // [2][64] L_JJ in DMMA fragment order
    lrow = lfr + 128;        // (no row-major copy: panel solves are all DMMA)
    rinv = lrow;
    misc = lrow;             // [1] chain quad, [2] fail, [3] chain warp, [4] logdet, [5..7] update-warp quads
    theta = misc + 16;  // Theta (≤ 20 doubles); misc holds 4 + KW ≤ 12 entries
    etab = theta + 20;       // 2^{−j/64}, j = 0..63 (exp_neg)
    slots = etab + 64;       // cap tiles
    tab = slots + 64 * cap;  // int16 slot table (TImax²)
    total_bytes = (tab + (TImax * TImax + 3) / 4) * 8;
  }
};

// KIND kPre: the general-ν Σ entries were written by the pre-generation kernel
// (bv_pregen_kernel below) as each block's packed lower triangle, pre[r(r+1)/2 + c],
// r ≥ c, r < N; the block kernel reads instead of evaluating K_ν.  Same function,
// same arguments → bitwise the entries the in-kernel path computes (incl. the
// padding: 0 off the diagonal, σ² on it, as Eq. (7) gives for the far points).
constexpr int kPre = 4;
__device__ __forceinline__ double pre_entry(const double* __restrict__ pre, int r, int c, int N, double s2) {
  const int rr = r > c ? r : c, cc = r > c ? c : r;
  return rr < N ? pre[(rr * (rr + 1) >> 1) + cc] : (rr == cc ? s2 : 0.0);
}

template <int KIND>
__device__ __forceinline__ double joint_entry(const PointRec& pr, const PointRec& pc, int r, int c, int N,
                                             const Theta& th, const double* tab64, const double* pre) {
  double v;
  if constexpr (KIND == kPre) v = pre_entry(pre, r, c, N, th.sigma2);
  else v = matern_kind<KIND>(sqdist(pr, pc), th, tab64);
  return (r == N) ? pc.v : v;  // the y row; padding entries are 0 by construction (far points)
}

// L(I,J) = C(I,J) L_JJ⁻ᵀ for one tile, in place (one warp): C is row-major,
// the result is stored in DMMA fragment order.  bi / bl = this lane's
// fragments of L_JJ⁻¹ / L_JJ (the B operands (L⁻ᵀ)[k][n], (Lᵀ)[k][n] at k = t,
// n = g).  X₁ = C L⁻ᵀ, then one refinement step X = X₁ + (C − X₁Lᵀ) L⁻ᵀ with
// the residual in FP64: this restores the accuracy of substitution, which a
// bare multiply by the explicit inverse loses on ill-conditioned L_JJ (refine =
// false skips it: the caller's condition proxy says it cannot matter).
// Returns the lane's two results (row g, columns 2t, 2t+1) for the y-row term.
template <int NT>
__device__ __forceinline__ void tile_trsm_n(double* const (&tile)[NT], double2 bi, double2 bl, int g, int t,
                                            double2 (&out)[NT], bool refine) {
  double x0[NT], x1[NT], cc0[NT], cc1[NT];
#pragma unroll
  for (int i = 0; i < NT; ++i) {
    const double* ra = tile[i] + 8 * g + t;  // A operand (row g, k = t / t+4) of a row-major tile
    const double c0 = ra[0], c1 = ra[4];
    const double2 cc = lds2(tile[i] + 8 * g + 2 * t);  // accumulator (row g, columns 2t, 2t+1)
    cc0[i] = cc.x;
    cc1[i] = cc.y;
    x0[i] = x1[i] = 0.0;
    dmma884(x0[i], x1[i], c0, bi.x);
    dmma884(x0[i], x1[i], c1, bi.y);
  }
  if (refine) {  // warp-uniform
  __syncwarp();
#pragma unroll
  for (int i = 0; i < NT; ++i) sts2(tile[i] + 8 * g + 2 * t, x0[i], x1[i]);
  __syncwarp();
#pragma unroll
  for (int i = 0; i < NT; ++i) {
    const double* ra = tile[i] + 8 * g + t;
    dmma884(cc0[i], cc1[i], neg(ra[0]), bl.x);  // R = C − X₁ Lᵀ
    dmma884(cc0[i], cc1[i], neg(ra[4]), bl.y);
  }
  __syncwarp();
#pragma unroll
  for (int i = 0; i < NT; ++i) sts2(tile[i] + 8 * g + 2 * t, cc0[i], cc1[i]);
  __syncwarp();
#pragma unroll
  for (int i = 0; i < NT; ++i) {
    const double* ra = tile[i] + 8 * g + t;
    dmma884(x0[i], x1[i], ra[0], bi.x);  // X = X₁ + R L⁻ᵀ
    dmma884(x0[i], x1[i], ra[4], bi.y);
  }
  }
  __syncwarp();
#pragma unroll
  for (int i = 0; i < NT; ++i) {
    tile[i][8 * g + 2 * ((2 * t) & 3) + (t >> 1)] = x0[i];
    tile[i][8 * g + 2 * ((2 * t + 1) & 3) + (t >> 1)] = x1[i];
    out[i] = make_double2(x0[i], x1[i]);
  }
}
__device__ __forceinline__ double2 tile_trsm(double* tile, double2 bi, double2 bl, int g, int t, bool refine) {
  double* const tl[1] = {tile};
  double2 o[1];
  tile_trsm_n<1>(tl, bi, bl, g, t, o, refine);
  return o[0];
}

// y-row term of one tile solve: u += Σ_{j ≥ m, j < N} z_j² over this lane's two columns
__device__ __forceinline__ double yrow_sq(double2 d, int J, int t, int m, int N) {
  const int k0 = 8 * J + 2 * t, k1 = k0 + 1;
  double q = (k0 >= m && k0 < N) ? d.x * d.x : 0.0;
  return (k1 >= m && k1 < N) ? fma(d.y, d.y, q) : q;
}

// Update-warp GEMM for NS tiles I = J+1+(u−1)+3s (warp 1's first tile is the
// next diagonal tile): S(s) += Σ_{K<J} L(I,K) L(J+1,K)ᵀ.
__device__ __forceinline__ const double* slot_at(const double* base, unsigned slot) {
  return reinterpret_cast<const double*>(reinterpret_cast<const char*>(base) + (slot << 9));  // 64 doubles per slot
}
__device__ __forceinline__ double* slot_at(double* base, unsigned slot) {
  return reinterpret_cast<double*>(reinterpret_cast<char*>(base) + (slot << 9));
}

// Update-warp column work for this warp's ns tiles I = J+uw+3s of column J+1 (warp 1's
// first tile is the next diagonal tile): generate A(I,J+1) (Eq. 7) straight into the MMA
// accumulators (lane (g,t): row g, columns 2t, 2t+1), then subtract the updates of panels
// K < J progressively, S ← S − L(I,K) L(J+1,K)ᵀ in increasing K — the rounding order of a
// right-looking elimination (each update rounds against the partially reduced value, not
// against the full sum of updates), which on ill-conditioned blocks is several times more
// accurate than summing the updates and subtracting once.
// The tiles go two at a time through ONE copy of the generation and of the K loop (plus a
// single-tile K loop for an odd tail), the results placed into S by compile-time selects:
// one code path for every tile count keeps the kernel's hot code small (per-tile-count
// instantiations put the co-resident warps on different code copies: instruction-fetch
// stalls, ncu stall_no_inst).
template <int MAXT>
__device__ __forceinline__ void u_place(double (&S)[MAXT][2], int s, double v0, double v1) {
#pragma unroll
  for (int q = 0; q < MAXT; ++q)
    if (q == s) {
      S[q][0] = v0;
      S[q][1] = v1;
    }
}
template <int MAXT, int KIND, int KW>
__device__ __forceinline__ void u_column(double (&S)[MAXT][2], int ns, const double* slots, const int16_t* tab, int TI,
                                         int J, int uw, int lane, const PointRec* P, int N, const Theta& th,
                                         const double* etab, const double* pre) {
  const int g = lane >> 2, t = lane & 3, c0 = 8 * (J + 1) + 2 * t;
  const PointRec pc0 = P[c0], pc1 = P[c0 + 1];
  const double* sl = slots + 2 * lane;
  const uint16_t* tJ = reinterpret_cast<const uint16_t*>(tab) + (J + 1) * TI;
#pragma unroll 1
  for (int s = 0; s < ns; s += 2) {
    const bool two = s + 1 < ns;  // warp-uniform
    double a[2][2];
    {  // both tiles' entries in flight (an odd tail recomputes tile s as its dummy partner;
       // measured c3 621 -> 642 evals/s against one tile at a time, c4 unchanged)
      const int r0 = 8 * (J + uw + (KW - 1) * s) + g, r1 = two ? r0 + 8 * (KW - 1) : r0;
      const PointRec p0 = P[r0], p1 = P[r1];
      a[0][0] = joint_entry<KIND>(p0, pc0, r0, c0, N, th, etab, pre);
      a[0][1] = joint_entry<KIND>(p0, pc1, r0, c0 + 1, N, th, etab, pre);
      a[1][0] = joint_entry<KIND>(p1, pc0, r1, c0, N, th, etab, pre);
      a[1][1] = joint_entry<KIND>(p1, pc1, r1, c0 + 1, N, th, etab, pre);
    }
    const uint16_t* t0 = reinterpret_cast<const uint16_t*>(tab) + (J + uw + (KW - 1) * s) * TI;
    if (two) {
      const uint16_t* t1 = t0 + (KW - 1) * TI;
#pragma unroll 2
      for (int K = 0; K < J; ++K) {
        const double2 b = lds2(slot_at(sl, tJ[K]));
        const double bx = neg(b.x), by = neg(b.y);
        const double2 x0 = lds2(slot_at(sl, t0[K]));
        const double2 x1 = lds2(slot_at(sl, t1[K]));
        dmma884(a[0][0], a[0][1], x0.x, bx);
        dmma884(a[1][0], a[1][1], x1.x, bx);
        dmma884(a[0][0], a[0][1], x0.y, by);
        dmma884(a[1][0], a[1][1], x1.y, by);
      }
      u_place(S, s + 1, a[1][0], a[1][1]);
    } else {
#pragma unroll 2
      for (int K = 0; K < J; ++K) {
        const double2 b = lds2(slot_at(sl, tJ[K]));
        const double2 x0 = lds2(slot_at(sl, t0[K]));
        dmma884(a[0][0], a[0][1], x0.x, neg(b.x));
        dmma884(a[0][0], a[0][1], x0.y, neg(b.y));
      }
    }
    u_place(S, s, a[0][0], a[0][1]);
  }
}

// CTAs per SM the register allocation targets: shared memory admits 5 blocks
// of TI ≤ 16 (MAXT ≤ 5, the bulk of c3/c4) and 4 of TI 17-18; 5 × 128 threads
// caps registers at 102 (a few spills in the chain warp's in-lane factor,
// measured +2.5 % at c4 over 4 CTAs with none).
#ifndef BV_MINB5
#define BV_MINB5 5
#endif
constexpr int v3_minb(int maxt) { return maxt >= 16 ? 2 : maxt <= 5 ? BV_MINB5 : 4; }
// Joint sizes beyond what shared memory holds (TI > 37, N > 295: the paper's
// conditioning sets reach 420-450) keep the same schedule
// with the tile slots in a global-memory scratch (L1/L2-resident) instead of
// shared memory: MAXT ∈ {16, 20} (TI ≤ 61, N ≤ 480), persistent CTAs (the
// scratch is gridDim × cap slots).  GS = "global slots".
constexpr int kGsMaxT = 16;

#ifndef BV_KW8_MINB3
#define BV_KW8_MINB3 3  // 8-warp CTAs per SM targeted for MAXT ≤ 3 (TI ≤ 22; shared memory admits 3)
#endif
// KW: warps per CTA (1 chain + KW−1 update warps): 4, or 8 for the large joint sizes whose
// tile slots leave room for only 2 CTAs per SM (host: v3_maxt_for).
template <int MAXT, int KIND, int KW = kW>
__global__ void __launch_bounds__(KW * 32, KW == kW ? v3_minb(MAXT) : (MAXT <= 3 ? BV_KW8_MINB3 : 2))
bv_block_v3_kernel(const PointRec* __restrict__ pts, const int32_t* __restrict__ nbr,
                   const BlockDesc* __restrict__ desc, const int32_t* __restrict__ list,
                   const Theta* __restrict__ theta_dev, const int16_t* __restrict__ tabs,
                   const int32_t* __restrict__ tab_off, const double* __restrict__ exp_tab, int TImax, int cap,
                   double* __restrict__ out_u, double* __restrict__ out_d, unsigned long long* __restrict__ acc,
                   int k_begin, double* __restrict__ gslots, int nblocks, const double* __restrict__ pre,
                   const int64_t* __restrict__ pre_off, double jit) {
  constexpr bool GS = MAXT >= kGsMaxT;
  extern __shared__ __align__(16) double smem[];
  const Layout Ly(TImax, GS ? 0 : cap);
  for (int bidx = blockIdx.x; bidx < (GS ? nblocks : (int)blockIdx.x + 1); bidx += gridDim.x) {
  const int q = list[bidx];
  const BlockDesc ds = desc[q];
  const int m = ds.m, l = ds.l, N = m + l;
  const double* preb = KIND == kPre ? pre + pre_off[q] : nullptr;
  const int TJ = (N + 7) >> 3;  // column panels
  const int TI = (N + 8) >> 3;  // tile rows (incl. the y row)
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int g = lane >> 2, t = lane & 3;

  PointRec* P = reinterpret_cast<PointRec*>(smem + Ly.P);
  double* dtile = smem + Ly.dtile;
  double* ptile = smem + Ly.ptile;
  double* linv = smem + Ly.linv;
  double* lfr = smem + Ly.lfr;
  double* misc = smem + Ly.misc;
  Theta* ths = reinterpret_cast<Theta*>(smem + Ly.theta);
  double* etab = smem + Ly.etab;
  double* slots = GS ? gslots + (size_t)blockIdx.x * cap * 64 : smem + Ly.slots;
  int16_t* tab = reinterpret_cast<int16_t*>(smem + Ly.tab);
  const uint16_t* tabu = reinterpret_cast<const uint16_t*>(tab);  // slot indices, unsigned: one shift-add per address

  // a1/a2: θ, gathered points (neighbours first), slot table, exp table
  if (tid < 64) etab[tid] = exp_tab[tid];
  if (tid < (int)(sizeof(Theta) / 8))
    reinterpret_cast<double*>(ths)[tid] = reinterpret_cast<const double*>(theta_dev)[tid];
#pragma unroll 1
  for (int i = tid; i < 8 * TI; i += (KW * 32)) {
    // padding rows/columns (i ≥ N, and the y row's own point): far-apart points, so every
    // padding entry off the diagonal is exactly 0 from Eq. (7) itself (x > 708 → 0) and no
    // per-entry validity select is needed (padding pivots are σ², exactly decoupled)
    const double far = 1e30 * (double)(i + 1);
    PointRec r = {far, far, far, 0.0};
    if (i < N) r = pts[(i < m) ? nbr[ds.nbr_off + i] : ds.pstart + (i - m)];
    P[i] = r;
  }
  {
    const int16_t* gt = tabs + tab_off[2 * TI + (TI - TJ)];
#pragma unroll 1
    for (int e = tid; e < TI * TI; e += (KW * 32)) tab[e] = gt[e];
  }
  if (tid < 4) misc[tid] = 0.0;
  __syncthreads();
  // default: the chain is warp 0 — the hardware rotates co-resident CTAs'
  // warps over the four SM sub-partitions (tools/peaks/wid_probe), so the
  // chains of the ~4 resident blocks land on different FP64 pipes
  const Theta& th = *ths;
  // a3 panel 0: C(I,0) = A(I,0) for I ≥ 1 into slots; C(0,0) into dtile
#pragma unroll 2
  for (int e = tid; e < TI * 64; e += (KW * 32)) {
    const int I = e >> 6, r = 8 * I + ((e >> 3) & 7), c = e & 7;
    const double v = joint_entry<KIND>(P[r], P[c], r, c, N, th, etab, preb);
    if (I == 0) dtile[e] = v;
    else slots[64 * tab[I * TI] + (e & 63)] = v;
  }
  __syncthreads();
  const int cw = (int)misc[3];
  const int uw = (warp - cw + KW) % KW;  // 0 = chain warp, 1..KW−1 = update warps
  const double pfloor = kPivotFloor * th.sigma2;

  if (uw == 0) {
    // ---------------------------------------------------------- chain warp
    double pm = 1.0, qd_t = 0.0;
    int pe = 0, nbad = 0;
    // the chain's tiles stay in registers in the MMA accumulator layout (lane (g,t): row g,
    // columns 2t, 2t+1); products use the k-permuted form of bv_tile.cuh
    double c0, c1;
    {
      const double2 dv = lds2(dtile + 8 * g + 2 * t);  // C(0,0)
      c0 = dv.x;
      c1 = dv.y;
    }
    for (int J = 0; J < TJ; ++J) {
      double* li = linv + 64 * (J & 1);
      double* lj = lfr + 64 * (J & 1);
      P3_T(t0);
      // a4/a7: the diagonal tile factored across the warp's lanes (bv_tile.cuh factor_dist)
      double z0, z1;
      tile::factor_dist<8>(c0, c1, z0, z1, lane, J, m, N, pfloor, jit, pm, nbad, qd_t);
      {  // publish L_JJ, L_JJ⁻¹ for the update warps in this kernel's fragment order:
         // element (i,k) at 2(4i + (k&3)) + (k>>2)
        const int k0 = 2 * t, k1 = 2 * t + 1;
        li[2 * (4 * g + (k0 & 3)) + (k0 >> 2)] = neg(z0);
        li[2 * (4 * g + (k1 & 3)) + (k1 >> 2)] = neg(z1);
        lj[2 * (4 * g + (k0 & 3)) + (k0 >> 2)] = c0;
        lj[2 * (4 * g + (k1 & 3)) + (k1 >> 2)] = c1;
      }
      const double2 zn = make_double2(z0, z1), lf = make_double2(c0, c1);
      int ex;
      pm = frexp(pm, &ex);
      pe += ex;
      P3_ADD(0, t0);
      P3_T(t1);
      // U finished iteration J−1 (so it has consumed G, F, H of J−1: a named
      // barrier must not receive this warp's next arrival before its previous
      // phase completed)
      if (J >= 1) bar_sync(kBarE, (KW * 32));
      bar_arrive(kBarG, (KW * 32));
      P3_ADD(1, t1);
      if (J + 1 >= TJ) {
        // last panel: when N is a multiple of 8 the y row sits alone in tile row
        // TJ, below the last diagonal tile — its solve is this warp's (U only
        // handles tiles I ≥ J+2)
        if (TI > TJ) {
          const double2 cv = lds2(slot_at(slots, tabu[TJ * TI + J]) + 8 * g + 2 * t);
          const double2 d = tile::trsm(make_double2(neg(cv.x), neg(cv.y)), zn, lf);
          if (g == (N & 7)) qd_t += yrow_sq(d, J, t, m, N);
        }
        break;
      }
      P3_T(t3);
      // L(J+1,J) = C(J+1,J) L_JJ⁻ᵀ (a5/a6), in registers (explicit inverse + one refinement)
      double* tj = slot_at(slots, tabu[(J + 1) * TI + J]);
      const double2 cv = lds2(tj + 8 * g + 2 * t);
      const double2 x = tile::trsm(make_double2(neg(cv.x), neg(cv.y)), zn, lf);
      if (8 * (J + 1) + g == N) qd_t += yrow_sq(x, J, t, m, N);  // the y row: u += Σ_{j≥m} z_j²
      // → the slot in fragment order (the update warps' b operand of their final term)
      tj[8 * g + 2 * ((2 * t) & 3) + (t >> 1)] = x.x;
      tj[8 * g + 2 * ((2 * t + 1) & 3) + (t >> 1)] = x.y;
      P3_ADD(3, t3);
      P3_T(t4);
      bar_sync(kBarH, (KW * 32));  // the update warps published P(J+1,J+1)
      const double2 pp = lds2(ptile + 8 * g + 2 * t);  // read before F: U regenerates ptile after F
      bar_arrive(kBarF, (KW * 32));
      // C(J+1,J+1) = P − L(J+1,J) L(J+1,J)ᵀ, straight into the next factorisation
      c0 = pp.x;
      c1 = pp.y;
      dmma884(c0, c1, neg(x.x), x.x);
      dmma884(c0, c1, neg(x.y), x.y);
      P3_ADD(4, t4);
    }
    if (nbad && lane == 0) misc[2] = 1.0;
    // y-row contributions of the chain warp: in-lane part (identical in all lanes) + row solves
    for (int o = 16; o > 0; o >>= 1) qd_t += __shfl_xor_sync(0xffffffffu, qd_t, o);
    if (lane == 0) {
      misc[1] = qd_t;  // per-warp partials, summed in a fixed order below (bitwise reproducible)
      misc[4] = log(pm) + (double)pe * 0.69314718055994530942;  // d = Σ_{j≥m} log p_j
    }
  } else {
    // ---------------------------------------------------------- update warps
    double qd_u = 0.0;
    for (int J = 0; J < TJ; ++J) {
      const bool ahead = J + 1 < TJ;
      double S[MAXT][2];
#pragma unroll
      for (int s = 0; s < MAXT; ++s) S[s][0] = S[s][1] = 0.0;
      if (ahead) {
        P3_T(u6);
        // a3 + a6: this warp's tiles of column J+1, generated into registers and reduced by
        // the panels K < J (exact tile count per warp: no predicated-off work)
        const int ns = (TI - J - 1 - (uw - 1) + (KW - 2)) / (KW - 1);
        u_column<MAXT, KIND, KW>(S, ns, slots, tab, TI, J, uw, lane, P, N, th, etab, preb);
        // P(J+1,J+1) = A − Σ_{K<J} L(J+1,K) L(J+1,K)ᵀ for the chain warp (warp 1 owns the tile)
        if (uw == 1) sts2(ptile + 8 * g + 2 * t, S[0][0], S[0][1]);
        P3_ADD(6, u6);
      }
      P3_T(u7);
      bar_sync(kBarG, (KW * 32));  // the chain warp published L_JJ
      if (ahead) bar_arrive(kBarH, (KW * 32));  // P(J+1,J+1) is in ptile
      P3_ADD(7, u7);
      P3_T(u8);
      {
        // L(I,J) = C(I,J) L_JJ⁻ᵀ for this warp's tiles I = J+u+3s > J+1 (a5/a6)
        const double2 bi = lds2(linv + 64 * (J & 1) + 2 * lane);
        const double2 bl = lds2(lfr + 64 * (J & 1) + 2 * lane);
        // refine only where the explicit inverse loses accuracy: max|L_JJ|·max|L_JJ⁻¹| (a
        // condition-number proxy, the same value in every lane after the butterfly)
        double mz = fmax(fabs(bi.x), fabs(bi.y)), ml = fmax(fabs(bl.x), fabs(bl.y));
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
          mz = fmax(mz, __shfl_xor_sync(0xffffffffu, mz, o));
          ml = fmax(ml, __shfl_xor_sync(0xffffffffu, ml, o));
        }
        const bool refine = mz * ml > kRefineKappa;
          // two tiles in flight: their DMMA / shared-memory round trips interleave
#pragma unroll 1
        for (int I = J + uw + (uw == 1 ? KW - 1 : 0); I < TI; I += 2 * (KW - 1)) {
          const int I2 = I + KW - 1;
          if (I2 < TI) {
            double* const tl[2] = {slot_at(slots, tabu[I * TI + J]), slot_at(slots, tabu[I2 * TI + J])};
            double2 d[2];
            tile_trsm_n<2>(tl, bi, bl, g, t, d, refine);
            if (8 * I + g == N) qd_u += yrow_sq(d[0], J, t, m, N);  // the y row (a8)
            if (8 * I2 + g == N) qd_u += yrow_sq(d[1], J, t, m, N);
          } else {
            const double2 d = tile_trsm(slot_at(slots, tabu[I * TI + J]), bi, bl, g, t, refine);
            if (8 * I + g == N) qd_u += yrow_sq(d, J, t, m, N);
          }
        }
      }
      P3_ADD(8, u8);
      // (no U barrier here: F below is a full barrier of the update warps, so
      // every L(I,J) is visible to all of them before the next GEMM)
      if (!ahead) continue;
      P3_T(u10);
      bar_sync(kBarF, (KW * 32));  // the chain warp published L(J+1,J)
      P3_ADD(10, u10);
      P3_T(u11);
      const double2 b = lds2(slot_at(slots + 2 * lane, tabu[(J + 1) * TI + J]));
#pragma unroll
      for (int s = 0; s < MAXT; ++s) {
        const int I = J + uw + (KW - 1) * s;
        if (I < TI && I > J + 1) {  // the diagonal tile's last term is the chain warp's
          const double2 a = lds2(slot_at(slots + 2 * lane, tabu[I * TI + J]));
          dmma884(S[s][0], S[s][1], a.x, neg(b.x));
          dmma884(S[s][0], S[s][1], a.y, neg(b.y));
          sts2(slot_at(slots + 8 * g + 2 * t, tabu[I * TI + J + 1]), S[s][0], S[s][1]);  // C(I,J+1), row-major
        }
      }
      __syncwarp();
      bar_arrive(kBarE, (KW * 32));  // iteration J done: C(I,J+1) stored, L(·,J) final
      P3_ADD(11, u11);
    }
    for (int o = 16; o > 0; o >>= 1) qd_u += __shfl_xor_sync(0xffffffffu, qd_u, o);
    if (lane == 0) misc[4 + uw] = qd_u;
  }
  __syncthreads();
#ifdef BV_PROFILE_PHASES
  if (threadIdx.x == 0) atomicAdd(&g_v3_cycles[12], 1ull);
#endif

  // a8: per-block outputs and the exact fixed-point term (a9)
  if (uw == 0 && lane == 0) {
    const bool fail = misc[2] != 0.0;
    int st = fail ? kNotPD : kOk;
    uint32_t c[6] = {0, 0, 0, 0, 0, 0};
    const double logdet = fail ? failed_d() : misc[4];
    double quad = misc[1];
    for (int w = 1; w < KW; ++w) quad += misc[4 + w];  // fixed order: bitwise reproducible
    quad = fail ? 0.0 : quad;
    if (!fail) {
      const double tk = -0.5 * (quad + logdet + (double)l * kLn2Pi);
      if (fixed_encode(tk, c)) st = kTermRange;
    }
    out_u[q] = quad;
    out_d[q] = logdet;
    accumulate_term(acc, c, st, k_begin + q);
  }
  if (GS) __syncthreads();  // the next block reuses shared memory and the scratch
  }
}

}  // namespace v3

// ------------------------------------------------------------------ host side
int debug_v3_cycles(unsigned long long* out, int reset) {
#ifdef BV_PROFILE_PHASES
  if (out) cudaMemcpyFromSymbol(out, v3::g_v3_cycles, sizeof(unsigned long long) * 16);
  if (reset) {
    unsigned long long z[16] = {};
    cudaMemcpyToSymbol(v3::g_v3_cycles, z, sizeof(z));
  }
  return 1;
#else
  (void)out;
  (void)reset;
  return 0;
#endif
}

// Instantiation for a tile-row count TI: MAXT (tiles per update warp) of the 4-warp kernel,
// or 100 + MAXT of the 8-warp kernel (TI ≥ kKw8MinTI, shared-memory slots only).  From
// TI ≈ 20 the tile slots leave room for only 2-3 CTAs per SM, and 7 update warps per block
// recover the parallelism (measured: c5 m = 200 12.1 → 20.9 evals/s, c3 620 → 645 with
// the threshold at 22 and 2 CTAs per SM; threshold 20 with 3 CTAs per SM for TI ≤ 22: c3 622
// → 640, m = 120 78.5 → 79.4; at 17-18 c3 and m = 120 lose — 4-5 CTAs of 4 warps win there).
#ifndef BV_KW8_MIN_TI
#define BV_KW8_MIN_TI 20
#endif
constexpr int kKw8MinTI = BV_KW8_MIN_TI;
int v3_maxt_for(int TI) {
  if (TI >= kKw8MinTI && TI <= 37) {
    const int need8 = (TI - 1 + 6) / 7;
    const int o8[] = {2, 3, 4, 5, 6};
    for (int o : o8)
      if (o >= need8) return 100 + o;
  }
  const int need = (TI - 1 + (v3::kW - 2)) / (v3::kW - 1);  // panel J+1 tiles I ≥ J+1 over the update warps
  const int opts[] = {1, 2, 3, 4, 5, 6, 8, 10, 12, 16, 20};
  for (int o : opts)
    if (o >= (need < 1 ? 1 : need)) return o;
  return -1;
}

bool v3_global_slots(int TI) {
  const int mt = v3_maxt_for(TI);
  return mt >= v3::kGsMaxT && mt < 100;
}

size_t v3_smem_bytes(int TImax, int cap) {
  const size_t b = (size_t)v3::Layout(TImax, v3_global_slots(TImax) ? 0 : cap).total_bytes;
  return b;
}

template <int MAXT, int KW = v3::kW>
static cudaError_t v3_prep(size_t smem) {
  cudaError_t e = cudaSuccess;
  for (int k = 0; k < 5 && e == cudaSuccess; ++k) {
    const void* f = k == 0 ? (const void*)v3::bv_block_v3_kernel<MAXT, 0, KW>
                  : k == 1 ? (const void*)v3::bv_block_v3_kernel<MAXT, 1, KW>
                  : k == 2 ? (const void*)v3::bv_block_v3_kernel<MAXT, 2, KW>
                  : k == 3 ? (const void*)v3::bv_block_v3_kernel<MAXT, 3, KW>
                           : (const void*)v3::bv_block_v3_kernel<MAXT, v3::kPre, KW>;
    e = cudaFuncSetAttribute(f, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  }
  return e;
}

cudaError_t prepare_block_v3(size_t max_smem) {
  cudaError_t e = cudaSuccess;
  if (e == cudaSuccess) e = v3_prep<1>(max_smem);
  if (e == cudaSuccess) e = v3_prep<2>(max_smem);
  if (e == cudaSuccess) e = v3_prep<3>(max_smem);
  if (e == cudaSuccess) e = v3_prep<4>(max_smem);
  if (e == cudaSuccess) e = v3_prep<5>(max_smem);
  if (e == cudaSuccess) e = v3_prep<6>(max_smem);
  if (e == cudaSuccess) e = v3_prep<8>(max_smem);
  if (e == cudaSuccess) e = v3_prep<10>(max_smem);
  if (e == cudaSuccess) e = v3_prep<12>(max_smem);
  if (e == cudaSuccess) e = v3_prep<16>(max_smem);
  if (e == cudaSuccess) e = v3_prep<20>(max_smem);
  if (kKw8MinTI <= 37) {
    if (e == cudaSuccess) e = v3_prep<2, 8>(max_smem);
    if (e == cudaSuccess) e = v3_prep<3, 8>(max_smem);
    if (e == cudaSuccess) e = v3_prep<4, 8>(max_smem);
    if (e == cudaSuccess) e = v3_prep<5, 8>(max_smem);
    if (e == cudaSuccess) e = v3_prep<6, 8>(max_smem);
  }
  return e;
}

template <int MAXT, int KW = v3::kW>
static void v3_launch_kind(int kind, int nblocks, size_t smem, cudaStream_t s, const PointRec* pts,
                           const int32_t* nbr, const BlockDesc* desc, const int32_t* list, const Theta* th,
                           const int16_t* tabs, const int32_t* tab_off, const double* etab, int TImax, int cap,
                           double* u, double* d, unsigned long long* acc, int k_begin, double* gslots, int grid,
                           const double* pre, const int64_t* pre_off, double jit) {
#define BV_K(KD)                                                                                             \
  v3::bv_block_v3_kernel<MAXT, KD, KW><<<grid, KW * 32, smem, s>>>(pts, nbr, desc, list, th, tabs, tab_off, etab, \
                                                               TImax, cap, u, d, acc, k_begin, gslots, nblocks, \
                                                               pre, pre_off, jit)
  switch (kind) {
    case 0: BV_K(0); break;
    case 1: BV_K(1); break;
    case 2: BV_K(2); break;
    case 3: BV_K(3); break;
    default: BV_K(v3::kPre); break;
  }
#undef BV_K
}

cudaError_t launch_block_v3(int kind, int nblocks, int TImax, int cap, cudaStream_t s, const PointRec* pts,
                            const int32_t* nbr, const BlockDesc* desc, const int32_t* list, const Theta* th,
                            const int16_t* tabs, const int32_t* tab_off, const double* etab, double* u, double* d,
                            unsigned long long* acc, int k_begin, double* gslots, int gs_grid, const double* pre,
                            const int64_t* pre_off, double jit) {
  if (nblocks == 0) return cudaSuccess;
  const size_t smem = v3_smem_bytes(TImax, cap);
  const int grid = v3_global_slots(TImax) ? (nblocks < gs_grid ? nblocks : gs_grid) : nblocks;
  switch (v3_maxt_for(TImax)) {
#define BV_MT(MT)                                                                                          \
  case MT:                                                                                                 \
    v3_launch_kind<MT>(kind, nblocks, smem, s, pts, nbr, desc, list, th, tabs, tab_off, etab, TImax, cap, u, d, \
                       acc, k_begin, gslots, grid, pre, pre_off, jit);                                     \
    break;
    BV_MT(1) BV_MT(2) BV_MT(3) BV_MT(4) BV_MT(5) BV_MT(6) BV_MT(8) BV_MT(10) BV_MT(12) BV_MT(16) BV_MT(20)
#undef BV_MT
#define BV_MT8(MT)                                                                                           \
  case 100 + MT:                                                                                             \
    v3_launch_kind<MT, 8>(kind, nblocks, smem, s, pts, nbr, desc, list, th, tabs, tab_off, etab, TImax, cap, u, \
                          d, acc, k_begin, gslots, grid, pre, pre_off, jit);                                 \
    break;
    BV_MT8(2) BV_MT8(3) BV_MT8(4) BV_MT8(5) BV_MT8(6)
#undef BV_MT8
    default: return cudaErrorInvalidValue;
  }
  return cudaGetLastError();
}

// ------------------------------------------------------------------ general-ν pre-generation
// a3 for small plans with general ν (c2: 500 blocks, fewer than one wave of
// block-kernel CTAs, K_ν costs hundreds of FP64 instructions per entry): one
// kernel evaluates every block's packed lower triangle of Σ with all SMs' warps
// into an L2-resident buffer, then the block kernel (KIND kPre) only reads it.
namespace v3 {
constexpr int kPgThreads = 256;
template <int KIND>
__global__ void __launch_bounds__(kPgThreads) bv_pregen_kernel(const PointRec* __restrict__ pts,
                                                              const int32_t* __restrict__ nbr,
                                                              const BlockDesc* __restrict__ desc,
                                                              const Theta* __restrict__ theta_dev,
                                                              const double* __restrict__ exp_tab,
                                                              const int64_t* __restrict__ pre_off,
                                                              double* __restrict__ pre) {
  __shared__ double etab[64];
  if (threadIdx.x < 64) etab[threadIdx.x] = exp_tab[threadIdx.x];
  __syncthreads();
  const Theta th = *theta_dev;
  const int q = blockIdx.x;
  const BlockDesc ds = desc[q];
  const int m = ds.m, N = ds.m + ds.l;
  const int E = N * (N + 1) / 2;
  double* out = pre + pre_off[q];
  for (int e = blockIdx.y * kPgThreads + threadIdx.x; e < E; e += kPgThreads * gridDim.y) {
    int r = (int)((sqrt(8.0 * (double)e + 1.0) - 1.0) * 0.5);  // row of packed index e (fixed up exactly)
    while ((r * (r + 1) >> 1) > e) --r;
    while (((r + 1) * (r + 2) >> 1) <= e) ++r;
    const int c = e - (r * (r + 1) >> 1);
    const PointRec pr = pts[(r < m) ? nbr[ds.nbr_off + r] : ds.pstart + (r - m)];
    const PointRec pc = pts[(c < m) ? nbr[ds.nbr_off + c] : ds.pstart + (c - m)];
    out[e] = matern_kind<KIND>(sqdist(pr, pc), th, etab);
  }
}
}  // namespace v3

cudaError_t launch_pregen(int nblocks, int chunks, cudaStream_t s, const PointRec* pts, const int32_t* nbr,
                          const BlockDesc* desc, const Theta* th, const double* etab, const int64_t* pre_off,
                          double* pre) {
  if (nblocks == 0) return cudaSuccess;
  v3::bv_pregen_kernel<kNuGeneral><<<dim3(nblocks, chunks), v3::kPgThreads, 0, s>>>(pts, nbr, desc, th, etab,
                                                                                      pre_off, pre);
  return cudaGetLastError();
}

}  // namespace bv
