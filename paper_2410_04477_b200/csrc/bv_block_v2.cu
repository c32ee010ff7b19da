// bv_block_v2.cu — the block kernel: left-looking 8×8-tiled joint Cholesky
// with FP64 tensor-core (DMMA m8n8k4) panel updates, one CTA per block.
//
// What it computes (per permuted position k; Alg. 1 l.10-29):
// the Cholesky factor of the augmented joint matrix
//        ⎡ Σcon    Σcross  y_NN ⎤      rows 0..m−1   : neighbours (given order)
//        ⎢ Σcrossᵀ Σlk     y_B  ⎥      rows m..N−1   : block points (ascending id)
//        ⎣ y_NNᵀ   y_Bᵀ    ·    ⎦      row  N        : observations (never a pivot)
// Its leading m×m factor is L = chol(Σcon) (l.17), its off-diagonal panel is
// Σ'crossᵀ = (L⁻¹Σcross)ᵀ (l.18), the trailing l×l factor is
// L' = chol(Σlk − Σ'crossᵀΣ'cross) (l.20-24), and row N holds
// [L⁻¹y_NN ; L'⁻¹(y_B − μnew)] (l.19, l.21, l.25).  Hence
//   d_k = 2 Σ_{j≥m} log L_jj = Σ_{j≥m} log p_j,   u_k = Σ_{j≥m} L_Nj²   (l.26-27).
//
// Design:
//  * tiles of 8×8; panel J = columns 8J..8J+7; rows up to N (the y row);
//  * left-looking: panel J's tiles C(I,J) = A(I,J) − Σ_{K<J} L(I,K) L(J,K)ᵀ, the
//    sum accumulated in registers by DMMA.8x8x4, A generated on the fly from
//    the gathered points (Matérn, Eq. 7) — the covariance never touches HBM;
//  * one warp per CTA factors the diagonal tiles (the block's serial pivot
//    chain); it is the warp that runs on SM sub-partition 0 (%warpid mod 4),
//    so the chains of all co-resident CTAs share one sub-partition while the
//    three update warps of every CTA fill the other three FP64 pipes with the
//    bulk (generation and DMMA) — no DMMA burst ever queues ahead of a pivot;
//  * rows below the diagonal are solved one row per thread (forward
//    substitution, not an explicit inverse), in place;
//  * each tile lives in one shared-memory slot from generation (C, row-major)
//    through the in-place solve (L, DMMA fragment order) to its last use;
//    slots are recycled by a per-(TI,TJ) table built once on the host
//    (bv_host.cpp: SlotTables) — at most ≈ T²/4 tiles are live;
//  * L tiles in fragment order: element (g, k) at 2·(4g + (k&3)) + (k>>2), so
//    one LDS.128 per lane yields both k-halves; a row keeps the same 64 bytes
//    in both layouts, which is what makes the solve in place.
#include <cuda_runtime.h>
#include <stdint.h>

#include "bv_common.cuh"
#include "matern.cuh"

namespace bv {

namespace {

constexpr int kW = 4;         // warps per CTA: 1 diagonal warp + 3 update warps
constexpr int kNT = kW * 32;  // threads per CTA
#ifndef BV_GEN_UNROLL
#define BV_GEN_UNROLL 4
#endif
constexpr int kGenUnroll = BV_GEN_UNROLL;  // Matérn entries in flight per thread

__device__ __forceinline__ void dmma884(double& d0, double& d1, double a, double b) {
  asm("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
      : "+d"(d0), "+d"(d1)
      : "d"(a), "d"(b));
}

__device__ __forceinline__ double2 lds2(const double* p) { return *reinterpret_cast<const double2*>(p); }
__device__ __forceinline__ void sts2(double* p, double a, double b) {
  *reinterpret_cast<double2*>(p) = make_double2(a, b);
}

// One 8-double row (64 bytes) of a tile, moved as four 16-byte chunks in a
// rotated order: thread row g touches chunk (k + g/2) mod 4 at step k, so the
// 8 rows of a tile hit 8 distinct bank groups (row stride 64 B would otherwise
// make even/odd rows collide 4-way).  Shared memory bandwidth is this
// kernel's scarcest resource.
__device__ __forceinline__ double2 sel4(const double2 (&v)[4], int i) {
  const double2 a = (i & 1) ? v[1] : v[0];
  const double2 b = (i & 1) ? v[3] : v[2];
  return (i & 2) ? b : a;
}
__device__ __forceinline__ void ld_row_rot(const double* row, int rot, double2 (&ch)[4]) {
  double2 t[4];
#pragma unroll
  for (int k = 0; k < 4; ++k) t[k] = lds2(row + 2 * ((k + rot) & 3));
#pragma unroll
  for (int q = 0; q < 4; ++q) ch[q] = sel4(t, (q - rot) & 3);  // chunk q was loaded at step (q − rot) mod 4
}
__device__ __forceinline__ void st_row_rot(double* row, int rot, const double2 (&ch)[4]) {
#pragma unroll
  for (int k = 0; k < 4; ++k) {
    const int q = (k + rot) & 3;
    const double2 v = sel4(ch, q);
    sts2(row + 2 * q, v.x, v.y);
  }
}

}  // namespace

#ifdef BV_PROFILE_PHASES
// Debug-only phase timers (cycles summed over CTAs): 0 prologue, 1 phase A
// (diag warp), 2 phase A (update warps), 3 sync after A, 4 phase B, 5 sync
// after B, 6 phase C + sync, 7 CTAs, 8 GEMM part of 2, 9 generation part of 2.
__device__ unsigned long long g_phase_cycles[10];
#define PH_T(v) long long v = clock64()
#define PH_ADD(i, v0)                                                                                   \
  do {                                                                                                  \
    if ((threadIdx.x & 31) == 0) atomicAdd(&g_phase_cycles[i], (unsigned long long)(clock64() - (v0))); \
  } while (0)
#else
#define PH_T(v)
#define PH_ADD(i, v0)
#endif

// Shared-memory carve-up (in doubles) for a bucket with at most TImax tile rows
// and `cap` tile slots.
struct V2Layout {
  int P, diag, rinv, misc, theta, etab, slots, tab, total_bytes;
  __host__ __device__ V2Layout(int TImax, int cap) {
    P = 0;                   // PointRec[8·TImax]
    diag = P + 32 * TImax;   // factored diagonal tile (row-major lower; diagonal = L_jj)
    rinv = diag + 64;        // 1/L_jj of the diagonal tile
    misc = rinv + 8;         // [0] logdet, [1] quad, [2] fail, [3] diagonal warp
    theta = misc + 8;        // Theta copy (16 doubles + ints → 20 doubles)
    etab = theta + 20;       // 2^{−j/64}, j = 0..63 (exp_neg table)
    slots = etab + 64;       // cap tiles
    tab = slots + 64 * cap;  // int16 slot table (TImax²), in doubles:
    total_bytes = (tab + (TImax * TImax + 3) / 4) * 8;
  }
};

// Covariance entry (r, c) of the augmented joint matrix (a3; Eq. 7): rows/cols
// < N are points, row N is the observation row, everything else is padding.
// Branch-free for the closed forms: every lane evaluates the covariance, then
// selects (P holds 8·TI zero-padded records, so the loads are in bounds).
template <int KIND>
__device__ __forceinline__ double joint_entry(const PointRec& pr, const PointRec& pc, int r, int c, int N,
                                             const Theta& th, const double* tab64) {
  double v = matern_kind<KIND>(sqdist(pr, pc), th, tab64);
  v = (r == N) ? pc.v : v;
  return (c >= N || r > N) ? 0.0 : v;
}

// One warp, in-lane (every lane holds the whole tile; no shuffles or memory
// in the pivot chain, ~55 cycles per pivot): Cholesky of the diagonal tile
// held row-major (lower part) in its slot.  Publishes L's strict lower part
// and 1/L_jj (0 on padding columns); accumulates, in the caller's registers,
// the product of the block pivots j ≥ m (for d, one log per block), the y
// row's Σ_{j≥m} L_Nj² when the y row sits inside this tile (for u), and the
// count of bad pivots (non-PD).
__device__ __forceinline__ void factor_diag_tile(const double* tile, double* diagL, double* rinv, int J, int m, int N,
                                                 int lane, double pfloor, double& prod, int& nbad, double& qd) {
  const int nreal = N - 8 * J;  // columns j < nreal are real pivots
  const int jm = m - 8 * J;     // columns j ≥ jm belong to the block (contribute to d)
  const int yr = N - 8 * J;     // the y row inside this tile (N not a multiple of 8)
  double a[8][8];
#pragma unroll
  for (int i = 0; i < 8; ++i)
#pragma unroll
    for (int k = 0; k <= i; ++k) a[i][k] = tile[8 * i + k];
#pragma unroll
  for (int j = 0; j < 8; ++j) {
    double p = a[j][j];
    // non-PD (reading G15): a pivot not above kPivotFloor·σ² — FP64-singular
    const bool ok = (p > pfloor) & (p <= 1.7976931348623157e308);
    const bool real = j < nreal;
    nbad += (real & !ok) ? 1 : 0;
    p = (real & ok) ? p : 1.0;
    prod *= (j >= jm) ? p : 1.0;
    const double r = rsqrt_pos(p);
    const double rv = real ? r : 0.0;
    const double lv = p * r;  // L_jj = √p (≤ 1 ulp)
    // L_ij = a_ij / L_jj: scale by r, then one residual correction so each
    // entry is rounded on its own (a systematic per-column scale error would be
    // amplified by the ill-conditioned Schur complements of late blocks)
#pragma unroll
    for (int i = j + 1; i < 8; ++i) {
      const double x = a[i][j] * rv;
      a[i][j] = fma(fma(-x, lv, a[i][j]), rv, x);
    }
#pragma unroll
    for (int i = j + 1; i < 8; ++i)
#pragma unroll
      for (int k = j + 1; k <= i; ++k) a[i][k] = fma(-a[i][j], a[k][j], a[i][k]);
    // column j is final: publish it now (frees its registers for the rest)
    if (lane == 0) {
#pragma unroll
      for (int i = j + 1; i < 8; ++i) diagL[8 * i + j] = a[i][j];
      diagL[9 * j] = lv;  // the diagonal slots hold L_jj
      rinv[j] = rv;
    }
  }
#pragma unroll
  for (int i = 1; i < 8; ++i)
    if (i == yr) {
#pragma unroll
      for (int k = 0; k < i; ++k)
        if (k >= jm) qd = fma(a[i][k], a[i][k], qd);
    }
}

// Panel update on the tensor cores for the NS tiles I = J+1+(u−1)+3s of update
// warp u: S(s) += Σ_{K<J} L(I,K) L(J+1,K)ᵀ, two DMMA.8x8x4 per (tile, K).
template <int NS, int MAXT>
__device__ __forceinline__ void panel_gemm(double (&S0)[MAXT][2], const double* slots, const int16_t* tab, int TI,
                                           int J, int uw, int lane) {
  const int16_t* tJ = tab + (J + 1) * TI;
  const int16_t* tI[NS];
#pragma unroll
  for (int s = 0; s < NS; ++s) tI[s] = tab + (J + uw + (kW - 1) * s) * TI;
#pragma unroll 2
  for (int K = 0; K < J; ++K) {
    const double2 b = lds2(slots + 64 * tJ[K] + 2 * lane);
#pragma unroll
    for (int s = 0; s < NS; ++s) {
      const double2 a = lds2(slots + 64 * tI[s][K] + 2 * lane);
      dmma884(S0[s][0], S0[s][1], a.x, b.x);
      dmma884(S0[s][0], S0[s][1], a.y, b.y);
    }
  }
}

// a3: generate the row-major tiles I = I0 .. TI−1 of column panel J into their
// slots: one thread per row r (8 entries, the 8 column points are the same for
// every thread — broadcast loads — so 8 independent Matérn chains are in
// flight per thread), each row stored with rotated 16-byte chunks.
#ifndef BV_GEN_ROWS
#define BV_GEN_ROWS 0
#endif
template <int KIND>
__device__ __forceinline__ void gen_tiles(const PointRec* P, int N, const Theta& th, const double* etab,
                                          double* slots, const int16_t* tab, int TI, int I0, int J, int thr, int nthr) {
#if BV_GEN_ROWS
  const int rows = (TI - I0) * 8;
#pragma unroll 1
  for (int rr = thr; rr < rows; rr += nthr) {
    const int I = I0 + (rr >> 3), g = rr & 7, r = 8 * I + g;
    const PointRec pr = P[r];
    double v[8];
#pragma unroll
    for (int k = 0; k < 8; ++k) {
      const int c = 8 * J + k;
      v[k] = joint_entry<KIND>(pr, P[c], r, c, N, th, etab);
    }
    const double2 ch[4] = {make_double2(v[0], v[1]), make_double2(v[2], v[3]), make_double2(v[4], v[5]),
                           make_double2(v[6], v[7])};
    st_row_rot(slots + 64 * tab[I * TI + J] + 8 * g, g >> 1, ch);
  }
#else
  // one entry per thread per step, kGenUnroll steps in flight; consecutive
  // threads take consecutive columns of a row (column points broadcast per row)
  const int total = (TI - I0) * 64;
#pragma unroll(kGenUnroll)
  for (int e = thr; e < total; e += nthr) {
    const int I = I0 + (e >> 6);
    const int r = 8 * I + ((e >> 3) & 7);
    const int c = 8 * J + (e & 7);
    slots[64 * tab[I * TI + J] + (e & 63)] = joint_entry<KIND>(P[r], P[c], r, c, N, th, etab);
  }
#endif
}

#ifndef BV_MINB
#define BV_MINB 4  // CTAs per SM the register allocation targets (4 × 128 threads → ≤ 128 registers)
#endif

template <int MAXT, int KIND>
__global__ void __launch_bounds__(kNT, BV_MINB)
bv_block_v2_kernel(const PointRec* __restrict__ pts, const int32_t* __restrict__ nbr,
                   const BlockDesc* __restrict__ desc, const int32_t* __restrict__ list,
                   const Theta* __restrict__ theta_dev, const int16_t* __restrict__ tabs,
                   const int32_t* __restrict__ tab_off, const double* __restrict__ exp_tab, int TImax, int cap,
                   double* __restrict__ out_u, double* __restrict__ out_d, unsigned long long* __restrict__ acc,
                   int k_begin) {
  extern __shared__ __align__(16) double smem[];
  const V2Layout Ly(TImax, cap);
  const int q = list[blockIdx.x];
  const BlockDesc ds = desc[q];
  const int m = ds.m, l = ds.l, N = m + l;
  const int TJ = (N + 7) >> 3;  // column panels (pivots 0..N−1)
  const int TI = (N + 8) >> 3;  // tile rows (rows 0..N, incl. the y row)
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int g = lane >> 2, t = lane & 3;

  PointRec* P = reinterpret_cast<PointRec*>(smem + Ly.P);
  double* diagL = smem + Ly.diag;
  double* rinv = smem + Ly.rinv;
  double* misc = smem + Ly.misc;
  Theta* ths = reinterpret_cast<Theta*>(smem + Ly.theta);
  double* slots = smem + Ly.slots;
  int16_t* tab = reinterpret_cast<int16_t*>(smem + Ly.tab);
  double* etab = smem + Ly.etab;

  // a1/a2: θ, gathered points (neighbours first), slot table, exp table
  if (tid < 64) etab[tid] = exp_tab[tid];
  if (tid < (int)(sizeof(Theta) / 8))
    reinterpret_cast<double*>(ths)[tid] = reinterpret_cast<const double*>(theta_dev)[tid];
#pragma unroll 1
  for (int i = tid; i < 8 * TI; i += kNT) {
    PointRec r = {0.0, 0.0, 0.0, 0.0};
    if (i < N) r = pts[(i < m) ? nbr[ds.nbr_off + i] : ds.pstart + (i - m)];
    P[i] = r;
  }
  {
    const int16_t* gt = tabs + tab_off[2 * TI + (TI - TJ)];
#pragma unroll 1
    for (int e = tid; e < TI * TI; e += kNT) tab[e] = gt[e];
  }
  if (tid < 4) misc[tid] = 0.0;
  __syncthreads();
  // The diagonal warp is the one on sub-partition 0 (a CTA's four warps sit on
  // the four sub-partitions); warp 0 if none reports it.
  {
    unsigned wid;
    asm volatile("mov.u32 %0, %%warpid;" : "=r"(wid));
    if (lane == 0 && (wid & 3u) == 0u) misc[3] = (double)warp;
  }
  __syncthreads();
  const int dwarp = (int)misc[3];
  const int uw = (warp - dwarp) & (kW - 1);  // 0 = diagonal warp, 1..3 = update warps
  const int utid = (uw - 1) * 32 + lane;     // 0..95 among the update warps
  const Theta& th = *ths;
  // diagonal-warp accumulators (registers, whole block): Π pivots as pm·2^pe,
  // y-row quadratic form inside diagonal tiles, bad-pivot count
  double pm = 1.0, qd = 0.0;
  int pe = 0, nbad = 0;
  PH_T(t_pro);

  // panel 0: C(I,0) = A(I,0) (nothing to subtract yet), all warps
  gen_tiles<KIND>(P, N, th, etab, slots, tab, TI, 0, 0, tid, kNT);
  __syncthreads();
  PH_ADD(0, t_pro);

  // Pipeline per panel J (the slots of column J hold the final C(I,J), I ≥ J,
  // row-major, on entry — each tile is staged in the slot its L will occupy):
  //   A: the diagonal warp factors tile (J,J) while the update warps u = 1..3
  //      generate A(·,J+1) into column J+1's slots and accumulate, in registers
  //      on the tensor cores, S(I) = Σ_{K<J} L(I,K) L(J+1,K)ᵀ, I = J+1+(u−1)+3s;
  //   B: all warps: L(I,J) = C(I,J) L(J,J)⁻ᵀ for I > J, one row per thread, in
  //      place (a row occupies the same 64 bytes in both layouts);
  //   C: update warps: C(I,J+1) = A − S(I) − L(I,J) L(J+1,J)ᵀ in place.
  for (int J = 0; J < TJ; ++J) {
    const bool ahead = (J + 1 < TJ);
    double S0[MAXT][2];  // one DMMA chain per tile; tiles interleave for ILP
#pragma unroll
    for (int s = 0; s < MAXT; ++s) S0[s][0] = S0[s][1] = 0.0;
    PH_T(t_a);
    if (uw == 0) {
      factor_diag_tile(slots + 64 * tab[J * TI + J], diagL, rinv, J, m, N, lane, kPivotFloor * th.sigma2, pm, nbad,
                       qd);
      int ex;
      pm = frexp(pm, &ex);  // keep the running product of ≤ N pivots in range
      pe += ex;
      if (nbad && lane == 0) misc[2] = 1.0;
      PH_ADD(1, t_a);
    } else if (ahead) {
      PH_T(t_gen);
      gen_tiles<KIND>(P, N, th, etab, slots, tab, TI, J + 1, J + 1, utid, (kW - 1) * 32);
      PH_ADD(9, t_gen);
      PH_T(t_gm);
      // exactly ns = ⌈(TI−J−1−(u−1))/3⌉ tiles: no predicated-off DMMA issue
      const int ns = (TI - J - 1 - (uw - 1) + (kW - 2)) / (kW - 1);
      switch (ns) {
#define BV_NS(n)                                                                          \
  case n:                                                                                 \
    if (MAXT >= n) panel_gemm<(MAXT >= n ? n : 1), MAXT>(S0, slots, tab, TI, J, uw, lane); \
    break;
        BV_NS(1) BV_NS(2) BV_NS(3) BV_NS(4) BV_NS(5) BV_NS(6) BV_NS(7) BV_NS(8) BV_NS(9) BV_NS(10) BV_NS(11)
        BV_NS(12)
#undef BV_NS
        default: break;
      }
#ifdef BV_PROFILE_PHASES
      if (S0[0][0] == 12345.678) misc[7] = S0[0][1];
#endif
      PH_ADD(8, t_gm);
      PH_ADD(2, t_a);
    }
    PH_T(t_s1);
    __syncthreads();
    PH_ADD(3, t_s1);
    if (misc[2] != 0.0) break;
    PH_T(t_b);

    // B: rows below the diagonal tile (a5/a6), solved in place into fragment order
    const int rows = (TI - J - 1) * 8;
    for (int rr = tid; rr < rows; rr += kNT) {
      const int I = J + 1 + (rr >> 3);
      const int gg = rr & 7;
      double* src = slots + 64 * tab[I * TI + J] + 8 * gg;  // C(I,J) row gg → L(I,J) row gg
      double c[8], x[8];
      {
        double2 ch[4];
        ld_row_rot(src, gg >> 1, ch);
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          c[2 * q] = ch[q].x;
          c[2 * q + 1] = ch[q].y;
        }
      }
#pragma unroll
      for (int k = 0; k < 8; ++k) {
        double tv = c[k];
#pragma unroll
        for (int kk = 0; kk < k; ++kk) tv = fma(-x[kk], diagL[8 * k + kk], tv);
        // tv / L_kk: scaled by 1/L_kk, then one residual correction (rinv = 0 on
        // padding columns → x = 0)
        const double xk = tv * rinv[k];
        x[k] = fma(fma(-xk, diagL[9 * k], tv), rinv[k], xk);
      }
      if (8 * I + gg == N) {  // the y row: u = Σ_{j≥m} z_j² (a8)
        double qd = 0.0;
#pragma unroll
        for (int k = 0; k < 8; ++k)
          if (8 * J + k >= m && 8 * J + k < N) qd = fma(x[k], x[k], qd);
        misc[1] += qd;
      }
      {  // fragment order: chunk q of the row holds (L[q], L[q+4])
        const double2 ch[4] = {make_double2(x[0], x[4]), make_double2(x[1], x[5]), make_double2(x[2], x[6]),
                               make_double2(x[3], x[7])};
        st_row_rot(src, gg >> 1, ch);
      }
    }
    PH_ADD(4, t_b);
    PH_T(t_s2);
    __syncthreads();
    PH_ADD(5, t_s2);
    if (!ahead) break;
    PH_T(t_c);

    // C: last term of panel J+1's update, then publish C(I,J+1) in place
    if (uw > 0) {
      const double2 b = lds2(slots + 64 * tab[(J + 1) * TI + J] + 2 * lane);
#pragma unroll
      for (int s = 0; s < MAXT; ++s) {
        const int I = J + uw + (kW - 1) * s;
        if (I < TI) {
          const double2 a = lds2(slots + 64 * tab[I * TI + J] + 2 * lane);
          dmma884(S0[s][0], S0[s][1], a.x, b.x);
          dmma884(S0[s][0], S0[s][1], a.y, b.y);
          double* cp = slots + 64 * tab[I * TI + J + 1] + 8 * g + 2 * t;
          const double2 av = lds2(cp);
          sts2(cp, av.x - S0[s][0], av.y - S0[s][1]);
        }
      }
    }
    __syncthreads();
    PH_ADD(6, t_c);
  }
#ifdef BV_PROFILE_PHASES
  if (threadIdx.x == 0) atomicAdd(&g_phase_cycles[7], 1ull);
#endif

  // ---- a8: per-block outputs and the exact fixed-point term (the diagonal
  // warp holds d's pivot product; u's TRSM part is in misc[1], visible since
  // the loop's last barrier)
  if (uw == 0 && lane == 0) {
    const bool fail = misc[2] != 0.0;
    int st = fail ? kNotPD : kOk;
    uint32_t c[6] = {0, 0, 0, 0, 0, 0};
    const double logdet = fail ? failed_d() : log(pm) + (double)pe * 0.69314718055994530942;  // d = Σ_{j≥m} log p_j
    const double quad = fail ? 0.0 : misc[1] + qd;
    if (!fail) {
      const double tk = -0.5 * (quad + logdet + (double)l * kLn2Pi);
      if (fixed_encode(tk, c)) st = kTermRange;
    }
    out_u[q] = quad;
    out_d[q] = logdet;
    accumulate_term(acc, c, st, k_begin + q);  // a9
  }
}

// ------------------------------------------------------------------ host side
int debug_phase_cycles(unsigned long long* out, int reset) {
#ifdef BV_PROFILE_PHASES
  if (out) cudaMemcpyFromSymbol(out, g_phase_cycles, sizeof(unsigned long long) * 10);
  if (reset) {
    unsigned long long z[10] = {0, 0, 0, 0, 0, 0, 0, 0, 0, 0};
    cudaMemcpyToSymbol(g_phase_cycles, z, sizeof(z));
  }
  return 1;
#else
  (void)out;
  (void)reset;
  return 0;
#endif
}

int v2_maxt_for(int TI) {
  const int need = (TI - 1 + (kW - 2)) / (kW - 1);  // panel J+1 tiles over the update warps
  const int opts[] = {1, 2, 3, 4, 5, 6, 8, 10, 12};
  for (int o : opts)
    if (o >= need) return o;
  return -1;
}

size_t v2_smem_bytes(int TImax, int cap) { return (size_t)V2Layout(TImax, cap).total_bytes; }

template <int MAXT>
static cudaError_t prep_kinds(size_t smem) {
  cudaError_t e = cudaSuccess;
  if (e == cudaSuccess)
    e = cudaFuncSetAttribute(bv_block_v2_kernel<MAXT, 0>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e == cudaSuccess)
    e = cudaFuncSetAttribute(bv_block_v2_kernel<MAXT, 1>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e == cudaSuccess)
    e = cudaFuncSetAttribute(bv_block_v2_kernel<MAXT, 2>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e == cudaSuccess)
    e = cudaFuncSetAttribute(bv_block_v2_kernel<MAXT, 3>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  return e;
}

cudaError_t prepare_block_v2(size_t max_smem) {
  cudaError_t e = cudaSuccess;
  if (e == cudaSuccess) e = prep_kinds<1>(max_smem);
  if (e == cudaSuccess) e = prep_kinds<2>(max_smem);
  if (e == cudaSuccess) e = prep_kinds<3>(max_smem);
  if (e == cudaSuccess) e = prep_kinds<4>(max_smem);
  if (e == cudaSuccess) e = prep_kinds<5>(max_smem);
  if (e == cudaSuccess) e = prep_kinds<6>(max_smem);
  if (e == cudaSuccess) e = prep_kinds<8>(max_smem);
  if (e == cudaSuccess) e = prep_kinds<10>(max_smem);
  if (e == cudaSuccess) e = prep_kinds<12>(max_smem);
  return e;
}

template <int MAXT>
static void launch_kind(int kind, int nblocks, size_t smem, cudaStream_t s, const PointRec* pts, const int32_t* nbr,
                        const BlockDesc* desc, const int32_t* list, const Theta* th, const int16_t* tabs,
                        const int32_t* tab_off, const double* etab, int TImax, int cap, double* u, double* d,
                        unsigned long long* acc, int k_begin) {
#define BV_K(KD)                                                                                              \
  bv_block_v2_kernel<MAXT, KD><<<nblocks, kNT, smem, s>>>(pts, nbr, desc, list, th, tabs, tab_off, etab, TImax, \
                                                          cap, u, d, acc, k_begin)
  switch (kind) {
    case 0: BV_K(0); break;
    case 1: BV_K(1); break;
    case 2: BV_K(2); break;
    default: BV_K(3); break;
  }
#undef BV_K
}

cudaError_t launch_block_v2(int kind, int nblocks, int TImax, int cap, cudaStream_t s, const PointRec* pts,
                            const int32_t* nbr, const BlockDesc* desc, const int32_t* list, const Theta* th,
                            const int16_t* tabs, const int32_t* tab_off, const double* etab, double* u, double* d,
                            unsigned long long* acc, int k_begin) {
  if (nblocks == 0) return cudaSuccess;
  const size_t smem = v2_smem_bytes(TImax, cap);
  switch (v2_maxt_for(TImax)) {
#define BV_MT(MT)                                                                                                \
  case MT:                                                                                                       \
    launch_kind<MT>(kind, nblocks, smem, s, pts, nbr, desc, list, th, tabs, tab_off, etab, TImax, cap, u, d, acc, \
                    k_begin);                                                                                   \
    break;
    BV_MT(1) BV_MT(2) BV_MT(3) BV_MT(4) BV_MT(5) BV_MT(6) BV_MT(8) BV_MT(10) BV_MT(12)
#undef BV_MT
    default: return cudaErrorInvalidValue;
  }
  return cudaGetLastError();
}

}  // namespace bv
