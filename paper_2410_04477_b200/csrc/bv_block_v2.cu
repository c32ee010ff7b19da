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
//    sum accumulated in registers by DMMA.8x8x4 (two accumulator chains), A
//    generated on the fly from the gathered points (Matérn, Eq. 7) — the
//    covariance never touches HBM;
//  * diagonal tile factored in-lane by warp 0 (8 pivots, rsqrt), rows below
//    solved one row per thread (forward substitution, not an explicit inverse);
//  * only the live part of L is kept in shared memory: L(I,K) is needed from
//    panel K+1 to panel I, so at panel J the live set is {K < J ≤ I}, at most
//    T²/4 tiles; slots are recycled through a per-(TI,TJ) table computed once
//    on the host (bv_host.cpp: build_slot_tables);
//  * L tiles are stored in DMMA fragment order: element (g, k) at
//    2·(4g + (k&3)) + (k>>2), so one LDS.128 per lane yields both k-halves.
#include <cuda_runtime.h>
#include <stdint.h>

#include "bv_common.cuh"
#include "matern.cuh"

namespace bv {

namespace {

constexpr int kW = 4;            // warps per CTA
constexpr int kNT = kW * 32;     // threads per CTA

__device__ __forceinline__ void dmma884(double& d0, double& d1, double a, double b) {
  asm("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
      : "+d"(d0), "+d"(d1)
      : "d"(a), "d"(b));
}

__device__ __forceinline__ double2 lds2(const double* p) { return *reinterpret_cast<const double2*>(p); }
__device__ __forceinline__ void sts2(double* p, double a, double b) {
  *reinterpret_cast<double2*>(p) = make_double2(a, b);
}

}  // namespace

#ifdef BV_PROFILE_PHASES
// Debug-only phase timers (cycles summed over CTAs): 0 prologue, 1 phase A
// (diag warp), 2 phase A (update warps), 3 sync after A, 4 phase B, 5 sync
// after B, 6 phase C + sync, 7 CTAs, 8 GEMM part of 2, 9 generation part of 2.
__device__ unsigned long long g_phase_cycles[10];
#define PH_T(v) long long v = clock64()
#define PH_ADD(i, v0) do { if ((threadIdx.x & 31) == 0) atomicAdd(&g_phase_cycles[i], (unsigned long long)(clock64() - (v0))); } while (0)
#else
#define PH_T(v)
#define PH_ADD(i, v0)
#endif

// Shared-memory carve-up (in doubles) for a bucket with at most TImax tile rows
// and `cap` L slots.
struct V2Layout {
  int P, stage, stage2, diag, rinv, misc, theta, etab, slots, tab, total_bytes;
  __host__ __device__ V2Layout(int TImax, int cap) {
    P = 0;                          // PointRec[8·TImax]
    stage = P + 32 * TImax;         // TImax tiles, row-major 8×8 (panel J)
    stage2 = stage + 64 * TImax;    // the same for panel J+1 (double buffer)
    diag = stage2 + 64 * TImax;     // factored diagonal tile (row-major lower)
    rinv = diag + 64;               // 1/L_jj of the diagonal tile
    misc = rinv + 8;                // [0] logdet, [1] quad, [2] fail
    theta = misc + 8;               // Theta copy (16 doubles + ints → 20 doubles)
    etab = theta + 20;              // 2^{−j/64}, j = 0..63 (exp_neg table)
    slots = etab + 64;              // cap L tiles in fragment order
    tab = slots + 64 * cap;         // int16 slot table (TImax²), in doubles:
    total_bytes = (tab + (TImax * TImax + 3) / 4) * 8;
  }
};

// Covariance entry (r, c) of the augmented joint matrix (a3; Eq. 7): rows/cols
// < N are points, row N is the observation row, everything else is padding.
// Branch-free for the closed forms: every lane evaluates the covariance, then
// selects (P holds 8·TI zero-padded records, so the loads are in bounds).
template <int KIND>
__device__ __forceinline__ double joint_entry(const PointRec* P, int r, int c, int N, const Theta& th,
                                             const double* tab64) {
  const PointRec pc = P[c];
  double v = matern_kind<KIND>(sqdist(P[r], pc), th, tab64);
  v = (r == N) ? pc.v : v;
  return (c >= N || r > N) ? 0.0 : v;
}

// One warp, in-lane: Cholesky of the diagonal tile held row-major in `stage`
// (lower part).  Publishes L's strict lower part (incl. the y row when it sits
// inside this tile) and 1/L_jj (0 on padding columns), adds the panel's
// Σ_{j≥m} log p_j to d, and raises the non-PD flag.
__device__ __forceinline__ void factor_diag_tile(const double* stage, double* diagL, double* rinv, double* misc,
                                                 int J, int m, int N, int lane) {
  double a[8][8];
#pragma unroll
  for (int i = 0; i < 8; ++i)
#pragma unroll
    for (int j = 0; j <= i; ++j) a[i][j] = stage[8 * i + j];
  double rv[8];
  double prod = 1.0;  // Π_{j≥m} p_j over this panel (≤ 8 pivots: no over/underflow for sane θ)
  int nbad = 0;
  const int nreal = N - 8 * J;   // columns j < nreal are real pivots
  const int jm = m - 8 * J;      // columns j ≥ jm belong to the block (contribute to d)
#pragma unroll
  for (int j = 0; j < 8; ++j) {
    double p = a[j][j];
    const bool ok = (p > 0.0) & (p <= 1.7976931348623157e308);
    const bool real = j < nreal;
    nbad += (real & !ok) ? 1 : 0;
    p = (real & ok) ? p : 1.0;
    prod *= (j >= jm) ? p : 1.0;
    rv[j] = real ? rsqrt_pos(p) : 0.0;
#pragma unroll
    for (int i = j + 1; i < 8; ++i) a[i][j] *= rv[j];
#pragma unroll
    for (int i = j + 1; i < 8; ++i)
#pragma unroll
      for (int k = j + 1; k <= i; ++k) a[i][k] = fma(-a[i][j], a[k][j], a[i][k]);
  }
#pragma unroll
  for (int i = 0; i < 8; ++i)
    if (lane == i) {
#pragma unroll
      for (int j = 0; j < i; ++j) diagL[8 * i + j] = a[i][j];
      rinv[i] = rv[i];
    }
  if (lane == 0) {
    misc[0] += log(prod);  // d = Σ_{j≥m} log p_j (a8)
    if (nbad) misc[2] = 1.0;
  }
}

// a3: generate the row-major tiles I = I0 .. I0+ntiles−1 of column panel J
// into dst (tile i at dst + 64·i), entries spread over `nthr` threads.  A
// plain loop (two entries in flight per thread): one copy of the Matérn code
// keeps the kernel inside the instruction cache.
template <int KIND>
__device__ __forceinline__ void gen_tiles(const PointRec* P, int N, const Theta& th, const double* tab64, double* dst,
                                          int I0, int ntiles, int J, int thr, int nthr) {
  const int total = ntiles * 64;
#pragma unroll 2
  for (int e = thr; e < total; e += nthr) {
    const int r = 8 * I0 + (e >> 3);  // (tile, row) flattened: 8·(I0 + e/64) + (e/8)%8
    const int c = 8 * J + (e & 7);
    dst[e] = joint_entry<KIND>(P, r, c, N, th, tab64);
  }
}

template <int MAXT, int KIND>
__global__ void __launch_bounds__(kNT, 4)
bv_block_v2_kernel(const PointRec* __restrict__ pts, const int32_t* __restrict__ nbr,
                   const BlockDesc* __restrict__ desc, const int32_t* __restrict__ list,
                   const Theta* __restrict__ theta_dev, const int16_t* __restrict__ tabs,
                   const int32_t* __restrict__ tab_off, const double* __restrict__ exp_tab, int TImax, int cap,
                   double* __restrict__ out_u, double* __restrict__ out_d, uint32_t* __restrict__ limbs,
                   int32_t* __restrict__ status) {
  extern __shared__ __align__(16) double smem[];
  const V2Layout Ly(TImax, cap);
  const int q = list[blockIdx.x];
  const BlockDesc ds = desc[q];
  const int m = ds.m, l = ds.l, N = m + l;
  const int TJ = (N + 7) >> 3;  // column panels (pivots 0..N−1)
  const int TI = (N + 8) >> 3;  // tile rows (rows 0..N, incl. the y row)
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int g = lane >> 2, t = lane & 3;
  // Role rotation across co-resident CTAs: the diagonal warp is blockIdx mod 4,
  // the update warps are numbered u = 1..3 after it.
  const int dwarp = blockIdx.x & 3;
  const int uw = (warp - dwarp) & 3;  // 0 = diagonal warp, 1..3 = update warps
  const int utid = (uw - 1) * 32 + lane;  // 0..95 among the update warps

  PointRec* P = reinterpret_cast<PointRec*>(smem + Ly.P);
  double* stage = smem + Ly.stage;
  double* stage2 = smem + Ly.stage2;
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
  if (tid < 8) misc[tid] = 0.0;
  __syncthreads();
  const Theta& th = *ths;
  PH_T(t_pro);

  // panel 0: C(I,0) = A(I,0) (nothing to subtract yet), all warps
  gen_tiles<KIND>(P, N, th, etab, stage, 0, TI, 0, tid, kNT);
  __syncthreads();
  PH_ADD(0, t_pro);

  // Pipeline per panel J (stage holds the final C(I,J), I ≥ J, tile I at
  // stage + 64·(I−J), on entry):
  //   A: the diagonal warp factors tile (J,J) while the update warps u = 1..3
  //      generate A(·,J+1) into stage2 and accumulate, in registers on the
  //      tensor cores, S(I) = Σ_{K<J} L(I,K) L(J+1,K)ᵀ for I = J+1+(u−1)+3s;
  //   B: all warps: L(I,J) = C(I,J) L(J,J)⁻ᵀ for I > J, one row per thread;
  //   C: update warps: C(I,J+1) = A − S(I) − L(I,J) L(J+1,J)ᵀ in stage2; swap.
  for (int J = 0; J < TJ; ++J) {
    const bool ahead = (J + 1 < TJ);
    double S0[MAXT][2];  // one DMMA chain per tile; tiles interleave for ILP
#pragma unroll
    for (int s = 0; s < MAXT; ++s) S0[s][0] = S0[s][1] = 0.0;
    PH_T(t_a);
    if (uw == 0) {
      factor_diag_tile(stage, diagL, rinv, misc, J, m, N, lane);
      PH_ADD(1, t_a);
    } else if (ahead) {
      PH_T(t_gen);
      gen_tiles<KIND>(P, N, th, etab, stage2, J + 1, TI - J - 1, J + 1, utid, 96);
      PH_ADD(9, t_gen);
      PH_T(t_gm);
      const int16_t* tJ = tab + (J + 1) * TI;
#pragma unroll 2
      for (int K = 0; K < J; ++K) {
        const double2 b = lds2(slots + 64 * tJ[K] + 2 * lane);
#pragma unroll
        for (int s = 0; s < MAXT; ++s) {
          const int I = J + uw + (kW - 1) * s;
          if (I < TI) {
            const double2 a = lds2(slots + 64 * tab[I * TI + K] + 2 * lane);
            dmma884(S0[s][0], S0[s][1], a.x, b.x);
            dmma884(S0[s][0], S0[s][1], a.y, b.y);
          }
        }
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

    // B: rows below the diagonal tile (a5/a6), stored in fragment order
    if (tid == 0) {  // the y row inside the diagonal tile (N not a multiple of 8)
      const int yr = N - 8 * J;
      if (yr > 0 && yr < 8) {
        double qd = 0.0;
#pragma unroll 1
        for (int j = 0; j < yr; ++j)
          if (8 * J + j >= m) qd = fma(diagL[8 * yr + j], diagL[8 * yr + j], qd);
        misc[1] += qd;
      }
    }
    const int rows = (TI - J - 1) * 8;
    for (int rr = tid; rr < rows; rr += kNT) {
      const int I = J + 1 + (rr >> 3);
      const int gg = rr & 7;
      const double* src = stage + 64 * (I - J) + 8 * gg;
      double c[8], x[8];
#pragma unroll
      for (int k = 0; k < 8; k += 2) {
        const double2 v = lds2(src + k);
        c[k] = v.x;
        c[k + 1] = v.y;
      }
#pragma unroll
      for (int k = 0; k < 8; ++k) {
        double tv = c[k];
#pragma unroll
        for (int kk = 0; kk < k; ++kk) tv = fma(-x[kk], diagL[8 * k + kk], tv);
        x[k] = tv * rinv[k];  // rinv = 0 on padding columns → x = 0
      }
      if (8 * I + gg == N) {  // the y row: u = Σ_{j≥m} z_j² (a8)
        double qd = 0.0;
#pragma unroll
        for (int k = 0; k < 8; ++k)
          if (8 * J + k >= m && 8 * J + k < N) qd = fma(x[k], x[k], qd);
        misc[1] += qd;
      }
      double* dst = slots + 64 * tab[I * TI + J] + 8 * gg;
#pragma unroll
      for (int k = 0; k < 4; ++k) sts2(dst + 2 * k, x[k], x[k + 4]);
    }
    PH_ADD(4, t_b);
    PH_T(t_s2);
    __syncthreads();
    PH_ADD(5, t_s2);
    if (!ahead) break;
    PH_T(t_c);

    // C: last term of panel J+1's update, then publish C(I,J+1)
    if (uw > 0) {
      const double2 b = lds2(slots + 64 * tab[(J + 1) * TI + J] + 2 * lane);
#pragma unroll
      for (int s = 0; s < MAXT; ++s) {
        const int I = J + uw + (kW - 1) * s;
        if (I < TI) {
          const double2 a = lds2(slots + 64 * tab[I * TI + J] + 2 * lane);
          dmma884(S0[s][0], S0[s][1], a.x, b.x);
          dmma884(S0[s][0], S0[s][1], a.y, b.y);
          double* cp = stage2 + 64 * (I - J - 1) + 8 * g + 2 * t;
          const double2 av = lds2(cp);
          sts2(cp, av.x - S0[s][0], av.y - S0[s][1]);
        }
      }
    }
    double* tmp = stage;
    stage = stage2;
    stage2 = tmp;
    __syncthreads();
    PH_ADD(6, t_c);
  }
#ifdef BV_PROFILE_PHASES
  if (threadIdx.x == 0) atomicAdd(&g_phase_cycles[7], 1ull);
#endif

  // ---- a8: per-block outputs and the exact fixed-point term
  if (tid == 0) {
    const bool fail = misc[2] != 0.0;
    int st = fail ? kNotPD : kOk;
    uint32_t c[6] = {0, 0, 0, 0, 0, 0};
    const double logdet = fail ? 0.0 : misc[0];
    const double quad = fail ? 0.0 : misc[1];
    if (!fail) {
      const double tk = -0.5 * (quad + logdet + (double)l * kLn2Pi);
      if (fixed_encode(tk, c)) st = kTermRange;
    }
    out_u[q] = quad;
    out_d[q] = logdet;
#pragma unroll
    for (int i = 0; i < 6; ++i) limbs[(size_t)q * 6 + i] = c[i];
    status[q] = st;
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
  const int need = (TI - 1 + (kW - 2)) / (kW - 1);  // panel J+1 tiles over warps 1..3
  const int opts[] = {2, 4, 5, 6, 8, 10, 12};
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
  if (e == cudaSuccess) e = prep_kinds<2>(max_smem);
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
                        uint32_t* limbs, int32_t* status) {
#define BV_K(KD)                                                                                             \
  bv_block_v2_kernel<MAXT, KD><<<nblocks, kNT, smem, s>>>(pts, nbr, desc, list, th, tabs, tab_off, etab, TImax, \
                                                          cap, u, d, limbs, status)
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
                            uint32_t* limbs, int32_t* status) {
  if (nblocks == 0) return cudaSuccess;
  const size_t smem = v2_smem_bytes(TImax, cap);
  switch (v2_maxt_for(TImax)) {
    case 2: launch_kind<2>(kind, nblocks, smem, s, pts, nbr, desc, list, th, tabs, tab_off, etab, TImax, cap, u, d, limbs, status); break;
    case 4: launch_kind<4>(kind, nblocks, smem, s, pts, nbr, desc, list, th, tabs, tab_off, etab, TImax, cap, u, d, limbs, status); break;
    case 5: launch_kind<5>(kind, nblocks, smem, s, pts, nbr, desc, list, th, tabs, tab_off, etab, TImax, cap, u, d, limbs, status); break;
    case 6: launch_kind<6>(kind, nblocks, smem, s, pts, nbr, desc, list, th, tabs, tab_off, etab, TImax, cap, u, d, limbs, status); break;
    case 8: launch_kind<8>(kind, nblocks, smem, s, pts, nbr, desc, list, th, tabs, tab_off, etab, TImax, cap, u, d, limbs, status); break;
    case 10: launch_kind<10>(kind, nblocks, smem, s, pts, nbr, desc, list, th, tabs, tab_off, etab, TImax, cap, u, d, limbs, status); break;
    case 12: launch_kind<12>(kind, nblocks, smem, s, pts, nbr, desc, list, th, tabs, tab_off, etab, TImax, cap, u, d, limbs, status); break;
    default: return cudaErrorInvalidValue;
  }
  return cudaGetLastError();
}

}  // namespace bv
