// bv_block_w.cu — the warp-per-block kernel: ONE WARP per block, the whole joint
// matrix in REGISTERS (joint sizes N ≤ 8·TI − 1, TI ≤ kWMaxTI = 16), many blocks per SM.
// The host sends every bucket with TI ≤ 10 here, and the buckets with TI ≤ 16 that hold at
// least 2,048 blocks of the plan (bv_host.cpp: one warp per block needs a full wave of warps).
//
// Same mathematics as the large-block kernel (Alg. 1 l.10-29, PAPER.md:593-632,
// fused into one Cholesky of the joint matrix with the y row appended, DESIGN.md
// §4), for the small conditioning sets of c5 at m = 30 (N median 49): there a
// block's whole elimination is a few thousand FP64 MMAs, too little to split
// across warps, so each warp owns one block and the SM's ~12-20 resident warps
// (one per block) hide each other's latency.
//
// The tiles live in registers, negated (Ĉ = −C), one double2 per lane per tile in
// the MMA accumulator layout (bv_tile.cuh): lane (g,t) holds row g, columns 2t and
// 2t+1.  Left-looking over the column panels K (all compile-time: TI is a template
// parameter, the panel loop is unrolled, so every tile index and every MMA is
// static and nothing is predicated), per panel:
//   generate A(I,K), I ≥ K (Eq. 7; a compact loop staged through shared memory,
//     then into registers);
//   Ĉ(I,K) += L(I,K') L(K,K')ᵀ for K' = 0..K−1 in that order — progressive
//     subtraction, the rounding order of a right-looking elimination;
//   factor Ĉ(K,K) across the warp's lanes (factor_dist below: the pivot, the scaled
//     column and the inverse's rows move by shuffles — no 32-lane redundant in-lane
//     factorisation); L_KK and −L_KK⁻¹ come out already in the B-fragment form;
//   L(I,K) = C(I,K) L_KK⁻ᵀ for I > K (tile::trsm: explicit inverse + one FP64
//     refinement step).
// Only the L tiles still to be read (rows ≥ K of the panels < K) and panel K are
// live: ≈ (TI/2)² + TI tiles instead of TI(TI+1)/2, which keeps the register file
// at 16+ resident blocks per SM.
#include <cuda_runtime.h>
#include <stdint.h>

#include "bv_tile.cuh"

namespace bv {
namespace wk {

using namespace tile;
constexpr int kWMaxTI = 16;
// Generated tiles in flight per lane: 1 (measured: 4 → 2 c5 m = 60 256.3 -> 269.8 evals/s,
// m = 30 unchanged; 2 → 1 m = 30 690 -> 711, m = 60 262 -> 268 — fewer live temporaries next
// to the register tiles, and one generation copy per panel).
constexpr int kGenFly = 1;
// The diagonal factorisation's pivot loop is a rolled loop here (factor_dist<1>): the
// kernel is unrolled over its panels, so an unrolled pivot loop would put TI copies of
// ~350 instructions into the code (TI = 7: 7.3k → 4.7k SASS instructions; measured
// c5 m = 30 664 -> 689 evals/s; instruction fetch, ncu stall_no_instruction, was the
// largest stall).  A rolled PANEL loop (generation and factorisation once, the register-tile
// parts reached by a compare chain) measured slower still (663 at m = 30): the unrolled
// panels let one panel's generation overlap the previous panel's pivot chain.

__host__ __device__ constexpr int ntiles(int TI) { return TI * (TI + 1) / 2; }
__host__ __device__ constexpr int tidx(int I, int K) { return (I * (I + 1) >> 1) + K; }

// Shared memory (doubles): the gathered points, a staging buffer for one generated
// panel (generation is a compact runtime loop; the tiles then move to registers),
// θ and the exp table.
struct Layout {
  int P, G, theta, etab, total;
  __host__ __device__ constexpr Layout(int TI)
      : P(0), G(32 * TI), theta(G + 64 * TI), etab(theta + (int)(sizeof(Theta) / 8)), total(etab + 64) {}
  __host__ __device__ constexpr int bytes() const { return 8 * total; }
};
// Resident warps (= blocks) per SM the register budget targets (live tiles ≈ (TI/2)² + TI).
// (measured with one generated tile in flight: TI ≥ 9 at 14 instead of 12 blocks, c5 m = 60
// 267.8 -> 277.3 evals/s; 16 for TI ≥ 9 or TI = 8, or 18 for TI 6-7: no gain or slower)
// (TI 11-16 for the large buckets: TI = 16 needs the full 255 registers and
// still spills ~400 B per thread; capping it lower spills more, and it measured faster than
// the CTA kernel anyway)
__host__ __device__ constexpr int minb_for(int TI) {
  return TI >= 15 ? 8 : TI >= 13 ? 10 : TI >= 11 ? 12 : TI >= 8 ? 14 : TI >= 6 ? 16 : 20;
}

template <int TI, int KIND>
__global__ void __launch_bounds__(32, minb_for(TI)) bv_block_w_kernel(
    const PointRec* __restrict__ pts, const int32_t* __restrict__ nbr, const BlockDesc* __restrict__ desc,
    const int32_t* __restrict__ list, const Theta* __restrict__ theta_dev, const double* __restrict__ exp_tab,
    double* __restrict__ out_u, double* __restrict__ out_d, unsigned long long* __restrict__ acc, int k_begin,
    const double* __restrict__ pre, const int64_t* __restrict__ pre_off, double jit) {
  constexpr Layout Ly(TI);
  constexpr int NT = ntiles(TI);
  extern __shared__ __align__(16) double smem[];
  PointRec* P = reinterpret_cast<PointRec*>(smem + Ly.P);
  double* G = smem + Ly.G;
  Theta* ths = reinterpret_cast<Theta*>(smem + Ly.theta);
  double* etab = smem + Ly.etab;

  const int q = list[blockIdx.x];
  const BlockDesc ds = desc[q];
  const int m = ds.m, l = ds.l, N = m + l;
  const int TJ = (N + 7) >> 3;  // column panels: TI or TI − 1 (TI = (N + 8) >> 3, the bucket)
  const int lane = threadIdx.x, g = lane >> 2, t = lane & 3;
  const double* preb = KIND == kPre ? pre + pre_off[q] : nullptr;

  // a1/a2: θ, exp table, gathered points (neighbours first); padding = far points
  etab[lane] = exp_tab[lane];
  etab[lane + 32] = exp_tab[lane + 32];
  if (lane < (int)(sizeof(Theta) / 8)) reinterpret_cast<double*>(ths)[lane] = reinterpret_cast<const double*>(theta_dev)[lane];
#pragma unroll 1
  for (int i = lane; i < 8 * TI; i += 32) {
    const double far = 1e30 * (double)(i + 1);
    PointRec r = {far, far, far, 0.0};
    if (i < N) r = pts[(i < m) ? nbr[ds.nbr_off + i] : ds.pstart + (i - m)];
    P[i] = r;
  }
  __syncwarp();
  const Theta& th = *ths;

  const int Iy = N >> 3, gy = N & 7;
  const double pfloor = kPivotFloor * th.sigma2;
  double pm = 1.0, qd = 0.0;
  int pe = 0, nbad = 0;
  double2 T[NT];
#pragma unroll
  for (int K = 0; K < TI; ++K) {
    if (K < TJ) {  // uniform (only the last panel can be absent)
      // a3: panel K, tiles I = K..TI−1, kGenFly in flight, staged through shared memory
#pragma unroll 1
      for (int i0 = K; i0 < TI; i0 += kGenFly) {
        double2 v[kGenFly];
#pragma unroll
        for (int u = 0; u < kGenFly; ++u) v[u] = gen_tile<KIND>(P, i0 + u < TI ? i0 + u : TI - 1, K, g, t, N, th, etab, preb);
#pragma unroll
        for (int u = 0; u < kGenFly; ++u)
          if (i0 + u < TI) sts2(G + 64 * (i0 + u) + 2 * lane, v[u].x, v[u].y);
      }
      __syncwarp();
#pragma unroll
      for (int I = K; I < TI; ++I) T[tidx(I, K)] = lds2(G + 64 * I + 2 * lane);
      __syncwarp();
      // a6: progressive subtraction of the earlier panels, K' ascending
#pragma unroll
      for (int Kp = 0; Kp < K; ++Kp)
#pragma unroll
        for (int I = K; I < TI; ++I) {
          double2& c = T[tidx(I, K)];
          dmma(c.x, c.y, T[tidx(I, Kp)].x, T[tidx(K, Kp)].x);
          dmma(c.x, c.y, T[tidx(I, Kp)].y, T[tidx(K, Kp)].y);
        }
      // a4/a7: the diagonal tile (positive C = −Ĉ)
      double c0 = neg(T[tidx(K, K)].x), c1 = neg(T[tidx(K, K)].y), z0, z1;
      factor_dist<1>(c0, c1, z0, z1, lane, K, m, N, pfloor, jit, pm, nbad, qd);
      int ex;
      pm = frexp(pm, &ex);
      pe += ex;
      const double2 zn = make_double2(z0, z1), lf = make_double2(c0, c1);
      // a5/a6: L(I,K) for I > K
#pragma unroll
      for (int I = K + 1; I < TI; ++I) {
        T[tidx(I, K)] = trsm(T[tidx(I, K)], zn, lf);
        if (I == Iy && g == gy) qd += yrow_sq(T[tidx(I, K)], K, t, m, N);
      }
    }
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) qd += __shfl_xor_sync(0xffffffffu, qd, o);

  // a8: per-block outputs and the exact fixed-point term (a9)
  if (lane == 0) {
    const bool fail = nbad != 0;
    int st = fail ? kNotPD : kOk;
    uint32_t cc[6] = {0, 0, 0, 0, 0, 0};
    const double logdet = fail ? failed_d() : log(pm) + (double)pe * 0.69314718055994530942;  // d = Σ_{j≥m} log p_j
    const double quad = fail ? 0.0 : qd;
    if (!fail) {
      const double tk = -0.5 * (quad + logdet + (double)l * kLn2Pi);
      if (fixed_encode(tk, cc)) st = kTermRange;
    }
    out_u[q] = quad;
    out_d[q] = logdet;
    accumulate_term(acc, cc, st, k_begin + q);
  }
}

}  // namespace wk

// ------------------------------------------------------------------ host side
int w_max_ti() { return wk::kWMaxTI; }
size_t w_smem_bytes(int TI) { return (size_t)wk::Layout(TI).bytes(); }

template <int TI>
static cudaError_t w_prep_ti() {
  const int smem = wk::Layout(TI).bytes();
  cudaError_t e = cudaSuccess;
  const void* f[5] = {(const void*)wk::bv_block_w_kernel<TI, 0>, (const void*)wk::bv_block_w_kernel<TI, 1>,
                      (const void*)wk::bv_block_w_kernel<TI, 2>, (const void*)wk::bv_block_w_kernel<TI, 3>,
                      (const void*)wk::bv_block_w_kernel<TI, tile::kPre>};
  for (int k = 0; k < 5 && e == cudaSuccess; ++k) e = cudaFuncSetAttribute(f[k], cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  return e;
}

template <int TI>
static cudaError_t w_launch_ti(int kind, int nblocks, cudaStream_t s, const PointRec* pts, const int32_t* nbr,
                               const BlockDesc* desc, const int32_t* list, const Theta* th, const double* etab,
                               double* u, double* d, unsigned long long* acc, int k_begin, const double* pre,
                               const int64_t* pre_off, double jit) {
  const int smem = wk::Layout(TI).bytes();
#define BV_K(KD)                                                                                          \
  wk::bv_block_w_kernel<TI, KD><<<nblocks, 32, smem, s>>>(pts, nbr, desc, list, th, etab, u, d, acc, k_begin, \
                                                          pre, pre_off, jit)
  switch (kind) {
    case 0: BV_K(0); break;
    case 1: BV_K(1); break;
    case 2: BV_K(2); break;
    case 3: BV_K(3); break;
    default: BV_K(tile::kPre); break;
  }
#undef BV_K
  return cudaGetLastError();
}

cudaError_t prepare_block_w() {
  cudaError_t e = cudaSuccess;
#define BV_P(T) if (e == cudaSuccess) e = w_prep_ti<T>();
  BV_P(1) BV_P(2) BV_P(3) BV_P(4) BV_P(5) BV_P(6) BV_P(7) BV_P(8) BV_P(9) BV_P(10) BV_P(11) BV_P(12) BV_P(13) BV_P(14) BV_P(15) BV_P(16)
#undef BV_P
  return e;
}

cudaError_t launch_block_w(int kind, int nblocks, int TI, cudaStream_t s, const PointRec* pts, const int32_t* nbr,
                           const BlockDesc* desc, const int32_t* list, const Theta* th, const double* etab, double* u,
                           double* d, unsigned long long* acc, int k_begin, const double* pre, const int64_t* pre_off,
                           double jit) {
  if (nblocks == 0) return cudaSuccess;
  switch (TI) {
#define BV_T(T)                                                                                                  \
  case T:                                                                                                        \
    return w_launch_ti<T>(kind, nblocks, s, pts, nbr, desc, list, th, etab, u, d, acc, k_begin, pre, pre_off, jit);
    BV_T(1) BV_T(2) BV_T(3) BV_T(4) BV_T(5) BV_T(6) BV_T(7) BV_T(8) BV_T(9) BV_T(10) BV_T(11) BV_T(12) BV_T(13) BV_T(14) BV_T(15) BV_T(16)
#undef BV_T
    default: return cudaErrorInvalidValue;
  }
}

}  // namespace bv
