// bv_block_w.cu — the small-block kernel: ONE WARP per block (joint sizes N ≤ 8·TI−1,
// TI ≤ kWMaxTI), many blocks per SM.
//
// Same mathematics as the large-block kernel (Alg. 1 l.10-29, PAPER.md:593-632,
// fused into one Cholesky of the joint matrix with the y row appended, DESIGN.md
// §4), for the small conditioning sets of c5 at m = 30 (N median 49): there a
// block's whole elimination is a few thousand FP64 MMAs, too little to split
// across warps without the hand-offs dominating, so each warp owns one block
// and the SM's ~12-16 resident warps (one per block) hide each other's pivot
// chains.  No barriers beyond __syncwarp.
//
// The packed lower triangle of 8×8 tiles lives in shared memory, negated, in the
// MMA accumulator layout (bv_tile.cuh).  Right-looking: per column panel J the
// diagonal tile is factored in-lane (tile::factor_tile), column J is solved
// (L(I,J) = C(I,J) L_JJ⁻ᵀ, FP64 MMA with one refinement step) and the trailing
// tiles get Ĉ(I,K) += L(I,J) L(K,J)ᵀ.  Solves and updates run in batches of
// four independent tiles (loads, then MMAs, then stores) so their MMA latency
// chains overlap.
#include <cuda_runtime.h>
#include <stdint.h>

#include "bv_tile.cuh"

namespace bv {
namespace wk {

using namespace tile;
constexpr int kWMaxTI = 10;
constexpr int kB = 4;  // tiles in flight per batch

__host__ __device__ constexpr int ntiles(int TI) { return TI * (TI + 1) / 2; }
__host__ __device__ constexpr int tidx(int I, int K) { return (I * (I + 1) >> 1) + K; }

struct Layout {
  int P, T, zb, lb, theta, etab, tab, total;
  __host__ __device__ constexpr Layout(int TI)
      : P(0),
        T(32 * TI),                  // packed lower tiles, tidx(I,K)
        zb(T + 64 * ntiles(TI)),     // −L_JJ⁻¹, row-major
        lb(zb + 64),                 // L_JJ, row-major
        theta(lb + 64),
        etab(theta + (int)(sizeof(Theta) / 8)),
        tab(etab + 64),              // int16 (I | K << 8), tiles in column-major order
        total(tab + (ntiles(TI) + 3) / 4) {}
  __host__ __device__ constexpr int bytes() const { return 8 * total; }
};

__device__ __forceinline__ void dmma_if(double& d0, double& d1, double a, double b, int p) {
  asm("{\n .reg .pred q;\n setp.ne.b32 q, %4, 0;\n"
      " @q mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n}\n"
      : "+d"(d0), "+d"(d1)
      : "d"(a), "d"(b), "r"(p));
}
__device__ __forceinline__ double2 trsm_if(double2 c, double2 zn, double2 lj, int p) {
  double x0 = 0.0, x1 = 0.0;
  dmma_if(x0, x1, c.x, zn.x, p);
  dmma_if(x0, x1, c.y, zn.y, p);
  dmma_if(c.x, c.y, x0, lj.x, p);
  dmma_if(c.x, c.y, x1, lj.y, p);
  dmma_if(x0, x1, c.x, zn.x, p);
  dmma_if(x0, x1, c.y, zn.y, p);
  return make_double2(x0, x1);
}

template <int TI, int KIND>
__global__ void __launch_bounds__(32) bv_block_w_kernel(
    const PointRec* __restrict__ pts, const int32_t* __restrict__ nbr, const BlockDesc* __restrict__ desc,
    const int32_t* __restrict__ list, const Theta* __restrict__ theta_dev, const double* __restrict__ exp_tab,
    double* __restrict__ out_u, double* __restrict__ out_d, unsigned long long* __restrict__ acc, int k_begin,
    const double* __restrict__ pre, const int64_t* __restrict__ pre_off, double jit) {
  constexpr Layout Ly(TI);
  extern __shared__ __align__(16) double smem[];
  PointRec* P = reinterpret_cast<PointRec*>(smem + Ly.P);
  double* T = smem + Ly.T;
  double* zb = smem + Ly.zb;
  double* lb = smem + Ly.lb;
  Theta* ths = reinterpret_cast<Theta*>(smem + Ly.theta);
  double* etab = smem + Ly.etab;
  int16_t* tab = reinterpret_cast<int16_t*>(smem + Ly.tab);

  const int q = list[blockIdx.x];
  const BlockDesc ds = desc[q];
  const int m = ds.m, l = ds.l, N = m + l;
  const int TJ = (N + 7) >> 3;  // column panels; TI = (N + 8) >> 3 (the bucket)
  const int lane = threadIdx.x, g = lane >> 2, t = lane & 3;
  const double* preb = KIND == kPre ? pre + pre_off[q] : nullptr;

  // a1/a2: θ, exp table, gathered points (neighbours first), tile list
  etab[lane] = exp_tab[lane];
  etab[lane + 32] = exp_tab[lane + 32];
  if (lane < (int)(sizeof(Theta) / 8)) reinterpret_cast<double*>(ths)[lane] = reinterpret_cast<const double*>(theta_dev)[lane];
#pragma unroll 1
  for (int i = lane; i < 8 * TI; i += 32) {
    const double far = 1e30 * (double)(i + 1);  // padding: far points (exact zeros off the diagonal)
    PointRec r = {far, far, far, 0.0};
    if (i < N) r = pts[(i < m) ? nbr[ds.nbr_off + i] : ds.pstart + (i - m)];
    P[i] = r;
  }
  int ntl = 0;  // tiles of the lower triangle, column-major (K < TJ): column K starts at colstart(K)
  for (int K = 0; K < TJ; ++K)
    for (int I = K; I < TI; ++I) {
      if (ntl % 32 == lane) tab[ntl] = (int16_t)(I | (K << 8));
      ++ntl;
    }
  __syncwarp();
  const Theta& th = *ths;

  // a3: every tile of the lower triangle, batches of kB in flight
#pragma unroll 1
  for (int e0 = 0; e0 < ntl; e0 += kB) {
    double2 v[kB];
#pragma unroll
    for (int u = 0; u < kB; ++u) {
      const int e = e0 + u < ntl ? e0 + u : ntl - 1;
      const int c = tab[e];
      v[u] = gen_tile<KIND>(P, c & 0xff, c >> 8, g, t, N, th, etab, preb);
    }
#pragma unroll
    for (int u = 0; u < kB; ++u) {
      const int e = e0 + u < ntl ? e0 + u : ntl - 1;
      const int c = tab[e];
      sts2(T + 64 * tidx(c & 0xff, c >> 8) + 2 * lane, v[u].x, v[u].y);
    }
  }
  __syncwarp();

  const int Iy = N >> 3, gy = N & 7;
  const double pfloor = kPivotFloor * th.sigma2;
  double pm = 1.0, qd = 0.0, qd_in = 0.0;
  int pe = 0, nbad = 0, cs = 0;  // cs = colstart(J)
#pragma unroll 1
  for (int J = 0; J < TJ; ++J) {
    factor_tile<true>(T + 64 * tidx(J, J), lb, zb, J, m, N, lane, pfloor, jit, pm, nbad, qd_in);  // a4/a7
    int ex;
    pm = frexp(pm, &ex);
    pe += ex;
    __syncwarp();
    const double2 zn = lds2(zb + 2 * lane), lf = lds2(lb + 2 * lane);
    // a5/a6: column J, I = J+1 .. TI−1
#pragma unroll 1
    for (int I0 = J + 1; I0 < TI; I0 += kB) {
      double2 c[kB];
#pragma unroll
      for (int u = 0; u < kB; ++u) c[u] = lds2(T + 64 * tidx(I0 + u < TI ? I0 + u : TI - 1, J) + 2 * lane);
#pragma unroll
      for (int u = 0; u < kB; ++u) c[u] = trsm_if(c[u], zn, lf, I0 + u < TI);
#pragma unroll
      for (int u = 0; u < kB; ++u) {
        const int I = I0 + u;
        if (I < TI) {
          sts2(T + 64 * tidx(I, J) + 2 * lane, c[u].x, c[u].y);
          if (I == Iy && g == gy) qd += yrow_sq(c[u], J, t, m, N);
        }
      }
    }
    __syncwarp();
    // a6: trailing tiles (I,K), J < K ≤ I, K < TJ — the suffix of the column-major list
    cs += TI - J;
#pragma unroll 1
    for (int e0 = cs; e0 < ntl; e0 += kB) {
      double2 c[kB], a[kB], b[kB];
      int ti[kB];
#pragma unroll
      for (int u = 0; u < kB; ++u) {
        const int e = e0 + u < ntl ? e0 + u : ntl - 1;
        const int cc = tab[e], I = cc & 0xff, K = cc >> 8;
        ti[u] = tidx(I, K);
        c[u] = lds2(T + 64 * ti[u] + 2 * lane);
        a[u] = lds2(T + 64 * tidx(I, J) + 2 * lane);
        b[u] = lds2(T + 64 * tidx(K, J) + 2 * lane);
      }
#pragma unroll
      for (int u = 0; u < kB; ++u) {
        const int p = e0 + u < ntl;
        dmma_if(c[u].x, c[u].y, a[u].x, b[u].x, p);
        dmma_if(c[u].x, c[u].y, a[u].y, b[u].y, p);
      }
#pragma unroll
      for (int u = 0; u < kB; ++u)
        if (e0 + u < ntl) sts2(T + 64 * ti[u] + 2 * lane, c[u].x, c[u].y);
    }
    __syncwarp();
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) qd += __shfl_xor_sync(0xffffffffu, qd, o);

  // a8: per-block outputs and the exact fixed-point term (a9)
  if (lane == 0) {
    const bool fail = nbad != 0;
    int st = fail ? kNotPD : kOk;
    uint32_t cc[6] = {0, 0, 0, 0, 0, 0};
    const double logdet = fail ? failed_d() : log(pm) + (double)pe * 0.69314718055994530942;  // d = Σ_{j≥m} log p_j
    const double quad = fail ? 0.0 : qd + qd_in;
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
  for (int k = 0; k < 5 && e == cudaSuccess; ++k) {
    e = cudaFuncSetAttribute(f[k], cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    if (e == cudaSuccess)
      e = cudaFuncSetAttribute(f[k], cudaFuncAttributePreferredSharedMemoryCarveout, cudaSharedmemCarveoutMaxShared);
  }
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
  BV_P(1) BV_P(2) BV_P(3) BV_P(4) BV_P(5) BV_P(6) BV_P(7) BV_P(8) BV_P(9) BV_P(10)
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
    BV_T(1) BV_T(2) BV_T(3) BV_T(4) BV_T(5) BV_T(6) BV_T(7) BV_T(8) BV_T(9) BV_T(10)
#undef BV_T
    default: return cudaErrorInvalidValue;
  }
}

}  // namespace bv
