// bv_cv.cu — classic-Vecchia throughput kernel: block size 1.
//
// Classic Vecchia is block Vecchia with every block a single point
// ("a special case when each block size is 1"; univariate
// conditionals).  For such a position the joint matrix of
// Alg. 1 (l.10-27) is (m+1)×(m+1): m neighbours, then the
// point itself, with the y row appended.  After eliminating the m neighbour
// columns the last pivot is the conditional variance σ²_cond and the y row's
// last entry is y − μ_cond, so
//     d = log σ²_cond,   u = (y − μ_cond)² / σ²_cond           (l.24-27 with l = 1).
// One WARP per position (m ≤ 31, so the joint matrix has ≤ 32 rows): lane i
// holds row i in registers (fully unrolled, statically indexed), the y row is
// held column-wise (lane k keeps entry (N, k)), and each elimination step
// broadcasts column j through a 33-double shared-memory buffer.  No barriers
// beyond __syncwarp; 4 independent positions per CTA.  LDLᵀ-ordered (no square
// roots): the pivots are the Schur complements themselves.
#include <cuda_runtime.h>
#include <stdint.h>

#include "bv_common.cuh"
#include "matern.cuh"

namespace bv {

constexpr int kCvWarps = 4;

template <int KIND>
__global__ void __launch_bounds__(kCvWarps * 32) bv_cv_kernel(const PointRec* __restrict__ pts,
                                                              const int32_t* __restrict__ nbr,
                                                              const BlockDesc* __restrict__ desc,
                                                              const int32_t* __restrict__ list, int count,
                                                              const Theta* __restrict__ theta_dev,
                                                              const double* __restrict__ exp_tab,
                                                              double* __restrict__ out_u, double* __restrict__ out_d,
                                                              unsigned long long* __restrict__ acc, int k_begin) {
  __shared__ double etab[64];
  __shared__ __align__(16) double thbuf[sizeof(Theta) / 8];
  __shared__ __align__(32) PointRec P[kCvWarps][32];
  __shared__ __align__(16) double colbuf[kCvWarps][32];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  if (tid < 64) etab[tid] = exp_tab[tid];
  if (tid < (int)(sizeof(Theta) / 8)) thbuf[tid] = reinterpret_cast<const double*>(theta_dev)[tid];
  const int idx = blockIdx.x * kCvWarps + warp;
  const bool active = idx < count;  // warp-uniform
  const int q = active ? list[idx] : 0;
  const BlockDesc ds = desc[q];
  const int m = ds.m, N = m + 1;  // l = 1
  if (active && lane < N) P[warp][lane] = pts[lane < m ? nbr[ds.nbr_off + lane] : ds.pstart];
  __syncthreads();
  if (!active) return;
  const Theta& th = *reinterpret_cast<const Theta*>(thbuf);
  const PointRec pi = P[warp][lane < N ? lane : 0];

  // a3: row `lane` of the joint lower triangle; the y row column-wise
  double r[32];
#pragma unroll
  for (int k = 0; k < 32; ++k) {
    double v = 0.0;
    if (k <= lane && lane < N) v = matern_kind<KIND>(sqdist(pi, P[warp][k]), th, etab);
    r[k] = v;
  }
  double yk = lane < N ? pi.v : 0.0;

  // a4-a7: eliminate the m neighbour columns (pivots j = 0..m−1)
  const double pfloor = kPivotFloor * th.sigma2;
  int bad = 0;
  double* cb = colbuf[warp];
#pragma unroll
  for (int j = 0; j < 31; ++j) {
    if (j >= m) break;  // warp-uniform
    cb[lane] = r[j];    // column j (entries of rows ≥ j are the live ones)
    __syncwarp();
    const double p = cb[j];
    const double yj = __shfl_sync(0xffffffffu, yk, j);
    bad |= !(p > pfloor) || !(p <= 1.7976931348623157e308);
    const double inv = 1.0 / p;
    const double w = r[j] * inv;  // A(i,j)/p_j for this lane's row i > j
    if (lane > j) {
#pragma unroll
      for (int k = j + 1; k < 32; ++k)
        if (k <= lane) r[k] = fma(-w, cb[k], r[k]);
    }
    if (lane > j) yk = fma(-yj, cb[lane] * inv, yk);  // y row: A(N,k) −= A(N,j) A(k,j)/p_j
    __syncwarp();
  }
  // a8: the point's pivot and y entry live in lane m = N − 1
  double plast = 0.0;
#pragma unroll
  for (int k = 0; k < 32; ++k)
    if (k == m) plast = r[k];
  bad = __any_sync(0xffffffffu, bad);
  if (lane == m) {
    const bool fail = bad || !(plast > pfloor) || !(plast <= 1.7976931348623157e308);
    int st = fail ? kNotPD : kOk;
    uint32_t c[6] = {0, 0, 0, 0, 0, 0};
    const double d = fail ? failed_d() : log(plast);
    const double u = fail ? 0.0 : yk * yk / plast;
    if (!fail) {
      const double t = -0.5 * (u + d + kLn2Pi);
      if (fixed_encode(t, c)) st = kTermRange;
    }
    out_u[q] = u;
    out_d[q] = d;
    accumulate_term(acc, c, st, k_begin + q);
  }
}

cudaError_t launch_cv(int kind, int count, cudaStream_t s, const PointRec* pts, const int32_t* nbr,
                      const BlockDesc* desc, const int32_t* list, const Theta* th, const double* etab, double* u,
                      double* d, unsigned long long* acc, int k_begin) {
  if (count == 0) return cudaSuccess;
  const int grid = (count + kCvWarps - 1) / kCvWarps;
  switch (kind) {
    case 0: bv_cv_kernel<0><<<grid, kCvWarps * 32, 0, s>>>(pts, nbr, desc, list, count, th, etab, u, d, acc, k_begin); break;
    case 1: bv_cv_kernel<1><<<grid, kCvWarps * 32, 0, s>>>(pts, nbr, desc, list, count, th, etab, u, d, acc, k_begin); break;
    case 2: bv_cv_kernel<2><<<grid, kCvWarps * 32, 0, s>>>(pts, nbr, desc, list, count, th, etab, u, d, acc, k_begin); break;
    default: bv_cv_kernel<3><<<grid, kCvWarps * 32, 0, s>>>(pts, nbr, desc, list, count, th, etab, u, d, acc, k_begin); break;
  }
  return cudaGetLastError();
}

}  // namespace bv
