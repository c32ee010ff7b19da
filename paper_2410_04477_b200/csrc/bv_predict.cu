// bv_predict.cu — block-Vecchia prediction, Alg. 2 of arXiv 2410.04477
// (§2.3).
//
// For prediction block B*_i with m_i training neighbours NN (l.6) the paper
// forms Σcon = K(NN, NN), Σcross = K(NN, B*), Σlk = K(B*, B*) (l.7-9) and
//     μ_B* = Σcrossᵀ Σcon⁻¹ y_NN,     Σ_B* = Σlk − Σcrossᵀ Σcon⁻¹ Σcross    (l.10-11)
// (Σcross read as m×l, reading G8).  Both are the Schur complement of the
// joint matrix
//        ⎡ Σcon    Σcross ⎤            ⎡ y_NN ⎤
//        ⎣ Σcrossᵀ Σlk    ⎦  with the  ⎣  0   ⎦  row appended,
// after eliminating its first m columns: the trailing l×l block is Σ_B* and
// the trailing part of the appended row is 0 − μ_B*.  So one CTA per
// prediction block generates the joint lower triangle (Matérn, Eq. (7)) into
// shared memory and runs m right-looking elimination steps; no Σ ever touches
// HBM, and no second factorisation is needed (the paper returns Σ_B* itself,
// "for conditional simulations", l.15; PAPER.md:242 takes its diagonal).
//
// Not the likelihood hot path (the paper predicts once per fit): two columns
// per pass over the trailing matrix (bitwise the same as two rank-1 steps),
// all 16 warps on the trailing update (512 threads, two CTAs per SM: the pass
// is latency-bound; at c4 512 threads beat 256 by 15 %, the two-column pass
// another 1.45x; a register-cached column j and a generic 4-column panel
// (2.61 ms vs 2.31) did not help), packed columns as
// in bv_kernels.cu's v1 kernel.
#include <cuda_runtime.h>
#include <stdint.h>

#include "bv_common.cuh"
#include "matern.cuh"

namespace bv {

namespace {
// packed lower triangle by columns, column j holds rows j..N (row N = the appended row)
__device__ __forceinline__ int pk_off(int j, int Na) { return j * Na - (j * (j - 1)) / 2; }
}  // namespace

constexpr int kPredNT = 512;

__global__ void __launch_bounds__(kPredNT, 2) bv_predict_kernel(const PointRec* __restrict__ train,
                                                             const PointRec* __restrict__ newp,
                                                             const int32_t* __restrict__ nbr,
                                                             const BlockDesc* __restrict__ desc,
                                                             const Theta* __restrict__ theta_dev,
                                                             const int64_t* __restrict__ cov_off,
                                                             double* __restrict__ mean, double* __restrict__ var,
                                                             double* __restrict__ cov, int32_t* __restrict__ status) {
  extern __shared__ __align__(16) double smem[];
  const int b = blockIdx.x;
  const BlockDesc ds = desc[b];
  const int m = ds.m, l = ds.l, N = m + l, Na = N + 1;
  const Theta th = *theta_dev;
  PointRec* P = reinterpret_cast<PointRec*>(smem);
  double* A = smem + 4 * N;
  const int tid = threadIdx.x;

  // l.6-7: neighbours (training records carry y) first, then the block's new points (appended row 0)
  for (int i = tid; i < N; i += kPredNT) {
    PointRec r;
    if (i < m) {
      r = train[nbr[ds.nbr_off + i]];
    } else {
      r = newp[ds.pstart + (i - m)];
      r.v = 0.0;
    }
    P[i] = r;
  }
  __syncthreads();
  // l.7-9: Σcon, Σcross, Σlk (lower triangle of the joint matrix) + the appended row
  for (int j = 0; j < N; ++j) {
    double* cj = A + pk_off(j, Na);
    const PointRec pj = P[j];
    for (int i = j + tid; i <= N; i += kPredNT) cj[i - j] = (i < N) ? matern_from_d2(sqdist(P[i], pj), th) : pj.v;
  }
  __syncthreads();
  // Σcon⁻¹ applied by eliminating the first m columns (l.10-11)
  int fail = 0;
  for (int j = 0; j < m; j += 2) {
    const double* cj = A + pk_off(j, Na);
    const double p = cj[0];
    if (!(p > kPivotFloor * th.sigma2) || !isfinite(p)) {  // uniform across the CTA (reading G15)
      fail = 1;
      break;
    }
    const double inv = 1.0 / p;
    if (j + 1 == m) {  // last (odd) column: one rank-1 step
      // trailing update, one warp per column k = j+1..N−1 (rows k..N, the appended row included)
      for (int k = j + 1 + (tid >> 5); k < N; k += kPredNT / 32) {
        double* ck = A + pk_off(k, Na);
        const double w = cj[k - j] * inv;
        for (int i = k + (tid & 31); i <= N; i += 32) ck[i - k] = fma(-cj[i - j], w, ck[i - k]);
      }
      __syncthreads();
      break;
    }
    // two columns per pass over the trailing matrix: column j+1 first takes step j's update,
    // then every later column takes step j's and step j+1's FMAs back to back — the same
    // operations in the same order as two rank-1 steps, so the result is bitwise identical
    double* c1 = A + pk_off(j + 1, Na);
    {
      const double w = cj[1] * inv;
      for (int i = j + 1 + tid; i <= N; i += kPredNT) c1[i - j - 1] = fma(-cj[i - j], w, c1[i - j - 1]);
    }
    __syncthreads();
    const double p1 = c1[0];
    if (!(p1 > kPivotFloor * th.sigma2) || !isfinite(p1)) {
      fail = 1;
      break;
    }
    const double inv1 = 1.0 / p1;
    for (int k = j + 2 + (tid >> 5); k < N; k += kPredNT / 32) {
      double* ck = A + pk_off(k, Na);
      const double w0 = cj[k - j] * inv;
      const double w1 = c1[k - j - 1] * inv1;
      for (int i = k + (tid & 31); i <= N; i += 32) {
        const double x = fma(-cj[i - j], w0, ck[i - k]);
        ck[i - k] = fma(-c1[i - j - 1], w1, x);
      }
    }
    __syncthreads();
  }
  // l.12: μ_B* = −(appended row), Σ_B* = trailing block; var = its diagonal
  if (!fail) {
    for (int a = tid; a < l; a += kPredNT) {
      const int c = m + a;
      const double* cc = A + pk_off(c, Na);
      mean[ds.pstart + a] = -cc[N - c];
      if (var) var[ds.pstart + a] = cc[0];
    }
    if (cov) {
      double* cb = cov + cov_off[b];
      for (int e = tid; e < l * l; e += kPredNT) {
        const int a = e / l, c = e - a * l;
        const int hi = a > c ? a : c, lo = a > c ? c : a;
        cb[e] = A[pk_off(m + lo, Na) + (hi - lo)];
      }
    }
  }
  if (tid == 0) status[b] = fail ? kNotPD : kOk;
}

size_t predict_smem_bytes(int N) { return (size_t)N * 32 + (size_t)(N + 1) * (N + 2) / 2 * 8; }

cudaError_t prepare_predict(size_t smem) {
  return cudaFuncSetAttribute(bv_predict_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
}

cudaError_t launch_predict(int nblocks, size_t smem, cudaStream_t s, const PointRec* train, const PointRec* newp,
                           const int32_t* nbr, const BlockDesc* desc, const Theta* th, const int64_t* cov_off,
                           double* mean, double* var, double* cov, int32_t* status) {
  if (nblocks == 0) return cudaSuccess;
  bv_predict_kernel<<<nblocks, kPredNT, smem, s>>>(train, newp, nbr, desc, th, cov_off, mean, var, cov, status);
  return cudaGetLastError();
}

}  // namespace bv
