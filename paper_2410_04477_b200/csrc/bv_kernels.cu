// bv_kernels.cu — sm_100a kernels of the block-Vecchia log-likelihood.
//
// Per permuted position k the path is Alg. 1 l.10-29:
// gather → Matérn (l.11-13) → POTRF Σcon (l.17) → TRSM/TRSV (l.18-19) →
// GEMM/GEMV Schur complement (l.20-23) → POTRF Σnew (l.24) → TRSV (l.25) →
// dot / logdet (l.26-27) → term t_k (l.29).  All of it is ONE elimination of
// the joint matrix
//        ⎡ Σcon    Σcross  y_NN ⎤
//        ⎢ Σcrossᵀ Σlk     y_B  ⎥      (N = m + l rows, plus the y row)
//        ⎣ y_NNᵀ   y_Bᵀ    ·    ⎦
// in exact arithmetic: after the first m pivots the trailing block is Σnew
// and the y row holds y_B − μnew in the L⁻¹ basis; the last l pivots p_j give
// d = Σ_{j≥m} log p_j (= 2 log det L') and the forward-eliminated y row gives
// u = Σ_{j≥m} z_j²/p_j (= vᵀv).  (DESIGN.md §4 derives this; the oracle keeps
// Alg. 1's nine separate steps.)
#include <cuda_runtime.h>
#include <stdint.h>

#include "bv_common.cuh"
#include "matern.cuh"

namespace bv {

// ---------------------------------------------------------------------------
// v1 kernel: one CTA per block, whole augmented lower triangle in shared
// memory (packed by columns), one right-looking elimination step per column.
// Column j occupies rows j..N (row N = the y row):
//   off(j) = j·(N+1) − j(j−1)/2,  entry (i, j) at off(j) + i − j.
__device__ __forceinline__ int col_off(int j, int Na) { return j * Na - (j * (j - 1)) / 2; }

template <int NT>
__global__ void __launch_bounds__(NT) bv_block_v1_kernel(const PointRec* __restrict__ pts,
                                                         const int32_t* __restrict__ nbr,
                                                         const BlockDesc* __restrict__ desc,
                                                         const int32_t* __restrict__ list,
                                                         const Theta* __restrict__ theta_dev,
                                                         double* __restrict__ out_u, double* __restrict__ out_d,
                                                         unsigned long long* __restrict__ acc, int k_begin,
                                                         double jit) {
  extern __shared__ __align__(16) double smem[];
  const int q = list[blockIdx.x];
  const BlockDesc ds = desc[q];
  const int m = ds.m, l = ds.l, N = m + l, Na = N + 1;
  const Theta th = *theta_dev;
  PointRec* P = reinterpret_cast<PointRec*>(smem);  // N records
  double* A = smem + 4 * N;                          // packed augmented lower triangle
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  constexpr int NW = NT / 32;

  // a2. gather: neighbours first (rows 0..m−1), then the block's points
  for (int i = tid; i < N; i += NT) {
    const int src = (i < m) ? nbr[ds.nbr_off + i] : ds.pstart + (i - m);
    P[i] = pts[src];
  }
  __syncthreads();
  // a3. covariance generation (lower triangle) + the y row
  for (int j = 0; j < N; ++j) {
    double* cj = A + col_off(j, Na);
    const PointRec pj = P[j];
    for (int i = j + tid; i <= N; i += NT) {
      double v;
      if (i < N) v = matern_from_d2(sqdist(P[i], pj), th);
      else v = pj.v;
      if (i == j) v += jit;  // optional jitter retry: ε·σ² on the joint diagonal (reading G15b)
      cj[i - j] = v;
    }
  }
  __syncthreads();

  // a4-a7. elimination, one column per step; column j itself is never written
  double logdet = 0.0, quad = 0.0;
  int fail = 0;
  for (int j = 0; j < N; ++j) {
    const double* cj = A + col_off(j, Na);
    const double p = cj[0];
    if (!(p > kPivotFloor * th.sigma2) || !isfinite(p)) {  // uniform across the CTA (reading G15)
      fail = 1;
      break;
    }
    const double inv = 1.0 / p;
    if (tid == 0 && j >= m) {  // a8. d = Σ log p_j ; u = Σ z_j²/p_j
      logdet += log(p);
      const double z = cj[N - j];
      quad += z * z * inv;
    }
    for (int k = j + 1 + warp; k < N; k += NW) {
      double* ck = A + col_off(k, Na);
      const double w = cj[k - j] * inv;
      for (int i = k + lane; i <= N; i += 32) ck[i - k] -= cj[i - j] * w;
    }
    __syncthreads();
  }
  if (tid == 0) {
    int st = fail ? kNotPD : kOk;
    uint32_t c[6] = {0, 0, 0, 0, 0, 0};
    if (!fail) {
      const double t = -0.5 * (quad + logdet + (double)l * kLn2Pi);
      if (fixed_encode(t, c)) st = kTermRange;
      out_u[q] = quad;
      out_d[q] = logdet;
    } else {
      out_u[q] = 0.0;
      out_d[q] = failed_d();
    }
    accumulate_term(acc, c, st, k_begin + q);  // a9
  }
}

// e2e: scatter host-order observations into the permuted point records.
__global__ void bv_scatter_y_kernel(const double* __restrict__ y, const int32_t* __restrict__ perm_of_id, int64_t n,
                                    PointRec* __restrict__ pts) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) pts[perm_of_id[i]].v = y[i];
}

// ------------------------------------------------------------------ launchers
size_t v1_smem_bytes(int Nmax) {
  const size_t Na = (size_t)Nmax + 1;
  const size_t packed = (size_t)Nmax * Na - ((size_t)Nmax * (Nmax - 1)) / 2;
  return (4 * (size_t)Nmax + packed) * sizeof(double);
}

constexpr int kV1Threads = 256;

// Called once in bv_setup (outside stream capture) with the largest bucket.
cudaError_t prepare_block_v1(int Nmax) {
  return cudaFuncSetAttribute(bv_block_v1_kernel<kV1Threads>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                              (int)v1_smem_bytes(Nmax));
}

cudaError_t launch_block_v1(int nblocks, int Nmax, cudaStream_t s, const PointRec* pts, const int32_t* nbr,
                            const BlockDesc* desc, const int32_t* list, const Theta* th, double* u, double* d,
                            unsigned long long* acc, int k_begin, double jit) {
  constexpr int NT = kV1Threads;
  const size_t smem = v1_smem_bytes(Nmax);
  if (nblocks == 0) return cudaSuccess;
  bv_block_v1_kernel<NT><<<nblocks, NT, smem, s>>>(pts, nbr, desc, list, th, u, d, acc, k_begin, jit);
  return cudaGetLastError();
}

cudaError_t launch_scatter_y(const double* y, const int32_t* perm_of_id, int64_t n, PointRec* pts, cudaStream_t s) {
  if (n == 0) return cudaSuccess;
  bv_scatter_y_kernel<<<(unsigned)((n + 255) / 256), 256, 0, s>>>(y, perm_of_id, n, pts);
  return cudaGetLastError();
}

}  // namespace bv
