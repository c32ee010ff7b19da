// bv_kernels.cu — small helper kernels of the host runtime.
//
// The e2e entry point bv_loglik_host_y copies the caller's observations (host
// order) to the device and scatters them into the permuted point records the
// block kernels gather from (the y row of every joint matrix, Alg. 1 l.14,
// PAPER.md:597).
#include <cuda_runtime.h>
#include <stdint.h>

#include "bv_common.cuh"
#include "matern.cuh"

namespace bv {

// e2e: scatter host-order observations into the permuted point records.
__global__ void bv_scatter_y_kernel(const double* __restrict__ y, const int32_t* __restrict__ perm_of_id, int64_t n,
                                    PointRec* __restrict__ pts) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) pts[perm_of_id[i]].v = y[i];
}

// ------------------------------------------------------------------ launchers
cudaError_t launch_scatter_y(const double* y, const int32_t* perm_of_id, int64_t n, PointRec* pts, cudaStream_t s) {
  if (n == 0) return cudaSuccess;
  bv_scatter_y_kernel<<<(unsigned)((n + 255) / 256), 256, 0, s>>>(y, perm_of_id, n, pts);
  return cudaGetLastError();
}

}  // namespace bv
