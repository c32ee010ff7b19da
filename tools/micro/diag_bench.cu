// Microbenchmark: latency of one diagonal-tile factorisation (the block's
// serial chain) in isolation — one warp, clock64 around N calls.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -I paper_2410_04477_b200/csrc tools/micro/diag_bench.cu
#include <cstdio>
#include <cuda_runtime.h>
#define BV_MINB 4
#include "../../paper_2410_04477_b200/csrc/bv_block_v2.cu"
#include "diag_variants.cuh"

using namespace bv;

__global__ void diag_lat(double* out, long long* cyc, int iters) {
  __shared__ __align__(16) double tile[64], diagL[64], rinv[8], misc[8];
  const int lane = threadIdx.x;
  // SPD tile: A = I*9 + ones
  for (int e = lane; e < 64; e += 32) tile[e] = ((e >> 3) == (e & 7) ? 9.0 : 0.0) + 1.0 + 0.01 * (e & 7);
  if (lane < 8) misc[lane] = 0.0;
  __syncwarp();
  long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
    factor_diag_tile(tile, diagL, rinv, misc, 0, 0, 1000, lane);
    __syncwarp();
  }
  long long t1 = clock64();
  if (lane == 0) { cyc[0] = (t1 - t0) / iters; out[0] = misc[0] + diagL[9] + rinv[3]; }
}

template <bool ONE>
__global__ void diag_fast_lat(double* out, long long* cyc, int iters, int slot) {
  __shared__ __align__(16) double tile[64], diagL[64], rinv[8];
  const int lane = threadIdx.x;
  for (int e = lane; e < 64; e += 32) tile[e] = ((e >> 3) == (e & 7) ? 9.0 : 0.0) + 1.0 + 0.01 * (e & 7);
  __syncwarp();
  double prod = 1.0, qd = 0.0; int nbad = 0;
  long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
    diag_inlane_fast<ONE>(tile, diagL, rinv, 0, 0, 1000, lane, prod, nbad, qd);
    int ex; prod = frexp(prod, &ex); nbad += ex & 0;
    __syncwarp();
  }
  long long t1 = clock64();
  if (lane == 0) { cyc[slot] = (t1 - t0) / iters; out[slot] = prod + diagL[9] + rinv[3] + nbad + qd; }
}

__global__ void log_lat(double* out, long long* cyc, int iters) {
  double x = 1.7 + threadIdx.x * 1e-3;
  long long t0 = clock64();
  for (int i = 0; i < iters; ++i) x = log(x) + 1.5;
  long long t1 = clock64();
  if (threadIdx.x == 0) { cyc[1] = (t1 - t0) / iters; out[1] = x; }
}

__global__ void rsq_lat(double* out, long long* cyc, int iters) {
  double x = 1.7 + threadIdx.x * 1e-3;
  long long t0 = clock64();
  for (int i = 0; i < iters; ++i) x = rsqrt_pos(x) + 1.5;
  long long t1 = clock64();
  if (threadIdx.x == 0) { cyc[2] = (t1 - t0) / iters; out[2] = x; }
}

__global__ void rsq_err(double* out) {
  // max relative error of rsqrt_pos1 / rsqrt_pos vs 1/sqrt (IEEE sqrt + IEEE div), over a log-spaced sweep
  double e1 = 0, e2 = 0;
  for (int i = 0; i < 4096; ++i) {
    const double x = exp2(-60.0 + 120.0 * ((blockIdx.x * 32 + threadIdx.x) * 4096 + i) / (4096.0 * 32 * 64));
    const double ref = 1.0 / sqrt(x);
    e1 = fmax(e1, fabs(rsqrt_pos1(x) - ref) / ref);
    e2 = fmax(e2, fabs(rsqrt_pos(x) - ref) / ref);
  }
  atomicMax((unsigned long long*)&out[4], __double_as_longlong(e1));
  atomicMax((unsigned long long*)&out[5], __double_as_longlong(e2));
}

int main() {
  double* d; long long* c; cudaMalloc(&d, 64); cudaMalloc(&c, 64);
  diag_lat<<<1, 32>>>(d, c, 1000); log_lat<<<1, 32>>>(d, c, 1000); rsq_lat<<<1, 32>>>(d, c, 1000);
  diag_fast_lat<false><<<1, 32>>>(d, c, 1000, 3); diag_fast_lat<true><<<1, 32>>>(d, c, 1000, 4);
  cudaDeviceSynchronize();
  long long h[5]; cudaMemcpy(h, c, 40, cudaMemcpyDeviceToHost);
  cudaMemset(d, 0, 64); rsq_err<<<64, 32>>>(d); double hd[6]; cudaMemcpy(hd, d, 48, cudaMemcpyDeviceToHost);
  printf("{\"rsqrt_pos1_max_rel_err\": %.3e, \"rsqrt_pos_max_rel_err\": %.3e}\n", hd[4], hd[5]);
  printf("{\"diag_tile_factor_cycles\": %lld, \"log_cycles\": %lld, \"rsqrt_pos_plus_add_cycles\": %lld, \"inlane_fast\": %lld, \"inlane_fast_onestep\": %lld}\n", h[0], h[1], h[2], h[3], h[4]);
  return 0;
}
