// Do DMMA.8x8x4 and DFMA share one FP64 datapath per SM sub-partition?
// Half the warps run DMMA chains, half DFMA chains; compare the combined
// FLOP rate with each alone.  nvcc -gencode arch=compute_100a,code=sm_100a -O3
#include <cstdio>
#include <cuda_runtime.h>
__global__ void mix(double* out, int iters, int mode) {
  const int w = threadIdx.x >> 5;
  const bool do_dmma = (mode == 0) || (mode == 2 && (w & 1));
  const bool do_dfma = (mode == 1) || (mode == 2 && !(w & 1));
  double s = 0;
  if (do_dmma) {
    double a = threadIdx.x * 1e-3, b = 1.0 - threadIdx.x * 1e-4, c[8][2];
    for (int k = 0; k < 8; ++k) c[k][0] = c[k][1] = 0;
    for (int i = 0; i < iters; ++i)
#pragma unroll
      for (int k = 0; k < 8; ++k)
        asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                     : "+d"(c[k][0]), "+d"(c[k][1]) : "d"(a), "d"(b));
    for (int k = 0; k < 8; ++k) s += c[k][0] + c[k][1];
  }
  if (do_dfma) {
    double acc[8];
    for (int c = 0; c < 8; ++c) acc[c] = threadIdx.x * 1e-9 + c;
    for (int i = 0; i < iters * 8; ++i)
#pragma unroll
      for (int c = 0; c < 8; ++c) acc[c] = fma(acc[c], 1.0000001, 1e-9);
    for (int c = 0; c < 8; ++c) s += acc[c];
  }
  if (s == 1234.5) out[0] = s;
}
int main() {
  double* d; cudaMalloc(&d, 8);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  const int blocks = 148 * 4, threads = 512, iters = 4096;
  const char* names[] = {"dmma only (all warps)", "dfma only (all warps)", "half dmma + half dfma"};
  for (int mode = 0; mode < 3; ++mode) {
    mix<<<blocks, threads>>>(d, 16, mode);
    cudaDeviceSynchronize();
    cudaEventRecord(e0);
    mix<<<blocks, threads>>>(d, iters, mode);
    cudaEventRecord(e1); cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    double warps = (double)blocks * threads / 32;
    double fl_dmma = (mode == 0 ? warps : mode == 2 ? warps / 2 : 0) * iters * 8 * 512.0;
    double fl_dfma = (mode == 1 ? warps : mode == 2 ? warps / 2 : 0) * iters * 8 * 8 * 64.0;
    printf("{\"probe\":\"%s\",\"ms\":%.3f,\"dmma_tflops\":%.2f,\"dfma_tflops\":%.2f,\"total_tflops\":%.2f}\n", names[mode], ms,
           fl_dmma / ms / 1e9, fl_dfma / ms / 1e9, (fl_dmma + fl_dfma) / ms / 1e9);
  }
  return 0;
}
