// FP64 box facts for B200: DFMA and DMMA m8n8k4 throughput,
// and the latencies that bound a small-matrix Cholesky's pivot chain.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o fp64_peak fp64_peak.cu
#include <cstdio>
#include <cstdlib>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("CUDA %s at %d\n", cudaGetErrorString(e), __LINE__); exit(1);} } while (0)

template <int CH>
__global__ void dfma_tput(double* out, int iters, double a, double b) {
  double acc[CH];
#pragma unroll
  for (int c = 0; c < CH; ++c) acc[c] = threadIdx.x * 1e-9 + c;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int c = 0; c < CH; ++c) acc[c] = fma(acc[c], a, b);
  }
  double s = 0;
#pragma unroll
  for (int c = 0; c < CH; ++c) s += acc[c];
  if (s == 12345.678) out[0] = s;
}

__global__ void dmma_tput(double* out, int iters) {
  double a = threadIdx.x * 1e-3, b = 1.0 - threadIdx.x * 1e-4;
  double c[8][2];
#pragma unroll
  for (int k = 0; k < 8; ++k) { c[k][0] = 0; c[k][1] = 0; }
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int k = 0; k < 8; ++k)
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                   : "+d"(c[k][0]), "+d"(c[k][1]) : "d"(a), "d"(b));
  }
  double s = 0;
#pragma unroll
  for (int k = 0; k < 8; ++k) s += c[k][0] + c[k][1];
  if (s == 12345.678) out[0] = s;
}

// latency probes: one thread, dependent chain, clock64
__global__ void lat_probe(double* out, long long* cyc, double x0) {
  double x = x0;
  long long t0, t1;
  // DFMA latency
  t0 = clock64();
  for (int i = 0; i < 256; ++i) x = fma(x, 1.0000001, 1e-12);
  t1 = clock64(); cyc[0] = (t1 - t0); out[0] = x;
  // rsqrt (precise) latency
  x = x0 + 1.5; t0 = clock64();
  for (int i = 0; i < 64; ++i) x = rsqrt(x) + 1.0;
  t1 = clock64(); cyc[1] = (t1 - t0); out[1] = x;
  // div latency
  x = x0 + 1.5; t0 = clock64();
  for (int i = 0; i < 64; ++i) x = 1.0 / x + 1.0;
  t1 = clock64(); cyc[2] = (t1 - t0); out[2] = x;
  // sqrt latency
  x = x0 + 1.5; t0 = clock64();
  for (int i = 0; i < 64; ++i) x = sqrt(x) + 1.0;
  t1 = clock64(); cyc[3] = (t1 - t0); out[3] = x;
  // exp latency
  x = x0 * 1e-3; t0 = clock64();
  for (int i = 0; i < 64; ++i) x = exp(-x) ;
  t1 = clock64(); cyc[4] = (t1 - t0); out[4] = x;
  // shfl latency (64-bit)
  x = x0; t0 = clock64();
  for (int i = 0; i < 64; ++i) x = __shfl_sync(0xffffffffu, x, (threadIdx.x + 1) & 31) + 1.0;
  t1 = clock64(); cyc[5] = (t1 - t0); out[5] = x;
  // log latency
  x = x0 + 2.0; t0 = clock64();
  for (int i = 0; i < 64; ++i) x = log(x) + 2.0;
  t1 = clock64(); cyc[6] = (t1 - t0); out[6] = x;
}

// DMMA latency: dependent chain through accumulator
__global__ void dmma_lat(double* out, long long* cyc) {
  double a = threadIdx.x * 1e-3, b = 1.0;
  double c0 = 0, c1 = 0;
  long long t0 = clock64();
  for (int i = 0; i < 128; ++i)
    asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                 : "+d"(c0), "+d"(c1) : "d"(a), "d"(b));
  long long t1 = clock64();
  if (threadIdx.x == 0) cyc[0] = t1 - t0;
  out[threadIdx.x] = c0 + c1;
}

int main() {
  cudaDeviceProp p; CK(cudaGetDeviceProperties(&p, 0));
  int clk_khz = 0; cudaDeviceGetAttribute(&clk_khz, cudaDevAttrClockRate, 0);
  printf("{\"gpu\":\"%s\",\"sms\":%d,\"smem_optin\":%zu,\"regs_per_sm\":%d,\"clock_khz_attr\":%d}\n",
         p.name, p.multiProcessorCount, p.sharedMemPerBlockOptin, p.regsPerMultiprocessor, clk_khz);
  double* d_out; long long* d_cyc;
  CK(cudaMalloc(&d_out, 4096 * sizeof(double))); CK(cudaMalloc(&d_cyc, 64 * sizeof(long long)));
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  int sms = p.multiProcessorCount;
  // DFMA throughput: grid = sms*8 blocks of 256 threads, 8 chains
  for (int rep = 0; rep < 2; ++rep) {
    int iters = 1 << 16; int blocks = sms * 8, threads = 256;
    dfma_tput<8><<<blocks, threads>>>(d_out, 64, 1.0000001, 1e-9);
    CK(cudaDeviceSynchronize());
    cudaEventRecord(e0);
    dfma_tput<8><<<blocks, threads>>>(d_out, iters, 1.0000001, 1e-9);
    cudaEventRecord(e1); CK(cudaEventSynchronize(e1));
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    double flops = 2.0 * 8 * (double)iters * blocks * threads;
    printf("{\"probe\":\"dfma\",\"tflops\":%.3f,\"ms\":%.3f}\n", flops / ms / 1e9, ms);
  }
  for (int rep = 0; rep < 2; ++rep) {
    int iters = 1 << 14; int blocks = sms * 8, threads = 256;
    dmma_tput<<<blocks, threads>>>(d_out, 64);
    CK(cudaDeviceSynchronize());
    cudaEventRecord(e0);
    dmma_tput<<<blocks, threads>>>(d_out, iters);
    cudaEventRecord(e1); CK(cudaEventSynchronize(e1));
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    double flops = 2.0 * 256 * 8 * (double)iters * blocks * (threads / 32);
    printf("{\"probe\":\"dmma_m8n8k4\",\"tflops\":%.3f,\"ms\":%.3f}\n", flops / ms / 1e9, ms);
  }
  lat_probe<<<1, 32>>>(d_out, d_cyc, 0.75); CK(cudaDeviceSynchronize());
  long long cyc[8]; CK(cudaMemcpy(cyc, d_cyc, sizeof(cyc), cudaMemcpyDeviceToHost));
  printf("{\"probe\":\"latency_cyc\",\"dfma\":%.2f,\"rsqrt_plus_add\":%.2f,\"rcpdiv_plus_add\":%.2f,\"sqrt_plus_add\":%.2f,\"exp\":%.2f,\"shfl64_plus_add\":%.2f,\"log_plus_add\":%.2f}\n",
         cyc[0] / 256.0, cyc[1] / 64.0, cyc[2] / 64.0, cyc[3] / 64.0, cyc[4] / 64.0, cyc[5] / 64.0, cyc[6] / 64.0);
  dmma_lat<<<1, 32>>>(d_out, d_cyc); CK(cudaDeviceSynchronize());
  CK(cudaMemcpy(cyc, d_cyc, sizeof(long long), cudaMemcpyDeviceToHost));
  printf("{\"probe\":\"latency_cyc\",\"dmma_m8n8k4\":%.2f}\n", cyc[0] / 128.0);
  return 0;
}
