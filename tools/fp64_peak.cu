// FP64 peak microbenchmark for B200 (sm_100a): DFMA (SIMT) vs DMMA (mma.sync f64).
// Establishes the roofline denominator for the Gram pass (SURVEY.md §8(d) "FP64: measured
// on the box with a DMMA microbenchmark"). Prints one JSON line.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o fp64_peak fp64_peak.cu
#include <cstdio>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { \
  fprintf(stderr, "CUDA %s at %s:%d\n", cudaGetErrorString(e), __FILE__, __LINE__); return 1; } } while (0)

template <int CHAINS>
__global__ void dfma_loop(double* out, int iters, double s) {
  double acc[CHAINS];
#pragma unroll
  for (int c = 0; c < CHAINS; ++c) acc[c] = threadIdx.x * 1e-9 + c;
  const double m = 0.999999, a = s;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int c = 0; c < CHAINS; ++c) acc[c] = fma(acc[c], m, a);
  }
  double t = 0;
#pragma unroll
  for (int c = 0; c < CHAINS; ++c) t += acc[c];
  if (t == 12345.678) out[0] = t;  // never true; keeps the loop alive
}

template <int ACC>
__global__ void dmma_loop(double* out, int iters, double s) {
  double d[ACC][2];
  double a = threadIdx.x * 1e-3 + s, b = 1.0 - threadIdx.x * 1e-4;
#pragma unroll
  for (int c = 0; c < ACC; ++c) { d[c][0] = 0; d[c][1] = 0; }
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int c = 0; c < ACC; ++c)
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                   : "+d"(d[c][0]), "+d"(d[c][1]) : "d"(a), "d"(b));
  }
  double t = 0;
#pragma unroll
  for (int c = 0; c < ACC; ++c) t += d[c][0] + d[c][1];
  if (t == 12345.678) out[0] = t;
}

template <typename K>
static float time_kernel(K kern, int grid, int block, int iters, double* out) {
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0); cudaEventCreate(&e1);
  for (int w = 0; w < 3; ++w) kern<<<grid, block>>>(out, iters, 0.5);
  cudaDeviceSynchronize();
  float best = 1e30f;
  for (int r = 0; r < 10; ++r) {
    cudaEventRecord(e0);
    kern<<<grid, block>>>(out, iters, 0.5);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    if (ms < best) best = ms;
  }
  return best;
}

int main() {
  int dev = 0, nsm = 0, clk = 0;
  CK(cudaSetDevice(dev));
  CK(cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev));
  CK(cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, dev));
  double* out; CK(cudaMalloc(&out, 64));
  printf("{\"sms\": %d, \"clock_khz\": %d", nsm, clk);
  // DFMA: 2 flops per FMA
  {
    const int iters = 1 << 14, block = 256;
    for (int occ : {2, 4, 8}) {
      int grid = nsm * occ;
      float ms = time_kernel(dfma_loop<8>, grid, block, iters, out);
      CK(cudaGetLastError());
      double flops = 2.0 * 8 * iters * (double)grid * block;
      printf(", \"dfma_occ%d_tflops\": %.3f", occ, flops / (ms * 1e-3) / 1e12);
    }
  }
  // DMMA m8n8k4: 8*8*4 = 256 FMA = 512 flops per warp-instruction
  {
    const int iters = 1 << 13;
    for (int wps : {4, 8, 16}) {
      int block = 32 * wps, grid = nsm * 2;
      float ms = time_kernel(dmma_loop<8>, grid, block, iters, out);
      CK(cudaGetLastError());
      double flops = 512.0 * 8 * iters * (double)grid * wps;
      printf(", \"dmma_w%d_tflops\": %.3f", wps, flops / (ms * 1e-3) / 1e12);
    }
    for (int wps : {4, 8}) {
      int block = 32 * wps, grid = nsm * 2;
      float ms = time_kernel(dmma_loop<4>, grid, block, iters, out);
      CK(cudaGetLastError());
      double flops = 512.0 * 4 * iters * (double)grid * wps;
      printf(", \"dmma_acc4_w%d_tflops\": %.3f", wps, flops / (ms * 1e-3) / 1e12);
    }
  }
  printf("}\n");
  return 0;
}
