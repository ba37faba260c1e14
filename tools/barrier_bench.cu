// Microbenchmark (developer tool): cost of a grid-wide counter barrier among C co-resident CTAs
// of 512 threads on B200, with and without a 16 KB L2 vector reload per iteration.
#include <cstdio>
#include <cuda_runtime.h>
__device__ __forceinline__ void red_release_add(unsigned* p, unsigned v) {
  asm volatile("red.release.gpu.global.add.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ unsigned ld_relaxed(const unsigned* p) {
  unsigned v;
  asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__global__ void bar_kernel(unsigned* cnt, int iters, int reload, double* vec, double* sink) {
  __shared__ double sv[2048];
  const unsigned C = gridDim.x;
  double acc = 0.0;
  for (int t = 0; t < iters; ++t) {
    if (reload && threadIdx.x < 2) vec[(t & 1) * 2048 + blockIdx.x * 2 + threadIdx.x] = t;
    __syncthreads();
    if (threadIdx.x == 0) {
      red_release_add(cnt, 1u);
      const unsigned target = (t + 1) * C;
      while (ld_relaxed(cnt) < target) {}
      asm volatile("fence.acq_rel.gpu;" ::: "memory");
    }
    __syncthreads();
    if (reload) {
      for (int k = threadIdx.x; k < 2000; k += blockDim.x) sv[k] = __ldcg(&vec[(t & 1) * 2048 + k]);
      __syncthreads();
      acc += sv[(threadIdx.x * 7) & 1023];
    }
  }
  if (acc == -1.0) sink[0] = acc;
}
int main() {
  unsigned* cnt;
  double *vec, *sink;
  cudaMalloc(&cnt, 4);
  cudaMalloc(&vec, 2 * 2048 * 8);
  cudaMalloc(&sink, 8);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  const int iters = 20000;
  for (int reload = 0; reload < 2; ++reload)
    for (int C : {8, 16, 34, 64, 100, 148}) {
      cudaMemset(cnt, 0, 4);
      bar_kernel<<<C, 512>>>(cnt, 100, reload, vec, sink);
      cudaMemset(cnt, 0, 4);
      cudaEventRecord(a);
      bar_kernel<<<C, 512>>>(cnt, iters, reload, vec, sink);
      cudaEventRecord(b);
      cudaEventSynchronize(b);
      float ms;
      cudaEventElapsedTime(&ms, a, b);
      printf("{\"C\": %d, \"reload\": %d, \"us_per_barrier\": %.3f}\n", C, reload, ms * 1e3 / iters);
    }
  return 0;
}
