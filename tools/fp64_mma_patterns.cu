// FP64 tensor-core operand-pattern microbenchmark (B200, sm_100a): how fast does DMMA.8x8x4
// run when each instruction uses different A/B fragments (as in a Gram tile) rather than the
// same registers? Compares with a register-blocked DFMA micro-tile. Prints one JSON line.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o fp64_mma_patterns fp64_mma_patterns.cu
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ void dmma(double& d0, double& d1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
               : "+d"(d0), "+d"(d1) : "d"(a), "d"(b));
}

// R x C accumulators, distinct A/B fragments per row/col (register-resident)
template <int R, int C>
__global__ void dmma_grid(double* out, int iters) {
  double acc[R][C][2];
  double a[R], b[C];
#pragma unroll
  for (int r = 0; r < R; ++r) a[r] = threadIdx.x * 1e-3 + r;
#pragma unroll
  for (int c = 0; c < C; ++c) b[c] = 1.0 - threadIdx.x * 1e-4 - c * 1e-2;
#pragma unroll
  for (int r = 0; r < R; ++r)
#pragma unroll
    for (int c = 0; c < C; ++c) acc[r][c][0] = acc[r][c][1] = 0.0;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int r = 0; r < R; ++r)
#pragma unroll
      for (int c = 0; c < C; ++c) dmma(acc[r][c][0], acc[r][c][1], a[r], b[c]);
#pragma unroll
    for (int r = 0; r < R; ++r) a[r] = __shfl_xor_sync(0xffffffff, a[r], 1);
  }
  double t = 0;
#pragma unroll
  for (int r = 0; r < R; ++r)
#pragma unroll
    for (int c = 0; c < C; ++c) t += acc[r][c][0] + acc[r][c][1];
  if (t == 1234.5) out[0] = t;
}

// same, fragments loaded from shared memory every k-step (as in the Gram kernel)
template <int R, int C>
__global__ void dmma_grid_lds(double* out, int iters) {
  __shared__ double tile[4 * 136];
  for (int i = threadIdx.x; i < 4 * 136; i += blockDim.x) tile[i] = i * 1e-3;
  __syncthreads();
  const int lane = threadIdx.x & 31;
  double acc[R][C][2];
#pragma unroll
  for (int r = 0; r < R; ++r)
#pragma unroll
    for (int c = 0; c < C; ++c) acc[r][c][0] = acc[r][c][1] = 0.0;
  const int base = (lane & 3) * 132 + (lane >> 2);
  for (int i = 0; i < iters; ++i) {
    double a[R], b[C];
#pragma unroll
    for (int r = 0; r < R; ++r) a[r] = tile[base + 8 * r];
#pragma unroll
    for (int c = 0; c < C; ++c) b[c] = tile[base + 64 + 8 * c];
#pragma unroll
    for (int r = 0; r < R; ++r)
#pragma unroll
      for (int c = 0; c < C; ++c) dmma(acc[r][c][0], acc[r][c][1], a[r], b[c]);
  }
  double t = 0;
#pragma unroll
  for (int r = 0; r < R; ++r)
#pragma unroll
    for (int c = 0; c < C; ++c) t += acc[r][c][0] + acc[r][c][1];
  if (t == 1234.5) out[0] = t;
}

// same as dmma_grid_lds but each DMMA predicated by a runtime mask (as the Gram kernel's
// diagonal / edge rectangles): do predicated-off DMMAs still occupy the pipe?
template <int R, int C>
__global__ void dmma_grid_mask(double* out, int iters, unsigned mask) {
  __shared__ double tile[4 * 136];
  for (int i = threadIdx.x; i < 4 * 136; i += blockDim.x) tile[i] = i * 1e-3;
  __syncthreads();
  const int lane = threadIdx.x & 31;
  double acc[R][C][2];
#pragma unroll
  for (int r = 0; r < R; ++r)
#pragma unroll
    for (int c = 0; c < C; ++c) acc[r][c][0] = acc[r][c][1] = 0.0;
  const int base = (lane & 3) * 132 + (lane >> 2);
  for (int i = 0; i < iters; ++i) {
    double a[R], b[C];
#pragma unroll
    for (int r = 0; r < R; ++r) a[r] = tile[base + 8 * r];
#pragma unroll
    for (int c = 0; c < C; ++c) b[c] = tile[base + 64 + 8 * c];
#pragma unroll
    for (int r = 0; r < R; ++r)
#pragma unroll
      for (int c = 0; c < C; ++c)
        if ((mask >> (r * C + c)) & 1u) dmma(acc[r][c][0], acc[r][c][1], a[r], b[c]);
  }
  double t = 0;
#pragma unroll
  for (int r = 0; r < R; ++r)
#pragma unroll
    for (int c = 0; c < C; ++c) t += acc[r][c][0] + acc[r][c][1];
  if (t == 1234.5) out[0] = t;
}

// SIMT DFMA micro-tile: each thread an 8x8 block of outputs, operands from smem
__global__ void dfma_tile(double* out, int iters) {
  __shared__ double sa[4][128], sb[4][128];
  for (int i = threadIdx.x; i < 512; i += blockDim.x) { (&sa[0][0])[i] = i * 1e-3; (&sb[0][0])[i] = 1 - i * 1e-4; }
  __syncthreads();
  const int tx = threadIdx.x & 15, ty = threadIdx.x >> 4;
  double acc[8][8];
#pragma unroll
  for (int r = 0; r < 8; ++r)
#pragma unroll
    for (int c = 0; c < 8; ++c) acc[r][c] = 0.0;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      double a[8], b[8];
#pragma unroll
      for (int r = 0; r < 8; r += 2) { double2 v = *reinterpret_cast<double2*>(&sa[k][(ty * 8 + r) & 127]); a[r] = v.x; a[r + 1] = v.y; }
#pragma unroll
      for (int c = 0; c < 8; c += 2) { double2 v = *reinterpret_cast<double2*>(&sb[k][(tx * 8 + c) & 127]); b[c] = v.x; b[c + 1] = v.y; }
#pragma unroll
      for (int r = 0; r < 8; ++r)
#pragma unroll
        for (int c = 0; c < 8; ++c) acc[r][c] = fma(a[r], b[c], acc[r][c]);
    }
  }
  double t = 0;
#pragma unroll
  for (int r = 0; r < 8; ++r)
#pragma unroll
    for (int c = 0; c < 8; ++c) t += acc[r][c];
  if (t == 1234.5) out[0] = t;
}

template <typename K>
static float timeit(K k, int grid, int block, int iters, double* out) {
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  for (int w = 0; w < 2; ++w) k<<<grid, block>>>(out, iters);
  cudaDeviceSynchronize();
  float best = 1e30f;
  for (int r = 0; r < 5; ++r) {
    cudaEventRecord(e0);
    k<<<grid, block>>>(out, iters);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    best = ms < best ? ms : best;
  }
  return best;
}

int main() {
  int nsm;
  cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0);
  double* out;
  cudaMalloc(&out, 64);
  const int it = 4096;
  printf("{");
  for (int wps : {4, 8, 12, 16}) {
    float ms = timeit(dmma_grid<4, 4>, nsm, 32 * wps, it, out);
    printf("\"grid44_w%d\": %.2f, ", wps, 512.0 * 16 * it * nsm * wps / (ms * 1e-3) / 1e12);
  }
  for (int wps : {4, 8}) {
    float ms = timeit(dmma_grid<4, 8>, nsm, 32 * wps, it, out);
    printf("\"grid48_w%d\": %.2f, ", wps, 512.0 * 32 * it * nsm * wps / (ms * 1e-3) / 1e12);
  }
  for (int wps : {4, 8, 12}) {
    float ms = timeit(dmma_grid_lds<4, 4>, nsm, 32 * wps, it, out);
    printf("\"lds44_w%d\": %.2f, ", wps, 512.0 * 16 * it * nsm * wps / (ms * 1e-3) / 1e12);
  }
  for (int wps : {4, 8}) {
    float ms = timeit(dmma_grid_lds<4, 8>, nsm, 32 * wps, it, out);
    printf("\"lds48_w%d\": %.2f, ", wps, 512.0 * 32 * it * nsm * wps / (ms * 1e-3) / 1e12);
  }
  {
    // upper-triangle mask of a 4x4 diagonal rectangle: 10 of 16 DMMAs active
    const unsigned tri = 0xF | (0xE << 4) | (0xC << 8) | (0x8 << 12);
    for (unsigned m : {0xFFFFu, tri}) {
      cudaEvent_t e0, e1;
      cudaEventCreate(&e0);
      cudaEventCreate(&e1);
      dmma_grid_mask<4, 4><<<nsm, 32 * 12>>>(out, it, m);
      cudaEventRecord(e0);
      dmma_grid_mask<4, 4><<<nsm, 32 * 12>>>(out, it, m);
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
      float ms;
      cudaEventElapsedTime(&ms, e0, e1);
      int active = __builtin_popcount(m);
      printf("\"mask44_w12_active%d_useful_tflops\": %.2f, ", active,
             512.0 * active * it * nsm * 12 / (ms * 1e-3) / 1e12);
    }
  }
  {
    float ms = timeit(dmma_grid<1, 1>, nsm * 2, 128, it * 8, out);
    printf("\"grid11_w4x2\": %.2f, ", 512.0 * it * 8 * nsm * 2 * 4 / (ms * 1e-3) / 1e12);
  }
  for (int thr : {256}) {
    float ms = timeit(dfma_tile, nsm, thr, it / 4, out);
    printf("\"dfma_tile8x8_t%d\": %.2f", thr, 2.0 * 64 * 4 * (it / 4) * nsm * (double)thr / (ms * 1e-3) / 1e12);
  }
  printf("}\n");
  return 0;
}
