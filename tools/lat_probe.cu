// Latency microbenchmarks for the path solver's per-iteration chain (developer tool): dependent
// DFMA, DADD, fp64 division, LDS.64, SHFL of a double, bar.sync / bar.red.or with 8 warps.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/lat_probe tools/lat_probe.cu
#include <cstdio>

__global__ void probe(double* out, long long* cyc, double x0, int n) {
  __shared__ double sm[256];
  const int tid = threadIdx.x;
  sm[tid] = x0 + tid;
  __syncthreads();
  double x = x0 + tid * 1e-9, y = 1.0000001;
  long long t0, t1;
  // dependent DFMA chain
  t0 = clock64();
  for (int i = 0; i < n; ++i) x = fma(x, y, 1e-12);
  t1 = clock64();
  if (tid == 0) cyc[0] = t1 - t0;
  // dependent DADD chain
  t0 = clock64();
  for (int i = 0; i < n; ++i) x = x + y;
  t1 = clock64();
  if (tid == 0) cyc[1] = t1 - t0;
  // dependent division chain
  t0 = clock64();
  for (int i = 0; i < n; ++i) x = (x + 1.0) / y;
  t1 = clock64();
  if (tid == 0) cyc[2] = t1 - t0;
  // dependent LDS chain (address depends on the loaded value)
  int idx = tid;
  t0 = clock64();
  for (int i = 0; i < n; ++i) idx = ((int)sm[idx & 255] + i) & 255;
  t1 = clock64();
  if (tid == 0) cyc[3] = t1 - t0;
  x += idx;
  // dependent shuffle chain
  t0 = clock64();
  for (int i = 0; i < n; ++i) x = __shfl_xor_sync(0xffffffffu, x, 1) + 1.0;
  t1 = clock64();
  if (tid == 0) cyc[4] = t1 - t0;
  // barriers (all 8 warps)
  __syncthreads();
  t0 = clock64();
  for (int i = 0; i < n; ++i) __syncthreads();
  t1 = clock64();
  if (tid == 0) cyc[5] = t1 - t0;
  int pr = 0;
  t0 = clock64();
  for (int i = 0; i < n; ++i) pr = __syncthreads_or((tid == (i & 255)) ^ pr);
  t1 = clock64();
  if (tid == 0) cyc[6] = t1 - t0;
  x += pr;
  // LDS + DFMA + STS + barrier round trip (the iteration skeleton)
  t0 = clock64();
  for (int i = 0; i < n; ++i) {
    const double v = sm[(tid + i) & 255];
    sm[tid] = fma(v, y, 1e-12);
    __syncthreads();
  }
  t1 = clock64();
  if (tid == 0) cyc[7] = t1 - t0;
  out[tid] = x + sm[tid];
}

int main() {
  double* out;
  long long* cyc;
  cudaMalloc(&out, 256 * sizeof(double));
  cudaMallocManaged(&cyc, 16 * sizeof(long long));
  const int n = 4096;
  for (int rep = 0; rep < 2; ++rep) probe<<<1, 256>>>(out, cyc, 1.0, n);
  cudaDeviceSynchronize();
  const char* names[8] = {"dfma", "dadd", "ddiv", "lds_dep", "shfl_f64+dadd", "bar.sync(8w)", "bar.red.or(8w)",
                          "lds+dfma+sts+bar"};
  for (int i = 0; i < 8; ++i) printf("%-18s %.1f cycles\n", names[i], (double)cyc[i] / n);
  return 0;
}
