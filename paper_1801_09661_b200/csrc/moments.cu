// moments.cu — f3: column sums X^T 1 and 1^T y per fold, for the intercept
// (R#3: centering from sufficient statistics, G_c = G - n xbar xbar^T, c_c = c - n xbar ybar) and
// the standardization of centred columns (R#2).
//
// One HBM-bound pass over [X | y]: CTAs own (column chunk, row segment) tiles; thread t of a
// chunk owns one column, so the per-fold accumulators in shared memory are never shared
// between threads; the rows of a segment are read row by row (coalesced across the chunk).
// Segment partials are summed in a fixed order by a second kernel (deterministic).
#include <algorithm>
#include <string>

#include "common.cuh"
#include "internal.h"

namespace oem {

constexpr int MOM_THREADS = 256;
constexpr int MOM_MAXK = 64;  // folds held in shared memory per CTA

// part[seg][k][p + 1]: column sums of fold k over the segment's rows (column p = y)
__global__ void __launch_bounds__(MOM_THREADS) moments_kernel(const double* __restrict__ X, const double* __restrict__ y,
                                                               int64_t n, int p, int64_t ldx, int K, int off_mod,
                                                               int64_t seg_rows, double* __restrict__ part) {
  extern __shared__ double acc[];  // [K][MOM_THREADS + 1]
  const int col = blockIdx.x * MOM_THREADS + threadIdx.x;   // col == p is the y column
  const int seg = blockIdx.y;
  const int64_t r0 = (int64_t)seg * seg_rows, r1 = min(n, r0 + seg_rows);
  for (int k = 0; k < K; ++k) acc[k * (MOM_THREADS + 1) + threadIdx.x] = 0.0;
  if (col <= p) {
    int f = (int)((off_mod + r0) % K);
    int64_t i = r0;
    for (; i + 4 <= r1; i += 4) {  // four rows in flight
      double v[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) v[u] = col < p ? __ldg(X + (i + u) * ldx + col) : __ldg(y + i + u);
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        acc[f * (MOM_THREADS + 1) + threadIdx.x] += v[u];
        if (++f == K) f = 0;
      }
    }
    for (; i < r1; ++i) {
      acc[f * (MOM_THREADS + 1) + threadIdx.x] += col < p ? X[i * ldx + col] : y[i];
      if (++f == K) f = 0;
    }
    for (int k = 0; k < K; ++k) part[((size_t)seg * K + k) * (p + 1) + col] = acc[k * (MOM_THREADS + 1) + threadIdx.x];
  }
}

__global__ void moments_reduce_kernel(const double* __restrict__ part, int nseg, int K, int p, double* __restrict__ xsum,
                                      double* __restrict__ ysum) {
  const int64_t total = (int64_t)K * (p + 1);
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < total; t += (int64_t)gridDim.x * blockDim.x) {
    double s = 0.0;
    for (int g = 0; g < nseg; ++g) s += part[(size_t)g * total + t];  // fixed order
    const int k = (int)(t / (p + 1)), j = (int)(t % (p + 1));
    if (j < p) xsum[(size_t)k * p + j] = s;
    else ysum[k] = s;
  }
}

}  // namespace oem

using namespace oem;

extern "C" oem_status oem_gram_moments(oem_ctx* ctx, const double* X, const double* y, int64_t n_local, int32_t p,
                                       int64_t ldx, int64_t row_offset, int32_t K, double* xsum, double* ysum,
                                       void* stream) {
  if (!ctx) OEM_FAIL(OEM_ERR_INVALID_ARG, "null oem_ctx");
  OEM_CUDA_TRY(cudaSetDevice(ctx->device));
  if (p < 1 || n_local < 0 || ldx < p) OEM_FAIL(OEM_ERR_DIM, "oem_gram_moments: need p >= 1, n_local >= 0, ldx >= p");
  if (K < 1) OEM_FAIL(OEM_ERR_INVALID_ARG, "oem_gram_moments: K >= 1");
  if (K > MOM_MAXK) OEM_FAIL(OEM_ERR_UNSUPPORTED, "oem_gram_moments: K > 64");
  if (!xsum || !ysum || (n_local > 0 && (!X || !y))) OEM_FAIL(OEM_ERR_INVALID_ARG, "oem_gram_moments: null pointer");
  cudaStream_t st = (cudaStream_t)stream;
  const int nchunk = (p + 1 + MOM_THREADS - 1) / MOM_THREADS;
  int nseg = (int)std::max<int64_t>(1, std::min<int64_t>((ctx->num_sms * 8 + nchunk - 1) / nchunk, (n_local + 1023) / 1024));
  const int64_t seg_rows = n_local > 0 ? (n_local + nseg - 1) / nseg : 1;
  if (n_local == 0) nseg = 0;
  const size_t total = (size_t)K * (p + 1);
  OEM_CUDA_TRY(ctx->mom_part.ensure(sizeof(double) * std::max<size_t>(1, (size_t)nseg * total)));
  double* part = ctx->mom_part.as<double>();
  const int off_mod = (int)(((row_offset % K) + K) % K);
  if (nseg > 0) {
    const size_t smem = sizeof(double) * (size_t)K * (MOM_THREADS + 1);
    OEM_CUDA_TRY(cudaFuncSetAttribute(moments_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    ++ctx->launches;
    moments_kernel<<<dim3((unsigned)nchunk, (unsigned)nseg), MOM_THREADS, smem, st>>>(X, y, n_local, p, ldx, K, off_mod,
                                                                                       seg_rows, part);
    OEM_CUDA_TRY(cudaGetLastError());
  }
  // the K*p + K outputs are contiguous per array; reduce into a packed buffer then combine ranks
  OEM_CUDA_TRY(ctx->mom_out.ensure(sizeof(double) * total));
  double* packed = ctx->mom_out.as<double>();
  ++ctx->launches;
  moments_reduce_kernel<<<(int)std::min<size_t>(1024, (total + 255) / 256), 256, 0, st>>>(part, nseg, K, p, packed,
                                                                                           packed + (size_t)K * p);
  OEM_CUDA_TRY(cudaGetLastError());
  oem_status s = allreduce_sum(ctx, packed, total, st);
  if (s != OEM_OK) return s;
  OEM_CUDA_TRY(cudaMemcpyAsync(xsum, packed, sizeof(double) * (size_t)K * p, cudaMemcpyDeviceToDevice, st));
  OEM_CUDA_TRY(cudaMemcpyAsync(ysum, packed + (size_t)K * p, sizeof(double) * K, cudaMemcpyDeviceToDevice, st));
  return OEM_OK;
}
