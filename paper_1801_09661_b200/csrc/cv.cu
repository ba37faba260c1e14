// cv.cu — f2: the fast cross-validation error curve and model selection of
// xval.oem, from the fold sums of one Gram pass (no second pass over X).
//
// The method (§3): the K complement fits use A_(k) = d_(k) I - sum_{c != k}
// X_c^T X_c, i.e. only the per-fold sufficient statistics. Their held-out error needs nothing
// else: for the fit b on the complement of fold k, sum_{i in fold k} (y_i - x_i^T b)^2
// = y_k^T y_k - 2 b^T X_k^T y_k + b^T X_k^T X_k b, all three of which the fold-segmented Gram
// pass already produced (R#33). cv.oem's outputs (P:L601-616 best.model / lambda.min,
// P:L659-660 lambda.1se, P:L689-690 cvup / cvlo) follow from the per-fold errors (R#34-35).
//
// Kernels: cv_err_kernel — one CTA per (lambda block, penalty, fold); the fold Gram rows stream
// from L2/HBM once per block of LB coefficient vectors (LB <= 8 held in shared memory), each
// warp forms row dots t = G_k b for its rows and accumulates b^T t and b^T c_k in a fixed order
// (deterministic). cv_summary_kernel — one CTA: cvm, cvsd, lambda_min, lambda_1se, best model.
#include <algorithm>
#include <string>
#include <vector>

#include "common.cuh"
#include "internal.h"

namespace oem {

constexpr int CV_LB = 8;       // coefficient vectors per CTA
constexpr int CV_THREADS = 256;

__global__ void __launch_bounds__(CV_THREADS) cv_err_kernel(const double* __restrict__ Gf, const double* __restrict__ cf,
                                                             const double* __restrict__ yyf, const double* __restrict__ nk,
                                                             const double* __restrict__ beta, int boff, int p, int nP, int L,
                                                             int LB, const double* __restrict__ xsf,
                                                             const double* __restrict__ ysf,
                                                             const double* __restrict__ b0u, double* __restrict__ err) {
  extern __shared__ __align__(16) double bs[];  // [LB][p]
  __shared__ double red[CV_THREADS / 32][3 * CV_LB];
  const int l0 = blockIdx.x * LB, q = blockIdx.y, k = blockIdx.z;
  const int nb = min(LB, L - l0);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, nw = CV_THREADS / 32;
  // CV: the complement fit of fold k is unit k+1 of the fold-mode path output (boff = 1);
  // compute.loss: unit k's own fit (boff = 0)
  const double* b0 = beta + (((size_t)(k + boff) * nP + q) * L + l0) * p;
  for (int e = threadIdx.x; e < nb * p; e += CV_THREADS) bs[e] = b0[e];
  __syncthreads();
  const double* G = Gf + (size_t)k * p * p;
  const double* c = cf + (size_t)k * p;
  // with an intercept (b0u != null): b^T X_k^T 1 from the fold's column sums (R#33)
  const double* xs = b0u ? xsf + (size_t)k * p : nullptr;
  double quad[CV_LB], lin[CV_LB], lsum[CV_LB];
#pragma unroll
  for (int b = 0; b < CV_LB; ++b) { quad[b] = 0.0; lin[b] = 0.0; lsum[b] = 0.0; }
  for (int j = warp; j < p; j += nw) {
    const double* gr = G + (size_t)j * p;
    double t[CV_LB];
#pragma unroll
    for (int b = 0; b < CV_LB; ++b) t[b] = 0.0;
    for (int kk = lane; kk < p; kk += 32) {
      const double g = gr[kk];
#pragma unroll
      for (int b = 0; b < CV_LB; ++b)
        if (b < nb) t[b] = fma(g, bs[b * p + kk], t[b]);
    }
#pragma unroll
    for (int b = 0; b < CV_LB; ++b) {
      if (b >= nb) break;
      double v = t[b];
#pragma unroll
      for (int o = 16; o >= 1; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
      const double bj = bs[b * p + j];
      quad[b] = fma(bj, v, quad[b]);       // b^T G_k b, rows in this warp's order
      lin[b] = fma(bj, c[j], lin[b]);      // b^T X_k^T y_k
      if (xs) lsum[b] = fma(bj, xs[j], lsum[b]);  // b^T X_k^T 1
    }
  }
  if (lane == 0)
#pragma unroll
    for (int b = 0; b < CV_LB; ++b) {
      red[warp][b] = quad[b];
      red[warp][CV_LB + b] = lin[b];
      red[warp][2 * CV_LB + b] = lsum[b];
    }
  __syncthreads();
  if (threadIdx.x < nb) {
    const int b = threadIdx.x;
    double qs = 0.0, ls = 0.0, ss = 0.0;
    for (int w = 0; w < nw; ++w) { qs += red[w][b]; ls += red[w][CV_LB + b]; ss += red[w][2 * CV_LB + b]; }  // fixed order
    double e = yyf[k] - 2.0 * ls + qs;
    if (b0u) {  // sum_i (y_i - b0 - x_i^T b)^2 = the above - 2 b0 1^T y_k + 2 b0 b^T X_k^T 1 + n_k b0^2
      const double b0 = b0u[((size_t)(k + boff) * nP + q) * L + l0 + b];
      e += b0 * (2.0 * ss - 2.0 * ysf[k] + nk[k] * b0);
    }
    err[((size_t)k * nP + q) * L + l0 + b] = e / nk[k];
  }
}

// cvm(l) = sum_k n_k e_k(l) / n; cvsd(l) = sqrt(sum_k n_k (e_k(l) - cvm(l))^2 / n / (K - 1));
// lambda_min = first minimiser of cvm (the larger lambda on ties, R#35); lambda_1se = the
// largest lambda with cvm <= cvm(lambda_min) + cvsd(lambda_min); best = penalty with the
// smallest min cvm (the earlier penalty on ties).
__global__ void cv_summary_kernel(const double* __restrict__ err, const double* __restrict__ nk, int K, int nP, int L,
                                  double* __restrict__ cvm, double* __restrict__ cvsd, int* __restrict__ sel) {
  double n = 0.0;
  for (int k = 0; k < K; ++k) n += nk[k];
  for (int e = threadIdx.x; e < nP * L; e += blockDim.x) {
    const int q = e / L, l = e % L;
    double m = 0.0;
    for (int k = 0; k < K; ++k) m += nk[k] * err[((size_t)k * nP + q) * L + l];
    m /= n;
    double v = 0.0;
    for (int k = 0; k < K; ++k) {
      const double dv = err[((size_t)k * nP + q) * L + l] - m;
      v += nk[k] * dv * dv;
    }
    cvm[e] = m;
    cvsd[e] = sqrt(v / n / (double)(K - 1));
  }
  __syncthreads();
  if (threadIdx.x < nP) {
    const int q = threadIdx.x;
    const double* cm = cvm + (size_t)q * L;
    int im = 0;
    for (int l = 1; l < L; ++l)
      if (cm[l] < cm[im]) im = l;
    const double thr = cm[im] + cvsd[(size_t)q * L + im];
    int i1 = im;
    for (int l = 0; l <= im; ++l)
      if (cm[l] <= thr) { i1 = l; break; }
    sel[q] = im;
    sel[nP + q] = i1;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    int best = 0;
    for (int q = 1; q < nP; ++q)
      if (cvm[(size_t)q * L + sel[q]] < cvm[(size_t)best * L + sel[best]]) best = q;
    sel[2 * nP] = best;
  }
}

}  // namespace oem

using namespace oem;

extern "C" oem_status oem_cv_error(oem_ctx* ctx, const double* G_folds, const double* xty_folds,
                                   const double* yty_folds, const int64_t* counts, int32_t K, int32_t p, int32_t nP,
                                   int32_t L, const double* beta, const double* xsum_folds,
                                   const double* ysum_folds, const double* intercept, double* err, double* cvm,
                                   double* cvsd, int32_t* idx_min, int32_t* idx_1se, int32_t* best, void* stream) {
  if (!ctx) OEM_FAIL(OEM_ERR_INVALID_ARG, "null oem_ctx");
  OEM_CUDA_TRY(cudaSetDevice(ctx->device));
  if (!G_folds || !xty_folds || !yty_folds || !counts || !beta || !err || !cvm || !cvsd)
    OEM_FAIL(OEM_ERR_INVALID_ARG, "oem_cv_error: null pointer");
  if (intercept && (!xsum_folds || !ysum_folds))
    OEM_FAIL(OEM_ERR_INVALID_ARG, "oem_cv_error: an intercept needs the fold column sums xsum_folds / ysum_folds");
  if (K < 2 || p < 1 || nP < 1 || L < 1) OEM_FAIL(OEM_ERR_DIM, "oem_cv_error: need K >= 2, p, nP, L >= 1");
  if (nP > 64) OEM_FAIL(OEM_ERR_UNSUPPORTED, "oem_cv_error: more than 64 penalties");
  for (int k = 0; k < K; ++k)
    if (counts[k] <= 0) OEM_FAIL(OEM_ERR_EMPTY_FOLD, "oem_cv_error: fold " + std::to_string(k) + " is empty");
  int LB = std::min(CV_LB, L);
  while (LB > 1 && (size_t)LB * p * 8 > 200 * 1024) --LB;
  if ((size_t)LB * p * 8 > 200 * 1024) OEM_FAIL(OEM_ERR_UNSUPPORTED, "oem_cv_error: p too large for one coefficient vector in shared memory");
  cudaStream_t st = (cudaStream_t)stream;
  // scratch: n_k as doubles, selection indices
  OEM_CUDA_TRY(ctx->path_small.ensure(sizeof(double) * (K + 2 * nP + 8)));
  double* nk = ctx->path_small.as<double>();
  int* sel = reinterpret_cast<int*>(nk + K);
  std::vector<double> hn(K);
  for (int k = 0; k < K; ++k) hn[k] = (double)counts[k];
  OEM_CUDA_TRY(cudaMemcpyAsync(nk, hn.data(), sizeof(double) * K, cudaMemcpyHostToDevice, st));
  const size_t smem = (size_t)LB * p * 8;
  OEM_CUDA_TRY(cudaFuncSetAttribute(cv_err_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)std::max<size_t>(smem, 1)));
  dim3 grid((unsigned)((L + LB - 1) / LB), (unsigned)nP, (unsigned)K);
  ++ctx->launches;
  cv_err_kernel<<<grid, CV_THREADS, smem, st>>>(G_folds, xty_folds, yty_folds, nk, beta, 1, p, nP, L, LB, xsum_folds,
                                                ysum_folds, intercept, err);
  OEM_CUDA_TRY(cudaGetLastError());
  ++ctx->launches;
  cv_summary_kernel<<<1, 256, 0, st>>>(err, nk, K, nP, L, cvm, cvsd, sel);
  OEM_CUDA_TRY(cudaGetLastError());
  std::vector<int> hs(2 * nP + 1);
  OEM_CUDA_TRY(cudaMemcpyAsync(hs.data(), sel, sizeof(int) * (2 * nP + 1), cudaMemcpyDeviceToHost, st));
  OEM_CUDA_TRY(cudaStreamSynchronize(st));
  for (int q = 0; q < nP; ++q) {
    if (idx_min) idx_min[q] = hs[q];
    if (idx_1se) idx_1se[q] = hs[nP + q];
  }
  if (best) *best = hs[2 * nP];
  return OEM_OK;
}

extern "C" oem_status oem_path_loss(oem_ctx* ctx, const double* G, const double* xty, const double* yty,
                                    const int64_t* counts, int32_t nG, int32_t p, int32_t nP, int32_t L,
                                    const double* beta, double* loss, void* stream) {
  if (!ctx) OEM_FAIL(OEM_ERR_INVALID_ARG, "null oem_ctx");
  OEM_CUDA_TRY(cudaSetDevice(ctx->device));
  if (!G || !xty || !yty || !counts || !beta || !loss) OEM_FAIL(OEM_ERR_INVALID_ARG, "oem_path_loss: null pointer");
  if (nG < 1 || p < 1 || nP < 1 || L < 1) OEM_FAIL(OEM_ERR_DIM, "oem_path_loss: need nG, p, nP, L >= 1");
  for (int g = 0; g < nG; ++g)
    if (counts[g] <= 0) OEM_FAIL(OEM_ERR_EMPTY_FOLD, "oem_path_loss: count " + std::to_string(g) + " is 0");
  int LB = std::min(CV_LB, L);
  if ((size_t)p * 8 > 200 * 1024) OEM_FAIL(OEM_ERR_UNSUPPORTED, "oem_path_loss: p too large");
  while (LB > 1 && (size_t)LB * p * 8 > 200 * 1024) --LB;
  cudaStream_t st = (cudaStream_t)stream;
  OEM_CUDA_TRY(ctx->path_small.ensure(sizeof(double) * (nG + 8)));
  double* nk = ctx->path_small.as<double>();
  std::vector<double> hn(nG);
  for (int g = 0; g < nG; ++g) hn[g] = (double)counts[g];
  OEM_CUDA_TRY(cudaMemcpyAsync(nk, hn.data(), sizeof(double) * nG, cudaMemcpyHostToDevice, st));
  const size_t smem = (size_t)LB * p * 8;
  OEM_CUDA_TRY(cudaFuncSetAttribute(cv_err_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)std::max<size_t>(smem, 1)));
  dim3 grid((unsigned)((L + LB - 1) / LB), (unsigned)nP, (unsigned)nG);
  ++ctx->launches;
  cv_err_kernel<<<grid, CV_THREADS, smem, st>>>(G, xty, yty, nk, beta, 0, p, nP, L, LB, nullptr, nullptr, nullptr, loss);
  OEM_CUDA_TRY(cudaGetLastError());
  return OEM_OK;
}
