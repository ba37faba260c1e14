// logit_ub.cu — f1: the Hessian upper-bound logistic step (PAPER.md P:L385-389
// "we optionally employ an approximation to the Hessian using an upper-bound of w_i = 0.25").
//
// With w_i = 1/4 the weighted Gram of every outer step is X^T X / 4: it is formed ONCE by the
// plain Gram pass (a2), and d_w once from it. The working response z = eta + (y - mu)/0.25
// (R#27) then gives X^T W z = (X^T X / 4) beta + X^T (y - mu), so each outer step only needs
// the gradient g = X^T (y - sigma(X beta)): one streaming pass over [X | y] that is HBM-bound
// (8 (p+1) bytes and ~4p flops per row), instead of a weighted SYRK per step.
//
// logit_grad_kernel: warps own interleaved rows of a contiguous per-CTA row range; lane l holds
// columns {2l, 2l+1} + 64 s (16-byte loads, coalesced), beta in registers; per row eta is a
// warp-wide reduction, then g += (y - mu) x stays in registers. Per-CTA partials are summed in
// a fixed order (warp order, then CTA order in logit_grad_reduce_kernel): deterministic.
#include <algorithm>
#include <string>
#include <vector>

#include "common.cuh"
#include "internal.h"

namespace oem {

constexpr int LG_THREADS = 256;
constexpr int LG_WARPS = LG_THREADS / 32;

__device__ __forceinline__ double softplus_dev(double e) { return e > 0.0 ? e + log1p(exp(-e)) : log1p(exp(e)); }

template <int PS, bool LL>  // double2 slots per lane: p <= 64 * PS; LL: also the log-likelihood
__global__ void __launch_bounds__(LG_THREADS, PS >= 8 ? 1 : 2) logit_grad_kernel(const double* __restrict__ X, const double* __restrict__ y,
                                                                const double* __restrict__ beta, int64_t n, int p,
                                                                int64_t ldx, int64_t rows_per_cta,
                                                                double* __restrict__ part) {
  __shared__ double acc[64 * PS + 1];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t r0 = (int64_t)blockIdx.x * rows_per_cta;
  const int64_t r1 = min(n, r0 + rows_per_cta);
  double2 b[PS], g[PS];
#pragma unroll
  for (int s = 0; s < PS; ++s) {
    const int c = 2 * (lane + 32 * s);
    b[s].x = c < p ? beta[c] : 0.0;
    b[s].y = c + 1 < p ? beta[c + 1] : 0.0;
    g[s] = make_double2(0.0, 0.0);
  }
  double ll = 0.0;
  constexpr int RB = PS <= 2 ? 4 : 2;  // rows per warp step
  for (int64_t i0 = r0 + warp * RB; i0 < r1; i0 += LG_WARPS * RB) {
    double2 x[RB][PS];
    double yv[RB];
#pragma unroll
    for (int rb = 0; rb < RB; ++rb) {
      const int64_t i = i0 + rb;
      const bool ok = i < r1;
      const double* xr = X + (ok ? i : r0) * ldx;
#pragma unroll
      for (int s = 0; s < PS; ++s) {
        const int c = 2 * (lane + 32 * s);
        // rows are 16-byte aligned with an even pitch (checked at the ABI), so the pair at
        // c = p-1 (p odd) stays inside the padded row; its second half is masked
        x[rb][s] = (ok && c < p) ? __ldg(reinterpret_cast<const double2*>(xr + c)) : make_double2(0.0, 0.0);
        if (c + 1 >= p) x[rb][s].y = 0.0;
      }
      yv[rb] = ok ? __ldg(y + i) : 0.0;
    }
    // eta of every row of the step (butterfly sums: every lane holds all of them); lane rb does
    // row rb's scalar work (exp, division, log-likelihood) once, not the whole warp per row
    double e[RB];
#pragma unroll
    for (int rb = 0; rb < RB; ++rb) {
      double v = 0.0;
#pragma unroll
      for (int s = 0; s < PS; ++s) v = fma(b[s].x, x[rb][s].x, fma(b[s].y, x[rb][s].y, v));
#pragma unroll
      for (int o = 16; o >= 1; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
      e[rb] = v;
    }
    double rmine = 0.0;
#pragma unroll
    for (int rb = 0; rb < RB; ++rb)
      if (lane == rb && i0 + rb < r1) {
        const double mu = 1.0 / (1.0 + exp(-e[rb]));   // sigma(eta)
        rmine = yv[rb] - mu;
        if (LL) ll += yv[rb] * e[rb] - softplus_dev(e[rb]);
      }
#pragma unroll
    for (int rb = 0; rb < RB; ++rb) {
      const double r = __shfl_sync(0xffffffffu, rmine, rb);   // 0 for rows past the segment
#pragma unroll
      for (int s = 0; s < PS; ++s) {
        g[s].x = fma(r, x[rb][s].x, g[s].x);
        g[s].y = fma(r, x[rb][s].y, g[s].y);
      }
    }
  }
  // the log-likelihood terms sit on lanes 0 .. RB-1: fixed-order butterfly to every lane
#pragma unroll
  for (int o = 16; o >= 1; o >>= 1) ll += __shfl_xor_sync(0xffffffffu, ll, o);
  // per-CTA sum in warp order (deterministic), one warp at a time into shared memory
  for (int w = 0; w < LG_WARPS; ++w) {
    if (warp == w) {
#pragma unroll
      for (int s = 0; s < PS; ++s) {
        const int c = 2 * (lane + 32 * s);
        acc[c] = (w == 0 ? 0.0 : acc[c]) + g[s].x;
        acc[c + 1] = (w == 0 ? 0.0 : acc[c + 1]) + g[s].y;
      }
      if (lane == 0) acc[64 * PS] = (w == 0 ? 0.0 : acc[64 * PS]) + ll;
    }
    __syncthreads();
  }
  double* out = part + (size_t)blockIdx.x * (p + 1);
  for (int j = threadIdx.x; j <= p; j += LG_THREADS) out[j] = acc[j < p ? j : 64 * PS];
}

// out[j] = sum over CTAs (fixed order) of part[cta][j], j <= p (out[p] = loglik)
__global__ void logit_grad_reduce_kernel(const double* __restrict__ part, int ncta, int p, double* __restrict__ out) {
  for (int j = blockIdx.x * blockDim.x + threadIdx.x; j <= p; j += gridDim.x * blockDim.x) {
    double s = 0.0;
    for (int c = 0; c < ncta; ++c) s += part[(size_t)c * (p + 1) + j];
    out[j] = s;
  }
}

// raw right-hand side of the upper-bound step: c_j = sum_k G_jk beta_k + 4 g_j, so that
// c / (4n) = (X^T X / 4n) beta + X^T (y - mu) / n = X^T W z / n with w = 1/4 (R#27)
__global__ void ub_rhs_kernel(const double* __restrict__ G, const double* __restrict__ beta, const double* __restrict__ g,
                              int p, double* __restrict__ c) {
  const int warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, lane = threadIdx.x & 31;
  if (warp >= p) return;
  const double* gr = G + (size_t)warp * p;
  double s = 0.0;
  for (int k = lane; k < p; k += 32) s = fma(gr[k], beta[k], s);
#pragma unroll
  for (int o = 16; o >= 1; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
  if (lane == 0) c[warp] = s + 4.0 * g[warp];
}

oem_status ub_rhs(oem_ctx* ctx, const double* G, const double* beta, const double* g, int p, double* c, cudaStream_t st) {
  ++ctx->launches;
  ub_rhs_kernel<<<(p * 32 + 255) / 256, 256, 0, st>>>(G, beta, g, p, c);
  OEM_CUDA_TRY(cudaGetLastError());
  return OEM_OK;
}

template <int PS>
static oem_status launch_lg(int grid, const double* X, const double* y, const double* beta, int64_t n, int p,
                            int64_t ldx, int64_t rpc, double* part, bool ll, cudaStream_t st) {
  if (ll) logit_grad_kernel<PS, true><<<grid, LG_THREADS, 0, st>>>(X, y, beta, n, p, ldx, rpc, part);
  else logit_grad_kernel<PS, false><<<grid, LG_THREADS, 0, st>>>(X, y, beta, n, p, ldx, rpc, part);
  OEM_CUDA_TRY(cudaGetLastError());
  return OEM_OK;
}

// g (p) and loglik (1) as raw sums over this rank's rows into out[0..p]; allreduced over ranks.
// want_ll = 0: out[p] = 0 (the upper-bound fit stops on the change in beta and needs no
// log-likelihood; dropping its log1p / exp per row takes a third of the per-row fp64 work)
oem_status logit_grad_pass(oem_ctx* ctx, const double* X, const double* y01, const double* beta, int64_t n_local,
                           int p, int64_t ldx, double* out, cudaStream_t st, int want_ll) {
  if (p > 512) OEM_FAIL(OEM_ERR_UNSUPPORTED, "oem_logit_grad: p > 512 (register-resident beta and gradient)");
  const int grid = std::max(1, std::min<int>(ctx->num_sms * 4, (int)((n_local + 255) / 256)));
  const int64_t rpc = n_local > 0 ? (n_local + grid - 1) / grid : 0;
  OEM_CUDA_TRY(ctx->lg_part.ensure(sizeof(double) * (size_t)grid * (p + 1)));
  double* part = ctx->lg_part.as<double>();
  if (n_local == 0) {
    OEM_CUDA_TRY(cudaMemsetAsync(out, 0, sizeof(double) * (p + 1), st));
  } else {
    PhaseTimer tm(ctx, PH_GRAM, st);
    ++ctx->launches;
    oem_status s;
    if (p <= 64) s = launch_lg<1>(grid, X, y01, beta, n_local, p, ldx, rpc, part, want_ll != 0, st);
    else if (p <= 128) s = launch_lg<2>(grid, X, y01, beta, n_local, p, ldx, rpc, part, want_ll != 0, st);
    else if (p <= 256) s = launch_lg<4>(grid, X, y01, beta, n_local, p, ldx, rpc, part, want_ll != 0, st);
    else s = launch_lg<8>(grid, X, y01, beta, n_local, p, ldx, rpc, part, want_ll != 0, st);
    if (s != OEM_OK) return s;
    PhaseTimer tm2(ctx, PH_REDUCE, st);
    ++ctx->launches;
    logit_grad_reduce_kernel<<<(p + 256) / 256, 256, 0, st>>>(part, grid, p, out);
    OEM_CUDA_TRY(cudaGetLastError());
  }
  return allreduce_sum(ctx, out, (size_t)p + 1, st);
}

}  // namespace oem

using namespace oem;

extern "C" oem_status oem_logit_grad(oem_ctx* ctx, const double* X, const double* y01, const double* beta,
                                     int64_t n_local, int32_t p, int64_t ldx, double* g, double* loglik, void* stream) {
  if (!ctx) OEM_FAIL(OEM_ERR_INVALID_ARG, "null oem_ctx");
  OEM_CUDA_TRY(cudaSetDevice(ctx->device));
  if (p < 1 || n_local < 0 || ldx < p) OEM_FAIL(OEM_ERR_DIM, "oem_logit_grad: need p >= 1, n_local >= 0, ldx >= p");
  if (!g || !beta || (n_local > 0 && (!X || !y01))) OEM_FAIL(OEM_ERR_INVALID_ARG, "oem_logit_grad: null pointer");
  if (n_local > 0 && ((reinterpret_cast<uintptr_t>(X) & 15) || (ldx & 1)))
    OEM_FAIL(OEM_ERR_ALIGN, "oem_logit_grad: X must be 16-byte aligned with an even ldx");
  cudaStream_t st = (cudaStream_t)stream;
  OEM_CUDA_TRY(ctx->lg_out.ensure(sizeof(double) * (p + 1)));
  double* out = ctx->lg_out.as<double>();
  oem_status s = logit_grad_pass(ctx, X, y01, beta, n_local, p, ldx, out, st, loglik != nullptr);
  if (s != OEM_OK) return s;
  OEM_CUDA_TRY(cudaMemcpyAsync(g, out, sizeof(double) * p, cudaMemcpyDeviceToDevice, st));
  if (loglik) OEM_CUDA_TRY(cudaMemcpyAsync(loglik, out + p, sizeof(double), cudaMemcpyDeviceToDevice, st));
  return OEM_OK;
}
