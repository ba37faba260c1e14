// logistic.cu — the proximal-Newton logistic path (§4) driven to
// convergence on the device: a4 fused weighted Gram per outer step (gram.cu, MODE_WEIGHTED),
// a6-a9 single-lambda OEM inner solve (path.cu), and a one-CTA kernel for the outer test
// max |beta_new - beta|. The host loop reads one scalar per outer step.
#include <cmath>
#include <cstring>
#include <vector>

#include "common.cuh"
#include "internal.h"

namespace oem {

// delta = max_j |nb_j - b_j|, then b <- nb (one CTA, deterministic tree).
__global__ void delta_copy_kernel(const double* __restrict__ nb, double* __restrict__ b, int p, double* delta) {
  __shared__ double red[32];
  double m = 0.0;
  for (int j = threadIdx.x; j < p; j += blockDim.x) {
    const double v = nb[j];
    m = fmax(m, fabs(v - b[j]));
    b[j] = v;
  }
  for (int o = 16; o > 0; o >>= 1) m = fmax(m, __shfl_xor_sync(0xffffffffu, m, o));
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = m;
  __syncthreads();
  if (threadIdx.x == 0) {
    double r = 0.0;
    for (int i = 0; i < (int)(blockDim.x >> 5); ++i) r = fmax(r, red[i]);
    *delta = r;
  }
}

}  // namespace oem

using namespace oem;

extern "C" void oem_logistic_cfg_default(oem_logistic_cfg* c) {
  if (!c) return;
  c->nlambda = 50;
  c->lambda_min_ratio = 1e-3;
  c->lambda = nullptr;
  c->tol_in = 1e-11;
  c->maxit_in = 100000;
  c->tol_out = 1e-10;
  c->outer_maxit = 100;
  c->eps = 1e-5;
  c->d_squarings = 12;
  c->var_w = nullptr;
  c->group = nullptr;
  c->ngroups = 0;
  c->grp_w = nullptr;
  c->hessian_upper_bound = 0;
}

extern "C" oem_status oem_fit_logistic(oem_ctx* ctx, const double* X, const double* y01, int64_t n_local, int32_t p,
                                       int64_t ldx, const oem_penalty* pen, const oem_logistic_cfg* cfg_in,
                                       double* beta_out, double* lambda_out, int32_t* outer_iters,
                                       int64_t* inner_iters, uint8_t* converged, void* stream) {
  if (!ctx || !pen || !beta_out || !lambda_out || !outer_iters || !inner_iters || !converged)
    OEM_FAIL(OEM_ERR_INVALID_ARG, "oem_fit_logistic: null pointer");
  OEM_CUDA_TRY(cudaSetDevice(ctx->device));
  oem_logistic_cfg cfg;
  if (cfg_in) cfg = *cfg_in;
  else oem_logistic_cfg_default(&cfg);
  if (pen->family > OEM_GRP_SCAD || pen->family < OEM_LASSO)
    OEM_FAIL(OEM_ERR_INVALID_ARG, "oem_fit_logistic: families lasso, EN, MCP, SCAD, group lasso / MCP / SCAD");
  const bool grp = pen->family >= OEM_GRP_LASSO;
  if (grp && (!cfg.group || cfg.ngroups < 1)) OEM_FAIL(OEM_ERR_INVALID_ARG, "oem_fit_logistic: group penalty needs cfg.group");
  if (cfg.group)
    for (int j = 0; j < p; ++j)
      if (cfg.group[j] < 0 || cfg.group[j] >= cfg.ngroups) OEM_FAIL(OEM_ERR_INVALID_ARG, "oem_fit_logistic: group id out of range");
  if (cfg.nlambda < 1 || cfg.outer_maxit < 1 || !(cfg.tol_out > 0.0))
    OEM_FAIL(OEM_ERR_INVALID_ARG, "oem_fit_logistic: need nlambda >= 1, outer_maxit >= 1, tol_out > 0");
  cudaStream_t st = (cudaStream_t)stream;
  const int L = cfg.nlambda;
  const size_t pp = (size_t)p * p;
  // workspace: Gw | cw | sc(2) | beta | beta_new | lam1 | d1 | delta | it1 (i64) | cv1 (u8)
  const size_t nd = pp + 5 * (size_t)p + 16;
  OEM_CUDA_TRY(ctx->logi.ensure(sizeof(double) * nd));
  double* Gw = ctx->logi.as<double>();
  double* cw = Gw + pp;
  double* sc = cw + p;
  double* beta = sc + 2;
  double* bnew = beta + p;
  double* lam1 = bnew + p;
  double* d1 = lam1 + 1;
  double* delta = d1 + 1;
  int64_t* it1 = reinterpret_cast<int64_t*>(delta + 1);
  uint8_t* cv1 = reinterpret_cast<uint8_t*>(it1 + 1);
  OEM_CUDA_TRY(cudaMemsetAsync(beta, 0, sizeof(double) * p, st));
  // global n
  int64_t n_total = n_local;
  if (ctx->nccl_comm) {
    // reuse the oem_gram row-count plumbing: sum over ranks through a tiny NCCL call
    double* tmp = delta;
    double v = (double)n_local;
    OEM_CUDA_TRY(cudaMemcpyAsync(tmp, &v, sizeof(double), cudaMemcpyHostToDevice, st));
    oem_status s = allreduce_sum(ctx, tmp, 1, st);
    if (s != OEM_OK) return s;
    OEM_CUDA_TRY(cudaMemcpyAsync(&v, tmp, sizeof(double), cudaMemcpyDeviceToHost, st));
    OEM_CUDA_TRY(cudaStreamSynchronize(st));
    n_total = (int64_t)llround(v);
  }
  if (n_total < 1) OEM_FAIL(OEM_ERR_DIM, "oem_fit_logistic: no rows");
  const bool ub = cfg.hessian_upper_bound != 0;
  oem_status s;
  double* gb = nullptr;  // upper-bound mode: X^T (y - mu) and loglik (p + 1)
  if (ub) {
    // f1: X^T X once (a2 pass + combine); the gradient at beta = 0 gives lambda_max (R#14)
    if (p > 512) OEM_FAIL(OEM_ERR_UNSUPPORTED, "oem_fit_logistic: hessian_upper_bound needs p <= 512");
    OEM_CUDA_TRY(ctx->lg_out.ensure(sizeof(double) * (2 * (size_t)p + 2)));
    gb = ctx->lg_out.as<double>() + p + 1;
    int64_t nt = 0;
    s = oem_gram(ctx, X, y01, n_local, p, ldx, Gw, cw, sc, &nt, stream);
    if (s != OEM_OK) return s;
    s = logit_grad_pass(ctx, X, y01, beta, n_local, p, ldx, gb, st, 0);
    if (s != OEM_OK) return s;
  } else {
    // a4 at beta = 0: gives lambda_max (R#14) and the first outer step's weighted Gram
    s = oem_gram_weighted(ctx, X, y01, beta, n_local, p, ldx, cfg.eps, Gw, cw, nullptr, stream);
    if (s != OEM_OK) return s;
  }
  std::vector<double> lam(L);
  if (cfg.lambda) {
    for (int l = 0; l < L; ++l) lam[l] = cfg.lambda[l];
  } else {
    std::vector<double> hc(p), hw(p, 1.0);
    OEM_CUDA_TRY(cudaMemcpyAsync(hc.data(), ub ? gb : cw, sizeof(double) * p, cudaMemcpyDeviceToHost, st));
    if (cfg.var_w) OEM_CUDA_TRY(cudaMemcpyAsync(hw.data(), cfg.var_w, sizeof(double) * p, cudaMemcpyDeviceToHost, st));
    OEM_CUDA_TRY(cudaStreamSynchronize(st));
    const double scale = pen->family == OEM_ENET ? pen->alpha : 1.0;
    double lmax = 0.0;
    // c_w at beta = 0 is sum_i x_ij (y_i - 1/2), normalised exactly as the path solver does
    // (times 1/n, prep_units_kernel), so beta = 0 is an exact fixed point at lambda_max
    const double inv_n = 1.0 / (double)n_total;
    if (!grp) {
      for (int j = 0; j < p; ++j)
        if (hw[j] > 0.0) lmax = std::fmax(lmax, std::fabs(hc[j] * inv_n) / (scale * hw[j]));
    } else {  // max_k ||c_{g_k}|| / c_k (R#12, R#14)
      std::vector<double> ss(cfg.ngroups, 0.0);
      std::vector<int> sz(cfg.ngroups, 0);
      for (int j = 0; j < p; ++j) {
        const double c = hc[j] * inv_n;
        ss[cfg.group[j]] += c * c;
        sz[cfg.group[j]]++;
      }
      for (int g = 0; g < cfg.ngroups; ++g) {
        const double cg = cfg.grp_w ? cfg.grp_w[g] : std::sqrt((double)sz[g]);
        if (cg > 0.0) lmax = std::fmax(lmax, std::sqrt(ss[g]) / cg);
      }
    }
    for (int l = 0; l < L; ++l)
      lam[l] = L == 1 ? lmax : lmax * std::exp(((double)l / (double)(L - 1)) * std::log(cfg.lambda_min_ratio));
  }
  OEM_CUDA_TRY(cudaMemcpyAsync(lambda_out, lam.data(), sizeof(double) * L, cudaMemcpyHostToDevice, st));
  oem_path_cfg pc;
  oem_path_cfg_default(&pc);
  pc.nlambda = 1;
  pc.tol = cfg.tol_in;
  pc.maxit = cfg.maxit_in;
  pc.var_w = cfg.var_w;
  pc.d_squarings = cfg.d_squarings;
  pc.group = cfg.group;
  pc.ngroups = cfg.ngroups;
  pc.grp_w = cfg.grp_w;
  bool have_gram = true;
  // upper-bound mode: G/(4n) and d_w are the same at every step; d_w is computed by the first
  // solve and passed in afterwards
  const int64_t n4 = 4 * n_total;
  bool have_d = false;
  double hd = 0.0;
  for (int l = 0; l < L; ++l) {
    int32_t o = 0;
    int64_t inner = 0;
    uint8_t ok = 0;
    pc.lambda = &lam[l];
    while (o < cfg.outer_maxit) {
      if (ub) {
        if (!have_gram) {
          s = logit_grad_pass(ctx, X, y01, beta, n_local, p, ldx, gb, st, 0);
          if (s != OEM_OK) return s;
        }
        s = ub_rhs(ctx, Gw, beta, gb, p, cw, st);  // c = X^T X beta + 4 X^T (y - mu)
        if (s != OEM_OK) return s;
      } else if (!have_gram) {
        s = oem_gram_weighted(ctx, X, y01, beta, n_local, p, ldx, cfg.eps, Gw, cw, nullptr, stream);
        if (s != OEM_OK) return s;
      }
      have_gram = false;
      if (ub) {
        s = oem_fit_path(ctx, Gw, cw, &n4, 1, p, pen, 1, &pc, have_d ? &hd : nullptr, beta, bnew, lam1, it1, cv1,
                         d1, stream);
        if (s == OEM_OK && !have_d) {
          OEM_CUDA_TRY(cudaMemcpyAsync(&hd, d1, sizeof(double), cudaMemcpyDeviceToHost, st));
          OEM_CUDA_TRY(cudaStreamSynchronize(st));
          have_d = true;
        }
      } else {
        s = oem_fit_path(ctx, Gw, cw, &n_total, 1, p, pen, 1, &pc, nullptr, beta, bnew, lam1, it1, cv1, d1, stream);
      }
      if (s != OEM_OK) return s;
      ++ctx->launches;
      delta_copy_kernel<<<1, 256, 0, st>>>(bnew, beta, p, delta);
      OEM_CUDA_TRY(cudaGetLastError());
      double hd = 0.0;
      int64_t hit = 0;
      OEM_CUDA_TRY(cudaMemcpyAsync(&hd, delta, sizeof(double), cudaMemcpyDeviceToHost, st));
      OEM_CUDA_TRY(cudaMemcpyAsync(&hit, it1, sizeof(int64_t), cudaMemcpyDeviceToHost, st));
      OEM_CUDA_TRY(cudaStreamSynchronize(st));
      ++o;
      inner += hit;
      if (!std::isfinite(hd)) OEM_FAIL(OEM_ERR_NONFINITE, "oem_fit_logistic: non-finite iterate");
      if (hd <= cfg.tol_out) { ok = 1; break; }
    }
    OEM_CUDA_TRY(cudaMemcpyAsync(beta_out + (size_t)l * p, beta, sizeof(double) * p, cudaMemcpyDeviceToDevice, st));
    outer_iters[l] = o;
    inner_iters[l] = inner;
    converged[l] = ok;
  }
  OEM_CUDA_TRY(cudaStreamSynchronize(st));
  return OEM_OK;
}
