// api.cu — the C ABI of liboem.so (include/oem.h): context, errors, NCCL plumbing and the
// Gram entry points (a2 oem_gram, a3 oem_gram_folds, a4 oem_gram_weighted, a5 combine).
#include <nccl.h>

#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>

#include "common.cuh"
#include "internal.h"

namespace oem {

static thread_local std::string g_last_error;
void set_error(const std::string& msg) { g_last_error = msg; }
bool poison_enabled() {
  static const bool on = [] {
    const char* e = std::getenv("OEM_POISON");
    return e && e[0] == '1';
  }();
  return on;
}

oem_status allreduce_sum(oem_ctx* ctx, double* buf, size_t count, cudaStream_t st) {
  if (!ctx->nccl_comm || count == 0) return OEM_OK;
  PhaseTimer tm(ctx, PH_ALLREDUCE, st);
  ncclResult_t r = ncclAllReduce(buf, buf, count, ncclFloat64, ncclSum, (ncclComm_t)ctx->nccl_comm, st);
  if (r != ncclSuccess) OEM_FAIL(OEM_ERR_NCCL, std::string("ncclAllReduce: ") + ncclGetErrorString(r));
  return OEM_OK;
}

static oem_status check_ctx(oem_ctx* ctx) {
  if (!ctx) OEM_FAIL(OEM_ERR_INVALID_ARG, "null oem_ctx");
  int dev = -1;
  OEM_CUDA_TRY(cudaGetDevice(&dev));
  if (dev != ctx->device) OEM_CUDA_TRY(cudaSetDevice(ctx->device));
  return OEM_OK;
}

static oem_status check_x(const double* X, const double* y, int64_t n_local, int32_t p, int64_t ldx, const char* who) {
  if (p < 1 || n_local < 0 || ldx < p) OEM_FAIL(OEM_ERR_DIM, std::string(who) + ": need p >= 1, n_local >= 0, ldx >= p");
  if (p > 16383) OEM_FAIL(OEM_ERR_UNSUPPORTED, std::string(who) + ": p > 16383");
  if (n_local > 0) {
    if (!X || !y) OEM_FAIL(OEM_ERR_INVALID_ARG, std::string(who) + ": null X or y");
    if ((reinterpret_cast<uintptr_t>(X) & 15) || (reinterpret_cast<uintptr_t>(y) & 15) || (ldx & 1))
      OEM_FAIL(OEM_ERR_ALIGN, std::string(who) + ": X and y must be 16-byte aligned and ldx even (TMA)");
    if (n_local > ((int64_t)1 << 31) - 64) OEM_FAIL(OEM_ERR_UNSUPPORTED, std::string(who) + ": n_local >= 2^31 per rank");
  }
  return OEM_OK;
}

oem_status host_allreduce_i64(oem_ctx* ctx, int64_t* vals, int n, cudaStream_t st) {
  // small integer sums (row counts) across ranks: through a context-owned device buffer and NCCL
  // int64 on the caller's stream (every collective of the communicator is issued on that stream,
  // in the same order on every rank)
  if (!ctx->nccl_comm) return OEM_OK;
  OEM_CUDA_TRY(ctx->counts_dev.ensure(sizeof(int64_t) * (size_t)n));
  int64_t* d = ctx->counts_dev.as<int64_t>();
  OEM_CUDA_TRY(cudaMemcpyAsync(d, vals, sizeof(int64_t) * n, cudaMemcpyHostToDevice, st));
  ncclResult_t r = ncclAllReduce(d, d, n, ncclInt64, ncclSum, (ncclComm_t)ctx->nccl_comm, st);
  if (r != ncclSuccess) OEM_FAIL(OEM_ERR_NCCL, std::string("ncclAllReduce(counts): ") + ncclGetErrorString(r));
  OEM_CUDA_TRY(cudaMemcpyAsync(vals, d, sizeof(int64_t) * n, cudaMemcpyDeviceToHost, st));
  OEM_CUDA_TRY(cudaStreamSynchronize(st));
  return OEM_OK;
}

}  // namespace oem

using namespace oem;

extern "C" {

const char* oem_status_string(oem_status s) {
  switch (s) {
    case OEM_OK: return "OEM_OK";
    case OEM_ERR_INVALID_ARG: return "OEM_ERR_INVALID_ARG";
    case OEM_ERR_DIM: return "OEM_ERR_DIM";
    case OEM_ERR_ALIGN: return "OEM_ERR_ALIGN";
    case OEM_ERR_EMPTY_FOLD: return "OEM_ERR_EMPTY_FOLD";
    case OEM_ERR_NONFINITE: return "OEM_ERR_NONFINITE";
    case OEM_ERR_CUDA: return "OEM_ERR_CUDA";
    case OEM_ERR_NCCL: return "OEM_ERR_NCCL";
    case OEM_ERR_NOMEM: return "OEM_ERR_NOMEM";
    case OEM_ERR_UNSUPPORTED: return "OEM_ERR_UNSUPPORTED";
  }
  return "OEM_ERR_UNKNOWN";
}

const char* oem_last_error(void) { return g_last_error.c_str(); }
const char* oem_version(void) { return "oem-b200 0.1 (sm_100a)"; }

oem_status oem_nccl_unique_id(void* uid128) {
  if (!uid128) OEM_FAIL(OEM_ERR_INVALID_ARG, "null uid buffer");
  ncclUniqueId id;
  ncclResult_t r = ncclGetUniqueId(&id);
  if (r != ncclSuccess) OEM_FAIL(OEM_ERR_NCCL, std::string("ncclGetUniqueId: ") + ncclGetErrorString(r));
  static_assert(sizeof(ncclUniqueId) == 128, "ncclUniqueId size");
  std::memcpy(uid128, &id, 128);
  return OEM_OK;
}

oem_status oem_ctx_create(int device, int nranks, int rank, const void* uid128, oem_ctx** out) {
  if (!out) OEM_FAIL(OEM_ERR_INVALID_ARG, "null out");
  *out = nullptr;
  if (nranks < 1 || rank < 0 || rank >= nranks) OEM_FAIL(OEM_ERR_INVALID_ARG, "bad nranks/rank");
  if (nranks > 1 && !uid128) OEM_FAIL(OEM_ERR_INVALID_ARG, "nranks > 1 needs the NCCL unique id");
  OEM_CUDA_TRY(cudaSetDevice(device));
  oem_ctx* c = new oem_ctx();
  c->device = device;
  c->nranks = nranks;
  c->rank = rank;
  cudaDeviceGetAttribute(&c->num_sms, cudaDevAttrMultiProcessorCount, device);
  if (uid128) {  // nranks == 1 with a uid: a one-rank communicator (the collective path on one GPU)
    ncclUniqueId id;
    std::memcpy(&id, uid128, 128);
    ncclComm_t comm;
    ncclResult_t r = ncclCommInitRank(&comm, nranks, id, rank);
    if (r != ncclSuccess) {
      delete c;
      OEM_FAIL(OEM_ERR_NCCL, std::string("ncclCommInitRank: ") + ncclGetErrorString(r));
    }
    c->nccl_comm = comm;
  }
  *out = c;
  return OEM_OK;
}

oem_status oem_ctx_destroy(oem_ctx* ctx) {
  if (!ctx) return OEM_OK;
  cudaSetDevice(ctx->device);
  cudaDeviceSynchronize();
  if (ctx->nccl_comm) ncclCommDestroy((ncclComm_t)ctx->nccl_comm);
  ctx->plans.clear();
  ctx->partial.release();
  ctx->partial2.release();
  ctx->counts_dev.release();
  ctx->partial_scal.release();
  ctx->packed.release();
  ctx->tail.release();
  ctx->plan_tables.release();
  ctx->path_ws.release();
  ctx->path_small.release();
  ctx->logi.release();
  ctx->drule_ws.release();
  ctx->wz.release();
  ctx->sparse_ws.release();
  ctx->gram_acc.release();
  ctx->lg_part.release();
  ctx->lg_out.release();
  ctx->mom_part.release();
  ctx->mom_out.release();
  ctx->stage0.release();
  ctx->stage1.release();
  if (ctx->copy_stream) cudaStreamDestroy(ctx->copy_stream);
  for (int i = 0; i < 2; ++i) {
    if (ctx->ev_copied[i]) cudaEventDestroy(ctx->ev_copied[i]);
    if (ctx->ev_used[i]) cudaEventDestroy(ctx->ev_used[i]);
  }
  for (auto& pe : ctx->pending) { cudaEventDestroy(pe.a); cudaEventDestroy(pe.b); }
  for (auto e : ctx->event_pool) cudaEventDestroy(e);
  delete ctx;
  return OEM_OK;
}

oem_status oem_ctx_set_timing(oem_ctx* ctx, int enable) {
  if (!ctx) OEM_FAIL(OEM_ERR_INVALID_ARG, "null oem_ctx");
  ctx->timing = enable != 0;
  return OEM_OK;
}

oem_status oem_ctx_stats(oem_ctx* ctx, oem_stats* out, int reset) {
  if (!ctx || !out) OEM_FAIL(OEM_ERR_INVALID_ARG, "null argument");
  OEM_CUDA_TRY(cudaSetDevice(ctx->device));
  for (auto& pe : ctx->pending) {
    OEM_CUDA_TRY(cudaEventSynchronize(pe.b));
    float ms = 0.f;
    OEM_CUDA_TRY(cudaEventElapsedTime(&ms, pe.a, pe.b));
    ctx->phase_ms[pe.phase] += ms;
    ctx->event_pool.push_back(pe.a);
    ctx->event_pool.push_back(pe.b);
  }
  ctx->pending.clear();
  out->launches = ctx->launches;
  out->gram_ms = ctx->phase_ms[PH_GRAM];
  out->reduce_ms = ctx->phase_ms[PH_REDUCE];
  out->allreduce_ms = ctx->phase_ms[PH_ALLREDUCE];
  out->power_ms = ctx->phase_ms[PH_POWER];
  out->path_ms = ctx->phase_ms[PH_PATH];
  if (reset) {
    ctx->launches = 0;
    for (double& v : ctx->phase_ms) v = 0.0;
  }
  return OEM_OK;
}

oem_status oem_gram(oem_ctx* ctx, const double* X, const double* y, int64_t n_local, int32_t p, int64_t ldx,
                    double* G, double* xty, double* yty, int64_t* n_total, void* stream) {
  oem_status s;
  if ((s = check_ctx(ctx)) != OEM_OK) return s;
  if ((s = check_x(X, y, n_local, p, ldx, "oem_gram")) != OEM_OK) return s;
  if (!G || !xty || !yty) OEM_FAIL(OEM_ERR_INVALID_ARG, "oem_gram: null output");
  cudaStream_t st = (cudaStream_t)stream;
  const int64_t psize = packed_size(p);
  OEM_CUDA_TRY(ctx->packed.ensure(sizeof(double) * (psize + 2)));
  double* packed = ctx->packed.as<double>();
  if ((s = gram_pass(ctx, MODE_PLAIN, X, y, nullptr, 0.0, n_local, p, ldx, 0, 1, packed, st)) != OEM_OK) return s;
  if ((s = allreduce_sum(ctx, packed, psize, st)) != OEM_OK) return s;
  if ((s = gram_unpack(ctx, packed, 1, p, G, xty, yty, st)) != OEM_OK) return s;
  if (n_total) {
    int64_t n = n_local;
    if ((s = host_allreduce_i64(ctx, &n, 1, st)) != OEM_OK) return s;
    *n_total = n;
  }
  return OEM_OK;
}

}  // extern "C"

// xsum[f*p + j] = sums[f*(p+2) + j] (j < p), ysum[f] = sums[f*(p+2) + p]
static oem_status unpack_sums(const double* sums, int nfold, int p, double* xsum, double* ysum, cudaStream_t st) {
  OEM_CUDA_TRY(cudaMemcpy2DAsync(xsum, sizeof(double) * p, sums, sizeof(double) * (p + 2), sizeof(double) * p, nfold,
                                 cudaMemcpyDeviceToDevice, st));
  OEM_CUDA_TRY(cudaMemcpy2DAsync(ysum, sizeof(double), sums + p, sizeof(double) * (p + 2), sizeof(double), nfold,
                                 cudaMemcpyDeviceToDevice, st));
  return OEM_OK;
}

// a3 (and its ones-column variant): K raw per-fold sums in one pass
static oem_status gram_folds_impl(oem_ctx* ctx, const double* X, const double* y, int64_t n_local, int32_t p,
                                  int64_t ldx, int64_t row_offset, int32_t K, double* G_folds, double* xty_folds,
                                  double* yty_folds, double* xsum_folds, double* ysum_folds, int64_t* counts,
                                  cudaStream_t st) {
  oem_status s;
  if (K < 1 || K > 65535) OEM_FAIL(OEM_ERR_INVALID_ARG, "oem_gram_folds: need 1 <= K <= 65535");
  if (row_offset < 0) OEM_FAIL(OEM_ERR_INVALID_ARG, "oem_gram_folds: row_offset < 0");
  if (!G_folds || !xty_folds || !yty_folds || !counts) OEM_FAIL(OEM_ERR_INVALID_ARG, "oem_gram_folds: null output");
  // fold sizes are arithmetic on the row indices (host): rows i with (off + i) mod K == k
  for (int k = 0; k < K; ++k) {
    const int64_t first = ((k - row_offset) % K + K) % K;  // first local row in fold k
    counts[k] = n_local > first ? (n_local - first + K - 1) / K : 0;
  }
  if ((s = host_allreduce_i64(ctx, counts, K, st)) != OEM_OK) return s;
  for (int k = 0; k < K; ++k)
    if (counts[k] == 0) OEM_FAIL(OEM_ERR_EMPTY_FOLD, "oem_gram_folds: fold " + std::to_string(k) + " has no rows");
  const int64_t psize = packed_size(p);
  const bool ones = xsum_folds != nullptr;
  const int64_t total = psize * K + (ones ? (int64_t)K * (p + 2) : 0);   // triangles | sums: one allreduce
  OEM_CUDA_TRY(ctx->packed.ensure(sizeof(double) * (total + 2)));
  double* packed = ctx->packed.as<double>();
  double* sums = ones ? packed + psize * K : nullptr;
  if ((s = gram_pass(ctx, MODE_FOLD, X, y, nullptr, 0.0, n_local, p, ldx, row_offset, K, packed, st, 0, 1, sums)) !=
      OEM_OK)
    return s;
  if ((s = allreduce_sum(ctx, packed, (size_t)total, st)) != OEM_OK) return s;
  if ((s = gram_unpack(ctx, packed, K, p, G_folds, xty_folds, yty_folds, st)) != OEM_OK) return s;
  return ones ? unpack_sums(sums, K, p, xsum_folds, ysum_folds, st) : OEM_OK;
}

extern "C" {

oem_status oem_gram_folds(oem_ctx* ctx, const double* X, const double* y, int64_t n_local, int32_t p, int64_t ldx,
                          int64_t row_offset, int32_t K, double* G_folds, double* xty_folds, double* yty_folds,
                          int64_t* counts, void* stream) {
  oem_status s;
  if ((s = check_ctx(ctx)) != OEM_OK) return s;
  if ((s = check_x(X, y, n_local, p, ldx, "oem_gram_folds")) != OEM_OK) return s;
  return gram_folds_impl(ctx, X, y, n_local, p, ldx, row_offset, K, G_folds, xty_folds, yty_folds, nullptr, nullptr,
                         counts, (cudaStream_t)stream);
}

oem_status oem_gram_sums(oem_ctx* ctx, const double* X, const double* y, int64_t n_local, int32_t p, int64_t ldx,
                         double* G, double* xty, double* yty, double* xsum, double* ysum, int64_t* n_total,
                         void* stream) {
  oem_status s;
  if ((s = check_ctx(ctx)) != OEM_OK) return s;
  if ((s = check_x(X, y, n_local, p, ldx, "oem_gram_sums")) != OEM_OK) return s;
  if (!G || !xty || !yty || !xsum || !ysum) OEM_FAIL(OEM_ERR_INVALID_ARG, "oem_gram_sums: null output");
  cudaStream_t st = (cudaStream_t)stream;
  const int64_t psize = packed_size(p);
  // packed triangle | sums [p + 2]: one allreduce for both
  OEM_CUDA_TRY(ctx->packed.ensure(sizeof(double) * (psize + p + 2)));
  double* packed = ctx->packed.as<double>();
  double* sums = packed + psize;
  if ((s = gram_pass(ctx, MODE_PLAIN, X, y, nullptr, 0.0, n_local, p, ldx, 0, 1, packed, st, 0, 1, sums)) != OEM_OK)
    return s;
  if ((s = allreduce_sum(ctx, packed, psize + p + 2, st)) != OEM_OK) return s;
  if ((s = gram_unpack(ctx, packed, 1, p, G, xty, yty, st)) != OEM_OK) return s;
  if ((s = unpack_sums(sums, 1, p, xsum, ysum, st)) != OEM_OK) return s;
  if (n_total) {
    int64_t n = n_local;
    if ((s = host_allreduce_i64(ctx, &n, 1, st)) != OEM_OK) return s;
    *n_total = n;
  }
  return OEM_OK;
}

oem_status oem_gram_folds_sums(oem_ctx* ctx, const double* X, const double* y, int64_t n_local, int32_t p,
                               int64_t ldx, int64_t row_offset, int32_t K, double* G_folds, double* xty_folds,
                               double* yty_folds, double* xsum_folds, double* ysum_folds, int64_t* counts,
                               void* stream) {
  oem_status s;
  if ((s = check_ctx(ctx)) != OEM_OK) return s;
  if ((s = check_x(X, y, n_local, p, ldx, "oem_gram_folds_sums")) != OEM_OK) return s;
  if (!xsum_folds || !ysum_folds) OEM_FAIL(OEM_ERR_INVALID_ARG, "oem_gram_folds_sums: null output");
  return gram_folds_impl(ctx, X, y, n_local, p, ldx, row_offset, K, G_folds, xty_folds, yty_folds, xsum_folds,
                         ysum_folds, counts, (cudaStream_t)stream);
}

oem_status oem_gram_weighted(oem_ctx* ctx, const double* X, const double* y01, const double* beta, int64_t n_local,
                             int32_t p, int64_t ldx, double eps, double* Gw, double* xtwz, double* scalars,
                             void* stream) {
  oem_status s;
  if ((s = check_ctx(ctx)) != OEM_OK) return s;
  if ((s = check_x(X, y01, n_local, p, ldx, "oem_gram_weighted")) != OEM_OK) return s;
  if (!beta || !Gw || !xtwz) OEM_FAIL(OEM_ERR_INVALID_ARG, "oem_gram_weighted: null pointer");
  if (!(eps > 0.0 && eps < 0.5)) OEM_FAIL(OEM_ERR_INVALID_ARG, "oem_gram_weighted: need 0 < eps < 0.5");
  cudaStream_t st = (cudaStream_t)stream;
  const int64_t psize = packed_size(p);
  OEM_CUDA_TRY(ctx->packed.ensure(sizeof(double) * (psize + 2)));
  double* packed = ctx->packed.as<double>();
  const int want_scal = scalars != nullptr;
  if ((s = gram_pass(ctx, MODE_WEIGHTED, X, y01, beta, eps, n_local, p, ldx, 0, 1, packed, st, 0, want_scal)) != OEM_OK)
    return s;
  if ((s = allreduce_sum(ctx, packed, psize + 2, st)) != OEM_OK) return s;
  if ((s = gram_unpack(ctx, packed, 1, p, Gw, xtwz, nullptr, st)) != OEM_OK) return s;
  if (scalars)
    OEM_CUDA_TRY(cudaMemcpyAsync(scalars, packed + psize, 2 * sizeof(double), cudaMemcpyDeviceToDevice, st));
  return OEM_OK;
}

}  // extern "C"
