// stream.cu — f4: out-of-core Gram passes, the big.oem analogue (§5.7,
// X too large for memory is kept out of core and the sufficient statistics are
// accumulated block by block; the OEM iterations need only the p x p result).
//
// X and y stay in (pinned) host memory. Row blocks are copied host -> device on the context's
// copy stream into two staging buffers while the Gram kernel (a2 / a3 on the FP64 tensor cores)
// consumes the other one on the caller's stream: transfer and contraction overlap, and device
// memory holds 2 blocks, not n rows. The packed partial statistics of every block are added in
// block order (gram_reduce_kernel with accumulate = 1), so the result is deterministic and equal
// (up to the order of the split-n sums) to the in-core pass over the same rows.
#include <algorithm>
#include <string>

#include "common.cuh"
#include "internal.h"

namespace oem {

static oem_status ensure_stream_state(oem_ctx* ctx) {
  if (!ctx->copy_stream) OEM_CUDA_TRY(cudaStreamCreateWithFlags(&ctx->copy_stream, cudaStreamNonBlocking));
  for (int i = 0; i < 2; ++i) {
    if (!ctx->ev_copied[i]) OEM_CUDA_TRY(cudaEventCreateWithFlags(&ctx->ev_copied[i], cudaEventDisableTiming));
    if (!ctx->ev_used[i]) OEM_CUDA_TRY(cudaEventCreateWithFlags(&ctx->ev_used[i], cudaEventDisableTiming));
  }
  return OEM_OK;
}

// One streamed pass: blocks of `block_rows` rows (the last one ragged); mode PLAIN or FOLD.
static oem_status stream_pass(oem_ctx* ctx, int mode, const double* Xh, const double* yh, int64_t n_local, int p,
                              int64_t ldx, int64_t row_offset, int K, int64_t block_rows, double* packed,
                              cudaStream_t st) {
  oem_status s;
  if ((s = ensure_stream_state(ctx)) != OEM_OK) return s;
  const int64_t nblk = (n_local + block_rows - 1) / block_rows;
  const size_t xbytes = sizeof(double) * (size_t)block_rows * ldx, ybytes = sizeof(double) * (size_t)block_rows;
  const size_t ybase = (xbytes + 255) / 256 * 256;
  OEM_CUDA_TRY(ctx->stage0.ensure(ybase + ybytes));
  OEM_CUDA_TRY(ctx->stage1.ensure(ybase + ybytes));
  char* stage[2] = {ctx->stage0.as<char>(), ctx->stage1.as<char>()};
  if (nblk == 0) return gram_pass(ctx, mode, nullptr, nullptr, nullptr, 0.0, 0, p, ldx, row_offset, K, packed, st, 0);
  // the copy stream starts after everything already queued on the compute stream
  OEM_CUDA_TRY(cudaEventRecord(ctx->ev_used[0], st));
  OEM_CUDA_TRY(cudaStreamWaitEvent(ctx->copy_stream, ctx->ev_used[0], 0));
  auto issue_copy = [&](int64_t b) -> oem_status {
    const int slot = (int)(b & 1);
    const int64_t r0 = b * block_rows, nr = std::min(block_rows, n_local - r0);
    if (b >= 2) OEM_CUDA_TRY(cudaStreamWaitEvent(ctx->copy_stream, ctx->ev_used[slot], 0));  // slot consumed
    OEM_CUDA_TRY(cudaMemcpyAsync(stage[slot], Xh + r0 * ldx, sizeof(double) * (size_t)nr * ldx,
                                 cudaMemcpyHostToDevice, ctx->copy_stream));
    OEM_CUDA_TRY(cudaMemcpyAsync(stage[slot] + ybase, yh + r0, sizeof(double) * (size_t)nr, cudaMemcpyHostToDevice,
                                 ctx->copy_stream));
    OEM_CUDA_TRY(cudaEventRecord(ctx->ev_copied[slot], ctx->copy_stream));
    return OEM_OK;
  };
  if ((s = issue_copy(0)) != OEM_OK) return s;
  for (int64_t b = 0; b < nblk; ++b) {
    const int slot = (int)(b & 1);
    if (b + 1 < nblk && (s = issue_copy(b + 1)) != OEM_OK) return s;
    OEM_CUDA_TRY(cudaStreamWaitEvent(st, ctx->ev_copied[slot], 0));
    const int64_t r0 = b * block_rows, nr = std::min(block_rows, n_local - r0);
    s = gram_pass(ctx, mode, reinterpret_cast<const double*>(stage[slot]),
                  reinterpret_cast<const double*>(stage[slot] + ybase), nullptr, 0.0, nr, p, ldx, row_offset + r0, K,
                  packed, st, b > 0 ? 1 : 0);
    if (s != OEM_OK) return s;
    OEM_CUDA_TRY(cudaEventRecord(ctx->ev_used[slot], st));
  }
  return OEM_OK;
}

static oem_status check_host(const double* Xh, const double* yh, int64_t n_local, int32_t p, int64_t ldx,
                             int64_t block_rows, const char* who) {
  if (p < 1 || n_local < 0 || ldx < p) OEM_FAIL(OEM_ERR_DIM, std::string(who) + ": need p >= 1, n_local >= 0, ldx >= p");
  if (p > 16383) OEM_FAIL(OEM_ERR_UNSUPPORTED, std::string(who) + ": p > 16383");
  if (n_local > 0 && (!Xh || !yh)) OEM_FAIL(OEM_ERR_INVALID_ARG, std::string(who) + ": null X or y");
  if (block_rows < 32 || block_rows > ((int64_t)1 << 31) - 64)
    OEM_FAIL(OEM_ERR_INVALID_ARG, std::string(who) + ": need 32 <= block_rows < 2^31");
  if (ldx & 1) OEM_FAIL(OEM_ERR_ALIGN, std::string(who) + ": ldx must be even (TMA row pitch)");
  return OEM_OK;
}

}  // namespace oem

using namespace oem;

extern "C" oem_status oem_gram_host(oem_ctx* ctx, const double* X, const double* y, int64_t n_local, int32_t p,
                                    int64_t ldx, int64_t block_rows, double* G, double* xty, double* yty,
                                    int64_t* n_total, void* stream) {
  if (!ctx) OEM_FAIL(OEM_ERR_INVALID_ARG, "null oem_ctx");
  OEM_CUDA_TRY(cudaSetDevice(ctx->device));
  oem_status s;
  if ((s = check_host(X, y, n_local, p, ldx, block_rows, "oem_gram_host")) != OEM_OK) return s;
  if (!G || !xty || !yty) OEM_FAIL(OEM_ERR_INVALID_ARG, "oem_gram_host: null output");
  cudaStream_t st = (cudaStream_t)stream;
  const int64_t psize = packed_size(p);
  OEM_CUDA_TRY(ctx->packed.ensure(sizeof(double) * (psize + 2)));
  double* packed = ctx->packed.as<double>();
  if ((s = stream_pass(ctx, MODE_PLAIN, X, y, n_local, p, ldx, 0, 1, block_rows, packed, st)) != OEM_OK) return s;
  if ((s = allreduce_sum(ctx, packed, psize, st)) != OEM_OK) return s;
  if ((s = gram_unpack(ctx, packed, 1, p, G, xty, yty, st)) != OEM_OK) return s;
  if (n_total) {
    int64_t n = n_local;
    if ((s = host_allreduce_i64(ctx, &n, 1, st)) != OEM_OK) return s;
    *n_total = n;
  }
  return OEM_OK;
}

extern "C" oem_status oem_gram_folds_host(oem_ctx* ctx, const double* X, const double* y, int64_t n_local, int32_t p,
                                          int64_t ldx, int64_t row_offset, int32_t K, int64_t block_rows,
                                          double* G_folds, double* xty_folds, double* yty_folds, int64_t* counts,
                                          void* stream) {
  if (!ctx) OEM_FAIL(OEM_ERR_INVALID_ARG, "null oem_ctx");
  OEM_CUDA_TRY(cudaSetDevice(ctx->device));
  oem_status s;
  if ((s = check_host(X, y, n_local, p, ldx, block_rows, "oem_gram_folds_host")) != OEM_OK) return s;
  if (K < 1 || K > 65535) OEM_FAIL(OEM_ERR_INVALID_ARG, "oem_gram_folds_host: need 1 <= K <= 65535");
  if (row_offset < 0) OEM_FAIL(OEM_ERR_INVALID_ARG, "oem_gram_folds_host: row_offset < 0");
  if (!G_folds || !xty_folds || !yty_folds || !counts) OEM_FAIL(OEM_ERR_INVALID_ARG, "oem_gram_folds_host: null output");
  cudaStream_t st = (cudaStream_t)stream;
  for (int k = 0; k < K; ++k) {
    const int64_t first = ((k - row_offset) % K + K) % K;
    counts[k] = n_local > first ? (n_local - first + K - 1) / K : 0;
  }
  if ((s = host_allreduce_i64(ctx, counts, K, st)) != OEM_OK) return s;
  for (int k = 0; k < K; ++k)
    if (counts[k] == 0) OEM_FAIL(OEM_ERR_EMPTY_FOLD, "oem_gram_folds_host: fold " + std::to_string(k) + " has no rows");
  const int64_t psize = packed_size(p);
  OEM_CUDA_TRY(ctx->packed.ensure(sizeof(double) * (psize * K + 2)));
  double* packed = ctx->packed.as<double>();
  if ((s = stream_pass(ctx, MODE_FOLD, X, y, n_local, p, ldx, row_offset, K, block_rows, packed, st)) != OEM_OK)
    return s;
  if ((s = allreduce_sum(ctx, packed, (size_t)psize * K, st)) != OEM_OK) return s;
  return gram_unpack(ctx, packed, K, p, G_folds, xty_folds, yty_folds, st);
}
