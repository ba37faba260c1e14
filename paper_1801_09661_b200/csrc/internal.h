// internal.h — liboem.so internals shared by the translation units (not part of the ABI).
#pragma once
#include <cuda.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include <map>
#include <memory>
#include <string>
#include <tuple>
#include <vector>

#include "../../include/oem.h"

namespace oem {

void set_error(const std::string& msg);

// Grown-on-demand device scratch owned by the context (freed in oem_ctx_destroy).
// With OEM_POISON=1 in the environment (a test mode) every ensure() fills the requested bytes
// with 0xFF (a NaN pattern for doubles), so a kernel that reads scratch it did not write shows up
// as a non-finite result instead of silently reusing a previous call's data.
bool poison_enabled();
struct DevBuf {
  void* ptr = nullptr;
  size_t bytes = 0;
  cudaError_t ensure(size_t need) {
    if (need > bytes) {
      if (ptr) cudaFree(ptr);
      ptr = nullptr;
      bytes = 0;
      cudaError_t e = cudaMalloc(&ptr, need);
      if (e != cudaSuccess) return e;
      bytes = need;
    }
    if (poison_enabled() && need > 0) return cudaMemset(ptr, 0xFF, need);
    return cudaSuccess;
  }
  template <typename T> T* as() const { return static_cast<T*>(ptr); }
  void release() {
    if (ptr) cudaFree(ptr);
    ptr = nullptr;
    bytes = 0;
  }
};

struct GramPlan;  // gram.cu

}  // namespace oem

namespace oem {
enum Phase { PH_GRAM = 0, PH_REDUCE = 1, PH_ALLREDUCE = 2, PH_POWER = 3, PH_PATH = 4, PH_NPHASE = 5 };
}

struct oem_ctx {
  int device = 0;
  int nranks = 1, rank = 0;
  int num_sms = 148;
  void* nccl_comm = nullptr;  // ncclComm_t
  oem::DevBuf partial, partial2, counts_dev, partial_scal, packed, tail, plan_tables, path_ws, path_small, logi, lg_part, lg_out, mom_part, mom_out, stage0, stage1, drule_ws, wz, sparse_ws, gram_acc;
  cudaStream_t copy_stream = nullptr;  // f4 host streaming: H2D copies overlap the Gram kernel
  cudaEvent_t ev_copied[2] = {nullptr, nullptr}, ev_used[2] = {nullptr, nullptr};
  std::map<std::tuple<int, int, int64_t, int, int>, std::shared_ptr<oem::GramPlan>> plans;
  // instrumentation (oem_ctx_set_timing / oem_ctx_stats)
  bool timing = false;
  int64_t launches = 0;
  double phase_ms[oem::PH_NPHASE] = {0, 0, 0, 0, 0};
  struct Pending { int phase; cudaEvent_t a, b; };
  std::vector<Pending> pending;
  std::vector<cudaEvent_t> event_pool;
};

namespace oem {

// Records CUDA events around a phase on the launching stream when timing is enabled.
struct PhaseTimer {
  oem_ctx* ctx;
  int phase;
  cudaStream_t st;
  cudaEvent_t a = nullptr;
  PhaseTimer(oem_ctx* c, int ph, cudaStream_t s) : ctx(c), phase(ph), st(s) {
    if (ctx->timing) { a = take(); cudaEventRecord(a, st); }
  }
  ~PhaseTimer() {
    if (a) {
      cudaEvent_t b = take();
      cudaEventRecord(b, st);
      ctx->pending.push_back({phase, a, b});
    }
  }
  cudaEvent_t take() {
    if (!ctx->event_pool.empty()) { cudaEvent_t e = ctx->event_pool.back(); ctx->event_pool.pop_back(); return e; }
    cudaEvent_t e;
    cudaEventCreate(&e);
    return e;
  }
};

// MODE_WZ (internal): the weighted pass of two-panel plans (p > 247), whose CTAs never see a whole
// row: w_i and z_i come precomputed per row (row_weights_kernel) through the y staging box.
enum GramMode { MODE_PLAIN = 0, MODE_FOLD = 1, MODE_WEIGHTED = 2, MODE_WZ = 3 };

// One pass over [X | y] producing the packed upper triangle of the augmented
// (p+1)x(p+1) Gram per fold (nfold = K for MODE_FOLD else 1), raw sums, this rank only.
// packed: nfold * psize (+2 scalars for MODE_WEIGHTED), psize = (p+1)(p+2)/2.
// ones = 1 (MODE_PLAIN / MODE_FOLD, not streamed): the pass is over [X | y | 1] and also writes
// sums[f][j] = column j of the ones column per fold (X^T 1 for j < p, 1^T y at p, the row count
// at p + 1; nfold * (p + 2) doubles), in the same pass.
oem_status gram_pass(oem_ctx* ctx, int mode, const double* X, const double* y, const double* beta, double eps,
                     int64_t n_local, int p, int64_t ldx, int64_t row_offset, int K, double* packed,
                     cudaStream_t st, int accumulate = 0, int want_scal = 1, double* sums = nullptr);
// packed (nfold blocks) -> full symmetric G (nfold*p*p), xty (nfold*p), yty (nfold)
oem_status gram_unpack(oem_ctx* ctx, const double* packed, int nfold, int p, double* G, double* xty, double* yty, cudaStream_t st);
inline int64_t packed_size(int p) { return (int64_t)(p + 1) * (p + 2) / 2; }

oem_status allreduce_sum(oem_ctx* ctx, double* buf, size_t count, cudaStream_t st);
// small host integer sums over ranks (row counts)
oem_status host_allreduce_i64(oem_ctx* ctx, int64_t* vals, int n, cudaStream_t st);

// f1 (logit_ub.cu): out[0..p) = X^T (y - sigma(X beta)), out[p] = loglik, raw sums allreduced
oem_status logit_grad_pass(oem_ctx* ctx, const double* X, const double* y01, const double* beta, int64_t n_local,
                           int p, int64_t ldx, double* out, cudaStream_t st, int want_ll = 1);
// a7 (drule.cu): d[u] = min(Gershgorin, trace(G_u^(2^S))^(1/2^S) (1 + 2Spu)) for the nU normalised
// p x p unit Grams Gn (R#5); d_out device [nU]
oem_status d_rule(oem_ctx* ctx, const double* Gn, int nU, int p, int S, double* d_out, cudaStream_t st);
// c = G beta + 4 g (the raw right-hand side of the upper-bound step)
oem_status ub_rhs(oem_ctx* ctx, const double* G, const double* beta, const double* g, int p, double* c, cudaStream_t st);

}  // namespace oem
