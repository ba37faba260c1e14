// gram.cu — K2/K3/K7: the Gram pass of OEM on sm_100a.
//
// What it computes: the sufficient statistics X^T X, X^T y,
// y^T y of the linear model as ONE symmetric rank-n update of the augmented matrix Z = [X | y]
// (upper triangle of Z^T Z only), optionally split by fold (fold(i) = (off+i) mod K)
// or weighted by the proximal-Newton weights with the working response in the augmented
// column (w_i = mu(1-mu), z_i = eta + (y - mu)/w, eta = x_i^T beta).
//
// How (B200-first):
//  * Row blocks of X (BK = 32 rows) and of y stream HBM -> shared memory through TMA
//    (cp.async.bulk.tensor, mbarrier complete_tx) in a multi-stage ring fed by one elected
//    producer thread; consumers release stages through a second mbarrier ring.
//  * The contraction runs on the FP64 tensor cores: mma.sync m8n8k4 f64 (SASS DMMA.8x8x4;
//    tcgen05 has no f64 kind on sm_100a). Each consumer warp owns one "job": a rectangle of 8x8
//    output blocks of the upper triangle with register accumulators. Jobs have compile-time
//    shapes (full 4x4 / 4x8 / 4xk rectangles, and upper triangles on the diagonal) so the
//    warp issues exactly the useful DMMAs: a predicated-off DMMA still costs a full pipe slot
//    on B200 (tools/fp64_mma_patterns.cu: 10 of 16 active -> 62% of peak).
//  * The smem row pitch is ld = 4 or 12 (mod 16) doubles so the fragment loads (4 rows x 8
//    columns per half-warp pair) are bank-conflict free; fragment addresses are one base
//    register plus compile-time offsets.
//  * Small p (8 ceil((p+1)/8) + 4 <= 256): one TMA box holds the whole augmented row ("single
//    panel"); jobs are spread over U CTA types that stream the same rows (the weighted pass
//    computes eta/w/z per row from the full row in smem, fused). Large p: 128-column panel
//    pairs (I, J), I <= J, one CTA type per tile, 4x8 jobs.
//  * Rows are split into segments (split-n); every (CTA type, segment) writes its own partial
//    blocks and a second kernel sums segments in a fixed order -> deterministic, no atomics.
//    The result is packed (upper triangle of the augmented matrix) for one NCCL allreduce
//    when the rows are sharded over GPUs.
#include <algorithm>
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <vector>

#include "common.cuh"
#include "internal.h"

namespace oem {

constexpr int BK = 32;      // rows per pipeline stage
constexpr int MAXST = 6;    // max pipeline stages
constexpr int NWC_MAX = 16; // consumer (MMA) warps per CTA: 16 for single-panel plans, 8 for two-panel ones
__host__ __device__ constexpr int nwc_of(bool two) { return two ? 8 : 16; }
constexpr int ORD_W = 2;    // ordered epilogue: interleaved accumulation chains per (fold, tile type)
constexpr int NRW = 2;      // WEIGHTED: row warps (eta, mu, w, z per row, one stage ahead of the MMA warps)
__host__ __device__ constexpr int gram_threads(int mode, bool two) { return (nwc_of(two) + (mode == 2 ? NRW : 0) + 1) * 32; }

// job kinds: shape (R x C blocks) and which blocks are issued. Full kinds F4c issue all 4 x c
// blocks; triangular kinds (T1..T4 and T4Fk = T4 followed by k full columns) issue (r, c) with
// c >= r. The Fxx/T4Fk kinds with C > 4 appear only in two-panel plans (128-column panels);
// F45..F47 and T4F1..T4F3 are trimmed jobs at the last panel (columns beyond the augmented
// matrix are never issued).
enum JobKind { J_NONE = 0, J_F44, J_T4, J_F41, J_F42, J_F43, J_T1, J_T2, J_T3, J_F48, J_T4F4,
               J_F45, J_F46, J_F47, J_T4F1, J_T4F2, J_T4F3, J_NKIND };
__host__ __device__ constexpr int kind_R(int k) {
  return k == J_NONE ? 0 : k == J_T1 ? 1 : k == J_T2 ? 2 : k == J_T3 ? 3 : 4;
}
__host__ __device__ constexpr int kind_C(int k) {
  return k == J_NONE ? 0 : k == J_F41 || k == J_T1 ? 1 : k == J_F42 || k == J_T2 ? 2
       : k == J_F43 || k == J_T3 ? 3 : k == J_F48 || k == J_T4F4 ? 8 : k == J_F45 || k == J_T4F1 ? 5
       : k == J_F46 || k == J_T4F2 ? 6 : k == J_F47 || k == J_T4F3 ? 7 : 4;
}
__host__ __device__ constexpr bool kind_tri(int k) {
  return k == J_T4 || k == J_T1 || k == J_T2 || k == J_T3 || k == J_T4F4 || k == J_T4F1 || k == J_T4F2 || k == J_T4F3;
}
// block (r, c) of the job is issued: all blocks for full kinds, c >= r for triangular ones
__host__ __device__ constexpr bool kind_active(int k, int r, int c) { return kind_tri(k) ? c >= r : true; }
// the kind with this shape (J_NONE if there is none)
static int kind_of(int R, int C, bool tri) {
  for (int k = 1; k < J_NKIND; ++k)
    if (kind_R(k) == R && kind_C(k) == C && kind_tri(k) == tri) return k;
  return J_NONE;
}
__host__ __device__ constexpr int kind_cost(int k) {
  int n = 0;
  for (int r = 0; r < kind_R(k); ++r)
    for (int c = 0; c < kind_C(k); ++c) n += kind_active(k, r, c) ? 1 : 0;
  return n;
}

struct Job {
  int32_t bi0, bj0;   // top-left 8x8 block (global block coordinates)
  int32_t kind;
  int32_t pad;
};
struct CtaDesc {
  int32_t a0, b0;     // first column of panel A / panel B
  int32_t same;       // panel B == panel A
  int32_t njob;       // consumer warps with work (arrivals per stage release)
  Job job[NWC_MAX];   // slot w = consumer warp w (SMSP w % 4); J_NONE = idle
};

struct GramParams {
  int p, nb, ld, U, nseg, ST, two_panel, nblk;
  int U_off;          // CTA types [0, U_off) are dispatched first (the costlier off-diagonal tiles)
  int64_t nrows;      // PLAIN/WEIGHTED: n_local rows; FOLD: nq = floor(n_local / K) full groups
  int64_t seg_rows;   // rows (FOLD: groups) per segment, multiple of BK
  int K, off_mod;     // FOLD
  int ytma, ystride;  // y through TMA (1D map, or 2D [nq][Kpad] map for folds); ys row stride
  const double* y;    // LDG fallback (odd K folds)
  const double* beta;
  double eps;
  int want_scal;          // WEIGHTED: accumulate sum w and the log-likelihood (else zeros)
  int ones;               // PLAIN / FOLD: a ones column at p + 1 (Z = [X | y | 1])
  double* partial;        // [nfold][nseg][nblk][64]
  int ordered;            // 1: segments add into accum in segment order (no partial buffer)
  unsigned* ticket;       // [ORD_W][U] next link of each chain allowed to add (zero at launch)
  double* accum;          // [ORD_W][nblk][64]
  double* partial_scal;   // WEIGHTED: [nseg][2]
  const CtaDesc* ctas;
  const int32_t* blk_of;  // [nb*nb] -> packed upper block index
  uint32_t xbox_bytes;    // one X box
  uint32_t ybox_bytes;    // y box per stage (0 if LDG fallback)
  int stage_doubles;      // per-stage smem footprint (doubles)
  int ys_off;             // offset of ys within a stage (doubles)
};

struct Cons {
  double* smem;
  uint64_t* full;
  uint64_t* empty;
  uint64_t* ready;    // WEIGHTED: row quantities of the stage are in shared memory
  int warp, lane, nst, seg, fold, kprime, u;
  int64_t r0, r1;
  int a0, b0;
  bool two;
  Job job;
  const double* beta_s;
  double* scal_s;     // WEIGHTED: [NRW][2] per-row-warp (sum w, loglik)
  int njob;           // consumer warps with a job in this CTA
  unsigned* done_s;   // ordered epilogue: warps of this CTA that have added their blocks
};

__device__ __forceinline__ unsigned ld_acquire_gpu(const unsigned* a) {
  unsigned v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(a) : "memory");
  return v;
}
__device__ __forceinline__ void st_release_gpu(unsigned* a, unsigned v) {
  asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(a), "r"(v) : "memory");
}

template <int MODE, int KIND>
__device__ __forceinline__ void consume(const GramParams& P, const Cons& cs) {
  constexpr int R = kind_R(KIND), C = kind_C(KIND);
  constexpr int RR = R > 0 ? R : 1, CC = C > 0 ? C : 1;
  const int ld = P.ld, lane = cs.lane;
  double acc[RR][CC][2];
#pragma unroll
  for (int r = 0; r < RR; ++r)
#pragma unroll
    for (int c = 0; c < CC; ++c) { acc[r][c][0] = 0.0; acc[r][c][1] = 0.0; }
  const int aoff = (lane & 3) * ld + 8 * cs.job.bi0 + (lane >> 2) - cs.a0;
  const int boff = (lane & 3) * ld + 8 * cs.job.bj0 + (lane >> 2) - cs.b0;
  // does this job's column range hold the augmented y column (copy it into the panel)?
  const int ycol = P.p - cs.b0;
  const bool ycopy = (MODE != MODE_WEIGHTED) && C > 0 && P.p >= 8 * cs.job.bj0 && P.p < 8 * (cs.job.bj0 + C);
  // ... and the ones column (1 for the segment's rows, 0 for the zero-filled rows past its end).
  // With the ones column the y column can also sit in the job's ROW range only (block rows ending
  // at p, columns in the next block, where the ones column opened a block): then y goes into the A
  // panel (for a shared panel, the same location any B-side writer fills with the same value)
  const bool onecopy = (MODE == MODE_PLAIN || MODE == MODE_FOLD) && C > 0 && P.ones && P.p + 1 >= 8 * cs.job.bj0 &&
                       P.p + 1 < 8 * (cs.job.bj0 + C);
  const bool ycopyA = (MODE == MODE_PLAIN || MODE == MODE_FOLD) && R > 0 && P.ones && !ycopy &&
                      P.p >= 8 * cs.job.bi0 && P.p < 8 * (cs.job.bi0 + R);
  const bool anycopy = ycopy || ycopyA || onecopy;   // warp-uniform: one branch per stage
  // the staged value for the augmented column: y (PLAIN), y of fold kprime (FOLD), z (WZ: ys holds (w, z) pairs)
  const int yidx = lane * P.ystride + (MODE == MODE_FOLD ? cs.kprime : MODE == MODE_WZ ? 1 : 0);
  int st = 0;
  uint32_t ph = 0;
  for (int s = 0; s < cs.nst; ++s) {
    mbar_wait(&cs.full[st], ph);
    if (MODE == MODE_WEIGHTED) mbar_wait(&cs.ready[st], ph);  // w_i and z_i of the stage's rows
    double* pa = cs.smem + (size_t)st * P.stage_doubles;
    double* pb = cs.two ? pa + (size_t)BK * ld : pa;
    double* ys = pa + P.ys_off;
    double* ws = ys + BK * P.ystride;
    if (MODE != MODE_WEIGHTED && anycopy) {
      if (ycopy) pb[lane * ld + ycol] = ys[yidx];
      if (ycopyA) pa[lane * ld + P.p - cs.a0] = ys[yidx];
      if (onecopy) pb[lane * ld + ycol + 1] = cs.r0 + (int64_t)s * BK + lane < cs.r1 ? 1.0 : 0.0;
      __syncwarp();
    }
    if (KIND != J_NONE) {
      const double* pak = pa + aoff;
      const double* pbk = pb + boff;
#pragma unroll
      for (int ks = 0; ks < BK / 4; ++ks) {
        double a[RR], b[CC];
#pragma unroll
        for (int r = 0; r < R; ++r) a[r] = pak[8 * r];
#pragma unroll
        for (int c = 0; c < C; ++c) b[c] = pbk[8 * c];
        if (MODE == MODE_WEIGHTED || MODE == MODE_WZ) {  // w_k scales row k (lane & 3) of one operand:
          // the A fragments, or the B fragments when the job has fewer block columns than rows
          // (both hold row k = lane & 3 of the stage; fewer DMULs on the DMMA warps)
          const double wk = MODE == MODE_WZ ? ys[2 * (ks * 4 + (lane & 3))] : ws[ks * 4 + (lane & 3)];
          if (C < R) {
#pragma unroll
            for (int c = 0; c < C; ++c) b[c] *= wk;
          } else {
#pragma unroll
            for (int r = 0; r < R; ++r) a[r] *= wk;
          }
        }
#pragma unroll
        for (int r = 0; r < R; ++r)
#pragma unroll
          for (int c = 0; c < C; ++c)
            if (kind_active(KIND, r, c)) dmma_8x8x4(acc[r][c][0], acc[r][c][1], a[r], b[c]);
        pak += 4 * ld;
        pbk += 4 * ld;
      }
    }
    if (MODE != MODE_WEIGHTED && anycopy) fence_proxy_async_smem();  // generic smem writes precede the next TMA refill
    __syncwarp();
    if (cs.lane == 0) mbar_arrive(&cs.empty[st]);
    if (++st == P.ST) { st = 0; ph ^= 1u; }
  }
  // epilogue, ordered plans: add this segment's blocks into the (fold, tile type)'s running sums
  // after the previous segment's CTA of the same tile type has added its own (a ticket per
  // (fold, tile type), released once every job warp of the CTA is done), so every entry is
  // ((seg 0 + seg 1) + seg 2) + ... in segment order: deterministic, the same order as the
  // partial-buffer reduction, without the partial buffer (L2 read-modify-writes, never HBM)
  if (KIND != J_NONE && P.ordered) {
    // ORD_W interleaved chains (segment s joins chain s % ORD_W as its (s / ORD_W)-th link): the
    // CTAs of one tile type that run in the same wave are never neighbours in a chain
    const int chain = cs.seg % ORD_W, link = cs.seg / ORD_W;
    unsigned* tk = P.ticket + (size_t)chain * P.U + cs.u;   // ordered plans have one fold
    if (lane == 0)
      while (ld_acquire_gpu(tk) != (unsigned)link) __nanosleep(32);
    __syncwarp();
    double* out = P.accum + (size_t)chain * P.nblk * 64;
#pragma unroll
    for (int r = 0; r < R; ++r)
#pragma unroll
      for (int c = 0; c < C; ++c)
        if (kind_active(KIND, r, c)) {
          const int idx = P.blk_of[(cs.job.bi0 + r) * P.nb + cs.job.bj0 + c];
          double2* o = reinterpret_cast<double2*>(out + (size_t)idx * 64 + (lane >> 2) * 8 + 2 * (lane & 3));
          double2 v = make_double2(acc[r][c][0], acc[r][c][1]);
          if (link > 0) {   // L2 only: the previous link was added by another SM
            const double2 prev = __ldcg(o);
            v.x = prev.x + v.x;
            v.y = prev.y + v.y;
          }
          __stcg(o, v);
        }
    __threadfence();
    __syncwarp();
    if (lane == 0 && atomicAdd(cs.done_s, 1u) == (unsigned)cs.njob - 1u) st_release_gpu(tk, (unsigned)link + 1u);
    return;
  }
  // epilogue: this (fold, segment)'s partial blocks
  if (KIND != J_NONE) {
    double* out = P.partial + ((size_t)(cs.fold * P.nseg + cs.seg) * P.nblk) * 64;
#pragma unroll
    for (int r = 0; r < R; ++r)
#pragma unroll
      for (int c = 0; c < C; ++c)
        if (kind_active(KIND, r, c)) {
          const int idx = P.blk_of[(cs.job.bi0 + r) * P.nb + cs.job.bj0 + c];
          *reinterpret_cast<double2*>(out + (size_t)idx * 64 + (lane >> 2) * 8 + 2 * (lane & 3)) =
              make_double2(acc[r][c][0], acc[r][c][1]);
        }
  }
}

// WEIGHTED row warps (R#25): per row of the stage, eta = x_i^T beta,
// mu = sigma(eta) clamped to [eps, 1-eps], w = mu(1-mu), z = eta + (y - mu)/w; w goes to ws[k]
// and z into the augmented column of the smem tile, so the MMA warps form sum w [x|z][x|z]^T.
// Running one stage ahead of the MMA warps (ready[] ring) keeps the DMMA pipe busy.
__device__ __forceinline__ void weighted_rows(const GramParams& P, const Cons& cs, int rw) {
  const int ld = P.ld, lane = cs.lane;
  constexpr int LPR = 32 * NRW / BK;                       // lanes per row
  const int k = rw * (BK / NRW) + lane / LPR, sub = lane % LPR;
  double sw = 0.0, sll = 0.0;
  int st = 0;
  uint32_t ph = 0;
  for (int s = 0; s < cs.nst; ++s) {
    mbar_wait(&cs.full[st], ph);
    double* pa = cs.smem + (size_t)st * P.stage_doubles;
    double* ys = pa + P.ys_off;
    double* ws = ys + BK * P.ystride;
    const double* xr = pa + k * ld;
    // eta = x_i^T beta: lane `sub` takes the column pairs 2 sub + 2 LPR t (16-byte loads; the
    // row pitch and beta_s are even and zero beyond p), four pairs in flight per step
    double e0 = 0.0, e1 = 0.0, e2 = 0.0, e3 = 0.0;
    const double2* x2 = reinterpret_cast<const double2*>(xr);
    const double2* b2 = reinterpret_cast<const double2*>(cs.beta_s);
    const int np2 = (P.p + 1) >> 1;  // column pairs covering p (beta_s[p] == 0)
    int t = sub;
    for (; t + 3 * LPR < np2; t += 4 * LPR) {
      const double2 xa = x2[t], xb = x2[t + LPR], xc = x2[t + 2 * LPR], xd = x2[t + 3 * LPR];
      const double2 ba = b2[t], bb = b2[t + LPR], bc = b2[t + 2 * LPR], bd = b2[t + 3 * LPR];
      e0 = fma(xa.x, ba.x, fma(xa.y, ba.y, e0));
      e1 = fma(xb.x, bb.x, fma(xb.y, bb.y, e1));
      e2 = fma(xc.x, bc.x, fma(xc.y, bc.y, e2));
      e3 = fma(xd.x, bd.x, fma(xd.y, bd.y, e3));
    }
    for (; t < np2; t += LPR) {
      const double2 xa = x2[t], ba = b2[t];
      e0 = fma(xa.x, ba.x, fma(xa.y, ba.y, e0));
    }
    double e = (e0 + e1) + (e2 + e3);
#pragma unroll
    for (int o = 1; o < LPR; o <<= 1) e += __shfl_xor_sync(0xffffffffu, e, o);
    const int64_t row = cs.r0 + (int64_t)s * BK + k;
    const bool valid = row < cs.r1;
    const double yk = ys[k];
    double w = 0.0, z = 0.0, ex = 0.0;
    if (valid) {
      ex = exp(-e);
      double mu = 1.0 / (1.0 + ex);
      mu = fmin(fmax(mu, P.eps), 1.0 - P.eps);
      w = mu * (1.0 - mu);
      z = e + (yk - mu) / w;
    }
    if (sub == 0) {
      ws[k] = w;
      pa[k * ld + P.p] = z;
    }
    fence_proxy_async_smem();  // these generic writes precede the stage's next TMA refill
    __syncwarp();
    if (lane == 0) {
      mbar_arrive(&cs.ready[st]);
      mbar_arrive(&cs.empty[st]);
    }
    // off the critical path (the MMA warps already have the stage): sum w and the
    // log-likelihood, once per segment (CTA type 0 writes them), only when the caller asked:
    // the row warps' scalar fp64 work shares the sub-partitions with the DMMA warps (measured:
    // 0.5 ms of an 8.7 ms cfg5 pass). log(1 + e^eta) = eta + log1p(e^-eta) reuses ex; when ex
    // overflows (eta < -709) the term is e^eta = 0 to double precision.
    if (P.want_scal && cs.u == 0 && valid && sub == 0) {
      sw += w;
      sll += yk * e - (isinf(ex) ? 0.0 : e + log1p(ex));
    }
    if (++st == P.ST) { st = 0; ph ^= 1u; }
  }
  // fixed-order reductions: lanes 0, LPR, 2 LPR, .. hold their rows' sums; then warps in order
#pragma unroll
  for (int o = LPR; o < 32; o <<= 1) {
    sw += __shfl_xor_sync(0xffffffffu, sw, o);
    sll += __shfl_xor_sync(0xffffffffu, sll, o);
  }
  if (lane == 0) { cs.scal_s[2 * rw] = sw; cs.scal_s[2 * rw + 1] = sll; }
  named_bar_sync(1, NRW * 32);
  if (rw == 0 && lane == 0 && cs.u == 0) {
    double a = 0.0, b = 0.0;
    for (int w = 0; w < NRW; ++w) { a += cs.scal_s[2 * w]; b += cs.scal_s[2 * w + 1]; }
    P.partial_scal[cs.seg * 2 + 0] = a;
    P.partial_scal[cs.seg * 2 + 1] = b;
  }
}

// WZ pre-pass (two-panel weighted plans, R#25): one HBM-bound pass over [X | y] that
// forms, per row, eta = x_i^T beta, mu = sigma(eta) clamped to [eps, 1-eps], w = mu(1-mu),
// z = eta + (y - mu)/w -> wz[i] = (w_i, z_i) (the same formulas, in the same order, as
// weighted_rows); with want_scal, per-CTA (sum w, log-likelihood) partials in warp order.
// Warps own blocks of 32 rows of a contiguous per-CTA range; lanes take 16-byte column pairs
// (four in flight); beta lives in shared memory (zero past p).
constexpr int RW_THREADS = 256;
__global__ void __launch_bounds__(RW_THREADS) row_weights_kernel(const double* __restrict__ X, const double* __restrict__ y,
                                                                 const double* __restrict__ beta, int64_t n, int p,
                                                                 int64_t ldx, double eps, int64_t rows_per_cta,
                                                                 int want_scal, double2* __restrict__ wz,
                                                                 double* __restrict__ pscal) {
  extern __shared__ __align__(16) double bsm[];
  __shared__ double red[RW_THREADS / 32][2];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, nw = RW_THREADS / 32;
  const int np2 = (p + 1) >> 1;
  for (int j = threadIdx.x; j < 2 * np2; j += RW_THREADS) bsm[j] = j < p ? beta[j] : 0.0;
  __syncthreads();
  const double2* b2 = reinterpret_cast<const double2*>(bsm);
  const int64_t r0 = (int64_t)blockIdx.x * rows_per_cta, r1 = min(n, r0 + rows_per_cta);
  double sw = 0.0, sll = 0.0;
  // a warp takes 32 rows per step: their dot products one by one (lanes over column pairs, four
  // pairs in flight, butterfly sum), lane k keeping eta of row k; then the per-row scalar work
  // (exp, clamp, two divisions) runs once per lane instead of once per row on a whole warp
  for (int64_t i0 = r0 + 32 * warp; i0 < r1; i0 += 32 * nw) {
    double eta = 0.0;
    const int nrow = r1 - i0 < 32 ? (int)(r1 - i0) : 32;
    for (int k = 0; k < nrow; ++k) {
      const double2* x2 = reinterpret_cast<const double2*>(X + (i0 + k) * ldx);
      double a0 = 0.0, a1 = 0.0, a2 = 0.0, a3 = 0.0;
      int t = lane;
      for (; t + 96 < np2; t += 128) {
        double2 xa = __ldg(x2 + t), xb = __ldg(x2 + t + 32), xc = __ldg(x2 + t + 64), xd = __ldg(x2 + t + 96);
        const double2 ba = b2[t], bb = b2[t + 32], bc = b2[t + 64], bd = b2[t + 96];
        a0 = fma(xa.x, ba.x, fma(xa.y, ba.y, a0));
        a1 = fma(xb.x, bb.x, fma(xb.y, bb.y, a1));
        a2 = fma(xc.x, bc.x, fma(xc.y, bc.y, a2));
        if (2 * (t + 96) + 1 >= p) xd.y = 0.0;  // the last pair may hold the pad element of an odd p
        a3 = fma(xd.x, bd.x, fma(xd.y, bd.y, a3));
      }
      for (; t < np2; t += 32) {
        double2 xa = __ldg(x2 + t);
        if (2 * t + 1 >= p) xa.y = 0.0;  // the pad element of an odd p (never trusted)
        a0 = fma(xa.x, b2[t].x, fma(xa.y, b2[t].y, a0));
      }
      double v = (a0 + a1) + (a2 + a3);
#pragma unroll
      for (int o = 16; o >= 1; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
      if (lane == k) eta = v;
    }
    if (lane < nrow) {
      const int64_t i = i0 + lane;
      const double ee = eta, yk = __ldg(y + i);
      const double ex = exp(-ee);
      double mu = 1.0 / (1.0 + ex);
      mu = fmin(fmax(mu, eps), 1.0 - eps);
      const double w = mu * (1.0 - mu);
      wz[i] = make_double2(w, ee + (yk - mu) / w);
      if (want_scal) {
        sw += w;
        sll += yk * ee - (isinf(ex) ? 0.0 : ee + log1p(ex));
      }
    }
  }
  if (!want_scal) return;
#pragma unroll
  for (int o = 16; o >= 1; o >>= 1) {   // butterfly over the lanes, fixed order
    sw += __shfl_xor_sync(0xffffffffu, sw, o);
    sll += __shfl_xor_sync(0xffffffffu, sll, o);
  }
  if (lane == 0) { red[warp][0] = sw; red[warp][1] = sll; }
  __syncthreads();
  if (threadIdx.x < 2) {
    double a = 0.0;
    for (int w = 0; w < nw; ++w) a += red[w][threadIdx.x];  // warp order
    pscal[2 * blockIdx.x + threadIdx.x] = a;
  }
}

template <int MODE, bool TWO>
__global__ void __launch_bounds__(gram_threads(MODE, TWO), 1)
gram_kernel(const __grid_constant__ CUtensorMap tmX, const __grid_constant__ CUtensorMap tmY, const GramParams P) {
  extern __shared__ __align__(128) double smem[];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  // work items (CTA type u, segment, fold): the U_off costlier types first (longest-processing-
  // time order keeps the last wave short), each group ordered segment-major so CTAs running
  // together stream the same rows (L2 reuse across tile types)
  const int nf = MODE == MODE_FOLD ? P.K : 1;
  const int off_items = P.U_off * P.nseg * nf;
  int u, rest;
  if ((int)blockIdx.x < off_items) {
    u = blockIdx.x % P.U_off;
    rest = blockIdx.x / P.U_off;
  } else {
    const int b2 = blockIdx.x - off_items, ud = P.U - P.U_off;
    u = P.U_off + b2 % ud;
    rest = b2 / ud;
  }
  __shared__ double scal_s[2 * NRW];
  __shared__ __align__(8) uint64_t ready_s[MAXST];
  __shared__ unsigned done_s;
  Cons cs;
  cs.done_s = &done_s;
  cs.scal_s = scal_s;
  cs.u = u;
  cs.seg = rest % P.nseg;
  cs.fold = rest / P.nseg;  // 0 unless MODE_FOLD
  cs.smem = smem;
  double* beta_s = smem + (size_t)P.ST * P.stage_doubles;  // WEIGHTED: ld doubles
  cs.full = reinterpret_cast<uint64_t*>(beta_s + (MODE == MODE_WEIGHTED ? P.ld : 0));
  cs.empty = cs.full + MAXST;
  cs.ready = ready_s;
  cs.beta_s = beta_s;
  cs.r0 = (int64_t)cs.seg * P.seg_rows;
  cs.r1 = min(P.nrows, cs.r0 + P.seg_rows);
  cs.nst = cs.r1 > cs.r0 ? (int)((cs.r1 - cs.r0 + BK - 1) / BK) : 0;
  cs.kprime = (MODE == MODE_FOLD) ? ((cs.fold - P.off_mod) % P.K + P.K) % P.K : 0;
  const CtaDesc* cd = P.ctas + u;
  cs.a0 = cd->a0;
  cs.b0 = cd->b0;
  cs.two = TWO && !cd->same;
  const int njob = cd->njob;
  cs.njob = njob;
  const int nconsumers = njob + (MODE == MODE_WEIGHTED ? NRW : 0);  // arrivals per stage release
  const int full_count = P.ytma ? 1 : 32;

  if (threadIdx.x == 0) {
    done_s = 0u;
    for (int s = 0; s < P.ST; ++s) {
      mbar_init(&cs.full[s], full_count);
      mbar_init(&cs.empty[s], nconsumers);
      if (MODE == MODE_WEIGHTED) mbar_init(&cs.ready[s], NRW);
    }
    fence_mbar_init();
    tma_prefetch(&tmX);
    if (P.ytma) tma_prefetch(&tmY);
  }
  if (MODE == MODE_WEIGHTED)
    for (int j = threadIdx.x; j < P.ld; j += blockDim.x) beta_s[j] = j < P.p ? P.beta[j] : 0.0;
  __syncthreads();

  cs.warp = warp;
  cs.lane = lane;
  constexpr int NWC = nwc_of(TWO);
  if (MODE == MODE_WEIGHTED && warp >= NWC && warp < NWC + NRW) {
    weighted_rows(P, cs, warp - NWC);
    return;
  }
  if (warp == gram_threads(MODE, TWO) / 32 - 1) {
    // ------------------------------------------------------------ producer warp
    if (!P.ytma || lane == 0) {
      int st = 0;
      uint32_t ph = 0;
      const uint32_t bytes = (cs.two ? 2u : 1u) * P.xbox_bytes + P.ybox_bytes;
      for (int s = 0; s < cs.nst; ++s) {
        mbar_wait(&cs.empty[st], ph ^ 1u);
        double* pa = smem + (size_t)st * P.stage_doubles;
        double* pb = pa + (size_t)BK * P.ld;
        double* ys = pa + P.ys_off;
        const int rr = (int)(cs.r0 + (int64_t)s * BK);
        if (lane == 0) {
          asm volatile("mbarrier.expect_tx.relaxed.cta.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(&cs.full[st])),
                       "r"(bytes)
                       : "memory");
          if (MODE == MODE_FOLD) {
            tma_load_3d(pa, &tmX, &cs.full[st], cs.a0, cs.kprime, rr);
            if (cs.two) tma_load_3d(pb, &tmX, &cs.full[st], cs.b0, cs.kprime, rr);
            if (P.ytma) tma_load_2d(ys, &tmY, &cs.full[st], 0, rr);
          } else {
            tma_load_2d(pa, &tmX, &cs.full[st], cs.a0, rr);
            if (cs.two) tma_load_2d(pb, &tmX, &cs.full[st], cs.b0, rr);
            if (MODE == MODE_WZ) tma_load_2d(ys, &tmY, &cs.full[st], 0, rr);   // (w, z) of the stage's rows
            else if (P.ytma) tma_load_1d(ys, &tmY, &cs.full[st], rr);
          }
        }
        if (!P.ytma) {  // odd-K folds: strided y through the producer's lanes
          const int64_t row = (int64_t)rr + lane;
          double yv = 0.0;
          if (row < cs.r1) yv = P.y[row * P.K + cs.kprime];
          ys[lane * P.ystride + cs.kprime] = yv;
        }
        mbar_arrive(&cs.full[st]);
        if (++st == P.ST) { st = 0; ph ^= 1u; }
      }
    }
    return;
  }
  // -------------------------------------------------------------- consumer warps
  cs.job = cd->job[warp];
  if (cs.job.kind == J_NONE) return;
  constexpr bool BIGJ = TWO;  // 4x8 jobs only in two-panel plans (registers)
  switch (cs.job.kind) {
    case J_F44: consume<MODE, J_F44>(P, cs); break;
    case J_T4: consume<MODE, J_T4>(P, cs); break;
    case J_F41: consume<MODE, J_F41>(P, cs); break;
    case J_F42: consume<MODE, J_F42>(P, cs); break;
    case J_F43: consume<MODE, J_F43>(P, cs); break;
    case J_T1: consume<MODE, J_T1>(P, cs); break;
    case J_T2: consume<MODE, J_T2>(P, cs); break;
    case J_T3: consume<MODE, J_T3>(P, cs); break;
    case J_F48: if (BIGJ) consume<MODE, J_F48>(P, cs); break;
    case J_T4F4: if (BIGJ) consume<MODE, J_T4F4>(P, cs); break;
    case J_F45: if (BIGJ) consume<MODE, J_F45>(P, cs); break;
    case J_F46: if (BIGJ) consume<MODE, J_F46>(P, cs); break;
    case J_F47: if (BIGJ) consume<MODE, J_F47>(P, cs); break;
    case J_T4F1: if (BIGJ) consume<MODE, J_T4F1>(P, cs); break;
    case J_T4F2: if (BIGJ) consume<MODE, J_T4F2>(P, cs); break;
    case J_T4F3: if (BIGJ) consume<MODE, J_T4F3>(P, cs); break;
    default: consume<MODE, J_NONE>(P, cs); break;
  }
}

// Sum the segment partials in a fixed order and scatter into the packed upper triangle of
// the augmented (p+1)x(p+1) matrix: packed[j*(p+1) - j(j-1)/2 + (l-j)], j <= l <= p.
__global__ void gram_reduce_kernel(const double* __restrict__ partial, int nfold, int nseg, int nblk,
                                   const int2* __restrict__ blk_coord, int p, const double* __restrict__ tail,
                                   double* __restrict__ packed, int64_t psize, const double* __restrict__ pscal,
                                   int nscal, int with_scal, int accumulate, double* __restrict__ sums) {
  const int64_t total = (int64_t)nfold * nblk * 64;
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < total; t += (int64_t)gridDim.x * blockDim.x) {
    const int e = (int)(t & 63);
    const int64_t fb = t >> 6;
    const int idx = (int)(fb % nblk);
    const int f = (int)(fb / nblk);
    const int2 bc = blk_coord[idx];
    const int j = 8 * bc.x + (e >> 3), l = 8 * bc.y + (e & 7);
    if (j > l || l > p + (sums ? 1 : 0)) continue;
    double s = 0.0;
    const double* src = partial + ((size_t)f * nseg * nblk + idx) * 64 + e;
    for (int g = 0; g < nseg; ++g) s += src[(size_t)g * nblk * 64];
    if (tail) s += tail[((size_t)f * nblk + idx) * 64 + e];
    if (l == p + 1) {   // the ones column: X^T 1, 1^T y, the row count
      sums[(size_t)f * (p + 2) + j] = s;
      continue;
    }
    double* dst = packed + (size_t)f * psize + (int64_t)j * (p + 1) - (int64_t)j * (j - 1) / 2 + (l - j);
    *dst = accumulate ? *dst + s : s;   // streamed row blocks add in block order (f4)
  }
  if (with_scal && blockIdx.x == 0 && threadIdx.x < 2) {
    double s = 0.0;
    for (int g = 0; g < nscal; ++g) s += pscal[g * 2 + threadIdx.x];
    packed[psize + threadIdx.x] = accumulate ? packed[psize + threadIdx.x] + s : s;
  }
}

// First level of the split-n reduction when there are many segments: chunk c of S sums the
// segments [c*per, (c+1)*per) in order; the output has the partial buffer's layout with nseg = S
// (so gram_reduce_kernel finishes it). Deterministic; spreads the segment loop over many threads.
__global__ void gram_chunk_kernel(const double* __restrict__ partial, int nfold, int nseg, int nblk, int S, int per,
                                  double* __restrict__ out, const double* __restrict__ pscal, double* __restrict__ oscal) {
  const int64_t total = (int64_t)nfold * S * nblk * 64;
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < total; t += (int64_t)gridDim.x * blockDim.x) {
    const int e = (int)(t & 63);
    const int64_t r = t >> 6;
    const int idx = (int)(r % nblk);
    const int64_t fc = r / nblk;
    const int c = (int)(fc % S), f = (int)(fc / S);
    const int g0 = c * per, g1 = min(nseg, g0 + per);
    double s = 0.0;
    for (int g = g0; g < g1; ++g) s += partial[(((size_t)f * nseg + g) * nblk + idx) * 64 + e];
    out[(((size_t)f * S + c) * nblk + idx) * 64 + e] = s;
  }
  if (pscal && blockIdx.x == 0)
    for (int i = threadIdx.x; i < 2 * S; i += blockDim.x) {
      const int c = i / 2, k = i % 2;
      double s = 0.0;
      for (int g = c * per; g < min(nseg, (c + 1) * per); ++g) s += pscal[g * 2 + k];
      oscal[i] = s;
    }
}

// FOLD tail: rows i in [nq*K, n_local) (fewer than K, so at most one per fold) as outer products.
__global__ void gram_fold_tail_kernel(const double* __restrict__ X, const double* __restrict__ y, int64_t ldx,
                                      int64_t n_local, int64_t nq, int K, int off_mod, int p, int nblk,
                                      const int2* __restrict__ blk_coord, double* __restrict__ tail, int ones) {
  const int64_t total = (int64_t)K * nblk * 64;
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < total; t += (int64_t)gridDim.x * blockDim.x) {
    const int e = (int)(t & 63);
    const int64_t fb = t >> 6;
    const int idx = (int)(fb % nblk);
    const int f = (int)(fb / nblk);
    const int kp = ((f - off_mod) % K + K) % K;
    const int64_t i = nq * K + kp;
    double v = 0.0;
    if (i < n_local) {
      const int2 bc = blk_coord[idx];
      const int j = 8 * bc.x + (e >> 3), l = 8 * bc.y + (e & 7);
      if (j <= p + ones && l <= p + ones) {   // z = [x_i | y_i | 1]
        const double zj = j < p ? X[i * ldx + j] : j == p ? y[i] : 1.0;
        const double zl = l < p ? X[i * ldx + l] : l == p ? y[i] : 1.0;
        v = zj * zl;
      }
    }
    tail[t] = v;
  }
}

__global__ void gram_unpack_kernel(const double* __restrict__ packed, int nfold, int p, double* __restrict__ G,
                                   double* __restrict__ xty, double* __restrict__ yty) {
  const int64_t psize = (int64_t)(p + 1) * (p + 2) / 2;
  const int64_t per = (int64_t)p * p + p + 1;
  const int64_t total = (int64_t)nfold * per;
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < total; t += (int64_t)gridDim.x * blockDim.x) {
    const int f = (int)(t / per);
    const int64_t q = t % per;
    const double* pk = packed + (size_t)f * psize;
    if (q < (int64_t)p * p) {
      int j = (int)(q / p), l = (int)(q % p);
      if (j > l) { int tmp = j; j = l; l = tmp; }
      G[(size_t)f * p * p + q] = pk[(int64_t)j * (p + 1) - (int64_t)j * (j - 1) / 2 + (l - j)];
    } else if (q < (int64_t)p * p + p) {
      const int j = (int)(q - (int64_t)p * p);
      xty[(size_t)f * p + j] = pk[(int64_t)j * (p + 1) - (int64_t)j * (j - 1) / 2 + (p - j)];
    } else if (yty) {
      yty[f] = pk[psize - 1];
    }
  }
}

// ------------------------------------------------------------------ host side: plans
struct GramPlan {
  int mode = 0, p = 0, nb = 0, ld = 0, two_panel = 0, U = 0, U_off = 0, nseg = 0, ST = 0, nblk = 0, ordered = 0;
  int64_t seg_rows = 0;
  size_t smem = 0;
  int stage_doubles = 0, ys_off = 0, ystride = 1, ytma = 1;
  uint32_t ybox_bytes = 0;
  std::vector<CtaDesc> ctas;
  CtaDesc* d_ctas = nullptr;
  int32_t* d_blk_of = nullptr;
  int2* d_blk_coord = nullptr;
  ~GramPlan() {
    if (d_ctas) cudaFree(d_ctas);
    if (d_blk_of) cudaFree(d_blk_of);
    if (d_blk_coord) cudaFree(d_blk_coord);
  }
};

// Spread jobs over CTA types (longest-processing-time first), then order each CTA's jobs so
// the 4 SM sub-partitions (warp w -> SMSP w % 4) carry similar DMMA counts.
// rw_bias: DMMA-block equivalents of row-warp work on SMSPs 0 and 1 (the weighted pass's two row
// warps are warps 16 and 17 of the CTA), so the packer gives those sub-partitions less DMMA work
static void pack_jobs(std::vector<Job>& jobs, int a0, int b0, int same, std::vector<CtaDesc>& out, int NWC,
                      int rw_bias = 0) {
  std::sort(jobs.begin(), jobs.end(),
            [](const Job& x, const Job& y) { return kind_cost(x.kind) > kind_cost(y.kind); });
  const int U = std::max<int>(1, ((int)jobs.size() + NWC - 1) / NWC);
  std::vector<std::vector<Job>> bins(U);
  std::vector<int> load(U, 0);
  for (auto& j : jobs) {
    int best = -1;
    for (int b = 0; b < U; ++b)
      if ((int)bins[b].size() < NWC && (best < 0 || load[b] < load[best])) best = b;
    bins[best].push_back(j);
    load[best] += kind_cost(j.kind);
  }
  for (auto& bin : bins) {
    CtaDesc cd;
    std::memset(&cd, 0, sizeof(cd));
    cd.a0 = a0; cd.b0 = b0; cd.same = same;
    std::vector<std::vector<Job>> sub(4);
    std::vector<int> sl{rw_bias, rw_bias, 0, 0};
    for (auto& j : bin) {  // already sorted by cost
      int best = -1;
      for (int q = 0; q < 4; ++q)
        if ((int)sub[q].size() * 4 + q < NWC && (best < 0 || sl[q] < sl[best])) best = q;
      sub[best].push_back(j);
      sl[best] += kind_cost(j.kind);
    }
    // warp w runs slot w (SMSP w % 4); idle slots hold J_NONE and exit early
    for (int w = 0; w < NWC_MAX; ++w) cd.job[w] = Job{0, 0, J_NONE, 0};
    int nj = 0;
    for (int q = 0; q < 4; ++q)
      for (size_t k = 0; k < sub[q].size(); ++k) { cd.job[q + 4 * k] = sub[q][k]; ++nj; }
    cd.njob = nj;  // busy warps = arrivals per stage release
    out.push_back(cd);
  }
}

static oem_status build_plan(oem_ctx* ctx, int mode, int p, int64_t nrows, int K, int ones, GramPlan& pl) {
  pl.mode = mode;
  pl.p = p;
  const int Pa = p + 1 + ones;   // augmented columns: [X | y] or [X | y | 1]
  const int nb_exact = (Pa + 7) / 8;
  const bool single = (8 * nb_exact + 4) <= 256;
  if ((mode == MODE_WEIGHTED && !single) || (mode == MODE_WZ && single))
    OEM_FAIL(OEM_ERR_UNSUPPORTED, "gram: weighted plan kind does not match p (internal)");
  pl.two_panel = single ? 0 : 1;
  // two-panel plans pad the block count to whole 128-column panels (zero columns, TMA fill)
  pl.nb = single ? nb_exact : (nb_exact + 15) / 16 * 16;
  pl.nblk = pl.nb * (pl.nb + 1) / 2;
  std::vector<int32_t> blk_of((size_t)pl.nb * pl.nb, -1);
  std::vector<int2> coord(pl.nblk);
  {
    int idx = 0;
    for (int bi = 0; bi < pl.nb; ++bi)
      for (int bj = bi; bj < pl.nb; ++bj) { blk_of[(size_t)bi * pl.nb + bj] = idx; coord[idx] = make_int2(bi, bj); ++idx; }
  }
  if (single) {
    pl.ld = 8 * pl.nb + 4;  // = 4 or 12 (mod 16): conflict-free fragment loads
    // One CTA per SM with 16 MMA warps (4 per SM sub-partition). Jobs are 4x4-block tiles of
    // the upper triangle, optionally with every full 4x4 tile split into two 4x2 ones; the tiling
    // whose packing gives the smaller (CTA types x busiest sub-partition) is kept: every CTA type
    // streams all rows, and a CTA's stage time is that of its busiest sub-partition.
    auto tile = [&](bool split) {
      std::vector<Job> jobs;
      for (int bi0 = 0; bi0 < pl.nb; bi0 += 4)
        for (int bj0 = bi0; bj0 < pl.nb; bj0 += 4) {
          const int Rr = std::min(4, pl.nb - bi0), Cc = std::min(4, pl.nb - bj0);
          if (bi0 == bj0) { jobs.push_back(Job{bi0, bj0, Rr == 4 ? J_T4 : Rr == 3 ? J_T3 : Rr == 2 ? J_T2 : J_T1, 0}); continue; }
          if (split && Cc == 4) {
            jobs.push_back(Job{bi0, bj0, J_F42, 0});
            jobs.push_back(Job{bi0, bj0 + 2, J_F42, 0});
          } else {
            jobs.push_back(Job{bi0, bj0, Cc == 4 ? J_F44 : Cc == 3 ? J_F43 : Cc == 2 ? J_F42 : J_F41, 0});
          }
        }
      return jobs;
    };
    auto score = [&](const std::vector<CtaDesc>& ctas) {
      int worst = 0;
      for (const auto& cd : ctas)
        for (int q = 0; q < 4; ++q) {
          int l = 0;
          for (int w = q; w < NWC_MAX; w += 4) l += kind_cost(cd.job[w].kind);
          worst = std::max(worst, l);
        }
      return (int64_t)ctas.size() * worst;
    };
    std::vector<CtaDesc> c0, c1;
    auto j0 = tile(false), j1 = tile(true);
    // the weighted pass's row warps (eta: p FMAs per row, exp, divisions) share sub-partitions 0
    // and 1 with DMMA warps; counting them as ~0.07 p blocks of DMMA work when packing measured
    // best (tools/rw_bias_sweep.sh, n = 5e6: p = 64 1.40 -> 1.37 ms, 100 2.52 -> 2.22, 150
    // 4.42 -> 4.19, 200 8.21 -> 7.76, 247 18.4 -> 13.9; OEM_GRAM_RW_BIAS overrides)
    const char* rwb = std::getenv("OEM_GRAM_RW_BIAS");
    const int rw_bias = rwb ? std::atoi(rwb) : mode == MODE_WEIGHTED ? (int)std::lround(0.07 * p) : 0;
    pack_jobs(j0, 0, 0, 1, c0, nwc_of(false), rw_bias);
    pack_jobs(j1, 0, 0, 1, c1, nwc_of(false), rw_bias);
    pl.ctas = score(c1) < score(c0) ? c1 : c0;
  } else {
    pl.ld = 132;  // 128-column panel + 4 (mod 16 = 4)
    const int np = pl.nb / 16;
    // off-diagonal tiles (I < J, 256 blocks) first, then the diagonal ones (136 blocks)
    std::vector<std::pair<int, int>> tiles;
    for (int I = 0; I < np; ++I)
      for (int J = I + 1; J < np; ++J) tiles.push_back({I, J});
    pl.U_off = (int)tiles.size();
    for (int I = 0; I < np; ++I) tiles.push_back({I, I});
    for (auto& tij : tiles) {
      const int I = tij.first, J = tij.second;
      {
        std::vector<Job> jobs;
        for (int r = 0; r < 4; ++r)
          for (int c = 0; c < 2; ++c) {
            const int bi0 = 16 * I + 4 * r, bj0 = 16 * J + 8 * c;
            if (I < J) { jobs.push_back(Job{bi0, bj0, J_F48, 0}); continue; }
            const int lr = 4 * r, lc = 8 * c;  // local block coordinates on a diagonal tile
            if (lc >= lr + 4) jobs.push_back(Job{bi0, bj0, J_F48, 0});
            else if (lc == lr) jobs.push_back(Job{bi0, bj0, J_T4F4, 0});
            else if (lc + 4 == lr) jobs.push_back(Job{bi0, bj0 + 4, J_T4, 0});
          }
        // trim blocks beyond the augmented matrix (last panel): block rows/cols >= nb_exact
        std::vector<Job> kept;
        for (auto& jb : jobs) {
          const int R0 = kind_R(jb.kind), C0 = kind_C(jb.kind);
          const int ru = std::min(R0, nb_exact - jb.bi0), cu = std::min(C0, nb_exact - jb.bj0);
          if (ru <= 0 || cu <= 0) continue;
          if (ru == R0 && cu == C0) { kept.push_back(jb); continue; }
          const int k = kind_of(ru, cu, kind_tri(jb.kind));
          kept.push_back(Job{jb.bi0, jb.bj0, k != J_NONE ? k : jb.kind, 0});
        }
        pack_jobs(kept, 128 * I, 128 * J, I == J, pl.ctas, nwc_of(true));
      }
    }
  }
  pl.U = (int)pl.ctas.size();
  // Two-panel fold / WZ plans dispatch the costlier off-diagonal tiles first (U_off), in up to 48
  // waves of long segments whose partial blocks a fixed-order kernel sums. DRAM traffic studies at
  // cfg4 (profiles/cfg4_l2_schedule_r02.md; the kernel is DMMA-bound with HBM at ~20% of its
  // peak, so re-reads cost no kernel time): that schedule reads X 4.6-4.9x from DRAM (372-389 GB)
  // at 288.3 ms; 384 waves of short segments, segment-major, every tile type of a segment
  // together (the plain two-panel default since round 2; OEM_GRAM_LPT=1 OEM_GRAM_WAVES=48 restores
  // the other) read 97.0-97.6 GB (1.21x) at the same kernel time but add 1.4 ms of reduction
  // (6.4 GB of partial blocks); the same schedule with the segments added in order into running
  // sums inside the kernel (OEM_GRAM_ORDERED=1: no partial blocks) reads 102.7 GB but runs
  // 294.9 ms.
  const char* ordv = std::getenv("OEM_GRAM_ORDERED");
  // (plain and WZ passes only: a fold pass splits every segment into K items whose same-tile
  // neighbours run in the same wave; cfg3 went 74.5 -> 124.5 ms ordered)
  pl.ordered = (pl.two_panel && mode != MODE_FOLD && ordv && ordv[0] == '1') ? 1 : 0;
  // plain two-panel passes default to the segment-major schedule of short segments (below): the
  // same kernel time with ~4x less DRAM traffic (cfg4: 388.6 -> 97.0 GB read, 1.21x the
  // algorithmic bytes; the whole call +1.4 ms = 0.5% for the larger split-n reduction). Fold
  // passes keep the costliest-first order: there the short segments cost kernel time (cfg3 384
  // waves: 44.3 GB = 1.10x but +1.2% kernel, +2.6% call; profiles/cfg4_l2_schedule_r02.md)
  const bool seg_major = pl.two_panel && mode == MODE_PLAIN && !pl.ordered;
  const char* lpt = std::getenv("OEM_GRAM_LPT");  // developer override (timing studies): 0 / 1
  const bool use_lpt = lpt ? lpt[0] == '1' : !pl.ordered && !seg_major;
  if (!pl.two_panel || pl.U_off == 0 || !use_lpt) pl.U_off = pl.U;
  // y staging: 1D TMA box (PLAIN/WEIGHTED); FOLD: 2D box [BK][Kpad] over y viewed as [nq][K]
  // (needs K*8 % 16 == 0, i.e. even K), else the producer's lanes load it
  if (mode == MODE_FOLD) {
    pl.ytma = (K % 2 == 0) && K <= 256;
    pl.ystride = pl.ytma ? K : K;  // smem row stride of ys in doubles
  } else if (mode == MODE_WZ) {   // (w, z) pairs: 2D box [BK][2]
    pl.ytma = 1;
    pl.ystride = 2;
  } else {
    pl.ytma = 1;
    pl.ystride = 1;
  }
  pl.ybox_bytes = pl.ytma ? (uint32_t)(BK * pl.ystride * 8) : 0;
  const int panels = pl.two_panel ? 2 : 1;
  pl.ys_off = panels * BK * pl.ld;
  pl.stage_doubles = pl.ys_off + BK * pl.ystride + (mode == MODE_WEIGHTED ? BK : 0);
  pl.stage_doubles = (pl.stage_doubles + 15) / 16 * 16;  // 128-byte aligned stages
  const size_t fixed = (mode == MODE_WEIGHTED ? pl.ld * 8 : 0) + 2 * MAXST * 8;
  // one CTA per SM (16 MMA warps for single-panel plans, 8 for two-panel ones): stages fill 220 KB
  const size_t whole = 220 * 1024;
  pl.ST = (int)std::min<size_t>(pl.two_panel ? 4 : MAXST, (whole - fixed) / ((size_t)pl.stage_doubles * 8));
  if (pl.ST < 2) OEM_FAIL(OEM_ERR_UNSUPPORTED, "gram: stage does not fit shared memory");
  pl.smem = (size_t)pl.ST * pl.stage_doubles * 8 + fixed;
  const int64_t units = std::max<int64_t>(1, (nrows + BK - 1) / BK);
  const int nfold = mode == MODE_FOLD ? K : 1;
  // segments: as many (CTA type, segment) items as a few whole waves over the SMs (below), but at
  // least 64 stages per segment (pipeline fill and the partial-block epilogue amortised; a whole
  // number of waves, so the last one is not a mostly idle partial wave)
  const char* wv = std::getenv("OEM_GRAM_WAVES");  // developer override (timing studies)
  const double per_wave = (double)ctx->num_sms / std::max(1, pl.U * nfold);  // segments per wave
  // single-panel plans (CTA types of equal cost) run best in very few waves: fewer segments, a
  // smaller split-n reduction, fewer pipeline fills. Measured (whole call): cfg2 4 waves 0.396 ms,
  // 2 waves 0.390, 1 wave 0.382; cfg5 weighted pass 33 waves 8.42 ms, 8 waves 8.19, 2 waves 8.16;
  // two-panel plans need many waves to balance their unequal tiles (cfg4: 8 waves 301 ms, 48: 288)
  const double w_fit = std::min(pl.ordered || seg_major ? 384.0 : pl.two_panel ? 48.0 : 2.0, (double)units / 64.0 / per_wave);
  const int waves = wv ? std::max(1, std::atoi(wv)) : std::max(1, (int)std::ceil(w_fit));
  int64_t want = std::max<int64_t>(1, (int64_t)std::llround(waves * per_wave));
  want = std::min<int64_t>(want, std::max<int64_t>(1, units / 8));
  pl.seg_rows = ((units + want - 1) / want) * BK;
  pl.nseg = (int)std::max<int64_t>(1, (nrows + pl.seg_rows - 1) / pl.seg_rows);
  cudaError_t e;
  if ((e = cudaMalloc(&pl.d_ctas, sizeof(CtaDesc) * pl.ctas.size())) != cudaSuccess ||
      (e = cudaMemcpy(pl.d_ctas, pl.ctas.data(), sizeof(CtaDesc) * pl.ctas.size(), cudaMemcpyHostToDevice)) != cudaSuccess ||
      (e = cudaMalloc(&pl.d_blk_of, sizeof(int32_t) * blk_of.size())) != cudaSuccess ||
      (e = cudaMemcpy(pl.d_blk_of, blk_of.data(), sizeof(int32_t) * blk_of.size(), cudaMemcpyHostToDevice)) != cudaSuccess ||
      (e = cudaMalloc(&pl.d_blk_coord, sizeof(int2) * coord.size())) != cudaSuccess ||
      (e = cudaMemcpy(pl.d_blk_coord, coord.data(), sizeof(int2) * coord.size(), cudaMemcpyHostToDevice)) != cudaSuccess)
    OEM_FAIL(OEM_ERR_CUDA, std::string("gram plan tables: ") + cudaGetErrorString(e));
  return OEM_OK;
}

// ------------------------------------------------------------------ TMA descriptors
typedef CUresult (*PFN_encodeTiled)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                    const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                    CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
static PFN_encodeTiled get_encode() {
  static PFN_encodeTiled fn = nullptr;
  if (!fn) {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<PFN_encodeTiled>(p);
  }
  return fn;
}

static oem_status make_map(CUtensorMap* map, const double* X, int rank, const cuuint64_t* dims,
                           const cuuint64_t* strides_bytes, const cuuint32_t* box) {
  PFN_encodeTiled enc = get_encode();
  if (!enc) OEM_FAIL(OEM_ERR_CUDA, "cuTensorMapEncodeTiled unavailable");
  cuuint32_t estr[3] = {1, 1, 1};
  CUresult r = enc(map, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, rank, const_cast<double*>(X), dims, strides_bytes, box, estr,
                   CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                   CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) {
    std::string d = "cuTensorMapEncodeTiled failed (code " + std::to_string((int)r) + ") rank " + std::to_string(rank) +
                    " addr%16=" + std::to_string((uintptr_t)X % 16) + " dims";
    for (int i = 0; i < rank; ++i) d += " " + std::to_string((unsigned long long)dims[i]);
    d += " box";
    for (int i = 0; i < rank; ++i) d += " " + std::to_string(box[i]);
    d += " strides";
    for (int i = 0; i + 1 < rank; ++i) d += " " + std::to_string((unsigned long long)strides_bytes[i]);
    OEM_FAIL(OEM_ERR_CUDA, d);
  }
  return OEM_OK;
}

template <int MODE, bool TWO>
static oem_status launch_t(const GramPlan& pl, const CUtensorMap& mx, const CUtensorMap& my, const GramParams& P,
                           int nfold, cudaStream_t st) {
  auto kern = gram_kernel<MODE, TWO>;
  // opt-in dynamic shared memory, raised on demand; the attribute is per device (a process may
  // drive several devices through several contexts), so the cache is too
  static thread_local size_t attr_smem[64] = {};
  int dev = 0;
  OEM_CUDA_TRY(cudaGetDevice(&dev));
  size_t& cur = attr_smem[dev & 63];
  if (pl.smem > cur) {
    OEM_CUDA_TRY(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)pl.smem));
    cur = pl.smem;
  }
  dim3 grid((unsigned)(pl.U * pl.nseg * nfold));
  kern<<<grid, gram_threads(MODE, TWO), pl.smem, st>>>(mx, my, P);
  OEM_CUDA_TRY(cudaGetLastError());
  return OEM_OK;
}

oem_status gram_pass(oem_ctx* ctx, int mode, const double* X, const double* y, const double* beta, double eps,
                     int64_t n_local, int p, int64_t ldx, int64_t row_offset, int K, double* packed, cudaStream_t st,
                     int accumulate, int want_scal, double* sums) {
  const int ones = sums ? 1 : 0;
  if (ones && (mode == MODE_WEIGHTED || accumulate))
    OEM_FAIL(OEM_ERR_UNSUPPORTED, "gram: the ones column is for single plain / fold passes (internal)");
  const int nfold = mode == MODE_FOLD ? K : 1;
  const int64_t psize = packed_size(p);
  const int64_t nq = mode == MODE_FOLD ? n_local / K : n_local;
  // the weighted pass of two-panel plans: row weights first (HBM-bound), then the WZ contraction
  const bool wz = mode == MODE_WEIGHTED && (8 * ((p + 1 + 7) / 8) + 4) > 256;
  const int kmode = wz ? (int)MODE_WZ : mode;
  if (n_local == 0 || nq == 0) {
    if (!accumulate)
      OEM_CUDA_TRY(cudaMemsetAsync(packed, 0, sizeof(double) * (nfold * psize + (mode == MODE_WEIGHTED ? 2 : 0)), st));
    if (sums) OEM_CUDA_TRY(cudaMemsetAsync(sums, 0, sizeof(double) * nfold * (p + 2), st));
    if (mode != MODE_FOLD || n_local == 0) return OEM_OK;
  }
  auto key = std::make_tuple(kmode, p, nq, K, ones);
  std::shared_ptr<GramPlan> plp;
  auto it = ctx->plans.find(key);
  if (it != ctx->plans.end()) plp = it->second;
  else {
    plp = std::make_shared<GramPlan>();
    oem_status s = build_plan(ctx, kmode, p, std::max<int64_t>(nq, 1), K, ones, *plp);
    if (s != OEM_OK) return s;
    ctx->plans[key] = plp;
  }
  const GramPlan& pl = *plp;
  double* accum = nullptr;
  unsigned* ticket = nullptr;
  if (pl.ordered) {   // running sums [ORD_W][nblk][64] + tickets [ORD_W][U] (one fold)
    const size_t acc_bytes = sizeof(double) * (size_t)ORD_W * pl.nblk * 64;
    OEM_CUDA_TRY(ctx->gram_acc.ensure(acc_bytes + sizeof(unsigned) * (size_t)ORD_W * pl.U + 256));
    accum = ctx->gram_acc.as<double>();
    ticket = reinterpret_cast<unsigned*>(ctx->gram_acc.as<char>() + (acc_bytes + 255) / 256 * 256);
    OEM_CUDA_TRY(cudaMemsetAsync(ticket, 0, sizeof(unsigned) * (size_t)ORD_W * pl.U, st));
  } else {
    const size_t part_bytes = sizeof(double) * (size_t)nfold * pl.nseg * pl.nblk * 64;
    OEM_CUDA_TRY(ctx->partial.ensure(part_bytes));
  }
  OEM_CUDA_TRY(ctx->partial_scal.ensure(sizeof(double) * 2 * (size_t)pl.nseg + 16));
  double* tail = nullptr;
  if (mode == MODE_FOLD && n_local % K != 0) {
    OEM_CUDA_TRY(ctx->tail.ensure(sizeof(double) * (size_t)K * pl.nblk * 64));
    tail = ctx->tail.as<double>();
  }
  int nscal = nq > 0 ? pl.nseg : 0;   // WEIGHTED: (sum w, loglik) partials to add in order
  const double* yin = y;
  if (wz && nq > 0) {
    // per-row (w, z) and the scalar partials, one HBM-bound pass (row_weights_kernel)
    const int64_t rows_per = std::max<int64_t>(64, (n_local + 4 * ctx->num_sms - 1) / (4 * ctx->num_sms));
    const int nb_rw = (int)((n_local + rows_per - 1) / rows_per);
    OEM_CUDA_TRY(ctx->wz.ensure(sizeof(double) * 2 * (size_t)n_local));
    OEM_CUDA_TRY(ctx->partial_scal.ensure(sizeof(double) * 2 * (size_t)std::max(nb_rw, pl.nseg) + 16));
    const size_t bsmem = sizeof(double) * (size_t)(2 * ((p + 1) / 2));
    if (bsmem > 48 * 1024)
      OEM_CUDA_TRY(cudaFuncSetAttribute(row_weights_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bsmem));
    PhaseTimer tm(ctx, PH_GRAM, st);
    ++ctx->launches;
    row_weights_kernel<<<nb_rw, RW_THREADS, bsmem, st>>>(X, y, beta, n_local, p, ldx, eps, rows_per, want_scal,
                                                          ctx->wz.as<double2>(), ctx->partial_scal.as<double>());
    OEM_CUDA_TRY(cudaGetLastError());
    nscal = want_scal ? nb_rw : 0;
    yin = ctx->wz.as<double>();
  }
  if (nq > 0) {
    CUtensorMap mx, my;
    std::memset(&my, 0, sizeof(my));
    const cuuint32_t boxw = (cuuint32_t)pl.ld;
    oem_status s;
    if (kmode == MODE_WZ) {
      cuuint64_t dims[2] = {(cuuint64_t)p, (cuuint64_t)n_local};
      cuuint64_t strides[1] = {(cuuint64_t)ldx * 8};
      cuuint32_t box[2] = {boxw, (cuuint32_t)BK};
      s = make_map(&mx, X, 2, dims, strides, box);
      if (s == OEM_OK) {
        cuuint64_t yd[2] = {2, (cuuint64_t)n_local};
        cuuint64_t ys[1] = {16};
        cuuint32_t yb[2] = {2, (cuuint32_t)BK};
        s = make_map(&my, yin, 2, yd, ys, yb);
      }
    } else if (mode == MODE_FOLD) {
      cuuint64_t dims[3] = {(cuuint64_t)p, (cuuint64_t)K, (cuuint64_t)nq};
      cuuint64_t strides[2] = {(cuuint64_t)ldx * 8, (cuuint64_t)ldx * 8 * K};
      cuuint32_t box[3] = {boxw, 1, (cuuint32_t)BK};
      s = make_map(&mx, X, 3, dims, strides, box);
      if (s == OEM_OK && pl.ytma) {
        cuuint64_t yd[2] = {(cuuint64_t)K, (cuuint64_t)nq};
        cuuint64_t ys[1] = {(cuuint64_t)K * 8};
        cuuint32_t yb[2] = {(cuuint32_t)K, (cuuint32_t)BK};
        s = make_map(&my, y, 2, yd, ys, yb);
      }
    } else {
      cuuint64_t dims[2] = {(cuuint64_t)p, (cuuint64_t)n_local};
      cuuint64_t strides[1] = {(cuuint64_t)ldx * 8};
      cuuint32_t box[2] = {boxw, (cuuint32_t)BK};
      s = make_map(&mx, X, 2, dims, strides, box);
      if (s == OEM_OK) {
        cuuint64_t yd[1] = {(cuuint64_t)n_local};
        cuuint32_t yb[1] = {(cuuint32_t)BK};
        cuuint64_t ydummy[1] = {(cuuint64_t)n_local * 8};  // rank 1: strides unused but must be non-null
        s = make_map(&my, y, 1, yd, ydummy, yb);
      }
    }
    if (s != OEM_OK) return s;
    GramParams P;
    std::memset(&P, 0, sizeof(P));
    P.p = p; P.nb = pl.nb; P.ld = pl.ld; P.U = pl.U; P.U_off = pl.U_off; P.nseg = pl.nseg; P.ST = pl.ST; P.two_panel = pl.two_panel;
    P.nblk = pl.nblk; P.nrows = nq; P.seg_rows = pl.seg_rows; P.K = K;
    P.off_mod = mode == MODE_FOLD ? (int)(((row_offset % K) + K) % K) : 0;
    P.ytma = pl.ytma; P.ystride = pl.ystride;
    P.y = y; P.beta = beta; P.eps = eps; P.want_scal = want_scal; P.ones = ones;
    P.partial = ctx->partial.as<double>();
    P.ordered = pl.ordered;
    P.ticket = ticket;
    P.accum = accum;
    P.partial_scal = ctx->partial_scal.as<double>();
    P.ctas = pl.d_ctas; P.blk_of = pl.d_blk_of;
    P.xbox_bytes = (uint32_t)(BK * pl.ld * 8);
    P.ybox_bytes = pl.ybox_bytes;
    P.stage_doubles = pl.stage_doubles;
    P.ys_off = pl.ys_off;
    oem_status ls;
    PhaseTimer tm(ctx, PH_GRAM, st);
    ++ctx->launches;
    if (!pl.two_panel) {
      if (mode == MODE_PLAIN) ls = launch_t<MODE_PLAIN, false>(pl, mx, my, P, nfold, st);
      else if (mode == MODE_FOLD) ls = launch_t<MODE_FOLD, false>(pl, mx, my, P, nfold, st);
      else ls = launch_t<MODE_WEIGHTED, false>(pl, mx, my, P, nfold, st);
    } else {
      if (mode == MODE_PLAIN) ls = launch_t<MODE_PLAIN, true>(pl, mx, my, P, nfold, st);
      else if (mode == MODE_FOLD) ls = launch_t<MODE_FOLD, true>(pl, mx, my, P, nfold, st);
      else ls = launch_t<MODE_WZ, true>(pl, mx, my, P, nfold, st);
    }
    if (ls != OEM_OK) return ls;
  }
  PhaseTimer tm_red(ctx, PH_REDUCE, st);
  if (tail) {
    ++ctx->launches;
    gram_fold_tail_kernel<<<std::max(1, std::min(1024, (int)((K * (int64_t)pl.nblk * 64 + 255) / 256))), 256, 0, st>>>(
        X, y, ldx, n_local, nq, K, (int)(((row_offset % K) + K) % K), p, pl.nblk, pl.d_blk_coord, tail, ones);
    OEM_CUDA_TRY(cudaGetLastError());
  }
  {
    const double* src = pl.ordered ? accum : ctx->partial.as<double>();
    const double* sscal = ctx->partial_scal.as<double>();
    // ordered plans: the segments are already summed into min(ORD_W, nseg) chains
    int nseg = nq > 0 ? (pl.ordered ? std::min(ORD_W, pl.nseg) : pl.nseg) : 0;
    if (nseg > 64) {  // two-level: chunks of `per` segments in parallel, then the final sum
      const int per = 16, S = (nseg + per - 1) / per;
      OEM_CUDA_TRY(ctx->partial2.ensure(sizeof(double) * (size_t)nfold * S * pl.nblk * 64 + sizeof(double) * (2 * S + 16)));
      double* out = ctx->partial2.as<double>();
      double* oscal = out + (size_t)nfold * S * pl.nblk * 64;
      const int64_t total = (int64_t)nfold * S * pl.nblk * 64;
      const int blocks = (int)std::max<int64_t>(1, std::min<int64_t>(ctx->num_sms * 16, (total + 255) / 256));
      ++ctx->launches;
      const bool chunk_scal = mode == MODE_WEIGHTED && !wz;   // the fused pass: scalars per segment
      gram_chunk_kernel<<<blocks, 256, 0, st>>>(src, nfold, nseg, pl.nblk, S, per, out,
                                                chunk_scal ? sscal : nullptr, oscal);
      OEM_CUDA_TRY(cudaGetLastError());
      src = out;
      if (chunk_scal) { sscal = oscal; nscal = S; }
      nseg = S;
    }
    const int64_t total = (int64_t)nfold * pl.nblk * 64;
    const int blocks = (int)std::max<int64_t>(1, std::min<int64_t>(ctx->num_sms * 8, (total + 255) / 256));
    ++ctx->launches;
    gram_reduce_kernel<<<blocks, 256, 0, st>>>(src, nfold, nseg, pl.nblk, pl.d_blk_coord, p, tail, packed, psize, sscal,
                                               nscal, mode == MODE_WEIGHTED, accumulate, sums);
    OEM_CUDA_TRY(cudaGetLastError());
  }
  return OEM_OK;
}

oem_status gram_unpack(oem_ctx* ctx, const double* packed, int nfold, int p, double* G, double* xty, double* yty,
                       cudaStream_t st) {
  PhaseTimer tm(ctx, PH_REDUCE, st);
  ++ctx->launches;
  const int64_t total = (int64_t)nfold * ((int64_t)p * p + p + 1);
  const int blocks = (int)std::max<int64_t>(1, std::min<int64_t>(4096, (total + 255) / 256));
  gram_unpack_kernel<<<blocks, 256, 0, st>>>(packed, nfold, p, G, xty, yty);
  OEM_CUDA_TRY(cudaGetLastError());
  return OEM_OK;
}

}  // namespace oem
