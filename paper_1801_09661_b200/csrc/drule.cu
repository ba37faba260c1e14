// drule.cu — a7 of the hot path on sm_100a: d >= lambda_1 of every normalised unit Gram.
//
// The method (§2.1): OEM needs d >= lambda_1(X^T X / n) (A = dI - X^T X
// positive semidefinite); d = lambda_1 converges fastest. Reading R#5:
//   d = min(Gershgorin max row sum, U_S),  U_S = trace(G^(2^S))^(1/2^S) * (1 + 2 S p u),
// an upper bound on lambda_1 for every symmetric PSD G (trace(G^m) = sum_i lambda_i^m), within a
// factor p^(2^-S) of it. G^(2^S) comes from S squarings of the trace-normalised matrix:
//   B_0 = G;  s_t = trace(B_t);  B_{t+1} = (B_t / s_t)^2;  log U_S = log s_0 + sum_t 2^-t log s_t.
//
// B200 design: ONE cooperative launch for all units and all S squarings. The squarings are
// p x p x p fp64 products, i.e. dense contractions: they run on the FP64 tensor cores
// (mma.sync m8n8k4 -> DMMA; tcgen05 has no f64 kind). B_t is symmetric, so only the tiles of the
// upper block triangle are computed (the mirror tile is written transposed: the same products in
// the same order, so the result stays bitwise symmetric), and both operands of a tile are row
// panels of B_t (B_t[k][j] = B_t[j][k]) -> every global load is a contiguous 256-byte row segment,
// staged through a 4-deep cp.async ring of 32-column chunks (three chunks in flight hide the L2
// latency). The whole p x p working set (8 MB at p = 1000) stays in L2 between squarings; B_t
// (t >= 1) is read with cp.async.cg (L2 only) because another SM wrote it since this SM last looked. Traces are
// per-diagonal-tile partial sums added in tile order (deterministic); one grid barrier
// (wrap-safe counter) separates the squarings.
#include <algorithm>
#include <cmath>
#include <string>

#include "common.cuh"
#include "internal.h"

namespace oem {

namespace {

// output tiles of DT x DT (64, or 32 for small problems: more CTAs share a squaring, since one
// SM's FP64 rate, ~250 GFLOP/s, bounds a tile's time)
constexpr int DK = 32;          // k-chunk staged in shared memory
constexpr int DPITCH = DK + 4;  // smem row pitch (doubles): 2 wavefronts per 8-byte fragment load
constexpr int DTHR = 256;       // 8 warps: 2 (rows of 32) x 4 (columns of 16)

struct DRuleArgs {
  const double* G;   // [nU][p][p] normalised unit Grams (read only)
  double* buf;       // [2][nU][p][pb] B_1, B_2, ... ping-pong (pb = p rounded up to even)
  double* tr;        // [S+1][nU][nb] partial traces of B_t per diagonal block
  double* gsl;       // [nU][nb] Gershgorin: max row abs-sum per row block
  unsigned* bar;     // grid barrier counter (zero at launch)
  double* d_out;     // [nU]
  int p, pb, nU, nb, ntile, S;   // pb: even row pitch of buf
};

__device__ __forceinline__ unsigned ld_acquire_u32(const unsigned* a) {
  unsigned v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(a) : "memory");
  return v;
}

// all CTAs of the (co-resident) grid; `target` = phase * gridDim.x, compared wrap-safe. The
// CTA barrier orders the CTA's writes before thread 0's release add (cumulative), the acquire
// poll orders the other CTAs' writes before the closing CTA barrier: no sequentially consistent
// fences (a fence.sc per CTA per squaring cost ~10 us at p = 200)
__device__ __forceinline__ void grid_sync(unsigned* bar, unsigned target) {
  __syncthreads();
  if (threadIdx.x == 0) {
    asm volatile("red.release.gpu.global.add.u32 [%0], %1;" ::"l"(bar), "r"(1u) : "memory");
    while ((int)(ld_acquire_u32(bar) - target) < 0) {}
  }
  __syncthreads();
}

// upper-triangle tile index -> (bi, bj), bi <= bj, row-major over the upper triangle
__device__ __forceinline__ void tile_ij(int t, int nb, int& bi, int& bj) {
  int i = 0;
  while (t >= nb - i) { t -= nb - i; ++i; }
  bi = i;
  bj = i + t;
}

__device__ __forceinline__ void cp_async_ca8(double* dst, const double* src) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(smem_u32(dst)), "l"(src) : "memory");
}
__device__ __forceinline__ void cp_async_cg16(double* dst, const double* src) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(smem_u32(dst)), "l"(src) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() { asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory"); }

constexpr int DNS = 4;                       // k-chunks in flight (cp.async ring)
template <int DT>
__global__ void __launch_bounds__(DTHR, 1) drule_kernel(const DRuleArgs A) {
  constexpr int DSTAGE = 2 * DT * DPITCH;      // doubles per ring stage (A and B panels)
  constexpr int MT = DT / 16, NT = DT / 32;    // 8x8 output blocks per warp: MT rows x NT columns
  extern __shared__ __align__(16) double dsm[];   // [DNS][2][DT][DPITCH]
  __shared__ double red[DTHR / 32];
  __shared__ double diag[DT];
  const int p = A.p, nb = A.nb, pb = A.pb, tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const size_t pp = (size_t)p * p, ppb = (size_t)p * pb;
  unsigned phase = 0;

  // ---- phase 0: Gershgorin row sums and the trace of B_0 = G, per (unit, row block)
  for (int w = blockIdx.x; w < A.nU * nb; w += gridDim.x) {
    const int u = w / nb, bi = w % nb;
    const double* Gu = A.G + (size_t)u * pp;
    double gm = 0.0, tr = 0.0;
    for (int r = bi * DT + warp; r < min(p, (bi + 1) * DT); r += DTHR / 32) {
      double s0 = 0.0, s1 = 0.0, s2 = 0.0, s3 = 0.0;   // four loads in flight
      int k = lane;
      for (; k + 96 < p; k += 128) {
        s0 += fabs(Gu[(size_t)r * p + k]);
        s1 += fabs(Gu[(size_t)r * p + k + 32]);
        s2 += fabs(Gu[(size_t)r * p + k + 64]);
        s3 += fabs(Gu[(size_t)r * p + k + 96]);
      }
      for (; k < p; k += 32) s0 += fabs(Gu[(size_t)r * p + k]);
      double s = (s0 + s1) + (s2 + s3);
#pragma unroll
      for (int o = 16; o >= 1; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
      gm = fmax(gm, s);
    }
    if (lane == 0) red[warp] = gm;
    if (tid < DT) diag[tid] = bi * DT + tid < p ? Gu[(size_t)(bi * DT + tid) * p + bi * DT + tid] : 0.0;
    __syncthreads();
    if (tid == 0) {
      for (int i = 0; i < DTHR / 32; ++i) gm = fmax(gm, red[i]);
      for (int i = 0; i < DT; ++i) tr += diag[i];  // fixed order
      A.gsl[(size_t)u * nb + bi] = gm;
      A.tr[(size_t)u * nb + bi] = tr;
    }
    __syncthreads();
  }
  grid_sync(A.bar, ++phase * gridDim.x);

  // ---- phases 1..S: B_{t+1} = (B_t / s_t)^2 on the upper block triangle
  const int wr = warp >> 2, wc = warp & 3;   // warp tile: rows wr DT/2 + [0, DT/2), columns wc DT/4 + [0, DT/4)
  const int nch = (p + DK - 1) / DK;
  for (int t = 0; t < A.S; ++t) {
    // B_0 = G (pitch p, never written by this launch: 8-byte cp.async through L1); B_t, t >= 1,
    // another SM wrote it since this SM last looked: 16-byte cp.async.cg (L2 only), even pitch pb
    const bool first = t == 0;
    const double* Bin = first ? A.G : A.buf + (size_t)((t - 1) & 1) * A.nU * ppb;
    const int ldin = first ? p : pb;
    double* Bout = A.buf + (size_t)(t & 1) * A.nU * ppb;
    for (int w = blockIdx.x; w < A.nU * A.ntile; w += gridDim.x) {
      const int u = w / A.ntile;
      int bi, bj;
      tile_ij(w % A.ntile, nb, bi, bj);
      double s = 0.0;
      for (int b = 0; b < nb; ++b) s += __ldcg(A.tr + ((size_t)t * A.nU + u) * nb + b);  // fixed order
      const double sc = s > 0.0 ? 1.0 / (s * s) : 0.0;
      const double* Bu = Bin + (size_t)u * (first ? pp : ppb);
      const int r0 = bi * DT, c0 = bj * DT;
      // stage chunk c (columns [c DK, c DK + DK)) of the row panels r0.. and c0.. into ring slot c % DNS
      auto issue = [&](int c) {
        if (c < nch) {
          double* As = dsm + (size_t)(c % DNS) * DSTAGE;
          double* Bs = As + DT * DPITCH;
          const int k0 = c * DK;
          if (first) {
#pragma unroll
            for (int i = 0; i < (DT * DK) / DTHR; ++i) {
              const int e = tid + i * DTHR, r = e / DK, kk = k0 + e % DK;
              double* da = As + r * DPITCH + e % DK;
              double* db = Bs + r * DPITCH + e % DK;
              if (r0 + r < p && kk < p) cp_async_ca8(da, Bu + (size_t)(r0 + r) * ldin + kk); else *da = 0.0;
              if (c0 + r < p && kk < p) cp_async_ca8(db, Bu + (size_t)(c0 + r) * ldin + kk); else *db = 0.0;
            }
          } else {
#pragma unroll
            for (int i = 0; i < (DT * DK) / (2 * DTHR); ++i) {
              const int e = 2 * (tid + i * DTHR), r = e / DK, kk = k0 + e % DK;   // column pairs
              double* da = As + r * DPITCH + e % DK;
              double* db = Bs + r * DPITCH + e % DK;
              // kk even, pitch even: a pair never straddles the row; its second element may be the
              // zero pad column p of an odd p (written by the epilogue)
              if (r0 + r < p && kk < p) cp_async_cg16(da, Bu + (size_t)(r0 + r) * ldin + kk); else { da[0] = 0.0; da[1] = 0.0; }
              if (c0 + r < p && kk < p) cp_async_cg16(db, Bu + (size_t)(c0 + r) * ldin + kk); else { db[0] = 0.0; db[1] = 0.0; }
            }
          }
        }
        cp_async_commit();   // one group per chunk index (empty past the end: uniform counting)
      };
      double acc[MT][NT][2];
#pragma unroll
      for (int i = 0; i < MT; ++i)
#pragma unroll
        for (int j = 0; j < NT; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;
#pragma unroll
      for (int c = 0; c < DNS - 1; ++c) issue(c);
      for (int c = 0; c < nch; ++c) {
        issue(c + DNS - 1);
        cp_async_wait<DNS - 1>();   // this thread's copies of chunk c have landed
        __syncthreads();            // ... and every thread's
        const double* As = dsm + (size_t)(c % DNS) * DSTAGE;
        const double* Bs = As + DT * DPITCH;
#pragma unroll
        for (int k4 = 0; k4 < DK; k4 += 4) {
          double a[MT], b[NT];
#pragma unroll
          for (int i = 0; i < MT; ++i) a[i] = As[(wr * (DT / 2) + i * 8 + (lane >> 2)) * DPITCH + k4 + (lane & 3)];
#pragma unroll
          for (int j = 0; j < NT; ++j) b[j] = Bs[(wc * (DT / 4) + j * 8 + (lane >> 2)) * DPITCH + k4 + (lane & 3)];
#pragma unroll
          for (int i = 0; i < MT; ++i)
#pragma unroll
            for (int j = 0; j < NT; ++j) dmma_8x8x4(acc[i][j][0], acc[i][j][1], a[i], b[j]);
        }
        __syncthreads();            // slot c % DNS is refilled by the next iteration's issue
      }
      cp_async_wait<0>();
      // epilogue: scale by 1/s_t^2, write the tile and (off the diagonal) its transpose; the pad
      // column p of an odd p is written as zero (the next squaring's 16-byte copies read it)
      double* Ou = Bout + (size_t)u * ppb;
#pragma unroll
      for (int i = 0; i < MT; ++i)
#pragma unroll
        for (int j = 0; j < NT; ++j)
#pragma unroll
          for (int e = 0; e < 2; ++e) {
            const int r = wr * (DT / 2) + i * 8 + (lane >> 2), c = wc * (DT / 4) + j * 8 + 2 * (lane & 3) + e;
            const double v = acc[i][j][e] * sc;
            if (r0 + r < p && c0 + c < p) {
              Ou[(size_t)(r0 + r) * pb + c0 + c] = v;
              if (bi != bj) Ou[(size_t)(c0 + c) * pb + r0 + r] = v;
            } else if (r0 + r < p && c0 + c == p && pb > p) {
              Ou[(size_t)(r0 + r) * pb + p] = 0.0;
            }
            if (bi == bj && r == c) diag[r] = r0 + r < p ? v : 0.0;
          }
      if (bi == bj) {
        __syncthreads();
        if (tid == 0) {
          double tr = 0.0;
          for (int i = 0; i < DT; ++i) tr += diag[i];  // fixed order
          A.tr[((size_t)(t + 1) * A.nU + u) * nb + bi] = tr;
        }
      }
    }
    grid_sync(A.bar, ++phase * gridDim.x);
  }

  // ---- d = min(Gershgorin, U_S)
  for (int u = blockIdx.x * DTHR + tid; u < A.nU; u += gridDim.x * DTHR) {
    double gm = 0.0;
    for (int b = 0; b < nb; ++b) gm = fmax(gm, __ldcg(A.gsl + (size_t)u * nb + b));
    double logU = 0.0;
    bool zero = false;
    for (int t = 0; t <= A.S; ++t) {
      double s = 0.0;
      for (int b = 0; b < nb; ++b) s += __ldcg(A.tr + ((size_t)t * A.nU + u) * nb + b);
      if (!(s > 0.0)) { zero = t == 0; break; }
      logU += ldexp(log(s), -t);
    }
    const double U = zero ? 0.0 : exp(logU) * (1.0 + 2.0 * (double)A.S * (double)p * 0x1p-53);
    A.d_out[u] = gm < U ? gm : U;
  }
}

}  // namespace

oem_status d_rule(oem_ctx* ctx, const double* Gn, int nU, int p, int S, double* d_out, cudaStream_t st) {
  if (S < 0 || S > 60) OEM_FAIL(OEM_ERR_INVALID_ARG, "d rule: need 0 <= squarings <= 60");
  // 64-wide tiles unless they leave most SMs idle (one unit at p <= ~300: cfg5's inner solves)
  const int nb64 = (p + 63) / 64;
  const int DT = (int64_t)nU * nb64 * (nb64 + 1) / 2 * 4 <= ctx->num_sms ? 32 : 64;
  const int nb = (p + DT - 1) / DT;
  const int ntile = nb * (nb + 1) / 2;
  const size_t pp = (size_t)p * p;
  size_t off = 0;
  auto take = [&](size_t bytes) { size_t o = off; off += (bytes + 255) / 256 * 256; return o; };
  const int pb = p + (p & 1);
  const size_t o_buf = take(S > 0 ? sizeof(double) * 2 * (size_t)nU * p * pb : 8);
  const size_t o_tr = take(sizeof(double) * (size_t)(S + 1) * nU * nb);
  const size_t o_gsl = take(sizeof(double) * (size_t)nU * nb);
  const size_t o_bar = take(sizeof(unsigned));
  OEM_CUDA_TRY(ctx->drule_ws.ensure(off));
  char* base = ctx->drule_ws.as<char>();
  OEM_CUDA_TRY(cudaMemsetAsync(base + o_bar, 0, sizeof(unsigned), st));
  DRuleArgs A;
  A.G = Gn;
  A.buf = reinterpret_cast<double*>(base + o_buf);
  A.tr = reinterpret_cast<double*>(base + o_tr);
  A.gsl = reinterpret_cast<double*>(base + o_gsl);
  A.bar = reinterpret_cast<unsigned*>(base + o_bar);
  A.d_out = d_out;
  A.p = p; A.pb = pb; A.nU = nU; A.nb = nb; A.ntile = ntile; A.S = S;
  const size_t smem = sizeof(double) * (size_t)DNS * 2 * DT * DPITCH;
  const void* kern = DT == 32 ? (const void*)drule_kernel<32> : (const void*)drule_kernel<64>;
  OEM_CUDA_TRY(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  int per_sm = 0;
  OEM_CUDA_TRY(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, DTHR, smem));
  const int work = std::max(nU * ntile, nU * nb);
  const int grid = std::max(1, std::min(work, ctx->num_sms * std::max(1, per_sm)));
  void* args[] = {&A};
  PhaseTimer tm(ctx, PH_POWER, st);
  ++ctx->launches;
  OEM_CUDA_TRY(cudaLaunchCooperativeKernel(kern, dim3(grid), dim3(DTHR), args, smem, st));
  return OEM_OK;
}

}  // namespace oem
