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
// panels of B_t (B_t[k][j] = B_t[j][k]) -> every global load is a contiguous 256-byte row segment.
// The whole p x p working set (8 MB at p = 1000) stays in L2 between squarings; reads use
// ld.global.cg because another SM wrote the data since this SM last looked. Traces are
// per-diagonal-tile partial sums added in tile order (deterministic); one grid barrier
// (wrap-safe counter) separates the squarings.
#include <algorithm>
#include <cmath>
#include <string>

#include "common.cuh"
#include "internal.h"

namespace oem {

namespace {

constexpr int DT = 64;          // output tile (rows and columns)
constexpr int DK = 32;          // k-chunk staged in shared memory
constexpr int DPITCH = DK + 4;  // smem row pitch (doubles): 2 wavefronts per 8-byte fragment load
constexpr int DTHR = 256;       // 8 warps: 2 (rows of 32) x 4 (columns of 16)

struct DRuleArgs {
  const double* G;   // [nU][p][p] normalised unit Grams (read only)
  double* buf;       // [2][nU][p][p] B_1, B_2, ... ping-pong
  double* tr;        // [S+1][nU][nb] partial traces of B_t per diagonal block
  double* gsl;       // [nU][nb] Gershgorin: max row abs-sum per row block
  unsigned* bar;     // grid barrier counter (zero at launch)
  double* d_out;     // [nU]
  int p, nU, nb, ntile, S;
};

__device__ __forceinline__ unsigned ld_acquire_u32(const unsigned* a) {
  unsigned v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(a) : "memory");
  return v;
}

// all CTAs of the (co-resident) grid; `target` = phase * gridDim.x, compared wrap-safe
__device__ __forceinline__ void grid_sync(unsigned* bar, unsigned target) {
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence();
    asm volatile("red.release.gpu.global.add.u32 [%0], %1;" ::"l"(bar), "r"(1u) : "memory");
    while ((int)(ld_acquire_u32(bar) - target) < 0) __nanosleep(32);
    __threadfence();
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

__device__ __forceinline__ double ldcg(const double* a, bool cg) { return cg ? __ldcg(a) : __ldg(a); }

__global__ void __launch_bounds__(DTHR, 1) drule_kernel(const DRuleArgs A) {
  __shared__ __align__(16) double As[DT * DPITCH];
  __shared__ __align__(16) double Bs[DT * DPITCH];
  __shared__ double red[DTHR / 32];
  __shared__ double diag[DT];
  const int p = A.p, nb = A.nb, tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const size_t pp = (size_t)p * p;
  unsigned phase = 0;

  // ---- phase 0: Gershgorin row sums and the trace of B_0 = G, per (unit, row block)
  for (int w = blockIdx.x; w < A.nU * nb; w += gridDim.x) {
    const int u = w / nb, bi = w % nb;
    const double* Gu = A.G + (size_t)u * pp;
    double gm = 0.0, tr = 0.0;
    for (int r = bi * DT + warp; r < min(p, (bi + 1) * DT); r += DTHR / 32) {
      double s = 0.0;
      for (int k = lane; k < p; k += 32) s += fabs(Gu[(size_t)r * p + k]);
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
  const int wr = warp >> 2, wc = warp & 3;
  for (int t = 0; t < A.S; ++t) {
    const bool cg = t > 0;  // B_0 = G was never written by this launch
    const double* Bin = t == 0 ? A.G : A.buf + (size_t)((t - 1) & 1) * A.nU * pp;
    double* Bout = A.buf + (size_t)(t & 1) * A.nU * pp;
    for (int w = blockIdx.x; w < A.nU * A.ntile; w += gridDim.x) {
      const int u = w / A.ntile;
      int bi, bj;
      tile_ij(w % A.ntile, nb, bi, bj);
      double s = 0.0;
      for (int b = 0; b < nb; ++b) s += __ldcg(A.tr + ((size_t)t * A.nU + u) * nb + b);  // fixed order
      const double sc = s > 0.0 ? 1.0 / (s * s) : 0.0;
      const double* Bu = Bin + (size_t)u * pp;
      const int r0 = bi * DT, c0 = bj * DT;
      double acc[4][2][2];
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 2; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;
      // register-staged prefetch of the next k-chunk (8 + 8 doubles per thread)
      double ra[8], rb[8];
      auto fetch = [&](int k0) {
#pragma unroll
        for (int i = 0; i < 8; ++i) {
          const int e = tid + i * DTHR, r = e / DK, kk = k0 + e % DK;
          ra[i] = (r0 + r < p && kk < p) ? ldcg(Bu + (size_t)(r0 + r) * p + kk, cg) : 0.0;
          rb[i] = (c0 + r < p && kk < p) ? ldcg(Bu + (size_t)(c0 + r) * p + kk, cg) : 0.0;
        }
      };
      fetch(0);
      for (int k0 = 0; k0 < p; k0 += DK) {
        __syncthreads();  // previous chunk's fragments consumed
#pragma unroll
        for (int i = 0; i < 8; ++i) {
          const int e = tid + i * DTHR;
          As[(e / DK) * DPITCH + e % DK] = ra[i];
          Bs[(e / DK) * DPITCH + e % DK] = rb[i];
        }
        __syncthreads();
        if (k0 + DK < p) fetch(k0 + DK);
#pragma unroll
        for (int k4 = 0; k4 < DK; k4 += 4) {
          double a[4], b[2];
#pragma unroll
          for (int i = 0; i < 4; ++i) a[i] = As[(wr * 32 + i * 8 + (lane >> 2)) * DPITCH + k4 + (lane & 3)];
#pragma unroll
          for (int j = 0; j < 2; ++j) b[j] = Bs[(wc * 16 + j * 8 + (lane >> 2)) * DPITCH + k4 + (lane & 3)];
#pragma unroll
          for (int i = 0; i < 4; ++i)
#pragma unroll
            for (int j = 0; j < 2; ++j) dmma_8x8x4(acc[i][j][0], acc[i][j][1], a[i], b[j]);
        }
      }
      // epilogue: scale by 1/s_t^2, write the tile and (off the diagonal) its transpose
      double* Ou = Bout + (size_t)u * pp;
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 2; ++j)
#pragma unroll
          for (int e = 0; e < 2; ++e) {
            const int r = wr * 32 + i * 8 + (lane >> 2), c = wc * 16 + j * 8 + 2 * (lane & 3) + e;
            const double v = acc[i][j][e] * sc;
            if (r0 + r < p && c0 + c < p) {
              Ou[(size_t)(r0 + r) * p + c0 + c] = v;
              if (bi != bj) Ou[(size_t)(c0 + c) * p + r0 + r] = v;
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
  const int nb = (p + DT - 1) / DT;
  const int ntile = nb * (nb + 1) / 2;
  const size_t pp = (size_t)p * p;
  size_t off = 0;
  auto take = [&](size_t bytes) { size_t o = off; off += (bytes + 255) / 256 * 256; return o; };
  const size_t o_buf = take(S > 0 ? sizeof(double) * 2 * (size_t)nU * pp : 8);
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
  A.p = p; A.nU = nU; A.nb = nb; A.ntile = ntile; A.S = S;
  int per_sm = 0;
  OEM_CUDA_TRY(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, drule_kernel, DTHR, 0));
  const int work = std::max(nU * ntile, nU * nb);
  const int grid = std::max(1, std::min(work, ctx->num_sms * std::max(1, per_sm)));
  void* args[] = {&A};
  PhaseTimer tm(ctx, PH_POWER, st);
  ++ctx->launches;
  OEM_CUDA_TRY(cudaLaunchCooperativeKernel((const void*)drule_kernel, dim3(grid), dim3(DTHR), args, 0, st));
  return OEM_OK;
}

}  // namespace oem
