// path.cu — a6, a8-a10 of the hot path on sm_100a: normalise the unit Grams, the lambda grid, and
// the OEM path iterations for every (Gram, penalty) unit (a7, d, runs in drule.cu in between).
//
// The method: OEM's EM step in closed form, u = X^T y + (dI - X^T X) beta
// (P:L171-172), followed by the penalty's thresholding M-step (eqs lasso / net /
// mcp / scad / glasso / gmcp / gscad), iterated to convergence along a warm-started lambda path
// (R#17-18), for several penalties sharing one Gram (§5.2) and for the K fold
// complements of fast CV (§3). d >= lambda_1 by the d rule R#5 (drule.cu).
//
// B200 design: one persistent cooperative launch. Each unit Gram g is owned by a group of C_g
// CTAs; CTA c keeps its slice of rows of G resident in shared memory for the whole path (the
// p x p matrix never leaves the SMs), and all penalties on that Gram are advanced together so
// each G element loaded from smem feeds nP FMAs (the "small GEMM across penalties"). A row is
// reduced by T_r lanes with xor-shuffles; coordinate-wise thresholds run on the row leader,
// group thresholds after a CTA-level exchange (groups never straddle CTAs). Per iteration the
// group exchanges the new beta through L2 (double-buffered) and meets at one barrier; the
// convergence test max |dbeta| uses a uint64 atomicMax (order independent, so deterministic).
// No host round-trip per iteration or per lambda.
#include <algorithm>
#include <cmath>
#include <cstring>
#include <numeric>
#include <type_traits>
#include <vector>

#include <cstdlib>
#include <string>

#include "common.cuh"
#include "internal.h"

namespace oem {

constexpr int PT = 512;          // threads per solver CTA
constexpr int MAXG = 4096;       // max groups (group penalties)

struct PathParams {
  int p, nP, L, nU;              // nU = number of unit Grams (nG')
  int ps;                        // smem row pitch (doubles)
  int T;                         // lanes per row
  int64_t maxit;
  double tol;
  const double* Gn;              // [nU][p][p] normalised (permuted) unit Grams
  const double* cn;              // [nU][p]
  const int* cta_unit;           // [ncta] unit of each CTA
  const int* cta_rank;           // [ncta] rank of the CTA within its unit group
  const int* unit_ncta;          // [nU]
  const int* cta_j0;             // [ncta] first row
  const int* cta_j1;             // [ncta] end row
  int smem_rows;                 // rows cached in smem (>= max rows per CTA, else G read from global)
  // penalties
  const int* fam;                // [nP]
  const double* gam;             // [nP]
  const double* alp;             // [nP]
  const double* var_w;           // [p] (permuted) or null
  int ngroups;
  const int* g_start;            // [ngroups] (permuted, contiguous)
  const int* g_end;
  const double* g_w;             // [ngroups]
  const int* g_of;               // [p] group id (permuted order) or null
  const int* perm;               // [p] original index of permuted coordinate j
  // lambda
  const double* lam_explicit;    // [L] or null
  double lmin_ratio;
  int shared_grid;               // fold mode: every unit uses unit 0's lambda_max
  const double* lmax_override;   // device scalar or null
  // state / outputs
  const double* d;               // [nU]
  const double* beta_init;       // [nU][nP][p] original order or null
  double* bbuf;                  // [2][nU][nP][p] exchange buffers
  unsigned long long* dslot;     // [3][nU][nP]
  unsigned int* bar;             // [nU][2] barrier counter / generation
  double* beta_out;              // [nU][nP][L][p] original order
  double* lam_out;               // [nU][nP][L]
  int64_t* it_out;
  uint8_t* cv_out;
  int* flags;                    // [0] non-finite, [1] invalid parameter
  unsigned long long* bad_iter;  // [nU] first iteration with a non-finite u (all ones = none)
};

// ---------------------------------------------------------------- group barrier (global memory)
__device__ __forceinline__ unsigned ld_acquire(const unsigned* p) {
  unsigned v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void group_barrier(unsigned* bar, int C) {
  __syncthreads();
  if (C > 1 && threadIdx.x == 0) {
    unsigned* cnt = bar;
    unsigned* gen = bar + 1;
    const unsigned g = ld_acquire(gen);
    __threadfence();
    if (atomicAdd(cnt, 1u) == (unsigned)C - 1u) {
      atomicExch(cnt, 0u);
      __threadfence();
      atomicAdd(gen, 1u);
    } else {
      while (ld_acquire(gen) == g) { __nanosleep(20); }
    }
    __threadfence();
  }
  __syncthreads();
}

// ---------------------------------------------------------------- thresholding operators (K6)
// exact transcriptions of PAPER.md §2.2; lam is the weighted level (w_j lambda or c_k lambda)
__device__ __forceinline__ double sgn(double u) { return u > 0.0 ? 1.0 : (u < 0.0 ? -1.0 : 0.0); }
__device__ __forceinline__ double pos(double a) { return a > 0.0 ? a : 0.0; }
// (a non-positive numerator gives pos(.) = 0 without dividing: the fp64 division routine is long,
// and the thresholded coordinates of a sparse path are mostly zero)
__device__ __forceinline__ double th_soft(double u, double lam, double d) {     // eq (lasso)
  const double t = fabs(u) - lam;
  return t > 0.0 ? sgn(u) * (t / d) : 0.0;
}
__device__ __forceinline__ double th_enet(double u, double lam, double a, double d) {  // eq (net)
  const double t = fabs(u) - lam * a;
  return t > 0.0 ? sgn(u) * (t / (d + lam * (1.0 - a))) : 0.0;
}
// (a zero numerator is returned without dividing: 0/x takes the slow path of the fp64 division
// routine on the GPU, and the thresholded coordinates of a sparse path are mostly zero)
__device__ __forceinline__ double th_mcp(double u, double lam, double g, double d) {   // eq (mcp)
  if (fabs(u) <= lam * g * d) {
    const double t = pos(fabs(u) - lam);
    return t > 0.0 ? sgn(u) * g * t / (g * d - 1.0) : 0.0;
  }
  return u / d;
}
__device__ __forceinline__ double th_scad(double u, double lam, double g, double d) {  // eq (scad)
  const double a = fabs(u);
  if (a <= (d + 1.0) * lam) {
    const double t = pos(a - lam);
    return t > 0.0 ? sgn(u) * t / d : 0.0;
  }
  if (a <= lam * g * d) return sgn(u) * ((g - 1.0) * a - lam * g) / ((g - 1.0) * d - 1.0);
  return u / d;
}
__device__ __forceinline__ double th_coord(int fam, double u, double lam, double g, double a, double d) {
  switch (fam) {
    case OEM_LASSO: return th_soft(u, lam, d);
    case OEM_ENET: return th_enet(u, lam, a, d);
    case OEM_MCP: return th_mcp(u, lam, g, d);
    default: return th_scad(u, lam, g, d);
  }
}

// The same operators with the constant divisors' reciprocals precomputed (rd = 1/d; rg = 1/(g d - 1)
// for MCP, 1/((g - 1) d - 1) for SCAD): each division becomes x r refined by one fused
// multiply-add on the exact remainder (q = x r, q += (x - q den) r), the correctly rounded
// quotient to within one ulp (~40 cycles of dependent FMAs instead of the ~130-cycle fp64
// division routine, measured by tools/lat_probe.cu). Used by the lean solver, whose iteration
// is one short dependent chain; the elastic net (a divisor that moves with lambda) divides.
__device__ __forceinline__ double div_r(double x, double den, double r) {
  const double q = x * r;
  return fma(fma(-q, den, x), r, q);
}
__device__ __forceinline__ double th_coord_r(int fam, double u, double lam, double g, double a, double d, double rd,
                                             double rg) {
  switch (fam) {
    case OEM_LASSO: {
      const double t = fabs(u) - lam;
      return t > 0.0 ? sgn(u) * div_r(t, d, rd) : 0.0;
    }
    case OEM_ENET: return th_enet(u, lam, a, d);
    case OEM_MCP:
      if (fabs(u) <= lam * g * d) {
        const double t = pos(fabs(u) - lam);
        return t > 0.0 ? div_r(sgn(u) * g * t, g * d - 1.0, rg) : 0.0;
      }
      return div_r(u, d, rd);
    default: {
      const double aa = fabs(u);
      if (aa <= (d + 1.0) * lam) {
        const double t = pos(aa - lam);
        return t > 0.0 ? div_r(sgn(u) * t, d, rd) : 0.0;
      }
      if (aa <= lam * g * d) return div_r(sgn(u) * ((g - 1.0) * aa - lam * g), (g - 1.0) * d - 1.0, rg);
      return div_r(u, d, rd);
    }
  }
}

// Sparse group lasso (eq sglasso; Table 1 with tau in the alpha field): the M-step
// minimiser is v_r = S(u_r, w_r lam tau, d) followed by the group shrink at level
// c lam (1 - tau) / d (exact composition, R#11). Returns f with beta_r = f * v_r.
__device__ __forceinline__ double sgl_factor(const double* ug, int a, int b, int stride, const double* wv, int wj0,
                                            double lam, double tau, double c, double d) {
  double s = 0.0;
  for (int r = a; r < b; ++r) {
    const double v = th_soft(ug[(size_t)r * stride], (wv ? wv[wj0 + r] : 1.0) * lam * tau, d);
    s += v * v;
  }
  const double nv = sqrt(s);
  return nv > 0.0 ? pos(1.0 - c * lam * (1.0 - tau) / (d * nv)) : 0.0;
}
// lambda_max of one group for the sparse group lasso (R#36): root of
// ||S(c_g, lam tau w_g, 1)|| = lam (1 - tau) c_g by bisection, nudged clear of the rounding
__device__ double sgl_lmax_group(const double* cc, int a, int b, const double* wv, double cg, double tau) {
  double hi = 0.0, s = 0.0;
  for (int j = a; j < b; ++j) {
    const double wj = wv ? wv[j] : 1.0;
    if (tau > 0.0 && wj > 0.0) hi = fmax(hi, fabs(cc[j]) / (tau * wj));
    s += cc[j] * cc[j];
  }
  if (tau < 1.0 && cg > 0.0) hi = fmax(hi, sqrt(s) / ((1.0 - tau) * cg));
  double lo = 0.0;
  for (int it = 0; it < 200 && hi > lo; ++it) {
    const double mid = 0.5 * (lo + hi);
    if (mid <= lo || mid >= hi) break;
    double t2 = 0.0;
    for (int j = a; j < b; ++j) {
      const double t = pos(fabs(cc[j]) - mid * tau * (wv ? wv[j] : 1.0));
      t2 += t * t;
    }
    if (sqrt(t2) > mid * (1.0 - tau) * cg) lo = mid;
    else hi = mid;
  }
  return hi * (1.0 + 1e-12);
}

// One group's M-step by a whole warp (eqs glasso / gmcp / gscad / sglasso): lanes
// own rows ra + lane + 32i, the norms are butterfly sums (fixed order), then every lane emits its
// rows' new coordinates through emit(r, nb). ug: u of the group's rows (index r).
template <class Emit>
__device__ __forceinline__ void group_mstep_warp(const double* ug, int ra, int rb, int fam, double lq, double gq,
                                                 double tau, double cg, double d, const double* wv, int j0, int lane,
                                                 Emit&& emit) {
  const bool sgl = fam == OEM_SGL;
  double ss = 0.0;
  for (int r = ra + lane; r < rb; r += 32) {
    const double v = sgl ? th_soft(ug[r], (wv ? wv[j0 + r] : 1.0) * lq * tau, d) : ug[r];
    ss += v * v;
  }
#pragma unroll
  for (int o = 16; o >= 1; o >>= 1) ss += __shfl_xor_sync(0xffffffffu, ss, o);
  const double nu = sqrt(ss);
  const double lw = cg * lq;
  double f;
  if (sgl) f = nu > 0.0 ? pos(1.0 - cg * lq * (1.0 - tau) / (d * nu)) : 0.0;   // R#11 (nu = ||v||)
  else if (fam == OEM_GRP_LASSO) f = nu > 0.0 ? pos(1.0 - lw / nu) : 0.0;
  else f = nu > 0.0 ? (fam == OEM_GRP_MCP ? th_mcp(nu, lw, gq, d) : th_scad(nu, lw, gq, d)) / nu : 0.0;
  for (int r = ra + lane; r < rb; r += 32) {
    const double nb = sgl ? f * th_soft(ug[r], (wv ? wv[j0 + r] : 1.0) * lq * tau, d)
                    : fam == OEM_GRP_LASSO ? ug[r] / d * f : f * ug[r];
    emit(r, nb);
  }
}

__device__ __forceinline__ void atomic_max_pos(unsigned long long* slot, double v) {
  // v >= 0: IEEE order equals unsigned-integer order of the bit patterns
  atomicMax(slot, (unsigned long long)__double_as_longlong(v));
}

// ---------------------------------------------------------------- prep: normalise unit Grams
// fold_mode = 0: unit g = G[g]/n_g. fold_mode = 1: unit 0 = (sum_k G_k)/n, unit k = (sum - G_{k-1})/(n - n_{k-1}).
// Coordinates are permuted so every group is contiguous: Gn[u][j][l] = Graw[perm[j]][perm[l]].
// f3 (R#2-3): per unit, in original coordinates, xbar_j = (X^T 1)_j / n, ybar = 1^T y / n (0 without
// an intercept) and inv_s_j = 1 / sd_j of the centred column (1 without standardization; 0 for a
// zero-variance column, which then drops out: its row/column of the unit Gram become 0).
__device__ __forceinline__ double unit_raw(const double* src, int nG, int u, int fold_mode, size_t stride, size_t off) {
  if (!fold_mode) return src[(size_t)u * stride + off];
  double s = 0.0;
  for (int k = 0; k < nG; ++k) s += src[(size_t)k * stride + off];  // fixed order
  return (u == 0) ? s : s - src[(size_t)(u - 1) * stride + off];    // total minus fold (R#20)
}
__global__ void unit_stats_kernel(const double* __restrict__ G, const double* __restrict__ xsum,
                                  const double* __restrict__ ysum, int nG, int p, int fold_mode,
                                  const double* __restrict__ inv_n, int standardize, double* __restrict__ mean,
                                  double* __restrict__ ybar, double* __restrict__ inv_s) {
  const int u = blockIdx.x;
  const double in = inv_n[u];
  if (threadIdx.x == 0) ybar[u] = ysum ? unit_raw(ysum, nG, u, fold_mode, 1, 0) * in : 0.0;
  for (int j = threadIdx.x; j < p; j += blockDim.x) {
    const double m = xsum ? unit_raw(xsum, nG, u, fold_mode, p, j) * in : 0.0;
    mean[(size_t)u * p + j] = m;
    double is = 1.0;
    if (standardize) {
      const double v = unit_raw(G, nG, u, fold_mode, (size_t)p * p, (size_t)j * p + j) * in - m * m;
      is = v > 0.0 ? 1.0 / sqrt(v) : 0.0;
    }
    inv_s[(size_t)u * p + j] = is;
  }
}

// After the solver: beta (original order) back to the original scale, beta_j = beta~_j inv_s_j,
// and the intercept b0 = ybar - xbar^T beta (one warp per (unit, penalty, lambda), fixed order).
__global__ void backtransform_kernel(double* __restrict__ beta, int nU, int nP, int L, int p,
                                     const double* __restrict__ mean, const double* __restrict__ ybar,
                                     const double* __restrict__ inv_s, double* __restrict__ b0) {
  const int w = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, lane = threadIdx.x & 31;
  if (w >= nU * nP * L) return;
  const int u = w / (nP * L);
  double* b = beta + (size_t)w * p;
  double s = 0.0;
  for (int j = lane; j < p; j += 32) {
    const double v = b[j] * inv_s[(size_t)u * p + j];
    b[j] = v;
    s = fma(mean[(size_t)u * p + j], v, s);
  }
#pragma unroll
  for (int o = 16; o >= 1; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
  if (lane == 0 && b0) b0[w] = ybar[u] - s;
}

__global__ void prep_units_kernel(const double* __restrict__ G, const double* __restrict__ xty, int nG, int p,
                                  int fold_mode, const double* __restrict__ inv_n, const int* __restrict__ perm,
                                  const double* __restrict__ mean, const double* __restrict__ ybar,
                                  const double* __restrict__ inv_s,
                                  double* __restrict__ Gn, double* __restrict__ cn, int* flags) {
  const int nU = fold_mode ? nG + 1 : nG;
  const int64_t per = (int64_t)p * p + p;
  const int64_t total = (int64_t)nU * per;
  const size_t pp = (size_t)p * p;
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < total; t += (int64_t)gridDim.x * blockDim.x) {
    const int u = (int)(t / per);
    const int64_t q = t % per;
    size_t off;
    int64_t stride;
    double* dst;
    if (q < (int64_t)p * p) {
      const int j = (int)(q / p), l = (int)(q % p);
      off = (size_t)perm[j] * p + perm[l];
      stride = (int64_t)pp;
      dst = Gn + (size_t)u * pp + q;
    } else {
      const int j = (int)(q - (int64_t)p * p);
      off = perm[j];
      stride = p;
      dst = cn + (size_t)u * p + j;
    }
    const double* src = q < (int64_t)p * p ? G : xty;
    double v;
    if (!fold_mode) {
      v = src[(size_t)u * stride + off];
    } else {
      double s = 0.0;
      for (int k = 0; k < nG; ++k) s += src[(size_t)k * stride + off];  // fixed order
      v = (u == 0) ? s : s - src[(size_t)(u - 1) * stride + off];    // total minus fold (R#20)
    }
    v = v * inv_n[u];
    if (mean) {  // centring and standardization (R#2-3); identity (bit for bit) when not requested
      const size_t mo = (size_t)u * p;
      if (q < (int64_t)p * p) {
        const int a = perm[(int)(q / p)], b = perm[(int)(q % p)];
        v = (v - mean[mo + a] * mean[mo + b]) * inv_s[mo + a] * inv_s[mo + b];
      } else {
        const int a = perm[(int)(q - (int64_t)p * p)];
        v = (v - mean[mo + a] * ybar[u]) * inv_s[mo + a];
      }
    }
    if (!isfinite(v)) flags[0] = 1;
    *dst = v;
  }
}

// ---------------------------------------------------------------- shared pieces of the persistent kernels
struct CtaView {
  int unit, rank, C, j0, j1, nr;
  const double* Gu;   // global rows of this unit
};

__device__ __forceinline__ CtaView cta_view(const PathParams& P) {
  CtaView v;
  v.unit = P.cta_unit[blockIdx.x];
  v.rank = P.cta_rank[blockIdx.x];
  v.C = P.unit_ncta[v.unit];
  v.j0 = P.cta_j0[blockIdx.x];
  v.j1 = P.cta_j1[blockIdx.x];
  v.nr = v.j1 - v.j0;
  v.Gu = P.Gn + (size_t)v.unit * P.p * P.p;
  return v;
}

// This CTA's rows of the unit Gram -> shared memory (resident for the whole launch).
__device__ __forceinline__ void load_rows(const PathParams& P, const CtaView& v, double* Gs) {
  for (int e = threadIdx.x; e < v.nr * P.p; e += blockDim.x) {
    const int r = e / P.p, k = e % P.p;
    Gs[r * P.ps + k] = v.Gu[(size_t)(v.j0 + r) * P.p + k];
  }
}

// deterministic block sum (fixed tree order); red needs 33 doubles
__device__ double block_sum(double x, double* red) {
  for (int o = 16; o > 0; o >>= 1) x += __shfl_xor_sync(0xffffffffu, x, o);
  const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
  __syncthreads();
  if (l == 0) red[w] = x;
  __syncthreads();
  if (threadIdx.x == 0) {
    double s = 0.0;
    for (int i = 0; i < (int)(blockDim.x >> 5); ++i) s += red[i];
    red[32] = s;
  }
  __syncthreads();
  const double r = red[32];
  __syncthreads();
  return r;
}
__device__ double block_max(double x, double* red) {
  for (int o = 16; o > 0; o >>= 1) x = fmax(x, __shfl_xor_sync(0xffffffffu, x, o));
  const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
  __syncthreads();
  if (l == 0) red[w] = x;
  __syncthreads();
  if (threadIdx.x == 0) {
    double s = 0.0;
    for (int i = 0; i < (int)(blockDim.x >> 5); ++i) s = fmax(s, red[i]);
    red[32] = s;
  }
  __syncthreads();
  const double r = red[32];
  __syncthreads();
  return r;
}

// w[r] = sum_k G[j0+r][k] * vec[k] for the local rows (T lanes per row, all lanes of every warp
// take part in each round so the width-T shuffles are convergent). Result in uv[r].
__device__ __forceinline__ void row_matvec(const PathParams& P, const CtaView& v, const double* Gs, const double* vec,
                                           double* uv, bool absval) {
  const int T = P.T, groups = blockDim.x / T;
  const int rg = threadIdx.x / T, tl = threadIdx.x % T;
  for (int rb = 0; rb < v.nr; rb += groups) {
    const int r = rb + rg;
    double a = 0.0;
    if (r < v.nr) {
      const double* grow = Gs + (size_t)r * P.ps;
      if (absval) for (int k = tl; k < P.p; k += T) a += fabs(grow[k]);
      else for (int k = tl; k < P.p; k += T) a = fma(grow[k], vec[k], a);
    }
    for (int o = T >> 1; o > 0; o >>= 1) a += __shfl_xor_sync(0xffffffffu, a, o, T);
    if (r < v.nr && tl == 0) uv[r] = a;
  }
}

// ---------------------------------------------------------------- K5: the persistent OEM path solver
template <int NPT>
__global__ void __launch_bounds__(PT, 1) path_kernel(const PathParams P) {
  extern __shared__ __align__(16) double sm[];
  const CtaView v = cta_view(P);
  const int p = P.p, nP = P.nP, L = P.L;
  double* Gs = sm;
  double* vec = Gs + (size_t)P.smem_rows * P.ps;         // current beta [NPT][ps] (all p coordinates)
  double* uv = vec + (size_t)NPT * P.ps;                  // u, then beta', local rows [NPT][smem_rows]
  __shared__ int s_lidx[NPT];
  __shared__ int64_t s_it[NPT];
  __shared__ double s_lam[NPT];
  __shared__ double s_lmax[NPT];
  __shared__ double s_delta[NPT];
  __shared__ int s_bad, s_stop;
  unsigned* bar = P.bar + 2 * v.unit;
  const double d = P.d[v.unit];
  const double* c = P.cn + (size_t)v.unit * p;

  load_rows(P, v, Gs);
  // warm start / cold start beta (full vector on every CTA), permuted order
  for (int q = 0; q < nP; ++q)
    for (int k = threadIdx.x; k < p; k += blockDim.x)
      vec[q * P.ps + k] = P.beta_init ? P.beta_init[((size_t)v.unit * nP + q) * p + P.perm[k]] : 0.0;
  // lambda_max per penalty (R#14), from this unit's c, or unit 0's in fold mode (R#22)
  if (threadIdx.x < nP) {
    const int q = threadIdx.x;
    const int fam = P.fam[q];
    const double* cc = P.shared_grid ? P.cn : c;
    double lm = 0.0;
    if (P.lmax_override) {
      lm = *P.lmax_override;
    } else if (fam == OEM_SGL) {
      for (int g = 0; g < P.ngroups; ++g)
        lm = fmax(lm, sgl_lmax_group(cc, P.g_start[g], P.g_end[g], P.var_w, P.g_w[g], P.alp[q]));
    } else if (fam >= OEM_GRP_LASSO) {
      for (int g = 0; g < P.ngroups; ++g) {
        const double cg = P.g_w[g];
        if (!(cg > 0.0)) continue;
        double s = 0.0;
        for (int j = P.g_start[g]; j < P.g_end[g]; ++j) s += cc[j] * cc[j];
        lm = fmax(lm, sqrt(s) / cg);
      }
    } else {
      const double sc = fam == OEM_ENET ? P.alp[q] : 1.0;
      for (int j = 0; j < p; ++j) {
        const double wj = P.var_w ? P.var_w[j] : 1.0;
        if (!(wj > 0.0)) continue;
        lm = fmax(lm, fabs(cc[j]) / (sc * wj));
      }
    }
    s_lmax[q] = lm;
    s_lidx[q] = 0;
    s_it[q] = 0;
    // parameter validity against the d in use (R#8): the paper's denominators must be > 0
    const double g = P.gam[q];
    bool bad = false;
    if (fam == OEM_MCP || fam == OEM_GRP_MCP) bad = !(g > 1.0) || !(g * d > 1.0);
    if (fam == OEM_SCAD || fam == OEM_GRP_SCAD) bad = !(g > 2.0) || !((g - 1.0) * d > 1.0);
    if (fam == OEM_ENET) bad = !(P.alp[q] >= 0.0 && P.alp[q] <= 1.0);
    if (bad) { atomicExch(&P.flags[1], 1); s_lidx[q] = L; }
  }
  if (threadIdx.x == 0) { s_bad = 0; s_stop = 0; }
  __syncthreads();
  auto lambda_at = [&](int q, int l) -> double {
    if (P.lam_explicit) return P.lam_explicit[l];
    if (L == 1) return s_lmax[q];
    return s_lmax[q] * exp(((double)l / (double)(L - 1)) * log(P.lmin_ratio));  // R#15
  };
  if (threadIdx.x < nP) {
    const int q = threadIdx.x;
    if (s_lidx[q] < L) s_lam[q] = lambda_at(q, 0);
    if (v.rank == 0)
      for (int l = 0; l < L; ++l) P.lam_out[((size_t)v.unit * nP + q) * L + l] = lambda_at(q, l);
  }
  __syncthreads();

  const int T = P.T, groups_rows = blockDim.x / T;
  const int rg = threadIdx.x / T, tl = threadIdx.x % T;
  const bool grp = P.g_of != nullptr;

  for (int64_t t = 0;; ++t) {
    uint32_t qmask = 0;  // units (penalties) still on their path; identical on every CTA of the group
    for (int q = 0; q < nP; ++q)
      if (s_lidx[q] < L) qmask |= 1u << q;
    if (!qmask) break;
    const int slot = (int)(t % 3);
    unsigned long long* ds = P.dslot + ((size_t)slot * P.nU + v.unit) * nP;
    // ---- E-step + M-step in closed form: u = c + d beta - G beta, local rows
    for (int rb = 0; rb < v.nr; rb += groups_rows) {
      const int r = rb + rg;
      double acc[NPT];
#pragma unroll
      for (int q = 0; q < NPT; ++q) acc[q] = 0.0;
      if (r < v.nr) {
        const double* grow = Gs + (size_t)r * P.ps;
        for (int k = tl; k < p; k += T) {
          const double g = grow[k];
#pragma unroll
          for (int q = 0; q < NPT; ++q)
            if ((qmask >> q) & 1u) acc[q] = fma(g, vec[q * P.ps + k], acc[q]);
        }
      }
#pragma unroll
      for (int q = 0; q < NPT; ++q) {
        if (!((qmask >> q) & 1u)) continue;
        double a = acc[q];
        for (int o = T >> 1; o > 0; o >>= 1) a += __shfl_xor_sync(0xffffffffu, a, o, T);
        if (tl == 0 && r < v.nr) {
          const int j = v.j0 + r;
          const double u = c[j] + d * vec[q * P.ps + j] - a;
          if (!isfinite(u)) s_bad = 1;
          if (!grp || P.fam[q] < OEM_GRP_LASSO) {  // coordinate-wise family (also when mixed with group ones)
            const double wj = P.var_w ? P.var_w[j] : 1.0;
            uv[q * P.smem_rows + r] = th_coord(P.fam[q], u, wj * s_lam[q], P.gam[q], P.alp[q], d);
          } else {
            uv[q * P.smem_rows + r] = u;
          }
        }
      }
    }
    __syncthreads();
    if (grp && v.nr > 0) {
      // group M-step (eqs glasso / gmcp / gscad): groups are contiguous, inside [j0, j1)
      const int g0 = P.g_of[v.j0], g1 = P.g_of[v.j1 - 1] + 1;
      for (int e = threadIdx.x; e < (g1 - g0) * nP; e += blockDim.x) {
        const int q = e % nP, gid = g0 + e / nP;
        if (!((qmask >> q) & 1u) || P.fam[q] < OEM_GRP_LASSO) continue;
        const int a = P.g_start[gid] - v.j0, b = P.g_end[gid] - v.j0;
        double* ug = uv + q * P.smem_rows;
        double s = 0.0;
        for (int r = a; r < b; ++r) s += ug[r] * ug[r];
        const double nu = sqrt(s);
        const double lam = P.g_w[gid] * s_lam[q];
        const int fam = P.fam[q];
        if (fam == OEM_SGL) {
          const double tau = P.alp[q];
          const double f = sgl_factor(ug, a, b, 1, P.var_w, v.j0, s_lam[q], tau, P.g_w[gid], d);
          for (int r = a; r < b; ++r)
            ug[r] = f * th_soft(ug[r], (P.var_w ? P.var_w[v.j0 + r] : 1.0) * s_lam[q] * tau, d);
        } else if (fam == OEM_GRP_LASSO) {
          const double f = nu > 0.0 ? pos(1.0 - lam / nu) : 0.0;     // (u/d)(1 - c lam/||u||)_+
          for (int r = a; r < b; ++r) ug[r] = ug[r] / d * f;
        } else {
          const double sc = nu > 0.0 ? (fam == OEM_GRP_MCP ? th_mcp(nu, lam, P.gam[q], d)
                                                          : th_scad(nu, lam, P.gam[q], d)) / nu
                                     : 0.0;
          for (int r = a; r < b; ++r) ug[r] = sc * ug[r];
        }
      }
      __syncthreads();
    }
    // ---- delta = max |beta' - beta| over local rows; publish beta'
    double* nb = P.bbuf + ((size_t)(t & 1) * P.nU + v.unit) * nP * p;
    for (int q = 0; q < nP; ++q) {
      if (!((qmask >> q) & 1u)) continue;
      double m = 0.0;
      for (int r = threadIdx.x; r < v.nr; r += blockDim.x) {
        const double b = uv[q * P.smem_rows + r];
        m = fmax(m, fabs(b - vec[q * P.ps + v.j0 + r]));
        if (v.C > 1) nb[(size_t)q * p + v.j0 + r] = b;
      }
      for (int o = 16; o > 0; o >>= 1) m = fmax(m, __shfl_xor_sync(0xffffffffu, m, o));
      if ((threadIdx.x & 31) == 0 && m > 0.0) atomic_max_pos(&ds[q], m);
    }
    // reset the slot used next iteration (3 rotating slots: no reader or writer is on it now)
    if (v.rank == 0 && threadIdx.x < nP) P.dslot[((size_t)((t + 1) % 3) * P.nU + v.unit) * nP + threadIdx.x] = 0ull;
    __syncthreads();
    if (threadIdx.x == 0 && s_bad) atomicMin(&P.bad_iter[v.unit], (unsigned long long)t);
    __threadfence();
    group_barrier(bar, v.C);
    // ---- every CTA of the group reads the same delta and the new beta
    if (threadIdx.x < nP) {
      const unsigned long long bits = __ldcg(&ds[threadIdx.x]);
      s_delta[threadIdx.x] = __longlong_as_double((long long)bits);
    }
    if (threadIdx.x == 0) s_stop = __ldcg(&P.bad_iter[v.unit]) <= (unsigned long long)t;
    if (v.C > 1) {
      for (int q = 0; q < nP; ++q) {
        if (!((qmask >> q) & 1u)) continue;
        for (int k = threadIdx.x; k < p; k += blockDim.x) vec[q * P.ps + k] = __ldcg(nb + (size_t)q * p + k);
      }
    } else {
      for (int q = 0; q < nP; ++q) {
        if (!((qmask >> q) & 1u)) continue;
        for (int r = threadIdx.x; r < v.nr; r += blockDim.x) vec[q * P.ps + v.j0 + r] = uv[q * P.smem_rows + r];
      }
    }
    __syncthreads();
    if (s_stop) {
      if (threadIdx.x == 0) atomicExch(&P.flags[0], 1);
      break;
    }
    // ---- per-unit convergence bookkeeping (identical decisions on every CTA of the group)
    for (int q = 0; q < nP; ++q) {
      if (!((qmask >> q) & 1u)) continue;
      const int64_t it = s_it[q] + 1;
      const bool conv = s_delta[q] <= P.tol;   // R#17: max_j |dbeta_j| <= tol
      if (conv || it >= P.maxit) {
        const int l = s_lidx[q];
        double* out = P.beta_out + (((size_t)v.unit * nP + q) * L + l) * p;
        for (int r = threadIdx.x; r < v.nr; r += blockDim.x) out[P.perm[v.j0 + r]] = vec[q * P.ps + v.j0 + r];
        __syncthreads();
        if (threadIdx.x == 0) {
          if (v.rank == 0) {
            P.it_out[((size_t)v.unit * nP + q) * L + l] = it;
            P.cv_out[((size_t)v.unit * nP + q) * L + l] = conv ? 1 : 0;
          }
          s_lidx[q] = l + 1;
          s_it[q] = 0;
          if (l + 1 < L) s_lam[q] = lambda_at(q, l + 1);
        }
      } else if (threadIdx.x == 0) {
        s_it[q] = it;
      }
      __syncthreads();
    }
  }
}

// ---------------------------------------------------------------- K4+K5 fused: the cluster solver
// One thread-block cluster per unit Gram (C <= 16 CTAs, one per SM). CTA `rank` owns rows
// [j0, j1) of the unit's normalised Gram; each thread keeps its share of those rows in
// registers (first EREG elements) and shared memory (the rest, thread-major so warp reads are
// conflict free) for the whole launch: the lambda grid (R#14-15) and
// the OEM paths all run from on-chip copies of G.
// Per iteration every CTA pushes its rows of the new beta (and its partial max |dbeta|) into the
// shared memory of every CTA of the cluster (DSMEM stores), then the cluster meets at one
// hardware barrier (barrier.cluster arrive.release / wait.acquire). beta and the partials are
// double-buffered by iteration parity, so no CTA overwrites data another may still read.
struct ClusterArgs {
  int C;          // CTAs per cluster (= per unit)
  int T;          // lanes per row
  int RG;         // row groups per CTA (= threads / T)
  int KPR;        // columns per thread per row = ceil(p / T)
  int NRT;        // rows per thread = ceil(max rows / RG)
  int S;          // shared-memory G slots per thread
  int pv;         // padded vector length (>= p)
  int maxrows;    // max rows per CTA (shared-memory row tables)
};

// (.aligned: every thread of the warp executes it convergently, so the warp is reconverged first;
// a warp arriving while one lane still runs a divergent tail of remote stores could complete the
// barrier before those stores are issued)
__device__ __forceinline__ void cluster_sync_all() {
  __syncwarp();
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}
__device__ __forceinline__ uint32_t cluster_rank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
// store a double into the shared memory of CTA `rank` of this cluster, at the address that
// `local` has in the calling CTA
__device__ __forceinline__ void st_cluster(double* local, uint32_t rank, double v) {
  if (gridDim.x == 0) return;  // (never) keeps the signature uniform for C == 1 callers
  uint32_t a = smem_u32(local), ra;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(ra) : "r"(a), "r"(rank));
  asm volatile("st.shared::cluster.f64 [%0], %1;" ::"r"(ra), "d"(v) : "memory");
}

// ---------------------------------------------------------------- K4+K5 lean: register-resident G
// For p <= 256 and nP <= 4 (cfg1, cfg2 and the logistic inner solves of cfg5). One cluster of
// C <= 4 CTAs per unit Gram; every thread keeps an R x KC tile of G in registers for the whole
// launch (rows rg + i*RG, columns tl + m*T), and the nP penalty vectors are multiplied together
// (the batched matvec: several penalties share A = dI - X^T X). One iteration:
// KC*NPT shared-memory loads, R*KC*NPT FMAs, a width-T reduce-scatter that leaves each
// (row, penalty) sum u_j on a single lane, the thresholding M-step on that lane,
// DSMEM stores of the new coordinate into every CTA of the cluster, a warp OR of the
// "|dbeta_j| > tol" bits and one hardware cluster barrier. The stopping rule (R#17,
// max_j |dbeta_j| <= tol) only needs that OR, so no floating-point max is reduced.
struct LeanArgs {
  int C;            // CTAs per unit (cluster size)
  int qsplit;       // 1: one cluster per (unit, penalty) (kernel instantiated with NPT = 1)
  int rows;         // max rows per CTA (= R * RG)
  int pvl;          // padded vector length (= KC * T >= p)
};

__device__ __forceinline__ void st_cl_f64(double* local, uint32_t rank, double v) {
  uint32_t a = smem_u32(local), ra;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(ra) : "r"(a), "r"(rank));
  asm volatile("st.shared::cluster.f64 [%0], %1;" ::"r"(ra), "d"(v) : "memory");
}
__device__ __forceinline__ void red_or_cl(uint32_t* local, uint32_t rank, uint32_t v) {
  uint32_t a = smem_u32(local), ra;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(ra) : "r"(a), "r"(rank));
  asm volatile("red.shared::cluster.or.b32 [%0], %1;" ::"r"(ra), "r"(v) : "memory");
}

// Reduce-scatter of V partial sums (padded to VP, a power of two dividing T) over the T lanes of a
// row group: recursive halving, then a butterfly; lane tl ends with the full sum of value index
// lean_vidx<VP,T>(tl). Fixed order of additions (deterministic).
template <int VP, int T>
__device__ __forceinline__ double lean_rs(double (&a)[VP], int tl) {
#pragma unroll
  for (int cnt = VP; cnt > 1; cnt >>= 1) {
    const int o = T * cnt / (2 * VP), half = cnt / 2;
    const bool up = (tl & o) != 0;
#pragma unroll
    for (int i = 0; i < half; ++i) {
      const double send = up ? a[i] : a[i + half];
      const double keep = up ? a[i + half] : a[i];
      a[i] = keep + __shfl_xor_sync(0xffffffffu, send, o);
    }
  }
#pragma unroll
  for (int o = T / (2 * VP); o >= 1; o >>= 1) a[0] += __shfl_xor_sync(0xffffffffu, a[0], o);
  return a[0];
}
template <int VP, int T>
__device__ __forceinline__ int lean_vidx(int tl) {
  int v = 0;
#pragma unroll
  for (int cnt = VP; cnt > 1; cnt >>= 1)
    if (tl & (T * cnt / (2 * VP))) v += cnt / 2;
  return v;
}
__host__ __device__ constexpr int pow2ceil(int v) { return v <= 1 ? 1 : 2 * pow2ceil((v + 1) / 2); }
// General form (VP may exceed T): halving over the offsets T/2 .. 1 while more than one value is
// left, then a butterfly if VP < T. Lane tl ends with CNT = max(1, VP/T) full sums in a[0..CNT),
// for the value indices lean_base<VP,T>(tl) + s.
template <int VP, int T>
__device__ __forceinline__ void lean_rs_gen(double (&a)[VP], int tl) {
#pragma unroll
  for (int k = 0; (T >> (k + 1)) >= 1; ++k) {
    const int o = T >> (k + 1), cnt = VP >> k;
    if (cnt > 1) {
      const int half = cnt / 2;
      const bool up = (tl & o) != 0;
#pragma unroll
      for (int i = 0; i < half; ++i) {
        const double send = up ? a[i] : a[i + half];
        const double keep = up ? a[i + half] : a[i];
        a[i] = keep + __shfl_xor_sync(0xffffffffu, send, o);
      }
    } else {
      a[0] += __shfl_xor_sync(0xffffffffu, a[0], o);
    }
  }
}
template <int VP, int T>
__device__ __forceinline__ int lean_base(int tl) {
  int v = 0;
#pragma unroll
  for (int k = 0; (T >> (k + 1)) >= 1; ++k) {
    const int o = T >> (k + 1), cnt = VP >> k;
    if (cnt > 1 && (tl & o)) v += cnt / 2;
  }
  return v;
}

// beta vectors in shared memory: penalties in pairs, [pair][k][2], so one 16-byte load per lane
// fetches two penalties and T consecutive lanes read T*16 contiguous bytes (conflict free)
template <int NPT>
__device__ __forceinline__ int vix(int q, int k, int pvl) {
  return NPT == 1 ? k : (q >> 1) * 2 * pvl + 2 * k + (q & 1);
}

// The matvec of one iteration, a[i*NPT + q] += sum_m G(i, m) b_q(tl + m T): the columns go in
// chunks of four whose shared-memory loads are all issued before their FMAs (one load latency per
// chunk instead of one per column; measured at cfg2, p = 100: the per-column form serialised 13
// load latencies per iteration). Columns m >= kcu are skipped a chunk at a time: entries past p
// are zero in the vector buffers and in the G tile, so the extra FMAs add exact zeros and each
// accumulator sums in the same order as a column-by-column loop.
template <int NPT, int RT, int KC, int T, int NV, int VP, class GEL>
__device__ __forceinline__ void lean_matvec(double (&a)[VP], const double* vc, int pvl, int kcu, int tl, GEL gel) {
  constexpr int MC = KC < 4 ? KC : 4;
  if constexpr (NV <= 2) {
    // one or two penalties per vector entry: software pipelined, the next chunk's loads issued
    // before this chunk's FMAs (the vector buffers hold KC * T entries, so loading a chunk past
    // kcu stays in bounds; it is never used). Same FMAs in the same order.
    constexpr bool SPLIT = VP <= 4;
    double a2[VP];
#pragma unroll
    for (int v = 0; v < VP; ++v) a2[v] = 0.0;
    double bn[MC][NV];
#pragma unroll
    for (int mm = 0; mm < MC; ++mm)
#pragma unroll
      for (int h = 0; h < NV; ++h) bn[mm][h] = vc[NV * (tl + mm * T) + h];   // layout [k][NV] (vix)
#pragma unroll
    for (int m0 = 0; m0 < KC; m0 += MC) {
      if (m0 >= kcu) break;
      double b[MC][NV];
#pragma unroll
      for (int mm = 0; mm < MC; ++mm)
#pragma unroll
        for (int q = 0; q < NV; ++q) b[mm][q] = bn[mm][q];
      if (m0 + MC < KC) {
#pragma unroll
        for (int mm = 0; mm < MC; ++mm) {
          const int k = tl + (m0 + MC + mm) * T;
          if (NV == 1) {
            bn[mm][0] = vc[k];
          } else {
            const double2 t2 = *reinterpret_cast<const double2*>(vc + 2 * k);
            bn[mm][0] = t2.x;
            bn[mm][1] = t2.y;
          }
        }
      }
      // two interleaved chains per sum (even / odd chunks) halve the dependent-FMA depth when a
      // thread has few sums; added at the end (a fixed order: deterministic)
      double* acc = (SPLIT && ((m0 / MC) & 1)) ? a2 : a;
#pragma unroll
      for (int mm = 0; mm < MC; ++mm)
#pragma unroll
        for (int i = 0; i < RT; ++i) {
          const double gv = gel(i, m0 + mm);
#pragma unroll
          for (int q = 0; q < NPT; ++q) acc[i * NPT + q] = fma(gv, b[mm][q], acc[i * NPT + q]);
        }
    }
    if (SPLIT)
#pragma unroll
      for (int v = 0; v < VP; ++v) a[v] += a2[v];
    return;
  }
#pragma unroll
  for (int m0 = 0; m0 < KC; m0 += MC) {
    if (m0 >= kcu) break;
    double b[MC][NV];
#pragma unroll
    for (int mm = 0; mm < MC; ++mm) {
      const int k = tl + (m0 + mm) * T;
      if (NPT == 1) {
        b[mm][0] = vc[k];
      } else {
#pragma unroll
        for (int h = 0; h < NV / 2; ++h) {
          const double2 t2 = *reinterpret_cast<const double2*>(vc + h * 2 * pvl + 2 * k);
          b[mm][2 * h] = t2.x;
          b[mm][2 * h + 1] = t2.y;
        }
      }
    }
#pragma unroll
    for (int mm = 0; mm < MC; ++mm)
#pragma unroll
      for (int i = 0; i < RT; ++i) {
        const double gv = gel(i, m0 + mm);
#pragma unroll
        for (int q = 0; q < NPT; ++q) a[i * NPT + q] = fma(gv, b[mm][q], a[i * NPT + q]);
      }
  }
}
// RS > 0: each thread row group also owns RS rows kept in SHARED memory (for units whose rows do
// not fit the register file, e.g. cfg3's eleven p = 500 Grams in clusters of 8). Thread (rg, tl)
// owns local rows rg*RT + i, i < RT = R + RS: i < R from registers, i >= R from shared memory.
template <int NPT, int R, int KC, int T, int RS = 0, int NTH = PT>
__global__ void __launch_bounds__(NTH, 1) fit_lean_kernel(const PathParams P, const LeanArgs A) {
  constexpr int RT = R + RS;
  constexpr int RG = NTH / T, V = RT * NPT, VP = pow2ceil(V), NW = NTH / 32;
  constexpr int NV = NPT == 1 ? 1 : 2 * ((NPT + 1) / 2);  // doubles per k in the vector layout
  static_assert((T & (T - 1)) == 0 && T <= 32 && (VP <= T || VP % T == 0), "lean layout");
  constexpr int CNT = VP >= T ? VP / T : 1;  // (row, penalty) sums each lane owns after the reduce-scatter
  extern __shared__ __align__(16) double sm[];
  __shared__ int s_fam[NPT], s_skip[NPT];
  __shared__ double s_gam[NPT], s_alp[NPT], s_lmax[NPT];
  __shared__ uint32_t F[3];
  const int p = P.p, nPg = P.nP, L = P.L, C = A.C;
  // penalty split (A.qsplit): cluster i fits penalty i % nPg of unit i / nPg alone (NPT = 1)
  const int clu = blockIdx.x / C;
  const int qoff = A.qsplit ? clu % nPg : 0, nP = A.qsplit ? 1 : nPg;
  constexpr int pvl = KC * T, rows = RT * RG;  // == A.pvl, A.rows (compile-time: immediate offsets)
  const int tid = threadIdx.x, rg = tid / T, tl = tid % T, warp = tid >> 5, lane = tid & 31;
  const uint32_t rank = cluster_rank();
  const int unit = A.qsplit ? clu / nPg : clu;
  const int j0 = P.cta_j0[blockIdx.x], j1 = P.cta_j1[blockIdx.x], nr = j1 - j0;
  const int kcu = (p + T - 1) / T;                       // column slots in use (warp-uniform)
  const bool wrows = (warp * (32 / T)) * RT < nr;        // this warp owns at least one row
  const double* Gu = P.Gn + (size_t)unit * p * p;
  const double* cu = P.cn + (size_t)unit * p;
  // shared memory: vec [2][pvl*NV] | gsm [RS*RG][pvl] | slots [2][C*NW] | uv [NPT][rows] | gw [rows] | ga, gb [rows]
  double* vec = sm;
  constexpr int vstride = pvl * NV;
  double* gsm = vec + (size_t)2 * vstride;
  double* slots = gsm + (size_t)RS * RG * pvl;
  double* uv = slots + (size_t)2 * C * NW;
  double* gw_s = uv + (size_t)NPT * rows;
  int* ga_s = reinterpret_cast<int*>(gw_s + rows);
  int* gb_s = ga_s + rows;
  auto sync_all = [&]() {
    if (C == 1) __syncthreads();
    else cluster_sync_all();
  };
  const bool grp = P.g_of != nullptr;
  const int g0 = (grp && nr > 0) ? P.g_of[j0] : 0;
  const int ng_loc = (grp && nr > 0) ? P.g_of[j1 - 1] + 1 - g0 : 0;
  for (int gg = tid; gg < ng_loc; gg += NTH) {
    gw_s[gg] = P.g_w[g0 + gg];
    ga_s[gg] = P.g_start[g0 + gg] - j0;
    gb_s[gg] = P.g_end[g0 + gg] - j0;
  }
  for (int k = tid; k < 2 * vstride; k += NTH) vec[k] = 0.0;
  for (int k = tid; k < 2 * C * NW; k += NTH) slots[k] = 0.0;
  if (tid < 3) F[tid] = 0u;
  // this thread's tile of G (rows rg*RT + i, columns tl + m*T): i < R in registers for the whole
  // launch, i >= R in shared memory (row rg*RS + i - R of gsm)
  double g[R][KC];
#pragma unroll
  for (int i = 0; i < R; ++i)
#pragma unroll
    for (int m = 0; m < KC; ++m) {
      const int r = rg * RT + i, k = tl + m * T;
      g[i][m] = (r < nr && k < p) ? Gu[(size_t)(j0 + r) * p + k] : 0.0;
    }
#pragma unroll
  for (int i = R; i < RT; ++i)
#pragma unroll
    for (int m = 0; m < KC; ++m) {
      const int r = rg * RT + i, k = tl + m * T;
      gsm[(size_t)(rg * RS + i - R) * pvl + k] = (r < nr && k < p) ? Gu[(size_t)(j0 + r) * p + k] : 0.0;
    }
  // element (i, m) of the thread's tile
  auto gel = [&](int i, int m) -> double {
    return i < R ? g[i < R ? i : 0][m] : gsm[(size_t)(rg * RS + i - R) * pvl + tl + m * T];
  };
  // the (row, penalty) sum this lane owns after the reduce-scatter
  const int vbase = lean_base<VP, T>(tl);
  const bool owner = VP >= T || (tl & (T / VP - 1)) == 0;
  int mq[CNT], mr[CNT], mj[CNT];
  bool act[CNT];
  double c_my[CNT], w_my[CNT];
#pragma unroll
  for (int s2 = 0; s2 < CNT; ++s2) {
    const int vidx = vbase + s2;
    mq[s2] = vidx % NPT;
    mr[s2] = rg * RT + vidx / NPT;
    act[s2] = owner && vidx < V && mr[s2] < nr;
    mj[s2] = j0 + mr[s2];
    c_my[s2] = act[s2] ? cu[mj[s2]] : 0.0;
    w_my[s2] = (act[s2] && P.var_w) ? P.var_w[mj[s2]] : 1.0;
  }
  cluster_sync_all();  // peers' buffers are zeroed before any remote store

  // a7: d (>= lambda_1, R#5) was computed for every unit by d_rule (drule.cu) before this launch
  const double d = P.d[unit];

  // ======================================================= a8: lambda grid (R#14-16, R#22)
  if (warp < NPT) {
    const int q = warp;
    double lm = 0.0;
    int fam = 0;
    double gq = 0.0, aq = 0.0;
    if (q < nP) {
      fam = P.fam[q + qoff]; gq = P.gam[q + qoff]; aq = P.alp[q + qoff];
      const double* cc = P.shared_grid ? P.cn : cu;
      if (P.lmax_override) {
        lm = *P.lmax_override;
      } else if (fam == OEM_SGL) {
        for (int gg = lane; gg < P.ngroups; gg += 32)
          lm = fmax(lm, sgl_lmax_group(cc, P.g_start[gg], P.g_end[gg], P.var_w, P.g_w[gg], aq));
      } else if (fam >= OEM_GRP_LASSO) {
        for (int gg = lane; gg < P.ngroups; gg += 32) {
          const double cg = P.g_w[gg];
          if (!(cg > 0.0)) continue;
          double s = 0.0;
          for (int j = P.g_start[gg]; j < P.g_end[gg]; ++j) s += cc[j] * cc[j];
          lm = fmax(lm, sqrt(s) / cg);
        }
      } else {
        const double scl = fam == OEM_ENET ? aq : 1.0;
        for (int j = lane; j < p; j += 32) {
          const double wj = P.var_w ? P.var_w[j] : 1.0;
          if (!(wj > 0.0)) continue;
          lm = fmax(lm, fabs(cc[j]) / (scl * wj));
        }
      }
#pragma unroll
      for (int o = 16; o >= 1; o >>= 1) lm = fmax(lm, __shfl_xor_sync(0xffffffffu, lm, o));
    }
    if (lane == 0) {
      s_fam[q] = fam; s_gam[q] = gq; s_alp[q] = aq; s_lmax[q] = lm;
      bool bad = false;  // parameter validity against the d in use (R#8)
      if (q < nP) {
        if (fam == OEM_MCP || fam == OEM_GRP_MCP) bad = !(gq > 1.0) || !(gq * d > 1.0);
        if (fam == OEM_SCAD || fam == OEM_GRP_SCAD) bad = !(gq > 2.0) || !((gq - 1.0) * d > 1.0);
        if (fam == OEM_ENET) bad = !(aq >= 0.0 && aq <= 1.0);
        if (bad && rank == 0) atomicExch(&P.flags[1], 1);
      }
      s_skip[q] = (q >= nP || bad) ? 1 : 0;
    }
  }
  // warm or cold start (permuted order) into buffer 0
  if (P.beta_init)
    for (int e = tid; e < nP * p; e += NTH) {
      const int q = e / p, k = e % p;
      vec[vix<NPT>(q, k, pvl)] = P.beta_init[((size_t)unit * nPg + q + qoff) * p + P.perm[k]];
    }
  __syncthreads();
  auto lam_at = [&](int q, int l) -> double {
    if (P.lam_explicit) return P.lam_explicit[l];
    if (L == 1) return s_lmax[q];
    return s_lmax[q] * exp(((double)l / (double)(L - 1)) * log(P.lmin_ratio));  // R#15
  };
  if (rank == 0)
    for (int e = tid; e < nP * L; e += NTH) {
      const int q = e / L, l = e % L;
      P.lam_out[((size_t)unit * nPg + q + qoff) * L + l] = lam_at(q, l);
    }
  int lidx[NPT], itc[NPT];
  double lam[NPT];
#pragma unroll
  for (int q = 0; q < NPT; ++q) {
    lidx[q] = s_skip[q] ? L : 0;
    itc[q] = 0;
    lam[q] = s_skip[q] ? 0.0 : lam_at(q, 0);
  }
  // the group M-step runs only if one of this cluster's penalties is a group family
  bool grpm = false;
  for (int q = 0; q < nP; ++q) grpm = grpm || (grp && s_fam[q] >= OEM_GRP_LASSO);
  int fam_my[CNT];
  double gam_my[CNT], alp_my[CNT], rg_my[CNT];
  const double rd = 1.0 / d;
#pragma unroll
  for (int s2 = 0; s2 < CNT; ++s2) {
    fam_my[s2] = s_fam[mq[s2]];
    gam_my[s2] = s_gam[mq[s2]];
    alp_my[s2] = s_alp[mq[s2]];
    rg_my[s2] = fam_my[s2] == OEM_MCP ? 1.0 / (gam_my[s2] * d - 1.0)
              : fam_my[s2] == OEM_SCAD ? 1.0 / ((gam_my[s2] - 1.0) * d - 1.0) : 0.0;
  }
  cluster_sync_all();  // every CTA's buffers are initialised before the first remote store

  // ======================================================= a9: OEM iterations
  uint32_t nan_seen = 0;
  for (int t = 0;; ++t) {
    uint32_t qmask = 0;
#pragma unroll
    for (int q = 0; q < NPT; ++q)
      if (lidx[q] < L) qmask |= 1u << q;
    if (!qmask) break;
    const int cur = t & 1, nxt = cur ^ 1;
    const double* vc = vec + (size_t)cur * vstride;
    double* vn = vec + (size_t)nxt * vstride;
    if (tid == 0) F[(t + 1) % 3] = 0u;
    // ---- E-step + M-step: u = c + d beta - G beta, all penalties at once
    double a[VP];
#pragma unroll
    for (int v = 0; v < VP; ++v) a[v] = 0.0;
    if (wrows) lean_matvec<NPT, RT, KC, T, NV>(a, vc, pvl, kcu, tl, gel);
    lean_rs_gen<VP, T>(a, tl);
    uint32_t bits = 0;
#pragma unroll
    for (int s2 = 0; s2 < CNT; ++s2) {
      if (!(act[s2] && ((qmask >> mq[s2]) & 1u))) continue;
      const int vi = vix<NPT>(mq[s2], mj[s2], pvl);
      const double bj = vc[vi];
      const double u = c_my[s2] + d * bj - a[s2];
      if (!isfinite(u)) bits |= 0x80000000u;
      if (!grp || fam_my[s2] < OEM_GRP_LASSO) {  // coordinate-wise family (also when mixed with group ones)
        double lq = 0.0;
#pragma unroll
        for (int q = 0; q < NPT; ++q)
          if (q == mq[s2]) lq = lam[q];
        const double nb = th_coord_r(fam_my[s2], u, w_my[s2] * lq, gam_my[s2], alp_my[s2], d, rd, rg_my[s2]);
        if (!(fabs(nb - bj) <= P.tol)) bits |= 1u << mq[s2];
        if (C == 1) vn[vi] = nb;
        else for (int rr = 0; rr < C; ++rr) st_cl_f64(&vn[vi], rr, nb);
      } else {
        uv[mq[s2] * rows + mr[s2]] = u;
      }
    }
    if (grpm) {
      // group M-step (eqs glasso / gmcp / gscad); groups lie inside [j0, j1)
      __syncthreads();
      for (int e = warp; e < ng_loc * nP; e += NW) {   // one warp per (group, penalty)
        const int q = e % nP, gl = e / nP;
        if (!((qmask >> q) & 1u) || s_fam[q] < OEM_GRP_LASSO) continue;
        double lq = 0.0;
#pragma unroll
        for (int qq = 0; qq < NPT; ++qq)
          if (qq == q) lq = lam[qq];
        group_mstep_warp(uv + q * rows, ga_s[gl], gb_s[gl], s_fam[q], lq, s_gam[q], s_alp[q], gw_s[gl], d, P.var_w, j0,
                         lane, [&](int r, double nb) {
                           const int vi = vix<NPT>(q, j0 + r, pvl);
                           if (!(fabs(nb - vc[vi]) <= P.tol)) bits |= 1u << q;
                           if (C == 1) vn[vi] = nb;
                           else for (int rr = 0; rr < C; ++rr) st_cl_f64(&vn[vi], rr, nb);
                         });
      }
    }
    uint32_t f;
    if (NPT == 1 && C == 1) {
      // one CTA, one penalty: the barrier itself ORs the "not converged" predicate (bar.red.or),
      // no shared flag word on the iteration's critical path. A non-finite u also leaves its
      // coordinate "not converged"; that is reduced every 64 iterations (sticky per thread)
      nan_seen |= bits >> 31;
      f = __syncthreads_or((int)(bits & 1u)) ? 1u : 0u;
      if ((t & 63) == 63 && __syncthreads_or((int)nan_seen)) f |= 0x80000000u;
    } else {
      bits = __reduce_or_sync(0xffffffffu, bits);
      if (lane == 0 && bits) {
        if (C == 1) atomicOr(&F[t % 3], bits);
        else for (int rr = 0; rr < C; ++rr) red_or_cl(&F[t % 3], rr, bits);
      }
      sync_all();
      f = F[t % 3];
    }
    if (f & 0x80000000u) {
      if (tid == 0) atomicExch(&P.flags[0], 1);
      break;
    }
    // ---- identical bookkeeping in every thread of every CTA of the cluster
#pragma unroll
    for (int q = 0; q < NPT; ++q) {
      if (!((qmask >> q) & 1u)) continue;
      const int it = itc[q] + 1;
      const bool conv = !((f >> q) & 1u);   // every |dbeta_j| <= tol (R#17)
      if (conv || it >= P.maxit) {
        const int l = lidx[q];
        double* out = P.beta_out + (((size_t)unit * nPg + q + qoff) * L + l) * p;
        for (int r = tid; r < nr; r += NTH) out[P.perm[j0 + r]] = vn[vix<NPT>(q, j0 + r, pvl)];
        if (rank == 0 && tid == 0) {
          P.it_out[((size_t)unit * nPg + q + qoff) * L + l] = it;
          P.cv_out[((size_t)unit * nPg + q + qoff) * L + l] = conv ? 1 : 0;
        }
        lidx[q] = l + 1;
        itc[q] = 0;
        if (l + 1 < L) lam[q] = lam_at(q, l + 1);
      } else {
        itc[q] = it;
      }
    }
  }
  // the periodic non-finite check of the one-CTA form, once more for the last iterations
  if (NPT == 1 && C == 1 && __syncthreads_or((int)nan_seen) && tid == 0) atomicExch(&P.flags[0], 1);
}

// ---------------------------------------------------------------- K4+K5 lean, grid-wide variant
// For units too large for one cluster (p up to 1024, e.g. cfg4's p = 1000 split over ~63-100
// CTAs): the same register-resident G tiles, batched penalties, reduce-scatter and OR-reduced
// stopping rule as fit_lean_kernel, but the C CTAs of a unit exchange through L2 instead of
// DSMEM: each CTA writes its new coordinates to a global double buffer and its "not converged"
// bits to a per-CTA slot, meets the unit's other CTAs at a counter barrier (release add /
// acquire poll, one per iteration), then copies the whole new vector back into shared memory
// (ld.global.cg: L2, never a stale L1 line). Cooperative launch: every CTA is co-resident.
struct GlobArgs {
  int Cmax;             // max CTAs per unit (slot stride)
  int qsplit;           // 1: one virtual unit per (unit, penalty), kernel instantiated with NPT = 1
  int nvu;              // virtual units (nU, or nU * nP with qsplit)
  int rows, pvl;
  double* gvec;         // [2][nU][NV * pvl]
  unsigned long long* gflag;  // [2][nU][Cmax] (iteration tag << 32) | not-converged bits (zero at launch)
  double* gslot;        // [2][nU][Cmax]
  unsigned* gcnt;       // [nU] barrier counters (zero at launch)
};

__device__ __forceinline__ void red_release_add(unsigned* p, unsigned v) {
  asm volatile("red.release.gpu.global.add.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ unsigned ld_relaxed(const unsigned* p) {
  unsigned v;
  asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void fence_acquire_gpu() { asm volatile("fence.acq_rel.gpu;" ::: "memory"); }
__device__ __forceinline__ void st_release_u64(unsigned long long* p, unsigned long long v) {
  asm volatile("st.release.gpu.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ unsigned long long ld_relaxed_u64(const unsigned long long* p) {
  unsigned long long v;
  asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}

template <int NPT, int R, int KC, int T, int RS = 0, int NTH = PT>
__global__ void __launch_bounds__(NTH, 1) fit_glob_kernel(const PathParams P, const GlobArgs A) {
  constexpr int RT = R + RS;  // rows per thread row group: R in registers, RS in shared memory
  constexpr int RG = NTH / T, V = RT * NPT, VP = pow2ceil(V), NW = NTH / 32;
  constexpr int NV = NPT == 1 ? 1 : 2 * ((NPT + 1) / 2);
  static_assert(VP <= T && (T & (T - 1)) == 0 && T <= 32, "lean layout");
  extern __shared__ __align__(16) double sm[];
  __shared__ int s_fam[NPT], s_skip[NPT];
  __shared__ double s_gam[NPT], s_alp[NPT], s_lmax[NPT];
  __shared__ uint32_t s_bits, s_all;
  __shared__ double s_red[NW], s_tot;
  const int p = P.p, nPg = P.nP, L = P.L;
  constexpr int pvl = KC * T, rows = RT * RG;  // == A.pvl, A.rows
  const int tid = threadIdx.x, rg = tid / T, tl = tid % T, warp = tid >> 5, lane = tid & 31;
  // virtual unit: a unit Gram, or with A.qsplit one (unit, penalty) pair fitted alone (NPT = 1)
  const int vu = P.cta_unit[blockIdx.x], rank = P.cta_rank[blockIdx.x], C = P.unit_ncta[vu];
  const int unit = A.qsplit ? vu / nPg : vu, qoff = A.qsplit ? vu % nPg : 0, nP = A.qsplit ? 1 : nPg;
  const int j0 = P.cta_j0[blockIdx.x], j1 = P.cta_j1[blockIdx.x], nr = j1 - j0;
  const int kcu = (p + T - 1) / T;
  const bool wrows = (warp * (32 / T)) * RT < nr;
  const double* Gu = P.Gn + (size_t)unit * p * p;
  const double* cu = P.cn + (size_t)unit * p;
  constexpr int vstride = pvl * NV;
  double* vec = sm;                                   // [2][vstride] (local copies)
  double* gsm = vec + (size_t)2 * vstride;            // [RS*RG][pvl] shared-memory rows of G
  double* uv = gsm + (size_t)RS * RG * pvl;           // [NPT][rows]
  double* gw_s = uv + (size_t)NPT * rows;
  int* ga_s = reinterpret_cast<int*>(gw_s + rows);
  int* gb_s = ga_s + rows;
  double* gvec = A.gvec + (size_t)vu * vstride;       // + par * nvu * vstride
  const size_t gpar = (size_t)A.nvu * vstride;
  unsigned long long* gflag = A.gflag + (size_t)vu * A.Cmax;  // + par * nvu * Cmax
  double* gslot = A.gslot + (size_t)vu * A.Cmax;
  const size_t spar = (size_t)A.nvu * A.Cmax;
  unsigned epoch = 0;
  // unit barrier: every CTA of the unit has published its writes (grid.sync pattern, per unit)
  // (bar.sync orders the CTA's writes before thread 0's release, which is cumulative; relaxed
  // polling, then one acquire fence: no L1 invalidation per poll)
  auto unit_sync = [&]() {
    __syncthreads();
    if (tid == 0) {
      red_release_add(&A.gcnt[vu], 1u);
      const unsigned target = (epoch + 1) * (unsigned)C;
      while ((int)(ld_relaxed(&A.gcnt[vu]) - target) < 0) {}  // wrap-safe
      fence_acquire_gpu();
    }
    ++epoch;
    __syncthreads();
  };
  const bool grp = P.g_of != nullptr;
  const int g0 = (grp && nr > 0) ? P.g_of[j0] : 0;
  const int ng_loc = (grp && nr > 0) ? P.g_of[j1 - 1] + 1 - g0 : 0;
  for (int gg = tid; gg < ng_loc; gg += NTH) {
    gw_s[gg] = P.g_w[g0 + gg];
    ga_s[gg] = P.g_start[g0 + gg] - j0;
    gb_s[gg] = P.g_end[g0 + gg] - j0;
  }
  for (int k = tid; k < 2 * vstride; k += NTH) vec[k] = 0.0;
  double g[R][KC];
#pragma unroll
  for (int i = 0; i < R; ++i)
#pragma unroll
    for (int m = 0; m < KC; ++m) {
      const int r = rg * RT + i, k = tl + m * T;
      g[i][m] = (r < nr && k < p) ? Gu[(size_t)(j0 + r) * p + k] : 0.0;
    }
#pragma unroll
  for (int i = R; i < RT; ++i)
#pragma unroll
    for (int m = 0; m < KC; ++m) {
      const int r = rg * RT + i, k = tl + m * T;
      gsm[(size_t)(rg * RS + i - R) * pvl + k] = (r < nr && k < p) ? Gu[(size_t)(j0 + r) * p + k] : 0.0;
    }
  auto gel = [&](int i, int m) -> double {
    return i < R ? g[i < R ? i : 0][m] : gsm[(size_t)(rg * RS + i - R) * pvl + tl + m * T];
  };
  const int vidx = lean_vidx<VP, T>(tl);
  const int mi = vidx / NPT, mq = vidx % NPT, mr = rg * RT + mi;
  const bool owner = (tl & (T / VP - 1)) == 0;
  const bool act = owner && vidx < V && mr < nr;
  const int mj = j0 + mr;
  const double c_my = act ? cu[mj] : 0.0;
  const double w_my = (act && P.var_w) ? P.var_w[mj] : 1.0;
  // CTA sum of one double per thread, in warp order; result in s_tot after the call
  auto cta_sum = [&](double x) {
#pragma unroll
    for (int o = 16; o >= 1; o >>= 1) x += __shfl_xor_sync(0xffffffffu, x, o);
    if (lane == 0) s_red[warp] = x;
    __syncthreads();
    if (tid == 0) {
      double t = 0.0;
      for (int w = 0; w < NW; ++w) t += s_red[w];
      s_tot = t;
    }
    __syncthreads();
    return s_tot;
  };
  // sum (or max) over the unit's CTAs of a per-CTA value, through the slots; fixed CTA order
  auto unit_reduce = [&](double mine, int par, bool is_max) -> double {
    if (tid == 0) gslot[par * spar + rank] = mine;
    unit_sync();
    if (warp == 0) {  // lane-strided loads, then a fixed butterfly: same order on every CTA
      double r = 0.0;
      for (int c = lane; c < C; c += 32) {
        const double v = __ldcg(&gslot[par * spar + c]);
        r = is_max ? fmax(r, v) : r + v;
      }
#pragma unroll
      for (int o = 16; o >= 1; o >>= 1) {
        const double v = __shfl_xor_sync(0xffffffffu, r, o);
        r = is_max ? fmax(r, v) : r + v;
      }
      if (lane == 0) s_tot = r;
    }
    __syncthreads();
    const double r = s_tot;
    __syncthreads();
    return r;
  };

  // a7: d (>= lambda_1, R#5) from d_rule (drule.cu)
  const double d = P.d[unit];
  int par = 0;

  // ======================================================= a8: lambda grid (R#14-16, R#22)
  if (warp < NPT) {
    const int q = warp;
    double lm = 0.0;
    int fam = 0;
    double gq = 0.0, aq = 0.0;
    if (q < nP) {
      fam = P.fam[q + qoff]; gq = P.gam[q + qoff]; aq = P.alp[q + qoff];
      const double* cc = P.shared_grid ? P.cn : cu;
      if (P.lmax_override) {
        lm = *P.lmax_override;
      } else if (fam == OEM_SGL) {
        for (int gg = lane; gg < P.ngroups; gg += 32)
          lm = fmax(lm, sgl_lmax_group(cc, P.g_start[gg], P.g_end[gg], P.var_w, P.g_w[gg], aq));
      } else if (fam >= OEM_GRP_LASSO) {
        for (int gg = lane; gg < P.ngroups; gg += 32) {
          const double cg = P.g_w[gg];
          if (!(cg > 0.0)) continue;
          double s = 0.0;
          for (int j = P.g_start[gg]; j < P.g_end[gg]; ++j) s += cc[j] * cc[j];
          lm = fmax(lm, sqrt(s) / cg);
        }
      } else {
        const double scl = fam == OEM_ENET ? aq : 1.0;
        for (int j = lane; j < p; j += 32) {
          const double wj = P.var_w ? P.var_w[j] : 1.0;
          if (!(wj > 0.0)) continue;
          lm = fmax(lm, fabs(cc[j]) / (scl * wj));
        }
      }
#pragma unroll
      for (int o = 16; o >= 1; o >>= 1) lm = fmax(lm, __shfl_xor_sync(0xffffffffu, lm, o));
    }
    if (lane == 0) {
      s_fam[q] = fam; s_gam[q] = gq; s_alp[q] = aq; s_lmax[q] = lm;
      bool bad = false;
      if (q < nP) {
        if (fam == OEM_MCP || fam == OEM_GRP_MCP) bad = !(gq > 1.0) || !(gq * d > 1.0);
        if (fam == OEM_SCAD || fam == OEM_GRP_SCAD) bad = !(gq > 2.0) || !((gq - 1.0) * d > 1.0);
        if (fam == OEM_ENET) bad = !(aq >= 0.0 && aq <= 1.0);
        if (bad && rank == 0) atomicExch(&P.flags[1], 1);
      }
      s_skip[q] = (q >= nP || bad) ? 1 : 0;
    }
  }
  if (P.beta_init)
    for (int e = tid; e < nP * p; e += NTH) {
      const int q = e / p, k = e % p;
      vec[vix<NPT>(q, k, pvl)] = P.beta_init[((size_t)unit * nPg + q + qoff) * p + P.perm[k]];
    }
  if (tid == 0) s_bits = 0u;
  __syncthreads();
  auto lam_at = [&](int q, int l) -> double {
    if (P.lam_explicit) return P.lam_explicit[l];
    if (L == 1) return s_lmax[q];
    return s_lmax[q] * exp(((double)l / (double)(L - 1)) * log(P.lmin_ratio));  // R#15
  };
  if (rank == 0)
    for (int e = tid; e < nP * L; e += NTH) {
      const int q = e / L, l = e % L;
      P.lam_out[((size_t)unit * nPg + q + qoff) * L + l] = lam_at(q, l);
    }
  int lidx[NPT], itc[NPT];
  double lam[NPT];
#pragma unroll
  for (int q = 0; q < NPT; ++q) {
    lidx[q] = s_skip[q] ? L : 0;
    itc[q] = 0;
    lam[q] = s_skip[q] ? 0.0 : lam_at(q, 0);
  }
  bool grpm = false;  // the group M-step runs only if one of this unit's penalties is a group family
  for (int q = 0; q < nP; ++q) grpm = grpm || (grp && s_fam[q] >= OEM_GRP_LASSO);
  const int fam_my = s_fam[mq];
  const double gam_my = s_gam[mq], alp_my = s_alp[mq];

  // ======================================================= a9: OEM iterations
  for (int t = 0;; ++t) {
    uint32_t qmask = 0;
#pragma unroll
    for (int q = 0; q < NPT; ++q)
      if (lidx[q] < L) qmask |= 1u << q;
    if (!qmask) break;
    const int cur = t & 1, nxt = cur ^ 1;
    const double* vc = vec + (size_t)cur * vstride;
    double* vn = vec + (size_t)nxt * vstride;
    double* gn = gvec + nxt * gpar;
    double a[VP];
#pragma unroll
    for (int v = 0; v < VP; ++v) a[v] = 0.0;
    if (wrows) lean_matvec<NPT, RT, KC, T, NV>(a, vc, pvl, kcu, tl, gel);
    const double s = lean_rs<VP, T>(a, tl);
    uint32_t bits = 0;
    if (act && ((qmask >> mq) & 1u)) {
      const int vi = vix<NPT>(mq, mj, pvl);
      const double bj = vc[vi];
      const double u = c_my + d * bj - s;
      if (!isfinite(u)) bits |= 0x80000000u;
      if (!grp || fam_my < OEM_GRP_LASSO) {  // coordinate-wise family (also when mixed with group ones)
        double lq = 0.0;
#pragma unroll
        for (int q = 0; q < NPT; ++q)
          if (q == mq) lq = lam[q];
        const double nb = th_coord(fam_my, u, w_my * lq, gam_my, alp_my, d);
        if (!(fabs(nb - bj) <= P.tol)) bits |= 1u << mq;
        gn[vi] = nb;
      } else {
        uv[mq * rows + mr] = u;
      }
    }
    if (grpm) {
      __syncthreads();
      for (int e = warp; e < ng_loc * nP; e += NW) {   // one warp per (group, penalty)
        const int q = e % nP, gl = e / nP;
        if (!((qmask >> q) & 1u) || s_fam[q] < OEM_GRP_LASSO) continue;
        double lq = 0.0;
#pragma unroll
        for (int qq = 0; qq < NPT; ++qq)
          if (qq == q) lq = lam[qq];
        group_mstep_warp(uv + q * rows, ga_s[gl], gb_s[gl], s_fam[q], lq, s_gam[q], s_alp[q], gw_s[gl], d, P.var_w, j0,
                         lane, [&](int r, double nb) {
                           const int vi = vix<NPT>(q, j0 + r, pvl);
                           if (!(fabs(nb - vc[vi]) <= P.tol)) bits |= 1u << q;
                           gn[vi] = nb;
                         });
      }
    }
    bits = __reduce_or_sync(0xffffffffu, bits);
    if (lane == 0 && bits) atomicOr(&s_bits, bits);
    __syncthreads();
    if (tid == 0) {
      gflag[(t & 1) * spar + rank] = s_bits;
      s_bits = 0u;
    }
    unit_sync();
    // the unit's new vector and flags, from L2: every load issued before any is used (one L2
    // round trip); 16-byte loads of penalty pairs (p <= 1024)
    constexpr int NLD = (1024 + NTH - 1) / NTH;  // loads per thread covering p <= 1024
    if (NPT == 1) {
      double tv[NLD];
#pragma unroll
      for (int u = 0; u < NLD; ++u) {
        const int k = tid + u * NTH;
        tv[u] = k < p ? __ldcg(&gn[k]) : 0.0;
      }
#pragma unroll
      for (int u = 0; u < NLD; ++u)
        if (tid + u * NTH < p) vn[tid + u * NTH] = tv[u];
    } else {
      double2 tv[NV / 2 > 0 ? NV / 2 : 1][NLD];
#pragma unroll
      for (int h = 0; h < NV / 2; ++h)
#pragma unroll
        for (int u = 0; u < NLD; ++u) {
          const int k = tid + u * NTH;
          tv[h][u] = k < p ? __ldcg(reinterpret_cast<const double2*>(gn + h * 2 * pvl) + k) : make_double2(0.0, 0.0);
        }
#pragma unroll
      for (int h = 0; h < NV / 2; ++h)
#pragma unroll
        for (int u = 0; u < NLD; ++u)
          if (tid + u * NTH < p) reinterpret_cast<double2*>(vn + h * 2 * pvl)[tid + u * NTH] = tv[h][u];
    }
    if (warp == 0) {
      uint32_t w = 0;
#pragma unroll 5
      for (int c = lane; c < C; c += 32) w |= (uint32_t)__ldcg(&gflag[(t & 1) * spar + c]);
      w = __reduce_or_sync(0xffffffffu, w);
      if (lane == 0) s_all = w;
    }
    __syncthreads();    const uint32_t f = s_all;
    if (f & 0x80000000u) {
      if (tid == 0) atomicExch(&P.flags[0], 1);
      break;
    }
#pragma unroll
    for (int q = 0; q < NPT; ++q) {
      if (!((qmask >> q) & 1u)) continue;
      const int it = itc[q] + 1;
      const bool conv = !((f >> q) & 1u);
      if (conv || it >= P.maxit) {
        const int l = lidx[q];
        double* out = P.beta_out + (((size_t)unit * nPg + q + qoff) * L + l) * p;
        for (int r = tid; r < nr; r += NTH) out[P.perm[j0 + r]] = vn[vix<NPT>(q, j0 + r, pvl)];
        if (rank == 0 && tid == 0) {
          P.it_out[((size_t)unit * nPg + q + qoff) * L + l] = it;
          P.cv_out[((size_t)unit * nPg + q + qoff) * L + l] = conv ? 1 : 0;
        }
        lidx[q] = l + 1;
        itc[q] = 0;
        if (l + 1 < L) lam[q] = lam_at(q, l + 1);
      } else {
        itc[q] = it;
      }
    }
  }
}

template <int NPT, int EREG>
__global__ void __launch_bounds__(PT, 1) fit_cluster_kernel(const PathParams P, const ClusterArgs A) {
  extern __shared__ __align__(16) double sm[];
  const int p = P.p, nP = P.nP, L = P.L, C = A.C, T = A.T, RG = A.RG, KPR = A.KPR, NRT = A.NRT;
  const int tid = threadIdx.x, rg = tid / T, tl = tid % T;
  const int rank = (int)cluster_rank();
  const int unit = blockIdx.x / C;
  const int cta = blockIdx.x;
  const int j0 = P.cta_j0[cta], j1 = P.cta_j1[cta], nr = j1 - j0;
  const double* Gu = P.Gn + (size_t)unit * p * p;
  const double* c = P.cn + (size_t)unit * p;
  // shared memory: G slots [S][PT] | vec [2][NPT][pv] | dl [2][C][NPT+2] | red [32][NPT+1] | uv [NPT][nr]
  double* gsm = sm;
  double* vec = gsm + (size_t)A.S * PT;
  double* dl = vec + (size_t)2 * NPT * A.pv;
  double* red = dl + (size_t)2 * C * (NPT + 2);
  double* uv = red + 32 * (NPT + 1);
  // per-row / per-group constants staged once: global loads after a cluster barrier miss L1
  double* c_s = uv + (size_t)NPT * A.maxrows;       // c_j, own rows
  double* w_s = c_s + A.maxrows;                     // var_w_j, own rows
  double* gw_s = w_s + A.maxrows;                    // group weights, local groups
  int* ga_s = reinterpret_cast<int*>(gw_s + A.maxrows);  // group start - j0
  int* gb_s = ga_s + A.maxrows;                          // group end - j0
  for (int r = tid; r < nr; r += PT) {
    c_s[r] = c[j0 + r];
    w_s[r] = P.var_w ? P.var_w[j0 + r] : 1.0;
  }
  // both vector buffers start at zero (padding beyond p is read by the row dots and must stay 0);
  // the cluster barrier orders the zeroing before any remote (DSMEM) write of a peer CTA
  for (int k = tid; k < 2 * NPT * A.pv; k += PT) vec[k] = 0.0;
  cluster_sync_all();
  const int g0 = (P.g_of && nr > 0) ? P.g_of[j0] : 0;
  const int ng_loc = (P.g_of && nr > 0) ? P.g_of[j1 - 1] + 1 - g0 : 0;
  for (int g = tid; g < ng_loc; g += PT) {
    gw_s[g] = P.g_w[g0 + g];
    ga_s[g] = P.g_start[g0 + g] - j0;
    gb_s[g] = P.g_end[g0 + g] - j0;
  }
  int famq[NPT];
  double gamq[NPT], alpq[NPT];
#pragma unroll
  for (int q = 0; q < NPT; ++q) {
    famq[q] = q < nP ? P.fam[q] : 0;
    gamq[q] = q < nP ? P.gam[q] : 0.0;
    alpq[q] = q < nP ? P.alp[q] : 0.0;
  }
  // ---- this thread's share of G: rows r = rg + ri*RG, columns k = tl + ci*T
  double greg[EREG];
#pragma unroll
  for (int e = 0; e < EREG; ++e) {
    const int r = rg, k = tl + e * T;
    greg[e] = (e < KPR && r < nr && k < p) ? Gu[(size_t)(j0 + r) * p + k] : 0.0;
  }
  for (int ri = 0; ri < NRT; ++ri)
    for (int ci = (ri == 0 ? EREG : 0); ci < KPR; ++ci) {
      const int slot = (ri == 0) ? ci - EREG : (KPR > EREG ? KPR - EREG : 0) + (ri - 1) * KPR + ci;
      const int r = rg + ri * RG, k = tl + ci * T;
      gsm[(size_t)slot * PT + tid] = (r < nr && k < p) ? Gu[(size_t)(j0 + r) * p + k] : 0.0;
    }
  // row-dot of this thread's elements against vector v (one penalty): partial sum
  auto rowdot = [&](int ri, const double* v) -> double {
    double a = 0.0;
    if (ri == 0) {
#pragma unroll
      for (int e = 0; e < EREG; ++e)
        if (e < KPR) a = fma(greg[e], v[tl + e * T], a);
      for (int ci = EREG; ci < KPR; ++ci) a = fma(gsm[(size_t)(ci - EREG) * PT + tid], v[tl + ci * T], a);
    } else {
      const int base = (KPR > EREG ? KPR - EREG : 0) + (ri - 1) * KPR;
      for (int ci = 0; ci < KPR; ++ci) a = fma(gsm[(size_t)(base + ci) * PT + tid], v[tl + ci * T], a);
    }
    return a;
  };
  auto reduce_T = [&](double a) -> double {
    for (int o = T >> 1; o > 0; o >>= 1) a += __shfl_xor_sync(0xffffffffu, a, o, T);
    return a;
  };
  const int warp = tid >> 5, lane = tid & 31, nwarps = PT / 32;

  // a7: d (>= lambda_1, R#5) from d_rule (drule.cu)
  const double d = P.d[unit];

  // ======================================================= a8: lambda grid (R#14-16, R#22)
  double lmax[NPT], lam[NPT];
  int lidx[NPT];
  int itc[NPT];
#pragma unroll
  for (int q = 0; q < NPT; ++q) {
    lmax[q] = 0.0;
    lidx[q] = L;
    itc[q] = 0;
    lam[q] = 0.0;
    if (q >= nP) continue;
    const int fam = P.fam[q];
    const double* cc = P.shared_grid ? P.cn : c;
    double lm = 0.0;
    if (P.lmax_override) {
      lm = *P.lmax_override;
    } else if (fam == OEM_SGL) {
      for (int g = 0; g < P.ngroups; ++g)
        lm = fmax(lm, sgl_lmax_group(cc, P.g_start[g], P.g_end[g], P.var_w, P.g_w[g], P.alp[q]));
    } else if (fam >= OEM_GRP_LASSO) {
      for (int g = 0; g < P.ngroups; ++g) {
        const double cg = P.g_w[g];
        if (!(cg > 0.0)) continue;
        double s = 0.0;
        for (int j = P.g_start[g]; j < P.g_end[g]; ++j) s += cc[j] * cc[j];
        lm = fmax(lm, sqrt(s) / cg);
      }
    } else {
      const double sc = fam == OEM_ENET ? P.alp[q] : 1.0;
      for (int j = 0; j < p; ++j) {
        const double wj = P.var_w ? P.var_w[j] : 1.0;
        if (!(wj > 0.0)) continue;
        lm = fmax(lm, fabs(cc[j]) / (sc * wj));
      }
    }
    lmax[q] = lm;
    // parameter validity against the d in use (R#8)
    const double g = P.gam[q];
    bool bad = false;
    if (fam == OEM_MCP || fam == OEM_GRP_MCP) bad = !(g > 1.0) || !(g * d > 1.0);
    if (fam == OEM_SCAD || fam == OEM_GRP_SCAD) bad = !(g > 2.0) || !((g - 1.0) * d > 1.0);
    if (fam == OEM_ENET) bad = !(P.alp[q] >= 0.0 && P.alp[q] <= 1.0);
    if (bad) {
      if (tid == 0) atomicExch(&P.flags[1], 1);
      continue;
    }
    lidx[q] = 0;
    lam[q] = P.lam_explicit ? P.lam_explicit[0] : lm;
    if (rank == 0)
      for (int l = tid; l < L; l += PT)
        P.lam_out[((size_t)unit * nP + q) * L + l] =
            P.lam_explicit ? P.lam_explicit[l]
                           : (L == 1 ? lm : lm * exp(((double)l / (double)(L - 1)) * log(P.lmin_ratio)));
  }
  // warm or cold start (permuted order), both parity buffers hold beta^(0) in slot 0
  for (int q = 0; q < NPT; ++q)
    for (int k = tid; k < A.pv; k += PT)
      vec[(size_t)q * A.pv + k] =
          (q < nP && k < p && P.beta_init) ? P.beta_init[((size_t)unit * nP + q) * p + P.perm[k]] : 0.0;
  __syncthreads();
  const bool grp = P.g_of != nullptr;

  // ======================================================= a9: OEM iterations
  for (int t = 0;; ++t) {
    uint32_t qmask = 0;
#pragma unroll
    for (int q = 0; q < NPT; ++q)
      if (q < nP && lidx[q] < L) qmask |= 1u << q;
    if (!qmask) break;
    const int cur = t & 1, nxt = cur ^ 1;
    const double* vc = vec + (size_t)cur * NPT * A.pv;
    double* vn = vec + (size_t)nxt * NPT * A.pv;
    double dmax[NPT];
    bool bad = false;
#pragma unroll
    for (int q = 0; q < NPT; ++q) dmax[q] = 0.0;
    // ---- E-step + M-step: u = c + d beta - G beta for this CTA's rows
    for (int ri = 0; ri < NRT; ++ri) {
      double acc[NPT];
#pragma unroll
      for (int q = 0; q < NPT; ++q) acc[q] = 0.0;
      if (ri == 0) {
#pragma unroll
        for (int e = 0; e < EREG; ++e) {
          if (e < KPR) {
            const int k = tl + e * T;
#pragma unroll
            for (int q = 0; q < NPT; ++q)
              if ((qmask >> q) & 1u) acc[q] = fma(greg[e], vc[q * A.pv + k], acc[q]);
          }
        }
        for (int ci = EREG; ci < KPR; ++ci) {
          const double g = gsm[(size_t)(ci - EREG) * PT + tid];
          const int k = tl + ci * T;
#pragma unroll
          for (int q = 0; q < NPT; ++q)
            if ((qmask >> q) & 1u) acc[q] = fma(g, vc[q * A.pv + k], acc[q]);
        }
      } else {
        const int base = (KPR > EREG ? KPR - EREG : 0) + (ri - 1) * KPR;
        for (int ci = 0; ci < KPR; ++ci) {
          const double g = gsm[(size_t)(base + ci) * PT + tid];
          const int k = tl + ci * T;
#pragma unroll
          for (int q = 0; q < NPT; ++q)
            if ((qmask >> q) & 1u) acc[q] = fma(g, vc[q * A.pv + k], acc[q]);
        }
      }
      const int r = rg + ri * RG;
#pragma unroll
      for (int q = 0; q < NPT; ++q) {
        if (!((qmask >> q) & 1u)) continue;
        const double a = reduce_T(acc[q]);
        if (tl == 0 && r < nr) {
          const int j = j0 + r;
          const double bj = vc[q * A.pv + j];
          const double u = c_s[r] + d * bj - a;
          if (!isfinite(u)) bad = true;
          if (!grp || famq[q] < OEM_GRP_LASSO) {  // coordinate-wise family (also when mixed with group ones)
            const double nb = th_coord(famq[q], u, w_s[r] * lam[q], gamq[q], alpq[q], d);
            dmax[q] = fmax(dmax[q], fabs(nb - bj));
            if (C == 1) vn[q * A.pv + j] = nb;
            else for (int rr = 0; rr < C; ++rr) st_cluster(&vn[q * A.pv + j], rr, nb);
          } else {
            uv[q * nr + r] = u;
          }
        }
      }
    }
    if (grp) {
      // group M-step (eqs glasso / gmcp / gscad); groups lie inside [j0, j1)
      __syncthreads();
      if (nr > 0) {
        for (int e = tid; e < ng_loc * nP; e += PT) {
          const int q = e % nP, gl = e / nP;
          if (!((qmask >> q) & 1u) || P.fam[q] < OEM_GRP_LASSO) continue;
          const int a = ga_s[gl], b = gb_s[gl];
          const double* ug = uv + q * nr;
          double s = 0.0;
          for (int r = a; r < b; ++r) s += ug[r] * ug[r];
          const double nu = sqrt(s);
          double lamq = 0.0, gq = 0.0;
          int fam = 0;
#pragma unroll
          for (int qq = 0; qq < NPT; ++qq)
            if (qq == q) { lamq = lam[qq]; gq = gamq[qq]; fam = famq[qq]; }
          const double lw = gw_s[gl] * lamq;
          double f;
          double tau = 0.0;
#pragma unroll
          for (int qq = 0; qq < NPT; ++qq)
            if (qq == q) tau = alpq[qq];
          if (fam == OEM_SGL) f = sgl_factor(ug, a, b, 1, P.var_w, j0, lamq, tau, gw_s[gl], d);
          else if (fam == OEM_GRP_LASSO) f = nu > 0.0 ? pos(1.0 - lw / nu) : 0.0;
          else f = nu > 0.0 ? (fam == OEM_GRP_MCP ? th_mcp(nu, lw, gq, d) : th_scad(nu, lw, gq, d)) / nu : 0.0;
          double m = 0.0;
          for (int r = a; r < b; ++r) {
            const double nb = fam == OEM_SGL ? f * th_soft(ug[r], (P.var_w ? P.var_w[j0 + r] : 1.0) * lamq * tau, d)
                            : fam == OEM_GRP_LASSO ? ug[r] / d * f : f * ug[r];
            const int j = j0 + r;
            m = fmax(m, fabs(nb - vc[q * A.pv + j]));
            if (C == 1) vn[q * A.pv + j] = nb;
            else for (int rr = 0; rr < C; ++rr) st_cluster(&vn[q * A.pv + j], rr, nb);
          }
#pragma unroll
          for (int qq = 0; qq < NPT; ++qq)
            if (qq == q) dmax[qq] = fmax(dmax[qq], m);
        }
      }
    }
    // ---- max |dbeta| per penalty: warp -> CTA -> every CTA of the cluster
#pragma unroll
    for (int q = 0; q < NPT; ++q) {
      double m = dmax[q];
      for (int o = 16; o > 0; o >>= 1) m = fmax(m, __shfl_xor_sync(0xffffffffu, m, o));
      if (lane == 0) red[warp * (NPT + 1) + q] = m;
    }
    {
      const unsigned anybad = __ballot_sync(0xffffffffu, bad);
      if (lane == 0) red[warp * (NPT + 1) + NPT] = anybad ? 1.0 : 0.0;
    }
    __syncthreads();
    if (tid <= NPT) {
      double m = 0.0;
      for (int w = 0; w < nwarps; ++w) m = fmax(m, red[w * (NPT + 1) + tid]);
      for (int rr = 0; rr < C; ++rr) st_cluster(&dl[(size_t)(cur * C + rank) * (NPT + 2) + tid], rr, m);
    }
    cluster_sync_all();
    // ---- identical bookkeeping in every thread of every CTA of the cluster
    double delta[NPT];
    bool stop = false;
#pragma unroll
    for (int q = 0; q < NPT; ++q) delta[q] = 0.0;
    for (int r = 0; r < C; ++r) {
      const double* dr = dl + (size_t)(cur * C + r) * (NPT + 2);
#pragma unroll
      for (int q = 0; q < NPT; ++q) delta[q] = fmax(delta[q], dr[q]);
      if (dr[NPT] != 0.0) stop = true;
    }
    if (stop) {
      if (tid == 0) atomicExch(&P.flags[0], 1);
      break;
    }
#pragma unroll
    for (int q = 0; q < NPT; ++q) {
      if (!((qmask >> q) & 1u)) continue;
      const int it = itc[q] + 1;
      const bool conv = delta[q] <= P.tol;   // R#17
      if (conv || it >= P.maxit) {
        const int l = lidx[q];
        double* out = P.beta_out + (((size_t)unit * nP + q) * L + l) * p;
        for (int r = tid; r < nr; r += PT) out[P.perm[j0 + r]] = vn[q * A.pv + j0 + r];
        if (rank == 0 && tid == 0) {
          P.it_out[((size_t)unit * nP + q) * L + l] = it;
          P.cv_out[((size_t)unit * nP + q) * L + l] = conv ? 1 : 0;
        }
        lidx[q] = l + 1;
        itc[q] = 0;
        if (l + 1 < L)
          lam[q] = P.lam_explicit ? P.lam_explicit[l + 1]
                                  : (L == 1 ? lmax[q]
                                            : lmax[q] * exp(((double)(l + 1) / (double)(L - 1)) * log(P.lmin_ratio)));
      } else {
        itc[q] = it;
      }
    }
  }
}

// cluster layout: smallest C whose per-thread share fits registers + shared memory
// ---------------------------------------------------------------- K5 active-set cluster solver
// For wide units (p > 256: cfg3's 500, cfg4's 1000) on tall data the coefficient paths are sparse
// (at lambda_min = 1e-3 lambda_max the null coordinates' |c_j| ~ 1/sqrt(n) stay below lambda), so
// G beta needs only the columns of G whose coordinate has ever been nonzero. One cluster of C <= 16
// CTAs per (unit, penalty); CTA c owns rows [j0, j1) (<= 64, groups never straddle CTAs) and keeps
// G[j][k] of its rows for the ACTIVE columns k in shared memory. Per iteration (P:L171-172 E-step,
// P:L239-297 M-steps): u_j = c_j + d b_j - sum over active k of G_jk b_k for every row (4 lanes per
// row, active columns interleaved), the threshold on the row's first lane, the new coordinate
// stored into every CTA's copy of the vector only where it changed (DSMEM), "needs another
// iteration" bits and the indices of coordinates that just became nonzero OR-ed into every CTA
// (red.shared::cluster.or), one hardware cluster barrier. After the barrier every CTA appends the
// newly active columns in ascending index order (identical on every CTA: the summation order is a
// deterministic function of the data) and loads their rows of G (G is symmetric: the contiguous
// row k). Columns beyond the shared-memory capacity are read from the L2-resident Gram.
// Skipping a column whose coordinate is exactly zero changes no sum (its terms are exact zeros);
// the sum order over the active list differs from the dense solvers' column order (rounding only).
//
// Screened compact iterations (the iterates are the paper's, up to rounding). Between full
// iterations the coordinates outside the active set A are provably still zero. At a full
// iteration t0 every inactive coordinate j (or inactive group g) has a zero-test slack
// tau - z(u(t0)) (z = |u_j|, or the group M-step's norm, tau its threshold; z is 1-Lipschitz in u),
// and for a later iteration s, u_j(s) - u_j(t0) = -sum_{k in A} G_jk (b_k(s-1) - b_k(t0-1)), so
// |du_j| <= ||G_{j,A}||_2 D with D = ||b(s-1) - b(t0-1)||_2 (a group: ||G_{g,A}||_F D). The full
// iteration measures those norms over A and every CTA forms the same minimum s_min of
// (tau - z - rounding) / ||G_{j,A}||; while D (+ a rounding term) <= s_min, the iteration restricted
// to the rows and columns of A equals the full iteration (every inactive threshold returns 0), so
// CTA 0 runs those iterations alone, in four warps (the matvec split by columns, one named barrier
// per iteration, two for group families) with G_AA in shared memory: no cluster barrier, no
// exchange. D is bounded by per-coordinate running maxima, checked
// every CW iterations and at the exit; a failed check rolls back to the last certified iterate and
// the cluster resumes full iterations (every lambda starts with one, which re-derives the slacks).
// For group families A holds whole groups.
struct ActArgs {
  int C;          // CTAs per cluster
  int amax;       // active columns cached per CTA
  int apitch;     // shared-memory pitch of a cached row (doubles)
  int rows;       // max rows per CTA (<= 64)
  int pw;         // 32-bit words of a p-bit set
  int screen;     // 1: screened compact iterations between full ones
  int ncmax;      // compact capacity (32, 64 or, 256-thread CTAs, 128 active coordinates; 0: no screening)
};

constexpr int ACT_T = 4;         // lanes per row
constexpr int CW = 8;            // compact iterations per screening check

__device__ __forceinline__ void st_cl_s32(int* local, uint32_t rank, int v) {
  uint32_t a = smem_u32(local), ra;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(ra) : "r"(a), "r"(rank));
  asm volatile("st.shared::cluster.s32 [%0], %1;" ::"r"(ra), "r"(v) : "memory");
}

template <int ACT_THREADS>       // 256 (64 rows per CTA) or 512 (128 rows per CTA)
__global__ void __launch_bounds__(ACT_THREADS, 1) fit_active_kernel(const PathParams P, const ActArgs A) {
  extern __shared__ __align__(16) double sm[];
  __shared__ uint32_t F[3];
  // per (CTA, warp) of a full iteration (parity t & 1): minimum screening slack, sum of (db_j)^2,
  // sum of b_j(t0-1)^2
  __shared__ double SLs[2][3][256];
  __shared__ int s_na;
  __shared__ double s_lmax;
  __shared__ int s_oc[2];                // compact phase: outcome, iterations
  __shared__ int cfl4[2][4];             // compact warps' flag words (iteration parity, warp)
  __shared__ double csum4[2][4];         // compact warps' partial sums (slot, warp)
  const int p = P.p, nPg = P.nP, L = P.L, C = A.C;
  const int clu = blockIdx.x / C;
  const int unit = clu / nPg, q = clu % nPg;   // one penalty per cluster
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31, r = tid / ACT_T, tl = tid % ACT_T;
  constexpr int NW = ACT_THREADS / 32;
  const uint32_t rank = cluster_rank();
  const int j0 = P.cta_j0[blockIdx.x], j1 = P.cta_j1[blockIdx.x], nr = j1 - j0;
  const double* Gu = P.Gn + (size_t)unit * p * p;
  const double* cu = P.cn + (size_t)unit * p;
  const int pv = (p + 1) & ~1;
  const int NCM = A.ncmax;
  // shared memory: vec [2][pv] | gc [NCM][NCM] | bcv [2][NCM] | res, ucv, cwv [NCM] | part [4][NCM] | ga [rows][apitch] |
  //                uv [2][rows] | gw, ga_s, gb_s [rows] | act [p] | abits, nbits [2][pw]
  double* vec = sm;
  double* gc = vec + 2 * (size_t)pv;
  double* bcv = gc + (size_t)NCM * NCM;
  double* res = bcv + 2 * (size_t)NCM;
  double* ucv = res + NCM;
  double* cwv = ucv + NCM;
  double* part = cwv + NCM;   // [4][NCM] compact matvec partial sums
  double* ga = part + 4 * (size_t)NCM;
  double* uv = ga + (size_t)A.rows * A.apitch;   // [2][rows]: u, then ||G_{j,A}||^2 (screening)
  double* gw_s = uv + 2 * A.rows;
  int* ga_s = reinterpret_cast<int*>(gw_s + A.rows);
  int* gb_s = ga_s + A.rows;
  int* act = gb_s + A.rows;
  uint32_t* abits = reinterpret_cast<uint32_t*>(act + p);
  uint32_t* nbits = abits + A.pw;   // [2][pw]
  const int fam = P.fam[q];
  const double gq = P.gam[q], aq = P.alp[q];
  const bool grp = P.g_of != nullptr && fam >= OEM_GRP_LASSO;
  const int g0 = (P.g_of && nr > 0) ? P.g_of[j0] : 0;
  const int ng_loc = (grp && nr > 0) ? P.g_of[j1 - 1] + 1 - g0 : 0;
  for (int gg = tid; gg < ng_loc; gg += ACT_THREADS) {
    gw_s[gg] = P.g_w[g0 + gg];
    ga_s[gg] = P.g_start[g0 + gg] - j0;
    gb_s[gg] = P.g_end[g0 + gg] - j0;
  }
  // warm or cold start (permuted order) into both buffers; the initial active set is its support
  // (whole groups for a group family)
  for (int k = tid; k < pv; k += ACT_THREADS) {
    const double b = (P.beta_init && k < p) ? P.beta_init[((size_t)unit * nPg + q) * p + P.perm[k]] : 0.0;
    vec[k] = b;
    vec[pv + k] = b;
  }
  for (int w = tid; w < 3 * A.pw; w += ACT_THREADS) abits[w] = 0u;
  if (tid < 3) F[tid] = 0u;
  __syncthreads();
  if (tid == 0) {
    int na = 0;
    if (P.beta_init) {
      for (int k = 0; k < p; ++k)
        if (vec[k] != 0.0) abits[k >> 5] |= 1u << (k & 31);
      if (grp)
        for (int gg = 0; gg < P.ngroups; ++gg) {
          bool on = false;
          for (int k = P.g_start[gg]; k < P.g_end[gg]; ++k) on = on || ((abits[k >> 5] >> (k & 31)) & 1u);
          if (on)
            for (int k = P.g_start[gg]; k < P.g_end[gg]; ++k) abits[k >> 5] |= 1u << (k & 31);
        }
      for (int k = 0; k < p; ++k)
        if ((abits[k >> 5] >> (k & 31)) & 1u) act[na++] = k;
    }
    s_na = na;
  }
  __syncthreads();
  int na = s_na;
  for (int e = tid; e < nr * min(na, A.amax); e += ACT_THREADS) {
    const int rr = e / min(na, A.amax), a = e % min(na, A.amax);
    ga[(size_t)rr * A.apitch + a] = Gu[(size_t)act[a] * p + j0 + rr];
  }
  const double d = P.d[unit];
  const double c_my = r < nr ? cu[j0 + r] : 0.0;
  const double w_my = (r < nr && P.var_w) ? P.var_w[j0 + r] : 1.0;
  // rounding scale of a computed u_j (gamma_{p+4}, times a safety factor of 4)
  const double gam_u = 4.0 * (p + 4) * 1.1102230246251565e-16;
  // ---- a8: lambda grid of this (unit, penalty) (R#14-16, R#22), as in the other solvers
  if (warp == 0) {
    double lm = 0.0;
    const double* cc = P.shared_grid ? P.cn : cu;
    if (P.lmax_override) {
      lm = *P.lmax_override;
    } else if (fam == OEM_SGL) {
      for (int gg = lane; gg < P.ngroups; gg += 32)
        lm = fmax(lm, sgl_lmax_group(cc, P.g_start[gg], P.g_end[gg], P.var_w, P.g_w[gg], aq));
    } else if (fam >= OEM_GRP_LASSO) {
      for (int gg = lane; gg < P.ngroups; gg += 32) {
        const double cg = P.g_w[gg];
        if (!(cg > 0.0)) continue;
        double sq = 0.0;
        for (int j = P.g_start[gg]; j < P.g_end[gg]; ++j) sq += cc[j] * cc[j];
        lm = fmax(lm, sqrt(sq) / cg);
      }
    } else {
      const double scl = fam == OEM_ENET ? aq : 1.0;
      for (int j = lane; j < p; j += 32) {
        const double wj = P.var_w ? P.var_w[j] : 1.0;
        if (!(wj > 0.0)) continue;
        lm = fmax(lm, fabs(cc[j]) / (scl * wj));
      }
    }
#pragma unroll
    for (int o = 16; o >= 1; o >>= 1) lm = fmax(lm, __shfl_xor_sync(0xffffffffu, lm, o));
    if (lane == 0) {
      s_lmax = lm;
      bool bad = false;  // parameter validity against the d in use (R#8)
      if (fam == OEM_MCP || fam == OEM_GRP_MCP) bad = !(gq > 1.0) || !(gq * d > 1.0);
      if (fam == OEM_SCAD || fam == OEM_GRP_SCAD) bad = !(gq > 2.0) || !((gq - 1.0) * d > 1.0);
      if (fam == OEM_ENET) bad = !(aq >= 0.0 && aq <= 1.0);
      if (bad) { atomicExch(&P.flags[1], 1); s_lmax = -1.0; }
    }
  }
  __syncthreads();
  if (s_lmax < 0.0) return;   // invalid parameters: every CTA of the cluster leaves together
  auto lam_at = [&](int l) -> double {
    if (P.lam_explicit) return P.lam_explicit[l];
    if (L == 1) return s_lmax;
    return s_lmax * exp(((double)l / (double)(L - 1)) * log(P.lmin_ratio));  // R#15
  };
  if (rank == 0)
    for (int l = tid; l < L; l += ACT_THREADS) P.lam_out[((size_t)unit * nPg + q) * L + l] = lam_at(l);
  int lidx = 0, itc = 0;
  double lam = lam_at(0);
  const double rd = 1.0 / d;
  // (the group families' norm thresholds are the coordinate MCP / SCAD ones)
  const double rgq = (fam == OEM_MCP || fam == OEM_GRP_MCP) ? 1.0 / (gq * d - 1.0)
                   : (fam == OEM_SCAD || fam == OEM_GRP_SCAD) ? 1.0 / ((gq - 1.0) * d - 1.0) : 0.0;
  int cfail = 0, cwait = 0;      // failed compact phases at this lambda; full iterations before the next
  int built_na = -1, built_pitch = 0;   // CTA 0: size of the active set whose G_AA is in gc, its pitch
  cluster_sync_all();  // every CTA initialised before the first remote store
  auto inA = [&](int k) -> bool { return (abits[k >> 5] >> (k & 31)) & 1u; };

  // ======================================================= a9: OEM iterations
  for (int t = 0; lidx < L; ++t) {
    const int cur = t & 1, par = t & 1;
    const double* vc = vec + (size_t)cur * pv;
    double* vn = vec + (size_t)(cur ^ 1) * pv;
    if (tid == 0) F[(t + 1) % 3] = 0u;
    // ---- E-step: u_j = c_j + d b_j - sum_{k active} G_jk b_k
    // (screening: r2 = ||G_{j,A}||^2 over the same active columns)
    double acc = 0.0, r2 = 0.0;
    if (r < nr) {
      const double* gr = ga + (size_t)r * A.apitch;
      const int nc = min(na, A.amax);
      int a = tl;
      for (; a + 3 * ACT_T < nc; a += 4 * ACT_T) {   // four independent loads in flight
        const double b0 = vc[act[a]], b1 = vc[act[a + ACT_T]], b2 = vc[act[a + 2 * ACT_T]], b3 = vc[act[a + 3 * ACT_T]];
        const double g0 = gr[a], g1 = gr[a + ACT_T], g2 = gr[a + 2 * ACT_T], g3 = gr[a + 3 * ACT_T];
        acc = fma(g0, b0, acc);
        acc = fma(g1, b1, acc);
        acc = fma(g2, b2, acc);
        acc = fma(g3, b3, acc);
        if (A.screen) r2 = fma(g3, g3, fma(g2, g2, fma(g1, g1, fma(g0, g0, r2))));
      }
      for (; a < nc; a += ACT_T) {
        const double g0 = gr[a];
        acc = fma(g0, vc[act[a]], acc);
        r2 = fma(g0, g0, r2);
      }
      for (a = A.amax + tl; a < na; a += ACT_T) {  // beyond capacity
        const double g0 = Gu[(size_t)act[a] * p + j0 + r];
        acc = fma(g0, vc[act[a]], acc);
        r2 = fma(g0, g0, r2);
      }
    }
#pragma unroll
    for (int o = ACT_T / 2; o >= 1; o >>= 1) {
      acc += __shfl_xor_sync(0xffffffffu, acc, o);
      r2 += __shfl_xor_sync(0xffffffffu, r2, o);
    }
    uint32_t bits = 0;
    double slk = INFINITY;   // this lane's screening slack (inactive coordinates / groups)
    const int j = j0 + r;
    double dsq = 0.0, bsq = 0.0;   // screening: this lane's sum of (db_j)^2 and of b_j^2
    auto emit = [&](int jj, double nb, bool req) {   // new coordinate jj: vector copies, flags, activation
      const double bj = vc[jj];
      dsq = fma(nb - bj, nb - bj, dsq);
      bsq = fma(bj, bj, bsq);
      if (!(fabs(nb - bj) <= P.tol)) bits |= 1u;
      if (nb != vn[jj])
        for (int rr = 0; rr < C; ++rr) st_cl_f64(&vn[jj], rr, nb);
      if (req && !inA(jj))
        for (int rr = 0; rr < C; ++rr) red_or_cl(&nbits[par * A.pw + (jj >> 5)], rr, 1u << (jj & 31));
    };
    if (tl == 0 && r < nr && lidx < L) {
      const double u = c_my + d * vc[j] - acc;
      if (!isfinite(u)) bits |= 0x80000000u;
      if (!grp) {
        const double nb = th_coord(fam, u, w_my * lam, gq, aq, d);
        emit(j, nb, nb != 0.0);
        // zero iff |u| <= tau (lasso, MCP, SCAD: w lam; elastic net: w lam alpha); u_j moves by at
        // most ||G_{j,A}|| ||db_A||, and its rounding by gam_u (|c_j| + ||G_{j,A}|| ||b||)
        if (A.screen && nb == 0.0 && !inA(j) && r2 > 0.0) {
          const double tau = w_my * lam * (fam == OEM_ENET ? aq : 1.0);
          slk = fmax((tau - fabs(u) - 2.0 * gam_u * fabs(c_my) - 1e-13 * tau) / (sqrt(r2) * (1.0 + 1e-12)), 0.0);
        }
      } else {
        uv[r] = u;
        uv[A.rows + r] = r2;
      }
    }
    if (grp) {
      // group M-step (eqs glasso / gmcp / gscad / sglasso; the arithmetic of
      // group_mstep_warp); groups lie inside [j0, j1). A group enters the active set whole.
      __syncthreads();
      const bool sgl = fam == OEM_SGL;
      for (int gl = warp; gl < ng_loc; gl += NW) {
        const int ra = ga_s[gl], rb = gb_s[gl];
        double ss = 0.0;
        for (int rr = ra + lane; rr < rb; rr += 32) {
          const double v = sgl ? th_soft(uv[rr], (P.var_w ? P.var_w[j0 + rr] : 1.0) * lam * aq, d) : uv[rr];
          ss += v * v;
        }
#pragma unroll
        for (int o = 16; o >= 1; o >>= 1) ss += __shfl_xor_sync(0xffffffffu, ss, o);
        const double nu = sqrt(ss);
        const double cg = gw_s[gl], lw = cg * lam;
        double f;
        if (sgl) f = nu > 0.0 ? pos(1.0 - cg * lam * (1.0 - aq) / (d * nu)) : 0.0;   // R#11 (nu = ||v||)
        else if (fam == OEM_GRP_LASSO) f = nu > 0.0 ? pos(1.0 - lw / nu) : 0.0;
        else f = nu > 0.0 ? (fam == OEM_GRP_MCP ? th_mcp(nu, lw, gq, d) : th_scad(nu, lw, gq, d)) / nu : 0.0;
        for (int rr = ra + lane; rr < rb; rr += 32) {
          const double nb = sgl ? f * th_soft(uv[rr], (P.var_w ? P.var_w[j0 + rr] : 1.0) * lam * aq, d)
                          : fam == OEM_GRP_LASSO ? uv[rr] / d * f : f * uv[rr];
          emit(j0 + rr, nb, f > 0.0);
        }
        // zero iff z <= tau: z = ||u_g|| against c_g lam, or (sparse group lasso) d ||v|| =
        // ||S(u_g, w lam tau)|| against c_g lam (1 - tau); both 1-Lipschitz in u_g, which moves by
        // at most ||G_{g,A}||_F ||db_A|| (rounding: gam_u (||c_g|| + ||G_{g,A}||_F ||b||))
        if (A.screen) {
          double f2 = 0.0, c2 = 0.0;
          for (int rr = ra + lane; rr < rb; rr += 32) {
            f2 += uv[A.rows + rr];
            c2 = fma(cu[j0 + rr], cu[j0 + rr], c2);
          }
#pragma unroll
          for (int o = 16; o >= 1; o >>= 1) {
            f2 += __shfl_xor_sync(0xffffffffu, f2, o);
            c2 += __shfl_xor_sync(0xffffffffu, c2, o);
          }
          if (f == 0.0 && !inA(j0 + ra) && f2 > 0.0) {
            const double tau = sgl ? cg * lam * (1.0 - aq) : lw;
            const double z = sgl ? d * nu : nu;
            // (the norm's own rounding: (n_g + 8) ulps relative, and 1e-13 for the M-step's test)
            const double rel = 1e-13 + 4.0 * 1.1102230246251565e-16 * (rb - ra + 8);
            slk = fmin(slk, fmax((tau - z - 2.0 * gam_u * sqrt(c2) - rel * tau) / (sqrt(f2) * (1.0 + 1e-12)), 0.0));
          }
        }
      }
    }
    if (A.screen) {
#pragma unroll
      for (int o = 16; o >= 1; o >>= 1) {
        slk = fmin(slk, __shfl_xor_sync(0xffffffffu, slk, o));
        dsq += __shfl_xor_sync(0xffffffffu, dsq, o);
        bsq += __shfl_xor_sync(0xffffffffu, bsq, o);
      }
      // every warp's minimum into its slot in every CTA (plain stores, read after the barrier;
      // parity t & 1: the slot is rewritten at t + 2, after the next barrier)
      if (lane == 0) {
        const int sl = rank * NW + warp;
        if (C == 1) {
          SLs[t & 1][0][sl] = slk; SLs[t & 1][1][sl] = dsq; SLs[t & 1][2][sl] = bsq;
        } else {
          for (int rr = 0; rr < C; ++rr) {
            st_cl_f64(&SLs[t & 1][0][sl], rr, slk);
            st_cl_f64(&SLs[t & 1][1][sl], rr, dsq);
            st_cl_f64(&SLs[t & 1][2][sl], rr, bsq);
          }
        }
      }
    }
    bits = __reduce_or_sync(0xffffffffu, bits);
    if (lane == 0 && bits)
      for (int rr = 0; rr < C; ++rr) red_or_cl(&F[t % 3], rr, bits);
    cluster_sync_all();
    const uint32_t f = F[t % 3];
    if (f & 0x80000000u) {
      if (tid == 0) atomicExch(&P.flags[0], 1);
      break;
    }
    // ---- newly active columns. Every warp checks the request words in parallel (the same answer
    // in every warp, so no block barrier when nothing changed, the common case); otherwise they
    // are appended in ascending index order on every CTA and their rows of G loaded.
    bool any = false;
    for (int w = lane; w < A.pw; w += 32) any = any || (nbits[par * A.pw + w] & ~abits[w]) != 0u;
    const bool grew = __any_sync(0xffffffffu, any);
    if (grew) {
      int added = 0;
      for (int w = 0; w < A.pw; ++w) {
        uint32_t nw = nbits[par * A.pw + w] & ~abits[w];
        while (nw) {
          const int k = 32 * w + __ffs(nw) - 1;
          nw &= nw - 1;
          if (tid == 0) act[na + added] = k;
          ++added;
        }
      }
      __syncthreads();   // act[] complete before the loads; every thread has read nbits / abits
      for (int e = tid; e < nr * added; e += ACT_THREADS) {
        const int rr = e / added, a = na + e % added;
        if (a < A.amax) ga[(size_t)rr * A.apitch + a] = Gu[(size_t)act[a] * p + j0 + rr];
      }
      for (int w = tid; w < A.pw; w += ACT_THREADS) {
        abits[w] |= nbits[par * A.pw + w];
        nbits[par * A.pw + w] = 0u;   // reused at t + 2 (after the next cluster barrier)
      }
      na += added;
      __syncthreads();
    }
    // ---- bookkeeping (identical in every thread of every CTA of the cluster)
    auto finish_lambda = [&](int it, bool conv) {
      double* out = P.beta_out + (((size_t)unit * nPg + q) * L + lidx) * p;
      for (int rr = tid; rr < nr; rr += ACT_THREADS) out[P.perm[j0 + rr]] = vn[j0 + rr];
      if (rank == 0 && tid == 0) {
        P.it_out[((size_t)unit * nPg + q) * L + lidx] = it;
        P.cv_out[((size_t)unit * nPg + q) * L + lidx] = conv ? 1 : 0;
      }
      ++lidx;
      itc = 0;
      cfail = 0;
      cwait = 0;
      if (lidx < L) lam = lam_at(lidx);
    };
    {
      const int it = itc + 1;
      const bool conv = !(f & 1u);   // every |dbeta_j| <= tol (R#17)
      if (conv || it >= P.maxit) {
        finish_lambda(it, conv);
        continue;
      }
      itc = it;
    }
    if (cwait > 0) --cwait;
    // (after an activation the next full iteration first measures ||G_{j,A}|| over the new A)
    if (!A.screen || cwait > 0 || grew || na == 0 || na > NCM) continue;
    // the cluster's minimum slack and the entry certificate, ||b(t0) - b(t0-1)||_2 against it (same
    // values, summed in the same order, on every CTA: a uniform decision)
    double smin = INFINITY, dsum = 0.0, bsum = 0.0;
    for (int k = lane; k < C * NW; k += 32) {
      smin = fmin(smin, SLs[t & 1][0][k]);
      dsum += SLs[t & 1][1][k];
      bsum += SLs[t & 1][2][k];
    }
#pragma unroll
    for (int o = 16; o >= 1; o >>= 1) {
      smin = fmin(smin, __shfl_xor_sync(0xffffffffu, smin, o));
      dsum += __shfl_xor_sync(0xffffffffu, dsum, o);
      bsum += __shfl_xor_sync(0xffffffffu, bsum, o);
    }
    if (!(sqrt(dsum) * (1.0 + 2.0 * gam_u) + 2.0 * gam_u * sqrt(bsum) <= smin * (1.0 - 1e-12))) continue;

    // ======================================================= screened compact phase (CTA 0)
    // A = act[0..na) (whole groups for group families, contiguous); b(t0) in vn, b(t0-1) in vc.
    if (rank == 0) {
      const int nc = na, ncp = (nc + 7) & ~7;
      // G_AA column-major with pitch 32 R (R = rows per lane of the compact warp: a compile-time
      // pitch in the loop), gc[k][i] = G[act[i]][act[k]], zero-padded, kept while A is unchanged.
      // Only the entries of new rows / columns are loaded (A only grows), four L2 loads in flight
      // per thread; padding columns [nc, ncp) are zero (rows >= nc are never used).
      const int pitch = nc <= 32 ? 32 : nc <= 64 ? 64 : 128;
      if (pitch != built_pitch) { built_na = -1; built_pitch = pitch; }
      if (nc != built_na) {
        const int b0 = built_na < 0 ? 0 : built_na, tot = ncp * nc;
        for (int e0 = tid; e0 < tot; e0 += 4 * ACT_THREADS) {
          double v[4];
          int at[4];
#pragma unroll
          for (int u4 = 0; u4 < 4; ++u4) {
            const int e = e0 + u4 * ACT_THREADS, k = e / nc, i = e - k * nc;
            at[u4] = (e < tot && (k >= b0 || i >= b0)) ? k * pitch + i : -1;
            v[u4] = (at[u4] >= 0 && k < nc) ? Gu[(size_t)act[k] * p + act[i]] : 0.0;
          }
#pragma unroll
          for (int u4 = 0; u4 < 4; ++u4)
            if (at[u4] >= 0) gc[at[u4]] = v[u4];
        }
        built_na = nc;
      }
      for (int i = tid; i < NCM; i += ACT_THREADS) {
        bcv[i] = i < nc ? vn[act[i]] : 0.0;
        bcv[NCM + i] = 0.0;
        cwv[i] = (i < nc && P.var_w) ? P.var_w[act[i]] : 1.0;
      }
      __syncthreads();
      if (warp < 4) {
        // Four warps (one per SM sub-partition, named barrier 1): in the matvec warp w sums the
        // columns [w ncp/4, (w+1) ncp/4) for every row (R rows per lane: lane + 32 h); the partial
        // sums meet in shared memory and are added in a fixed order; warp w then thresholds row
        // lane + 32 w. Divisions by constants use the refined reciprocal (within one ulp), group
        // norms rsqrt: the compact iterate equals the full one up to rounding.
        // FC: the coordinate family as a compile-time constant (no per-iteration dispatch), or 4 for
        // the group families (dispatched on `fam` inside)
        auto run = [&](auto RC, auto FC) {
          constexpr int R = decltype(RC)::value;   // 32-row blocks of the matvec (nc <= 32 R)
          constexpr int FAMC = decltype(FC)::value;
          constexpr int PR = 32 * R;               // gc pitch
          auto csync = []() { asm volatile("bar.sync 1, 128;" ::: "memory"); };
          const int i = lane + 32 * warp;          // this lane's row in the threshold step
          const bool valid = i < nc;
          const int ci = valid ? act[i] : 0;
          const double c_i = valid ? cu[ci] : 0.0, w_i = valid ? cwv[i] : 1.0;
          const double enden = d + w_i * lam * (1.0 - aq), rden = 1.0 / enden;
          int cga = i, cgb = i + 1;
          double cg_i = 0.0;
          if (grp && valid) {
            const int g = P.g_of[ci];
            cga = i - (ci - P.g_start[g]);
            cgb = cga + (P.g_end[g] - P.g_start[g]);
            cg_i = P.g_w[g];
          }
          double b = valid ? bcv[i] : 0.0;
          const double bref = valid ? vc[ci] : 0.0;
          double e = valid ? fabs(b - bref) : 0.0, bsnap = b;
          // sum over the four warps (warp sums, then a fixed order); slot alternates
          auto xsum = [&](double v, int slot) -> double {
#pragma unroll
            for (int o = 16; o >= 1; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
            if (lane == 0) csum4[slot][warp] = v;
            csync();
            return (csum4[slot][0] + csum4[slot][1]) + (csum4[slot][2] + csum4[slot][3]);
          };
          // ||b(t0-1)||_2 over A (every other coordinate is 0): the rounding term's scale;
          // se = sum_i e_i^2 >= ||b(s-1) - b(t0-1)||_2^2 over the iterations so far
          const double nbref = sqrt(xsum(bref * bref, 0));
          auto certified = [&](double se) -> bool {
            return sqrt(se) * (1.0 + 2.0 * gam_u) + 2.0 * gam_u * nbref <= smin;
          };
          const double se0 = xsum(e * e, 1);
          int it = 0, itsnap = 0, oc = 2, slot = 0;
          const bool sgl = fam == OEM_SGL;
          const int cfam = fam == OEM_GRP_MCP ? OEM_MCP : fam == OEM_GRP_SCAD ? OEM_SCAD : fam;
          const int ncq = ncp >> 2, k0 = warp * ncq;
          if (certified(se0)) {
            for (;;) {
              const double* bcur = bcv + (it & 1) * NCM;
              double* bnx = bcv + ((it & 1) ^ 1) * NCM;
              // ---- matvec partials over this warp's columns
              double a[R][2];
#pragma unroll
              for (int h = 0; h < R; ++h) a[h][0] = a[h][1] = 0.0;
              const double* gk = gc + (size_t)k0 * PR + lane;
              const double* xk = bcur + k0;
#pragma unroll 4
              for (int k = 0; k < ncq; k += 2, gk += 2 * PR, xk += 2) {
                const double2 x0 = *reinterpret_cast<const double2*>(xk);
#pragma unroll
                for (int h = 0; h < R; ++h) {
                  a[h][0] = fma(gk[32 * h], x0.x, a[h][0]);
                  a[h][1] = fma(gk[PR + 32 * h], x0.y, a[h][1]);
                }
              }
#pragma unroll
              for (int h = 0; h < R; ++h) part[warp * NCM + lane + 32 * h] = a[h][0] + a[h][1];
              csync();
              // ---- E-step and M-step of row i
              const int iu = valid ? i : 0;
              const double u = c_i + d * b - ((part[iu] + part[NCM + iu]) + (part[2 * NCM + iu] + part[3 * NCM + iu]));
              double nb = 0.0;
              if constexpr (FAMC == OEM_ENET) {   // eq (net): the divisor d + w lam (1 - alpha) is fixed in the phase
                const double t = fabs(u) - w_i * lam * aq;
                nb = t > 0.0 ? sgn(u) * div_r(t, enden, rden) : 0.0;
              } else if constexpr (FAMC < 4) {
                nb = th_coord_r(FAMC, u, w_i * lam, gq, aq, d, rd, rgq);
              } else {
                // the row's square (of u, or of its soft-threshold for the sparse group lasso),
                // then every row sums its group's squares
                const double vs = sgl ? th_coord_r(OEM_LASSO, u, w_i * lam * aq, 0.0, 0.0, d, rd, 0.0) : u;
                if (valid) ucv[i] = vs * vs;
                csync();
                double s0 = 0.0, s1 = 0.0, s2 = 0.0, s3 = 0.0;
                int rr = cga;
                if (valid) {
                  for (; rr + 3 < cgb; rr += 4) {
                    s0 += ucv[rr];
                    s1 += ucv[rr + 1];
                    s2 += ucv[rr + 2];
                    s3 += ucv[rr + 3];
                  }
                  for (; rr < cgb; ++rr) s0 += ucv[rr];
                }
                const double ss = (s0 + s1) + (s2 + s3);
                const double rnu = ss > 0.0 ? rsqrt(ss) : 0.0, nu = ss * rnu;
                const double lw = cg_i * lam;
                double fg;
                if (sgl) fg = pos(1.0 - cg_i * lam * (1.0 - aq) * rd * rnu);
                else if (fam == OEM_GRP_LASSO) fg = pos(1.0 - lw * rnu);
                else fg = th_coord_r(cfam, nu, lw, gq, 0.0, d, rd, rgq) * rnu;
                nb = sgl ? fg * vs : fam == OEM_GRP_LASSO ? u * rd * fg : fg * u;
              }
              int fl = 0;
              if (valid) {
                fl = (!(fabs(nb - b) <= P.tol) ? 1 : 0) | (!isfinite(u) ? 2 : 0);
                bnx[i] = nb;
                e = fmax(e, fabs(nb - bref));
                b = nb;
              }
              ++it;
              fl = __reduce_or_sync(0xffffffffu, fl);
              if (lane == 0) cfl4[it & 1][warp] = fl;
              csync();
              fl = (cfl4[it & 1][0] | cfl4[it & 1][1]) | (cfl4[it & 1][2] | cfl4[it & 1][3]);
              if (fl & 2) { oc = 4; break; }
              const bool conv = !(fl & 1);
              const bool capped = itc + it >= P.maxit;
              if (conv || capped || (it % CW) == 0) {
                if (!certified(xsum(e * e, slot))) {
                  oc = 2;
                  b = bsnap;
                  it = itsnap;
                  break;
                }
                slot ^= 1;
                bsnap = b;
                itsnap = it;
                if (conv) { oc = 1; break; }
                if (capped) { oc = 3; break; }
              }
            }
          }
          if (valid) res[i] = b;
          if (tid == 0) { s_oc[0] = oc; s_oc[1] = it; }
        };
        auto go = [&](auto RC) {
          if (grp) run(RC, std::integral_constant<int, 4>{});
          else if (fam == OEM_LASSO) run(RC, std::integral_constant<int, OEM_LASSO>{});
          else if (fam == OEM_ENET) run(RC, std::integral_constant<int, OEM_ENET>{});
          else if (fam == OEM_MCP) run(RC, std::integral_constant<int, OEM_MCP>{});
          else run(RC, std::integral_constant<int, OEM_SCAD>{});
        };
        if (nc <= 32) go(std::integral_constant<int, 1>{});
        else if (nc <= 64) go(std::integral_constant<int, 2>{});
        else if constexpr (ACT_THREADS == 256) go(std::integral_constant<int, 4>{});   // (register budget)
      }
      __syncthreads();
      const int oc = s_oc[0], its = s_oc[1];
      // the result into both vector buffers of every CTA, the outcome into every CTA
      for (int e = tid; e < nc * C; e += ACT_THREADS) {
        const int i = e % nc, rr = e / nc, k = act[i];
        st_cl_f64(&vec[k], rr, res[i]);
        st_cl_f64(&vec[pv + k], rr, res[i]);
      }
      if (tid == 0)
        for (int rr = 1; rr < C; ++rr) { st_cl_s32(&s_oc[0], rr, oc); st_cl_s32(&s_oc[1], rr, its); }
    }
    cluster_sync_all();
    const int oc = s_oc[0], its = s_oc[1];
    if (oc == 4) {
      if (tid == 0) atomicExch(&P.flags[0], 1);
      break;
    }
    itc += its;
    if (oc == 1 || oc == 3) {
      finish_lambda(itc, oc == 1);
    } else {
      ++cfail;
      cwait = 1 << min(cfail, 3);
    }
  }
  cluster_sync_all();   // no CTA leaves while a peer may still store into its shared memory
}

struct ClusterLayout {
  int C = 0, T = 1, RG = PT, KPR = 0, NRT = 1, S = 0, pv = 0, ereg = 32, maxrows = 0;
  size_t smem = 0;
  std::vector<int> j0, j1;
};

static bool make_cluster_layout(int nU, int p, int NPT, const std::vector<int>& gstart, int num_sms, int ereg,
                                ClusterLayout& lo) {
  lo.ereg = ereg;
  lo.pv = (p + 1) / 2 * 2 + 2;
  for (int C = 1; C <= 16; ++C) {
    // group-aligned cuts
    std::vector<int> cuts{0};
    for (int c = 1; c < C; ++c) {
      const int target = (int)((int64_t)p * c / C);
      int best = target;
      if (!gstart.empty()) {
        best = -1;
        for (int b : gstart)
          if (b > cuts.back() && b < p && (best < 0 || std::abs(b - target) < std::abs(best - target))) best = b;
        if (best < 0) break;
      }
      if (best > cuts.back() && best < p) cuts.push_back(best);
    }
    cuts.push_back(p);
    if ((int)cuts.size() - 1 != C) continue;
    int maxrows = 0;
    for (int c = 0; c < C; ++c) maxrows = std::max(maxrows, cuts[c + 1] - cuts[c]);
    int T = 32;
    while (T > 1 && PT / T < maxrows) T >>= 1;
    const int RG = PT / T;
    const int NRT = (maxrows + RG - 1) / RG;
    const int KPR = (p + T - 1) / T;
    const int S = std::max(0, KPR - ereg) + (NRT - 1) * KPR;
    // vectors are read at every column index a thread owns (tl + ci*T < KPR*T): pad to that
    lo.pv = std::max((p + 1) / 2 * 2 + 2, (KPR * T + 1) / 2 * 2);
    const size_t smem = ((size_t)S * PT + (size_t)2 * NPT * lo.pv + (size_t)2 * C * (NPT + 2) + 32 * (NPT + 1) +
                         (size_t)NPT * maxrows + (size_t)5 * maxrows + 8) * 8;
    if (smem > 200 * 1024) continue;
    if ((int64_t)nU * C > 8L * num_sms) return false;
    lo.C = C; lo.T = T; lo.RG = RG; lo.KPR = KPR; lo.NRT = NRT; lo.S = S; lo.smem = smem; lo.maxrows = maxrows;
    lo.j0.clear(); lo.j1.clear();
    for (int u = 0; u < nU; ++u)
      for (int c = 0; c < C; ++c) { lo.j0.push_back(cuts[c]); lo.j1.push_back(cuts[c + 1]); }
    return true;
  }
  return false;
}

template <int NPT>
static oem_status launch_cluster(const PathParams& P, const ClusterArgs& A, int nU, size_t smem, cudaStream_t st) {
  auto kern = fit_cluster_kernel<NPT, (NPT <= 1 ? 32 : NPT == 2 ? 24 : NPT == 4 ? 16 : 8)>;
  OEM_CUDA_TRY(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  if (A.C > 8) OEM_CUDA_TRY(cudaFuncSetAttribute(kern, cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3((unsigned)(nU * A.C));
  cfg.blockDim = dim3(PT);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = (unsigned)A.C;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  OEM_CUDA_TRY(cudaLaunchKernelEx(&cfg, kern, P, A));
  return OEM_OK;
}

// ---------------------------------------------------------------- lean solver: host layout / launch
struct LeanLayout {
  int variant = -1;  // default: 7 (p <= 128), 9 (p <= 256), 10 (p <= 512); the rest via OEM_LEAN_VARIANT
  int C = 1, rows = 0, pvl = 0;
  size_t smem = 0;
  std::vector<int> cuts;  // C + 1 row cuts (group aligned)
};

static bool lean_layout_try(int p, int NPT, const std::vector<int>& gstart, int v, int R, int KC, int T, int RS,
                            int NTH, LeanLayout& lo);

static bool make_lean_layout(int p, int NPT, const std::vector<int>& gstart, LeanLayout& lo) {
  // variants: rows per CTA = R * 512 / T, columns = KC * T
  // variant 5: 32 register rows + 32 shared-memory rows per CTA (p <= 512, clusters of <= 8)
  // variant 6: 256 threads (8 warps, 4 rows per thread): less per-iteration overhead at p <= 128
  // variants 7, 8: four lanes per row (short reduce-scatter, 32-column FMA chains), 256 / 512 threads
  // variant 9: 256 threads, 4 rows x 16 columns per thread (the 256-thread form of variant 2)
  // variant 10: 256 threads, 4 register + 4 shared-memory rows per thread (the 256-thread form of 5)
  // variant 11: 256 threads, 4 register + 4 shared-memory rows x 16 columns per thread, 16 lanes
  // per row (128 rows per CTA: p <= 256 in clusters of 2)
  // variant 12: 256 threads, 2 rows x 16 columns per thread, 16 lanes per row (32 rows per CTA:
  // p <= 256 in clusters of up to 8)
  static const int R_[13] = {1, 2, 2, 1, 1, 2, 4, 2, 1, 4, 4, 4, 2},
                   KC_[13] = {8, 16, 16, 8, 16, 16, 16, 32, 32, 16, 16, 16, 16},
                   T_[13] = {8, 8, 16, 16, 16, 32, 8, 4, 4, 16, 32, 16, 16},
                   RS_[13] = {0, 0, 0, 0, 0, 2, 0, 0, 0, 0, 4, 4, 0},
                   NTH_[13] = {PT, PT, PT, PT, PT, PT, 256, 256, PT, 256, 256, 256, 256};
  // measured (path phase, one B200): p = 20 variant 0 0.83 -> 7 0.76 us/iteration; p = 100
  // (cfg2) 1 1.01 -> 7 0.88; p = 200 (cfg5 inner solves) 2 96.7 ms -> 9 83.2 ms; p = 500 (cfg3)
  // 5 2.49 -> 10 2.18 us/iteration
  // p = 200 (sparse workload paths, 2 penalties): variant 9 (C = 4) 2.96 -> 12 (C = 7) 2.16
  // us/iteration, 11 (C = 2) 4.79; variant 12 needs groups of <= 32 columns, else 9
  std::vector<int> cand = p <= 128 ? std::vector<int>{7} : p <= 256 ? std::vector<int>{12, 9}
                        : p <= 512 ? std::vector<int>{10} : std::vector<int>{};
  if (const char* ev = std::getenv("OEM_LEAN_VARIANT")) {  // developer override (timing studies)
    const int f = std::atoi(ev);
    if (f >= 0 && f < 13 && KC_[f] * T_[f] >= p) cand = {f};
  }
  if (NPT > 4) return false;
  for (int v : cand)
    if (lean_layout_try(p, NPT, gstart, v, R_[v], KC_[v], T_[v], RS_[v], NTH_[v], lo)) return true;
  return false;
}

static bool lean_layout_try(int p, int NPT, const std::vector<int>& gstart, int v, int R, int KC, int T, int RS,
                            int NTH, LeanLayout& lo) {
  const int rows = (R + RS) * (NTH / T);
  // contiguous row blocks of <= rows rows, cut only at group starts (greedy packing)
  std::vector<int> cuts{0};
  if (gstart.empty()) {
    const int C = (p + rows - 1) / rows;
    for (int c = 1; c <= C; ++c) cuts.push_back((int)((int64_t)p * c / C));
  } else {
    std::vector<int> starts(gstart);
    std::sort(starts.begin(), starts.end());
    starts.push_back(p);
    int last = 0;  // last feasible cut candidate inside the current block
    for (size_t i = 1; i < starts.size(); ++i) {
      const int b = starts[i];
      if (b - cuts.back() > rows) {
        if (last <= cuts.back()) return false;  // a group larger than one CTA's rows
        cuts.push_back(last);
        if (b - cuts.back() > rows) return false;
      }
      last = b;
    }
    if (cuts.back() != p) cuts.push_back(p);
  }
  const int C = (int)cuts.size() - 1;
  if (C < 1 || C > 8) return false;
  lo.variant = v;
  lo.C = C;
  lo.rows = rows;
  lo.pvl = KC * T;
  lo.cuts = cuts;
  const int NV = NPT == 1 ? 1 : 2 * ((NPT + 1) / 2);
  lo.smem = ((size_t)2 * NV * lo.pvl + (size_t)RS * (NTH / T) * lo.pvl + (size_t)2 * C * (NTH / 32) +
             (size_t)NPT * rows + rows) * 8 +
            (size_t)2 * rows * 4 + 16;
  return true;
}

template <int NPT, int R, int KC, int T>
static oem_status launch_lean_t(const PathParams& P, const LeanArgs& A, int nU, size_t smem, cudaStream_t st) {
  auto kern = fit_lean_kernel<NPT, R, KC, T>;
  OEM_CUDA_TRY(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3((unsigned)(nU * A.C));
  cfg.blockDim = dim3(PT);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = (unsigned)A.C;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  OEM_CUDA_TRY(cudaLaunchKernelEx(&cfg, kern, P, A));
  return OEM_OK;
}

template <int NPT>
static oem_status launch_lean_t5(const PathParams& P, const LeanArgs& A, int nU, size_t smem, cudaStream_t st) {
  auto kern = fit_lean_kernel<NPT, 2, 16, 32, 2>;
  OEM_CUDA_TRY(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3((unsigned)(nU * A.C));
  cfg.blockDim = dim3(PT);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = (unsigned)A.C;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  OEM_CUDA_TRY(cudaLaunchKernelEx(&cfg, kern, P, A));
  return OEM_OK;
}

template <int NPT, int R, int KC, int T, int NTH, int RS = 0>
static oem_status launch_lean_nth(const PathParams& P, const LeanArgs& A, int nU, size_t smem, cudaStream_t st) {
  auto kern = fit_lean_kernel<NPT, R, KC, T, RS, NTH>;
  OEM_CUDA_TRY(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3((unsigned)(nU * A.C));
  cfg.blockDim = dim3(NTH);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = (unsigned)A.C;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  OEM_CUDA_TRY(cudaLaunchKernelEx(&cfg, kern, P, A));
  return OEM_OK;
}

template <int NPT>
static oem_status launch_lean_v(const PathParams& P, const LeanArgs& A, int nU, const LeanLayout& lo, cudaStream_t st) {
  if (lo.variant == 0) return launch_lean_t<NPT, 1, 8, 8>(P, A, nU, lo.smem, st);
  if (lo.variant == 1) return launch_lean_t<NPT, 2, 16, 8>(P, A, nU, lo.smem, st);
  if (lo.variant == 3) return launch_lean_t<NPT, 1, 8, 16>(P, A, nU, lo.smem, st);
  if (lo.variant == 4) return launch_lean_t<NPT, 1, 16, 16>(P, A, nU, lo.smem, st);
  if (lo.variant == 5) return launch_lean_t5<NPT>(P, A, nU, lo.smem, st);
  if (lo.variant == 6) return launch_lean_nth<NPT, 4, 16, 8, 256>(P, A, nU, lo.smem, st);
  if (lo.variant == 7) return launch_lean_nth<NPT, 2, 32, 4, 256>(P, A, nU, lo.smem, st);
  if (lo.variant == 8) return launch_lean_nth<NPT, 1, 32, 4, PT>(P, A, nU, lo.smem, st);
  if (lo.variant == 9) return launch_lean_nth<NPT, 4, 16, 16, 256>(P, A, nU, lo.smem, st);
  if (lo.variant == 10) return launch_lean_nth<NPT, 4, 16, 32, 256, 4>(P, A, nU, lo.smem, st);
  if (lo.variant == 11) return launch_lean_nth<NPT, 4, 16, 16, 256, 4>(P, A, nU, lo.smem, st);
  if (lo.variant == 12) return launch_lean_nth<NPT, 2, 16, 16, 256>(P, A, nU, lo.smem, st);
  return launch_lean_t<NPT, 2, 16, 16>(P, A, nU, lo.smem, st);
}

template <typename K>
static oem_status coop_launch(K kern, int grid, size_t smem, cudaStream_t st, void** args, int nth = PT) {
  OEM_CUDA_TRY(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  OEM_CUDA_TRY(cudaLaunchCooperativeKernel((const void*)kern, dim3(grid), dim3(nth), args, smem, st));
  return OEM_OK;
}

// ---------------------------------------------------------------- grid-wide lean solver: layout / launch
struct GlobLayout {
  int variant = -1;  // 0: R1 KC32 T32 (16 rows / CTA, p <= 1024), 1: R2 KC16 T32 (32 rows, p <= 512),
                     // 2: R1 RS1 KC32 T32 (16 register + 16 shared-memory rows, p <= 1024, split),
                     // 3: R2 RS2 KC32 T32 on 256 threads (the same 32 rows as 2)
  bool split = false;
  int nvu = 0;
  int C = 0, rows = 0, pvl = 0;
  size_t smem = 0;
  std::vector<int> cuts;
};

template <int NPT, int R, int KC, int T, int RS = 0, int NTH = PT>
static int glob_capacity(size_t smem, int num_sms) {
  int per = 0;
  if (cudaFuncSetAttribute(fit_glob_kernel<NPT, R, KC, T, RS, NTH>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                           (int)smem) != cudaSuccess ||
      cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, fit_glob_kernel<NPT, R, KC, T, RS, NTH>, NTH, smem) !=
          cudaSuccess)
    return 0;
  return per * num_sms;
}

// split = true: one virtual unit per (unit, penalty), NPT = 1, 32 rows per CTA (16 of them in
// shared memory for p > 512) so that nU * nP units stay co-resident.
static bool make_glob_layout(int nU, int p, int nP, const std::vector<int>& gstart, int num_sms, GlobLayout& lo,
                             bool split = false) {
  if (nP > 4 || p > 1024) return false;
  // split, p > 512: the 256-thread layout (measured at cfg4: variant 2 4.66 -> 3 4.36 us/iteration)
  int v = p <= 512 ? 1 : split ? 3 : 0;
  if (const char* ev = std::getenv("OEM_GLOB_VARIANT"))  // developer override (timing studies)
    if (split && p > 512 && std::atoi(ev) == 2) v = 2;
  const int rows = v == 0 ? 16 : 32, pvl = v == 1 ? 16 * 32 : 32 * 32, rs = v == 2 || v == 3 ? 16 : 0;
  const int nvu = split ? nU * nP : nU, NPTe = split ? 1 : nP;
  std::vector<int> cuts{0};
  if (gstart.empty()) {
    const int C = (p + rows - 1) / rows;
    for (int c = 1; c <= C; ++c) cuts.push_back((int)((int64_t)p * c / C));
  } else {
    std::vector<int> starts(gstart);
    std::sort(starts.begin(), starts.end());
    starts.push_back(p);
    int last = 0;
    for (size_t i = 1; i < starts.size(); ++i) {
      const int b = starts[i];
      if (b - cuts.back() > rows) {
        if (last <= cuts.back()) return false;
        cuts.push_back(last);
        if (b - cuts.back() > rows) return false;
      }
      last = b;
    }
    if (cuts.back() != p) cuts.push_back(p);
  }
  const int C = (int)cuts.size() - 1;
  const int NV = NPTe == 1 ? 1 : 2 * ((NPTe + 1) / 2);
  const size_t smem = ((size_t)2 * NV * pvl + (size_t)rs * pvl + (size_t)NPTe * rows + rows) * 8 +
                      (size_t)2 * rows * 4 + 16;
  int cap = 0;
  if (v == 3) {
    cap = glob_capacity<1, 2, 32, 32, 2, 256>(smem, num_sms);
  } else if (v == 2) {
    cap = glob_capacity<1, 1, 32, 32, 1>(smem, num_sms);
  } else if (v == 0) {
    cap = NPTe == 1 ? glob_capacity<1, 1, 32, 32>(smem, num_sms) : NPTe == 2 ? glob_capacity<2, 1, 32, 32>(smem, num_sms)
        : NPTe == 3 ? glob_capacity<3, 1, 32, 32>(smem, num_sms) : glob_capacity<4, 1, 32, 32>(smem, num_sms);
  } else {
    cap = NPTe == 1 ? glob_capacity<1, 2, 16, 32>(smem, num_sms) : NPTe == 2 ? glob_capacity<2, 2, 16, 32>(smem, num_sms)
        : NPTe == 3 ? glob_capacity<3, 2, 16, 32>(smem, num_sms) : glob_capacity<4, 2, 16, 32>(smem, num_sms);
  }
  if ((int64_t)nvu * C > cap) return false;
  lo.variant = v;
  lo.C = C;
  lo.rows = rows;
  lo.pvl = pvl;
  lo.smem = smem;
  lo.cuts = cuts;
  lo.split = split;
  lo.nvu = nvu;
  return true;
}

template <int NPT>
static oem_status launch_glob_v(const PathParams& P, const GlobArgs& A, int grid, const GlobLayout& lo, cudaStream_t st) {
  void* args[] = {const_cast<PathParams*>(&P), const_cast<GlobArgs*>(&A)};
  if (lo.variant == 0) return coop_launch(fit_glob_kernel<NPT, 1, 32, 32>, grid, lo.smem, st, args);
  if (lo.variant == 2) return coop_launch(fit_glob_kernel<1, 1, 32, 32, 1>, grid, lo.smem, st, args);
  if (lo.variant == 3) return coop_launch(fit_glob_kernel<1, 2, 32, 32, 2, 256>, grid, lo.smem, st, args, 256);
  return coop_launch(fit_glob_kernel<NPT, 2, 16, 32>, grid, lo.smem, st, args);
}

// ---------------------------------------------------------------- active-set solver: host layout / launch
struct ActLayout {
  int C = 0, rows = 0, amax = 0, apitch = 0, pw = 0, nth = 256, ncmax = 0;
  size_t smem = 0;
  std::vector<int> cuts;
};
// ncmax: capacity of the screened compact iterations (G_AA of up to ncmax active coordinates in
// CTA 0's shared memory), 0 without screening
static bool make_act_layout(int p, const std::vector<int>& gstart, ActLayout& lo, int nth, int ncmax = 0) {
  const int maxrows = nth / ACT_T;   // 64 or 128
  std::vector<int> cuts{0};
  if (gstart.empty()) {
    const int C = (p + maxrows - 1) / maxrows;
    for (int c = 1; c <= C; ++c) cuts.push_back((int)((int64_t)p * c / C));
  } else {   // cut only at group starts (greedy packing), as the lean layout
    std::vector<int> starts(gstart);
    std::sort(starts.begin(), starts.end());
    starts.push_back(p);
    int last = 0;
    for (size_t i = 1; i < starts.size(); ++i) {
      const int b = starts[i];
      if (b - cuts.back() > maxrows) {
        if (last <= cuts.back()) return false;
        cuts.push_back(last);
        if (b - cuts.back() > maxrows) return false;
      }
      last = b;
    }
    if (cuts.back() != p) cuts.push_back(p);
  }
  const int C = (int)cuts.size() - 1;
  if (C < 1 || C > 16) return false;
  int rows = 0;
  for (int c = 0; c < C; ++c) rows = std::max(rows, cuts[c + 1] - cuts[c]);
  lo.C = C;
  lo.nth = nth;
  lo.rows = rows;
  lo.cuts = cuts;
  lo.pw = (p + 31) / 32;
  const int pv = (p + 1) & ~1;
  lo.ncmax = ncmax;
  const size_t fixed = (size_t)2 * pv * 8 + (size_t)ncmax * ncmax * 8 + (size_t)9 * ncmax * 8 +
                       (size_t)rows * 8 * 3 + (size_t)rows * 4 * 2 + (size_t)p * 4 + (size_t)3 * lo.pw * 4 + 64;
  const size_t cap = 200 * 1024;
  if (fixed + (size_t)rows * 8 * 8 > cap) return false;
  int apitch = (int)std::min<size_t>((cap - fixed) / ((size_t)rows * 8), (size_t)p + 2);
  apitch -= (apitch % 2);   // keep rows 16-byte aligned
  lo.apitch = apitch;
  lo.amax = std::min(apitch, p);
  lo.smem = fixed + (size_t)rows * apitch * 8;
  return true;
}
template <int NTH>
static oem_status launch_active(const PathParams& P, const ActArgs& A, int nclusters, size_t smem, cudaStream_t st) {
  auto kern = fit_active_kernel<NTH>;
  OEM_CUDA_TRY(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  if (A.C > 8) OEM_CUDA_TRY(cudaFuncSetAttribute(kern, cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3((unsigned)(nclusters * A.C));
  cfg.blockDim = dim3(NTH);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = (unsigned)A.C;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  OEM_CUDA_TRY(cudaLaunchKernelEx(&cfg, kern, P, A));
  return OEM_OK;
}

// ---------------------------------------------------------------- host side
struct Layout {
  std::vector<int> unit, rank, ncta, j0, j1;
  int smem_rows = 0, ps = 0, T = 1, ncta_total = 0, Cmax = 1;
  size_t smem = 0;
};

// Split each unit's rows over C CTAs (cut at group boundaries) so the rows fit shared memory,
// and all nU*C CTAs are co-resident (cooperative launch, one CTA per SM).
static bool make_layout(int nU, int p, int NPT, const std::vector<int>& gstart, int num_sms, size_t smem_cap,
                        Layout& lo, std::string& why) {
  lo.ps = p + 2 - (p & 1);        // even pitch...
  if ((lo.ps % 16) == 0 || (lo.ps % 16) == 8) lo.ps += 2;  // ...not a multiple of 8 doubles
  auto bytes_for = [&](int rows) { return ((size_t)rows * lo.ps + (size_t)NPT * lo.ps + (size_t)NPT * rows) * 8; };
  int fit = 0;
  while (fit < p && bytes_for(fit + 1) <= smem_cap) ++fit;
  if (fit < 1) { why = "one row does not fit shared memory"; return false; }
  int C = (p + fit - 1) / fit;
  for (;;) {
    std::vector<int> cuts{0};
    for (int c = 1; c < C; ++c) {
      const int target = (int)((int64_t)p * c / C);
      int best = target;
      if (!gstart.empty()) {
        best = -1;
        for (int b : gstart)
          if (b > cuts.back() && b < p && (best < 0 || std::abs(b - target) < std::abs(best - target))) best = b;
        if (best < 0) break;
      }
      if (best > cuts.back() && best < p) cuts.push_back(best);
    }
    cuts.push_back(p);
    int maxrows = 0;
    for (size_t c = 0; c + 1 < cuts.size(); ++c) maxrows = std::max(maxrows, cuts[c + 1] - cuts[c]);
    if (bytes_for(maxrows) > smem_cap) {
      if (C >= p) { why = "rows do not fit shared memory"; return false; }
      ++C;
      continue;
    }
    C = (int)cuts.size() - 1;
    if ((int64_t)C * nU > num_sms) {
      why = "needs " + std::to_string((int64_t)C * nU) + " co-resident CTAs (> SM count)";
      return false;
    }
    lo.smem_rows = maxrows;
    lo.smem = bytes_for(maxrows) + 64 * 8;
    lo.Cmax = C;
    for (int u = 0; u < nU; ++u)
      for (int c = 0; c < C; ++c) {
        lo.unit.push_back(u);
        lo.rank.push_back(c);
        lo.j0.push_back(cuts[c]);
        lo.j1.push_back(cuts[c + 1]);
      }
    lo.ncta.assign(nU, C);
    lo.ncta_total = nU * C;
    int T = 1;
    while (T < 32 && PT / (T * 2) >= maxrows) T *= 2;
    lo.T = T;
    return true;
  }
}

}  // namespace oem

using namespace oem;

extern "C" void oem_path_cfg_default(oem_path_cfg* cfg) {
  if (!cfg) return;
  cfg->nlambda = 100;
  cfg->lambda_min_ratio = 1e-3;
  cfg->lambda = nullptr;
  cfg->tol = 1e-11;
  cfg->maxit = 100000;
  cfg->var_w = nullptr;
  cfg->group = nullptr;
  cfg->ngroups = 0;
  cfg->grp_w = nullptr;
  cfg->d_squarings = 12;
  cfg->fold_mode = 0;
  cfg->lambda_max_override = nullptr;
  cfg->standardize = 0;
  cfg->xsum = nullptr;
  cfg->ysum = nullptr;
  cfg->intercept_out = nullptr;
}


static int ereg_for(int NPT) { return NPT <= 1 ? 32 : NPT == 2 ? 24 : NPT == 4 ? 16 : 8; }

extern "C" oem_status oem_fit_path(oem_ctx* ctx, const double* G, const double* xty, const int64_t* counts,
                                   int32_t nG, int32_t p, const oem_penalty* pens, int32_t nP,
                                   const oem_path_cfg* cfg_in, const double* d_in, const double* beta_init,
                                   double* beta_out, double* lambda_out, int64_t* iters_out, uint8_t* converged_out,
                                   double* d_out, void* stream) {
  if (!ctx) OEM_FAIL(OEM_ERR_INVALID_ARG, "null oem_ctx");
  OEM_CUDA_TRY(cudaSetDevice(ctx->device));
  oem_path_cfg cfg;
  if (cfg_in) cfg = *cfg_in;
  else oem_path_cfg_default(&cfg);
  cudaStream_t st = (cudaStream_t)stream;
  if (!G || !xty || !counts || !pens || !beta_out || !lambda_out || !iters_out || !converged_out || !d_out)
    OEM_FAIL(OEM_ERR_INVALID_ARG, "oem_fit_path: null pointer");
  if (p < 1 || nG < 1) OEM_FAIL(OEM_ERR_DIM, "oem_fit_path: need p >= 1, nG >= 1");
  if (p > 16383) OEM_FAIL(OEM_ERR_UNSUPPORTED, "oem_fit_path: p > 16383");
  if (nP < 1 || nP > 8) OEM_FAIL(OEM_ERR_INVALID_ARG, "oem_fit_path: 1 <= nP <= 8 penalties per call");
  if (cfg.nlambda < 1) OEM_FAIL(OEM_ERR_INVALID_ARG, "oem_fit_path: nlambda < 1");
  if (!cfg.lambda && !(cfg.lambda_min_ratio > 0.0 && cfg.lambda_min_ratio < 1.0) && cfg.nlambda > 1)
    OEM_FAIL(OEM_ERR_INVALID_ARG, "oem_fit_path: need 0 < lambda_min_ratio < 1");
  if (!(cfg.tol > 0.0) || cfg.maxit < 1) OEM_FAIL(OEM_ERR_INVALID_ARG, "oem_fit_path: need tol > 0, maxit >= 1");
  if (cfg.maxit > 2000000000LL) cfg.maxit = 2000000000LL;
  if (cfg.d_squarings < 0 || cfg.d_squarings > 60) OEM_FAIL(OEM_ERR_INVALID_ARG, "oem_fit_path: need 0 <= d_squarings <= 60");
  const int fold = cfg.fold_mode ? 1 : 0;
  const int nU = fold ? nG + 1 : nG;
  const int L = cfg.nlambda;
  bool any_grp = false;
  for (int q = 0; q < nP; ++q) {
    const int f = pens[q].family;
    if (f < OEM_LASSO || f > OEM_SGL) OEM_FAIL(OEM_ERR_INVALID_ARG, "oem_fit_path: unknown penalty family");
    if (f == OEM_SGL && !(pens[q].alpha >= 0.0 && pens[q].alpha <= 1.0))
      OEM_FAIL(OEM_ERR_INVALID_ARG, "oem_fit_path: sparse group lasso tau (alpha field) outside [0,1]");
    if (f >= OEM_GRP_LASSO) any_grp = true;
    if (f == OEM_ENET && !(pens[q].alpha >= 0.0 && pens[q].alpha <= 1.0))
      OEM_FAIL(OEM_ERR_INVALID_ARG, "oem_fit_path: elastic-net alpha outside [0,1]");
    if ((f == OEM_MCP || f == OEM_GRP_MCP) && !(pens[q].gamma > 1.0)) OEM_FAIL(OEM_ERR_INVALID_ARG, "MCP needs gamma > 1");
    if ((f == OEM_SCAD || f == OEM_GRP_SCAD) && !(pens[q].gamma > 2.0)) OEM_FAIL(OEM_ERR_INVALID_ARG, "SCAD needs gamma > 2");
  }
  if (any_grp && (!cfg.group || cfg.ngroups < 1)) OEM_FAIL(OEM_ERR_INVALID_ARG, "group penalties need cfg.group");
  // normalisers (R#1, R#20)
  std::vector<double> inv_n(nU);
  {
    int64_t tot = 0;
    for (int g = 0; g < nG; ++g) {
      if (counts[g] <= 0) OEM_FAIL(OEM_ERR_EMPTY_FOLD, "oem_fit_path: count " + std::to_string(g) + " is 0");
      tot += counts[g];
    }
    for (int u = 0; u < nU; ++u) {
      int64_t nn = !fold ? counts[u] : (u == 0 ? tot : tot - counts[u - 1]);
      if (nn <= 0) OEM_FAIL(OEM_ERR_EMPTY_FOLD, "oem_fit_path: empty training set");
      inv_n[u] = 1.0 / (double)nn;
    }
  }
  // groups -> permutation making them contiguous (stable by id)
  std::vector<int> perm(p), gstart, gend, g_of_perm;
  std::vector<double> gw;
  std::iota(perm.begin(), perm.end(), 0);
  if (cfg.group) {
    for (int j = 0; j < p; ++j)
      if (cfg.group[j] < 0 || cfg.group[j] >= cfg.ngroups) OEM_FAIL(OEM_ERR_INVALID_ARG, "group id out of range");
    if (cfg.ngroups > MAXG) OEM_FAIL(OEM_ERR_UNSUPPORTED, "more than 4096 groups");
    std::stable_sort(perm.begin(), perm.end(), [&](int a, int b) { return cfg.group[a] < cfg.group[b]; });
    gstart.assign(cfg.ngroups, 0);
    gend.assign(cfg.ngroups, 0);
    g_of_perm.assign(p, 0);
    std::vector<int> size(cfg.ngroups, 0);
    for (int j = 0; j < p; ++j) size[cfg.group[j]]++;
    int s = 0;
    for (int g = 0; g < cfg.ngroups; ++g) { gstart[g] = s; s += size[g]; gend[g] = s; }
    for (int j = 0; j < p; ++j) g_of_perm[j] = cfg.group[perm[j]];
    gw.resize(cfg.ngroups);
    for (int g = 0; g < cfg.ngroups; ++g) {
      gw[g] = cfg.grp_w ? cfg.grp_w[g] : std::sqrt((double)size[g]);  // R#12
      if (!(gw[g] >= 0.0) || !std::isfinite(gw[g])) OEM_FAIL(OEM_ERR_INVALID_ARG, "group weight must be >= 0");
    }
  }
  const int NPT = nP <= 1 ? 1 : nP <= 2 ? 2 : nP <= 4 ? 4 : 8;
  // ---- solver layout: a thread-block cluster per unit when the rows fit on-chip (C <= 16),
  // else the cooperative global-barrier solver
  const char* force = std::getenv("OEM_PATH_SOLVER");
  ClusterLayout cl;
  Layout lo;
  LeanLayout ll;
  // active-set clusters with screened compact iterations (tall-data paths are sparse) for p > 256
  // and p <= 128; the register-resident lean clusters for 128 < p <= 256, whose 32-row CTAs make
  // a full iteration cheap (measured, B200: the sparse workload's p = 200 paths, ~6 iterations per
  // lambda, 1.41 ms lean vs 3.64 ms screened; cfg5's inner solves 39.8 vs 37.6 ms; cfg2, p = 100,
  // 6.65 ms lean vs 4.70 ms screened). Without screening (OEM_SCREEN=0, timing studies) the
  // active-set clusters for p > 256 and the lean clusters below. OEM_PATH_SOLVER=active / lean /
  // global / cluster / batched forces a variant (tests, timing studies)
  const char* scr = std::getenv("OEM_SCREEN");
  const int ncmax = (scr && std::string(scr) == "0") ? 0 : (scr && std::string(scr) == "32") ? 32 : 64;
  ActLayout al;
  const std::string fs = force ? std::string(force) : std::string();
  // (128-row CTAs when that gives a smaller cluster: fewer CTAs meet at each barrier)
  const bool want_act = fs == "active" || (fs.empty() && (p > 256 || (ncmax > 0 && p <= 128)));
  const std::vector<int> gs_act = any_grp ? gstart : std::vector<int>();
  ActLayout al128;
  const char* ath = std::getenv("OEM_ACT_THREADS");   // developer override (timing studies): 256 / 512
  const int force_th = ath ? std::atoi(ath) : 0;
  // (256-thread CTAs hold up to 128 compact rows, 4 per lane, when p <= 256)
  const int ncmax256 = (ncmax == 64 && p <= 256 && p > 64) ? 128 : ncmax;
  const bool act256 = want_act && force_th != 512 &&
                      (make_act_layout(p, gs_act, al, 256, ncmax256) || make_act_layout(p, gs_act, al, 256, ncmax));
  const bool act512 =
      want_act && (p > 512 || force_th == 512) && force_th != 256 && make_act_layout(p, gs_act, al128, 512, ncmax);
  if (act512 && (!act256 || al128.C < al.C)) al = al128;
  const bool use_act = act256 || act512;
  const bool use_lean = !use_act && !(fs == "global" || fs == "cluster") &&
                        make_lean_layout(p, nP, any_grp ? gstart : std::vector<int>(), ll);
  GlobLayout gl;
  const bool glob_ok = !use_act && !use_lean && !(force && (std::string(force) == "global" || std::string(force) == "cluster"));
  const bool use_glob =
      glob_ok && ((nP > 1 && !(force && std::string(force) == "batched") &&
                   make_glob_layout(nU, p, nP, any_grp ? gstart : std::vector<int>(), ctx->num_sms, gl, true)) ||
                  make_glob_layout(nU, p, nP, any_grp ? gstart : std::vector<int>(), ctx->num_sms, gl, false));
  bool use_cluster = !use_act && !use_lean && !use_glob && !(force && std::string(force) == "global") &&
                     make_cluster_layout(nU, p, NPT, any_grp ? gstart : std::vector<int>(), ctx->num_sms,
                                         ereg_for(NPT), cl);
  std::string why;
  if (!use_act && !use_lean && !use_glob && !use_cluster &&
      !make_layout(nU, p, NPT, any_grp ? gstart : std::vector<int>(), ctx->num_sms, 200 * 1024, lo, why))
    OEM_FAIL(OEM_ERR_UNSUPPORTED, "oem_fit_path: persistent solver layout: " + why);
  // penalty split: with SMs to spare, each (unit, penalty) gets its own cluster (NPT = 1: no
  // cross-penalty divergence, and each penalty stops when its own path ends)
  LeanLayout ll1;
  const bool qsplit = use_lean && nP > 1 && !(force && std::string(force) == "batched") &&
                      make_lean_layout(p, 1, any_grp ? gstart : std::vector<int>(), ll1) &&
                      (int64_t)nU * nP * ll1.C <= ctx->num_sms;
  if (qsplit) ll = ll1;
  std::vector<int> t_unit, t_rank, t_ncta, t_j0, t_j1;
  if (use_act) {
    for (int u = 0; u < nU; ++u)
      for (int q = 0; q < nP; ++q)
        for (int c = 0; c < al.C; ++c) {
          t_unit.push_back(u); t_rank.push_back(c); t_j0.push_back(al.cuts[c]); t_j1.push_back(al.cuts[c + 1]);
        }
    t_ncta.assign(nU, al.C);
  } else if (use_lean) {
    for (int u = 0; u < nU; ++u)
      for (int q = 0; q < (qsplit ? nP : 1); ++q)
        for (int c = 0; c < ll.C; ++c) {
          t_unit.push_back(u); t_rank.push_back(c); t_j0.push_back(ll.cuts[c]); t_j1.push_back(ll.cuts[c + 1]);
        }
    t_ncta.assign(nU, ll.C);
  } else if (use_glob) {
    for (int u = 0; u < gl.nvu; ++u)  // virtual units (unit, or (unit, penalty) when split)
      for (int c = 0; c < gl.C; ++c) {
        t_unit.push_back(u); t_rank.push_back(c); t_j0.push_back(gl.cuts[c]); t_j1.push_back(gl.cuts[c + 1]);
      }
    t_ncta.assign(gl.nvu, gl.C);
  } else if (use_cluster) {
    for (int u = 0; u < nU; ++u)
      for (int c = 0; c < cl.C; ++c) { t_unit.push_back(u); t_rank.push_back(c); }
    t_ncta.assign(nU, cl.C);
    t_j0 = cl.j0;
    t_j1 = cl.j1;
  } else {
    t_unit = lo.unit; t_rank = lo.rank; t_ncta = lo.ncta; t_j0 = lo.j0; t_j1 = lo.j1;
  }
  const int ncta_total = (int)t_unit.size();
  if (any_grp) {
    for (size_t i = 0; i < t_j0.size(); ++i)
      for (int g = 0; g < cfg.ngroups; ++g)
        if (gstart[g] < t_j0[i] && gend[g] > t_j0[i])
          OEM_FAIL(OEM_ERR_UNSUPPORTED, "oem_fit_path: a group is larger than one solver CTA's rows");
  }
  const int Cmax = use_act ? al.C : use_lean ? ll.C : use_glob ? gl.C : use_cluster ? cl.C : lo.Cmax;
  // ---- workspace (device)
  const size_t pp = (size_t)p * p;
  size_t off = 0;
  auto take = [&](size_t bytes) { size_t o = off; off += (bytes + 255) / 256 * 256; return o; };
  const size_t o_Gn = take(sizeof(double) * nU * pp);
  const size_t o_cn = take(sizeof(double) * nU * p);
  const size_t o_bbuf = take(sizeof(double) * 2 * nU * nP * p);
  const size_t o_bad = take(sizeof(unsigned long long) * nU);
  const size_t o_dslot = take(sizeof(unsigned long long) * 3 * nU * nP);
  const int nvu_ws = use_glob ? std::max(nU, gl.nvu) : nU;  // virtual units (grid solver split)
  const size_t o_bar = take(sizeof(unsigned) * 2 * nvu_ws);
  const size_t o_flags = take(sizeof(int) * 4);
  const size_t o_invn = take(sizeof(double) * nU);
  const size_t o_perm = take(sizeof(int) * p);
  const size_t o_gof = take(sizeof(int) * p);
  const size_t o_gs = take(sizeof(int) * std::max<size_t>(1, gstart.size()));
  const size_t o_ge = take(sizeof(int) * std::max<size_t>(1, gend.size()));
  const size_t o_gw = take(sizeof(double) * std::max<size_t>(1, gw.size()));
  const size_t o_varw = take(sizeof(double) * p);
  const size_t o_fam = take(sizeof(int) * nP);
  const size_t o_gam = take(sizeof(double) * nP);
  const size_t o_alp = take(sizeof(double) * nP);
  const size_t o_lam = take(sizeof(double) * L);
  const size_t o_lmax = take(sizeof(double));
  const size_t o_cu = take(sizeof(int) * ncta_total);
  const size_t o_cr = take(sizeof(int) * ncta_total);
  const size_t o_un = take(sizeof(int) * nvu_ws);
  const size_t o_j0 = take(sizeof(int) * ncta_total);
  const size_t o_j1 = take(sizeof(int) * ncta_total);
  const size_t o_d = take(sizeof(double) * nU);
  const int gNV = nP == 1 ? 1 : 2 * ((nP + 1) / 2);
  const int gNVe = (use_glob && gl.split) ? 1 : gNV;
  const size_t o_gvec = take(use_glob ? sizeof(double) * 2 * (size_t)nvu_ws * gNVe * gl.pvl : 8);
  const size_t o_gflag = take(use_glob ? sizeof(unsigned long long) * 2 * (size_t)nvu_ws * Cmax : 8);
  const size_t o_gslot = take(use_glob ? sizeof(double) * 2 * (size_t)nvu_ws * Cmax : 8);
  const bool centre = cfg.xsum != nullptr || cfg.ysum != nullptr;
  const bool xform = centre || cfg.standardize;
  if (centre && !(cfg.xsum && cfg.ysum)) OEM_FAIL(OEM_ERR_INVALID_ARG, "oem_fit_path: intercept needs both xsum and ysum");
  const size_t o_mean = take(sizeof(double) * (xform ? (size_t)nU * p : 1));
  const size_t o_ybar = take(sizeof(double) * nU);
  const size_t o_invs = take(sizeof(double) * (xform ? (size_t)nU * p : 1));
  const size_t o_host_end = off;
  OEM_CUDA_TRY(ctx->path_ws.ensure(off));
  char* base = ctx->path_ws.as<char>();
  std::vector<char> hb(o_host_end - o_invn, 0);
  auto put = [&](size_t o, const void* src, size_t bytes) { if (bytes) std::memcpy(hb.data() + (o - o_invn), src, bytes); };
  put(o_invn, inv_n.data(), sizeof(double) * nU);
  put(o_perm, perm.data(), sizeof(int) * p);
  if (cfg.group) {
    put(o_gof, g_of_perm.data(), sizeof(int) * p);
    put(o_gs, gstart.data(), sizeof(int) * gstart.size());
    put(o_ge, gend.data(), sizeof(int) * gend.size());
    put(o_gw, gw.data(), sizeof(double) * gw.size());
  }
  std::vector<int> fam(nP);
  std::vector<double> gam(nP), alp(nP);
  for (int q = 0; q < nP; ++q) { fam[q] = pens[q].family; gam[q] = pens[q].gamma; alp[q] = pens[q].alpha; }
  put(o_fam, fam.data(), sizeof(int) * nP);
  put(o_gam, gam.data(), sizeof(double) * nP);
  put(o_alp, alp.data(), sizeof(double) * nP);
  if (cfg.lambda) put(o_lam, cfg.lambda, sizeof(double) * L);
  if (cfg.lambda_max_override) put(o_lmax, cfg.lambda_max_override, sizeof(double));
  put(o_cu, t_unit.data(), sizeof(int) * ncta_total);
  put(o_cr, t_rank.data(), sizeof(int) * ncta_total);
  put(o_un, t_ncta.data(), sizeof(int) * t_ncta.size());
  put(o_j0, t_j0.data(), sizeof(int) * ncta_total);
  put(o_j1, t_j1.data(), sizeof(int) * ncta_total);
  if (d_in) put(o_d, d_in, sizeof(double) * nU);
  if (cfg.var_w) {
    std::vector<double> tmp(p), wp(p);
    OEM_CUDA_TRY(cudaMemcpyAsync(tmp.data(), cfg.var_w, sizeof(double) * p, cudaMemcpyDeviceToHost, st));
    OEM_CUDA_TRY(cudaStreamSynchronize(st));
    for (int j = 0; j < p; ++j) {
      wp[j] = tmp[perm[j]];
      if (!(wp[j] >= 0.0) || !std::isfinite(wp[j])) OEM_FAIL(OEM_ERR_INVALID_ARG, "variable weights must be >= 0");
    }
    put(o_varw, wp.data(), sizeof(double) * p);
  }
  OEM_CUDA_TRY(cudaMemcpyAsync(base + o_invn, hb.data(), hb.size(), cudaMemcpyHostToDevice, st));
  OEM_CUDA_TRY(cudaMemsetAsync(base + o_dslot, 0, (o_invn - o_dslot), st));  // dslot, bar, flags
  OEM_CUDA_TRY(cudaMemsetAsync(base + o_bad, 0xff, sizeof(unsigned long long) * nU, st));
  double* Gn = reinterpret_cast<double*>(base + o_Gn);
  double* cn = reinterpret_cast<double*>(base + o_cn);
  int* flags = reinterpret_cast<int*>(base + o_flags);
  // ---- a6 normalise (+ fold complements, + permutation)
  {
    const int64_t total = (int64_t)nU * ((int64_t)pp + p);
    const int blocks = (int)std::max<int64_t>(1, std::min<int64_t>(ctx->num_sms * 8, (total + 255) / 256));
    PhaseTimer tm(ctx, PH_PATH, st);
    ++ctx->launches;
    if (xform) {
      ++ctx->launches;
      unit_stats_kernel<<<nU, 256, 0, st>>>(G, cfg.xsum, cfg.ysum, nG, p, fold, reinterpret_cast<double*>(base + o_invn),
                                             cfg.standardize ? 1 : 0, reinterpret_cast<double*>(base + o_mean),
                                             reinterpret_cast<double*>(base + o_ybar), reinterpret_cast<double*>(base + o_invs));
      OEM_CUDA_TRY(cudaGetLastError());
    }
    prep_units_kernel<<<blocks, 256, 0, st>>>(G, xty, nG, p, fold, reinterpret_cast<double*>(base + o_invn),
                                              reinterpret_cast<int*>(base + o_perm),
                                              xform ? reinterpret_cast<double*>(base + o_mean) : nullptr,
                                              reinterpret_cast<double*>(base + o_ybar),
                                              reinterpret_cast<double*>(base + o_invs), Gn, cn, flags);
    OEM_CUDA_TRY(cudaGetLastError());
  }
  PathParams P;
  std::memset(&P, 0, sizeof(P));
  P.p = p; P.nP = nP; P.L = L; P.nU = nU; P.maxit = cfg.maxit; P.tol = cfg.tol;
  P.Gn = Gn; P.cn = cn;
  P.cta_unit = reinterpret_cast<int*>(base + o_cu);
  P.cta_rank = reinterpret_cast<int*>(base + o_cr);
  P.unit_ncta = reinterpret_cast<int*>(base + o_un);
  P.cta_j0 = reinterpret_cast<int*>(base + o_j0);
  P.cta_j1 = reinterpret_cast<int*>(base + o_j1);
  P.fam = reinterpret_cast<int*>(base + o_fam);
  P.gam = reinterpret_cast<double*>(base + o_gam);
  P.alp = reinterpret_cast<double*>(base + o_alp);
  P.var_w = cfg.var_w ? reinterpret_cast<double*>(base + o_varw) : nullptr;
  P.ngroups = cfg.group ? cfg.ngroups : 0;
  P.g_start = reinterpret_cast<int*>(base + o_gs);
  P.g_end = reinterpret_cast<int*>(base + o_ge);
  P.g_w = reinterpret_cast<double*>(base + o_gw);
  P.g_of = any_grp ? reinterpret_cast<int*>(base + o_gof) : nullptr;
  P.perm = reinterpret_cast<int*>(base + o_perm);
  P.lam_explicit = cfg.lambda ? reinterpret_cast<double*>(base + o_lam) : nullptr;
  P.lmin_ratio = cfg.lambda_min_ratio;
  P.shared_grid = fold;
  P.lmax_override = cfg.lambda_max_override ? reinterpret_cast<double*>(base + o_lmax) : nullptr;
  P.d = reinterpret_cast<double*>(base + o_d);
  P.beta_init = beta_init;
  P.bbuf = reinterpret_cast<double*>(base + o_bbuf);
  P.dslot = reinterpret_cast<unsigned long long*>(base + o_dslot);
  P.bar = reinterpret_cast<unsigned*>(base + o_bar);
  P.beta_out = beta_out; P.lam_out = lambda_out; P.it_out = iters_out; P.cv_out = converged_out;
  P.flags = flags;
  P.bad_iter = reinterpret_cast<unsigned long long*>(base + o_bad);
  double* dptr = reinterpret_cast<double*>(base + o_d);
  // ---- a7 d per unit (R#5) unless given: one cooperative launch over all units (drule.cu)
  if (!d_in) {
    oem_status s = d_rule(ctx, Gn, nU, p, cfg.d_squarings, dptr, st);
    if (s != OEM_OK) return s;
  }
  if (use_glob) {
    // ---- a7-a10 fused in one cooperative launch: register-resident G, C CTAs per unit over L2
    P.ps = 0; P.T = 0; P.smem_rows = 0;
    GlobArgs A;
    A.Cmax = Cmax; A.rows = gl.rows; A.pvl = gl.pvl; A.qsplit = gl.split ? 1 : 0; A.nvu = gl.nvu;
    A.gvec = reinterpret_cast<double*>(base + o_gvec);
    A.gflag = reinterpret_cast<unsigned long long*>(base + o_gflag);
    OEM_CUDA_TRY(cudaMemsetAsync(A.gflag, 0, sizeof(unsigned long long) * 2 * (size_t)nvu_ws * Cmax, st));
    A.gslot = reinterpret_cast<double*>(base + o_gslot);
    A.gcnt = reinterpret_cast<unsigned*>(base + o_bar);   // zeroed with dslot / bar / flags
    PhaseTimer tm(ctx, PH_PATH, st);
    ++ctx->launches;
    oem_status s;
    const int grid = gl.nvu * gl.C;
    if (gl.split) s = launch_glob_v<1>(P, A, grid, gl, st);
    else if (nP == 1) s = launch_glob_v<1>(P, A, grid, gl, st);
    else if (nP == 2) s = launch_glob_v<2>(P, A, grid, gl, st);
    else if (nP == 3) s = launch_glob_v<3>(P, A, grid, gl, st);
    else s = launch_glob_v<4>(P, A, grid, gl, st);
    if (s != OEM_OK) return s;
  } else if (use_act) {
    // ---- a8-a10 in one launch: an active-set cluster per (unit, penalty)
    P.ps = 0; P.T = 0; P.smem_rows = 0;
    ActArgs A;
    A.C = al.C; A.amax = al.amax; A.apitch = al.apitch; A.rows = al.rows; A.pw = al.pw;
    A.screen = al.ncmax > 0 ? 1 : 0; A.ncmax = al.ncmax;
    PhaseTimer tm(ctx, PH_PATH, st);
    ++ctx->launches;
    oem_status s = al.nth == 512 ? launch_active<512>(P, A, nU * nP, al.smem, st)
                                 : launch_active<256>(P, A, nU * nP, al.smem, st);
    if (s != OEM_OK) return s;
  } else if (use_lean) {
    // ---- a7-a10 fused in one launch: register-resident G, one cluster per unit
    P.ps = 0; P.T = 0; P.smem_rows = 0;
    LeanArgs A;
    A.C = ll.C; A.rows = ll.rows; A.pvl = ll.pvl; A.qsplit = qsplit ? 1 : 0;
    PhaseTimer tm(ctx, PH_PATH, st);
    ++ctx->launches;
    oem_status s;
    if (qsplit) s = launch_lean_v<1>(P, A, nU * nP, ll, st);
    else if (nP == 1) s = launch_lean_v<1>(P, A, nU, ll, st);
    else if (nP == 2) s = launch_lean_v<2>(P, A, nU, ll, st);
    else if (nP == 3) s = launch_lean_v<3>(P, A, nU, ll, st);
    else s = launch_lean_v<4>(P, A, nU, ll, st);
    if (s != OEM_OK) return s;
  } else if (use_cluster) {
    // ---- a7-a10 fused in one cluster launch (d, lambda grid, paths)
    P.ps = 0; P.T = cl.T; P.smem_rows = 0;
    ClusterArgs A;
    A.C = cl.C; A.T = cl.T; A.RG = cl.RG; A.KPR = cl.KPR; A.NRT = cl.NRT; A.S = cl.S; A.pv = cl.pv;
    A.maxrows = cl.maxrows;
    PhaseTimer tm(ctx, PH_PATH, st);
    ++ctx->launches;
    oem_status s;
    if (NPT == 1) s = launch_cluster<1>(P, A, nU, cl.smem, st);
    else if (NPT == 2) s = launch_cluster<2>(P, A, nU, cl.smem, st);
    else if (NPT == 4) s = launch_cluster<4>(P, A, nU, cl.smem, st);
    else s = launch_cluster<8>(P, A, nU, cl.smem, st);
    if (s != OEM_OK) return s;
  } else {
    P.ps = lo.ps; P.T = lo.T; P.smem_rows = lo.smem_rows;
    // ---- a8-a10 lambda grid + OEM paths
    void* args[] = {&P};
    PhaseTimer tm(ctx, PH_PATH, st);
    ++ctx->launches;
    oem_status s;
    if (NPT == 1) s = coop_launch(path_kernel<1>, lo.ncta_total, lo.smem, st, args);
    else if (NPT == 2) s = coop_launch(path_kernel<2>, lo.ncta_total, lo.smem, st, args);
    else if (NPT == 4) s = coop_launch(path_kernel<4>, lo.ncta_total, lo.smem, st, args);
    else s = coop_launch(path_kernel<8>, lo.ncta_total, lo.smem, st, args);
    if (s != OEM_OK) return s;
  }
  if (xform) {
    const int warps = nU * nP * L;
    ++ctx->launches;
    backtransform_kernel<<<(warps * 32 + 255) / 256, 256, 0, st>>>(
        beta_out, nU, nP, L, p, reinterpret_cast<double*>(base + o_mean), reinterpret_cast<double*>(base + o_ybar),
        reinterpret_cast<double*>(base + o_invs), centre ? cfg.intercept_out : nullptr);
    OEM_CUDA_TRY(cudaGetLastError());
  } else if (cfg.intercept_out) {
    OEM_CUDA_TRY(cudaMemsetAsync(cfg.intercept_out, 0, sizeof(double) * (size_t)nU * nP * L, st));
  }
  OEM_CUDA_TRY(cudaMemcpyAsync(d_out, dptr, sizeof(double) * nU, cudaMemcpyDeviceToDevice, st));
  int hflags[4] = {0, 0, 0, 0};
  OEM_CUDA_TRY(cudaMemcpyAsync(hflags, flags, sizeof(hflags), cudaMemcpyDeviceToHost, st));
  OEM_CUDA_TRY(cudaStreamSynchronize(st));
  if (hflags[0]) OEM_FAIL(OEM_ERR_NONFINITE, "oem_fit_path: non-finite value in the Gram or the iterates");
  if (hflags[1])
    OEM_FAIL(OEM_ERR_INVALID_ARG, "oem_fit_path: MCP needs gamma*d > 1 and SCAD (gamma-1)*d > 1 for the d in use (R#8)");
  return OEM_OK;
}
