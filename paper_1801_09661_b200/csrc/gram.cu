// gram.cu — K2/K3/K7: the Gram pass of OEM on sm_100a.
//
// What it computes: the sufficient statistics X^T X, X^T y,
// y^T y of the linear model as ONE symmetric rank-n update of the augmented matrix Z = [X | y]
// (upper triangle of Z^T Z only), optionally split by fold (fold(i) = (off+i) mod K)
// or weighted by the proximal-Newton weights with the working response in the augmented
// column (w_i = mu(1-mu), z_i = eta + (y - mu)/w, eta = x_i^T beta).
//
// How (B200-first):
//  * Row blocks of X (BK = 32 rows) stream HBM -> shared memory through TMA
//    (cp.async.bulk.tensor, mbarrier complete_tx) in a multi-stage ring fed by one producer
//    warp; y (or y01) rides along as an extra column filled by the producer's lanes.
//  * The contraction runs on the FP64 tensor cores: mma.sync m8n8k4 f64 (SASS DMMA.8x8x4;
//    tcgen05 has no f64 kind on sm_100a). Each consumer warp owns a rectangle of R x C 8x8
//    output blocks of the upper triangle with register accumulators; blocks below the
//    diagonal are skipped. The smem row pitch is ld = 4 or 12 (mod 16) doubles so the
//    fragment loads (4 rows x 8 columns per half-warp pair) are bank-conflict free.
//  * Small p (p+1 <= 248): the whole augmented row fits one TMA box ("single panel"); the
//    triangle's rectangles are spread over U CTA types that all stream the same rows
//    (the weighted pass computes eta/w/z per row from the full row in smem, fused).
//    Large p: 128-column panel pairs (I, J), I <= J, one CTA type per tile, 4x8 rectangles.
//  * Rows are split into segments (split-n); every (CTA type, segment) writes its own
//    partial blocks and a second kernel sums segments in a fixed order -> deterministic,
//    no atomics. The result is packed (upper triangle of the augmented matrix) for a single
//    NCCL allreduce when the rows are sharded over GPUs.
#include <algorithm>
#include <cstring>
#include <vector>

#include "common.cuh"
#include "internal.h"

namespace oem {

constexpr int BK = 32;      // rows per pipeline stage
constexpr int MAXST = 6;    // max pipeline stages
constexpr int MAXNW = 12;   // max consumer warps

struct RectDesc {
  int32_t bi0, bj0;   // top-left 8x8 block (global block coordinates)
  uint32_t mask;      // active blocks, bit r*C + c  (block (bi0+r, bj0+c) with bi <= bj < nb)
  int32_t pad;
};
struct CtaDesc {
  int32_t a0, b0;     // first column of panel A / panel B
  int32_t same;       // panel B == panel A
  int32_t nrect;
  RectDesc rect[MAXNW];
};

struct GramParams {
  int p, nb, ld, U, nseg, ST, two_panel, nblk;
  int64_t nrows;      // PLAIN/WEIGHTED: n_local rows; FOLD: nq = floor(n_local / K) full groups
  int64_t seg_rows;   // rows (FOLD: groups) per segment, multiple of BK
  int K, off_mod;     // FOLD
  const double* y;
  const double* beta;
  double eps;
  double* partial;        // [nfold][nseg][nblk][64]
  double* partial_scal;   // WEIGHTED: [nseg][2]
  const CtaDesc* ctas;
  const int32_t* blk_of;  // [nb*nb] -> packed upper block index or -1
  uint32_t tma_bytes;     // bytes of one TMA box (one per panel per stage)
  int stage_doubles;      // per-stage smem footprint (doubles)
};

template <int R, int C, int NW, int MODE>
__global__ void __launch_bounds__((NW + 1) * 32, 1)
gram_kernel(const __grid_constant__ CUtensorMap tmX, const GramParams P) {
  extern __shared__ __align__(128) double smem[];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int u = blockIdx.x % P.U;
  const int rest = blockIdx.x / P.U;
  const int seg = rest % P.nseg;
  const int fold = rest / P.nseg;  // 0 unless MODE_FOLD
  const int ld = P.ld;

  double* beta_s = smem + (size_t)P.ST * P.stage_doubles;                       // WEIGHTED: ld doubles
  uint64_t* full = reinterpret_cast<uint64_t*>(beta_s + (MODE == MODE_WEIGHTED ? ld : 0));
  uint64_t* empty = full + MAXST;
  __shared__ double scal_s[MAXNW][2];

  const int64_t r0 = (int64_t)seg * P.seg_rows;
  const int64_t r1 = min(P.nrows, r0 + P.seg_rows);
  const int nst = r1 > r0 ? (int)((r1 - r0 + BK - 1) / BK) : 0;
  const int kprime = (MODE == MODE_FOLD) ? ((fold - P.off_mod) % P.K + P.K) % P.K : 0;

  const CtaDesc* cd = P.ctas + u;
  const int a0 = cd->a0, b0 = cd->b0;
  const bool two = P.two_panel && !cd->same;

  if (threadIdx.x == 0) {
    for (int s = 0; s < P.ST; ++s) {
      mbar_init(&full[s], 32);
      mbar_init(&empty[s], NW);
    }
    fence_mbar_init();
    tma_prefetch(&tmX);
  }
  if (MODE == MODE_WEIGHTED)
    for (int j = threadIdx.x; j < ld; j += blockDim.x) beta_s[j] = j < P.p ? P.beta[j] : 0.0;
  __syncthreads();

  if (warp == NW) {
    // ------------------------------------------------------------ producer warp
    for (int s = 0; s < nst; ++s) {
      const int st = s % P.ST;
      const uint32_t ph = (uint32_t)(s / P.ST) & 1u;
      mbar_wait(&empty[st], ph ^ 1u);
      double* pa = smem + (size_t)st * P.stage_doubles;
      double* pb = pa + (size_t)BK * ld;
      double* ys = pa + (size_t)(P.two_panel ? 2 : 1) * BK * ld;
      const int64_t rr = r0 + (int64_t)s * BK;
      if (lane == 0) {
        asm volatile("mbarrier.expect_tx.relaxed.cta.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(&full[st])),
                     "r"(two ? 2u * P.tma_bytes : P.tma_bytes)
                     : "memory");
        if (MODE == MODE_FOLD) {
          tma_load_3d(pa, &tmX, &full[st], a0, kprime, (int)rr);
          if (two) tma_load_3d(pb, &tmX, &full[st], b0, kprime, (int)rr);
        } else {
          tma_load_2d(pa, &tmX, &full[st], a0, (int)rr);
          if (two) tma_load_2d(pb, &tmX, &full[st], b0, (int)rr);
        }
      }
      // the augmented column: y rows of this stage (0 beyond the end)
      const int64_t row = rr + lane;
      double yv = 0.0;
      if (row < r1) {
        if (MODE == MODE_FOLD) yv = P.y[row * P.K + kprime];
        else yv = P.y[row];
      }
      ys[lane] = yv;
      mbar_arrive(&full[st]);
    }
    return;
  }

  // -------------------------------------------------------------- consumer warps
  RectDesc rd;
  if (warp < cd->nrect) rd = cd->rect[warp];
  else { rd.bi0 = 0; rd.bj0 = 0; rd.mask = 0u; }
  uint32_t rowmask = 0, colmask = 0;
#pragma unroll
  for (int r = 0; r < R; ++r)
#pragma unroll
    for (int c = 0; c < C; ++c)
      if ((rd.mask >> (r * C + c)) & 1u) { rowmask |= 1u << r; colmask |= 1u << c; }
  int offA[R], offB[C];
#pragma unroll
  for (int r = 0; r < R; ++r) offA[r] = (lane & 3) * ld + 8 * (rd.bi0 + r) + (lane >> 2) - a0;
#pragma unroll
  for (int c = 0; c < C; ++c) offB[c] = (lane & 3) * ld + 8 * (rd.bj0 + c) + (lane >> 2) - b0;

  double acc[R][C][2];
#pragma unroll
  for (int r = 0; r < R; ++r)
#pragma unroll
    for (int c = 0; c < C; ++c) { acc[r][c][0] = 0.0; acc[r][c][1] = 0.0; }

  double sw = 0.0, sll = 0.0;  // WEIGHTED scalars (lane 0 of each warp)
  const int ycol_b = P.p - b0;  // column of y inside panel B (valid if 0 <= ycol_b < ld)

  for (int s = 0; s < nst; ++s) {
    const int st = s % P.ST;
    const uint32_t ph = (uint32_t)(s / P.ST) & 1u;
    mbar_wait(&full[st], ph);
    double* pa = smem + (size_t)st * P.stage_doubles;
    double* pb = two ? pa + (size_t)BK * ld : pa;
    double* ys = pa + (size_t)(P.two_panel ? 2 : 1) * BK * ld;
    double* ws = ys + BK;

    if (MODE != MODE_WEIGHTED) {
      if (warp == 0 && ycol_b >= 0 && ycol_b < ld) pb[lane * ld + ycol_b] = ys[lane];
    } else {
      // fused proximal-Newton row quantities: eta, mu (clamped), w, z
      const int64_t rr = r0 + (int64_t)s * BK;
      for (int k = warp; k < BK; k += NW) {
        double e = 0.0;
        for (int j = lane; j < P.p; j += 32) e = fma(pa[k * ld + j], beta_s[j], e);
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) e += __shfl_xor_sync(0xffffffffu, e, o);
        if (lane == 0) {
          double w = 0.0, z = 0.0;
          if (rr + k < r1) {
            double mu = 1.0 / (1.0 + exp(-e));
            mu = fmin(fmax(mu, P.eps), 1.0 - P.eps);
            w = mu * (1.0 - mu);
            const double yk = ys[k];
            z = e + (yk - mu) / w;
            sw += w;
            sll += yk * e - (e > 0.0 ? e + log1p(exp(-e)) : log1p(exp(e)));
          }
          ws[k] = w;
          pa[k * ld + P.p] = z;
        }
      }
    }
    named_bar_sync(1, NW * 32);

#pragma unroll
    for (int ks = 0; ks < BK / 4; ++ks) {
      const double* pak = pa + ks * 4 * ld;
      const double* pbk = pb + ks * 4 * ld;
      double a[R], b[C];
      double wk = 1.0;
      if (MODE == MODE_WEIGHTED) wk = ws[ks * 4 + (lane & 3)];
#pragma unroll
      for (int r = 0; r < R; ++r) {
        a[r] = 0.0;
        if ((rowmask >> r) & 1u) {
          a[r] = pak[offA[r]];
          if (MODE == MODE_WEIGHTED) a[r] *= wk;
        }
      }
#pragma unroll
      for (int c = 0; c < C; ++c) b[c] = ((colmask >> c) & 1u) ? pbk[offB[c]] : 0.0;
#pragma unroll
      for (int r = 0; r < R; ++r)
#pragma unroll
        for (int c = 0; c < C; ++c)
          if ((rd.mask >> (r * C + c)) & 1u) dmma_8x8x4(acc[r][c][0], acc[r][c][1], a[r], b[c]);
    }
    fence_proxy_async_smem();  // generic-proxy smem writes above precede the next TMA refill
    __syncwarp();
    if (lane == 0) mbar_arrive(&empty[st]);
  }

  // -------------------------------------------------------------- epilogue
  double* out = P.partial + ((size_t)(fold * P.nseg + seg) * P.nblk) * 64;
#pragma unroll
  for (int r = 0; r < R; ++r)
#pragma unroll
    for (int c = 0; c < C; ++c)
      if ((rd.mask >> (r * C + c)) & 1u) {
        const int idx = P.blk_of[(rd.bi0 + r) * P.nb + rd.bj0 + c];
        double2 v = make_double2(acc[r][c][0], acc[r][c][1]);
        *reinterpret_cast<double2*>(out + (size_t)idx * 64 + (lane >> 2) * 8 + 2 * (lane & 3)) = v;
      }
  if (MODE == MODE_WEIGHTED) {
    if (lane == 0) { scal_s[warp][0] = sw; scal_s[warp][1] = sll; }
    named_bar_sync(1, NW * 32);
    if (threadIdx.x == 0 && u == 0) {
      double a = 0.0, b = 0.0;
      for (int w = 0; w < NW; ++w) { a += scal_s[w][0]; b += scal_s[w][1]; }
      P.partial_scal[seg * 2 + 0] = a;
      P.partial_scal[seg * 2 + 1] = b;
    }
  }
}

// Sum the segment partials in a fixed order and scatter into the packed upper triangle of
// the augmented (p+1)x(p+1) matrix: packed[j*(p+1) - j(j-1)/2 + (l-j)], j <= l <= p.
__global__ void gram_reduce_kernel(const double* __restrict__ partial, int nfold, int nseg, int nblk,
                                   const int2* __restrict__ blk_coord, int p, const double* __restrict__ tail,
                                   double* __restrict__ packed, int64_t psize, const double* __restrict__ pscal,
                                   int with_scal) {
  const int64_t total = (int64_t)nfold * nblk * 64;
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < total; t += (int64_t)gridDim.x * blockDim.x) {
    const int e = (int)(t & 63);
    const int64_t fb = t >> 6;
    const int idx = (int)(fb % nblk);
    const int f = (int)(fb / nblk);
    const int2 bc = blk_coord[idx];
    const int j = 8 * bc.x + (e >> 3), l = 8 * bc.y + (e & 7);
    if (j > l || l > p) continue;
    double s = 0.0;
    const double* src = partial + ((size_t)f * nseg * nblk + idx) * 64 + e;
    for (int g = 0; g < nseg; ++g) s += src[(size_t)g * nblk * 64];
    if (tail) s += tail[((size_t)f * nblk + idx) * 64 + e];
    packed[(size_t)f * psize + (int64_t)j * (p + 1) - (int64_t)j * (j - 1) / 2 + (l - j)] = s;
  }
  if (with_scal && blockIdx.x == 0 && threadIdx.x < 2) {
    double s = 0.0;
    for (int g = 0; g < nseg; ++g) s += pscal[g * 2 + threadIdx.x];
    packed[psize + threadIdx.x] = s;
  }
}

// FOLD tail: rows i in [nq*K, n_local) (fewer than K, so at most one per fold) as outer products.
__global__ void gram_fold_tail_kernel(const double* __restrict__ X, const double* __restrict__ y, int64_t ldx,
                                      int64_t n_local, int64_t nq, int K, int off_mod, int p, int nblk,
                                      const int2* __restrict__ blk_coord, double* __restrict__ tail) {
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
      if (j <= p && l <= p) {
        const double zj = j < p ? X[i * ldx + j] : y[i];
        const double zl = l < p ? X[i * ldx + l] : y[i];
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
  int mode = 0, p = 0, nb = 0, ld = 0, two_panel = 0, U = 0, nseg = 0, ST = 0, nblk = 0;
  int R = 4, C = 4, NW = 12;
  int64_t seg_rows = 0;
  size_t smem = 0;
  uint32_t tma_bytes = 0;
  int stage_doubles = 0;
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

static int popc(uint32_t x) { return __builtin_popcount(x); }

// Assign rectangles to CTA types (longest-processing-time first), then order each CTA's
// rectangles so the 4 SM sub-partitions (warp w -> SMSP w % 4) carry similar DMMA counts.
static void pack_rects(std::vector<RectDesc>& rects, int NW, int a0, int b0, int same, std::vector<CtaDesc>& out) {
  std::sort(rects.begin(), rects.end(), [](const RectDesc& x, const RectDesc& y) { return popc(x.mask) > popc(y.mask); });
  const int U = std::max<int>(1, ((int)rects.size() + NW - 1) / NW);
  std::vector<std::vector<RectDesc>> bins(U);
  std::vector<int> load(U, 0);
  for (auto& r : rects) {
    int best = -1;
    for (int b = 0; b < U; ++b)
      if ((int)bins[b].size() < NW && (best < 0 || load[b] < load[best])) best = b;
    bins[best].push_back(r);
    load[best] += popc(r.mask);
  }
  for (auto& bin : bins) {
    CtaDesc cd;
    std::memset(&cd, 0, sizeof(cd));
    cd.a0 = a0; cd.b0 = b0; cd.same = same;
    // SMSP balancing: LPT over 4 sub-partitions, slot w = sub + 4 * k
    std::vector<std::vector<RectDesc>> sub(4);
    std::vector<int> sl(4, 0);
    for (auto& r : bin) {  // bin is sorted by cost already
      int best = -1;
      for (int q = 0; q < 4; ++q)
        if ((int)sub[q].size() * 4 + q < NW && (best < 0 || sl[q] < sl[best])) best = q;
      sub[best].push_back(r);
      sl[best] += popc(r.mask);
    }
    int nrect = 0;
    RectDesc empty_rect{0, 0, 0u, 0};
    for (int w = 0; w < NW; ++w) cd.rect[w] = empty_rect;
    for (int q = 0; q < 4; ++q)
      for (size_t k = 0; k < sub[q].size(); ++k) {
        int w = q + 4 * (int)k;
        cd.rect[w] = sub[q][k];
        nrect = std::max(nrect, w + 1);
      }
    cd.nrect = nrect;
    out.push_back(cd);
  }
}

static oem_status build_plan(oem_ctx* ctx, int mode, int p, int64_t nrows, int K, GramPlan& pl) {
  pl.mode = mode;
  pl.p = p;
  const int Pa = p + 1;
  pl.nb = (Pa + 7) / 8;
  const int r8 = pl.nb * 8;
  const bool single = (r8 + 4) <= 256;
  if (mode == MODE_WEIGHTED && !single)
    OEM_FAIL(OEM_ERR_UNSUPPORTED, "oem_gram_weighted: p > 247 is not supported by the fused single-panel kernel");
  pl.two_panel = single ? 0 : 1;
  pl.nblk = pl.nb * (pl.nb + 1) / 2;
  std::vector<int32_t> blk_of((size_t)pl.nb * pl.nb, -1);
  std::vector<int2> coord(pl.nblk);
  {
    int idx = 0;
    for (int bi = 0; bi < pl.nb; ++bi)
      for (int bj = bi; bj < pl.nb; ++bj) { blk_of[(size_t)bi * pl.nb + bj] = idx; coord[idx] = make_int2(bi, bj); ++idx; }
  }
  auto mk_mask = [&](int bi0, int bj0, int R, int C) {
    uint32_t m = 0;
    for (int r = 0; r < R; ++r)
      for (int c = 0; c < C; ++c) {
        int bi = bi0 + r, bj = bj0 + c;
        if (bi <= bj && bj < pl.nb) m |= 1u << (r * C + c);
      }
    return m;
  };
  if (single) {
    pl.R = 4; pl.C = 4; pl.NW = 12;
    pl.ld = r8 + 4;  // = 4 or 12 (mod 16): conflict-free fragment loads
    std::vector<RectDesc> rects;
    for (int bi0 = 0; bi0 < pl.nb; bi0 += 4)
      for (int bj0 = bi0; bj0 < pl.nb; bj0 += 4) {
        uint32_t m = mk_mask(bi0, bj0, 4, 4);
        if (m) rects.push_back(RectDesc{bi0, bj0, m, 0});
      }
    pack_rects(rects, pl.NW, 0, 0, 1, pl.ctas);
  } else {
    pl.R = 4; pl.C = 8; pl.NW = 8;
    pl.ld = 132;  // 128-column panel + 4 (mod 16 = 4)
    const int np = (Pa + 127) / 128;
    for (int I = 0; I < np; ++I)
      for (int J = I; J < np; ++J) {
        std::vector<RectDesc> rects;
        for (int r = 0; r < 4; ++r)
          for (int c = 0; c < 2; ++c) {
            int bi0 = 16 * I + 4 * r, bj0 = 16 * J + 8 * c;
            uint32_t m = mk_mask(bi0, bj0, 4, 8);
            if (m) rects.push_back(RectDesc{bi0, bj0, m, 0});
          }
        if (rects.empty()) continue;
        pack_rects(rects, pl.NW, 128 * I, 128 * J, I == J, pl.ctas);
      }
  }
  pl.U = (int)pl.ctas.size();
  const int panels = pl.two_panel ? 2 : 1;
  pl.stage_doubles = panels * BK * pl.ld + BK * (mode == MODE_WEIGHTED ? 2 : 1);
  pl.stage_doubles = (pl.stage_doubles + 15) / 16 * 16;  // 128-byte aligned stages
  const size_t budget = 220 * 1024;
  const size_t fixed = (mode == MODE_WEIGHTED ? pl.ld * 8 : 0) + 2 * MAXST * 8;
  pl.ST = (int)std::min<size_t>(4, (budget - fixed) / ((size_t)pl.stage_doubles * 8));
  if (pl.ST < 2) OEM_FAIL(OEM_ERR_UNSUPPORTED, "gram: stage does not fit shared memory");
  pl.smem = (size_t)pl.ST * pl.stage_doubles * 8 + fixed;
  // segments: enough (CTA type, segment) items for several waves over the SMs
  const int64_t units = std::max<int64_t>(1, (nrows + BK - 1) / BK);  // BK-row units
  const int nfold = mode == MODE_FOLD ? K : 1;
  int64_t want = (int64_t)ctx->num_sms * 4 / std::max(1, pl.U * nfold);
  want = std::max<int64_t>(1, std::min<int64_t>(want, units / 4 > 0 ? units / 4 : 1));
  pl.seg_rows = ((units + want - 1) / want) * BK;
  pl.nseg = (int)std::max<int64_t>(1, (nrows + pl.seg_rows - 1) / pl.seg_rows);
  // device tables
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
  if (r != CUDA_SUCCESS) OEM_FAIL(OEM_ERR_CUDA, "cuTensorMapEncodeTiled failed (code " + std::to_string((int)r) + ")");
  return OEM_OK;
}

template <int R, int C, int NW, int MODE>
static oem_status launch_t(const GramPlan& pl, const CUtensorMap& map, const GramParams& P, int nfold, cudaStream_t st) {
  auto kern = gram_kernel<R, C, NW, MODE>;
  static size_t attr_smem = 0;  // opt-in dynamic shared memory, raised on demand
  if (pl.smem > attr_smem) {
    OEM_CUDA_TRY(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)pl.smem));
    attr_smem = pl.smem;
  }
  dim3 grid((unsigned)(pl.U * pl.nseg * nfold));
  kern<<<grid, (NW + 1) * 32, pl.smem, st>>>(map, P);
  OEM_CUDA_TRY(cudaGetLastError());
  return OEM_OK;
}

oem_status gram_pass(oem_ctx* ctx, int mode, const double* X, const double* y, const double* beta, double eps,
                     int64_t n_local, int p, int64_t ldx, int64_t row_offset, int K, double* packed, cudaStream_t st) {
  const int nfold = mode == MODE_FOLD ? K : 1;
  const int64_t psize = packed_size(p);
  const int64_t nq = mode == MODE_FOLD ? n_local / K : n_local;
  if (n_local == 0 || nq == 0) {
    // nothing to stream through the tensor-core kernel
    OEM_CUDA_TRY(cudaMemsetAsync(packed, 0, sizeof(double) * (nfold * psize + (mode == MODE_WEIGHTED ? 2 : 0)), st));
    if (mode != MODE_FOLD || n_local == 0) return OEM_OK;
  }
  auto key = std::make_tuple(mode, p, nq, K);
  std::shared_ptr<GramPlan> plp;
  auto it = ctx->plans.find(key);
  if (it != ctx->plans.end()) plp = it->second;
  else {
    plp = std::make_shared<GramPlan>();
    oem_status s = build_plan(ctx, mode, p, std::max<int64_t>(nq, 1), K, *plp);
    if (s != OEM_OK) return s;
    ctx->plans[key] = plp;
  }
  const GramPlan& pl = *plp;
  // workspace
  const size_t part_bytes = sizeof(double) * (size_t)nfold * pl.nseg * pl.nblk * 64;
  OEM_CUDA_TRY(ctx->partial.ensure(part_bytes));
  OEM_CUDA_TRY(ctx->partial_scal.ensure(sizeof(double) * 2 * (size_t)pl.nseg + 16));
  double* tail = nullptr;
  if (mode == MODE_FOLD && n_local % K != 0) {
    OEM_CUDA_TRY(ctx->tail.ensure(sizeof(double) * (size_t)K * pl.nblk * 64));
    tail = ctx->tail.as<double>();
  }
  if (nq > 0) {
    CUtensorMap map;
    const cuuint32_t boxw = (cuuint32_t)pl.ld;
    oem_status s;
    if (mode == MODE_FOLD) {
      cuuint64_t dims[3] = {(cuuint64_t)p, (cuuint64_t)K, (cuuint64_t)nq};
      cuuint64_t strides[2] = {(cuuint64_t)ldx * 8, (cuuint64_t)ldx * 8 * K};
      cuuint32_t box[3] = {boxw, 1, (cuuint32_t)BK};
      s = make_map(&map, X, 3, dims, strides, box);
    } else {
      cuuint64_t dims[2] = {(cuuint64_t)p, (cuuint64_t)n_local};
      cuuint64_t strides[1] = {(cuuint64_t)ldx * 8};
      cuuint32_t box[2] = {boxw, (cuuint32_t)BK};
      s = make_map(&map, X, 2, dims, strides, box);
    }
    if (s != OEM_OK) return s;
    GramParams P;
    std::memset(&P, 0, sizeof(P));
    P.p = p; P.nb = pl.nb; P.ld = pl.ld; P.U = pl.U; P.nseg = pl.nseg; P.ST = pl.ST; P.two_panel = pl.two_panel;
    P.nblk = pl.nblk; P.nrows = nq; P.seg_rows = pl.seg_rows; P.K = K;
    P.off_mod = mode == MODE_FOLD ? (int)(((row_offset % K) + K) % K) : 0;
    P.y = y; P.beta = beta; P.eps = eps;
    P.partial = ctx->partial.as<double>();
    P.partial_scal = ctx->partial_scal.as<double>();
    P.ctas = pl.d_ctas; P.blk_of = pl.d_blk_of;
    P.tma_bytes = (uint32_t)(BK * pl.ld * 8);  // bytes of one box; off-diagonal tiles load two
    P.stage_doubles = pl.stage_doubles;
    oem_status ls;
    if (!pl.two_panel) {
      if (mode == MODE_PLAIN) ls = launch_t<4, 4, 12, MODE_PLAIN>(pl, map, P, nfold, st);
      else if (mode == MODE_FOLD) ls = launch_t<4, 4, 12, MODE_FOLD>(pl, map, P, nfold, st);
      else ls = launch_t<4, 4, 12, MODE_WEIGHTED>(pl, map, P, nfold, st);
    } else {
      if (mode == MODE_PLAIN) ls = launch_t<4, 8, 8, MODE_PLAIN>(pl, map, P, nfold, st);
      else ls = launch_t<4, 8, 8, MODE_FOLD>(pl, map, P, nfold, st);
    }
    if (ls != OEM_OK) return ls;
  }
  if (tail) {
    gram_fold_tail_kernel<<<std::max(1, std::min(1024, (int)((K * (int64_t)pl.nblk * 64 + 255) / 256))), 256, 0, st>>>(
        X, y, ldx, n_local, nq, K, (int)(((row_offset % K) + K) % K), p, pl.nblk, pl.d_blk_coord, tail);
    OEM_CUDA_TRY(cudaGetLastError());
  }
  {
    const int64_t total = (int64_t)nfold * pl.nblk * 64;
    const int blocks = (int)std::max<int64_t>(1, std::min<int64_t>(ctx->num_sms * 8, (total + 255) / 256));
    gram_reduce_kernel<<<blocks, 256, 0, st>>>(ctx->partial.as<double>(), nfold, nq > 0 ? pl.nseg : 0, pl.nblk,
                                               pl.d_blk_coord, p, tail, packed, psize, ctx->partial_scal.as<double>(),
                                               mode == MODE_WEIGHTED);
    OEM_CUDA_TRY(cudaGetLastError());
  }
  return OEM_OK;
}

oem_status gram_unpack(const double* packed, int nfold, int p, double* G, double* xty, double* yty, cudaStream_t st) {
  const int64_t total = (int64_t)nfold * ((int64_t)p * p + p + 1);
  const int blocks = (int)std::max<int64_t>(1, std::min<int64_t>(4096, (total + 255) / 256));
  gram_unpack_kernel<<<blocks, 256, 0, st>>>(packed, nfold, p, G, xty, yty);
  OEM_CUDA_TRY(cudaGetLastError());
  return OEM_OK;
}

}  // namespace oem
