// sparse.cu — f4: the Gram pass over a SPARSE design (§5.8, P:L894-928:
// "oem() and cv.oem() can accept sparse design matrices ... a substantial computational speedup").
//
// What it computes: exactly the a2 statistics of the augmented matrix
// Z = [X | y] — G_jk = sum_i x_ij x_ik (j <= k), X^T y, y^T y — with X given in compressed sparse
// row form (row_ptr, col, val; columns strictly ascending within each row). Only the products of
// nonzeros exist: row i contributes m_i (m_i + 1) / 2 + m_i + 1 terms (m_i = its nonzeros), so
// the pass is bound by reading the CSR arrays, not by the p^2 arithmetic of the dense kernel.
//
// B200 design (deterministic: every accumulator has one owner thread and a data-fixed order):
//  * One CTA per SM holds a SLICE of the packed upper triangle of Z^T Z in shared memory (rows
//    [J_u, J_{u+1}) of the triangle; p = 200 fits one slice, 162 KB) and streams a contiguous row
//    segment of the CSR arrays: one producer warp stages chunks of up to 256 rows / 768 nonzeros
//    (row_ptr, y, col, val) into a 3-deep shared-memory ring with cp.async (completion through
//    mbarrier arrive.noinc); four mask warps and 16 owner warps process them.
//  * Owner lanes OWN triangle rows (columns): column c belongs to warp c % 16 (4 owner warps per
//    SM sub-partition), lane (c / 16) % L; it alone updates G[j][k >= j] and G[j][p] for its
//    columns. Per chunk the mask warps first mark, for every owned column j, which of the chunk's
//    rows hold a nonzero in column j (a 256-bit row mask per column in the stage, set with
//    shared-memory atomicOr: a bitwise OR is order-free); each owner walks its masks in ascending
//    row order and, for every row with x_ij != 0, adds x_ij x_ik for the row's nonzeros k >= j and
//    x_ij y_i. Work per chunk is proportional to the chunk's nonzeros and their row neighbours, with
//    no conflicts and no redundant scanning; owner warps are coupled only through the ring
//    (imbalance between chunks averages out). y^T y is a fixed-order warp sum per mask warp and
//    chunk, added in warp order by the owner of the augmented column p.
//  * Segments write their slice to a partial buffer; a second kernel adds the segments in a
//    fixed order into the packed triangle (the NCCL allreduce and the unpack are shared with the
//    dense path).
#include <algorithm>
#include <string>
#include <vector>

#include "common.cuh"
#include "internal.h"

namespace oem {

namespace {

constexpr int SP_WARPS = 16;                    // owner (consumer) warps; a lane owns columns
constexpr int SP_LGW = 4;                       // log2(SP_WARPS)
constexpr int SP_PROD = SP_WARPS;               // warp index of the producer
constexpr int SP_MASKW = SP_WARPS + 1;          // warp index of the first mask builder
constexpr int SP_NMASK = 4;                     // mask-builder warps (rows 32 m + lane + 128 t)
constexpr int SP_THREADS = (SP_WARPS + 1 + SP_NMASK) * 32;
constexpr int SP_ST = 3;                        // ring depth
constexpr int SP_ROWS = 256;                    // rows per stage (max)
constexpr int SP_MW = SP_ROWS / 32;             // mask words per column
constexpr int SP_ENT = 768;                     // nonzeros per stage (max): p <= SP_ENT
constexpr size_t SP_SMEM_MAX = 227 * 1024;

struct SpStage {  // shared-memory layout of one ring stage (byte offsets); masks follow at `mask`
  static constexpr int rp = 0;
  static constexpr int y = rp + (SP_ROWS + 1) * 8;
  static constexpr int val = y + SP_ROWS * 8;
  static constexpr int col = val + SP_ENT * 8;
  static constexpr int hdr = col + SP_ENT * 4;   // int R, pad, int64 e0, double yy[SP_NMASK] (the chunk's y^T y)
  static constexpr int rs = hdr + 16 + 8 * SP_NMASK;   // int16 [SP_ROWS + 1]: row offsets relative to e0 (mask warps)
  static constexpr int summ = (rs + 2 * (SP_ROWS + 1) + 15) / 16 * 16;   // one byte per mask slot: its non-empty words
};
// The masks are stored word-major and, within a word, in OWNER order: with L = 2^lgl lanes per
// owner warp per round (the least power of two with SP_WARPS L >= ncol, at most 32), column c is
// owned by warp c % SP_WARPS, lane (c / SP_WARPS) % L, so the slice's columns spread over all
// owner warps (4 per SM sub-partition, hiding each other's shared-memory latency), and its mask
// slot is round * SP_WARPS L + warp L + lane: an owner warp's mask loads hit distinct banks.
// Word w of column c sits at mask[w * mask_ld(ncol) + slot(c)].
__host__ __device__ constexpr int lg_lanes(int ncol) {   // log2 of the lanes per owner warp per round
  int l = 0;
  while ((SP_WARPS << l) < ncol && l < 5) ++l;
  return l;
}
__host__ __device__ constexpr int mask_ld(int ncol) {
  const int nl = SP_WARPS << lg_lanes(ncol);
  return (ncol + nl - 1) / nl * nl;
}
__device__ __forceinline__ int mask_slot(int c, int lgl) {
  return (c & ~((SP_WARPS << lgl) - 1)) | ((c & (SP_WARPS - 1)) << lgl) | ((c >> SP_LGW) & ((1 << lgl) - 1));
}
// the masks follow the per-slot summary bytes (mask_ld(ncol) of them)
__host__ __device__ constexpr int mask_off(int ncol) { return (SpStage::summ + mask_ld(ncol) + 127) / 128 * 128; }
__host__ __device__ constexpr int stage_bytes(int ncol) { return mask_off(ncol) + (mask_ld(ncol) * SP_MW * 4 + 127) / 128 * 128; }

struct SpParams {
  const int64_t* row_ptr;
  const int32_t* col;
  const double* val;
  const double* y;
  int64_t n;
  int p, U, nseg;
  int64_t seg_rows;
  const int* slice_j0;   // [U+1] first triangle row of each slice
  int cap;               // entries per slice buffer (max over slices)
  int sbytes;            // bytes per ring stage (mask columns of the widest slice)
  double* partial;       // [U][nseg][cap]
};

#ifdef SP_PROFILE
// developer instrumentation: cycles each role spends waiting on its ring barrier vs in total (CTA 0)
#define SP_WAIT(bar, par)                               \
  do {                                                  \
    const long long t_ = clock64();                     \
    mbar_wait(bar, par);                                \
    prof_wait += clock64() - t_;                        \
  } while (0)
#define SP_REPORT(role)                                                                              \
  if (blockIdx.x == 0 && lane == 0)                                                                  \
    printf("SP_PROFILE %s warp %d wait %lld total %lld chunks %d\n", role, warp, prof_wait,          \
           clock64() - prof_t0, prof_chunks)
#else
#define SP_WAIT(bar, par) mbar_wait(bar, par)
#define SP_REPORT(role)
#endif

__device__ __forceinline__ int64_t tri_off(int64_t j, int64_t pa) { return j * pa - j * (j - 1) / 2; }  // packed index of (j, j)

__device__ __forceinline__ void cp_async8(void* dst, const void* src) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(smem_u32(dst)), "l"(src) : "memory");
}
__device__ __forceinline__ void cp_async4(void* dst, const void* src) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"(smem_u32(dst)), "l"(src) : "memory");
}
__device__ __forceinline__ void cp_async_arrive_noinc(uint64_t* bar) {
  asm volatile("cp.async.mbarrier.arrive.noinc.shared::cta.b64 [%0];" ::"r"(smem_u32(bar)) : "memory");
}

// Ring protocol per stage s: producer fills rows / nonzeros -> full[s] (32 cp.async arrivals +
// the header arrive); the mask warps mark the owned columns' rows and the chunk's y^T y ->
// ready[s]; every owner warp walks its columns, clears their mask words -> empty[s]. Owner warps
// are coupled only through the ring, so a warp slowed by a dense column in one chunk catches up
// on the next (up to SP_ST chunks of slack).
__global__ void __launch_bounds__(SP_THREADS, 1) sparse_gram_kernel(const SpParams P) {
  extern __shared__ __align__(128) unsigned char sbytes[];
  __shared__ __align__(8) uint64_t full[SP_ST], ready[SP_ST], empty[SP_ST];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
#ifdef SP_PROFILE
  long long prof_wait = 0, prof_t0 = clock64();
  int prof_chunks = 0;
#endif
  const int u = blockIdx.x % P.U, seg = blockIdx.x / P.U;
  const int p = P.p;
  const int64_t pa = p + 1;
  const int64_t r0 = (int64_t)seg * P.seg_rows, r1 = min(P.n, r0 + P.seg_rows);
  const int J0 = P.slice_j0[u], J1 = P.slice_j0[u + 1], ncol = J1 - J0, mld = mask_ld(ncol), lgl = lg_lanes(ncol);
  const int64_t base = tri_off(J0, pa), nent = tri_off(J1, pa) - base;
  double* gs = reinterpret_cast<double*>(sbytes + (size_t)SP_ST * P.sbytes);
  for (int64_t e = threadIdx.x; e < nent; e += SP_THREADS) gs[e] = 0.0;
  for (int s = 0; s < SP_ST; ++s) {
    uint32_t* m = reinterpret_cast<uint32_t*>(sbytes + (size_t)s * P.sbytes + mask_off(ncol));
    for (int e = threadIdx.x; e < mask_ld(ncol) * SP_MW; e += SP_THREADS) m[e] = 0u;
    uint32_t* sm4 = reinterpret_cast<uint32_t*>(sbytes + (size_t)s * P.sbytes + SpStage::summ);
    for (int e = threadIdx.x; e < mld / 4; e += SP_THREADS) sm4[e] = 0u;
  }
  if (threadIdx.x == 0) {
    for (int s = 0; s < SP_ST; ++s) {
      mbar_init(&full[s], 33);          // 32 cp.async arrivals (noinc) + the header arrive
      mbar_init(&ready[s], 32 * SP_NMASK);   // every lane of the mask warps
      mbar_init(&empty[s], SP_WARPS);   // lane 0 of every owner warp
    }
    fence_mbar_init();
  }
  __syncthreads();

  if (warp == SP_PROD) {
    // ---------------------------------------------------------------- producer warp
    int st = 0;
    uint32_t ph = 0;
    int64_t r = r0;
    // row offsets of the next chunk's first row and of its full-size end, loaded one chunk ahead
    // (their global-load latency overlaps the wait for a free stage)
    int64_t pf_lo = 0, pf_hi = 0;
    if (lane == 0 && r < r1) {
      pf_lo = P.row_ptr[r];
      pf_hi = P.row_ptr[r + (r1 - r < (int64_t)SP_ROWS ? r1 - r : (int64_t)SP_ROWS)];
    }
    for (;;) {
      SP_WAIT(&empty[st], ph ^ 1u);
      unsigned char* sb = sbytes + (size_t)st * P.sbytes;
      int R = 0;
      int64_t e0 = 0, e1 = 0;
      if (lane == 0 && r < r1) {
        // the largest R <= SP_ROWS whose nonzeros fit the stage (binary search on row_ptr)
        const int full_r = (int)(r1 - r < (int64_t)SP_ROWS ? r1 - r : (int64_t)SP_ROWS);
        int hi = full_r;
        e0 = pf_lo;
        if (pf_hi - e0 <= SP_ENT) {
          R = hi;
        } else {
          int lo = 1;  // a single row always fits (p <= SP_ENT)
          while (lo < hi) {
            const int mid = (lo + hi + 1) / 2;
            if (P.row_ptr[r + mid] - e0 <= SP_ENT) lo = mid;
            else hi = mid - 1;
          }
          R = lo;
        }
        e1 = R == full_r ? pf_hi : P.row_ptr[r + R];
        // prefetch the next chunk's bounds (it starts at r + R)
        const int64_t rn = r + R;
        if (rn < r1) {
          pf_lo = e1;
          pf_hi = P.row_ptr[rn + (r1 - rn < (int64_t)SP_ROWS ? r1 - rn : (int64_t)SP_ROWS)];
        }
      }
      R = __shfl_sync(0xffffffffu, R, 0);
      e0 = __shfl_sync(0xffffffffu, e0, 0);
      e1 = __shfl_sync(0xffffffffu, e1, 0);
      int64_t* rp_s = reinterpret_cast<int64_t*>(sb + SpStage::rp);
      double* y_s = reinterpret_cast<double*>(sb + SpStage::y);
      double* v_s = reinterpret_cast<double*>(sb + SpStage::val);
      int32_t* c_s = reinterpret_cast<int32_t*>(sb + SpStage::col);
      for (int q = lane; q <= R && R > 0; q += 32) cp_async8(rp_s + q, P.row_ptr + r + q);
      for (int q = lane; q < R; q += 32) cp_async8(y_s + q, P.y + r + q);
      const int ne = (int)(e1 - e0);
      for (int q = lane; q < ne; q += 32) {
        cp_async8(v_s + q, P.val + e0 + q);
        cp_async4(c_s + q, P.col + e0 + q);
      }
      cp_async_arrive_noinc(&full[st]);
      if (lane == 0) {
        int* h = reinterpret_cast<int*>(sb + SpStage::hdr);
        h[0] = R;
        *reinterpret_cast<int64_t*>(h + 2) = e0;
        mbar_arrive(&full[st]);
      }
      if (++st == SP_ST) { st = 0; ph ^= 1u; }
      if (R == 0) break;  // the terminating (empty) stage has been published
      r += R;
#ifdef SP_PROFILE
      ++prof_chunks;
#endif
    }
    SP_REPORT("producer");
    return;
  }

  if (warp >= SP_MASKW) {
    const int m = warp - SP_MASKW;
    // ---------------------------------------------------------------- mask warp
    int st = 0;
    uint32_t ph = 0;
    for (;;) {
      SP_WAIT(&full[st], ph);
      unsigned char* sb = sbytes + (size_t)st * P.sbytes;
      int* h = reinterpret_cast<int*>(sb + SpStage::hdr);
      const int R = h[0];
      const int64_t e0 = *reinterpret_cast<const int64_t*>(h + 2);
      const int64_t* rp_s = reinterpret_cast<const int64_t*>(sb + SpStage::rp);
      const double* y_s = reinterpret_cast<const double*>(sb + SpStage::y);
      const int32_t* c_s = reinterpret_cast<const int32_t*>(sb + SpStage::col);
      int16_t* rs = reinterpret_cast<int16_t*>(sb + SpStage::rs);
      uint32_t* summ = reinterpret_cast<uint32_t*>(sb + SpStage::summ);
      uint32_t* mask = reinterpret_cast<uint32_t*>(sb + mask_off(ncol));
      // the stage's masks and summaries start from zero (the owners only read them): the mask
      // warps clear them, then meet at a named barrier before marking
      const int tm = 32 * m + lane;
      for (int e = tm; e < mld * SP_MW / 4; e += 32 * SP_NMASK) reinterpret_cast<uint4*>(mask)[e] = make_uint4(0u, 0u, 0u, 0u);
      for (int e = tm; e < mld / 4; e += 32 * SP_NMASK) summ[e] = 0u;
      named_bar_sync(1, 32 * SP_NMASK);
      double yy = 0.0;
      if (tm == 0) rs[R] = (int16_t)(rp_s[R] - e0);
      for (int q = tm; q < R; q += 32 * SP_NMASK) {   // warp m, lane: rows 32 m + lane + 128 t
        const int a0 = (int)(rp_s[q] - e0), a1 = (int)(rp_s[q + 1] - e0);
        rs[q] = (int16_t)a0;
        for (int a = a0; a < a1; ++a) {
          const int c = c_s[a] - J0;
          if (c >= 0 && c < ncol) {
            const int sl = mask_slot(c, lgl);
            atomicOr(&mask[(q >> 5) * mld + sl], 1u << (q & 31));
            atomicOr(&summ[sl >> 2], 1u << ((q >> 5) + 8 * (sl & 3)));   // word q/32 of slot sl is non-empty
          }
        }
        yy = fma(y_s[q], y_s[q], yy);
      }
#pragma unroll
      for (int o = 16; o >= 1; o >>= 1) yy += __shfl_xor_sync(0xffffffffu, yy, o);   // fixed order
      if (lane == 0) reinterpret_cast<double*>(h + 4)[m] = yy;
      __syncwarp();
      mbar_arrive(&ready[st]);
      if (++st == SP_ST) { st = 0; ph ^= 1u; }
      if (R == 0) break;
#ifdef SP_PROFILE
      ++prof_chunks;
#endif
    }
    SP_REPORT("mask");
    return;
  }

  // ------------------------------------------------------------------ owner warps
  // owner (warp, lane < 2^lgl) holds mask slot ct (+ one round of SP_WARPS << lgl slots per trip)
  // and owns columns (lane << SP_LGW) + warp (+ the same per trip)
  const int ct = (warp << lgl) | lane;
  int st = 0;
  uint32_t ph = 0;
  for (;;) {
    SP_WAIT(&ready[st], ph);
    unsigned char* sb = sbytes + (size_t)st * P.sbytes;
    const int* h = reinterpret_cast<const int*>(sb + SpStage::hdr);
    const int R = h[0];
    if (R == 0) break;
    const int16_t* rs = reinterpret_cast<const int16_t*>(sb + SpStage::rs);
    const double* y_s = reinterpret_cast<const double*>(sb + SpStage::y);
    const double* v_s = reinterpret_cast<const double*>(sb + SpStage::val);
    const int32_t* c_s = reinterpret_cast<const int32_t*>(sb + SpStage::col);
    const uint32_t* summ = reinterpret_cast<const uint32_t*>(sb + SpStage::summ);
    const uint32_t* mask = reinterpret_cast<const uint32_t*>(sb + mask_off(ncol));
    for (int i = 0;; i += SP_WARPS << lgl) {
      const int c = i + (lane << SP_LGW) + warp;   // the column of mask slot i + ct
      if (lane >> lgl || c >= ncol) break;
      const int j = J0 + c;
      double* grow = gs + (tri_off(j, pa) - base) - j;   // grow[k] = G[j][k]
      if (j == p) {   // the augmented column: y^T y of the chunk
        const double* yyc = reinterpret_cast<const double*>(h + 4);
        double yy = yyc[0];
#pragma unroll
        for (int mm = 1; mm < SP_NMASK; ++mm) yy += yyc[mm];   // fixed order
        grow[p] += yy;
        continue;
      }
      // the column's non-empty mask words (its summary byte), then their set bits in ascending
      // row order, each lane at its own pace (a word is loaded when the walk reaches it)
      const int sl = i + ct;
      uint32_t nzw = (summ[sl >> 2] >> (8 * (sl & 3))) & 0xffu;
      int w = 0;
      uint32_t bits = 0u;
      for (;;) {   // one set bit per trip: a lane's trip count is its column's nonzeros in the chunk
        if (!bits) {
          if (!nzw) break;
          w = __ffs(nzw) - 1;
          nzw &= nzw - 1;
          bits = mask[w * mld + sl];
        }
        const int q = 32 * w + __ffs(bits) - 1;
        bits &= bits - 1;
        const int a0 = rs[q];
        const int a1 = rs[q + 1];
        // the row's nonzero in column j, four columns per probe: the row's columns ascend and
        // are distinct, so the first match is it (slots past the row end come after it)
        int a = a0;
        for (;; a += 4) {
          const int k0 = c_s[a], k1 = c_s[a + 1], k2 = c_s[a + 2], k3 = c_s[a + 3];
          if (k0 == j) break;
          if (k1 == j) { a += 1; break; }
          if (k2 == j) { a += 2; break; }
          if (k3 == j) { a += 3; break; }
        }
        const double va = v_s[a];
        // the row's columns are distinct, so these read-modify-writes never alias: the loads
        // of a pair are issued before either store
        int b = a;
        for (; b + 1 < a1; b += 2) {
          const int k0 = c_s[b], k1 = c_s[b + 1];
          const double g0 = grow[k0], g1 = grow[k1];
          const double x0 = v_s[b], x1 = v_s[b + 1];
          grow[k0] = g0 + va * x0;
          grow[k1] = g1 + va * x1;
        }
        if (b < a1) grow[c_s[b]] += va * v_s[b];
        grow[p] += va * y_s[q];
      }
    }
    __syncwarp();
    if (lane == 0) mbar_arrive(&empty[st]);
    if (++st == SP_ST) { st = 0; ph ^= 1u; }
#ifdef SP_PROFILE
    ++prof_chunks;
#endif
  }
  SP_REPORT("owner");
  // epilogue: every owner writes its columns' triangle rows to this segment's partial
  double* out = P.partial + ((size_t)u * P.nseg + seg) * P.cap;
  for (int c = (lane << SP_LGW) + warp; !(lane >> lgl) && c < ncol; c += SP_WARPS << lgl) {   // the same columns as above (no CTA barrier needed)
    const int64_t a0 = tri_off(J0 + c, pa) - base, a1 = tri_off(J0 + c + 1, pa) - base;
    for (int64_t e = a0; e < a1; ++e) out[e] = gs[e];
  }
}

// packed[base_u + e] = sum over segments (fixed order) of partial[u][seg][e]
__global__ void sparse_reduce_kernel(const double* __restrict__ partial, int U, int nseg, int cap,
                                     const int* __restrict__ slice_j0, int p, double* __restrict__ packed,
                                     int accumulate) {
  const int64_t pa = p + 1;
  const int64_t total = (int64_t)U * cap;
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < total; t += (int64_t)gridDim.x * blockDim.x) {
    const int u = (int)(t / cap);
    const int64_t e = t % cap;
    const int64_t base = tri_off(slice_j0[u], pa), nent = tri_off(slice_j0[u + 1], pa) - base;
    if (e >= nent) continue;
    double s = 0.0;
    for (int g = 0; g < nseg; ++g) s += partial[((size_t)u * nseg + g) * cap + e];
    packed[base + e] = accumulate ? packed[base + e] + s : s;
  }
}

}  // namespace

}  // namespace oem

using namespace oem;

extern "C" oem_status oem_gram_csr(oem_ctx* ctx, const int64_t* row_ptr, const int32_t* col, const double* val,
                                   const double* y, int64_t n_local, int32_t p, double* G, double* xty, double* yty,
                                   int64_t* n_total, void* stream) {
  if (!ctx) OEM_FAIL(OEM_ERR_INVALID_ARG, "null oem_ctx");
  OEM_CUDA_TRY(cudaSetDevice(ctx->device));
  if (p < 1 || n_local < 0) OEM_FAIL(OEM_ERR_DIM, "oem_gram_csr: need p >= 1, n_local >= 0");
  if (p > SP_ENT) OEM_FAIL(OEM_ERR_UNSUPPORTED, "oem_gram_csr: p > 768 (a row must fit one staging chunk)");
  if (!G || !xty || !yty) OEM_FAIL(OEM_ERR_INVALID_ARG, "oem_gram_csr: null output");
  if (n_local > 0 && (!row_ptr || !y || !col || !val)) OEM_FAIL(OEM_ERR_INVALID_ARG, "oem_gram_csr: null input");
  if (n_local > ((int64_t)1 << 40)) OEM_FAIL(OEM_ERR_UNSUPPORTED, "oem_gram_csr: n_local too large");
  cudaStream_t st = (cudaStream_t)stream;
  const int64_t pa = p + 1, psize = packed_size(p);
  // slices of the packed triangle (rows of Z^T Z): a slice's entries (8 bytes each) sit in shared
  // memory beside the ring, whose stages carry a row mask per slice column (4 * SP_MW bytes)
  std::vector<int> sj;
  int64_t cap = 0;
  int sbytes = 0;
  for (int64_t budget = (int64_t)SP_SMEM_MAX - 1024 - (int64_t)SP_ST * SpStage::summ; budget > 0; budget -= 4096) {
    sj.assign(1, 0);
    int64_t cur = 0;
    for (int j = 0; j <= p; ++j) {
      const int64_t need = 8 * (pa - j) + (int64_t)SP_ST * (4 * SP_MW + 1);
      if (cur + need > budget && cur > 0) { sj.push_back(j); cur = 0; }
      cur += need;
    }
    sj.push_back(p + 1);
    cap = 0;
    int ncol = 0;
    for (size_t u = 0; u + 1 < sj.size(); ++u) {
      const int64_t a = sj[u], b = sj[u + 1];
      cap = std::max<int64_t>(cap, (b * pa - b * (b - 1) / 2) - (a * pa - a * (a - 1) / 2));
      ncol = std::max(ncol, (int)(b - a));
    }
    sbytes = stage_bytes(ncol);
    if ((size_t)SP_ST * sbytes + (size_t)cap * 8 <= SP_SMEM_MAX - 1024) break;
  }
  const int U = (int)sj.size() - 1;
  const int nseg = (int)std::max<int64_t>(1, std::min<int64_t>((n_local + 1023) / 1024, std::max(1, ctx->num_sms / U)));
  const int64_t seg_rows = n_local > 0 ? (n_local + nseg - 1) / nseg : 1;
  // workspace: partial [U][nseg][cap] | packed | tables
  size_t off = 0;
  auto take = [&](size_t bytes) { size_t o = off; off += (bytes + 255) / 256 * 256; return o; };
  const size_t o_part = take(sizeof(double) * (size_t)U * nseg * cap);
  const size_t o_pack = take(sizeof(double) * (size_t)(psize + 2));
  const size_t o_sj = take(sizeof(int) * sj.size());
  OEM_CUDA_TRY(ctx->sparse_ws.ensure(off));
  char* base = ctx->sparse_ws.as<char>();
  OEM_CUDA_TRY(cudaMemcpyAsync(base + o_sj, sj.data(), sizeof(int) * sj.size(), cudaMemcpyHostToDevice, st));
  double* packed = reinterpret_cast<double*>(base + o_pack);
  if (n_local == 0) {
    OEM_CUDA_TRY(cudaMemsetAsync(packed, 0, sizeof(double) * psize, st));
  } else {
    SpParams P;
    P.row_ptr = row_ptr; P.col = col; P.val = val; P.y = y; P.n = n_local; P.p = p; P.U = U; P.nseg = nseg;
    P.seg_rows = seg_rows;
    P.slice_j0 = reinterpret_cast<int*>(base + o_sj);
    P.cap = (int)cap;
    P.sbytes = sbytes;
    P.partial = reinterpret_cast<double*>(base + o_part);
    const size_t smem = (size_t)SP_ST * sbytes + (size_t)cap * 8;
    OEM_CUDA_TRY(cudaFuncSetAttribute(sparse_gram_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    {
      PhaseTimer tm(ctx, PH_GRAM, st);
      ++ctx->launches;
      sparse_gram_kernel<<<U * nseg, SP_THREADS, smem, st>>>(P);
      OEM_CUDA_TRY(cudaGetLastError());
    }
    PhaseTimer tm(ctx, PH_REDUCE, st);
    ++ctx->launches;
    const int64_t total = (int64_t)U * cap;
    sparse_reduce_kernel<<<(int)std::max<int64_t>(1, std::min<int64_t>(ctx->num_sms * 8, (total + 255) / 256)), 256, 0,
                           st>>>(P.partial, U, nseg, (int)cap, P.slice_j0, p, packed, 0);
    OEM_CUDA_TRY(cudaGetLastError());
  }
  oem_status s = allreduce_sum(ctx, packed, (size_t)psize, st);
  if (s != OEM_OK) return s;
  s = gram_unpack(ctx, packed, 1, p, G, xty, yty, st);
  if (s != OEM_OK) return s;
  if (n_total) {
    int64_t nn = n_local;
    if ((s = host_allreduce_i64(ctx, &nn, 1, st)) != OEM_OK) return s;
    *n_total = nn;
  }
  return OEM_OK;
}
