// sparse.cu — f4: the Gram pass over a SPARSE design (§5.8, P:L894-928:
// "oem() and cv.oem() can accept sparse design matrices ... a substantial computational speedup").
//
// What it computes: exactly the a2 statistics of the augmented matrix
// Z = [X | y] — G_jk = sum_i x_ij x_ik (j <= k), X^T y, y^T y — with X given in compressed sparse
// row form (row_ptr, col, val; columns strictly ascending within each row). Only the products of
// nonzeros exist: row i contributes m_i (m_i + 1) / 2 + m_i + 1 terms (m_i = its nonzeros), so
// the pass is bound by reading the CSR arrays, not by the p^2 arithmetic of the dense kernel.
//
// B200 design (deterministic, no atomics):
//  * One CTA per SM holds a SLICE of the packed upper triangle of Z^T Z in shared memory (rows
//    [J_u, J_{u+1}) of the triangle, up to ~22k entries = 175 KB; p = 200 fits one slice) and
//    streams a contiguous row segment of the CSR arrays: one producer warp stages chunks of up to
//    256 rows / 768 nonzeros (row_ptr, y, col, val) into a 4-deep shared-memory ring with
//    cp.async (completion through mbarrier arrive.noinc), eight consumer warps read them.
//  * Every consumer warp OWNS a contiguous range of triangle rows j and scans every staged row
//    (lane = row), emitting only its own pairs (j, k >= j), (j, p) and (p, p): no two warps ever
//    touch the same entry. Inside a warp, lanes emit one pair per round; lanes that hit the same
//    entry in a round are grouped with __match_any_sync and summed in lane order by the group
//    leader -> every entry accumulates in an order fixed by the data, bitwise reproducible.
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

constexpr int SP_WARPS = 8;                     // consumer warps
constexpr int SP_THREADS = (SP_WARPS + 1) * 32; // + one producer warp
constexpr int SP_ST = 4;                        // ring depth
constexpr int SP_ROWS = 256;                    // rows per stage (max)
constexpr int SP_ENT = 768;                     // nonzeros per stage (max): p <= SP_ENT
constexpr int SP_STAGE_BYTES = ((SP_ROWS + 1) * 8 + SP_ROWS * 8 + SP_ENT * 4 + SP_ENT * 8 + 32 + 127) / 128 * 128;
constexpr size_t SP_SMEM_MAX = 227 * 1024;

struct SpStage {  // shared-memory layout of one ring stage (byte offsets)
  static constexpr int rp = 0;
  static constexpr int y = rp + (SP_ROWS + 1) * 8;
  static constexpr int val = y + SP_ROWS * 8;
  static constexpr int col = val + SP_ENT * 8;
  static constexpr int hdr = col + SP_ENT * 4;  // {int R; int base_shift} then int64 e0
};

struct SpParams {
  const int64_t* row_ptr;
  const int32_t* col;
  const double* val;
  const double* y;
  int64_t n;
  int p, U, nseg;
  int64_t seg_rows;
  const int* slice_j0;   // [U+1] first triangle row of each slice
  const int* warp_j0;    // [U][SP_WARPS+1] first triangle row of each consumer warp
  int cap;               // entries per slice buffer (max over slices)
  double* partial;       // [U][nseg][cap]
};

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

__global__ void __launch_bounds__(SP_THREADS, 1) sparse_gram_kernel(const SpParams P) {
  extern __shared__ __align__(128) unsigned char sbytes[];
  __shared__ __align__(8) uint64_t full[SP_ST], empty[SP_ST];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int u = blockIdx.x % P.U, seg = blockIdx.x / P.U;
  const int p = P.p;
  const int64_t pa = p + 1;
  const int64_t r0 = (int64_t)seg * P.seg_rows, r1 = min(P.n, r0 + P.seg_rows);
  const int J0 = P.slice_j0[u];
  const int64_t base = tri_off(J0, pa);
  double* gs = reinterpret_cast<double*>(sbytes + (size_t)SP_ST * SP_STAGE_BYTES);
  const int64_t nent = tri_off(P.slice_j0[u + 1], pa) - base;
  for (int64_t e = threadIdx.x; e < nent; e += SP_THREADS) gs[e] = 0.0;
  if (threadIdx.x == 0) {
    for (int s = 0; s < SP_ST; ++s) {
      mbar_init(&full[s], 33);        // 32 cp.async arrivals (noinc) + the header arrive
      mbar_init(&empty[s], SP_WARPS);
    }
    fence_mbar_init();
  }
  __syncthreads();

  if (warp == SP_WARPS) {
    // ---------------------------------------------------------------- producer warp
    int st = 0;
    uint32_t ph = 0;
    int64_t r = r0;
    for (;;) {
      mbar_wait(&empty[st], ph ^ 1u);
      unsigned char* sb = sbytes + (size_t)st * SP_STAGE_BYTES;
      int R = 0;
      int64_t e0 = 0, e1 = 0;
      if (lane == 0 && r < r1) {
        // the largest R <= SP_ROWS whose nonzeros fit the stage (binary search on row_ptr)
        int hi = (int)(r1 - r < (int64_t)SP_ROWS ? r1 - r : (int64_t)SP_ROWS);
        e0 = P.row_ptr[r];
        if (P.row_ptr[r + hi] - e0 <= SP_ENT) {
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
        e1 = P.row_ptr[r + R];
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
    }
    return;
  }

  // ------------------------------------------------------------------ consumer warps
  const int jw0 = P.warp_j0[u * (SP_WARPS + 1) + warp], jw1 = P.warp_j0[u * (SP_WARPS + 1) + warp + 1];
  const bool own_pp = jw0 <= p && p < jw1;   // this warp owns the (p, p) entry: y^T y
  int st = 0;
  uint32_t ph = 0;
  for (;;) {
    mbar_wait(&full[st], ph);
    const unsigned char* sb = sbytes + (size_t)st * SP_STAGE_BYTES;
    const int* h = reinterpret_cast<const int*>(sb + SpStage::hdr);
    const int R = h[0];
    if (R == 0) break;
    const int64_t e0 = *reinterpret_cast<const int64_t*>(h + 2);
    const int64_t* rp_s = reinterpret_cast<const int64_t*>(sb + SpStage::rp);
    const double* y_s = reinterpret_cast<const double*>(sb + SpStage::y);
    const double* v_s = reinterpret_cast<const double*>(sb + SpStage::val);
    const int32_t* c_s = reinterpret_cast<const int32_t*>(sb + SpStage::col);
    if (jw0 < jw1) {
      for (int q0 = 0; q0 < R; q0 += 32) {
        const int q = q0 + lane;
        // this lane's row: entries [a, end) of the stage, the first one with column >= jw0
        int a = 0, end = 0, b = 0, phase = 2;  // phase 0: pairs (j_a, k_b) / (j_a, p); 1: (p, p); 2: done
        double yq = 0.0;
        if (q < R) {
          a = (int)(rp_s[q] - e0);
          end = (int)(rp_s[q + 1] - e0);
          yq = y_s[q];
          while (a < end && c_s[a] < jw0) ++a;
          if (a < end && c_s[a] < jw1) { phase = 0; b = a; }
          else phase = own_pp ? 1 : 2;
        }
        for (;;) {
          const bool has = phase < 2;
          const unsigned act = __ballot_sync(0xffffffffu, has);
          if (!act) break;
          if (has) {
            int64_t key;
            double prod;
            if (phase == 0) {
              const int j = c_s[a];
              const double va = v_s[a];
              const bool isy = b == end;
              const int k = isy ? p : c_s[b];
              prod = va * (isy ? yq : v_s[b]);
              key = tri_off(j, pa) + (k - j);
            } else {
              prod = yq * yq;
              key = tri_off(p, pa);
            }
            const unsigned grp = __match_any_sync(act, (unsigned long long)key);
            const int leader = __ffs(grp) - 1;
            double s = prod;
            if (grp != (1u << lane)) {   // lanes of one group sum in lane order (fixed)
              s = 0.0;
              unsigned m = grp;
              while (m) {
                const int src = __ffs(m) - 1;
                m &= m - 1;
                s += __shfl_sync(grp, prod, src);
              }
            }
            if (lane == leader) gs[key - base] += s;
            // advance
            if (phase == 0) {
              if (++b > end) {
                ++a;
                if (a < end && c_s[a] < jw1) b = a;
                else phase = own_pp ? 1 : 2;
              }
            } else {
              phase = 2;
            }
          }
        }
      }
    }
    __syncwarp();
    if (lane == 0) mbar_arrive(&empty[st]);
    if (++st == SP_ST) { st = 0; ph ^= 1u; }
  }
  // epilogue: this warp's entries of the slice -> the segment's partial
  const int64_t a0 = tri_off(jw0, pa) - base, a1 = tri_off(jw1, pa) - base;
  double* out = P.partial + ((size_t)u * P.nseg + seg) * P.cap;
  for (int64_t e = a0 + lane; e < a1; e += 32) out[e] = gs[e];
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
  // slices of the packed triangle (rows of Z^T Z) that fit the shared memory beside the ring
  const int64_t cap_max = (int64_t)(SP_SMEM_MAX - (size_t)SP_ST * SP_STAGE_BYTES - 1024) / 8;
  std::vector<int> sj{0};
  {
    int64_t cur = 0;
    for (int j = 0; j <= p; ++j) {
      const int64_t len = pa - j;
      if (cur + len > cap_max) { sj.push_back(j); cur = 0; }
      cur += len;
    }
    sj.push_back(p + 1);
  }
  const int U = (int)sj.size() - 1;
  int64_t cap = 0;
  for (int u = 0; u < U; ++u) {
    const int64_t a = sj[u], b = sj[u + 1];
    cap = std::max<int64_t>(cap, (b * pa - b * (b - 1) / 2) - (a * pa - a * (a - 1) / 2));
  }
  // consumer warps of a slice split its triangle rows evenly (the work of row j is ~ the
  // nonzeros of column j, uniform for the paper's random patterns)
  std::vector<int> wj((size_t)U * (SP_WARPS + 1));
  for (int u = 0; u < U; ++u)
    for (int w = 0; w <= SP_WARPS; ++w) wj[(size_t)u * (SP_WARPS + 1) + w] = sj[u] + (int)((int64_t)(sj[u + 1] - sj[u]) * w / SP_WARPS);
  const int nseg = (int)std::max<int64_t>(1, std::min<int64_t>((n_local + 1023) / 1024, std::max(1, ctx->num_sms / U)));
  const int64_t seg_rows = n_local > 0 ? (n_local + nseg - 1) / nseg : 1;
  // workspace: partial [U][nseg][cap] | packed | tables
  size_t off = 0;
  auto take = [&](size_t bytes) { size_t o = off; off += (bytes + 255) / 256 * 256; return o; };
  const size_t o_part = take(sizeof(double) * (size_t)U * nseg * cap);
  const size_t o_pack = take(sizeof(double) * (size_t)(psize + 2));
  const size_t o_sj = take(sizeof(int) * sj.size());
  const size_t o_wj = take(sizeof(int) * wj.size());
  OEM_CUDA_TRY(ctx->sparse_ws.ensure(off));
  char* base = ctx->sparse_ws.as<char>();
  OEM_CUDA_TRY(cudaMemcpyAsync(base + o_sj, sj.data(), sizeof(int) * sj.size(), cudaMemcpyHostToDevice, st));
  OEM_CUDA_TRY(cudaMemcpyAsync(base + o_wj, wj.data(), sizeof(int) * wj.size(), cudaMemcpyHostToDevice, st));
  double* packed = reinterpret_cast<double*>(base + o_pack);
  if (n_local == 0) {
    OEM_CUDA_TRY(cudaMemsetAsync(packed, 0, sizeof(double) * psize, st));
  } else {
    SpParams P;
    P.row_ptr = row_ptr; P.col = col; P.val = val; P.y = y; P.n = n_local; P.p = p; P.U = U; P.nseg = nseg;
    P.seg_rows = seg_rows;
    P.slice_j0 = reinterpret_cast<int*>(base + o_sj);
    P.warp_j0 = reinterpret_cast<int*>(base + o_wj);
    P.cap = (int)cap;
    P.partial = reinterpret_cast<double*>(base + o_part);
    const size_t smem = (size_t)SP_ST * SP_STAGE_BYTES + (size_t)cap * 8;
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
