// datagen_cuda.cu — device implementation of the seeded input generator (include/oem_datagen.h).
//
// Not part of the method. Written separately from datagen_host.c from the same specification;
// every floating-point operation is an explicit round-to-nearest intrinsic (__dmul_rn,
// __dadd_rn, __ddiv_rn, __dsqrt_rn) so no FMA contraction can change the bits, and X, y match
// the host generator exactly. Untimed: it only makes the inputs resident in HBM.
#include <cuda_runtime.h>
#include <stdint.h>

#include "../include/oem_datagen.h"

namespace {

__device__ __forceinline__ void philox(uint64_t seed, uint32_t a, uint32_t b, uint32_t c, uint32_t s, uint32_t w[4]) {
  uint32_t c0 = a, c1 = b, c2 = c, c3 = s;
  uint32_t k0 = (uint32_t)(seed & 0xffffffffu), k1 = (uint32_t)(seed >> 32);
#pragma unroll
  for (int r = 0; r < 10; ++r) {
    if (r > 0) { k0 += 0x9E3779B9u; k1 += 0xBB67AE85u; }
    const uint32_t hi0 = __umulhi(0xD2511F53u, c0), lo0 = 0xD2511F53u * c0;
    const uint32_t hi1 = __umulhi(0xCD9E8D57u, c2), lo1 = 0xCD9E8D57u * c2;
    const uint32_t n0 = hi1 ^ c1 ^ k0, n2 = hi0 ^ c3 ^ k1;
    c0 = n0; c1 = lo1; c2 = n2; c3 = lo0;
  }
  w[0] = c0; w[1] = c1; w[2] = c2; w[3] = c3;
}

__device__ __forceinline__ double uniform01(uint32_t wa, uint32_t wb) {
  const uint64_t k = ((((uint64_t)wa) << 32) | (uint64_t)wb) >> 12;
  return __dmul_rn(__ull2double_rn(2 * k + 1), 0x1.0p-53);
}

#define MUL __dmul_rn
#define ADD __dadd_rn
#define SUB __dsub_rn
#define DIV __ddiv_rn

__device__ double ln_sw(double x) {
  int e;
  double m = frexp(x, &e);
  if (m < 0x1.6a09e667f3bcdp-1) { m = MUL(m, 2.0); e = e - 1; }
  const double s = DIV(SUB(m, 1.0), ADD(m, 1.0));
  const double s2 = MUL(s, s);
  double t = 0x1.642c8590b2164p-5;
  t = ADD(MUL(t, s2), 0x1.8618618618618p-5);
  t = ADD(MUL(t, s2), 0x1.af286bca1af28p-5);
  t = ADD(MUL(t, s2), 0x1.e1e1e1e1e1e1ep-5);
  t = ADD(MUL(t, s2), 0x1.1111111111111p-4);
  t = ADD(MUL(t, s2), 0x1.3b13b13b13b14p-4);
  t = ADD(MUL(t, s2), 0x1.745d1745d1746p-4);
  t = ADD(MUL(t, s2), 0x1.c71c71c71c71cp-4);
  t = ADD(MUL(t, s2), 0x1.2492492492492p-3);
  t = ADD(MUL(t, s2), 0x1.999999999999ap-3);
  t = ADD(MUL(t, s2), 0x1.5555555555555p-2);
  t = ADD(MUL(t, s2), 1.0);
  const double lnm = MUL(MUL(2.0, s), t);
  return ADD(MUL((double)e, 0x1.62e42fefa39efp-1), lnm);
}

__device__ double exp_sw(double x) {
  if (x > 700.0) return __longlong_as_double(0x7ff0000000000000LL);
  if (x < -740.0) return 0.0;
  const double k = floor(ADD(MUL(x, 0x1.71547652b82fep+0), 0.5));
  const double r = SUB(SUB(x, MUL(k, 0x1.62e4200000000p-1)), MUL(k, 0x1.fdf473de00000p-22));
  double t = 0x1.6124613a86d09p-33;
  t = ADD(MUL(t, r), 0x1.1eed8eff8d898p-29);
  t = ADD(MUL(t, r), 0x1.ae64567f544e4p-26);
  t = ADD(MUL(t, r), 0x1.27e4fb7789f5cp-22);
  t = ADD(MUL(t, r), 0x1.71de3a556c734p-19);
  t = ADD(MUL(t, r), 0x1.a01a01a01a01ap-16);
  t = ADD(MUL(t, r), 0x1.a01a01a01a01ap-13);
  t = ADD(MUL(t, r), 0x1.6c16c16c16c17p-10);
  t = ADD(MUL(t, r), 0x1.1111111111111p-7);
  t = ADD(MUL(t, r), 0x1.5555555555555p-5);
  t = ADD(MUL(t, r), 0x1.5555555555555p-3);
  t = ADD(MUL(t, r), 0x1.0000000000000p-1);
  t = ADD(MUL(t, r), 1.0);
  t = ADD(MUL(t, r), 1.0);
  return ldexp(t, (int)k);
}

__device__ void sincos_quarter(double a, double* s, double* c) {
  const double a2 = MUL(a, a);
  double ps = 0x1.952c77030ad4ap-49;
  ps = ADD(MUL(ps, a2), -0x1.ae7f3e733b81fp-41);
  ps = ADD(MUL(ps, a2), 0x1.6124613a86d09p-33);
  ps = ADD(MUL(ps, a2), -0x1.ae64567f544e4p-26);
  ps = ADD(MUL(ps, a2), 0x1.71de3a556c734p-19);
  ps = ADD(MUL(ps, a2), -0x1.a01a01a01a01ap-13);
  ps = ADD(MUL(ps, a2), 0x1.1111111111111p-7);
  ps = ADD(MUL(ps, a2), -0x1.5555555555555p-3);
  *s = ADD(a, MUL(MUL(a, a2), ps));
  double pc = -0x1.6827863b97d97p-53;
  pc = ADD(MUL(pc, a2), 0x1.ae7f3e733b81fp-45);
  pc = ADD(MUL(pc, a2), -0x1.93974a8c07c9dp-37);
  pc = ADD(MUL(pc, a2), 0x1.1eed8eff8d898p-29);
  pc = ADD(MUL(pc, a2), -0x1.27e4fb7789f5cp-22);
  pc = ADD(MUL(pc, a2), 0x1.a01a01a01a01ap-16);
  pc = ADD(MUL(pc, a2), -0x1.6c16c16c16c17p-10);
  pc = ADD(MUL(pc, a2), 0x1.5555555555555p-5);
  pc = ADD(MUL(pc, a2), -0x1.0000000000000p-1);
  *c = ADD(1.0, MUL(a2, pc));
}

__device__ void sincos2pi_sw(double u, double* s, double* c) {
  const double t = MUL(u, 4.0);
  const int q = (int)t;
  const double f = SUB(t, (double)q);
  const bool swap = f > 0.5;
  const double h = swap ? SUB(1.0, f) : f;
  double sa, ca;
  sincos_quarter(MUL(h, 0x1.921fb54442d18p+0), &sa, &ca);
  const double sq = swap ? ca : sa, cq = swap ? sa : ca;
  switch (q & 3) {
    case 0: *s = sq; *c = cq; break;
    case 1: *s = cq; *c = -sq; break;
    case 2: *s = -sq; *c = -cq; break;
    default: *s = -cq; *c = sq; break;
  }
}

__device__ void normal_pair(const uint32_t w[4], double* z0, double* z1) {
  const double u1 = uniform01(w[0], w[1]);
  const double u2 = uniform01(w[2], w[3]);
  const double r = __dsqrt_rn(MUL(-2.0, ln_sw(u1)));
  double s, c;
  sincos2pi_sw(u2, &s, &c);
  *z0 = MUL(r, c);
  *z1 = MUL(r, s);
}

// SPARSE: the pattern draw u_ij of stream 5 (words 0,1 for even j, 2,3 for odd j) is < d
__device__ __forceinline__ bool kept(const dg_spec& sp, uint64_t gi, int j) {
  uint32_t w[4];
  philox(sp.seed, (uint32_t)gi, (uint32_t)(gi >> 32), (uint32_t)(j >> 1), 5u, w);
  const double u = (j & 1) ? uniform01(w[2], w[3]) : uniform01(w[0], w[1]);
  return u < sp.rho;
}

constexpr int ROWS = 128, CH = 32;

__global__ void __launch_bounds__(ROWS) rows_kernel(dg_spec sp, const double* __restrict__ beta, int64_t row0,
                                                     int64_t nrows, double* __restrict__ X, int64_t ldx,
                                                     double* __restrict__ y) {
  __shared__ double tile[ROWS][CH + 1];
  const int t = threadIdx.x;
  const int64_t rb = (int64_t)blockIdx.x * ROWS;
  const int64_t r = rb + t;
  const bool active = r < nrows;
  const uint64_t gi = (uint64_t)(row0 + r);
  const int p = sp.p;
  const double sq_rho = __dsqrt_rn(SUB(1.0, MUL(sp.rho, sp.rho)));
  const double sq_r = __dsqrt_rn(sp.rho), sq_1r = __dsqrt_rn(SUB(1.0, sp.rho));
  double z0 = 0, z1 = 0, g0 = 0, g1 = 0, prev = 0.0, eta = 0.0;
  int64_t gpair = -1;
  for (int c0 = 0; c0 < p; c0 += CH) {
    if (active) {
      for (int jj = 0; jj < CH && c0 + jj < p; ++jj) {
        const int j = c0 + jj;
        if ((j & 1) == 0) {
          uint32_t w[4];
          philox(sp.seed, (uint32_t)gi, (uint32_t)(gi >> 32), (uint32_t)(j >> 1), 0u, w);
          normal_pair(w, &z0, &z1);
        }
        const double z = (j & 1) ? z1 : z0;
        double x;
        if (sp.design == DG_AR1) {
          x = (j == 0) ? z : ADD(MUL(sp.rho, prev), MUL(sq_rho, z));
          prev = x;
        } else if (sp.design == DG_BLOCK) {
          const int k = j / sp.group_size;
          if ((k >> 1) != gpair) {
            uint32_t w[4];
            philox(sp.seed, (uint32_t)gi, (uint32_t)(gi >> 32), (uint32_t)(k >> 1), 1u, w);
            normal_pair(w, &g0, &g1);
            gpair = k >> 1;
          }
          x = ADD(MUL(sq_r, (k & 1) ? g1 : g0), MUL(sq_1r, z));
        } else if (sp.design == DG_SPARSE) {
          x = kept(sp, gi, j) ? z : 0.0;
        } else {
          x = z;
        }
        tile[t][jj] = x;
        const double b = beta[j];
        if (b != 0.0) eta = ADD(eta, MUL(x, b));
      }
    }
    __syncthreads();
    for (int e = t; e < ROWS * CH; e += ROWS) {
      const int rr = e / CH, cc = e % CH;
      if (rb + rr < nrows && c0 + cc < p) X[(rb + rr) * ldx + c0 + cc] = tile[rr][cc];
    }
    __syncthreads();
  }
  if (active && y) {
    uint32_t w[4];
    if (sp.response == DG_LINEAR) {
      philox(sp.seed, (uint32_t)gi, (uint32_t)(gi >> 32), 0u, 2u, w);
      double e0, e1;
      normal_pair(w, &e0, &e1);
      y[r] = ADD(eta, MUL(sp.sigma, e0));
    } else {
      philox(sp.seed, (uint32_t)gi, (uint32_t)(gi >> 32), 0u, 4u, w);
      const double u = uniform01(w[0], w[1]);
      const double pr = DIV(1.0, ADD(1.0, exp_sw(-eta)));
      y[r] = (u < pr) ? 1.0 : 0.0;
    }
  }
}

// SPARSE in CSR form: one thread per row (the pattern of a row is a pure function of (i, j))
__global__ void csr_count_kernel(dg_spec sp, int64_t row0, int64_t nrows, int64_t* __restrict__ counts) {
  const int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (r >= nrows) return;
  const uint64_t gi = (uint64_t)(row0 + r);
  int64_t c = 0;
  for (int j = 0; j < sp.p; ++j) c += kept(sp, gi, j) ? 1 : 0;
  counts[r] = c;
}

__global__ void csr_fill_kernel(dg_spec sp, const double* __restrict__ beta, int64_t row0, int64_t nrows,
                                const int64_t* __restrict__ row_ptr, int32_t* __restrict__ col,
                                double* __restrict__ val, double* __restrict__ y) {
  const int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (r >= nrows) return;
  const uint64_t gi = (uint64_t)(row0 + r);
  int64_t e = row_ptr[r];
  double eta = 0.0, z0 = 0.0, z1 = 0.0;
  int drawn = -1;   // column pair whose normals z0, z1 hold
  for (int j = 0; j < sp.p; ++j) {
    if (!kept(sp, gi, j)) continue;
    if ((j >> 1) != drawn) {
      uint32_t w[4];
      philox(sp.seed, (uint32_t)gi, (uint32_t)(gi >> 32), (uint32_t)(j >> 1), 0u, w);
      normal_pair(w, &z0, &z1);
      drawn = j >> 1;
    }
    const double x = (j & 1) ? z1 : z0;
    col[e] = j;
    val[e] = x;
    ++e;
    const double b = beta ? beta[j] : 0.0;
    if (b != 0.0) eta = ADD(eta, MUL(x, b));
  }
  if (y) {
    uint32_t w[4];
    if (sp.response == DG_LINEAR) {
      philox(sp.seed, (uint32_t)gi, (uint32_t)(gi >> 32), 0u, 2u, w);
      double e0, e1;
      normal_pair(w, &e0, &e1);
      y[r] = ADD(eta, MUL(sp.sigma, e0));
    } else {
      philox(sp.seed, (uint32_t)gi, (uint32_t)(gi >> 32), 0u, 4u, w);
      const double u = uniform01(w[0], w[1]);
      const double pr = DIV(1.0, ADD(1.0, exp_sw(-eta)));
      y[r] = (u < pr) ? 1.0 : 0.0;
    }
  }
}

}  // namespace

extern "C" int dg_csr_count_cuda(const dg_spec* spec, int64_t row0, int64_t nrows, int64_t* counts, void* stream) {
  if (!spec || spec->design != DG_SPARSE || !counts || nrows < 0 || row0 < 0 || spec->p < 1) return -1;
  if (nrows == 0) return 0;
  csr_count_kernel<<<(unsigned)((nrows + 255) / 256), 256, 0, (cudaStream_t)stream>>>(*spec, row0, nrows, counts);
  return cudaGetLastError() == cudaSuccess ? 0 : -2;
}

extern "C" int dg_csr_fill_cuda(const dg_spec* spec, const double* beta, int64_t row0, int64_t nrows,
                                const int64_t* row_ptr, int32_t* col, double* val, double* y, void* stream) {
  if (!spec || spec->design != DG_SPARSE || !row_ptr || !col || !val || nrows < 0 || row0 < 0 || spec->p < 1) return -1;
  if (y && !beta) return -1;
  if (nrows == 0) return 0;
  csr_fill_kernel<<<(unsigned)((nrows + 255) / 256), 256, 0, (cudaStream_t)stream>>>(*spec, beta, row0, nrows, row_ptr,
                                                                                      col, val, y);
  return cudaGetLastError() == cudaSuccess ? 0 : -2;
}

extern "C" int dg_rows_cuda(const dg_spec* spec, const double* beta, int64_t row0, int64_t nrows, double* X,
                            int64_t ldx, double* y, void* stream) {
  if (!spec || !beta || !X || nrows < 0 || row0 < 0 || ldx < spec->p || spec->p < 1) return -1;
  if (spec->design < 0 || spec->design > 3 || spec->response < 0 || spec->response > 1) return -1;
  if (spec->design == DG_BLOCK && spec->group_size < 1) return -1;
  if (nrows == 0) return 0;
  const int64_t blocks = (nrows + ROWS - 1) / ROWS;
  rows_kernel<<<(unsigned)blocks, ROWS, 0, (cudaStream_t)stream>>>(*spec, beta, row0, nrows, X, ldx, y);
  return cudaGetLastError() == cudaSuccess ? 0 : -2;
}
