/* datagen_host.c — host implementation of the seeded input generator (include/oem_datagen.h).
 *
 * Not part of the method: it draws X, beta and y for the paper's simulation designs
 * (§6.1 AR(1) Gaussian design; L1137-1149 §6.3 logistic design) and the
 * BASELINE.json configs. Compiled with -ffp-contract=off so every +,-,*,/ is one IEEE
 * round-to-nearest operation, matching the device implementation (datagen_cuda.cu) bit for bit.
 * Written separately from the device file, from the specification in oem_datagen.h.
 */
#include "../include/oem_datagen.h"

#include <math.h>
#include <stdlib.h>
#include <string.h>

/* ---------------- Philox4x32-10 ---------------- */
#define PHILOX_M0 0xD2511F53u
#define PHILOX_M1 0xCD9E8D57u
#define PHILOX_W0 0x9E3779B9u
#define PHILOX_W1 0xBB67AE85u

void dg_philox4x32_10(const uint32_t ctr[4], const uint32_t key[2], uint32_t out[4]) {
  uint32_t c0 = ctr[0], c1 = ctr[1], c2 = ctr[2], c3 = ctr[3];
  uint32_t k0 = key[0], k1 = key[1];
  for (int r = 0; r < 10; ++r) {
    if (r > 0) { k0 += PHILOX_W0; k1 += PHILOX_W1; }
    uint64_t p0 = (uint64_t)PHILOX_M0 * c0;
    uint64_t p1 = (uint64_t)PHILOX_M1 * c2;
    uint32_t n0 = (uint32_t)(p1 >> 32) ^ c1 ^ k0;
    uint32_t n1 = (uint32_t)p1;
    uint32_t n2 = (uint32_t)(p0 >> 32) ^ c3 ^ k1;
    uint32_t n3 = (uint32_t)p0;
    c0 = n0; c1 = n1; c2 = n2; c3 = n3;
  }
  out[0] = c0; out[1] = c1; out[2] = c2; out[3] = c3;
}

static void philox(uint64_t seed, uint32_t a, uint32_t b, uint32_t c, uint32_t s, uint32_t w[4]) {
  uint32_t ctr[4] = {a, b, c, s};
  uint32_t key[2] = {(uint32_t)(seed & 0xffffffffu), (uint32_t)(seed >> 32)};
  dg_philox4x32_10(ctr, key, w);
}

/* uniform in (0,1): k = 52 high bits of (wa:wb), u = (2k+1) * 2^-53 (exact). */
static double uniform01(uint32_t wa, uint32_t wb) {
  uint64_t k = ((((uint64_t)wa) << 32) | (uint64_t)wb) >> 12;
  return (double)(2 * k + 1) * 0x1.0p-53;
}

/* ---------------- software math: only +,-,*,/,sqrt ---------------- */
double dg_ln(double x) {
  int e;
  double m = frexp(x, &e);                 /* x = m * 2^e, m in [0.5, 1) */
  if (m < 0x1.6a09e667f3bcdp-1) { m = m * 2.0; e = e - 1; }
  double s = (m - 1.0) / (m + 1.0);
  double s2 = s * s;
  double t = 0x1.642c8590b2164p-5;         /* 1/23 */
  t = t * s2 + 0x1.8618618618618p-5;       /* 1/21 */
  t = t * s2 + 0x1.af286bca1af28p-5;       /* 1/19 */
  t = t * s2 + 0x1.e1e1e1e1e1e1ep-5;       /* 1/17 */
  t = t * s2 + 0x1.1111111111111p-4;       /* 1/15 */
  t = t * s2 + 0x1.3b13b13b13b14p-4;       /* 1/13 */
  t = t * s2 + 0x1.745d1745d1746p-4;       /* 1/11 */
  t = t * s2 + 0x1.c71c71c71c71cp-4;       /* 1/9 */
  t = t * s2 + 0x1.2492492492492p-3;       /* 1/7 */
  t = t * s2 + 0x1.999999999999ap-3;       /* 1/5 */
  t = t * s2 + 0x1.5555555555555p-2;       /* 1/3 */
  t = t * s2 + 1.0;
  double lnm = (2.0 * s) * t;
  return (double)e * 0x1.62e42fefa39efp-1 + lnm;
}

double dg_exp(double x) {
  if (x > 700.0) return INFINITY;
  if (x < -740.0) return 0.0;
  double k = floor(x * 0x1.71547652b82fep+0 + 0.5);
  double r = (x - k * 0x1.62e4200000000p-1) - k * 0x1.fdf473de00000p-22;
  double t = 0x1.6124613a86d09p-33;        /* 1/13! */
  t = t * r + 0x1.1eed8eff8d898p-29;       /* 1/12! */
  t = t * r + 0x1.ae64567f544e4p-26;       /* 1/11! */
  t = t * r + 0x1.27e4fb7789f5cp-22;       /* 1/10! */
  t = t * r + 0x1.71de3a556c734p-19;       /* 1/9! */
  t = t * r + 0x1.a01a01a01a01ap-16;       /* 1/8! */
  t = t * r + 0x1.a01a01a01a01ap-13;       /* 1/7! */
  t = t * r + 0x1.6c16c16c16c17p-10;       /* 1/6! */
  t = t * r + 0x1.1111111111111p-7;        /* 1/5! */
  t = t * r + 0x1.5555555555555p-5;        /* 1/4! */
  t = t * r + 0x1.5555555555555p-3;        /* 1/3! */
  t = t * r + 0x1.0000000000000p-1;        /* 1/2! */
  t = t * r + 1.0;
  t = t * r + 1.0;
  return ldexp(t, (int)k);
}

static void sincos_quarter(double a, double* s, double* c) {
  /* a in [0, pi/4] */
  double a2 = a * a;
  double ps = 0x1.952c77030ad4ap-49;
  ps = ps * a2 + -0x1.ae7f3e733b81fp-41;
  ps = ps * a2 + 0x1.6124613a86d09p-33;
  ps = ps * a2 + -0x1.ae64567f544e4p-26;
  ps = ps * a2 + 0x1.71de3a556c734p-19;
  ps = ps * a2 + -0x1.a01a01a01a01ap-13;
  ps = ps * a2 + 0x1.1111111111111p-7;
  ps = ps * a2 + -0x1.5555555555555p-3;
  *s = a + (a * a2) * ps;
  double pc = -0x1.6827863b97d97p-53;
  pc = pc * a2 + 0x1.ae7f3e733b81fp-45;
  pc = pc * a2 + -0x1.93974a8c07c9dp-37;
  pc = pc * a2 + 0x1.1eed8eff8d898p-29;
  pc = pc * a2 + -0x1.27e4fb7789f5cp-22;
  pc = pc * a2 + 0x1.a01a01a01a01ap-16;
  pc = pc * a2 + -0x1.6c16c16c16c17p-10;
  pc = pc * a2 + 0x1.5555555555555p-5;
  pc = pc * a2 + -0x1.0000000000000p-1;
  *c = 1.0 + a2 * pc;
}

void dg_sincos2pi(double u, double* s, double* c) {
  double t = u * 4.0;
  int q = (int)t;
  double f = t - (double)q;
  int swap = f > 0.5;
  double h = swap ? (1.0 - f) : f;
  double sa, ca;
  sincos_quarter(h * 0x1.921fb54442d18p+0, &sa, &ca);
  double sq = swap ? ca : sa, cq = swap ? sa : ca; /* sin/cos of f*pi/2 */
  switch (q & 3) {
    case 0: *s = sq; *c = cq; break;
    case 1: *s = cq; *c = -sq; break;
    case 2: *s = -sq; *c = -cq; break;
    default: *s = -cq; *c = sq; break;
  }
}

static void normal_pair(const uint32_t w[4], double* z0, double* z1) {
  double u1 = uniform01(w[0], w[1]);
  double u2 = uniform01(w[2], w[3]);
  double r = sqrt(-2.0 * dg_ln(u1));
  double s, c;
  dg_sincos2pi(u2, &s, &c);
  *z0 = r * c;
  *z1 = r * s;
}

/* ---------------- beta ---------------- */
static int spec_ok(const dg_spec* sp) {
  if (!sp || sp->n < 0 || sp->p < 1) return 0;
  if (sp->design < 0 || sp->design > 3) return 0;
  if (sp->design == DG_SPARSE && !(sp->rho >= 0.0 && sp->rho <= 1.0)) return 0;
  if (sp->design == DG_BLOCK && (sp->group_size < 1 || sp->rho < 0.0 || sp->rho > 1.0)) return 0;
  if (sp->design == DG_AR1 && !(sp->rho > -1.0 && sp->rho < 1.0)) return 0;
  if (sp->response < 0 || sp->response > 1) return 0;
  if (sp->beta_kind < 0 || sp->beta_kind > 3) return 0;
  if (sp->beta_kind == DG_BETA_ACTIVE_GROUPS &&
      (sp->group_size < 1 || sp->p % sp->group_size != 0 || sp->nnz > sp->p / sp->group_size)) return 0;
  if ((sp->beta_kind == DG_BETA_UNIFORM || sp->beta_kind == DG_BETA_NORMAL) && (sp->nnz < 0 || sp->nnz > sp->p)) return 0;
  return 1;
}

static double beta_value(const dg_spec* sp, uint32_t t) {
  uint32_t w[4];
  philox(sp->seed, t, 1u, 0u, 3u, w);
  if (sp->beta_kind == DG_BETA_UNIFORM) {
    double u = uniform01(w[0], w[1]);
    return sp->beta_lo + (sp->beta_hi - sp->beta_lo) * u;
  }
  double z0, z1;
  normal_pair(w, &z0, &z1);
  return z0;
}

static void fisher_yates(const dg_spec* sp, int32_t m, int32_t k, int32_t* perm) {
  for (int32_t j = 0; j < m; ++j) perm[j] = j;
  for (int32_t t = 0; t < k; ++t) {
    uint32_t w[4];
    philox(sp->seed, (uint32_t)t, 0u, 0u, 3u, w);
    int32_t j = t + (int32_t)(((uint64_t)w[0] * (uint64_t)(m - t)) >> 32);
    int32_t tmp = perm[t]; perm[t] = perm[j]; perm[j] = tmp;
  }
}

static int cmp_i32(const void* a, const void* b) {
  int32_t x = *(const int32_t*)a, y = *(const int32_t*)b;
  return (x > y) - (x < y);
}

int dg_beta(const dg_spec* sp, double* beta) {
  if (!spec_ok(sp) || !beta) return -1;
  if (sp->beta_kind == DG_BETA_EXPLICIT) return 0;
  for (int32_t j = 0; j < sp->p; ++j) beta[j] = 0.0;
  if (sp->beta_kind == DG_BETA_ACTIVE_GROUPS) {
    int32_t G = sp->p / sp->group_size;
    int32_t* perm = (int32_t*)malloc(sizeof(int32_t) * (size_t)G);
    if (!perm) return -1;
    fisher_yates(sp, G, sp->nnz, perm);
    qsort(perm, (size_t)sp->nnz, sizeof(int32_t), cmp_i32);
    uint32_t t = 0;
    for (int32_t a = 0; a < sp->nnz; ++a)
      for (int32_t j = perm[a] * sp->group_size; j < (perm[a] + 1) * sp->group_size; ++j)
        beta[j] = beta_value(sp, t++);
    free(perm);
    return 0;
  }
  int32_t* perm = (int32_t*)malloc(sizeof(int32_t) * (size_t)sp->p);
  if (!perm) return -1;
  fisher_yates(sp, sp->p, sp->nnz, perm);
  qsort(perm, (size_t)sp->nnz, sizeof(int32_t), cmp_i32);
  for (int32_t t = 0; t < sp->nnz; ++t) beta[perm[t]] = beta_value(sp, (uint32_t)t);
  free(perm);
  return 0;
}

/* ---------------- rows ---------------- */
typedef struct {
  int64_t cached_pair;   /* pair index of z cache, or -1 */
  double z0, z1;
  int64_t cached_gpair;
  double g0, g1;
} rowcache;

static double z_of(const dg_spec* sp, uint64_t gi, int32_t j, rowcache* rc) {
  int64_t m = j >> 1;
  if (rc->cached_pair != m) {
    uint32_t w[4];
    philox(sp->seed, (uint32_t)gi, (uint32_t)(gi >> 32), (uint32_t)m, 0u, w);
    normal_pair(w, &rc->z0, &rc->z1);
    rc->cached_pair = m;
  }
  return (j & 1) ? rc->z1 : rc->z0;
}

/* SPARSE: the pattern draw u_ij of stream 5 (words 0,1 for even j, 2,3 for odd j) */
static int kept(const dg_spec* sp, uint64_t gi, int32_t j) {
  uint32_t w[4];
  philox(sp->seed, (uint32_t)gi, (uint32_t)(gi >> 32), (uint32_t)(j >> 1), 5u, w);
  double u = (j & 1) ? uniform01(w[2], w[3]) : uniform01(w[0], w[1]);
  return u < sp->rho;
}

static double g_of(const dg_spec* sp, uint64_t gi, int32_t k, rowcache* rc) {
  int64_t m = k >> 1;
  if (rc->cached_gpair != m) {
    uint32_t w[4];
    philox(sp->seed, (uint32_t)gi, (uint32_t)(gi >> 32), (uint32_t)m, 1u, w);
    normal_pair(w, &rc->g0, &rc->g1);
    rc->cached_gpair = m;
  }
  return (k & 1) ? rc->g1 : rc->g0;
}

int dg_rows_host(const dg_spec* sp, const double* beta, int64_t row0, int64_t nrows,
                 int32_t col0, int32_t ncols, double* X, int64_t ldx, double* y) {
  if (!spec_ok(sp) || row0 < 0 || nrows < 0 || col0 < 0 || ncols < 0 || col0 + ncols > sp->p) return -1;
  if (ncols > 0 && (!X || ldx < ncols)) return -1;
  if (y && !beta) return -1;
  const int32_t p = sp->p;
  /* columns needed per row: requested range, plus every support column when y is wanted */
  char* need = (char*)calloc((size_t)p, 1);
  double* row = (double*)malloc(sizeof(double) * (size_t)p);
  if (!need || !row) { free(need); free(row); return -1; }
  int32_t jmax = col0 + ncols - 1;
  for (int32_t j = col0; j < col0 + ncols; ++j) need[j] = 1;
  if (y)
    for (int32_t j = 0; j < p; ++j)
      if (beta[j] != 0.0) { need[j] = 1; if (j > jmax) jmax = j; }
  const double sq_rho = sqrt(1.0 - sp->rho * sp->rho);
  const double sq_r = sqrt(sp->rho), sq_1r = sqrt(1.0 - sp->rho);
  for (int64_t r = 0; r < nrows; ++r) {
    uint64_t gi = (uint64_t)(row0 + r);
    rowcache rc = {-1, 0.0, 0.0, -1, 0.0, 0.0};
    if (sp->design == DG_AR1) {
      for (int32_t j = 0; j <= jmax; ++j) {
        double z = z_of(sp, gi, j, &rc);
        row[j] = (j == 0) ? z : sp->rho * row[j - 1] + sq_rho * z;
      }
    } else {
      for (int32_t j = 0; j <= jmax; ++j) {
        if (!need[j]) continue;
        double z = z_of(sp, gi, j, &rc);
        if (sp->design == DG_IID) row[j] = z;
        else if (sp->design == DG_SPARSE) row[j] = kept(sp, gi, j) ? z : 0.0;
        else row[j] = sq_r * g_of(sp, gi, j / sp->group_size, &rc) + sq_1r * z;
      }
    }
    for (int32_t j = 0; j < ncols; ++j) X[r * ldx + j] = row[col0 + j];
    if (y) {
      double eta = 0.0;
      for (int32_t j = 0; j <= jmax; ++j)
        if (beta[j] != 0.0) eta = eta + row[j] * beta[j];
      uint32_t w[4];
      if (sp->response == DG_LINEAR) {
        philox(sp->seed, (uint32_t)gi, (uint32_t)(gi >> 32), 0u, 2u, w);
        double e0, e1;
        normal_pair(w, &e0, &e1);
        y[r] = eta + sp->sigma * e0;
      } else {
        philox(sp->seed, (uint32_t)gi, (uint32_t)(gi >> 32), 0u, 4u, w);
        double u = uniform01(w[0], w[1]);
        double pr = 1.0 / (1.0 + dg_exp(-eta));
        y[r] = (u < pr) ? 1.0 : 0.0;
      }
    }
  }
  free(need);
  free(row);
  return 0;
}
