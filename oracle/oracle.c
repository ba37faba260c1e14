/* oracle.c — plain CPU reference of the OEM hot path. TEST INFRASTRUCTURE ONLY (see oracle.h).
 *
 * Deliberately naive: triple loops, no blocking, no fusion, one formula per line in the paper's
 * order and notation. Sums over the n rows use compensated accumulation of exact products so
 * that the comparison against the GPU measures the GPU's rounding, not the oracle's.
 */
#include "oracle.h"

#include <math.h>
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

/* ---------------- compensated accumulation ----------------
 * acc = (s, c): value s + c. add_prod adds a*b exactly up to one final rounding: the product
 * is split into p = fl(a*b) and its exact error e = fma(a, b, -p) (TwoProduct), p is added with
 * Neumaier's TwoSum-style compensation and e goes straight into the compensation term. */
static inline void acc_add(double* s, double* c, double x) {
  double t = *s + x;
  if (fabs(*s) >= fabs(x)) *c += (*s - t) + x;
  else *c += (x - t) + *s;
  *s = t;
}
static inline void acc_add_prod(double* s, double* c, double a, double b) {
  double p = a * b;
  double e = fma(a, b, -p);
  acc_add(s, c, p);
  *c += e;
}

/* ---------------- O1 Gram ---------------- */
/* state layout: [Gs p*p][Gc p*p][xs p][xc p][ys 1][yc 1] */
void orc_gram_begin(int32_t p, double* state) {
  memset(state, 0, sizeof(double) * 2 * ((size_t)p * p + p + 1));
}

static void gram_rows(const double* X, const double* y, int64_t r0, int64_t r1, int32_t p, int64_t ldx,
                      double* Gs, double* Gc, double* xs, double* xc, double* ys, double* yc) {
  for (int64_t i = r0; i < r1; ++i) {
    const double* xi = X + i * ldx;
    for (int32_t j = 0; j < p; ++j) {
      for (int32_t k = j; k < p; ++k) acc_add_prod(&Gs[(size_t)j * p + k], &Gc[(size_t)j * p + k], xi[j], xi[k]);
      acc_add_prod(&xs[j], &xc[j], xi[j], y[i]);
    }
    acc_add_prod(ys, yc, y[i], y[i]);
  }
}

void orc_gram_add(const double* X, const double* y, int64_t n, int32_t p, int64_t ldx, double* state,
                  int nthreads) {
  size_t pp = (size_t)p * p;
  if (nthreads < 1) nthreads = 1;
  if ((int64_t)nthreads > n) nthreads = n > 0 ? (int)n : 1;
  size_t per = 2 * (pp + p + 1);
  double* part = (double*)calloc(per * (size_t)nthreads, sizeof(double));
  /* static row blocks, one per thread; merged below in thread order (deterministic) */
#pragma omp parallel for num_threads(nthreads) schedule(static, 1)
  for (int t = 0; t < nthreads; ++t) {
    int64_t r0 = n * t / nthreads, r1 = n * (t + 1) / nthreads;
    double* b = part + per * (size_t)t;
    gram_rows(X, y, r0, r1, p, ldx, b, b + pp, b + 2 * pp, b + 2 * pp + p, b + 2 * pp + 2 * p,
              b + 2 * pp + 2 * p + 1);
  }
  double *Gs = state, *Gc = state + pp, *xs = state + 2 * pp, *xc = xs + p, *ys = xc + p, *yc = ys + 1;
  for (int t = 0; t < nthreads; ++t) {
    double* b = part + per * (size_t)t;
    for (size_t q = 0; q < pp; ++q) { acc_add(&Gs[q], &Gc[q], b[q]); acc_add(&Gs[q], &Gc[q], b[pp + q]); }
    for (int32_t j = 0; j < p; ++j) { acc_add(&xs[j], &xc[j], b[2 * pp + j]); acc_add(&xs[j], &xc[j], b[2 * pp + p + j]); }
    acc_add(ys, yc, b[2 * pp + 2 * p]);
    acc_add(ys, yc, b[2 * pp + 2 * p + 1]);
  }
  free(part);
}

void orc_gram_end(int32_t p, const double* state, double* G, double* xty, double* yty) {
  size_t pp = (size_t)p * p;
  const double *Gs = state, *Gc = state + pp, *xs = state + 2 * pp, *xc = xs + p, *ys = xc + p, *yc = ys + 1;
  for (int32_t j = 0; j < p; ++j)
    for (int32_t k = j; k < p; ++k) {
      double v = Gs[(size_t)j * p + k] + Gc[(size_t)j * p + k];
      G[(size_t)j * p + k] = v;
      G[(size_t)k * p + j] = v; /* symmetric: the upper sum is the definition, mirrored */
    }
  for (int32_t j = 0; j < p; ++j) xty[j] = xs[j] + xc[j];
  *yty = *ys + *yc;
}

void orc_gram(const double* X, const double* y, int64_t n, int32_t p, int64_t ldx, double* G,
              double* xty, double* yty, int nthreads) {
  double* st = (double*)malloc(sizeof(double) * 2 * ((size_t)p * p + p + 1));
  orc_gram_begin(p, st);
  orc_gram_add(X, y, n, p, ldx, st, nthreads);
  orc_gram_end(p, st, G, xty, yty);
  free(st);
}

/* ---------------- O2 fold Grams ---------------- */
void orc_gram_folds(const double* X, const double* y, int64_t n, int32_t p, int64_t ldx,
                    int64_t row_offset, int32_t K, double* Gk, double* xtyk, double* ytyk,
                    int64_t* counts, int nthreads) {
  size_t pp = (size_t)p * p;
  /* rows of fold k gathered into a contiguous copy, then O1 on that copy */
  for (int32_t k = 0; k < K; ++k) {
    int64_t nk = 0;
    for (int64_t i = 0; i < n; ++i)
      if ((row_offset + i) % K == k) ++nk;
    double* Xk = (double*)malloc(sizeof(double) * (size_t)(nk > 0 ? nk : 1) * (size_t)p);
    double* yk = (double*)malloc(sizeof(double) * (size_t)(nk > 0 ? nk : 1));
    int64_t r = 0;
    for (int64_t i = 0; i < n; ++i)
      if ((row_offset + i) % K == k) {
        memcpy(Xk + r * p, X + i * ldx, sizeof(double) * (size_t)p);
        yk[r] = y[i];
        ++r;
      }
    orc_gram(Xk, yk, nk, p, p, Gk + (size_t)k * pp, xtyk + (size_t)k * p, ytyk + k, nthreads);
    counts[k] = nk;
    free(Xk);
    free(yk);
  }
}

void orc_fold_complements(const double* Gk, const double* xtyk, int32_t K, int32_t p,
                          double* Gminus, double* xtyminus) {
  size_t pp = (size_t)p * p;
  for (int32_t k = 0; k < K; ++k) {
    for (size_t q = 0; q < pp; ++q) {
      double s = 0.0, c = 0.0;
      for (int32_t m = 0; m < K; ++m)
        if (m != k) acc_add(&s, &c, Gk[(size_t)m * pp + q]);
      Gminus[(size_t)k * pp + q] = s + c;
    }
    for (int32_t j = 0; j < p; ++j) {
      double s = 0.0, c = 0.0;
      for (int32_t m = 0; m < K; ++m)
        if (m != k) acc_add(&s, &c, xtyk[(size_t)m * p + j]);
      xtyminus[(size_t)k * p + j] = s + c;
    }
  }
}

/* ---------------- O3 weighted Gram ---------------- */
static double softplus(double eta) { /* log(1 + exp(eta)), evaluated without overflow */
  return eta > 0.0 ? eta + log1p(exp(-eta)) : log1p(exp(eta));
}

void orc_gram_weighted(const double* X, const double* y01, const double* beta, int64_t n, int32_t p,
                       int64_t ldx, double eps, double* Gw, double* cw, double* scalars, int nthreads) {
  size_t pp = (size_t)p * p;
  if (nthreads < 1) nthreads = 1;
  if ((int64_t)nthreads > n) nthreads = n > 0 ? (int)n : 1;
  size_t per = 2 * (pp + p + 2);
  double* part = (double*)calloc(per * (size_t)nthreads, sizeof(double));
#pragma omp parallel for num_threads(nthreads) schedule(static, 1)
  for (int t = 0; t < nthreads; ++t) {
    int64_t r0 = n * t / nthreads, r1 = n * (t + 1) / nthreads;
    double* b = part + per * (size_t)t;
    double *Gs = b, *Gc = b + pp, *xs = b + 2 * pp, *xc = xs + p, *sc = xc + p; /* sc: sw, swc, ll, llc */
    for (int64_t i = r0; i < r1; ++i) {
      const double* xi = X + i * ldx;
      double eta = 0.0;
      for (int32_t j = 0; j < p; ++j) eta += xi[j] * beta[j];
      double mu = 1.0 / (1.0 + exp(-eta));
      if (mu < eps) mu = eps;
      if (mu > 1.0 - eps) mu = 1.0 - eps;
      double w = mu * (1.0 - mu);
      double z = eta + (y01[i] - mu) / w;
      for (int32_t j = 0; j < p; ++j) {
        double wxj = w * xi[j];
        for (int32_t k = j; k < p; ++k) acc_add_prod(&Gs[(size_t)j * p + k], &Gc[(size_t)j * p + k], wxj, xi[k]);
        acc_add_prod(&xs[j], &xc[j], wxj, z);
      }
      acc_add(&sc[0], &sc[1], w);
      acc_add(&sc[2], &sc[3], y01[i] * eta - softplus(eta));
    }
  }
  for (size_t q = 0; q < pp; ++q) Gw[q] = 0.0;
  double fs[2 * 2] = {0, 0, 0, 0};
  double* Gs = (double*)calloc(2 * pp + 2 * (size_t)p, sizeof(double));
  for (int t = 0; t < nthreads; ++t) {
    double* b = part + per * (size_t)t;
    for (size_t q = 0; q < pp; ++q) { acc_add(&Gs[q], &Gs[pp + q], b[q]); acc_add(&Gs[q], &Gs[pp + q], b[pp + q]); }
    for (int32_t j = 0; j < p; ++j) {
      acc_add(&Gs[2 * pp + j], &Gs[2 * pp + p + j], b[2 * pp + j]);
      acc_add(&Gs[2 * pp + j], &Gs[2 * pp + p + j], b[2 * pp + p + j]);
    }
    double* sc = b + 2 * pp + 2 * p;
    acc_add(&fs[0], &fs[1], sc[0]); acc_add(&fs[0], &fs[1], sc[1]);
    acc_add(&fs[2], &fs[3], sc[2]); acc_add(&fs[2], &fs[3], sc[3]);
  }
  for (int32_t j = 0; j < p; ++j)
    for (int32_t k = j; k < p; ++k) {
      double v = Gs[(size_t)j * p + k] + Gs[pp + (size_t)j * p + k];
      Gw[(size_t)j * p + k] = v;
      Gw[(size_t)k * p + j] = v;
    }
  for (int32_t j = 0; j < p; ++j) cw[j] = Gs[2 * pp + j] + Gs[2 * pp + p + j];
  scalars[0] = fs[0] + fs[1];
  scalars[1] = fs[2] + fs[3];
  free(Gs);
  free(part);
}

/* ---------------- O4 eigenvalues / d ---------------- */
void orc_eig_jacobi(const double* A0, int32_t p, double* evals) {
  /* cyclic Jacobi rotations (Golub & Van Loan, Alg. 8.5.3) until the off-diagonal is negligible */
  double* A = (double*)malloc(sizeof(double) * (size_t)p * p);
  memcpy(A, A0, sizeof(double) * (size_t)p * p);
  for (int sweep = 0; sweep < 100; ++sweep) {
    double off = 0.0, tot = 0.0;
    for (int32_t i = 0; i < p; ++i)
      for (int32_t j = 0; j < p; ++j) {
        double a = A[(size_t)i * p + j] * A[(size_t)i * p + j];
        tot += a;
        if (i != j) off += a;
      }
    if (off <= 1e-34 * tot || off == 0.0) break;
    for (int32_t q = 0; q < p; ++q)
      for (int32_t r = q + 1; r < p; ++r) {
        double aqr = A[(size_t)q * p + r];
        if (aqr == 0.0) continue;
        double aqq = A[(size_t)q * p + q], arr = A[(size_t)r * p + r];
        double tau = (arr - aqq) / (2.0 * aqr);
        double t = (tau >= 0.0 ? 1.0 : -1.0) / (fabs(tau) + sqrt(1.0 + tau * tau));
        double c = 1.0 / sqrt(1.0 + t * t), s = t * c;
        for (int32_t k = 0; k < p; ++k) { /* A <- A J (columns q, r) */
          double akq = A[(size_t)k * p + q], akr = A[(size_t)k * p + r];
          A[(size_t)k * p + q] = c * akq - s * akr;
          A[(size_t)k * p + r] = s * akq + c * akr;
        }
        for (int32_t k = 0; k < p; ++k) { /* A <- J^T A (rows q, r) */
          double aqk = A[(size_t)q * p + k], ark = A[(size_t)r * p + k];
          A[(size_t)q * p + k] = c * aqk - s * ark;
          A[(size_t)r * p + k] = s * aqk + c * ark;
        }
      }
  }
  for (int32_t i = 0; i < p; ++i) evals[i] = A[(size_t)i * p + i];
  /* ascending insertion sort */
  for (int32_t i = 1; i < p; ++i) {
    double v = evals[i];
    int32_t j = i - 1;
    while (j >= 0 && evals[j] > v) { evals[j + 1] = evals[j]; --j; }
    evals[j + 1] = v;
  }
  free(A);
}

/* The d rule (R#5): d = min(Gershgorin, U_S), U_S = trace(A^(2^S))^(1/2^S).
 * For symmetric PSD A with eigenvalues l_1 >= ... >= l_p >= 0, trace(A^m) = sum_i l_i^m, so
 * l_1 <= trace(A^m)^(1/m) <= p^(1/m) l_1: U_S is an upper bound on l_1 for every A (whatever
 * its eigenvectors), and within a factor p^(1/2^S) of it. A^(2^S) is formed by S squarings of
 * the trace-normalised matrix (the power method applied to all p basis vectors at once):
 *   B_0 = A; s_t = trace(B_t); B_{t+1} = (B_t / s_t)^2;
 *   log U_S = log s_0 + sum_{t=1..S} 2^-t log s_t     (A^(2^t) = c_t B_t / s_t, c_t = c_{t-1}^2 s_t),
 * times the rounding allowance (1 + 2 S p u).
 * Naive triple-loop products (rows in parallel; each entry is one plain dot product). */
double orc_d_rule(const double* A, int32_t p, int32_t squarings, double* U_out, double* gersh_out) {
  size_t pp = (size_t)p * p;
  double gersh = 0.0;
  for (int32_t j = 0; j < p; ++j) {
    double s = 0.0;
    for (int32_t k = 0; k < p; ++k) s += fabs(A[(size_t)j * p + k]);
    if (s > gersh) gersh = s;
  }
  double* B = (double*)malloc(sizeof(double) * pp);
  double* C = (double*)malloc(sizeof(double) * pp);
  memcpy(B, A, sizeof(double) * pp);
  double s = 0.0;
  for (int32_t j = 0; j < p; ++j) s += B[(size_t)j * p + j];
  double logU = s > 0.0 ? log(s) : -INFINITY;
  for (int32_t t = 1; t <= squarings && s > 0.0; ++t) {
    /* B <- B / s, then C = B B. B stays exactly symmetric (C_jk and C_kj are the same products
     * summed in the same order), so B_mk is read as B_km: a row-by-row dot product. */
    for (size_t e = 0; e < pp; ++e) B[e] /= s;
#pragma omp parallel for schedule(static)
    for (int32_t j = 0; j < p; ++j)
      for (int32_t k = 0; k < p; ++k) {
        double acc = 0.0;
        for (int32_t m = 0; m < p; ++m) acc += B[(size_t)j * p + m] * B[(size_t)k * p + m];
        C[(size_t)j * p + k] = acc;
      }
    double* tmp = B; B = C; C = tmp;
    s = 0.0;
    for (int32_t j = 0; j < p; ++j) s += B[(size_t)j * p + j];
    logU += ldexp(log(s), -t);
  }
  free(B);
  free(C);
  /* rounding allowance: the S squarings perturb the top of the spectrum by about S p u
   * relative (u = 2^-53), so U is inflated by (1 + 2 S p u) to stay >= lambda_1 in fp64 */
  double U = exp(logU) * (1.0 + 2.0 * (double)squarings * (double)p * ldexp(1.0, -53));
  if (U_out) *U_out = U;
  if (gersh_out) *gersh_out = gersh;
  return gersh < U ? gersh : U;
}

/* ---------------- thresholding operators ---------------- */
static double sgn(double u) { return u > 0.0 ? 1.0 : (u < 0.0 ? -1.0 : 0.0); }
static double pos(double a) { return a > 0.0 ? a : 0.0; }

double orc_soft(double u, double lam, double d) { /* S(u, lam, d) = sign(u)((|u| - lam)/d)_+ */
  return sgn(u) * pos((fabs(u) - lam) / d);
}
double orc_enet(double u, double lam, double alpha, double d) { /* sign(u)((|u|-w a l)/(d + w(1-a) l))_+ */
  return sgn(u) * pos((fabs(u) - lam * alpha) / (d + lam * (1.0 - alpha)));
}
double orc_mcp(double u, double lam, double gamma, double d) {
  if (fabs(u) <= lam * gamma * d) return sgn(u) * gamma * pos(fabs(u) - lam) / (gamma * d - 1.0);
  return u / d;
}
double orc_scad(double u, double lam, double gamma, double d) {
  double a = fabs(u);
  if (a <= (d + 1.0) * lam) return sgn(u) * pos(a - lam) / d;
  if (a <= lam * gamma * d) return sgn(u) * ((gamma - 1.0) * a - lam * gamma) / ((gamma - 1.0) * d - 1.0);
  return u / d;
}
static double norm2(const double* u, int32_t m) {
  double s = 0.0;
  for (int32_t i = 0; i < m; ++i) s += u[i] * u[i];
  return sqrt(s);
}
void orc_grp_lasso(const double* u, int32_t m, double lam, double d, double* out) {
  double nu = norm2(u, m);
  double f = nu > 0.0 ? pos(1.0 - lam / nu) : 0.0; /* 0/0 -> beta_g = 0 (R#10) */
  for (int32_t i = 0; i < m; ++i) out[i] = u[i] / d * f;
}
void orc_grp_mcp(const double* u, int32_t m, double lam, double gamma, double d, double* out) {
  double nu = norm2(u, m);
  double s = nu > 0.0 ? orc_mcp(nu, lam, gamma, d) / nu : 0.0;
  for (int32_t i = 0; i < m; ++i) out[i] = s * u[i];
}
void orc_grp_scad(const double* u, int32_t m, double lam, double gamma, double d, double* out) {
  double nu = norm2(u, m);
  double s = nu > 0.0 ? orc_scad(nu, lam, gamma, d) / nu : 0.0;
  for (int32_t i = 0; i < m; ++i) out[i] = s * u[i];
}

/* Sparse group lasso (P:L291-297 eq sglasso). The printed G(v, c lam (1 - tau), 1) is the
   proximal map only at d = 1; the M-step minimises (d/2)||b||^2 - u^T b + lam tau sum w|b| +
   lam (1 - tau) c ||b||, whose minimiser is the soft threshold followed by the group shrink of
   v = S(u, w lam tau, d) at level c lam (1 - tau) / d (R#11). */
void orc_sgl(const double* u, const double* w, int32_t m, double lam, double tau, double c, double d, double* out) {
  for (int32_t i = 0; i < m; ++i) out[i] = orc_soft(u[i], (w ? w[i] : 1.0) * lam * tau, d);
  double nv = norm2(out, m);
  double f = nv > 0.0 ? pos(1.0 - c * lam * (1.0 - tau) / (d * nv)) : 0.0;
  for (int32_t i = 0; i < m; ++i) out[i] *= f;
}

/* ---------------- lambda grid ---------------- */
static int is_group(int family) { return family >= ORC_GRP_LASSO; }

/* sparse group lasso: the smallest lambda at which beta_g = 0 is a fixed point from beta = 0 is
   the root of ||S(c_g, lam tau w_g, 1)|| = lam (1 - tau) c_g (decreasing in lam), by bisection
   (R#36) */
static double sgl_group_lmax(const double* cg_vec, const double* wg, int32_t m, double cg, double tau) {
  double hi = 0.0;
  for (int32_t i = 0; i < m; ++i) {
    double wi = wg ? wg[i] : 1.0;
    if (tau > 0.0 && wi > 0.0) hi = fmax(hi, fabs(cg_vec[i]) / (tau * wi));
  }
  if (tau < 1.0 && cg > 0.0) hi = fmax(hi, norm2(cg_vec, m) / ((1.0 - tau) * cg));
  double lo = 0.0;
  for (int it = 0; it < 200 && hi > lo; ++it) {
    double mid = 0.5 * (lo + hi);
    if (mid <= lo || mid >= hi) break;
    double s = 0.0;
    for (int32_t i = 0; i < m; ++i) {
      double t = pos(fabs(cg_vec[i]) - mid * tau * (wg ? wg[i] : 1.0));
      s += t * t;
    }
    if (sqrt(s) > mid * (1.0 - tau) * cg) lo = mid; else hi = mid;
  }
  return hi * (1.0 + 1e-12);  /* R#36: clear of the rounding at the root, so the operator is exactly 0 there */
}

static double group_weight(const int32_t* group, int32_t p, int32_t g, const double* grp_w) {
  if (grp_w) return grp_w[g];
  int32_t m = 0;
  for (int32_t j = 0; j < p; ++j) m += group[j] == g;
  return sqrt((double)m);
}

double orc_lambda_max(int family, double alpha, const double* c, int32_t p, const double* w,
                      const int32_t* group, int32_t ngroups, const double* grp_w) {
  double lmax = 0.0;
  if (family == ORC_SGL) {
    double* cgv = (double*)malloc(sizeof(double) * (size_t)p);
    double* wgv = (double*)malloc(sizeof(double) * (size_t)p);
    for (int32_t g = 0; g < ngroups; ++g) {
      double cg = group_weight(group, p, g, grp_w);
      int32_t m = 0;
      for (int32_t j = 0; j < p; ++j)
        if (group[j] == g) { cgv[m] = c[j]; wgv[m] = w ? w[j] : 1.0; ++m; }
      double v = sgl_group_lmax(cgv, wgv, m, cg, alpha);
      if (v > lmax) lmax = v;
    }
    free(cgv);
    free(wgv);
    return lmax;
  }
  if (is_group(family)) {
    for (int32_t g = 0; g < ngroups; ++g) {
      double cg = group_weight(group, p, g, grp_w);
      if (!(cg > 0.0)) continue;
      double s = 0.0;
      for (int32_t j = 0; j < p; ++j)
        if (group[j] == g) s += c[j] * c[j];
      double v = sqrt(s) / cg;
      if (v > lmax) lmax = v;
    }
    return lmax;
  }
  double scale = (family == ORC_ENET) ? alpha : 1.0;
  for (int32_t j = 0; j < p; ++j) {
    double wj = w ? w[j] : 1.0;
    if (!(wj > 0.0)) continue;
    double v = fabs(c[j]) / (scale * wj);
    if (v > lmax) lmax = v;
  }
  return lmax;
}

void orc_lambda_grid(double lmax, int32_t L, double ratio, double* lambdas) {
  if (L == 1) { lambdas[0] = lmax; return; }
  for (int32_t i = 0; i < L; ++i) lambdas[i] = lmax * exp(((double)i / (double)(L - 1)) * log(ratio));
}

/* ---------------- O6 OEM path ---------------- */
static void threshold_all(int family, const double* u, int32_t p, double d, double lambda, double gamma,
                          double alpha, const double* w, const int32_t* group, int32_t ngroups,
                          const double* grp_w, double* out) {
  if (!is_group(family)) {
    for (int32_t j = 0; j < p; ++j) {
      double lam = (w ? w[j] : 1.0) * lambda;
      switch (family) {
        case ORC_LASSO: out[j] = orc_soft(u[j], lam, d); break;
        case ORC_ENET: out[j] = orc_enet(u[j], lam, alpha, d); break;
        case ORC_MCP: out[j] = orc_mcp(u[j], lam, gamma, d); break;
        default: out[j] = orc_scad(u[j], lam, gamma, d); break;
      }
    }
    return;
  }
  double* ug = (double*)malloc(sizeof(double) * (size_t)p);
  double* og = (double*)malloc(sizeof(double) * (size_t)p);
  double* wg = (double*)malloc(sizeof(double) * (size_t)p);
  for (int32_t g = 0; g < ngroups; ++g) {
    int32_t m = 0;
    for (int32_t j = 0; j < p; ++j)
      if (group[j] == g) { wg[m] = w ? w[j] : 1.0; ug[m++] = u[j]; }
    double lam = group_weight(group, p, g, grp_w) * lambda;
    if (family == ORC_SGL) orc_sgl(ug, wg, m, lambda, alpha, group_weight(group, p, g, grp_w), d, og);
    else if (family == ORC_GRP_LASSO) orc_grp_lasso(ug, m, lam, d, og);
    else if (family == ORC_GRP_MCP) orc_grp_mcp(ug, m, lam, gamma, d, og);
    else orc_grp_scad(ug, m, lam, gamma, d, og);
    m = 0;
    for (int32_t j = 0; j < p; ++j)
      if (group[j] == g) out[j] = og[m++];
  }
  free(ug);
  free(og);
  free(wg);
}

int orc_oem_path(const double* G, const double* c, int32_t p, double d, int family, double gamma,
                 double alpha, const double* w, const int32_t* group, int32_t ngroups,
                 const double* grp_w, const double* lambdas, int32_t L, double tol, int64_t maxit,
                 const double* beta_init, double* beta_out, int64_t* iters, uint8_t* conv) {
  if (!(d > 0.0)) return -1;
  if (family == ORC_MCP || family == ORC_GRP_MCP) { if (!(gamma > 1.0) || !(gamma * d > 1.0)) return -1; }
  if (family == ORC_SCAD || family == ORC_GRP_SCAD) { if (!(gamma > 2.0) || !((gamma - 1.0) * d > 1.0)) return -1; }
  if (family == ORC_ENET && !(alpha >= 0.0 && alpha <= 1.0)) return -1;
  if (is_group(family) && (!group || ngroups < 1)) return -1;
  if (family == ORC_SGL && !(alpha >= 0.0 && alpha <= 1.0)) return -1;
  double* beta = (double*)malloc(sizeof(double) * (size_t)p);
  double* u = (double*)malloc(sizeof(double) * (size_t)p);
  double* nb = (double*)malloc(sizeof(double) * (size_t)p);
  for (int32_t j = 0; j < p; ++j) beta[j] = beta_init ? beta_init[j] : 0.0;
  for (int32_t l = 0; l < L; ++l) {
    int64_t t = 0;
    uint8_t ok = 0;
    while (t < maxit) {
      /* E-step + M-step in closed form: u = X^T y + (dI - X^T X) beta */
      for (int32_t j = 0; j < p; ++j) {
        double gb = 0.0;
        for (int32_t k = 0; k < p; ++k) gb += G[(size_t)j * p + k] * beta[k];
        u[j] = c[j] + d * beta[j] - gb;
      }
      threshold_all(family, u, p, d, lambdas[l], gamma, alpha, w, group, ngroups, grp_w, nb);
      double delta = 0.0;
      for (int32_t j = 0; j < p; ++j) {
        double a = fabs(nb[j] - beta[j]);
        if (a > delta) delta = a;
        beta[j] = nb[j];
      }
      ++t;
      if (delta <= tol) { ok = 1; break; }
    }
    memcpy(beta_out + (size_t)l * p, beta, sizeof(double) * (size_t)p);
    iters[l] = t;
    conv[l] = ok;
  }
  free(beta);
  free(u);
  free(nb);
  return 0;
}

/* ---------------- objective (Table 1 penalty forms) ---------------- */
static double p_mcp(double b, double lam, double gamma) {
  double a = fabs(b);
  return a <= gamma * lam ? lam * a - a * a / (2.0 * gamma) : gamma * lam * lam / 2.0;
}
static double p_scad(double b, double lam, double gamma) {
  double a = fabs(b);
  if (a <= lam) return lam * a;
  if (a <= gamma * lam) return -(a * a - 2.0 * gamma * lam * a + lam * lam) / (2.0 * (gamma - 1.0));
  return (gamma + 1.0) * lam * lam / 2.0;
}

double orc_objective(const double* G, const double* c, int32_t p, const double* beta, int family,
                     double lambda, double gamma, double alpha, const double* w,
                     const int32_t* group, int32_t ngroups, const double* grp_w) {
  double q = 0.0;
  for (int32_t j = 0; j < p; ++j) {
    double gb = 0.0;
    for (int32_t k = 0; k < p; ++k) gb += G[(size_t)j * p + k] * beta[k];
    q += 0.5 * beta[j] * gb - c[j] * beta[j];
  }
  double pen = 0.0;
  if (!is_group(family)) {
    for (int32_t j = 0; j < p; ++j) {
      double wj = w ? w[j] : 1.0;
      switch (family) {
        case ORC_LASSO: pen += lambda * wj * fabs(beta[j]); break;
        case ORC_ENET: pen += alpha * lambda * wj * fabs(beta[j]) + 0.5 * (1.0 - alpha) * lambda * wj * beta[j] * beta[j]; break;
        case ORC_MCP: pen += p_mcp(beta[j], lambda * wj, gamma); break;
        default: pen += p_scad(beta[j], lambda * wj, gamma); break;
      }
    }
  } else {
    for (int32_t g = 0; g < ngroups; ++g) {
      double s = 0.0;
      for (int32_t j = 0; j < p; ++j)
        if (group[j] == g) s += beta[j] * beta[j];
      double nb = sqrt(s), cg = group_weight(group, p, g, grp_w);
      if (family == ORC_SGL) {  /* Table 1: lam (1 - tau) sum c_k ||b_g|| + lam tau sum w_j |b_j| */
        pen += lambda * (1.0 - alpha) * cg * nb;
        for (int32_t j = 0; j < p; ++j)
          if (group[j] == g) pen += lambda * alpha * (w ? w[j] : 1.0) * fabs(beta[j]);
      } else if (family == ORC_GRP_LASSO) pen += lambda * cg * nb;
      else if (family == ORC_GRP_MCP) pen += p_mcp(nb, lambda * cg, gamma); /* R#9: no extra leading lambda */
      else pen += p_scad(nb, lambda * cg, gamma);
    }
  }
  return q + pen;
}

/* ---------------- O7 logistic ---------------- */
int orc_logistic_path(const double* X, const double* y01, int64_t n, int32_t p, int64_t ldx, int family,
                      double gamma, double alpha, const double* w, const int32_t* group, int32_t ngroups,
                      const double* grp_w, const double* lambdas, int32_t L, double eps, double tol_in,
                      int64_t maxit_in, double tol_out, int32_t outer_maxit, int32_t squarings,
                      double* beta_out, int32_t* outer_iters, int64_t* inner_iters, uint8_t* conv,
                      double* d_out, int nthreads) {
  for (int64_t i = 0; i < n; ++i)
    if (!(y01[i] == 0.0 || y01[i] == 1.0)) return -1;
  size_t pp = (size_t)p * p;
  double* Gw = (double*)malloc(sizeof(double) * pp);
  double* cw = (double*)malloc(sizeof(double) * (size_t)p);
  double* beta = (double*)calloc((size_t)p, sizeof(double));
  double* nb = (double*)malloc(sizeof(double) * (size_t)p);
  double sc[2];
  int64_t it1;
  uint8_t cv1;
  int rc = 0;
  for (int32_t l = 0; l < L && rc == 0; ++l) {
    int32_t o = 0;
    int64_t inner = 0;
    uint8_t ok = 0;
    while (o < outer_maxit) {
      orc_gram_weighted(X, y01, beta, n, p, ldx, eps, Gw, cw, sc, nthreads);
      for (size_t q = 0; q < pp; ++q) Gw[q] /= (double)n;
      for (int32_t j = 0; j < p; ++j) cw[j] /= (double)n;
      double dw = orc_d_rule(Gw, p, squarings, NULL, NULL);
      if (d_out && l == 0 && o == 0) *d_out = dw;
      rc = orc_oem_path(Gw, cw, p, dw, family, gamma, alpha, w, group, ngroups, grp_w, &lambdas[l], 1,
                        tol_in, maxit_in, beta, nb, &it1, &cv1);
      if (rc != 0) break;
      inner += it1;
      ++o;
      double delta = 0.0;
      for (int32_t j = 0; j < p; ++j) {
        double a = fabs(nb[j] - beta[j]);
        if (a > delta) delta = a;
        beta[j] = nb[j];
      }
      if (delta <= tol_out) { ok = 1; break; }
    }
    memcpy(beta_out + (size_t)l * p, beta, sizeof(double) * (size_t)p);
    outer_iters[l] = o;
    inner_iters[l] = inner;
    conv[l] = ok;
  }
  free(Gw);
  free(cw);
  free(beta);
  free(nb);
  return rc;
}
