/* oem_datagen.h — seeded synthetic-input generator shared by the oracle tests and the CUDA path.
 *
 * This module holds NONE of the method's arithmetic (no Gram, no threshold, no path): it only
 * draws the design X, the true coefficient vector beta and the response y of the paper's
 * simulation designs (§6.1 "we generate the design matrix from a
 * multivariate normal distribution with covariance matrix 0.5^|i-j|"; L1137-1149, §6.3 logistic
 * timings; BASELINE.json configs 1-5; SURVEY.md §8(d).2 generator specification).
 *
 * Two independent implementations exist, written separately from the same specification below:
 *   host   : datagen/datagen_host.c   -> datagen/libdatagen_host.so  (gcc, -ffp-contract=off)
 *   device : datagen/datagen_cuda.cu  -> datagen/libdatagen_cuda.so  (nvcc, explicit _rn intrinsics)
 * Both produce bit-identical X and y for the same spec (checked by row hashes in tests).
 *
 * SPECIFICATION (the contract both sides implement):
 *  - Philox4x32-10 (Salmon et al. 2011): multipliers M0=0xD2511F53, M1=0xCD9E8D57, key bumps
 *    W0=0x9E3779B9, W1=0xBB67AE85; 10 rounds; key = (seed & 0xffffffff, seed >> 32).
 *    Counters (c0,c1,c2,c3) per stream:
 *      stream 0  base normals z_ij   : (i_lo, i_hi, j>>1, 0)   columns 2m, 2m+1 share one call
 *      stream 1  group factors g_ik  : (i_lo, i_hi, k>>1, 1)
 *      stream 2  noise eps_i         : (i_lo, i_hi, 0, 2)
 *      stream 3  beta draws          : (t, s, 0, 3)            t = draw index, s = 0 index / 1 value
 *      stream 4  Bernoulli u_i       : (i_lo, i_hi, 0, 4)
 *      stream 5  sparsity pattern    : (i_lo, i_hi, j>>1, 5)   columns 2m, 2m+1 share one call
 *  - uniform(w_a, w_b): k = ((w_a << 32) | w_b) >> 12 (52 bits); u = (2k + 1) * 2^-53, exact, in (0,1).
 *  - normal pair from one call (w0..w3): u1 = uniform(w0,w1), u2 = uniform(w2,w3);
 *      r = sqrt(-2 * LN(u1)); (z_even, z_odd) = (r * COS2PI(u2), r * SIN2PI(u2)).
 *    LN, COS2PI, SIN2PI, EXP are the software routines defined in datagen_host.c / _cuda.cu
 *    using only IEEE +,-,*,/,sqrt (correctly rounded, no FMA contraction), so both sides agree
 *    bit for bit.
 *  - designs: IID x_ij = z_ij;  AR1 x_i0 = z_i0, x_ij = rho*x_i,j-1 + sqrt(1-rho^2)*z_ij;
 *    BLOCK x_ij = sqrt(r)*g_i,k(j) + sqrt(1-r)*z_ij with k(j) = j / group_size (group factors
 *    are the stream-1 normals).  SPARSE (the paper's rsparsematrix example):
 *    x_ij = z_ij if u_ij < d else 0, with d = rho (the density) and u_ij = uniform(w0,w1) (even j)
 *    or uniform(w2,w3) (odd j) of the stream-5 call of the pair; every cell independently (the
 *    expected density is d).  All products/sums evaluated left to right as written.
 *  - beta: partial Fisher-Yates over [0,m) (m = p, or the number of groups for ACTIVE_GROUPS):
 *    for t < nnz: w0 of counter (t,0,0,3); j = t + ((w0 * (m - t)) >> 32); swap(perm[t], perm[j]).
 *    values: counter (t,1,0,3), uniform(w0,w1) -> lo + (hi-lo)*u (UNIFORM) or the even normal
 *    of the pair (NORMAL). ACTIVE_GROUPS draws one value per column of each chosen group, the
 *    value draw index t running over chosen columns in ascending column order.
 *  - response: eta_i = sum over j ascending with beta_j != 0 of x_ij*beta_j (acc = acc + x*b,
 *    acc starts at +0.0); LINEAR y_i = eta_i + sigma*eps_i (eps_i = even normal of stream 2);
 *    LOGISTIC y_i = 1.0 if uniform(w0,w1) of stream 4 < 1/(1+EXP(-eta_i)) else 0.0.
 */
#ifndef OEM_DATAGEN_H
#define OEM_DATAGEN_H
#include <stdint.h>
#ifdef __cplusplus
extern "C" {
#endif

typedef enum { DG_IID = 0, DG_AR1 = 1, DG_BLOCK = 2, DG_SPARSE = 3 } dg_design;
typedef enum { DG_LINEAR = 0, DG_LOGISTIC = 1 } dg_response;
typedef enum { DG_BETA_EXPLICIT = 0, DG_BETA_UNIFORM = 1, DG_BETA_NORMAL = 2, DG_BETA_ACTIVE_GROUPS = 3 } dg_beta_kind;

typedef struct {
  uint64_t seed;
  int64_t n;          /* global number of rows */
  int32_t p;          /* number of columns */
  int32_t design;     /* dg_design */
  double rho;         /* AR(1) rho, within-group correlation r for DG_BLOCK, density d for DG_SPARSE */
  int32_t group_size; /* DG_BLOCK and DG_BETA_ACTIVE_GROUPS: contiguous groups of this size */
  int32_t response;   /* dg_response */
  double sigma;       /* noise sd (linear) */
  int32_t beta_kind;  /* dg_beta_kind */
  int32_t nnz;        /* nonzeros (UNIFORM/NORMAL) or number of active groups (ACTIVE_GROUPS) */
  double beta_lo, beta_hi; /* UNIFORM range */
} dg_spec;

/* Philox4x32-10 of one counter/key (exposed for known-answer tests). out: 4 words (host). */
void dg_philox4x32_10(const uint32_t ctr[4], const uint32_t key[2], uint32_t out[4]);

/* Host software math used by the generator (exposed for tests of the routines themselves). */
double dg_ln(double x);
double dg_exp(double x);
void dg_sincos2pi(double u, double* s, double* c);

/* beta_true (host, p doubles). Returns 0, or -1 on an invalid spec. For DG_BETA_EXPLICIT the
 * caller fills beta itself and this call only validates the spec. */
int dg_beta(const dg_spec* spec, double* beta);

/* Host rows [row0, row0+nrows) x columns [col0, col0+ncols) into X (row-major, leading
 * dimension ldx >= ncols; element (i, j) at X[i*ldx + (j-col0)]). y (nrows) if non-NULL.
 * beta: host p doubles (needed for y). Returns 0 or -1 on invalid arguments. */
int dg_rows_host(const dg_spec* spec, const double* beta, int64_t row0, int64_t nrows,
                 int32_t col0, int32_t ncols, double* X, int64_t ldx, double* y);

/* Device (libdatagen_cuda.so): full rows [row0,row0+nrows), all p columns, into device X
 * (row-major [nrows][ldx]) and device y (nrows). beta: DEVICE p doubles. Asynchronous on
 * `stream` (a cudaStream_t passed as void*). Returns 0, -1 invalid args, -2 CUDA launch error. */
int dg_rows_cuda(const dg_spec* spec, const double* beta, int64_t row0, int64_t nrows,
                 double* X, int64_t ldx, double* y, void* stream);

/* Device compressed-sparse-row form of the SPARSE design (rows [row0, row0+nrows), libdatagen_cuda.so):
 * dg_csr_count_cuda writes the nonzero count of every row (int64, nrows); after the caller's
 * exclusive prefix sum into row_ptr (nrows+1, row_ptr[0] = 0), dg_csr_fill_cuda writes the column
 * indices (int32, ascending within each row) and values of every nonzero, and y (nrows) if
 * non-NULL (eta over the nonzero support columns in ascending j, as above). Values equal the
 * dense generator's bit for bit. Asynchronous on `stream`. Returns 0, -1 (invalid), -2 (CUDA). */
int dg_csr_count_cuda(const dg_spec* spec, int64_t row0, int64_t nrows, int64_t* counts, void* stream);
int dg_csr_fill_cuda(const dg_spec* spec, const double* beta, int64_t row0, int64_t nrows,
                     const int64_t* row_ptr, int32_t* col, double* val, double* y, void* stream);

#ifdef __cplusplus
}
#endif
#endif
