/* oem.h — C ABI of liboem.so: the data-parallel hot path of the orthogonalizing EM (OEM)
 * algorithm for penalized least squares on tall data (Huling & Chien, arXiv 1801.09661),
 * B200-native (sm_100a).
 *
 * Citations: "P:Lnnn" = PAPER.md line nnn; "R#k" = reading k in DESIGN.md §3 (the paper's
 * silent/garbled points and the reading taken).
 *
 * Conventions (all entry points)
 *  - Pointers are DEVICE pointers unless marked (host). The caller owns every buffer it passes;
 *    the library never frees them. The oem_ctx owns its workspace (split-n partials, packed
 *    reduction buffers, the NCCL communicator) and releases it in oem_ctx_destroy.
 *  - Every call is enqueued on `stream` (a cudaStream_t passed as void*; NULL = legacy default
 *    stream). Calls that must read device results on the host (counts, maxit flags) synchronise
 *    that stream before returning, and say so.
 *  - X is row-major: element (i, j) at X[i*ldx + j], 0 <= i < n_local, 0 <= j < p, ldx >= p.
 *    TMA needs X and y 16-byte aligned and ldx even (row pitch a multiple of 16 B); otherwise
 *    OEM_ERR_ALIGN.
 *  - All arithmetic is IEEE fp64. Reductions use no atomics and a fixed order: for a fixed
 *    world size and inputs, outputs are bitwise reproducible.
 *  - Errors: the boundary never throws or aborts. Each call returns an oem_status;
 *    oem_last_error() returns a thread-local detail string for the last failing call.
 *  - Multi-GPU: one process per GPU. X is row-sharded; each rank passes its own rows. When the
 *    context holds a communicator (nranks > 1, or a uid given), the Gram entry points sum their raw outputs over all
 *    ranks with one ncclAllReduce (sum, fp64) on `stream` before returning, so every rank holds
 *    identical reduced statistics ("computed independently ... in parallel";
 *    P:L72-76 Gram quantities computed on a cluster).
 */
#ifndef OEM_H
#define OEM_H
#include <stdint.h>
#ifdef __cplusplus
extern "C" {
#endif

typedef struct oem_ctx oem_ctx;

typedef enum {
  OEM_OK = 0,
  OEM_ERR_INVALID_ARG = 1,  /* bad gamma/alpha/weights/groups/sizes, y not in {0,1} for logistic */
  OEM_ERR_DIM = 2,          /* dimension mismatch (SPEC DimensionMismatch) */
  OEM_ERR_ALIGN = 3,        /* X / y not 16-byte aligned or ldx odd (TMA constraints) */
  OEM_ERR_EMPTY_FOLD = 4,   /* a fold has no rows (SPEC EmptyFold) */
  OEM_ERR_NONFINITE = 5,    /* NaN/Inf in a Gram or in the path iterates (SPEC NonFinite) */
  OEM_ERR_CUDA = 6,
  OEM_ERR_NCCL = 7,
  OEM_ERR_NOMEM = 8,
  OEM_ERR_UNSUPPORTED = 9   /* a size this build does not handle (stated in the detail text) */
} oem_status;

const char* oem_status_string(oem_status s);
const char* oem_last_error(void);
const char* oem_version(void);

/* NCCL bootstrap: rank 0 calls oem_nccl_unique_id and broadcasts the 128 bytes to the other
 * ranks (e.g. through torch.distributed); every rank then calls oem_ctx_create with it. */
oem_status oem_nccl_unique_id(void* uid128 /*host, 128 bytes*/);
/* One context per (process, device). nranks == 1: uid may be NULL and no NCCL is used; with a uid
 * (from oem_nccl_unique_id in the same process) a one-rank communicator is created and every
 * entry point takes its multi-rank path (the allreduces run, as identities) on one GPU. */
oem_status oem_ctx_create(int device, int nranks, int rank, const void* uid128 /*host*/, oem_ctx** out);
oem_status oem_ctx_destroy(oem_ctx* ctx);

/* ---- a2 Gram pass (P:L171-172 A = dI - X^T X, u = X^T y + A beta; "the key
 * computational step in OEM is in forming the matrix A"; P:L328-333 O(np^2 + np)).
 * One pass over [X | y]: G = X^T X (full symmetric p*p written, row-major), xty = X^T y (p),
 * yty = y^T y (1). Raw sums over this rank's rows, allreduced when the context has a communicator; normalisation
 * (/n, R#1) happens in oem_fit_path. n_total (host, may be NULL) receives the global row count
 * (with a communicator a small NCCL allreduce on `stream`, after which the call synchronises it).
 * n_local = 0 is allowed (zero outputs). Errors: OEM_ERR_DIM (p < 1, ldx < p, n_local < 0),
 * OEM_ERR_ALIGN, OEM_ERR_UNSUPPORTED (p > 16383), OEM_ERR_CUDA, OEM_ERR_NCCL. */
oem_status oem_gram(oem_ctx* ctx, const double* X, const double* y, int64_t n_local, int32_t p,
                    int64_t ldx, double* G, double* xty, double* yty, int64_t* n_total, void* stream);

/* ---- a3 fold-segmented Gram (§3: A_(k) = d_(k) I - sum_{c != k} X_c^T X_c and
 * X_{-k}^T y_{-k} = sum_{c != k} X_c^T y_c; P:L336-339 folds computed independently).
 * One pass over X producing K raw per-fold sums: G_folds[k*p*p + j*p + l] (full symmetric),
 * xty_folds[k*p + j], yty_folds[k]; counts[k] (host) = global rows in fold k.
 * fold(i) = (row_offset + i) mod K for local row i (R#19); row_offset = this rank's first
 * global row. Errors: as oem_gram, plus OEM_ERR_INVALID_ARG (K < 1),
 * OEM_ERR_EMPTY_FOLD (a fold with no rows globally). Synchronises `stream` only with a communicator
 * (the per-rank counts are host arithmetic; their sum over ranks is one small NCCL allreduce on
 * `stream`, read back before the pass). */
oem_status oem_gram_folds(oem_ctx* ctx, const double* X, const double* y, int64_t n_local, int32_t p,
                          int64_t ldx, int64_t row_offset, int32_t K, double* G_folds,
                          double* xty_folds, double* yty_folds, int64_t* counts /*host K*/, void* stream);

/* ---- a2/a3 with a ones column (f3 intercept / standardization, R#2-3): the
 * same single pass over Z = [X | y | 1] (the ones column is formed in shared memory, no extra
 * HBM bytes), which also yields the column sums the intercept needs: xsum[j] = sum_i x_ij (p),
 * ysum = sum_i y_i (1), raw over this rank's rows and allreduced with G (one allreduce).
 * G, xty, yty, n_total exactly as oem_gram (the sums of the shared entries may differ from
 * oem_gram's in the last bits when the extra column changes the tiling). Replaces the second,
 * HBM-bound pass of oem_gram_moments for in-core data. Errors: as oem_gram. */
oem_status oem_gram_sums(oem_ctx* ctx, const double* X, const double* y, int64_t n_local, int32_t p,
                         int64_t ldx, double* G, double* xty, double* yty, double* xsum /*p*/,
                         double* ysum /*1*/, int64_t* n_total /*host, may be NULL*/, void* stream);
/* The fold-segmented form (a3 + f3): oem_gram_folds plus, per fold k, xsum_folds[k*p + j] and
 * ysum_folds[k] (the fold column sums oem_cv_error and an intercept fit take), one pass.
 * Errors: as oem_gram_folds. */
oem_status oem_gram_folds_sums(oem_ctx* ctx, const double* X, const double* y, int64_t n_local, int32_t p,
                               int64_t ldx, int64_t row_offset, int32_t K, double* G_folds,
                               double* xty_folds, double* yty_folds, double* xsum_folds /*K*p*/,
                               double* ysum_folds /*K*/, int64_t* counts /*host K*/, void* stream);

/* ---- a4 weighted Gram for the proximal-Newton logistic step (§4; working
 * responses z_i and weights w_i at P:L376-380; R#23-25). Per row: eta = x_i^T beta,
 * mu = 1/(1+exp(-eta)) clamped to [eps, 1-eps], w = mu(1-mu), z = eta + (y - mu)/w.
 * Outputs raw sums: Gw = sum w x x^T (full symmetric p*p), xtwz = sum w z x (p),
 * scalars (device, 2, or NULL) = {sum w, sum [y eta - log(1 + e^eta)] (log-likelihood)};
 * with scalars = NULL neither is formed (the row work is then ~5% cheaper; the logistic fit,
 * whose stopping rule is the change in beta, passes NULL).
 * beta (p, device) must be identical on every rank. y01 must hold 0.0/1.0 (not checked on the
 * device; the binding checks once per fit). p <= 247: eta, w, z are formed inside the Gram kernel
 * from the staged rows (one pass); larger p (two-panel plans, whose CTAs never hold a whole row):
 * one HBM-bound pass forms (w_i, z_i) per row, then the contraction reads them with the rows.
 * Errors: as oem_gram. */
oem_status oem_gram_weighted(oem_ctx* ctx, const double* X, const double* y01, const double* beta,
                             int64_t n_local, int32_t p, int64_t ldx, double eps, double* Gw,
                             double* xtwz, double* scalars, void* stream);

/* ---- a6-a10 normalise, d, lambda grid, OEM path (P:L147-158 Steps 1-2; P:L171-195;
 * P:L239-289 thresholding M-steps; §5.2 several penalties share A and X^T y).
 * Penalty families of Table 1, update equations at P:L243-289. */
typedef enum { OEM_LASSO = 0, OEM_ENET = 1, OEM_MCP = 2, OEM_SCAD = 3,
               OEM_GRP_LASSO = 4, OEM_GRP_MCP = 5, OEM_GRP_SCAD = 6,
               OEM_SGL = 7 /* sparse group lasso (Table 1), tau in the alpha field;
                              exact d-scaled composition of the two proximal maps (R#11) */ } oem_family;
typedef struct { int32_t family; double gamma; double alpha; } oem_penalty;
typedef struct {
  int32_t nlambda;          /* L >= 1 */
  double lambda_min_ratio;  /* 0 < r < 1 (R#15); default 1e-3 */
  const double* lambda;     /* host, optional explicit grid of L values shared by all units */
  double tol;               /* stop when max_j |beta'_j - beta_j| <= tol (R#17); default 1e-11 */
  int64_t maxit;            /* per-lambda update cap (not an error, R#17); default 1e5 */
  const double* var_w;      /* device, p or NULL (= 1, R#13) */
  const int32_t* group;     /* host, p group ids in [0, ngroups), or NULL */
  int32_t ngroups;
  const double* grp_w;      /* host, ngroups or NULL (= sqrt(group size), R#12) */
  int32_t d_squarings;      /* d rule (R#5): S in d = min(Gershgorin, trace(G^(2^S))^(1/2^S)); default 12 */
  int32_t fold_mode;        /* 1: inputs are K fold sums -> fit full data + K complements (R#20-22) */
  const double* lambda_max_override; /* host, optional: use this lambda_max for every unit */
  /* f3 (R#2-3): with xsum/ysum (device: nG*p raw column sums X^T 1 and nG raw 1^T y, in the
   * same layout as G/xty, e.g. from oem_gram_moments) the fit has an intercept: each unit's
   * statistics are centred, G - n xbar xbar^T and c - n xbar ybar, and intercept_out (device,
   * nG'*nP*L, may be NULL) receives b0 = ybar - xbar^T beta. standardize = 1 scales the
   * (centred) columns to unit variance before the fit and returns beta on the
   * original scale; columns of zero variance get beta = 0. */
  int32_t standardize;
  const double* xsum;
  const double* ysum;
  double* intercept_out;
} oem_path_cfg;

/* Fit paths from raw sufficient statistics. Inputs G (nG*p*p, full symmetric), xty (nG*p),
 * counts (host, nG): raw sums and their row counts. Gram g is normalised by counts[g] (R#1).
 * fold_mode = 0: nG' = nG units of Gram; fold_mode = 1: the nG = K inputs are fold sums; unit 0
 * is the full data (sum over folds, normalised by sum counts) and unit k (1..K) the complement
 * of fold k-1 (total minus fold, normalised by n - n_k, R#20), nG' = K + 1. d per unit by the
 * power rule (R#5, R#21) unless d_in (host, nG') is given. lambda grid per (unit, penalty) from
 * that unit's lambda_max (R#14, R#16) — in fold mode every unit shares unit 0's grid (R#22).
 * beta_init (device, nG'*nP*p) or NULL (= 0). Outputs (device): beta_out[nG'][nP][L][p],
 * lambda_out[nG'][nP][L], iters_out[nG'][nP][L] (int64), converged_out[nG'][nP][L] (uint8),
 * d_out[nG'] (double). Units run independently; a unit's lambda advances only when that unit
 * converges or hits maxit. Synchronises `stream` (reads the non-finite flag).
 * The iterates are the paper's; for p > 256 and p <= 128 the solver
 * iterates only the active block while a certificate proves every other coordinate's threshold
 * returns zero (developer overrides, read per call: OEM_SCREEN=0 turns that off,
 * OEM_PATH_SOLVER=active|lean|global|cluster|batched forces a solver layout).
 * Errors: OEM_ERR_INVALID_ARG (MCP gamma*d <= 1, SCAD (gamma-1)*d <= 1, alpha outside [0,1],
 * groups missing for group families, L < 1, bad ratio), OEM_ERR_EMPTY_FOLD (count 0),
 * OEM_ERR_NONFINITE, OEM_ERR_UNSUPPORTED (p > 16383), OEM_ERR_CUDA. */
oem_status oem_fit_path(oem_ctx* ctx, const double* G, const double* xty, const int64_t* counts /*host*/,
                        int32_t nG, int32_t p, const oem_penalty* pens /*host nP*/, int32_t nP,
                        const oem_path_cfg* cfg /*host*/, const double* d_in /*host or NULL*/,
                        const double* beta_init, double* beta_out, double* lambda_out,
                        int64_t* iters_out, uint8_t* converged_out, double* d_out, void* stream);

/* Default-initialise a path config (values listed above). */
void oem_path_cfg_default(oem_path_cfg* cfg);

/* ---- a4 + a6-a9 driven to convergence: the proximal-Newton logistic path (§4,
 * glmnet-style outer loop with OEM as the inner solver; R#23-27). For each lambda (warm start
 * from the previous solution): repeat { oem_gram_weighted at beta (allreduced over ranks);
 * normalise by n; d_w by the d rule (R#5); single-lambda OEM solve from beta } until
 * max_j |beta_new - beta| <= tol_out or outer_maxit. The lambda grid runs from lambda_max
 * (R#14, no intercept; c = (1/n) sum_i x_i (y_i - 1/2), the working statistic at beta = 0):
 * max_j |c_j| / (w_j [alpha for EN]) for the coordinate families, max_k ||c_{g_k}|| / c_k for
 * group lasso / MCP / SCAD (§6.3 fits group penalties to logistic models), down to
 * ratio * lambda_max (R#15), unless an explicit grid is given. The sparse group lasso is not
 * offered here (OEM_ERR_INVALID_ARG). Host loop: one scalar device->host read per outer step.
 * Outputs: beta_out (device, L*p), lambda_out (device, L), outer_iters / inner_iters /
 * converged (host, L). Errors: as oem_gram_weighted and oem_fit_path. */
typedef struct {
  int32_t nlambda; double lambda_min_ratio; const double* lambda /*host, optional*/;
  double tol_in; int64_t maxit_in; double tol_out; int32_t outer_maxit;
  double eps; int32_t d_squarings; const double* var_w /*device p or NULL*/;
  const int32_t* group; int32_t ngroups; const double* grp_w; /* host; group families as in oem_path_cfg */
  int32_t hessian_upper_bound; /* f1 (R#27): w_i = 1/4. The Gram X^T X and d_w are
                                  formed once (a2 pass); each outer step is one oem_logit_grad
                                  pass and c = X^T X beta + 4 X^T (y - mu), normalised by 4n.
                                  Needs p <= 512. */
} oem_logistic_cfg;
void oem_logistic_cfg_default(oem_logistic_cfg* cfg);  /* 50, 1e-3, NULL, 1e-11, 1e5, 1e-10, 100, 1e-5, 12, NULL, NULL, 0, NULL, 0 */

/* ---- f1 logistic gradient pass (P:L357-359 mu(x) = 1/(1 + exp(-x^T beta)); P:L385-389 the
 * upper-bound step needs only X^T (y - mu)). One HBM-bound pass over [X | y]: g = sum_i
 * (y_i - mu_i) x_i (p) and loglik = sum_i [y_i eta_i - log(1 + e^eta_i)] (1, device, or NULL: not
 * formed, which drops a third of the per-row fp64 work), raw sums over this
 * rank's rows, allreduced when the context has a communicator. beta (device, p) identical on every rank. No clamp of
 * mu (no division by w). Errors: OEM_ERR_DIM, OEM_ERR_ALIGN (X 16-byte aligned, ldx even),
 * OEM_ERR_UNSUPPORTED (p > 512), OEM_ERR_CUDA, OEM_ERR_NCCL. */
oem_status oem_logit_grad(oem_ctx* ctx, const double* X, const double* y01, const double* beta, int64_t n_local,
                          int32_t p, int64_t ldx, double* g, double* loglik, void* stream);
oem_status oem_fit_logistic(oem_ctx* ctx, const double* X, const double* y01, int64_t n_local, int32_t p,
                            int64_t ldx, const oem_penalty* pen /*host, one*/, const oem_logistic_cfg* cfg /*host*/,
                            double* beta_out, double* lambda_out, int32_t* outer_iters /*host L*/,
                            int64_t* inner_iters /*host L*/, uint8_t* converged /*host L*/, void* stream);

/* ---- f4 out-of-core Gram passes (the big.oem analogue, §5.7: X kept out of core,
 * the p x p statistics accumulated block by block). X (row-major, ldx even) and y are HOST
 * pointers, ideally pinned (cudaHostAlloc / torch pin_memory) so the copies run asynchronously:
 * blocks of block_rows rows are copied to two device staging buffers on an internal copy stream
 * while the Gram kernel consumes the other buffer on `stream`, and the block results are added
 * in block order (deterministic). Outputs and errors as oem_gram / oem_gram_folds (device
 * outputs), plus OEM_ERR_INVALID_ARG for block_rows < 32. Device memory used: 2 blocks.
 * The caller must keep X and y unchanged until `stream` has passed the call (the copies are
 * asynchronous). */
oem_status oem_gram_host(oem_ctx* ctx, const double* X /*host*/, const double* y /*host*/, int64_t n_local,
                         int32_t p, int64_t ldx, int64_t block_rows, double* G, double* xty, double* yty,
                         int64_t* n_total, void* stream);
oem_status oem_gram_folds_host(oem_ctx* ctx, const double* X /*host*/, const double* y /*host*/, int64_t n_local,
                               int32_t p, int64_t ldx, int64_t row_offset, int32_t K, int64_t block_rows,
                               double* G_folds, double* xty_folds, double* yty_folds, int64_t* counts /*host K*/,
                               void* stream);

/* ---- f4 sparse design (§5.8: oem() accepts sparse design matrices; "a substantial
 * computational speedup and reduction in memory usage"). The a2 statistics of one pass over a
 * design in compressed sparse row form: row_ptr (device int64, n_local + 1 offsets into col/val;
 * row i holds entries [row_ptr[i], row_ptr[i+1])), col (device int32, column indices strictly
 * ascending within each row, each in [0, p)), val (device fp64), y (device, n_local). Outputs,
 * communicator and n_total exactly as oem_gram: G = X^T X (full symmetric p*p), xty, yty,
 * raw sums over this rank's rows (the ranks' CSR blocks are their row shards), so the result
 * feeds oem_fit_path unchanged. Work and traffic scale with the nonzeros (each row contributes
 * the products of its nonzeros only). Deterministic (fixed partition and summation order).
 * The CSR precondition (ascending, in-range columns) is not checked on the device.
 * Errors: OEM_ERR_DIM, OEM_ERR_INVALID_ARG, OEM_ERR_UNSUPPORTED (p > 768), OEM_ERR_CUDA,
 * OEM_ERR_NCCL. */
oem_status oem_gram_csr(oem_ctx* ctx, const int64_t* row_ptr, const int32_t* col, const double* val,
                        const double* y, int64_t n_local, int32_t p, double* G, double* xty, double* yty,
                        int64_t* n_total /*host, may be NULL*/, void* stream);

/* ---- f3 column sums for the intercept / standardization (R#2-3): xsum[k*p + j] = sum of
 * x_ij over this rank's rows i of fold k (fold(i) = (row_offset + i) mod K, R#19; K = 1 for the
 * whole data), ysum[k] = sum of y_i; raw sums, allreduced when the context has a communicator. One HBM-bound pass.
 * Errors: OEM_ERR_DIM, OEM_ERR_INVALID_ARG (K < 1), OEM_ERR_UNSUPPORTED (K > 64), OEM_ERR_CUDA. */
oem_status oem_gram_moments(oem_ctx* ctx, const double* X, const double* y, int64_t n_local, int32_t p,
                            int64_t ldx, int64_t row_offset, int32_t K, double* xsum /*K*p*/,
                            double* ysum /*K*/, void* stream);

/* ---- f3 compute.loss: the loss of every fitted path point from the unit's
 * sufficient statistics alone (no pass over X, R#37): loss[g][q][l] = (yty_g - 2 b^T xty_g +
 * b^T G_g b) / n_g, the mean squared residual of b = beta[g][q][l] (no intercept; for a fit with
 * intercept pass the centred statistics). Inputs: raw G (nG*p*p), xty (nG*p), yty (nG), counts
 * (host nG), beta (nG*nP*L*p). The Gaussian log-likelihood is -n/2 (log(2 pi loss) + 1).
 * Errors: OEM_ERR_DIM, OEM_ERR_EMPTY_FOLD (count 0), OEM_ERR_UNSUPPORTED, OEM_ERR_CUDA. */
oem_status oem_path_loss(oem_ctx* ctx, const double* G, const double* xty, const double* yty,
                         const int64_t* counts /*host nG*/, int32_t nG, int32_t p, int32_t nP, int32_t L,
                         const double* beta, double* loss, void* stream);

/* ---- f2 fast cross-validation error and selection (§3; P:L601-616, L659-660,
 * L689-690 §5.4-5.5 cv.oem / xval.oem outputs; R#33-35). Inputs: the K raw fold sums of
 * oem_gram_folds (G_folds K*p*p, xty_folds K*p, yty_folds K, counts host K) and the coefficient
 * paths of oem_fit_path in fold_mode (beta (K+1)*nP*L*p; unit k+1 = fit on the complement of
 * fold k). No pass over X: err[k][q][l] = (yty_k - 2 b^T xty_k + b^T G_k b) / n_k is the held-out
 * mean squared error of b = beta[k+1][q][l] on fold k (R#33). A fit with an intercept (the
 * intercept_out of a fold-mode oem_path_cfg with xsum/ysum) passes intercept ((K+1)*nP*L,
 * device) with the fold column sums of oem_gram_moments (xsum_folds K*p, ysum_folds K); the
 * error is then of y - b0 - X b: the above + b0 (2 b^T xsum_k - 2 ysum_k + n_k b0) / n_k.
 * intercept = NULL: no intercept (xsum_folds / ysum_folds ignored, may be NULL).
 * Summaries per penalty q (device): cvm[q][l] = sum_k n_k err / n,
 * cvsd[q][l] = sqrt(sum_k n_k (err - cvm)^2 / n / (K-1)) (R#34).
 * Host outputs (may be NULL): idx_min[q] = first argmin_l cvm (the larger lambda on ties),
 * idx_1se[q] = smallest l with cvm[l] <= cvm[idx_min] + cvsd[idx_min] (the largest such lambda),
 * best = penalty with the smallest min cvm (the first on ties) (R#35). Synchronises `stream`.
 * Errors: OEM_ERR_DIM (K < 2, p/nP/L < 1), OEM_ERR_EMPTY_FOLD, OEM_ERR_INVALID_ARG (intercept
 * without the fold sums), OEM_ERR_UNSUPPORTED (nP > 64, 8p bytes > 200 KB), OEM_ERR_CUDA. */
oem_status oem_cv_error(oem_ctx* ctx, const double* G_folds, const double* xty_folds, const double* yty_folds,
                        const int64_t* counts /*host K*/, int32_t K, int32_t p, int32_t nP, int32_t L,
                        const double* beta, const double* xsum_folds, const double* ysum_folds,
                        const double* intercept, double* err, double* cvm, double* cvsd, int32_t* idx_min /*host nP*/,
                        int32_t* idx_1se /*host nP*/, int32_t* best /*host 1*/, void* stream);

/* ---- instrumentation (used by bench.py; no effect on results).
 * With timing enabled the library records CUDA events around its phases on the launching
 * stream; oem_ctx_stats synchronises those events and returns the accumulated device times. */
typedef struct {
  int64_t launches;      /* kernels this context launched (all phases) */
  double gram_ms;        /* Gram-pass tensor-core kernels (a2/a3/a4) */
  double reduce_ms;      /* split-n reduction, fold tail, unpack */
  double allreduce_ms;   /* NCCL combine (a5) */
  double power_ms;       /* d (a7) */
  double path_ms;        /* normalise + lambda grid + OEM path solver (a6, a8-a10) */
} oem_stats;
oem_status oem_ctx_set_timing(oem_ctx* ctx, int enable);
oem_status oem_ctx_stats(oem_ctx* ctx, oem_stats* out /*host*/, int reset);

#ifdef __cplusplus
}
#endif
#endif
