/* oracle.h — plain, slow, obviously-correct CPU reference of the OEM hot path.
 *
 * TEST INFRASTRUCTURE ONLY. Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
 * --impl reference leg may load liboracle.so. The product path (liboem.so and its binding)
 * never links, loads or calls anything here, and this file shares no code with it.
 *
 * Citations: "P:Lnnn" = /root/reference/PAPER.md line nnn (the paper, arXiv 1801.09661);
 * "S:Lnnn" = SPEC.md line nnn; readings "R#k" = DESIGN.md §3 reading k (= SURVEY.md §8(c).2 #k).
 * All arithmetic is IEEE fp64; sums over rows use compensated (Neumaier) accumulation of exact
 * products (TwoProduct by fma), so the oracle's own error is far below the 1e-12 parity bar.
 *
 * Pins (tests/test_oracle_*.py, marker "not gpu") tie every function to something other than
 * itself: exact integer arithmetic, closed forms, SPEC/paper worked values, library routines
 * (numpy eigvalsh / solve), brute-force enumeration and independent solvers.
 */
#ifndef OEM_ORACLE_H
#define OEM_ORACLE_H
#include <stdint.h>
#ifdef __cplusplus
extern "C" {
#endif

/* ---- O1 Gram ("A = Delta^T Delta", u = X^T y + A beta; "key computational
 * step ... forming the matrix A"; P:L328-333 O(np^2+np)). Raw sums, no normalization:
 * G[j*p+k] = sum_i x_ij x_ik (full symmetric p*p), xty[j] = sum_i x_ij y_i, yty = sum_i y_i^2.
 * X row-major with leading dimension ldx. Streaming form: state holds 2*(p*p+p+1) doubles. */
void orc_gram_begin(int32_t p, double* state);
void orc_gram_add(const double* X, const double* y, int64_t n, int32_t p, int64_t ldx, double* state,
                  int nthreads);
void orc_gram_end(int32_t p, const double* state, double* G, double* xty, double* yty);
void orc_gram(const double* X, const double* y, int64_t n, int32_t p, int64_t ldx, double* G,
              double* xty, double* yty, int nthreads);

/* ---- O2 fold Grams (§3: X partitioned into X_1..X_K; A_(k) built from
 * sum_{c != k} X_c^T X_c). fold(i) = (row_offset + i) mod K (R#19). Outputs K raw-sum Grams
 * Gk[k*p*p + j*p + l], xtyk[k*p + j], ytyk[k], counts[k]. */
void orc_gram_folds(const double* X, const double* y, int64_t n, int32_t p, int64_t ldx,
                    int64_t row_offset, int32_t K, double* Gk, double* xtyk, double* ytyk,
                    int64_t* counts, int nthreads);
/* Training statistics in the paper's own form sum_{c != k}, not total-minus-fold. */
void orc_fold_complements(const double* Gk, const double* xtyk, int32_t K, int32_t p,
                          double* Gminus, double* xtyminus);

/* ---- O3 weighted Gram for proximal Newton (§4; working response z and weights w
 * at P:L376-380; R#23-25). Per row: eta = x_i^T beta, mu = 1/(1+exp(-eta)) clamped to
 * [eps, 1-eps], w = mu(1-mu), z = eta + (y - mu)/w. Raw sums: Gw = sum w x x^T (full p*p),
 * cw = sum w z x, scalars[0] = sum w, scalars[1] = sum [y eta - log(1+exp(eta))]. */
void orc_gram_weighted(const double* X, const double* y01, const double* beta, int64_t n, int32_t p,
                       int64_t ldx, double eps, double* Gw, double* cw, double* scalars, int nthreads);

/* ---- O4 d (§2.1: OEM converges for d >= lambda_1(X^T X); d = lambda_1 fastest).
 * orc_eig_jacobi: all eigenvalues of symmetric A (p*p) by cyclic Jacobi (textbook), ascending.
 * orc_d_rule: the d rule of R#5: d = min(Gershgorin max row sum, U_S) with
 *   U_S = trace(A^(2^S))^(1/2^S) >= lambda_1 (A symmetric PSD), formed by S squarings of the
 *   trace-normalised matrix. Returns d; U / gersh optional outputs. */
void orc_eig_jacobi(const double* A, int32_t p, double* evals);
double orc_d_rule(const double* A, int32_t p, int32_t squarings, double* U, double* gersh);

/* ---- thresholding operators (§2.2, eqs lasso/net/mcp/scad/glasso/gmcp/gscad).
 * lam is the already-weighted level (w_j*lambda or c_k*lambda). */
double orc_soft(double u, double lam, double d);                          /* eq (lasso) */
double orc_enet(double u, double lam, double alpha, double d);            /* eq (net), lam = w_j*lambda */
double orc_mcp(double u, double lam, double gamma, double d);             /* eq (mcp) */
double orc_scad(double u, double lam, double gamma, double d);            /* eq (scad) */
/* group forms: u (m), out (m) */
void orc_grp_lasso(const double* u, int32_t m, double lam, double d, double* out);            /* eq (glasso) */
void orc_grp_mcp(const double* u, int32_t m, double lam, double gamma, double d, double* out); /* eq (gmcp) */
/* sparse group lasso M-step, exact d-scaled composition (R#11): v_i = S(u_i, w_i lam tau, d),
   out = v (1 - c lam (1 - tau) / (d ||v||))_+ ; w may be NULL (= 1) */
void orc_sgl(const double* u, const double* w, int32_t m, double lam, double tau, double c, double d, double* out);
void orc_grp_scad(const double* u, int32_t m, double lam, double gamma, double d, double* out);/* eq (gscad) */

/* ---- penalty families (Table 1) ---- */
enum { ORC_LASSO = 0, ORC_ENET = 1, ORC_MCP = 2, ORC_SCAD = 3, ORC_GRP_LASSO = 4, ORC_GRP_MCP = 5, ORC_GRP_SCAD = 6,
       ORC_SGL = 7 /* sparse group lasso, tau passed as alpha (R#11) */ };

/* lambda_max (R#14): smallest lambda for which beta = 0 is a fixed point. c is the normalized
 * X^T y / n. w: p or NULL (=1). group: p ids or NULL; grp_w: ngroups or NULL (= sqrt(size), R#12). */
double orc_lambda_max(int family, double alpha, const double* c, int32_t p, const double* w,
                      const int32_t* group, int32_t ngroups, const double* grp_w);
/* lambda_i = lmax * exp((i/(L-1)) ln ratio), i = 0..L-1 (R#15); L = 1 gives lmax. */
void orc_lambda_grid(double lmax, int32_t L, double ratio, double* lambdas);

/* ---- O6 OEM path (P:L147-158 Steps 1/2.1/2.2; P:L171-188 u = X^T y + A beta with
 * A = dI - X^T X; M-step = thresholding P:L239-289; warm starts R#18; stop rule R#17).
 * G: p*p full symmetric NORMALIZED Gram, c: normalized X^T y. For each lambda in order:
 *   repeat: u = c + d*beta - G beta; beta' = Theta(u); delta = max|beta'-beta|; beta = beta'
 *   until delta <= tol (converged) or maxit updates. beta_out: L*p; iters: L; conv: L.
 * Returns 0, or -1 on invalid parameters (gamma*d <= 1 for MCP, (gamma-1)*d <= 1 for SCAD, R#8). */
int orc_oem_path(const double* G, const double* c, int32_t p, double d, int family, double gamma,
                 double alpha, const double* w, const int32_t* group, int32_t ngroups,
                 const double* grp_w, const double* lambdas, int32_t L, double tol, int64_t maxit,
                 const double* beta_init, double* beta_out, int64_t* iters, uint8_t* conv);

/* Penalized least-squares objective from the Gram (R#1): 0.5 b^T G b - c^T b + P_lambda(b)
 * (differs from (1/2n)||y - Xb||^2 + P by the constant 0.5 yty/n). Table 1 penalty forms. */
double orc_objective(const double* G, const double* c, int32_t p, const double* beta, int family,
                     double lambda, double gamma, double alpha, const double* w,
                     const int32_t* group, int32_t ngroups, const double* grp_w);

/* ---- O7 logistic proximal Newton (§4; R#23-26). For each lambda (warm start):
 * repeat outer: O3 at beta; normalize by n; d_w by the d rule (squarings); inner OEM (O6) for
 * the single lambda from beta with the given penalty family (any of Table 1, groups as in O6;
 * tol_in, maxit_in); stop when max|beta_new - beta| <= tol_out or outer_maxit.
 * outer_iters: L; inner_iters: L (sum over outer steps); conv: L; d_out (optional): d_w of the
 * first outer step. Returns 0, -1 (y not 0/1) or -1 from O6 (invalid penalty parameters). */
int orc_logistic_path(const double* X, const double* y01, int64_t n, int32_t p, int64_t ldx, int family,
                      double gamma, double alpha, const double* w, const int32_t* group, int32_t ngroups,
                      const double* grp_w, const double* lambdas, int32_t L, double eps, double tol_in,
                      int64_t maxit_in, double tol_out, int32_t outer_maxit, int32_t squarings,
                      double* beta_out, int32_t* outer_iters, int64_t* inner_iters, uint8_t* conv,
                      double* d_out, int nthreads);

#ifdef __cplusplus
}
#endif
#endif
