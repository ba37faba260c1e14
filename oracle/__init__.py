"""oracle — plain CPU reference of the OEM hot path (§2-§4, arXiv 1801.09661).

TEST INFRASTRUCTURE ONLY. Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s
``cpu_baseline`` / ``--impl reference`` leg may import this package. The product path
(``paper_1801_09661_b200``) never imports it, and it imports nothing from the product path.

The arithmetic lives in ``oracle.c`` (naive loops, compensated fp64 sums); this module only
marshals numpy arrays through ctypes and composes the documented steps (normalize -> d ->
lambda grid -> path) in the paper's order. Each function names the passage it follows
("P:Lnnn" = PAPER.md line, "R#k" = reading k in DESIGN.md §3).

Parity status: every function below is pinned by a ``-m "not gpu"`` test in
``tests/test_oracle_*.py`` except where its docstring says "parity unpinned".
"""
from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SO = os.path.join(_HERE, "liboracle.so")

LASSO, ENET, MCP, SCAD, GRP_LASSO, GRP_MCP, GRP_SCAD, SGL = range(8)
FAMILY = {"lasso": LASSO, "enet": ENET, "mcp": MCP, "scad": SCAD,
          "grp_lasso": GRP_LASSO, "grp_mcp": GRP_MCP, "grp_scad": GRP_SCAD,
          "sgl": SGL}   # sparse group lasso: tau is passed as alpha (R#11)


def build(force: bool = False) -> str:
    """Compile liboracle.so (gcc; the checker is built, not used, by __graft_entry__.build())."""
    src = os.path.join(_HERE, "oracle.c")
    if force or not os.path.exists(_SO) or os.path.getmtime(_SO) < max(
            os.path.getmtime(src), os.path.getmtime(os.path.join(_HERE, "oracle.h"))):
        subprocess.check_call(["gcc", "-O2", "-mfma", "-ffp-contract=off", "-fopenmp", "-fPIC",
                               "-shared", "-o", _SO, src, "-lm"])
    return _SO


_lib = None


def lib():
    global _lib
    if _lib is None:
        build()
        _lib = ctypes.CDLL(_SO)
        d, i32, i64, p = ctypes.c_double, ctypes.c_int32, ctypes.c_int64, ctypes.c_void_p
        sig = {
            "orc_gram_begin": (None, [i32, p]),
            "orc_gram_add": (None, [p, p, i64, i32, i64, p, ctypes.c_int]),
            "orc_gram_end": (None, [i32, p, p, p, p]),
            "orc_gram": (None, [p, p, i64, i32, i64, p, p, p, ctypes.c_int]),
            "orc_gram_folds": (None, [p, p, i64, i32, i64, i64, i32, p, p, p, p, ctypes.c_int]),
            "orc_fold_complements": (None, [p, p, i32, i32, p, p]),
            "orc_gram_weighted": (None, [p, p, p, i64, i32, i64, d, p, p, p, ctypes.c_int]),
            "orc_eig_jacobi": (None, [p, i32, p]),
            "orc_d_rule": (d, [p, i32, i32, p, p]),
            "orc_soft": (d, [d, d, d]),
            "orc_enet": (d, [d, d, d, d]),
            "orc_mcp": (d, [d, d, d, d]),
            "orc_scad": (d, [d, d, d, d]),
            "orc_grp_lasso": (None, [p, i32, d, d, p]),
            "orc_grp_mcp": (None, [p, i32, d, d, d, p]),
            "orc_grp_scad": (None, [p, i32, d, d, d, p]),
            "orc_sgl": (None, [p, p, i32, d, d, d, d, p]),
            "orc_lambda_max": (d, [ctypes.c_int, d, p, i32, p, p, i32, p]),
            "orc_lambda_grid": (None, [d, i32, d, p]),
            "orc_oem_path": (ctypes.c_int, [p, p, i32, d, ctypes.c_int, d, d, p, p, i32, p, p, i32,
                                            d, i64, p, p, p, p]),
            "orc_objective": (d, [p, p, i32, p, ctypes.c_int, d, d, d, p, p, i32, p]),
            "orc_logistic_path": (ctypes.c_int, [p, p, i64, i32, i64, ctypes.c_int, d, d, p, p, i32,
                                                 p, p, i32, d, d, i64, d, i32, i32, p, p, p, p, p,
                                                 ctypes.c_int]),
        }
        for name, (res, args) in sig.items():
            f = getattr(_lib, name)
            f.restype = res
            f.argtypes = args
    return _lib


def _ptr(a):
    return None if a is None else a.ctypes.data_as(ctypes.c_void_p)


def _f64(a):
    return None if a is None else np.ascontiguousarray(a, dtype=np.float64)


def _nthreads(n):
    return max(1, min(os.cpu_count() or 1, 16))


# ---------------------------------------------------------------- O1 / O2 / O3
def gram(X, y, nthreads=None):
    """O1: raw G = X^T X (full symmetric), X^T y, y^T y."""
    X = _f64(X)
    y = _f64(y)
    n, p = X.shape
    G = np.empty((p, p))
    c = np.empty(p)
    yy = np.empty(1)
    lib().orc_gram(_ptr(X), _ptr(y), n, p, p, _ptr(G), _ptr(c), _ptr(yy), nthreads or _nthreads(n))
    return G, c, float(yy[0])


class GramAccumulator:
    """O1 in streaming form: add row blocks, then finalize (block-size invariant)."""

    def __init__(self, p):
        self.p = p
        self.state = np.zeros(2 * (p * p + p + 1))
        lib().orc_gram_begin(p, _ptr(self.state))
        self.n = 0

    def add(self, X, y, nthreads=None):
        X = _f64(X)
        y = _f64(y)
        n, p = X.shape
        assert p == self.p
        lib().orc_gram_add(_ptr(X), _ptr(y), n, p, p, _ptr(self.state), nthreads or _nthreads(n))
        self.n += n

    def result(self):
        p = self.p
        G = np.empty((p, p))
        c = np.empty(p)
        yy = np.empty(1)
        lib().orc_gram_end(p, _ptr(self.state), _ptr(G), _ptr(c), _ptr(yy))
        return G, c, float(yy[0])


def gram_folds(X, y, K, row_offset=0, nthreads=None):
    """O2: per-fold raw Grams with fold(i) = (row_offset + i) mod K (R#19)."""
    X = _f64(X)
    y = _f64(y)
    n, p = X.shape
    Gk = np.empty((K, p, p))
    ck = np.empty((K, p))
    yyk = np.empty(K)
    cnt = np.empty(K, dtype=np.int64)
    lib().orc_gram_folds(_ptr(X), _ptr(y), n, p, p, row_offset, K, _ptr(Gk), _ptr(ck), _ptr(yyk),
                         _ptr(cnt), nthreads or _nthreads(n))
    return Gk, ck, yyk, cnt


def fold_complements(Gk, ck):
    """O2: training statistics sum_{c != k} X_c^T X_c, sum_{c != k} X_c^T y_c."""
    Gk = _f64(Gk)
    ck = _f64(ck)
    K, p, _ = Gk.shape
    Gm = np.empty_like(Gk)
    cm = np.empty_like(ck)
    lib().orc_fold_complements(_ptr(Gk), _ptr(ck), K, p, _ptr(Gm), _ptr(cm))
    return Gm, cm


def gram_weighted(X, y01, beta, eps=1e-5, nthreads=None):
    """O3: raw G_w = sum w x x^T, c_w = sum w z x, (sum w, loglik) (R#23-25)."""
    X = _f64(X)
    y01 = _f64(y01)
    beta = _f64(beta)
    n, p = X.shape
    Gw = np.empty((p, p))
    cw = np.empty(p)
    sc = np.empty(2)
    lib().orc_gram_weighted(_ptr(X), _ptr(y01), _ptr(beta), n, p, p, eps, _ptr(Gw), _ptr(cw),
                            _ptr(sc), nthreads or _nthreads(n))
    return Gw, cw, sc


# ---------------------------------------------------------------- O4 d
def eig_jacobi(A):
    """O4: eigenvalues (ascending) of symmetric A by cyclic Jacobi (textbook)."""
    A = _f64(A)
    p = A.shape[0]
    ev = np.empty(p)
    lib().orc_eig_jacobi(_ptr(A), p, _ptr(ev))
    return ev


SQUARINGS = 12   # R#5: S, so U_S is within a factor p^(1/4096) of lambda_1 (0.17% at p = 1000)


def d_rule(A, squarings=SQUARINGS):
    """O4: d = min(Gershgorin, U_S), U_S = trace(A^(2^S))^(1/2^S) >= lambda_1 (R#5
    "d >= lambda_1 ... d = lambda_1 fastest"). Returns (d, U_S, Gershgorin)."""
    A = _f64(A)
    u = np.empty(1)
    gs = np.empty(1)
    d = lib().orc_d_rule(_ptr(A), A.shape[0], squarings, _ptr(u), _ptr(gs))
    return d, float(u[0]), float(gs[0])


# ---------------------------------------------------------------- thresholds
def soft(u, lam, d):
    return lib().orc_soft(u, lam, d)


def enet(u, lam, alpha, d):
    return lib().orc_enet(u, lam, alpha, d)


def mcp(u, lam, gamma, d):
    return lib().orc_mcp(u, lam, gamma, d)


def scad(u, lam, gamma, d):
    return lib().orc_scad(u, lam, gamma, d)


def grp_lasso(u, lam, d):
    u = _f64(u)
    out = np.empty_like(u)
    lib().orc_grp_lasso(_ptr(u), u.size, lam, d, _ptr(out))
    return out


def grp_mcp(u, lam, gamma, d):
    u = _f64(u)
    out = np.empty_like(u)
    lib().orc_grp_mcp(_ptr(u), u.size, lam, gamma, d, _ptr(out))
    return out


def grp_scad(u, lam, gamma, d):
    u = _f64(u)
    out = np.empty_like(u)
    lib().orc_grp_scad(_ptr(u), u.size, lam, gamma, d, _ptr(out))
    return out


def sgl(u, lam, tau, c, d, w=None):
    """Sparse group lasso M-step for one group, exact d-scaled composition (R#11)."""
    u = _f64(u)
    out = np.empty_like(u)
    lib().orc_sgl(_ptr(u), _ptr(_f64(w)), u.size, lam, tau, c, d, _ptr(out))
    return out


# ---------------------------------------------------------------- lambda grid / path
def _groups(group, ngroups):
    if group is None:
        return None, 0
    g = np.ascontiguousarray(group, dtype=np.int32)
    return g, int(ngroups if ngroups else g.max() + 1)


def lambda_max(family, c, w=None, group=None, ngroups=0, grp_w=None, alpha=1.0):
    """R#14: smallest lambda with beta = 0 a fixed point."""
    c = _f64(c)
    g, ng = _groups(group, ngroups)
    return lib().orc_lambda_max(FAMILY[family], alpha, _ptr(c), c.size, _ptr(_f64(w)), _ptr(g), ng,
                                _ptr(_f64(grp_w)))


def lambda_grid(lmax, L, ratio=1e-3):
    """R#15: lambda_i = lmax * exp((i/(L-1)) ln ratio)."""
    out = np.empty(L)
    lib().orc_lambda_grid(lmax, L, ratio, _ptr(out))
    return out


def oem_path(G, c, d, family, lambdas, gamma=3.0, alpha=1.0, w=None, group=None, ngroups=0,
             grp_w=None, tol=1e-11, maxit=100000, beta_init=None):
    """O6: warm-started OEM path u = c + d beta - G beta, beta = Theta(u).

    G, c: NORMALIZED Gram and X^T y. Returns (beta[L,p], iters[L], conv[L])."""
    G = _f64(G)
    c = _f64(c)
    lambdas = _f64(np.atleast_1d(lambdas))
    p = c.size
    L = lambdas.size
    g, ng = _groups(group, ngroups)
    B = np.empty((L, p))
    it = np.empty(L, dtype=np.int64)
    cv = np.empty(L, dtype=np.uint8)
    rc = lib().orc_oem_path(_ptr(G), _ptr(c), p, d, FAMILY[family], gamma, alpha, _ptr(_f64(w)),
                            _ptr(g), ng, _ptr(_f64(grp_w)), _ptr(lambdas), L, tol, maxit,
                            _ptr(_f64(beta_init)), _ptr(B), _ptr(it), _ptr(cv))
    if rc != 0:
        raise ValueError("oracle oem_path: invalid parameters (d, gamma, alpha or groups)")
    return B, it, cv.astype(bool)


def objective(G, c, beta, family, lam, gamma=3.0, alpha=1.0, w=None, group=None, ngroups=0,
              grp_w=None):
    """0.5 b^T G b - c^T b + P_lambda(b) with Table 1 penalties (R#1)."""
    G = _f64(G)
    c = _f64(c)
    beta = _f64(beta)
    g, ng = _groups(group, ngroups)
    return lib().orc_objective(_ptr(G), _ptr(c), c.size, _ptr(beta), FAMILY[family], lam, gamma,
                               alpha, _ptr(_f64(w)), _ptr(g), ng, _ptr(_f64(grp_w)))


def logistic_path(X, y01, lambdas, family="lasso", gamma=3.0, alpha=1.0, w=None, group=None,
                  ngroups=0, grp_w=None, eps=1e-5, tol_in=1e-11, maxit_in=100000, tol_out=1e-10,
                  outer_maxit=100, squarings=SQUARINGS, nthreads=None, return_d=False):
    """O7: proximal-Newton logistic path with OEM inner solves (R#23-26), any
    Table 1 family (groups as in O6). Returns (B[L,p], outer[L], inner[L], conv[L]) and, with
    return_d, the first outer step's d_w."""
    X = _f64(X)
    y01 = _f64(y01)
    lambdas = _f64(np.atleast_1d(lambdas))
    n, p = X.shape
    L = lambdas.size
    g, ng = _groups(group, ngroups)
    B = np.empty((L, p))
    oi = np.empty(L, dtype=np.int32)
    ii = np.empty(L, dtype=np.int64)
    cv = np.empty(L, dtype=np.uint8)
    d0 = np.zeros(1)
    rc = lib().orc_logistic_path(_ptr(X), _ptr(y01), n, p, p, FAMILY[family], gamma, alpha,
                                 _ptr(_f64(w)), _ptr(g), ng, _ptr(_f64(grp_w)), _ptr(lambdas), L,
                                 eps, tol_in, maxit_in, tol_out, outer_maxit, squarings, _ptr(B),
                                 _ptr(oi), _ptr(ii), _ptr(cv), _ptr(d0), nthreads or _nthreads(n))
    if rc != 0:
        raise ValueError("oracle logistic_path: y must be 0/1 and the penalty parameters valid")
    if return_d:
        return B, oi, ii, cv.astype(bool), float(d0[0])
    return B, oi, ii, cv.astype(bool)


# ---------------------------------------------------------------- composed fit (§8(a) a6-a10)
def fit_from_gram(G_raw, c_raw, n, penalties, nlambda=100, ratio=1e-3, d=None, tol=1e-11,
                  maxit=100000, w=None, group=None, ngroups=0, grp_w=None, squarings=SQUARINGS,
                  lambda_max_override=None):
    """a6 normalize (/n, R#1) -> a7 d (rule R#5, or the d given) -> a8 grid per family (R#14-16)
    -> a9 path per penalty. penalties: list of (family, gamma, alpha). Returns dict."""
    Gn = np.asarray(G_raw, dtype=np.float64) / n
    cn = np.asarray(c_raw, dtype=np.float64) / n
    if d is None:
        d = d_rule(Gn, squarings)[0]
    out = {"d": d, "beta": [], "lambda": [], "iters": [], "conv": []}
    for fam, gamma, alpha in penalties:
        lmax = lambda_max_override if lambda_max_override is not None else lambda_max(
            fam, cn, w, group, ngroups, grp_w, alpha)
        lam = lambda_grid(lmax, nlambda, ratio)
        B, it, cv = oem_path(Gn, cn, d, fam, lam, gamma, alpha, w, group, ngroups, grp_w, tol, maxit)
        out["beta"].append(B)
        out["lambda"].append(lam)
        out["iters"].append(it)
        out["conv"].append(cv)
    return out


# ---------------------------------------------------------------- f2: fast-CV error and selection
def cv_error(X, y, K, beta_units, row_offset=0, intercepts=None):
    """f2 held-out error by its plain definition (R#33): for fold k (rows with (row_offset + i)
    mod K == k, R#19) and the fit (b0, b) = (intercepts[k+1][q][l], beta_units[k+1][q][l]) on the
    complement of fold k, e_k(l) = (1/n_k) sum_{i in fold k} (y_i - b0 - x_i^T b)^2
    (b0 = 0 without intercepts). The held-out rows are streamed directly (a matmul per fold as the
    library step); the Gram identity the product uses is NOT used here. Returns err [K][nP][L]."""
    X = _f64(X)
    y = _f64(y)
    B = np.asarray(beta_units, dtype=np.float64)
    nU, nP, L, p = B.shape
    assert nU == K + 1 and p == X.shape[1]
    B0 = np.zeros((nU, nP, L)) if intercepts is None else np.asarray(intercepts, dtype=np.float64)
    fold = (row_offset + np.arange(X.shape[0])) % K
    err = np.empty((K, nP, L))
    for k in range(K):
        rows = fold == k
        Xk, yk = X[rows], y[rows]
        R = yk[:, None] - B0[k + 1].reshape(nP * L)[None, :] - Xk @ B[k + 1].reshape(nP * L, p).T
        err[k] = (np.sum(R * R, axis=0) / rows.sum()).reshape(nP, L)
    return err


def cv_summary(err, counts):
    """f2 cv.oem summaries (P:L601-616 best.model / lambda.min; P:L659-660 lambda.1se; R#34-35),
    explicit loops: cvm = sum_k n_k e_k / n; cvsd = sqrt(sum_k n_k (e_k - cvm)^2 / n / (K-1));
    lambda_min = first argmin (larger lambda on ties); lambda_1se = largest lambda (smallest
    index) with cvm <= cvm_min + cvsd_min; best = first penalty attaining the smallest min cvm."""
    err = np.asarray(err, dtype=np.float64)
    K, nP, L = err.shape
    nk = [float(c) for c in counts]
    n = sum(nk)
    cvm = np.zeros((nP, L))
    cvsd = np.zeros((nP, L))
    for q in range(nP):
        for l in range(L):
            m = sum(nk[k] * err[k, q, l] for k in range(K)) / n
            v = sum(nk[k] * (err[k, q, l] - m) ** 2 for k in range(K))
            cvm[q, l] = m
            cvsd[q, l] = np.sqrt(v / n / (K - 1))
    imin, i1se = [], []
    for q in range(nP):
        im = 0
        for l in range(1, L):
            if cvm[q, l] < cvm[q, im]:
                im = l
        thr = cvm[q, im] + cvsd[q, im]
        i1 = next(l for l in range(im + 1) if cvm[q, l] <= thr)
        imin.append(im)
        i1se.append(i1)
    best = 0
    for q in range(1, nP):
        if cvm[q, imin[q]] < cvm[best, imin[best]]:
            best = q
    return cvm, cvsd, imin, i1se, best


# ---------------------------------------------------------------- f1: Hessian upper-bound logistic
def logit_grad(X, y01, beta):
    """f1 gradient pass by its definition: g = sum_i (y_i - mu_i) x_i with
    mu_i = 1/(1 + exp(-x_i^T beta)), and loglik = sum_i [y_i eta_i - log(1 + e^eta_i)] (R#23).
    numpy fp64 (matvecs as the library step)."""
    X = _f64(X)
    y01 = _f64(y01)
    eta = X @ _f64(beta)
    mu = 1.0 / (1.0 + np.exp(-eta))
    return X.T @ (y01 - mu), float(np.sum(y01 * eta - np.logaddexp(0.0, eta)))


def logistic_path_ub(X, y01, lambdas, family="lasso", gamma=3.0, alpha=1.0, d=None, tol_in=1e-11,
                     maxit_in=100000, tol_out=1e-10, outer_maxit=1000, squarings=SQUARINGS,
                     group=None, ngroups=0, grp_w=None):
    """f1: the proximal-Newton logistic path with the Hessian upper bound w_i = 1/4
    (R#27), in the paper's order: per outer step the working responses
    z_i = eta_i + (y_i - mu_i)/w_i with w_i = 1/4, the weighted statistics
    G_w = (1/n) sum w x x^T, c_w = (1/n) sum w z x, d_w by the d rule (R#5)
    unless d is given, then the OEM inner solve for the single lambda from the current beta
    (O6); stop when max |dbeta| <= tol_out. Returns (B[L,p], outer[L], inner[L], conv[L])."""
    X = _f64(X)
    y01 = _f64(y01)
    lambdas = _f64(np.atleast_1d(lambdas))
    n, p = X.shape
    w = 0.25
    beta = np.zeros(p)
    B = np.empty((lambdas.size, p))
    oi = np.zeros(lambdas.size, dtype=np.int32)
    ii = np.zeros(lambdas.size, dtype=np.int64)
    cv = np.zeros(lambdas.size, dtype=bool)
    for l, lam in enumerate(lambdas):
        for o in range(outer_maxit):
            eta = X @ beta
            mu = 1.0 / (1.0 + np.exp(-eta))
            z = eta + (y01 - mu) / w
            Gw = (w * X).T @ X / n
            cw = X.T @ (w * z) / n
            dw = d if d is not None else d_rule(Gw, squarings)[0]
            nb, it, ok = oem_path(Gw, cw, dw, family, [lam], gamma, alpha, group=group, ngroups=ngroups,
                                  grp_w=grp_w, tol=tol_in, maxit=maxit_in, beta_init=beta)
            ii[l] += it[0]
            oi[l] = o + 1
            delta = np.max(np.abs(nb[0] - beta)) if p else 0.0
            beta = nb[0].copy()
            if delta <= tol_out:
                cv[l] = True
                break
        B[l] = beta
    return B, oi, ii, cv


# ---------------------------------------------------------------- f3: intercept, standardization, loss
def fit_transformed(X, y, penalties, nlambda=100, ratio=1e-3, standardize=False, intercept=False, d=None,
                    lambdas=None, tol=1e-11, maxit=100000, w=None, group=None, ngroups=0, grp_w=None,
                    squarings=SQUARINGS):
    """f3 by transforming the DATA (R#2-3), not the Gram: with an intercept, X and y are centred
    explicitly (x_ij - xbar_j, y_i - ybar); with standardization the (centred) columns are divided
    by sd_j = sqrt(mean(x_ij^2)) (P:L173-177 with the /n convention of R#1); then O1 Gram -> a6-a9
    (fit_from_gram, the given d and lambda grid if any) and the map back to the original scale:
    beta_j = beta~_j / sd_j (0 for a zero-variance column), b0 = ybar - xbar^T beta.
    Returns dict(beta [nP][L][p], intercept [nP][L], d, lambda)."""
    X = _f64(X).copy()
    y = _f64(y).copy()
    n, p = X.shape
    xbar = X.mean(axis=0) if intercept else np.zeros(p)
    ybar = float(y.mean()) if intercept else 0.0
    X -= xbar
    y -= ybar
    sd = np.sqrt(np.mean(X * X, axis=0)) if standardize else np.ones(p)
    inv = np.where(sd > 0, 1.0 / np.where(sd > 0, sd, 1.0), 0.0)
    X *= inv
    G, c, _ = gram(X, y)
    out = {"beta": [], "intercept": [], "lambda": []}
    if d is None:
        d = d_rule(G / n, squarings)[0]
    out["d"] = d
    for q, (fam, gamma, alpha) in enumerate(penalties):
        if lambdas is None:
            lm = lambda_max(fam, c / n, w, group, ngroups, grp_w, alpha)
            lam = lambda_grid(lm, nlambda, ratio)
        else:
            lam = _f64(lambdas[q])
        B, _, _ = oem_path(G / n, c / n, d, fam, lam, gamma, alpha, w, group, ngroups, grp_w, tol, maxit)
        B = B * inv
        out["beta"].append(B)
        out["intercept"].append(ybar - B @ xbar)
        out["lambda"].append(lam)
    return out


def path_loss(X, y, B):
    """f3 compute.loss by its definition (R#37): mean((y - X b)^2) for every b in B[..., p]."""
    X = _f64(X)
    y = _f64(y)
    B = np.asarray(B, dtype=np.float64)
    R = y[:, None] - X @ B.reshape(-1, B.shape[-1]).T
    return (np.sum(R * R, axis=0) / X.shape[0]).reshape(B.shape[:-1])
