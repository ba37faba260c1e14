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

LASSO, ENET, MCP, SCAD, GRP_LASSO, GRP_MCP, GRP_SCAD = range(7)
FAMILY = {"lasso": LASSO, "enet": ENET, "mcp": MCP, "scad": SCAD,
          "grp_lasso": GRP_LASSO, "grp_mcp": GRP_MCP, "grp_scad": GRP_SCAD}


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
            "orc_power_rule": (d, [p, i32, i32, d, p, p]),
            "orc_soft": (d, [d, d, d]),
            "orc_enet": (d, [d, d, d, d]),
            "orc_mcp": (d, [d, d, d, d]),
            "orc_scad": (d, [d, d, d, d]),
            "orc_grp_lasso": (None, [p, i32, d, d, p]),
            "orc_grp_mcp": (None, [p, i32, d, d, d, p]),
            "orc_grp_scad": (None, [p, i32, d, d, d, p]),
            "orc_lambda_max": (d, [ctypes.c_int, d, p, i32, p, p, i32, p]),
            "orc_lambda_grid": (None, [d, i32, d, p]),
            "orc_oem_path": (ctypes.c_int, [p, p, i32, d, ctypes.c_int, d, d, p, p, i32, p, p, i32,
                                            d, i64, p, p, p, p]),
            "orc_objective": (d, [p, p, i32, p, ctypes.c_int, d, d, d, p, p, i32, p]),
            "orc_logistic_path": (ctypes.c_int, [p, p, i64, i32, i64, p, i32, d, d, i64, d, i32,
                                                 i32, d, p, p, p, p, ctypes.c_int]),
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


def power_rule(A, iters=200, inflate=5e-3):
    """O4: d = min(Gershgorin, (1+inflate) RQ_iters) from v0 = 1/sqrt(p) (R#5)."""
    A = _f64(A)
    rq = np.empty(1)
    gs = np.empty(1)
    d = lib().orc_power_rule(_ptr(A), A.shape[0], iters, inflate, _ptr(rq), _ptr(gs))
    return d, float(rq[0]), float(gs[0])


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


def logistic_path(X, y01, lambdas, eps=1e-5, tol_in=1e-11, maxit_in=100000, tol_out=1e-10,
                  outer_maxit=100, power_iters=200, inflate=5e-3, nthreads=None):
    """O7: proximal-Newton lasso-logistic path with OEM inner solves (R#23-26)."""
    X = _f64(X)
    y01 = _f64(y01)
    lambdas = _f64(np.atleast_1d(lambdas))
    n, p = X.shape
    L = lambdas.size
    B = np.empty((L, p))
    oi = np.empty(L, dtype=np.int32)
    ii = np.empty(L, dtype=np.int64)
    cv = np.empty(L, dtype=np.uint8)
    rc = lib().orc_logistic_path(_ptr(X), _ptr(y01), n, p, p, _ptr(lambdas), L, eps, tol_in,
                                 maxit_in, tol_out, outer_maxit, power_iters, inflate, _ptr(B),
                                 _ptr(oi), _ptr(ii), _ptr(cv), nthreads or _nthreads(n))
    if rc != 0:
        raise ValueError("oracle logistic_path: y must be 0/1")
    return B, oi, ii, cv.astype(bool)


# ---------------------------------------------------------------- composed fit (§8(a) a6-a10)
def fit_from_gram(G_raw, c_raw, n, penalties, nlambda=100, ratio=1e-3, d=None, tol=1e-11,
                  maxit=100000, w=None, group=None, ngroups=0, grp_w=None, power_iters=200,
                  inflate=5e-3, lambda_max_override=None):
    """a6 normalize (/n, R#1) -> a7 d (rule R#5, or the d given) -> a8 grid per family (R#14-16)
    -> a9 path per penalty. penalties: list of (family, gamma, alpha). Returns dict."""
    Gn = np.asarray(G_raw, dtype=np.float64) / n
    cn = np.asarray(c_raw, dtype=np.float64) / n
    if d is None:
        d = power_rule(Gn, power_iters, inflate)[0]
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
