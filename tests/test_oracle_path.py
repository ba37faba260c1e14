"""Pins for oracle O5-O7 (lambda grid, OEM path, logistic proximal Newton).

Convex families (lasso, EN, group lasso) have a unique minimiser when G is positive definite,
so OEM's fixed point is pinned by the plain definition: OLS at lambda = 0 (normal equations),
ridge closed form, KKT conditions, exhaustive sign-pattern / region enumeration on tiny p and
an independent cyclic coordinate descent. MCP/SCAD are pinned on convex instances (gamma large
enough that 0.5 b^T G b + P is convex) by region enumeration."""
import itertools
from fractions import Fraction

import numpy as np
import pytest

import datagen as dg
import oracle as orc
from datagen.configs import CONFIGS, groups_of


def small_problem(seed, n, p, rho=0.3):
    rng = np.random.default_rng(seed)
    S = rho ** np.abs(np.subtract.outer(np.arange(p), np.arange(p)))
    X = rng.standard_normal((n, p)) @ np.linalg.cholesky(S).T
    beta = np.zeros(p)
    beta[: min(3, p)] = [1.5, -1.0, 0.5][: min(3, p)]
    y = X @ beta + rng.standard_normal(n)
    G, c, _ = orc.gram(X, y)
    return G / n, c / n


# ------------------------------------------------------------------ lambda_max / grid
def test_lambda_max_examples(golden):
    for ex in golden["lambda_max"]:
        lm = orc.lambda_max(ex["family"], np.array(ex["xty"]), group=ex.get("group"),
                            grp_w=ex.get("grp_w"))
        assert lm == ex["lambda_max"]


@pytest.mark.parametrize("family,alpha", [("lasso", 1.0), ("enet", 0.5), ("mcp", 1.0),
                                          ("scad", 1.0), ("grp_lasso", 1.0)])
def test_lambda_max_is_smallest_null_fixed_point(family, alpha):
    """beta = 0 is a fixed point at lambda_max but not at lambda_max (1 - 1e-3)."""
    G, c = small_problem(12, 400, 6)
    grp = np.array([0, 0, 1, 1, 2, 2], dtype=np.int32) if family.startswith("grp") else None
    d = orc.d_rule(G)[0]
    lm = orc.lambda_max(family, c, group=grp, alpha=alpha)
    b, it, _ = orc.oem_path(G, c, d, family, [lm], gamma=3.7, alpha=alpha, group=grp, maxit=1)
    assert not b.any()
    b, it, _ = orc.oem_path(G, c, d, family, [lm * (1 - 1e-3)], gamma=3.7, alpha=alpha, group=grp,
                            maxit=1)
    assert b.any()


def test_lambda_grid_shape():
    lam = orc.lambda_grid(2.0, 100, 1e-3)
    assert lam[0] == 2.0 and abs(lam[-1] - 2e-3) < 1e-15
    assert np.allclose(np.diff(np.log(lam)), np.log(1e-3) / 99, rtol=1e-12)
    assert list(orc.lambda_grid(3.0, 1, 1e-3)) == [3.0]


# ------------------------------------------------------------------ unpenalized / closed forms
def test_lambda_zero_is_ols():
    """lambda = 0 -> the normal-equation solution (north star)."""
    G, c = small_problem(13, 500, 8)
    d = orc.d_rule(G)[0]
    for fam in ("lasso", "mcp", "scad", "enet"):
        b, it, cv = orc.oem_path(G, c, d, fam, [0.0], gamma=3.0, alpha=0.5, tol=1e-14, maxit=200000)
        assert cv[0]
        assert np.max(np.abs(b[0] - np.linalg.solve(G, c))) < 1e-11


def test_orthogonal_design_one_step():
    """G = I, d = 1: one EM step gives beta = Theta(c) exactly."""
    rng = np.random.default_rng(14)
    c = rng.uniform(-3, 3, 6)
    G = np.eye(6)
    grp = np.array([0, 0, 0, 1, 1, 1], dtype=np.int32)
    for fam, op in (("lasso", lambda u: orc.soft(u, 0.7, 1.0)),
                    ("mcp", lambda u: orc.mcp(u, 0.7, 3.0, 1.0)),
                    ("scad", lambda u: orc.scad(u, 0.7, 3.7, 1.0))):
        gamma = 3.0 if fam == "mcp" else 3.7
        b, it, cv = orc.oem_path(G, c, 1.0, fam, [0.7], gamma=gamma, maxit=1)
        assert np.array_equal(b[0], [op(u) for u in c])
        b2, it2, cv2 = orc.oem_path(G, c, 1.0, fam, [0.7], gamma=gamma)
        # the second step recomputes u = (c + b) - b, equal to c up to one rounding
        assert np.max(np.abs(b2[0] - b[0])) <= 4e-16 * np.max(np.abs(c)) and it2[0] == 2 and cv2[0]
    b, _, _ = orc.oem_path(G, c, 1.0, "grp_lasso", [0.7], group=grp, maxit=1)
    w = np.sqrt(3.0)
    assert np.allclose(b[0], np.concatenate([orc.grp_lasso(c[:3], 0.7 * w, 1.0),
                                             orc.grp_lasso(c[3:], 0.7 * w, 1.0)]), rtol=0, atol=0)


def test_enet_alpha0_is_ridge():
    G, c = small_problem(15, 300, 7)
    d = orc.d_rule(G)[0]
    for lam in (0.01, 0.3, 2.0):
        b, _, cv = orc.oem_path(G, c, d, "enet", [lam], alpha=0.0, tol=1e-14)
        assert cv[0]
        assert np.max(np.abs(b[0] - np.linalg.solve(G + lam * np.eye(7), c))) < 1e-11


# ------------------------------------------------------------------ KKT along whole paths
def test_lasso_kkt_every_lambda_cfg1():
    cfg = CONFIGS["cfg1"]
    bt = dg.beta(cfg.spec, cfg.explicit_beta)
    X, y = dg.rows_host(cfg.spec, bt)
    G, c, _ = orc.gram(X, y)
    fit = orc.fit_from_gram(G, c, cfg.n, cfg.penalties, cfg.nlambda, tol=1e-11)
    Gn, cn = G / cfg.n, c / cfg.n
    gersh = np.abs(Gn).sum(1).max()
    B, lam = fit["beta"][0], fit["lambda"][0]
    assert fit["conv"][0].all()
    slack = 2 * gersh * 1e-11 * 10 + 1e-12
    for b, l in zip(B, lam):
        r = cn - Gn @ b
        nz = b != 0
        assert np.all(np.abs(r[~nz]) <= l + slack)
        assert np.all(np.abs(r[nz] - l * np.sign(b[nz])) <= slack)
    assert not B[0].any()                       # lambda_max nulls everything
    assert np.count_nonzero(B[-1]) >= 5         # the true support is recovered at small lambda


def test_group_lasso_kkt():
    G, c = small_problem(16, 600, 9)
    grp = np.repeat(np.arange(3), 3).astype(np.int32)
    d = orc.d_rule(G)[0]
    lm = orc.lambda_max("grp_lasso", c, group=grp)
    lams = orc.lambda_grid(lm, 20, 1e-2)
    B, _, cv = orc.oem_path(G, c, d, "grp_lasso", lams, group=grp, tol=1e-13)
    assert cv.all()
    for b, l in zip(B, lams):
        r = c - G @ b
        for g in range(3):
            s = slice(3 * g, 3 * g + 3)
            lw = l * np.sqrt(3)
            if not b[s].any():
                assert np.linalg.norm(r[s]) <= lw + 1e-10
            else:
                assert np.max(np.abs(r[s] - lw * b[s] / np.linalg.norm(b[s]))) < 1e-10


# ------------------------------------------------------------------ brute force on tiny p
def lasso_enumerate(G, c, lam):
    """Exact lasso minimiser by enumerating the 3^p sign patterns (each a linear solve)."""
    p = c.size
    best, bestb = np.inf, None
    for pat in itertools.product((-1, 0, 1), repeat=p):
        s = np.array(pat, dtype=float)
        A = np.nonzero(s)[0]
        b = np.zeros(p)
        if A.size:
            b[A] = np.linalg.solve(G[np.ix_(A, A)], c[A] - lam * s[A])
            if np.any(np.sign(b[A]) != s[A]):
                continue
        f = 0.5 * b @ G @ b - c @ b + lam * np.abs(b).sum()
        if f < best:
            best, bestb = f, b
    return bestb


def mcp_regions_enumerate(G, c, lam, gamma, kind):
    """Exact minimiser of 0.5 b'Gb - c'b + sum P(b_j) for MCP/SCAD on a convex instance by
    enumerating per-coordinate regions; on each region P is quadratic so the stationary point
    is a linear solve, kept if feasible."""
    p = c.size
    if kind == "mcp":  # regions: 0, (0, g lam] +/-, > g lam +/-
        regions = [(0, 0, 0.0, 0.0)]
        regions += [(s, 1, -1.0 / gamma, s * lam) for s in (1, -1)]   # P' = lam s - b/g
        regions += [(s, 2, 0.0, 0.0) for s in (1, -1)]
        bounds = {1: (0, gamma * lam), 2: (gamma * lam, np.inf)}
    else:
        regions = [(0, 0, 0.0, 0.0)]
        regions += [(s, 1, 0.0, s * lam) for s in (1, -1)]            # |b| <= lam: P' = lam s
        regions += [(s, 2, -1.0 / (gamma - 1), s * gamma * lam / (gamma - 1)) for s in (1, -1)]
        regions += [(s, 3, 0.0, 0.0) for s in (1, -1)]
        bounds = {1: (0, lam), 2: (lam, gamma * lam), 3: (gamma * lam, np.inf)}
    pen = (lambda b: sum(lam * abs(x) - x * x / (2 * gamma) if abs(x) <= gamma * lam else gamma * lam * lam / 2
                         for x in b)) if kind == "mcp" else (
        lambda b: sum(lam * abs(x) if abs(x) <= lam else (
            -(x * x - 2 * gamma * lam * abs(x) + lam * lam) / (2 * (gamma - 1)) if abs(x) <= gamma * lam
            else (gamma + 1) * lam * lam / 2) for x in b))
    best, bestb = np.inf, None
    for combo in itertools.product(regions, repeat=p):
        H = G.copy()
        rhs = c.copy()
        A = []
        for j, (s, r, curv, lin) in enumerate(combo):
            if r == 0:
                continue
            A.append(j)
            H[j, j] += curv
            rhs[j] -= lin
        b = np.zeros(p)
        if A:
            try:
                b[A] = np.linalg.solve(H[np.ix_(A, A)], rhs[A])
            except np.linalg.LinAlgError:
                continue
        ok = True
        for j, (s, r, _, _) in enumerate(combo):
            if r == 0:
                continue
            lo, hi = bounds[r]
            if not (np.sign(b[j]) == s and lo - 1e-14 <= abs(b[j]) <= hi + 1e-14):
                ok = False
        if not ok:
            continue
        f = 0.5 * b @ G @ b - c @ b + pen(b)
        if f < best:
            best, bestb = f, b
    return bestb


def test_lasso_brute_force_tiny_p():
    for seed in range(5):
        G, c = small_problem(100 + seed, 200, 3, rho=0.5)
        d = orc.d_rule(G)[0]
        for frac in (0.9, 0.5, 0.1, 0.01):
            lam = frac * orc.lambda_max("lasso", c)
            b, _, cv = orc.oem_path(G, c, d, "lasso", [lam], tol=1e-14)
            assert cv[0]
            assert np.max(np.abs(b[0] - lasso_enumerate(G, c, lam))) < 1e-11


@pytest.mark.parametrize("kind,gamma", [("mcp", 6.0), ("scad", 7.0)])
def test_nonconvex_brute_force_on_convex_instances(kind, gamma):
    """lambda_min(G) > 1/gamma (MCP) or > 1/(gamma-1) (SCAD): unique minimiser, so the OEM
    fixed point must equal it (R#30)."""
    for seed in range(4):
        G, c = small_problem(200 + seed, 300, 3, rho=0.2)
        lmin = np.linalg.eigvalsh(G)[0]
        assert lmin > (1 / gamma if kind == "mcp" else 1 / (gamma - 1))
        d = orc.d_rule(G)[0]
        for frac in (0.8, 0.4, 0.1):
            lam = frac * orc.lambda_max(kind, c)
            b, _, cv = orc.oem_path(G, c, d, kind, [lam], gamma=gamma, tol=1e-14)
            assert cv[0]
            assert np.max(np.abs(b[0] - mcp_regions_enumerate(G, c, lam, gamma, kind))) < 1e-10


def test_coordinate_descent_agreement():
    """An independent solver (cyclic coordinate descent, Friedman et al. 2010) on EN."""
    G, c = small_problem(17, 400, 10, rho=0.5)
    d = orc.d_rule(G)[0]
    lam, alpha = 0.05, 0.5
    b_oem, _, _ = orc.oem_path(G, c, d, "enet", [lam], alpha=alpha, tol=1e-14)
    b = np.zeros(10)
    for _ in range(5000):
        for j in range(10):
            r = c[j] - G[j] @ b + G[j, j] * b[j]
            b[j] = np.sign(r) * max(abs(r) - alpha * lam, 0) / (G[j, j] + (1 - alpha) * lam)
    assert np.max(np.abs(b_oem[0] - b)) < 1e-11


# ------------------------------------------------------------------ algorithm properties
@pytest.mark.parametrize("family", ["lasso", "mcp", "scad", "enet", "grp_lasso", "grp_mcp", "grp_scad", "sgl"])
def test_descent_each_iteration(family):
    """EM/MM: the objective never increases across OEM iterations when d >= lambda_1.
    For the sparse group lasso this also checks the exact composition (R#11) is the M-step."""
    G, c = small_problem(18, 500, 6, rho=0.5)
    grp = np.array([0, 0, 1, 1, 2, 2], dtype=np.int32) if family.startswith("grp") or family == "sgl" else None
    d = orc.d_rule(G)[0]
    lam = 0.2 * orc.lambda_max(family, c, group=grp, alpha=0.5)
    b = np.zeros(6)
    f = orc.objective(G, c, b, family, lam, 3.0, 0.5, group=grp)
    for _ in range(60):
        nb, _, _ = orc.oem_path(G, c, d, family, [lam], gamma=3.0, alpha=0.5, group=grp, maxit=1,
                                beta_init=b)
        f2 = orc.objective(G, c, nb[0], family, lam, 3.0, 0.5, group=grp)
        assert f2 <= f + 1e-14
        b, f = nb[0], f2


def test_convex_paths_independent_of_d():
    """OEM converges for every d >= lambda_1; convex fixed points do not depend on d."""
    G, c = small_problem(19, 500, 12, rho=0.5)
    lam1 = np.linalg.eigvalsh(G)[-1]
    lams = orc.lambda_grid(orc.lambda_max("lasso", c), 30)
    b1, it1, _ = orc.oem_path(G, c, lam1 * (1 + 1e-9), "lasso", lams)
    b2, it2, _ = orc.oem_path(G, c, 1.5 * lam1, "lasso", lams)
    assert np.max(np.abs(b1 - b2)) < 1e-8
    assert it1.sum() < it2.sum()  # d = lambda_1 converges fastest


def test_multi_penalty_grid_and_group_ids():
    cfg = CONFIGS["cfg4"]
    grp = groups_of(cfg)
    assert grp[0] == 0 and grp[-1] == 99 and np.all(np.bincount(grp) == 10)


def test_invalid_nonconvex_parameters():
    G, c = small_problem(20, 100, 3)
    with pytest.raises(ValueError):
        orc.oem_path(G, c, 1.0, "mcp", [0.1], gamma=0.9)   # gamma d <= 1 (R#8)
    with pytest.raises(ValueError):
        orc.oem_path(G, c, 1.0, "scad", [0.1], gamma=1.5)


# ------------------------------------------------------------------ logistic
def newton_mle(X, y, iters=50):
    b = np.zeros(X.shape[1])
    for _ in range(iters):
        mu = 1 / (1 + np.exp(-(X @ b)))
        H = (X * (mu * (1 - mu))[:, None]).T @ X
        b = b + np.linalg.solve(H, X.T @ (y - mu))
    return b


def logistic_data(seed, n, p):
    spec = dg.make_spec(seed, n, p, dg.DG_AR1, rho=0.5, response=dg.DG_LOGISTIC,
                        beta_kind=dg.DG_BETA_UNIFORM, nnz=3, beta_lo=-1.0, beta_hi=1.0)
    bt = dg.beta(spec)
    return dg.rows_host(spec, bt)


def test_logistic_lambda0_is_newton_mle():
    X, y = logistic_data(21, 2000, 4)
    B, oi, ii, cv = orc.logistic_path(X, y, [0.0])
    assert cv[0]
    assert np.max(np.abs(B[0] - newton_mle(X, y))) < 1e-8


def test_logistic_kkt_and_null_fixed_point():
    X, y = logistic_data(22, 3000, 8)
    n = X.shape[0]
    _, cw0, _ = orc.gram_weighted(X, y, np.zeros(8))
    lmax = np.max(np.abs(cw0 / n))          # = max |(1/n) sum x (y - 1/2)| (R#14)
    assert abs(lmax - np.max(np.abs(X.T @ (y - 0.5) / n))) < 1e-14
    lams = orc.lambda_grid(lmax, 15, 1e-2)
    B, oi, ii, cv = orc.logistic_path(X, y, lams)
    assert cv.all() and not B[0].any()
    for b, l in zip(B, lams):
        mu = 1 / (1 + np.exp(-(X @ b)))
        gr = X.T @ (y - mu) / n
        nz = b != 0
        assert np.all(np.abs(gr[~nz]) <= l + 1e-7)
        assert np.all(np.abs(gr[nz] - l * np.sign(b[nz])) <= 1e-7)
        assert np.all(mu * (1 - mu) <= 0.25)


def test_logistic_group_lasso_kkt():
    """O7 with the group lasso (P:L1146-1148 fits group penalties to logistic models): at every
    lambda the logistic group-lasso subgradient conditions hold, ||(1/n) X_g^T (y - mu)|| <=
    lambda c_g on zero groups and (1/n) X_g^T (y - mu) = lambda c_g b_g / ||b_g|| on the others,
    with c_g = sqrt(|g|) (R#12); beta = 0 at lambda_max = max_g ||c_g|| / c_g (R#14)."""
    X, y = logistic_data(24, 3000, 12)
    n, p = X.shape
    grp = (np.arange(p) // 3).astype(np.int32)
    _, cw0, _ = orc.gram_weighted(X, y, np.zeros(p))
    lmax = orc.lambda_max("grp_lasso", cw0 / n, group=grp)
    lams = orc.lambda_grid(lmax, 10, 1e-2)
    B, oi, ii, cv = orc.logistic_path(X, y, lams, family="grp_lasso", group=grp)
    assert cv.all() and not B[0].any()
    for b, l in zip(B, lams):
        gr = X.T @ (y - 1 / (1 + np.exp(-(X @ b)))) / n
        for g in range(p // 3):
            idx = grp == g
            nb = np.linalg.norm(b[idx])
            if nb == 0:
                assert np.linalg.norm(gr[idx]) <= l * np.sqrt(3) * (1 + 1e-6) + 1e-9
            else:
                assert np.max(np.abs(gr[idx] - l * np.sqrt(3) * b[idx] / nb)) <= 1e-7


def test_logistic_enet_kkt_and_mcp_scad_limits():
    """O7 with the elastic net: (1/n) X^T (y - mu) - lambda (1 - alpha) b = lambda alpha sign(b) on
    the support, |.| <= lambda alpha off it. MCP and SCAD: below their flat zone (|b_j| > gamma
    lambda, resp. > gamma lambda for SCAD) the penalty's derivative vanishes, so at a tiny lambda
    every coefficient is unpenalised and the path point is the Newton-Raphson MLE."""
    X, y = logistic_data(25, 2500, 5)
    n = X.shape[0]
    lams = [0.02, 0.005]
    B, oi, ii, cv = orc.logistic_path(X, y, lams, family="enet", alpha=0.5)
    assert cv.all()
    for b, l in zip(B, lams):
        gr = X.T @ (y - 1 / (1 + np.exp(-(X @ b)))) / n
        nz = b != 0
        assert np.all(np.abs(gr[~nz]) <= 0.5 * l + 1e-7)
        assert np.all(np.abs(gr[nz] - 0.5 * l * b[nz] - 0.5 * l * np.sign(b[nz])) <= 1e-7)
    mle = newton_mle(X, y)
    for fam, gam in (("mcp", 3.0), ("scad", 3.7)):
        lam = 0.1 * np.min(np.abs(mle)) / gam
        B, oi, ii, cv = orc.logistic_path(X, y, [lam], family=fam, gamma=gam, tol_out=1e-12)
        assert cv.all() and np.max(np.abs(B[0] - mle)) <= 1e-8, fam


# ---------------------------------------------------------------- f1 upper-bound logistic oracle
def test_logit_grad_zero_beta_exact():
    """beta = 0: mu = 1/2, g = X^T (y - 1/2) exactly on integer X (all partial sums are exact)."""
    rng = np.random.default_rng(21)
    X = rng.integers(-6, 7, size=(401, 7)).astype(float)
    y = (rng.random(401) < 0.4).astype(float)
    g, ll = orc.logit_grad(X, y, np.zeros(7))
    Xo = X.astype(int).astype(object)
    exact = [sum(Fraction(int(Xo[i, j])) * (Fraction(int(y[i])) - Fraction(1, 2)) for i in range(401)) for j in range(7)]
    assert np.array_equal(g, np.array([float(v) for v in exact]))
    assert abs(ll - 401 * (-np.log(2.0))) <= 1e-12 * 401


def test_logistic_ub_matches_exact_newton_fixed_point():
    """The upper-bound MM iteration and exact proximal Newton minimise the same convex
    objective (R#23-24), so their lasso paths agree at convergence; and lambda = 0 reproduces
    the unpenalised MLE from Newton-Raphson (numpy)."""
    rng = np.random.default_rng(22)
    n, p = 600, 4
    X = rng.standard_normal((n, p))
    bt = np.array([1.0, -0.5, 0.0, 0.25])
    y = (rng.random(n) < 1 / (1 + np.exp(-X @ bt))).astype(float)
    lam = [0.05, 0.01, 0.0]
    Bu, oi, ii, cv = orc.logistic_path_ub(X, y, lam, tol_out=1e-12)
    Be, _, _, cve = orc.logistic_path(X, y, lam, tol_out=1e-12)
    assert cv.all() and cve.all()
    assert np.max(np.abs(Bu - Be)) <= 1e-8
    b = np.zeros(p)
    for _ in range(50):
        mu = 1 / (1 + np.exp(-(X @ b)))
        b = b + np.linalg.solve((X * (mu * (1 - mu))[:, None]).T @ X, X.T @ (y - mu))
    assert np.max(np.abs(Bu[-1] - b)) <= 1e-8
    # the MM step never increases the penalised negative log-likelihood (descent)
    assert (oi >= 1).all()


def test_sgl_kkt_and_limits_on_path():
    """Sparse group lasso path (tau = 0.4): at the fixed point the subgradient conditions of
    0.5 b^T G b - c^T b + lam (1-tau) sum c_k ||b_g|| + lam tau sum |b_j| hold per group; tau = 0
    reproduces the group-lasso path and tau = 1 the lasso path."""
    G, c = small_problem(23, 800, 9, rho=0.4)
    grp = np.repeat(np.arange(3), 3).astype(np.int32)
    d = orc.d_rule(G)[0]
    tau = 0.4
    lams = orc.lambda_grid(orc.lambda_max("sgl", c, group=grp, alpha=tau), 12)
    B, _, cv = orc.oem_path(G, c, d, "sgl", lams, alpha=tau, group=grp, tol=1e-14)
    assert cv.all()
    ck = np.sqrt(3.0)
    for b, lam in zip(B, lams):
        r = c - G @ b                                   # = subgradient of the penalty
        for g in range(3):
            idx = grp == g
            bg, rg = b[idx], r[idx]
            if not bg.any():
                # 0 in the subdifferential: exists s in [-1,1]^m with ||rg - lam tau s|| <= lam (1-tau) ck
                z = np.sign(rg) * np.maximum(np.abs(rg) - lam * tau, 0)
                assert np.linalg.norm(z) <= lam * (1 - tau) * ck * (1 + 1e-9) + 1e-12
            else:
                nz = bg != 0
                s = np.where(nz, np.sign(bg), 0.0)
                res = rg - lam * tau * s - lam * (1 - tau) * ck * bg / np.linalg.norm(bg)
                assert np.all(np.abs(res[nz]) <= 1e-9)
                assert np.all(np.abs(rg[~nz] - lam * (1 - tau) * ck * bg[~nz] / np.linalg.norm(bg)) <= lam * tau + 1e-9)
    lg = orc.lambda_grid(orc.lambda_max("grp_lasso", c, group=grp), 8)
    B0, _, _ = orc.oem_path(G, c, d, "sgl", lg, alpha=0.0, group=grp, tol=1e-14)
    Bg, _, _ = orc.oem_path(G, c, d, "grp_lasso", lg, group=grp, tol=1e-14)
    assert np.max(np.abs(B0 - Bg)) <= 1e-12
    ll = orc.lambda_grid(orc.lambda_max("lasso", c), 8)
    B1, _, _ = orc.oem_path(G, c, d, "sgl", ll, alpha=1.0, group=grp, tol=1e-14)
    Bl, _, _ = orc.oem_path(G, c, d, "lasso", ll, tol=1e-14)
    assert np.max(np.abs(B1 - Bl)) <= 1e-12
