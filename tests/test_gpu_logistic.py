"""GPU parity for the proximal-Newton logistic path (a4 + a6-a9, oem_fit_logistic) against the
oracle's O7: per-lambda max |beta| difference <= 1e-8 and logistic KKT on the GPU
solution (R#23-27)."""
import numpy as np
import pytest

import datagen as dg
import oracle as orc
from datagen.configs import CONFIGS
from gpu_util import device_rows

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")


@pytest.fixture(scope="module")
def ctx():
    from paper_1801_09661_b200 import Context
    c = Context(0)
    yield c
    c.close()


@pytest.mark.parametrize("n,p,L", [(4000, 20, 12), (20_011, 200, 8), (6_001, 500, 4)])
def test_logistic_path_parity(ctx, n, p, L):
    from paper_1801_09661_b200 import oem_fit_logistic
    spec = CONFIGS["cfg5"].spec.replace(n=n, p=p, nnz=min(20, p // 2))
    bt = dg.beta(spec)
    Xd, yd = device_rows(spec, bt)
    X, y = dg.rows_host(spec, bt)
    fit = oem_fit_logistic(ctx, Xd, yd, ("lasso", 0.0, 1.0), nlambda=L)
    lam = fit.lam.cpu().numpy()
    _, cw0, _ = orc.gram_weighted(X, y, np.zeros(p))
    lmax = np.max(np.abs(cw0 / n))
    assert abs(lam[0] - lmax) <= 1e-13 * lmax
    assert np.allclose(lam, orc.lambda_grid(lmax, L), rtol=1e-13, atol=0)
    B, oi, ii, cv = orc.logistic_path(X, y, lam)
    Bg = fit.beta.cpu().numpy()
    assert np.max(np.abs(Bg - B)) <= 1e-8
    assert all(fit.conv) and cv.all()
    assert np.max(np.abs(np.array(fit.outer_iters) - oi)) <= 1
    assert not Bg[0].any()  # lambda_max: null model
    for b, l in zip(Bg, lam):  # lasso-logistic KKT
        mu = 1 / (1 + np.exp(-(X @ b)))
        g = X.T @ (y - mu) / n
        nz = b != 0
        assert np.all(np.abs(g[~nz]) <= l + 1e-7)
        assert np.all(np.abs(g[nz] - l * np.sign(b[nz])) <= 1e-7)


def test_logistic_lambda0_newton(ctx):
    from paper_1801_09661_b200 import oem_fit_logistic
    spec = CONFIGS["cfg5"].spec.replace(n=3000, p=5, nnz=3)
    bt = dg.beta(spec)
    X, y = dg.rows_host(spec, bt)
    Xp = np.zeros((X.shape[0], 6))  # row pitch must be even (16-byte TMA strides)
    Xp[:, :5] = X
    fit = oem_fit_logistic(ctx, torch.from_numpy(Xp).cuda()[:, :5], torch.from_numpy(y).cuda(), lambdas=[0.0])
    b = np.zeros(5)
    for _ in range(40):
        mu = 1 / (1 + np.exp(-(X @ b)))
        b = b + np.linalg.solve((X * (mu * (1 - mu))[:, None]).T @ X, X.T @ (y - mu))
    assert np.max(np.abs(fit.beta[0].cpu().numpy() - b)) < 1e-8


# ---------------------------------------------------------------- f1: Hessian upper bound (w = 1/4)
@pytest.mark.parametrize("n,p", [(20_011, 5), (9_000, 64), (9_001, 65), (30_000, 200), (4_000, 257)])
def test_logit_grad_parity(ctx, n, p):
    from paper_1801_09661_b200 import oem_logit_grad
    spec = CONFIGS["cfg5"].spec.replace(n=n, p=p, nnz=min(20, p))
    bt = dg.beta(spec)
    Xd, yd = device_rows(spec, bt)
    X, y = dg.rows_host(spec, bt)
    beta = 0.6 * bt + 0.01 * np.cos(np.arange(p))
    g, ll = oem_logit_grad(ctx, Xd, yd, torch.from_numpy(beta).cuda())
    go, llo = orc.logit_grad(X, y, beta)
    mu = 1 / (1 + np.exp(-(X @ beta)))
    cond = np.abs(X).T @ np.abs(y - mu)     # condition of each sum
    assert np.max(np.abs(g.cpu().numpy() - go) / cond) <= 1e-12
    assert abs(float(ll) - llo) <= 1e-12 * np.sum(np.abs(y * (X @ beta)) + np.logaddexp(0, X @ beta))


def test_logistic_upper_bound_path(ctx):
    """f1 path (R#27) against the oracle's upper-bound path and the exact-Hessian
    path: all three minimise the same convex objective, so they agree at convergence."""
    from paper_1801_09661_b200 import oem_fit_logistic
    spec = CONFIGS["cfg5"].spec.replace(n=12_000, p=30, nnz=8)
    bt = dg.beta(spec)
    Xd, yd = device_rows(spec, bt)
    X, y = dg.rows_host(spec, bt)
    fu = oem_fit_logistic(ctx, Xd, yd, nlambda=8, hessian_upper_bound=True, outer_maxit=1000)
    fe = oem_fit_logistic(ctx, Xd, yd, nlambda=8)
    lam = fu.lam.cpu().numpy()
    # the same lambda_max from two kernels' sums of x_ij (y_i - 1/2) (gradient pass vs weighted
    # pass at beta = 0): equal up to their rounding
    assert np.allclose(lam, fe.lam.cpu().numpy(), rtol=1e-14, atol=0)
    Bo, oi, ii, cv = orc.logistic_path_ub(X, y, lam)
    Bu = fu.beta.cpu().numpy()
    assert all(fu.conv) and cv.all()
    assert np.max(np.abs(Bu - Bo)) <= 1e-8
    assert np.max(np.abs(Bu - fe.beta.cpu().numpy())) <= 1e-7
    assert np.max(np.abs(np.array(fu.outer_iters) - oi)) <= 2


@pytest.mark.parametrize("pen,p,grouped", [
    (("enet", 0.0, 0.5), 40, False),
    (("mcp", 3.0, 1.0), 40, False),
    (("scad", 3.7, 1.0), 40, False),
    (("grp_lasso", 0.0, 1.0), 100, True),
    (("grp_mcp", 3.0, 1.0), 100, True),
    (("grp_scad", 3.7, 1.0), 100, True),
])
def test_logistic_every_family(ctx, pen, p, grouped):
    """Proximal-Newton OEM with every Table 1 family (§6.3 P:L1143-1148 fits MCP
    with gamma = 3 and group penalties with contiguous groups of 25 to logistic models), against
    the oracle's O7 with the same family, groups and lambda grid: lambda_max of the working
    statistic at beta = 0 (R#14), every beta at 1e-8, converged flags and outer step counts."""
    from paper_1801_09661_b200 import oem_fit_logistic
    n, L = 6000, 10
    spec = CONFIGS["cfg5"].spec.replace(n=n, p=p, nnz=min(10, p))
    bt = dg.beta(spec)
    Xd, yd = device_rows(spec, bt)
    X, y = dg.rows_host(spec, bt)
    grp = (np.arange(p) // 25).astype(np.int32) if grouped else None
    fam, gamma, alpha = pen
    fit = oem_fit_logistic(ctx, Xd, yd, pen, nlambda=L, group=grp)
    lam = fit.lam.cpu().numpy()
    _, cw0, _ = orc.gram_weighted(X, y, np.zeros(p))
    lmax = orc.lambda_max(fam, cw0 / n, group=grp, alpha=alpha)
    assert abs(lam[0] - lmax) <= 1e-13 * lmax
    assert np.allclose(lam, orc.lambda_grid(lmax, L), rtol=1e-13, atol=0)
    B, oi, ii, cv = orc.logistic_path(X, y, lam, family=fam, gamma=gamma, alpha=alpha, group=grp)
    Bg = fit.beta.cpu().numpy()
    assert np.max(np.abs(Bg - B)) <= 1e-8, np.max(np.abs(Bg - B))
    assert np.array_equal(np.array(fit.conv), cv)
    assert np.max(np.abs(np.array(fit.outer_iters) - oi)) <= 1
    assert not Bg[0].any()  # lambda_max: null model


def test_logistic_upper_bound_groups(ctx):
    """f1 upper-bound mode with the group lasso and group MCP ('For the MCP and
    group lasso, oem() with the Hessian upper-bound option is the fastest'), against the oracle's
    upper-bound path with the same groups."""
    from paper_1801_09661_b200 import oem_fit_logistic
    n, p, L = 8000, 100, 6
    spec = CONFIGS["cfg5"].spec.replace(n=n, p=p, nnz=10)
    bt = dg.beta(spec)
    Xd, yd = device_rows(spec, bt)
    X, y = dg.rows_host(spec, bt)
    grp = (np.arange(p) // 25).astype(np.int32)
    for pen in (("grp_lasso", 0.0, 1.0), ("grp_mcp", 3.0, 1.0)):
        fit = oem_fit_logistic(ctx, Xd, yd, pen, nlambda=L, group=grp, hessian_upper_bound=True,
                               outer_maxit=1000)
        lam = fit.lam.cpu().numpy()
        Bo, oi, ii, cv = orc.logistic_path_ub(X, y, lam, family=pen[0], gamma=pen[1], group=grp)
        assert all(fit.conv) and cv.all()
        assert np.max(np.abs(fit.beta.cpu().numpy() - Bo)) <= 1e-8, pen


def test_logistic_full_size_cfg5(ctx):
    """cfg5 at full size (n = 5e6, p = 200, 8 GB resident), in bench.py's launch configuration
    (exact-Hessian proximal Newton, weighted Gram recomputed each outer step), on an explicit
    grid of the first three lambda of the benched 50-point grid, against the oracle's O7 over all
    5e6 rows (host generator): every beta at 1e-8 and equal converged flags / outer step counts."""
    from paper_1801_09661_b200 import oem_fit_logistic
    cfg = CONFIGS["cfg5"]
    bt = dg.beta(cfg.spec)
    Xd, yd = device_rows(cfg.spec, bt)
    full = oem_fit_logistic(ctx, Xd, yd, cfg.penalties[0], nlambda=cfg.nlambda)
    lam = full.lam.cpu().numpy()[:3]
    fit = oem_fit_logistic(ctx, Xd, yd, cfg.penalties[0], lambdas=lam)
    Bg = fit.beta.cpu().numpy()
    assert np.array_equal(Bg, full.beta.cpu().numpy()[:3])  # explicit grid == the benched run's start
    del Xd, yd
    torch.cuda.empty_cache()
    X, y = dg.rows_host(cfg.spec, bt)
    _, cw0, _ = orc.gram_weighted(X, y, np.zeros(cfg.p))
    lmax = np.max(np.abs(cw0 / cfg.n))
    assert abs(lam[0] - lmax) <= 1e-13 * lmax
    B, oi, ii, cv = orc.logistic_path(X, y, lam)
    assert np.max(np.abs(Bg - B)) <= 1e-8, np.max(np.abs(Bg - B))
    assert np.array_equal(np.array(fit.conv), cv) and cv.all()
    assert np.max(np.abs(np.array(fit.outer_iters) - oi)) <= 1


def test_logistic_group_lasso_p250_exact_hessian(ctx):
    """The paper's §6.3 shape for grouped logistic regression (p up to 500, groups
    of 25, exact-Hessian proximal Newton): p = 250 runs the two-panel weighted pass every outer
    step; against O7 with the same groups."""
    from paper_1801_09661_b200 import oem_fit_logistic
    n, p, L = 5000, 250, 5
    spec = CONFIGS["cfg5"].spec.replace(n=n, p=p, nnz=10)
    bt = dg.beta(spec)
    Xd, yd = device_rows(spec, bt)
    X, y = dg.rows_host(spec, bt)
    grp = (np.arange(p) // 25).astype(np.int32)
    fit = oem_fit_logistic(ctx, Xd, yd, ("grp_lasso", 0.0, 1.0), nlambda=L, group=grp)
    lam = fit.lam.cpu().numpy()
    B, oi, ii, cv = orc.logistic_path(X, y, lam, family="grp_lasso", group=grp)
    assert np.max(np.abs(fit.beta.cpu().numpy() - B)) <= 1e-8
    assert np.array_equal(np.array(fit.conv), cv)


def test_logit_grad_without_loglik(ctx):
    """loglik=False (the upper-bound fit's call) gives the same gradient bit for bit."""
    from paper_1801_09661_b200 import oem_logit_grad
    spec = CONFIGS["cfg5"].spec.replace(n=7_001, p=90, nnz=9)
    bt = dg.beta(spec)
    Xd, yd = device_rows(spec, bt)
    beta = torch.from_numpy(0.5 * bt).cuda()
    g1, ll = oem_logit_grad(ctx, Xd, yd, beta)
    g2, none = oem_logit_grad(ctx, Xd, yd, beta, loglik=False)
    assert none is None and ll is not None and torch.equal(g1, g2)
