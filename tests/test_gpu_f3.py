"""GPU parity for f3: column sums (oem_gram_moments), the fit with intercept and standardization
(centring / scaling of the sufficient statistics in oem_fit_path, R#2-3) against the oracle's
data-transformation route, and compute.loss (oem_path_loss, R#37) against direct residuals."""
import numpy as np
import pytest

import datagen as dg
import oracle as orc
from datagen.configs import CONFIGS

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")


@pytest.fixture(scope="module")
def ctx():
    from paper_1801_09661_b200 import Context
    c = Context(0)
    yield c
    c.close()


def _shifted(n, p, seed):
    """cfg2-shaped rows, then columns shifted and scaled so centring and scaling matter."""
    spec = CONFIGS["cfg2"].spec.replace(n=n, p=p, nnz=min(8, p))
    bt = dg.beta(spec)
    X, y = dg.rows_host(spec, bt)
    rng = np.random.default_rng(seed)
    X = X * rng.uniform(0.3, 4.0, p) + rng.uniform(-3, 3, p)
    y = y + 2.5
    Xp = np.zeros((n, p + (p & 1)))
    Xp[:, :p] = X
    return X, y, torch.from_numpy(Xp).cuda()[:, :p], torch.from_numpy(y).cuda()


@pytest.mark.parametrize("n,p,K,off", [(5000, 7, 1, 0), (20_011, 300, 1, 0), (9_999, 40, 5, 3), (1_000, 513, 3, 11)])
def test_moments_parity(ctx, n, p, K, off):
    from paper_1801_09661_b200 import oem_gram_moments
    rng = np.random.default_rng(n)
    Xi = rng.integers(-9, 10, size=(n, p)).astype(float)   # integer data: sums exact, compare bitwise
    yi = rng.integers(-9, 10, size=n).astype(float)
    Xp = np.zeros((n, p + (p & 1)))
    Xp[:, :p] = Xi
    xs, ys = oem_gram_moments(ctx, torch.from_numpy(Xp).cuda()[:, :p], torch.from_numpy(yi).cuda(), K, off)
    fold = (off + np.arange(n)) % K
    for k in range(K):
        assert np.array_equal(xs[k].cpu().numpy(), Xi[fold == k].sum(axis=0))
        assert float(ys[k]) == yi[fold == k].sum()


@pytest.mark.parametrize("p,std", [(30, True), (30, False), (120, True), (300, True)])
def test_intercept_standardize_parity(ctx, p, std):
    from paper_1801_09661_b200 import oem_fit_path, oem_gram, oem_gram_moments
    n = 8000
    X, y, Xd, yd = _shifted(n, p, p)
    G, c, yy, nn = oem_gram(ctx, Xd, yd)
    xs, ys = oem_gram_moments(ctx, Xd, yd)
    pens = [("lasso", 0.0, 1.0), ("scad", 3.7, 1.0)]
    fit = oem_fit_path(ctx, G, c, [nn], pens, nlambda=15, standardize=std, xsum=xs, ysum=ys)
    d = float(fit.d[0])
    lams = [fit.lam[0, q].cpu().numpy() for q in range(2)]
    ref = orc.fit_transformed(X, y, pens, standardize=std, intercept=True, d=d, lambdas=lams)
    # the grid itself (lambda_max of the centred / scaled statistics, R#14)
    lref = orc.fit_transformed(X, y, pens[:1], nlambda=15, standardize=std, intercept=True, d=d)["lambda"][0]
    assert np.max(np.abs(lams[0] - lref) / lref) <= 1e-11
    for q in range(2):
        Bg = fit.beta[0, q].cpu().numpy()
        assert np.max(np.abs(Bg - ref["beta"][q])) <= 1e-8, np.max(np.abs(Bg - ref["beta"][q]))
        assert np.max(np.abs(fit.intercept[0, q].cpu().numpy() - ref["intercept"][q])) <= 1e-7


def test_intercept_fold_mode(ctx):
    """Fold sums of the moments follow the same total-minus-fold algebra as the Grams."""
    from paper_1801_09661_b200 import oem_fit_path, oem_gram_folds, oem_gram_moments
    n, p, K = 6000, 25, 4
    X, y, Xd, yd = _shifted(n, p, 7)
    Gk, ck, yyk, cnt = oem_gram_folds(ctx, Xd, yd, K)
    xs, ys = oem_gram_moments(ctx, Xd, yd, K)
    pens = [("lasso", 0.0, 1.0)]
    fit = oem_fit_path(ctx, Gk, ck, cnt, pens, nlambda=10, fold_mode=True, standardize=True, xsum=xs, ysum=ys)
    fold = np.arange(n) % K
    for u in (0, 2):
        rows = np.ones(n, bool) if u == 0 else fold != (u - 1)
        ref = orc.fit_transformed(X[rows], y[rows], pens, standardize=True, intercept=True,
                                  d=float(fit.d[u]), lambdas=[fit.lam[u, 0].cpu().numpy()])
        assert np.max(np.abs(fit.beta[u, 0].cpu().numpy() - ref["beta"][0])) <= 1e-8
        assert np.max(np.abs(fit.intercept[u, 0].cpu().numpy() - ref["intercept"][0])) <= 1e-7


def test_path_loss_parity(ctx):
    from paper_1801_09661_b200 import oem_fit_path, oem_gram, oem_path_loss
    spec = CONFIGS["cfg2"].spec.replace(n=12_000, p=60, nnz=8)
    bt = dg.beta(spec)
    X, y = dg.rows_host(spec, bt)
    Xd, yd = torch.from_numpy(X).cuda(), torch.from_numpy(y).cuda()
    G, c, yy, nn = oem_gram(ctx, Xd, yd)
    pens = [("lasso", 0.0, 1.0), ("mcp", 3.0, 1.0)]
    fit = oem_fit_path(ctx, G, c, [nn], pens, nlambda=20)
    loss = oem_path_loss(ctx, G, c, yy, [nn], fit.beta)
    ref = orc.path_loss(X, y, fit.beta.cpu().numpy())
    s = float(np.mean(y * y))
    assert np.max(np.abs(loss.cpu().numpy() - ref)) <= 1e-10 * s
    # at lambda_max (beta = 0) the loss is y^T y / n exactly
    assert float(loss[0, 0, 0]) == float(yy) / nn
