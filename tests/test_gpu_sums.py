"""GPU parity for the Gram pass with a ones column (oem_gram_sums / oem_gram_folds_sums): one pass
over Z = [X | y | 1] gives the a2/a3 statistics plus the f3 column sums X^T 1, 1^T y (R#2-3;
SURVEY §8(c) #3), with no second pass over X.

Integer-valued designs are compared bit for bit with exact integer sums (every partial sum is an
exact integer, so any summation order gives the same bits); shapes cover single-panel and
two-panel plans, p + 1 a multiple of 8 (the ones column then opens a new 8-column block) and not,
ragged row counts, folds with a tail (n mod K != 0) and a row offset. Real-valued designs are
compared with the oracle's Gram (scale-aware 1e-12, R#32), and an intercept fit fed by
the one-pass sums with the oracle's data-transformation route."""
import numpy as np
import pytest

import datagen as dg
import oracle as orc
from datagen.configs import CONFIGS
from gpu_util import scale_err, xty_err

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")


@pytest.fixture(scope="module")
def ctx():
    from paper_1801_09661_b200 import Context
    c = Context(0)
    yield c
    c.close()


def _dev(X):
    """X on the device with an even row pitch (TMA needs 16-byte row strides)."""
    n, p = X.shape
    Xp = np.zeros((n, p + (p & 1)))
    Xp[:, :p] = X
    return torch.from_numpy(Xp).cuda()[:, :p]


def _int_design(seed, n, p):
    rng = np.random.default_rng(seed)
    return rng.integers(-9, 10, size=(n, p)).astype(float), rng.integers(-9, 10, size=n).astype(float)


# p: 7 / 15 / 247 (p + 1 = 0 mod 8: the ones column opens a block; 247 also turns the plan
# two-panel), 30 / 100 (single panel), 300 / 1000 (two-panel)
@pytest.mark.parametrize("n,p", [(4_099, 7), (3_001, 15), (10_007, 30), (20_000, 100), (2_053, 247),
                                 (5_003, 300), (1_031, 1000)])
def test_sums_integer_bit_exact(ctx, n, p):
    from paper_1801_09661_b200 import oem_gram_sums
    X, y = _int_design(n + p, n, p)
    G, c, yy, xs, ys, nt = oem_gram_sums(ctx, _dev(X), torch.from_numpy(y).cuda())
    assert nt == n
    assert np.array_equal(G.cpu().numpy(), X.T @ X)
    assert np.array_equal(c.cpu().numpy(), X.T @ y)
    assert float(yy) == float(y @ y)
    assert np.array_equal(xs.cpu().numpy(), X.sum(axis=0))
    assert float(ys) == float(y.sum())


@pytest.mark.parametrize("n,p,K,off", [(9_999, 40, 5, 3), (4_000, 63, 10, 0), (1_037, 300, 3, 11), (13, 20, 5, 4)])
def test_folds_sums_integer_bit_exact(ctx, n, p, K, off):
    """Folds (off + i) mod K with a tail of n mod K rows (the tail kernel adds the ones column
    too); (13, 20, 5, 4): two full groups and a tail of three rows."""
    from paper_1801_09661_b200 import oem_gram_folds_sums
    X, y = _int_design(n * K + p, n, p)
    Gk, ck, yyk, xs, ys, cnt = oem_gram_folds_sums(ctx, _dev(X), torch.from_numpy(y).cuda(), K, off)
    fold = (off + np.arange(n)) % K
    for k in range(K):
        r = fold == k
        assert cnt[k] == int(r.sum())
        assert np.array_equal(Gk[k].cpu().numpy(), X[r].T @ X[r])
        assert np.array_equal(ck[k].cpu().numpy(), X[r].T @ y[r])
        assert float(yyk[k]) == float(y[r] @ y[r])
        assert np.array_equal(xs[k].cpu().numpy(), X[r].sum(axis=0))
        assert float(ys[k]) == float(y[r].sum())


def test_sums_empty_rows(ctx):
    from paper_1801_09661_b200 import oem_gram_sums
    X = torch.zeros((0, 12), dtype=torch.float64, device="cuda")
    y = torch.zeros(0, dtype=torch.float64, device="cuda")
    G, c, yy, xs, ys, nt = oem_gram_sums(ctx, X, y)
    assert nt == 0 and not G.any() and not c.any() and float(yy) == 0 and not xs.any() and float(ys) == 0


@pytest.mark.parametrize("name,n", [("cfg2", 50_021), ("cfg3", 30_011), ("cfg4", 12_007)])
def test_sums_real_parity(ctx, name, n):
    """Real-valued designs of the benched shapes (cfg2 p = 100 single panel; cfg3 p = 500 and
    cfg4 p = 1000 two-panel) against the oracle's Gram and fp64 column sums."""
    from paper_1801_09661_b200 import oem_gram_sums
    spec = CONFIGS[name].spec.replace(n=n)
    X, y = dg.rows_host(spec, dg.beta(spec))
    G, c, yy, xs, ys, nt = oem_gram_sums(ctx, _dev(X), torch.from_numpy(y).cuda())
    Go, co, yyo = orc.gram(X, y)
    assert scale_err(G.cpu().numpy(), Go) <= 1e-12
    assert xty_err(c.cpu().numpy(), co, Go, yyo) <= 1e-12
    assert abs(float(yy) - yyo) <= 1e-12 * yyo
    # column sums: error bound relative to sum |x_ij| (any summation order)
    xabs = np.abs(X).sum(axis=0)
    assert np.max(np.abs(xs.cpu().numpy() - X.sum(axis=0)) / xabs) <= 1e-12
    assert abs(float(ys) - y.sum()) <= 1e-12 * np.abs(y).sum()


@pytest.mark.parametrize("p,std", [(30, True), (300, False)])
def test_intercept_fit_from_one_pass(ctx, p, std):
    """The intercept / standardization fit (R#2-3) fed by the one-pass sums matches the oracle's
    data-transformation route (centre / scale the data, then fit)."""
    from paper_1801_09661_b200 import oem_fit_path, oem_gram_sums
    n = 8000
    spec = CONFIGS["cfg2"].spec.replace(n=n, p=p, nnz=min(8, p))
    X, y = dg.rows_host(spec, dg.beta(spec))
    rng = np.random.default_rng(p)
    X = X * rng.uniform(0.3, 4.0, p) + rng.uniform(-3, 3, p)
    y = y + 2.5
    G, c, yy, xs, ys, nn = oem_gram_sums(ctx, _dev(X), torch.from_numpy(y).cuda())
    pens = [("lasso", 0.0, 1.0), ("mcp", 3.0, 1.0)]
    fit = oem_fit_path(ctx, G, c, [nn], pens, nlambda=15, standardize=std, xsum=xs.reshape(1, p),
                       ysum=ys.reshape(1))
    d = float(fit.d[0])
    lams = [fit.lam[0, q].cpu().numpy() for q in range(2)]
    ref = orc.fit_transformed(X, y, pens, standardize=std, intercept=True, d=d, lambdas=lams)
    for q in range(2):
        assert np.max(np.abs(fit.beta[0, q].cpu().numpy() - ref["beta"][q])) <= 1e-8
        assert np.max(np.abs(fit.intercept[0, q].cpu().numpy() - ref["intercept"][q])) <= 1e-7


def test_cv_with_intercept_from_one_pass(ctx):
    """f2 with an intercept from one fold pass: the held-out error of y - b0 - X b on each fold
    equals the oracle's direct residuals (R#39)."""
    from paper_1801_09661_b200 import oem_cv_error, oem_fit_path, oem_gram_folds_sums
    n, p, K = 6000, 25, 4
    spec = CONFIGS["cfg2"].spec.replace(n=n, p=p, nnz=8)
    X, y = dg.rows_host(spec, dg.beta(spec))
    X = X + 1.5
    y = y - 3.0
    Gk, ck, yyk, xs, ys, cnt = oem_gram_folds_sums(ctx, _dev(X), torch.from_numpy(y).cuda(), K)
    fit = oem_fit_path(ctx, Gk, ck, cnt, [("lasso", 0.0, 1.0)], nlambda=10, fold_mode=True, xsum=xs, ysum=ys)
    cv = oem_cv_error(ctx, Gk, ck, yyk, cnt, fit.beta, intercept=fit.intercept, xsum_folds=xs, ysum_folds=ys)
    ref = orc.cv_error(X, y, K, fit.beta.cpu().numpy(), intercepts=fit.intercept.cpu().numpy())
    fold = np.arange(n) % K
    scale = np.array([np.mean((y[fold == k] - y.mean()) ** 2) for k in range(K)])[:, None, None]
    assert np.max(np.abs(cv.err.cpu().numpy() - ref) / scale) <= 1e-10
