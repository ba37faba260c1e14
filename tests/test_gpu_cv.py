"""GPU parity for f2 (oem_cv_error): the fast-CV held-out error from the fold sums (Gram
identity, no second pass) against the oracle's direct held-out residuals (R#33), and the cv.oem
summaries / selection against the oracle's explicit loops (R#34-35)."""
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


@pytest.mark.parametrize("n,p,K,pens,L", [
    (20_000, 40, 5, [("lasso", 0.0, 1.0), ("mcp", 3.0, 1.0)], 20),
    (20_011, 33, 10, [("lasso", 0.0, 1.0)], 15),        # ragged: n not a multiple of K
    (3_001, 130, 3, [("scad", 3.7, 1.0), ("enet", 0.0, 0.5), ("lasso", 0.0, 1.0)], 9),
])
def test_cv_error_parity(ctx, n, p, K, pens, L):
    from paper_1801_09661_b200 import oem_cv_error, oem_fit_path, oem_gram_folds
    spec = CONFIGS["cfg3"].spec.replace(n=n, p=p, nnz=min(10, p))
    bt = dg.beta(spec)
    Xd, yd = device_rows(spec, bt)
    X, y = dg.rows_host(spec, bt)
    Gk, ck, yyk, cnt = oem_gram_folds(ctx, Xd, yd, K)
    fit = oem_fit_path(ctx, Gk, ck, cnt, pens, nlambda=L, fold_mode=True)
    cv = oem_cv_error(ctx, Gk, ck, yyk, cnt, fit.beta)
    B = fit.beta.cpu().numpy()
    err_o = orc.cv_error(X, y, K, B)
    # tolerance: the identity's three terms are O(n_k mean(y_k^2)); fp64 rounding of the
    # sums leaves ~1e-13 of that scale, so compare relative to mean(y_k^2) (R#33)
    fold = np.arange(n) % K
    scale = np.array([np.mean(y[fold == k] ** 2) for k in range(K)])[:, None, None]
    err_g = cv.err.cpu().numpy()
    assert np.max(np.abs(err_g - err_o) / scale) <= 1e-10
    cvm_o, cvsd_o, imin_o, i1se_o, best_o = orc.cv_summary(err_o, cnt)
    s = float(np.mean(y ** 2))
    assert np.max(np.abs(cv.cvm.cpu().numpy() - cvm_o)) <= 1e-10 * s
    assert np.max(np.abs(cv.cvsd.cpu().numpy() - cvsd_o)) <= 1e-8 * s
    # selection: unique up to near-ties; the GPU's choices must attain the oracle's optimum
    for q in range(len(pens)):
        assert cvm_o[q, cv.idx_min[q]] <= cvm_o[q, imin_o[q]] + 1e-10 * s
        assert cvm_o[q, cv.idx_1se[q]] <= cvm_o[q, imin_o[q]] + cvsd_o[q, imin_o[q]] + 1e-10 * s
        assert cv.idx_1se[q] <= cv.idx_min[q]
        # lambda_1se is the LARGEST lambda (smallest index) within one SE: no smaller index may
        # satisfy the threshold by more than the rounding tolerance (R#35)
        thr = cvm_o[q, cv.idx_min[q]] + cvsd_o[q, cv.idx_min[q]]
        assert np.all(cvm_o[q, :cv.idx_1se[q]] > thr - 1e-10 * s), q
        if abs(cvm_o[q, imin_o[q]] - np.partition(cvm_o[q], 1)[1]) > 1e-9 * s:
            assert cv.idx_min[q] == imin_o[q]
    mins = [cvm_o[q, imin_o[q]] for q in range(len(pens))]
    assert mins[cv.best] <= min(mins) + 1e-10 * s


def test_cv_null_model_closed_form(ctx):
    """At lambda_max every complement fit is b = 0, so e_k = mean of y^2 over fold k exactly
    in the identity (b^T terms vanish): yty_k / n_k."""
    from paper_1801_09661_b200 import oem_cv_error, oem_fit_path, oem_gram_folds
    spec = CONFIGS["cfg3"].spec.replace(n=5000, p=20, nnz=5)
    bt = dg.beta(spec)
    Xd, yd = device_rows(spec, bt)
    Gk, ck, yyk, cnt = oem_gram_folds(ctx, Xd, yd, 4)
    fit = oem_fit_path(ctx, Gk, ck, cnt, [("lasso", 0.0, 1.0)], nlambda=5, fold_mode=True,
                       lambda_max=1e6)   # above every complement's own lambda_max
    cv = oem_cv_error(ctx, Gk, ck, yyk, cnt, fit.beta)
    assert not fit.beta[1:, :, 0].any()
    e0 = cv.err[:, 0, 0].cpu().numpy()
    assert np.array_equal(e0, yyk.cpu().numpy() / np.array(cnt, dtype=float))


def test_cv_errors(ctx):
    from paper_1801_09661_b200 import OemError, oem_cv_error
    G = torch.zeros((1, 3, 3), dtype=torch.float64, device="cuda")
    c = torch.zeros((1, 3), dtype=torch.float64, device="cuda")
    yy = torch.zeros(1, dtype=torch.float64, device="cuda")
    B = torch.zeros((2, 1, 2, 3), dtype=torch.float64, device="cuda")
    with pytest.raises(OemError) as e:
        oem_cv_error(ctx, G, c, yy, [5], B)
    assert e.value.status == "OEM_ERR_DIM"
    G2 = torch.zeros((2, 3, 3), dtype=torch.float64, device="cuda")
    with pytest.raises(OemError) as e:
        oem_cv_error(ctx, G2, torch.zeros((2, 3), dtype=torch.float64, device="cuda"),
                     torch.zeros(2, dtype=torch.float64, device="cuda"), [5, 0],
                     torch.zeros((3, 1, 2, 3), dtype=torch.float64, device="cuda"))
    assert e.value.status == "OEM_ERR_EMPTY_FOLD"


def test_cv_error_with_intercept(ctx):
    """fold-mode fits with an intercept are scored with it. The GPU forms the held-out
    error of y - b0 - X b from the fold sums and the fold column sums (R#33); the oracle streams
    the held-out rows directly (orc.cv_error with intercepts)."""
    from paper_1801_09661_b200 import oem_cv_error, oem_fit_path, oem_gram_folds, oem_gram_moments
    n, p, K = 9_001, 24, 5
    spec = CONFIGS["cfg3"].spec.replace(n=n, p=p, nnz=6)
    bt = dg.beta(spec)
    Xd, yd = device_rows(spec, bt)
    Xd = Xd + 0.75          # columns with nonzero means and a shifted response: the intercept matters
    yd = yd + 3.0
    X, y = Xd.cpu().numpy(), yd.cpu().numpy()
    Xp = torch.zeros((n, p), dtype=torch.float64, device="cuda")
    Xp.copy_(Xd)
    Gk, ck, yyk, cnt = oem_gram_folds(ctx, Xp, yd, K)
    xs, ys = oem_gram_moments(ctx, Xp, yd, K)
    pens = [("lasso", 0.0, 1.0), ("mcp", 3.0, 1.0)]
    fit = oem_fit_path(ctx, Gk, ck, cnt, pens, nlambda=12, fold_mode=True, xsum=xs, ysum=ys)
    cv = oem_cv_error(ctx, Gk, ck, yyk, cnt, fit.beta, intercept=fit.intercept, xsum_folds=xs, ysum_folds=ys)
    err_o = orc.cv_error(X, y, K, fit.beta.cpu().numpy(), intercepts=fit.intercept.cpu().numpy())
    fold = np.arange(n) % K
    scale = np.array([np.mean((y[fold == k] - y.mean()) ** 2) for k in range(K)])[:, None, None]
    assert np.max(np.abs(cv.err.cpu().numpy() - err_o) / scale) <= 1e-10
    # without the intercept the same coefficients score far worse: the correction is not a no-op
    cv0 = oem_cv_error(ctx, Gk, ck, yyk, cnt, fit.beta)
    assert float(cv0.cvm.min()) > 2 * float(cv.cvm.min())
