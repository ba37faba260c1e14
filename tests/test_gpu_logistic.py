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


@pytest.mark.parametrize("n,p,L", [(4000, 20, 12), (20_011, 200, 8)])
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
