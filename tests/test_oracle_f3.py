"""Pins for the f3 oracle pieces (intercept, standardization, compute.loss) against closed forms
and invariances (R#2-3, R#37)."""
import numpy as np

import oracle as orc


def _data(seed, n=700, p=6):
    rng = np.random.default_rng(seed)
    X = rng.standard_normal((n, p)) * rng.uniform(0.5, 3.0, p) + rng.uniform(-2, 2, p)
    y = 1.5 + X @ rng.normal(0, 1, p) + rng.standard_normal(n)
    return X, y


def test_intercept_lambda0_is_ols_with_intercept():
    X, y = _data(41)
    r = orc.fit_transformed(X, y, [("lasso", 0.0, 1.0)], lambdas=[[0.0]], intercept=True, tol=1e-14)
    A = np.hstack([np.ones((X.shape[0], 1)), X])
    sol = np.linalg.lstsq(A, y, rcond=None)[0]
    assert abs(r["intercept"][0][0] - sol[0]) <= 1e-9
    assert np.max(np.abs(r["beta"][0][0] - sol[1:])) <= 1e-9


def test_intercept_translation_invariance():
    """Shifting every column and y by constants leaves the slopes unchanged; the intercept moves
    by dy - shift^T beta."""
    X, y = _data(42)
    shift = np.array([3.0, -1.0, 0.5, 10.0, -4.0, 2.0])
    pens = [("lasso", 0.0, 1.0), ("mcp", 3.0, 1.0)]
    a = orc.fit_transformed(X, y, pens, nlambda=15, intercept=True, standardize=True)
    b = orc.fit_transformed(X + shift, y + 7.0, pens, nlambda=15, intercept=True, standardize=True, d=a["d"],
                            lambdas=a["lambda"])
    for q in range(2):
        assert np.max(np.abs(a["beta"][q] - b["beta"][q])) <= 1e-9
        assert np.max(np.abs(b["intercept"][q] - (a["intercept"][q] + 7.0 - a["beta"][q] @ shift))) <= 1e-8


def test_standardize_scale_equivariance_and_noop():
    """Scaling column j by k divides beta_j by k (standardized fit); already-standardized columns
    make standardization a no-op."""
    X, y = _data(43)
    k = np.array([2.0, 0.5, 1.0, 8.0, 1.0, 0.25])
    pens = [("lasso", 0.0, 1.0)]
    a = orc.fit_transformed(X, y, pens, nlambda=12, intercept=True, standardize=True)
    b = orc.fit_transformed(X * k, y, pens, nlambda=12, intercept=True, standardize=True, d=a["d"], lambdas=a["lambda"])
    assert np.max(np.abs(a["beta"][0] - b["beta"][0] * k)) <= 1e-9
    Z = X - X.mean(axis=0)
    Z /= np.sqrt(np.mean(Z * Z, axis=0))
    c = orc.fit_transformed(Z, y, pens, nlambda=12, intercept=True, standardize=True)
    e = orc.fit_transformed(Z, y, pens, nlambda=12, intercept=True, standardize=False, d=c["d"], lambdas=c["lambda"])
    assert np.max(np.abs(c["beta"][0] - e["beta"][0])) <= 1e-10


def test_zero_variance_column_gets_zero():
    X, y = _data(44)
    X[:, 2] = 5.0
    r = orc.fit_transformed(X, y, [("lasso", 0.0, 1.0)], nlambda=8, intercept=True, standardize=True)
    assert not r["beta"][0][:, 2].any()


def test_path_loss_closed_forms():
    X, y = _data(45, n=200, p=3)
    B = np.zeros((1, 2, 4, 3))
    assert np.allclose(orc.path_loss(X, y, B), np.mean(y * y), rtol=1e-14, atol=0)
    bstar = np.array([0.5, -0.25, 2.0])
    Xi = np.round(X * 4) / 4
    assert np.all(orc.path_loss(Xi, Xi @ bstar, bstar[None, None, None, :]) == 0.0)
