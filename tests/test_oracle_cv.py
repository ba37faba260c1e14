"""Pins for the f2 oracle (held-out error of fast CV and the cv.oem summaries) against closed
forms, exact rational arithmetic and hand-worked selections (R#33-35)."""
from fractions import Fraction

import numpy as np

import oracle as orc


def test_null_fit_is_mean_square_of_fold():
    """b = 0 (every fit at lambda_max): e_k = (1/n_k) sum_{i in fold k} y_i^2 (closed form)."""
    rng = np.random.default_rng(3)
    n, p, K = 103, 4, 5
    X = rng.standard_normal((n, p))
    y = rng.standard_normal(n)
    B = np.zeros((K + 1, 2, 3, p))
    err = orc.cv_error(X, y, K, B)
    for k in range(K):
        yk = y[np.arange(n) % K == k]
        assert np.allclose(err[k], np.mean(yk ** 2), rtol=1e-14, atol=0)


def test_exact_fit_has_zero_error():
    """y = X b* exactly with dyadic entries: residuals vanish exactly, so does the error."""
    rng = np.random.default_rng(4)
    n, p, K = 60, 3, 3
    X = rng.integers(-4, 5, size=(n, p)).astype(float)
    bstar = np.array([0.5, -1.0, 2.0])
    y = X @ bstar
    B = np.broadcast_to(bstar, (K + 1, 1, 2, p)).copy()
    assert np.all(orc.cv_error(X, y, K, B) == 0.0)


def test_row_offset_and_brute_force_rational():
    """Integer data, rational coefficients: compare with exact Fraction arithmetic on folds taken
    from a nonzero global row offset (fold(i) = (offset + i) mod K, R#19)."""
    rng = np.random.default_rng(5)
    n, p, K, off = 17, 2, 3, 7
    X = rng.integers(-3, 4, size=(n, p))
    y = rng.integers(-5, 6, size=n)
    B = rng.integers(-4, 5, size=(K + 1, 1, 2, p)) / 4.0
    err = orc.cv_error(X.astype(float), y.astype(float), K, B, row_offset=off)
    for k in range(K):
        rows = [i for i in range(n) if (off + i) % K == k]
        for l in range(2):
            b = [Fraction(v) for v in B[k + 1, 0, l]]
            s = sum((Fraction(int(y[i])) - sum(Fraction(int(X[i, j])) * b[j] for j in range(p))) ** 2 for i in rows)
            assert err[k, 0, l] == float(s / len(rows))


def test_intercept_rational_and_closed_form():
    """With intercepts the residual is y_i - b0 - x_i^T b (a fold-mode fit with an
    intercept must be scored with it). b = 0: e_k = mean over the fold of (y_i - b0)^2 = var_k +
    (ybar_k - b0)^2 (closed form); integer data with rational (b0, b): exact Fraction arithmetic."""
    rng = np.random.default_rng(9)
    n, p, K = 41, 3, 4
    X = rng.integers(-3, 4, size=(n, p))
    y = rng.integers(-5, 6, size=n)
    B = np.zeros((K + 1, 1, 2, p))
    B0 = np.array([0.0, 1.5, -2.0, 0.25, 3.0])[:, None, None] * np.ones((K + 1, 1, 2))
    err = orc.cv_error(X.astype(float), y.astype(float), K, B, intercepts=B0)
    for k in range(K):
        yk = y[np.arange(n) % K == k].astype(float)
        expect = np.var(yk) + (yk.mean() - B0[k + 1, 0, 0]) ** 2
        assert np.allclose(err[k], expect, rtol=1e-13, atol=0)
    B = rng.integers(-4, 5, size=(K + 1, 1, 2, p)) / 4.0
    B0 = rng.integers(-8, 9, size=(K + 1, 1, 2)) / 8.0
    err = orc.cv_error(X.astype(float), y.astype(float), K, B, intercepts=B0)
    for k in range(K):
        rows = [i for i in range(n) if i % K == k]
        for l in range(2):
            b = [Fraction(v) for v in B[k + 1, 0, l]]
            b0 = Fraction(B0[k + 1, 0, l])
            s = sum((Fraction(int(y[i])) - b0 - sum(Fraction(int(X[i, j])) * b[j] for j in range(p))) ** 2
                    for i in rows)
            assert err[k, 0, l] == float(s / len(rows))


def test_summary_two_folds_closed_form():
    """K = 2, equal folds: cvm = (e1 + e2)/2 and cvsd = |e1 - e2| / 2."""
    err = np.array([[[1.0, 4.0, 2.5]], [[3.0, 1.0, 2.5]]])
    cvm, cvsd, imin, i1se, best = orc.cv_summary(err, [10, 10])
    assert np.allclose(cvm[0], [2.0, 2.5, 2.5])
    assert np.allclose(cvsd[0], [1.0, 1.5, 0.0])
    assert imin == [0] and i1se == [0] and best == 0


def test_selection_rules_hand_worked():
    """lambda_min = first argmin; lambda_1se = largest lambda within one sd; best penalty."""
    K = 2
    # build err so that cvm = target exactly (equal folds, e1 = e2 = cvm -> cvsd = 0), then
    # split to get a chosen cvsd: e1 = m - s, e2 = m + s gives cvm = m, cvsd = s
    m = np.array([[5.0, 3.0, 2.0, 2.5, 4.0], [4.0, 1.5, 1.5, 3.0, 6.0]])
    s = np.array([[1.0, 1.0, 1.2, 1.0, 1.0], [0.0, 0.25, 0.0, 0.0, 0.0]])
    err = np.stack([m - s, m + s])
    cvm, cvsd, imin, i1se, best = orc.cv_summary(err, [7, 7])
    assert np.allclose(cvm, m) and np.allclose(cvsd, s)
    assert imin == [2, 1]            # ties in penalty 1 (1.5, 1.5) -> the larger lambda (index 1)
    assert i1se == [1, 1]            # penalty 0: threshold 3.2 admits index 1 (3.0) not 0 (5.0)
    assert best == 1                 # min cvm 1.5 < 2.0
