"""Pins for oracle O1-O3 (Gram, fold Grams, weighted Gram) against things other than itself:
SPEC worked values, exact rational / integer arithmetic, closed forms (Hadamard), library
routines (numpy BLAS) and algebraic identities in a different arithmetic form."""
from fractions import Fraction

import numpy as np
import pytest

import oracle as orc


def scale_err(A, B, diag):
    """Scale-aware error |dA_jk| / sqrt(A_jj A_kk) (reading R#32)."""
    s = np.sqrt(np.outer(diag, diag))
    return np.max(np.abs(A - B) / s)


def test_spec_worked_example(golden):
    ex = golden["gram"][0]
    X = np.array(ex["X"])
    y = np.array(ex["y"])
    G, c, yy = orc.gram(X, y)
    n = X.shape[0]
    assert np.array_equal(G / n, np.array(ex["xtx_over_n"]))
    assert np.array_equal(c / n, np.array(ex["xty_over_n"]))
    assert yy == 5.0


def test_integer_design_exact():
    """Integer-valued X: every partial sum is an exact integer < 2^53, so the oracle must equal
    exact integer arithmetic bit for bit."""
    rng = np.random.default_rng(1)
    n, p = 1500, 13
    Xi = rng.integers(-8, 9, size=(n, p))
    yi = rng.integers(-8, 9, size=n)
    G, c, yy = orc.gram(Xi.astype(float), yi.astype(float))
    Xo = Xi.astype(object)
    Gx = Xo.T.dot(Xo)
    cx = Xo.T.dot(yi.astype(object))
    assert np.array_equal(G, Gx.astype(float))
    assert np.array_equal(c, cx.astype(float))
    assert yy == float(sum(int(v) * int(v) for v in yi))


def test_compensated_sum_is_correctly_rounded():
    """Random real X with heavy cancellation: the oracle equals the exactly rounded rational sum
    (Fraction brute force) to within one ulp, far below the 1e-12 parity bar."""
    rng = np.random.default_rng(2)
    n, p = 300, 4
    X = rng.standard_normal((n, p)) * np.array([1.0, 1e8, 1e-8, 3.0])
    X[:, 3] = -X[:, 0] + rng.standard_normal(n) * 1e-9  # column 3 nearly cancels column 0
    y = rng.standard_normal(n)
    G, c, yy = orc.gram(X, y)
    for j in range(p):
        for k in range(p):
            exact = sum(Fraction(X[i, j]) * Fraction(X[i, k]) for i in range(n))
            assert abs(Fraction(G[j, k]) - exact) <= abs(exact) * Fraction(2, 2 ** 53) + Fraction(1, 2 ** 1074)
        exact = sum(Fraction(X[i, j]) * Fraction(y[i]) for i in range(n))
        assert abs(Fraction(c[j]) - exact) <= abs(exact) * Fraction(2, 2 ** 53)


def test_hadamard_closed_form():
    """+-1 Walsh-Hadamard design with n = 2^m: X^T X = n I exactly."""
    H = np.array([[1.0]])
    for _ in range(7):
        H = np.block([[H, H], [H, -H]])
    X = H[:, 1:20]  # 128 x 19, orthogonal columns
    G, c, _ = orc.gram(X, H[:, 0])
    assert np.array_equal(G, 128 * np.eye(19))
    assert np.array_equal(c, np.zeros(19))  # columns orthogonal to the all-ones column


def test_matches_blas_and_block_invariance():
    rng = np.random.default_rng(3)
    n, p = 2000, 9
    X = rng.standard_normal((n, p))
    y = rng.standard_normal(n)
    G, c, yy = orc.gram(X, y)
    d = np.diag(G)
    assert scale_err(G, X.T @ X, d) < 1e-13
    assert np.max(np.abs(c - X.T @ y) / np.sqrt(d * yy)) < 1e-13
    for block in (1, 7, n):
        acc = orc.GramAccumulator(p)
        for r in range(0, n, block):
            acc.add(X[r:r + block], y[r:r + block], nthreads=1)
        G2, c2, yy2 = acc.result()
        assert scale_err(G2, G, d) < 1e-15
        assert np.max(np.abs(c2 - c)) <= 1e-15 * np.max(np.abs(c))
    # thread count does not change the result beyond the last bit
    G3, _, _ = orc.gram(X, y, nthreads=5)
    assert scale_err(G3, G, d) < 1e-15


def test_folds_identities():
    rng = np.random.default_rng(4)
    n, p, K = 403, 5, 10  # ragged folds
    Xi = rng.integers(-8, 9, size=(n, p)).astype(float)
    yi = rng.integers(-8, 9, size=n).astype(float)
    G, c, yy = orc.gram(Xi, yi)
    Gk, ck, yyk, cnt = orc.gram_folds(Xi, yi, K, row_offset=3)
    # fold(i) = (3 + i) mod K
    assert list(cnt) == [sum(1 for i in range(n) if (3 + i) % K == k) for k in range(K)]
    assert np.array_equal(Gk.sum(0), G) and np.array_equal(ck.sum(0), c) and yyk.sum() == yy
    for k in range(K):
        rows = [(3 + i) % K == k for i in range(n)]
        Gd, cd, _ = orc.gram(Xi[rows], yi[rows])
        assert np.array_equal(Gk[k], Gd) and np.array_equal(ck[k], cd)
    Gm, cm = orc.fold_complements(Gk, ck)  # paper's form sum_{c != k}
    for k in range(K):
        assert np.array_equal(Gm[k], G - Gk[k]) and np.array_equal(cm[k], c - ck[k])
    # K = 1 equals the full Gram; K = n (leave-one-out) gives outer products
    G1, c1, _, n1 = orc.gram_folds(Xi, yi, 1)
    assert np.array_equal(G1[0], G) and n1[0] == n
    Xs, ys = Xi[:6], yi[:6]
    GL, cL, _, nL = orc.gram_folds(Xs, ys, 6)
    for i in range(6):
        assert np.array_equal(GL[i], np.outer(Xs[i], Xs[i])) and np.all(nL == 1)
    # K = 2: complement of fold 0 is the Gram computed directly on fold 1
    G2, c2, _, _ = orc.gram_folds(Xi, yi, 2)
    Gm2, cm2 = orc.fold_complements(G2, c2)
    Gd, cd, _ = orc.gram(Xi[1::2], yi[1::2])
    assert np.array_equal(Gm2[0], Gd) and np.array_equal(cm2[0], cd)


def test_weighted_at_zero_beta():
    """beta = 0: mu = 1/2, w = 1/4, z = 4y - 2, so G_w = G/4 and c_w = X^T (y - 1/2)
    exactly, and loglik = -n log 2."""
    rng = np.random.default_rng(5)
    n, p = 500, 6
    X = rng.integers(-8, 9, size=(n, p)).astype(float)
    y = (rng.random(n) < 0.4).astype(float)
    Gw, cw, sc = orc.gram_weighted(X, y, np.zeros(p))
    G, _, _ = orc.gram(X, y)
    assert np.array_equal(Gw, G / 4)
    Xo = X.astype(int).astype(object)
    exact = Xo.T.dot((2 * y.astype(int) - 1).astype(object))  # 2 * X^T (y - 1/2)
    assert np.array_equal(cw * 2, exact.astype(float))
    assert sc[0] == n / 4
    assert abs(sc[1] + n * np.log(2)) < 1e-10


def test_weighted_random_beta_identity():
    """Different arithmetic form: c_w = G_w beta + X^T (y - mu) (algebraically equal to
    sum w z x with z = eta + (y - mu)/w). Computed here with numpy."""
    rng = np.random.default_rng(6)
    n, p = 3000, 7
    X = rng.standard_normal((n, p))
    beta = rng.uniform(-0.5, 0.5, p)
    eta = X @ beta
    mu = 1 / (1 + np.exp(-eta))
    y = (rng.random(n) < mu).astype(float)
    Gw, cw, sc = orc.gram_weighted(X, y, beta)
    w = mu * (1 - mu)
    Gref = (X * w[:, None]).T @ X
    d = np.diag(Gref)
    assert scale_err(Gw, Gref, d) < 1e-12
    cref = Gref @ beta + X.T @ (y - mu)
    assert np.max(np.abs(cw - cref)) < 1e-11 * np.max(np.abs(cref))
    assert abs(sc[0] - w.sum()) < 1e-12 * w.sum()
    ll = np.sum(y * eta - np.logaddexp(0, eta))
    assert abs(sc[1] - ll) < 1e-11 * abs(ll)
    assert np.all(np.linalg.eigvalsh(Gw / n) <= np.linalg.eigvalsh(X.T @ X / n / 4).max() + 1e-12)


def test_weighted_clamp():
    """mu clamped to [eps, 1-eps] (R#25): w = eps(1-eps) for extreme eta."""
    X = np.array([[100.0], [-100.0]])
    Gw, cw, sc = orc.gram_weighted(X, np.array([1.0, 0.0]), np.array([1.0]), eps=1e-5)
    hi = 1 - 1e-5
    w = hi * (1 - hi) + 1e-5 * (1 - 1e-5)
    assert abs(sc[0] - w) < 1e-15 * w
    assert abs(Gw[0, 0] - w * 1e4) < 1e-15 * w * 1e4
