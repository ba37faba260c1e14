"""Generator pins (host side): Philox known answers, software math accuracy, design statistics.

The generator holds none of the method's arithmetic; these tests make sure the inputs are the
distributions the configs name (BASELINE.json configs; §6.1)."""
import json
import math
import os

import numpy as np
import pytest

import datagen as dg
from datagen.configs import CONFIGS

HERE = os.path.dirname(os.path.abspath(__file__))


def test_philox_known_answers():
    with open(os.path.join(HERE, "golden", "random123_philox_kat.json")) as f:
        kat = json.load(f)
    for v in kat["vectors"]:
        ctr = [int(x, 16) for x in v["ctr"]]
        key = [int(x, 16) for x in v["key"]]
        assert dg.philox(ctr, key) == [int(x, 16) for x in v["out"]]


def test_software_math_accuracy():
    rng = np.random.default_rng(0)
    h = dg.host()
    for x in np.concatenate([rng.random(2000), rng.random(200) * 1e-12, [2.0 ** -53, 1 - 2.0 ** -53]]):
        if x <= 0:
            continue
        assert abs(h.dg_ln(x) - math.log(x)) <= 4e-16 * max(1.0, abs(math.log(x)))
    for x in rng.uniform(-40, 40, 2000):
        assert abs(h.dg_exp(x) - math.exp(x)) <= 4e-15 * math.exp(x)
    import ctypes
    s, c = ctypes.c_double(), ctypes.c_double()
    for u in np.concatenate([rng.random(2000), [0.125, 0.25, 0.5, 0.75, 1e-17]]):
        h.dg_sincos2pi(u, ctypes.byref(s), ctypes.byref(c))
        assert abs(s.value - math.sin(2 * math.pi * u)) < 2e-15
        assert abs(c.value - math.cos(2 * math.pi * u)) < 2e-15


def test_iid_normals_statistics():
    spec = dg.make_spec(11, 20000, 8, dg.DG_IID, beta_kind=dg.DG_BETA_EXPLICIT)
    X, _ = dg.rows_host(spec, np.zeros(8), want_y=False)
    z = X.ravel()
    assert abs(z.mean()) < 0.02
    assert abs(z.var() - 1) < 0.02
    # 4th moment of N(0,1) is 3
    assert abs((z ** 4).mean() - 3) < 0.1
    C = np.corrcoef(X.T)
    assert np.max(np.abs(C - np.eye(8))) < 0.04


def test_ar1_and_block_correlation():
    spec = dg.make_spec(12, 40000, 6, dg.DG_AR1, rho=0.5, beta_kind=dg.DG_BETA_EXPLICIT)
    X, _ = dg.rows_host(spec, np.zeros(6), want_y=False)
    C = np.cov(X.T, bias=True)
    target = 0.5 ** np.abs(np.subtract.outer(np.arange(6), np.arange(6)))
    assert np.max(np.abs(C - target)) < 0.04
    spec = dg.make_spec(13, 40000, 6, dg.DG_BLOCK, rho=0.4, group_size=3,
                        beta_kind=dg.DG_BETA_EXPLICIT)
    X, _ = dg.rows_host(spec, np.zeros(6), want_y=False)
    C = np.cov(X.T, bias=True)
    g = np.arange(6) // 3
    target = np.where(g[:, None] == g[None, :], 0.4, 0.0) + 0.6 * np.eye(6)
    assert np.max(np.abs(C - target)) < 0.04


def test_column_and_row_subsets_are_consistent():
    for cfg in (CONFIGS["cfg2"].with_n(300), CONFIGS["cfg4"].with_n(100)):
        b = dg.beta(cfg.spec)
        Xf, yf = dg.rows_host(cfg.spec, b)
        Xs, ys = dg.rows_host(cfg.spec, b, row0=37, nrows=50, col0=13, ncols=29)
        assert np.array_equal(Xs, Xf[37:87, 13:42])
        assert np.array_equal(ys, yf[37:87])


def test_beta_recipes():
    b1 = dg.beta(CONFIGS["cfg1"].spec, CONFIGS["cfg1"].explicit_beta)
    assert list(b1[:5]) == [1.0, -1.0, 0.5, -0.5, 2.0] and not b1[5:].any()
    b2 = dg.beta(CONFIGS["cfg2"].spec)
    assert np.count_nonzero(b2) == 10 and np.all(np.abs(b2) <= 2)
    b3 = dg.beta(CONFIGS["cfg3"].spec)
    assert np.count_nonzero(b3) == 25
    b4 = dg.beta(CONFIGS["cfg4"].spec)
    active = np.nonzero(np.abs(b4.reshape(100, 10)).sum(1))[0]
    assert len(active) == 5 and np.all(b4.reshape(100, 10)[active] != 0)
    b5 = dg.beta(CONFIGS["cfg5"].spec)
    assert np.count_nonzero(b5) == 20 and np.all(np.abs(b5) <= 1)
    assert np.array_equal(b2, dg.beta(CONFIGS["cfg2"].spec))  # reproducible


def test_linear_response_model():
    cfg = CONFIGS["cfg2"].with_n(20000)
    b = dg.beta(cfg.spec)
    X, y = dg.rows_host(cfg.spec, b)
    r = y - X @ b
    assert abs(r.std() - 2.0) < 0.05  # noise sd 2
    assert abs(r.mean()) < 0.05


def test_logistic_response_model():
    cfg = CONFIGS["cfg5"].with_n(20000)
    b = dg.beta(cfg.spec)
    X, y = dg.rows_host(cfg.spec, b)
    assert set(np.unique(y)) <= {0.0, 1.0}
    pr = 1 / (1 + np.exp(-(X @ b)))
    # calibration: mean label matches mean probability
    assert abs(y.mean() - pr.mean()) < 0.015
    assert abs(((y - pr) * (X @ b)).mean()) < 0.05


def test_sparse_design_pattern():
    """SPARSE (include/oem_datagen.h): every cell is the IID design's z_ij kept with probability d
    (stream-5 uniform < d), so the kept values equal the IID generator's bit for bit and the
    density and the pattern's independence follow the binomial law."""
    d = 0.05
    spec = dg.make_spec(21, 20000, 40, dg.DG_SPARSE, rho=d, beta_kind=dg.DG_BETA_EXPLICIT)
    iid = dg.make_spec(21, 20000, 40, dg.DG_IID, beta_kind=dg.DG_BETA_EXPLICIT)
    X, _ = dg.rows_host(spec, np.zeros(40), want_y=False)
    Z, _ = dg.rows_host(iid, np.zeros(40), want_y=False)
    nz = X != 0
    assert np.array_equal(X[nz], Z[nz])
    m = nz.size
    assert abs(nz.mean() - d) < 5 * np.sqrt(d * (1 - d) / m)
    # the pattern is independent of the values: the kept values are N(0, 1)
    assert abs(X[nz].mean()) < 0.05 and abs(X[nz].var() - 1) < 0.06
    # column subsets and the response agree with the full rows
    bt = np.zeros(40)
    bt[[3, 17]] = [0.5, -1.25]
    spec2 = spec.replace(sigma=2.0)
    Xf, yf = dg.rows_host(spec2, bt, 100, 50)
    Xs, ys = dg.rows_host(spec2, bt, 100, 50, 10, 7)
    assert np.array_equal(Xs, Xf[:, 10:17]) and np.array_equal(ys, yf)
