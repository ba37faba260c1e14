"""GPU parity for the Gram passes (a2 oem_gram, a3 oem_gram_folds, a4 oem_gram_weighted)
through the C ABI, element by element against the oracle on identical seeded inputs.

Bar (north star): scale-aware relative 1e-12 (R#32); integer-valued designs are
bit-exact (every partial sum is an exact integer, so any summation order gives the same bits)."""
import numpy as np
import pytest

import datagen as dg
import oracle as orc
from datagen.configs import CONFIGS
from gpu_util import cfg4_oracle_sample, device_rows, scale_err, xty_err

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")


@pytest.fixture(scope="module")
def ctx():
    from paper_1801_09661_b200 import Context
    c = Context(0)
    yield c
    c.close()


def to_dev(a):
    return torch.from_numpy(np.ascontiguousarray(a)).cuda()


def int_design(seed, n, p, lo=-8, hi=9):
    rng = np.random.default_rng(seed)
    return rng.integers(lo, hi, size=(n, p)).astype(float), rng.integers(lo, hi, size=n).astype(float)


# ---------------------------------------------------------------- device generator
@pytest.mark.parametrize("name", ["cfg1", "cfg2", "cfg3", "cfg4", "cfg5"])
def test_device_generator_bit_identical(name):
    cfg = CONFIGS[name]
    bt = dg.beta(cfg.spec, cfg.explicit_beta)
    for row0, nrows in ((0, 70), (cfg.n - 37, 37), (cfg.n // 3, 129)):
        Xd, yd = device_rows(cfg.spec, bt, row0, nrows)
        Xh, yh = dg.rows_host(cfg.spec, bt, row0, nrows)
        assert np.array_equal(Xd.cpu().numpy(), Xh)
        assert np.array_equal(yd.cpu().numpy(), yh)


# ---------------------------------------------------------------- a2 Gram
@pytest.mark.parametrize("p", [1, 2, 7, 20, 31, 100, 127, 200, 247, 248, 300, 513])
def test_gram_integer_design_bit_exact(ctx, p):
    from paper_1801_09661_b200 import oem_gram
    n = 1000 + 37  # several stages and a ragged tail
    X, y = int_design(p, n, p)
    ldx = p + (p & 1)
    Xp = np.zeros((n, ldx))
    Xp[:, :p] = X
    Xd = to_dev(Xp)[:, :p]
    G, c, yy, nt = oem_gram(ctx, Xd, to_dev(y))
    Go, co, yyo = orc.gram(X, y)
    assert nt == n
    assert np.array_equal(G.cpu().numpy(), Go)
    assert np.array_equal(c.cpu().numpy(), co)
    assert float(yy) == yyo


@pytest.mark.parametrize("p,n", [(1024, 301), (2047, 157), (4095, 67)])
def test_gram_wide_p_bit_exact(ctx, p, n):
    """Two-panel plans far wider than any config (8 to 32 panels, 36 to 528 tile types, a ragged
    last panel): integer designs, bit-exact against the oracle, plain and fold passes."""
    from paper_1801_09661_b200 import oem_gram, oem_gram_folds
    X, y = int_design(p + n, n, p)
    ldx = p + (p & 1)
    Xp = np.zeros((n, ldx))
    Xp[:, :p] = X
    Xd = to_dev(Xp)[:, :p]
    G, c, yy, nt = oem_gram(ctx, Xd, to_dev(y))
    Go, co, yyo = orc.gram(X, y)
    assert nt == n and np.array_equal(G.cpu().numpy(), Go) and np.array_equal(c.cpu().numpy(), co)
    assert float(yy) == yyo
    if p <= 2047:
        Gk, ck, yyk, cnt = oem_gram_folds(ctx, Xd, to_dev(y), 3, row_offset=2)
        Gf, cf, yyf, cntf = orc.gram_folds(X, y, 3, row_offset=2)
        assert list(cnt) == list(cntf)
        assert np.array_equal(Gk.cpu().numpy(), Gf) and np.array_equal(ck.cpu().numpy(), cf)


@pytest.mark.parametrize("name,n", [("cfg1", 1000), ("cfg2", 30011), ("cfg3", 4099), ("cfg4", 2053),
                                    ("cfg5", 10007)])
def test_gram_configs_parity(ctx, name, n):
    from paper_1801_09661_b200 import oem_gram
    cfg = CONFIGS[name].with_n(n)
    bt = dg.beta(cfg.spec, cfg.explicit_beta)
    Xd, yd = device_rows(cfg.spec, bt)
    G, c, yy, nt = oem_gram(ctx, Xd, yd)
    X, y = dg.rows_host(cfg.spec, bt)
    Go, co, yyo = orc.gram(X, y)
    assert scale_err(G.cpu().numpy(), Go) <= 1e-12
    assert xty_err(c.cpu().numpy(), co, Go, yyo) <= 1e-12
    assert abs(float(yy) - yyo) <= 1e-12 * yyo
    # symmetric output, both triangles
    Gh = G.cpu().numpy()
    assert np.array_equal(Gh, Gh.T)


def test_gram_full_size_cfg2(ctx):
    """Full BASELINE size (n = 1e6, p = 100), in the launch configuration bench.py times."""
    from paper_1801_09661_b200 import oem_gram
    cfg = CONFIGS["cfg2"]
    bt = dg.beta(cfg.spec)
    Xd, yd = device_rows(cfg.spec, bt)
    G, c, yy, nt = oem_gram(ctx, Xd, yd)
    acc = orc.GramAccumulator(cfg.p)
    for r in range(0, cfg.n, 250_000):
        X, y = dg.rows_host(cfg.spec, bt, r, 250_000)
        acc.add(X, y)
    Go, co, yyo = acc.result()
    assert scale_err(G.cpu().numpy(), Go) <= 1e-12
    assert xty_err(c.cpu().numpy(), co, Go, yyo) <= 1e-12


def test_gram_full_n_column_subset_cfg4(ctx):
    """cfg4 at full n = 1e7 (80 GB resident), in bench.py's launch configuration: a 32 x 32
    sub-Gram over four column blocks in four different 128-column panels (diagonal and
    off-diagonal panel pairs, 528 distinct entries), X^T y and the f3 column sums on those columns,
    against the oracle's sums over all 1e7 rows (gpu_util.cfg4_oracle_sample)."""
    from paper_1801_09661_b200 import oem_gram, oem_gram_moments, oem_gram_sums
    cfg = CONFIGS["cfg4"]
    bt = dg.beta(cfg.spec)
    Xd, yd = device_rows(cfg.spec, bt)
    G, c, yy, nt = oem_gram(ctx, Xd, yd)
    xs, ysum = oem_gram_moments(ctx, Xd, yd, 1, 0)   # f3 column sums at full size, same launch shape
    G1, c1, yy1, xs1, ys1, nt1 = oem_gram_sums(ctx, Xd, yd)   # the same in one pass over [X | y | 1]
    del Xd
    torch.cuda.empty_cache()
    idx, Go, co, yyo, xso, xabs = cfg4_oracle_sample()
    assert np.max(np.abs(xs[0].cpu().numpy()[idx] - xso) / xabs) <= 1e-12
    assert nt1 == nt and np.max(np.abs(xs1.cpu().numpy()[idx] - xso) / xabs) <= 1e-12
    G1h = G1.cpu().numpy()
    assert scale_err(G1h[np.ix_(idx, idx)], Go) <= 1e-12
    assert xty_err(c1.cpu().numpy()[idx], co, Go, yyo) <= 1e-12 and abs(float(yy1) - yyo) <= 1e-12 * yyo
    del G1h
    Gh = G.cpu().numpy()
    assert scale_err(Gh[np.ix_(idx, idx)], Go) <= 1e-12
    assert xty_err(c.cpu().numpy()[idx], co, Go, yyo) <= 1e-12
    assert abs(float(yy) - yyo) <= 1e-12 * yyo
    # property at full size: G/n close to the population covariance (block 0.4)
    grp = np.arange(cfg.p) // 10
    S = np.where(grp[:, None] == grp[None, :], 0.4, 0.0) + 0.6 * np.eye(cfg.p)
    assert np.max(np.abs(Gh / cfg.n - S)) < 6 / np.sqrt(cfg.n) * 3


def test_gram_folds_full_size_cfg3(ctx):
    """cfg3 at full size (n = 1e7, p = 500, K = 10 folds, 40 GB resident), in the launch
    configuration bench.py times: the leading 16x16 block of every fold Gram against the oracle's
    fold sums over all 1e7 rows (host generator, those columns only: y would need every column,
    and X^T y per fold is checked at the smaller sizes of test_gram_folds_cfg3_parity)."""
    from paper_1801_09661_b200 import oem_gram_folds
    cfg = CONFIGS["cfg3"]
    bt = dg.beta(cfg.spec)
    Xd, yd = device_rows(cfg.spec, bt)
    Gk, ck, yyk, cnt = oem_gram_folds(ctx, Xd, yd, cfg.folds)
    del Xd
    torch.cuda.empty_cache()
    m, K = 16, cfg.folds
    Gs = np.zeros((K, m, m))
    for r in range(0, cfg.n, 1_000_000):
        X, _ = dg.rows_host(cfg.spec, bt, r, 1_000_000, 0, m, want_y=False)
        G1, _, _, _ = orc.gram_folds(X, np.zeros(X.shape[0]), K, row_offset=r)
        Gs += G1
    Gh = Gk.cpu().numpy()
    for k in range(K):
        assert scale_err(Gh[k, :m, :m], Gs[k]) <= 1e-12
    assert list(cnt) == [cfg.n // K] * K


def test_weighted_full_size_cfg5(ctx):
    """cfg5's weighted pass at full size (n = 5e6, p = 200, 8 GB resident) at a nonzero beta,
    against the oracle's compensated weighted Gram accumulated over 1e6-row blocks."""
    from paper_1801_09661_b200 import oem_gram_weighted
    cfg = CONFIGS["cfg5"]
    bt = dg.beta(cfg.spec)
    Xd, yd = device_rows(cfg.spec, bt)
    beta = 0.5 * bt + 0.01
    Gw, cw, sc = oem_gram_weighted(ctx, Xd, yd, to_dev(beta))
    from paper_1801_09661_b200 import oem_logit_grad
    g, ll = oem_logit_grad(ctx, Xd, yd, to_dev(beta))   # f1 gradient pass at full size
    del Xd
    torch.cuda.empty_cache()
    Go = np.zeros((cfg.p, cfg.p)); co = np.zeros(cfg.p); so = np.zeros(2); szz = 0.0
    go = np.zeros(cfg.p); llo = 0.0; cond = np.zeros(cfg.p); llc = 0.0
    for r in range(0, cfg.n, 1_000_000):
        X, y = dg.rows_host(cfg.spec, bt, r, 1_000_000)
        G1, c1, s1 = orc.gram_weighted(X, y, beta)
        Go += G1; co += c1; so += s1
        g1, l1 = orc.logit_grad(X, y, beta)
        go += g1; llo += l1
        eta1 = X @ beta
        cond += np.abs(X).T @ np.abs(y - 1 / (1 + np.exp(-eta1)))
        llc += np.sum(np.abs(y * eta1) + np.logaddexp(0, eta1))
        eta = X @ beta
        mu = np.clip(1 / (1 + np.exp(-eta)), 1e-5, 1 - 1e-5)
        w = mu * (1 - mu)
        szz += np.sum(w * (eta + (y - mu) / w) ** 2)
    assert scale_err(Gw.cpu().numpy(), Go) <= 1e-12
    # scale-aware for the augmented column: sqrt(Gw_jj * sum w z^2) (R#32 applied to [X | z])
    assert np.max(np.abs(cw.cpu().numpy() - co) / np.sqrt(np.diag(Go) * szz)) <= 1e-12
    assert abs(float(sc[0]) - so[0]) <= 1e-12 * so[0]
    assert abs(float(sc[1]) - so[1]) <= 1e-12 * abs(so[1])
    assert np.max(np.abs(g.cpu().numpy() - go) / cond) <= 1e-12
    assert abs(float(ll) - llo) <= 1e-12 * llc


def test_gram_edge_cases(ctx):
    from paper_1801_09661_b200 import OemError, oem_gram
    # n = 0: zero statistics
    X = torch.zeros((0, 4), dtype=torch.float64, device="cuda")
    y = torch.zeros(0, dtype=torch.float64, device="cuda")
    G, c, yy, nt = oem_gram(ctx, X, y)
    assert nt == 0 and not G.any() and not c.any() and float(yy) == 0
    # n = 1
    X1 = to_dev(np.array([[1.0, 2.0, 3.0, 4.0]]))
    G, c, yy, nt = oem_gram(ctx, X1, to_dev(np.array([2.0])))
    assert np.array_equal(G.cpu().numpy(), np.outer([1, 2, 3, 4], [1, 2, 3, 4]))
    assert np.array_equal(c.cpu().numpy(), [2, 4, 6, 8])
    # odd ldx -> alignment error from the boundary
    Xo = torch.zeros((10, 5), dtype=torch.float64, device="cuda")
    with pytest.raises(OemError) as e:
        oem_gram(ctx, Xo, torch.zeros(10, dtype=torch.float64, device="cuda"))
    assert e.value.status == "OEM_ERR_ALIGN"


def test_gram_deterministic(ctx):
    from paper_1801_09661_b200 import oem_gram
    cfg = CONFIGS["cfg3"].with_n(20000)
    bt = dg.beta(cfg.spec)
    Xd, yd = device_rows(cfg.spec, bt)
    a = oem_gram(ctx, Xd, yd)
    b = oem_gram(ctx, Xd, yd)
    assert torch.equal(a[0], b[0]) and torch.equal(a[1], b[1])


def test_logical_shards_sum(ctx):
    """Row sharding: per-shard Grams summed on the host equal the full Gram
    (integer design: exactly)."""
    from paper_1801_09661_b200 import oem_gram
    X, y = int_design(5, 4000, 36)
    Xd, yd = to_dev(X), to_dev(y)
    full = oem_gram(ctx, Xd, yd)[0].cpu().numpy()
    parts = [oem_gram(ctx, Xd[r:r + 500], yd[r:r + 500])[0].cpu().numpy() for r in range(0, 4000, 500)]
    assert np.array_equal(sum(parts), full)


# ---------------------------------------------------------------- a3 fold Grams
@pytest.mark.parametrize("p,K,n,off", [(20, 10, 1000, 0), (100, 10, 20037, 3), (129, 3, 999, 1),
                                       (500, 10, 3001, 0), (7, 1, 100, 0), (5, 2, 64, 5)])
def test_gram_folds_integer_bit_exact(ctx, p, K, n, off):
    from paper_1801_09661_b200 import oem_gram_folds
    X, y = int_design(p * 7 + K, n, p)
    ldx = p + (p & 1)
    Xp = np.zeros((n, ldx))
    Xp[:, :p] = X
    Gk, ck, yyk, cnt = oem_gram_folds(ctx, to_dev(Xp)[:, :p], to_dev(y), K, row_offset=off)
    Go, co, yyo, cnto = orc.gram_folds(X, y, K, row_offset=off)
    assert list(cnt) == list(cnto)
    assert np.array_equal(Gk.cpu().numpy(), Go)
    assert np.array_equal(ck.cpu().numpy(), co)
    assert np.array_equal(yyk.cpu().numpy(), yyo)


@pytest.mark.parametrize("lpt,waves", [("0", "384"), ("0", "1"), ("1", "384"), ("1", "3")])
def test_gram_schedule_overrides_bit_exact(monkeypatch, lpt, waves):
    """The work-item schedule overrides (OEM_GRAM_LPT, OEM_GRAM_WAVES; the L2-traffic study in
    profiles/cfg4_l2_schedule_r01.md) change only the order of the split-n sums: two-panel plain
    and fold passes on integer designs stay bit-exact against the oracle."""
    from paper_1801_09661_b200 import Context, oem_gram, oem_gram_folds
    monkeypatch.setenv("OEM_GRAM_LPT", lpt)
    monkeypatch.setenv("OEM_GRAM_WAVES", waves)
    c = Context(0)  # plans are cached per context: a fresh one reads the overrides
    try:
        p, n = 300, 8000 + 19
        X, y = int_design(41, n, p)
        Xd = to_dev(X)
        G, cc, yy, nt = oem_gram(c, Xd, to_dev(y))
        Go, co, yyo = orc.gram(X, y)
        assert np.array_equal(G.cpu().numpy(), Go) and np.array_equal(cc.cpu().numpy(), co) and float(yy) == yyo
        Gk, ck, yyk, cnt = oem_gram_folds(c, Xd, to_dev(y), 4, row_offset=1)
        Gf, cf, yyf, cntf = orc.gram_folds(X, y, 4, row_offset=1)
        assert list(cnt) == list(cntf)
        assert np.array_equal(Gk.cpu().numpy(), Gf) and np.array_equal(ck.cpu().numpy(), cf)
    finally:
        c.close()


def test_gram_folds_cfg3_parity(ctx):
    from paper_1801_09661_b200 import oem_gram_folds
    cfg = CONFIGS["cfg3"].with_n(10_013)
    bt = dg.beta(cfg.spec)
    Xd, yd = device_rows(cfg.spec, bt)
    Gk, ck, yyk, cnt = oem_gram_folds(ctx, Xd, yd, 10)
    X, y = dg.rows_host(cfg.spec, bt)
    Go, co, yyo, _ = orc.gram_folds(X, y, 10)
    for k in range(10):
        assert scale_err(Gk[k].cpu().numpy(), Go[k]) <= 1e-12
        assert xty_err(ck[k].cpu().numpy(), co[k], Go[k], yyo[k]) <= 1e-12


def test_empty_fold_error(ctx):
    from paper_1801_09661_b200 import OemError, oem_gram_folds
    X, y = int_design(1, 5, 4)
    with pytest.raises(OemError) as e:
        oem_gram_folds(ctx, to_dev(X), to_dev(y), 7)
    assert e.value.status == "OEM_ERR_EMPTY_FOLD"


# ---------------------------------------------------------------- a4 weighted Gram
def test_weighted_zero_beta_exact(ctx):
    from paper_1801_09661_b200 import oem_gram_weighted
    X, _ = int_design(9, 3001, 30)
    y = (np.random.default_rng(9).random(3001) < 0.3).astype(float)
    Gw, cw, sc = oem_gram_weighted(ctx, to_dev(X), to_dev(y), torch.zeros(30, dtype=torch.float64, device="cuda"))
    Go, co, sco = orc.gram_weighted(X, y, np.zeros(30))
    assert np.array_equal(Gw.cpu().numpy(), Go)      # w = 1/4 exactly, integer sums
    assert np.array_equal(cw.cpu().numpy(), co)      # w z = y - 1/2 exactly
    assert float(sc[0]) == sco[0]
    assert abs(float(sc[1]) - sco[1]) <= 1e-12 * abs(sco[1])


@pytest.mark.parametrize("n,p", [(10007, 200), (5000, 37), (777, 247)])
def test_weighted_parity(ctx, n, p):
    from paper_1801_09661_b200 import oem_gram_weighted
    cfg = CONFIGS["cfg5"]
    spec = cfg.spec.replace(n=n, p=p, nnz=min(20, p))
    bt = dg.beta(spec)
    Xd, yd = device_rows(spec, bt)
    X, y = dg.rows_host(spec, bt)
    beta = 0.7 * bt + 0.05
    Gw, cw, sc = oem_gram_weighted(ctx, Xd, yd, to_dev(beta))
    Go, co, sco = orc.gram_weighted(X, y, beta)
    assert scale_err(Gw.cpu().numpy(), Go) <= 1e-12
    # scale-aware for the augmented column: sqrt(Gw_jj * sum w z^2) (R#32 applied to [X | z])
    eta = X @ beta
    mu = np.clip(1 / (1 + np.exp(-eta)), 1e-5, 1 - 1e-5)
    w = mu * (1 - mu)
    szz = np.sum(w * (eta + (y - mu) / w) ** 2)
    assert np.max(np.abs(cw.cpu().numpy() - co) / np.sqrt(np.diag(Go) * szz)) <= 1e-12
    assert abs(float(sc[0]) - sco[0]) <= 1e-12 * sco[0]
    assert abs(float(sc[1]) - sco[1]) <= 1e-12 * abs(sco[1])


def test_weighted_extreme_eta_and_no_scalars(ctx):
    """eta spanning [-800, 800] (exp(-eta) overflows below -709, mu clamps at both ends) against
    the oracle; then scalars=False must give bit-identical G_w and X^T W z (the flag only drops
    the sum of w and the log-likelihood)."""
    from paper_1801_09661_b200 import oem_gram_weighted
    rng = np.random.default_rng(17)
    n, p = 4099, 24
    X = rng.standard_normal((n, p))
    X[:, 0] = np.linspace(-1.0, 1.0, n)          # eta = 800 x_0 + small terms
    y = (rng.random(n) < 0.5).astype(float)
    beta = np.zeros(p)
    beta[0] = 800.0
    beta[1:4] = [0.3, -0.2, 0.1]
    Xd, yd, bd = to_dev(X), to_dev(y), to_dev(beta)
    Gw, cw, sc = oem_gram_weighted(ctx, Xd, yd, bd)
    Go, co, sco = orc.gram_weighted(X, y, beta)
    assert scale_err(Gw.cpu().numpy(), Go) <= 1e-12
    eta = X @ beta
    mu = np.clip(1 / (1 + np.exp(-eta)), 1e-5, 1 - 1e-5)
    w = mu * (1 - mu)
    szz = np.sum(w * (eta + (y - mu) / w) ** 2)
    assert np.max(np.abs(cw.cpu().numpy() - co) / np.sqrt(np.diag(Go) * szz)) <= 1e-12
    assert abs(float(sc[0]) - sco[0]) <= 1e-12 * sco[0]
    assert abs(float(sc[1]) - sco[1]) <= 1e-12 * abs(sco[1])
    Gn, cn, sn = oem_gram_weighted(ctx, Xd, yd, bd, scalars=False)
    assert sn is None
    assert torch.equal(Gn, Gw) and torch.equal(cn, cw)


@pytest.mark.parametrize("n,p", [(6001, 248), (4001, 255), (3003, 500), (2011, 1000), (1001, 1031)])
def test_weighted_two_panel_parity(ctx, n, p):
    """p > 247 (two-panel plans; the paper's §6.3 logistic study varies p up to 500):
    the (w, z) pre-pass plus the WZ contraction against the oracle's weighted Gram (R#25), with
    the scalars; ragged tails (n not a multiple of 32) and a last panel holding the augmented
    column at every offset class."""
    from paper_1801_09661_b200 import oem_gram_weighted
    spec = CONFIGS["cfg5"].spec.replace(n=n, p=p, nnz=min(20, p))
    bt = dg.beta(spec)
    Xd, yd = device_rows(spec, bt)
    X, y = dg.rows_host(spec, bt)
    beta = 0.7 * bt + 0.02 * np.cos(np.arange(p))
    Gw, cw, sc = oem_gram_weighted(ctx, Xd, yd, to_dev(beta))
    Go, co, sco = orc.gram_weighted(X, y, beta)
    assert scale_err(Gw.cpu().numpy(), Go) <= 1e-12
    eta = X @ beta
    mu = np.clip(1 / (1 + np.exp(-eta)), 1e-5, 1 - 1e-5)
    w = mu * (1 - mu)
    szz = np.sum(w * (eta + (y - mu) / w) ** 2)
    assert np.max(np.abs(cw.cpu().numpy() - co) / np.sqrt(np.diag(Go) * szz)) <= 1e-12
    assert abs(float(sc[0]) - sco[0]) <= 1e-12 * sco[0]
    assert abs(float(sc[1]) - sco[1]) <= 1e-12 * abs(sco[1])
    Gn, cn, sn = oem_gram_weighted(ctx, Xd, yd, to_dev(beta), scalars=False)
    assert torch.equal(Gn, Gw) and torch.equal(cn, cw)


def test_weighted_two_panel_zero_beta_exact(ctx):
    """beta = 0: w = 1/4 and w z = y - 1/2 exactly, so on integer data G_w = X^T X / 4 and
    X^T W z = X^T (y - 1/2) are exact in any summation order: bit-exact at p = 300."""
    from paper_1801_09661_b200 import oem_gram_weighted
    X, _ = int_design(11, 2049, 300)
    y = (np.random.default_rng(11).random(2049) < 0.4).astype(float)
    Gw, cw, sc = oem_gram_weighted(ctx, to_dev(X), to_dev(y), torch.zeros(300, dtype=torch.float64, device="cuda"))
    Go, co, sco = orc.gram_weighted(X, y, np.zeros(300))
    assert np.array_equal(Gw.cpu().numpy(), Go)
    assert np.array_equal(cw.cpu().numpy(), co)
    assert float(sc[0]) == sco[0]


@pytest.mark.parametrize("sched", ["OEM_GRAM_ORDERED=1", "OEM_GRAM_LPT=0 OEM_GRAM_WAVES=384"])
def test_alternative_two_panel_schedules(sched, monkeypatch):
    """The DRAM-traffic schedules of profiles/cfg4_l2_schedule_r02.md (ordered in-kernel running
    sums; short segment-major segments): integer data stays bit-exact against the oracle in the
    plain pass, and the weighted (WZ) pass matches the oracle at 1e-12, with many segments."""
    from paper_1801_09661_b200 import Context, oem_gram, oem_gram_weighted
    for kv in sched.split():
        k, v = kv.split("=")
        monkeypatch.setenv(k, v)
    c = Context(0)   # fresh context: plans are built (and the schedule read) per context
    try:
        X, y = int_design(21, 70_001, 300)
        G, xty, yy, nt = oem_gram(c, to_dev(X), to_dev(y))
        Go, co, yyo = orc.gram(X, y)
        assert np.array_equal(G.cpu().numpy(), Go) and np.array_equal(xty.cpu().numpy(), co) and float(yy) == yyo
        spec = CONFIGS["cfg5"].spec.replace(n=30_011, p=260, nnz=10)
        bt = dg.beta(spec)
        Xd, yd = device_rows(spec, bt)
        Xh, yh = dg.rows_host(spec, bt)
        beta = 0.6 * bt
        Gw, cw, sc = oem_gram_weighted(c, Xd, yd, to_dev(beta))
        Gwo, cwo, sco = orc.gram_weighted(Xh, yh, beta)
        assert scale_err(Gw.cpu().numpy(), Gwo) <= 1e-12
        assert abs(float(sc[0]) - sco[0]) <= 1e-12 * sco[0]
    finally:
        c.close()
