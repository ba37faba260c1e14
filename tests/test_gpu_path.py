"""GPU parity for a6-a10 (normalise, d, lambda grid, OEM paths) through oem_fit_path.

The oracle runs the same algorithm with the GPU's d (paths depend on d for MCP/SCAD, DESIGN.md
R#30), the same lambda grid, tol and maxit; the bar is max |beta_gpu - beta_oracle| <= 1e-8 at
every lambda (north star), equal converged flags, and d within [lambda_1, 1.01 lambda_1]."""
import numpy as np
import pytest

import datagen as dg
import oracle as orc
from datagen.configs import CONFIGS, groups_of
from gpu_util import device_rows

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")

TOL_BETA = 1e-8


@pytest.fixture(scope="module")
def ctx():
    from paper_1801_09661_b200 import Context
    c = Context(0)
    yield c
    c.close()


def host_problem(cfg):
    bt = dg.beta(cfg.spec, cfg.explicit_beta)
    X, y = dg.rows_host(cfg.spec, bt)
    return bt, X, y


def check_d(d, Go, n, G_gpu=None):
    """a7 against the oracle (R#5): d_gpu equals the oracle's own rule on the oracle's statistics
    (up to the Gram's own 1e-12 parity), equals it on the GPU's statistics to 1e-12, and lies in
    [lambda_1, p^(2^-12) lambda_1] (the trace bound's guarantee), lambda_1 from numpy."""
    Gn = np.asarray(Go, dtype=float) / n
    d_ref = orc.d_rule(Gn)[0]
    assert abs(d - d_ref) <= 1e-11 * d_ref, (d, d_ref)
    if G_gpu is not None:
        d_same = orc.d_rule(np.asarray(G_gpu, dtype=float) / n)[0]
        assert abs(d - d_same) <= 1e-12 * d_same, (d, d_same)
    p = Gn.shape[0]
    lam1 = np.linalg.eigvalsh(Gn)[-1]
    assert lam1 * (1 - 1e-12) <= d <= lam1 * p ** (1 / 4096) * (1 + 1e-10) + 1e-300, (d, lam1)
    return d_ref


def check_fit(fit, Go, co, n, penalties, nlambda, unit=0, group=None, lambdas=None, w=None, G_gpu=None):
    """Every output of one unit against the oracle's OWN pipeline on the oracle's statistics:
    its d (R#5), its lambda grid (R#14-16) and its path solve (O6)."""
    d = float(fit.d[unit])
    Gn = Go / n
    d_ref = check_d(d, Go, n, G_gpu)
    for q, (fam, gamma, alpha) in enumerate(penalties):
        if lambdas is None:
            lmax = orc.lambda_max(fam, co / n, w=w, group=group, alpha=alpha)
            lam = orc.lambda_grid(lmax, nlambda)
        else:
            lam = np.asarray(lambdas, dtype=float)
        lg = fit.lam[unit, q].cpu().numpy()
        assert np.max(np.abs(lg - lam) / lam.clip(min=1e-300)) < 1e-13
        B, it, cv = orc.oem_path(Gn, co / n, d_ref, fam, lam, gamma, alpha, w=w, group=group)
        Bg = fit.beta[unit, q].cpu().numpy()
        err = np.max(np.abs(Bg - B))
        assert err <= TOL_BETA, (fam, err)
        assert np.array_equal(fit.conv[unit, q].cpu().numpy().astype(bool), cv)
        itg = fit.iters[unit, q].cpu().numpy()
        assert np.max(np.abs(itg - it)) <= max(2, 0.02 * it.max()), (itg - it)


def test_cfg1_lasso_path(ctx):
    from paper_1801_09661_b200 import oem_fit_path, oem_gram
    cfg = CONFIGS["cfg1"]
    bt, X, y = host_problem(cfg)
    G, c, yy, n = oem_gram(ctx, torch.from_numpy(X).cuda(), torch.from_numpy(y).cuda())
    fit = oem_fit_path(ctx, G, c, [n], cfg.penalties, nlambda=cfg.nlambda)
    Go, co, _ = orc.gram(X, y)
    check_fit(fit, Go, co, n, cfg.penalties, cfg.nlambda, G_gpu=G.cpu().numpy())
    # lambda_max nulls everything, the smallest lambda recovers the support
    assert not fit.beta[0, 0, 0].any()
    assert (fit.beta[0, 0, -1].abs() > 0.1).sum() >= 5


@pytest.mark.parametrize("n", [30011, 1_000_000])
def test_cfg2_three_penalties(ctx, n):
    """cfg2: lasso + MCP(3) + SCAD(3.7) paths of 100 lambda on one Gram, computed together."""
    from paper_1801_09661_b200 import oem_fit_path, oem_gram
    cfg = CONFIGS["cfg2"].with_n(n)
    bt = dg.beta(cfg.spec)
    Xd, yd = device_rows(cfg.spec, bt)
    G, c, yy, nn = oem_gram(ctx, Xd, yd)
    fit = oem_fit_path(ctx, G, c, [nn], cfg.penalties, nlambda=cfg.nlambda)
    acc = orc.GramAccumulator(cfg.p)
    for r in range(0, n, 250_000):
        X, y = dg.rows_host(cfg.spec, bt, r, min(250_000, n - r))
        acc.add(X, y)
    Go, co, _ = acc.result()
    check_fit(fit, Go, co, n, cfg.penalties, cfg.nlambda, G_gpu=G.cpu().numpy())
    # multi-penalty independence: lasso alone == lasso inside the batch, bit for bit
    fit1 = oem_fit_path(ctx, G, c, [nn], cfg.penalties[:1], nlambda=cfg.nlambda, d_in=[float(fit.d[0])])
    assert torch.equal(fit1.beta[0, 0], fit.beta[0, 0])


def test_cfg3_fold_mode(ctx):
    """cfg3 shape: 10 fold Grams in one pass, then full fit + 10 complement fits (fold_mode),
    shared lambda grid from the full data, per-unit d (R#20-22)."""
    from paper_1801_09661_b200 import oem_fit_path, oem_gram_folds
    cfg = CONFIGS["cfg3"].with_n(12_007)
    bt = dg.beta(cfg.spec)
    Xd, yd = device_rows(cfg.spec, bt)
    Gk, ck, yyk, cnt = oem_gram_folds(ctx, Xd, yd, 10)
    L = 20
    fit = oem_fit_path(ctx, Gk, ck, cnt, cfg.penalties, nlambda=L, fold_mode=True)
    X, y = dg.rows_host(cfg.spec, bt)
    Gf, cf, _, cnto = orc.gram_folds(X, y, 10)
    Gm, cm = orc.fold_complements(Gf, cf)
    n = X.shape[0]
    lmax0 = orc.lambda_max("lasso", cf.sum(0) / n)
    lam = orc.lambda_grid(lmax0, L)
    check_fit(fit, Gf.sum(0), cf.sum(0), n, cfg.penalties, L, unit=0, lambdas=lam)
    for k in range(10):
        check_fit(fit, Gm[k], cm[k], n - cnto[k], cfg.penalties, L, unit=k + 1, lambdas=lam)


def test_cfg3_full_size_cv_paths(ctx):
    """cfg3 at full size in bench.py's launch configuration: the K = 10 fold Grams of all n = 1e7
    rows (40 GB resident) in one pass, then the full-data fit and the 10 complement fits (fold
    mode, 100 lambda, lasso) in one launch; every unit checked against the oracle's path solve on
    the same statistics (the oracle forms the complements as sums of the other folds)."""
    from paper_1801_09661_b200 import oem_fit_path, oem_gram_folds
    cfg = CONFIGS["cfg3"]
    bt = dg.beta(cfg.spec)
    Xd, yd = device_rows(cfg.spec, bt)
    Gk, ck, yyk, cnt = oem_gram_folds(ctx, Xd, yd, cfg.folds)
    del Xd, yd
    torch.cuda.empty_cache()
    fit = oem_fit_path(ctx, Gk, ck, cnt, cfg.penalties, nlambda=cfg.nlambda, fold_mode=True)
    Gf, cf = Gk.cpu().numpy(), ck.cpu().numpy()
    Gm, cm = orc.fold_complements(Gf, cf)
    n = int(sum(cnt))
    lam = orc.lambda_grid(orc.lambda_max("lasso", cf.sum(0) / n), cfg.nlambda)
    check_fit(fit, Gf.sum(0), cf.sum(0), n, cfg.penalties, cfg.nlambda, unit=0, lambdas=lam)
    for k in range(cfg.folds):
        check_fit(fit, Gm[k], cm[k], n - cnt[k], cfg.penalties, cfg.nlambda, unit=k + 1, lambdas=lam)


def test_cfg4_group_lasso_and_enet(ctx):
    """cfg4 shape (p = 1000, 100 groups of 10, block-equicorrelated design): group lasso and
    EN(0.5) together, first 12 lambda of the 50-point grid (oracle time)."""
    from paper_1801_09661_b200 import oem_fit_path, oem_gram
    cfg = CONFIGS["cfg4"].with_n(20_000)
    bt = dg.beta(cfg.spec)
    Xd, yd = device_rows(cfg.spec, bt)
    G, c, yy, n = oem_gram(ctx, Xd, yd)
    grp = groups_of(cfg)
    X, y = dg.rows_host(cfg.spec, bt)
    Go, co, _ = orc.gram(X, y)
    Ls = []
    for fam, gamma, alpha in cfg.penalties:
        lmax = orc.lambda_max(fam, co / n, group=grp if fam.startswith("grp") else None, alpha=alpha)
        Ls.append(orc.lambda_grid(lmax, cfg.nlambda)[:12])
    for q, pen in enumerate(cfg.penalties):
        fit = oem_fit_path(ctx, G, c, [n], [pen], lambdas=Ls[q], group=grp, ngroups=100)
        check_fit(fit, Go, co, n, [pen], 12, group=grp if pen[0].startswith("grp") else None, lambdas=Ls[q])
    # both penalties in one launch agree with the separate launches
    both = oem_fit_path(ctx, G, c, [n], cfg.penalties, lambdas=Ls[0], group=grp, ngroups=100)
    one = oem_fit_path(ctx, G, c, [n], cfg.penalties[:1], lambdas=Ls[0], group=grp, ngroups=100,
                       d_in=[float(both.d[0])])
    assert torch.equal(both.beta[0, 0], one.beta[0, 0])


def test_cfg4_full_size_paths(ctx):
    """cfg4 at full size in bench.py's launch configuration: the Gram of all n = 1e7 rows (80 GB
    resident), then both 50-lambda paths (group lasso, EN(0.5)) in one launch of the grid-wide
    split solver, each checked against the oracle's path solve on the same Gram (host copy) at the
    GPU's d: lambda grid, every beta, converged flags and iteration counts."""
    from paper_1801_09661_b200 import oem_fit_path, oem_gram
    cfg = CONFIGS["cfg4"]
    bt = dg.beta(cfg.spec)
    Xd, yd = device_rows(cfg.spec, bt)
    G, c, yy, n = oem_gram(ctx, Xd, yd)
    del Xd, yd
    torch.cuda.empty_cache()
    grp = groups_of(cfg)
    fit = oem_fit_path(ctx, G, c, [n], cfg.penalties, nlambda=cfg.nlambda, group=grp, ngroups=100)
    Gh, ch = G.cpu().numpy(), c.cpu().numpy()
    d = float(fit.d[0])
    check_d(d, Gh, n, Gh)
    for q, (fam, gamma, alpha) in enumerate(cfg.penalties):
        g = grp if fam.startswith("grp") else None
        lam = orc.lambda_grid(orc.lambda_max(fam, ch / n, group=g, alpha=alpha), cfg.nlambda)
        lg = fit.lam[0, q].cpu().numpy()
        assert np.max(np.abs(lg - lam) / lam) < 1e-13
        B, it, cv = orc.oem_path(Gh / n, ch / n, d, fam, lg, gamma, alpha, group=g)
        assert np.max(np.abs(fit.beta[0, q].cpu().numpy() - B)) <= TOL_BETA, fam
        assert np.array_equal(fit.conv[0, q].cpu().numpy().astype(bool), cv)
        itg = fit.iters[0, q].cpu().numpy()
        assert np.max(np.abs(itg - it)) <= max(2, 0.02 * it.max()), (fam, itg - it)


def test_noncontiguous_groups_and_weights(ctx):
    from paper_1801_09661_b200 import oem_fit_path, oem_gram
    rng = np.random.default_rng(3)
    cfg = CONFIGS["cfg2"].with_n(5000)
    bt = dg.beta(cfg.spec)
    X, y = dg.rows_host(cfg.spec, bt)
    G, c, yy, n = oem_gram(ctx, torch.from_numpy(X).cuda(), torch.from_numpy(y).cuda())
    Go, co, _ = orc.gram(X, y)
    grp = rng.integers(0, 17, size=100).astype(np.int32)
    grp[:17] = np.arange(17)  # every id used
    gw = rng.uniform(0.5, 2.0, 17)
    pens = [("grp_lasso", 0.0, 1.0), ("grp_mcp", 3.0, 1.0), ("grp_scad", 3.7, 1.0)]
    fit = oem_fit_path(ctx, G, c, [n], pens, nlambda=25, group=grp, ngroups=17, grp_w=gw)
    d = float(fit.d[0])
    check_d(d, Go, n)
    for q, (fam, gamma, alpha) in enumerate(pens):
        lg = fit.lam[0, q].cpu().numpy()
        B, it, cv = orc.oem_path(Go / n, co / n, d, fam, lg, gamma, alpha, group=grp, grp_w=gw)
        assert np.max(np.abs(fit.beta[0, q].cpu().numpy() - B)) <= TOL_BETA
    w = torch.from_numpy(rng.uniform(0.0, 2.0, 100)).cuda()
    w[5] = 0.0  # unpenalized coordinate
    pens = [("lasso", 0.0, 1.0), ("enet", 0.0, 0.3), ("scad", 3.7, 1.0)]
    fit = oem_fit_path(ctx, G, c, [n], pens, nlambda=30, var_w=w)
    d = float(fit.d[0])
    check_d(d, Go, n)
    for q, (fam, gamma, alpha) in enumerate(pens):
        lg = fit.lam[0, q].cpu().numpy()
        lmax = orc.lambda_max(fam, co / n, w=w.cpu().numpy(), alpha=alpha)
        assert abs(lg[0] - lmax) <= 1e-13 * lmax
        B, it, cv = orc.oem_path(Go / n, co / n, d, fam, lg, gamma, alpha, w=w.cpu().numpy())
        assert np.max(np.abs(fit.beta[0, q].cpu().numpy() - B)) <= TOL_BETA


def test_lambda_zero_ols_and_warm_start(ctx):
    from paper_1801_09661_b200 import oem_fit_path, oem_gram
    cfg = CONFIGS["cfg1"].with_n(600)
    bt, X, y = host_problem(cfg)
    G, c, yy, n = oem_gram(ctx, torch.from_numpy(X).cuda(), torch.from_numpy(y).cuda())
    fit = oem_fit_path(ctx, G, c, [n], [("lasso", 0, 1), ("mcp", 3, 1)], lambdas=[0.0], tol=1e-14,
                       maxit=200000)
    ols = np.linalg.solve(X.T @ X, X.T @ y)
    for q in range(2):
        assert np.max(np.abs(fit.beta[0, q, 0].cpu().numpy() - ols)) < 1e-10
    # warm start from the solution: one update, converged
    init = fit.beta[:, :, 0, :].clone()
    fit2 = oem_fit_path(ctx, G, c, [n], [("lasso", 0, 1), ("mcp", 3, 1)], lambdas=[0.0], tol=1e-12,
                        beta_init=init, d_in=[float(fit.d[0])])
    assert int(fit2.iters.max()) <= 2


def test_invalid_parameters(ctx):
    from paper_1801_09661_b200 import OemError, oem_fit_path
    G = torch.eye(4, dtype=torch.float64, device="cuda") * 10
    c = torch.ones(4, dtype=torch.float64, device="cuda")
    with pytest.raises(OemError) as e:   # gamma * d = 0.9 * 1 <= 1 (R#8)
        oem_fit_path(ctx, G, c, [10], [("mcp", 1.5, 1.0)], nlambda=5, d_in=[0.5])
    assert e.value.status == "OEM_ERR_INVALID_ARG"
    with pytest.raises(OemError) as e:
        oem_fit_path(ctx, G, c, [10], [("grp_lasso", 0, 1.0)], nlambda=5)
    assert e.value.status == "OEM_ERR_INVALID_ARG"
    Gn = G.clone()
    Gn[1, 1] = float("nan")
    with pytest.raises(OemError) as e:
        oem_fit_path(ctx, Gn, c, [10], [("lasso", 0, 1.0)], nlambda=5, d_in=[2.0])
    assert e.value.status == "OEM_ERR_NONFINITE"


def test_maxit_flag_not_error(ctx):
    from paper_1801_09661_b200 import oem_fit_path, oem_gram
    cfg = CONFIGS["cfg2"].with_n(3000)
    bt, X, y = host_problem(cfg)
    G, c, yy, n = oem_gram(ctx, torch.from_numpy(X).cuda(), torch.from_numpy(y).cuda())
    fit = oem_fit_path(ctx, G, c, [n], [("lasso", 0, 1)], nlambda=10, maxit=3)
    assert int(fit.iters.max()) == 3
    assert not bool(fit.conv[0, 0, -1])
    Go, co, _ = orc.gram(X, y)
    B, it, cv = orc.oem_path(Go / n, co / n, float(fit.d[0]), "lasso", fit.lam[0, 0].cpu().numpy(), maxit=3)
    assert np.max(np.abs(fit.beta[0, 0].cpu().numpy() - B)) <= 1e-12
    assert np.array_equal(fit.iters[0, 0].cpu().numpy(), it)


@pytest.mark.parametrize("p,solver", [(100, None), (100, "cluster"), (120, "global"), (400, None)])
def test_sparse_group_lasso(ctx, p, solver, monkeypatch):
    """f3 sparse group lasso (exact composition R#11, lambda_max R#36) on every
    solver kernel (lean / cluster / global), with non-contiguous groups, group and variable
    weights, against the oracle at the GPU's d and lambda grid."""
    from paper_1801_09661_b200 import oem_fit_path, oem_gram
    if solver:
        monkeypatch.setenv("OEM_PATH_SOLVER", solver)
    rng = np.random.default_rng(p)
    spec = CONFIGS["cfg2"].spec.replace(n=6000, p=p, nnz=min(10, p))
    bt = dg.beta(spec)
    X, y = dg.rows_host(spec, bt)
    Xp = np.zeros((X.shape[0], p + (p & 1)))
    Xp[:, :p] = X
    G, c, yy, n = oem_gram(ctx, torch.from_numpy(Xp).cuda()[:, :p], torch.from_numpy(y).cuda())
    Go, co, _ = orc.gram(X, y)
    ng = p // 8
    grp = rng.integers(0, ng, size=p).astype(np.int32)
    grp[:ng] = np.arange(ng)
    gw = rng.uniform(0.5, 2.0, ng)
    w = rng.uniform(0.5, 1.5, p)
    pens = [("sgl", 0.0, 0.3), ("sgl", 0.0, 0.7), ("grp_lasso", 0.0, 1.0)]
    fit = oem_fit_path(ctx, G, c, [n], pens, nlambda=20, group=grp, ngroups=ng, grp_w=gw,
                       var_w=torch.from_numpy(w).cuda())
    d = float(fit.d[0])
    check_d(d, Go, n)
    for q, (fam, gamma, alpha) in enumerate(pens):
        lg = fit.lam[0, q].cpu().numpy()
        lmax = orc.lambda_max(fam, co / n, w=w, group=grp, ngroups=ng, grp_w=gw, alpha=alpha)
        assert abs(lg[0] - lmax) <= 1e-12 * lmax, (fam, lg[0], lmax)
        B, it, cv = orc.oem_path(Go / n, co / n, d, fam, lg, gamma, alpha, w=w, group=grp, ngroups=ng,
                                 grp_w=gw)
        Bg = fit.beta[0, q].cpu().numpy()
        assert np.max(np.abs(Bg - B)) <= TOL_BETA, (fam, np.max(np.abs(Bg - B)))
        assert np.array_equal(fit.conv[0, q].cpu().numpy().astype(bool), cv)
        assert np.max(np.abs(Bg[0])) <= 1e-12   # lambda_max: null up to the rounding at the root


@pytest.mark.parametrize("p,solver", [(60, None), (60, "cluster"), (60, "global"), (700, None)])
def test_mixed_group_and_coordinate_penalties(ctx, p, solver, monkeypatch):
    """Group and coordinate-wise families fitted in ONE launch (cfg4 runs group lasso + EN
    together): every penalty must match its own oracle path (each family keeps its own M-step)."""
    from paper_1801_09661_b200 import oem_fit_path, oem_gram
    if solver:
        monkeypatch.setenv("OEM_PATH_SOLVER", solver)
    spec = CONFIGS["cfg4"].spec.replace(n=4000, p=p, nnz=2)
    bt = dg.beta(spec)
    X, y = dg.rows_host(spec, bt)
    G, c, yy, n = oem_gram(ctx, torch.from_numpy(X).cuda(), torch.from_numpy(y).cuda())
    Go, co, _ = orc.gram(X, y)
    grp = (np.arange(p) // 10).astype(np.int32)
    pens = [("grp_lasso", 0.0, 1.0), ("enet", 0.0, 0.5), ("mcp", 3.0, 1.0), ("sgl", 0.0, 0.5)]
    fit = oem_fit_path(ctx, G, c, [n], pens, nlambda=12, group=grp, ngroups=p // 10)
    d = float(fit.d[0])
    check_d(d, Go, n)
    for q, (fam, gamma, alpha) in enumerate(pens):
        g = grp if fam in ("grp_lasso", "sgl") else None
        lg = fit.lam[0, q].cpu().numpy()
        lmax = orc.lambda_max(fam, co / n, group=g, ngroups=p // 10 if g is not None else 0, alpha=alpha)
        assert abs(lg[0] - lmax) <= 1e-12 * lmax
        B, it, cv = orc.oem_path(Go / n, co / n, d, fam, lg, gamma, alpha, group=g,
                                 ngroups=p // 10 if g is not None else 0)
        assert np.max(np.abs(fit.beta[0, q].cpu().numpy() - B)) <= TOL_BETA, fam


def test_many_penalties_and_wide_p_fallbacks(ctx):
    """Shapes outside the lean / grid solvers' templates take the fallback kernels: six penalties
    at once (NPT = 8) and p = 1100 (> 1024); both against the oracle."""
    from paper_1801_09661_b200 import oem_fit_path, oem_gram
    spec = CONFIGS["cfg2"].spec.replace(n=3000, p=40, nnz=6)
    bt = dg.beta(spec)
    X, y = dg.rows_host(spec, bt)
    G, c, yy, n = oem_gram(ctx, torch.from_numpy(X).cuda(), torch.from_numpy(y).cuda())
    Go, co, _ = orc.gram(X, y)
    pens = [("lasso", 0.0, 1.0), ("enet", 0.0, 0.3), ("mcp", 3.0, 1.0), ("scad", 3.7, 1.0),
            ("enet", 0.0, 0.8), ("mcp", 5.0, 1.0)]
    fit = oem_fit_path(ctx, G, c, [n], pens, nlambda=15)
    d = float(fit.d[0])
    check_d(d, Go, n)
    for q, (fam, gamma, alpha) in enumerate(pens):
        B, it, cv = orc.oem_path(Go / n, co / n, d, fam, fit.lam[0, q].cpu().numpy(), gamma, alpha)
        assert np.max(np.abs(fit.beta[0, q].cpu().numpy() - B)) <= TOL_BETA, fam
    spec = CONFIGS["cfg4"].spec.replace(n=2500, p=1100, nnz=3)
    bt = dg.beta(spec)
    X, y = dg.rows_host(spec, bt)
    G, c, yy, n = oem_gram(ctx, torch.from_numpy(X).cuda(), torch.from_numpy(y).cuda())
    Go, co, _ = orc.gram(X, y)
    fit = oem_fit_path(ctx, G, c, [n], [("lasso", 0.0, 1.0)], nlambda=6)
    B, it, cv = orc.oem_path(Go / n, co / n, float(fit.d[0]), "lasso", fit.lam[0, 0].cpu().numpy())
    assert np.max(np.abs(fit.beta[0, 0].cpu().numpy() - B)) <= TOL_BETA


@pytest.mark.parametrize("p", [1, 7, 64, 65, 128, 129, 256, 257, 512, 513, 1024])
def test_solver_variant_boundaries(ctx, p):
    """Every solver layout boundary (lean register / shared-memory variants, cluster sizes, the
    grid-wide solver, penalty split) with two units and two penalties, against the oracle."""
    from paper_1801_09661_b200 import oem_fit_path, oem_gram
    spec = CONFIGS["cfg2"].spec.replace(n=1500 + 3 * p, p=p, nnz=min(5, p))
    bt = dg.beta(spec)
    X, y = dg.rows_host(spec, bt)
    Xp = np.zeros((X.shape[0], p + (p & 1)))
    Xp[:, :p] = X
    Xd = torch.from_numpy(Xp).cuda()[:, :p]
    yd = torch.from_numpy(y).cuda()
    h = (X.shape[0] // 2) & ~1   # 16-byte aligned second block (TMA)
    G0, c0, _, n0 = oem_gram(ctx, Xd[:h], yd[:h])
    G1, c1, _, n1 = oem_gram(ctx, Xd[h:], yd[h:])
    G = torch.stack([G0, G1]); c = torch.stack([c0, c1])
    pens = [("lasso", 0.0, 1.0), ("mcp", 3.0, 1.0)]
    fit = oem_fit_path(ctx, G, c, [n0, n1], pens, nlambda=6)
    for u, (lo, hi, nn) in enumerate([(0, h, n0), (h, X.shape[0], n1)]):
        Go, co, _ = orc.gram(X[lo:hi], y[lo:hi])
        d = float(fit.d[u])
        check_d(d, Go, nn, G[u].cpu().numpy())
        for q, (fam, gamma, alpha) in enumerate(pens):
            B, it, cv = orc.oem_path(Go / nn, co / nn, d, fam, fit.lam[u, q].cpu().numpy(), gamma, alpha)
            assert np.max(np.abs(fit.beta[u, q].cpu().numpy() - B)) <= TOL_BETA, (p, u, fam)


@pytest.mark.parametrize("p", [100, 200, 300, 512])
def test_batched_penalties_every_lean_layout(ctx, p, monkeypatch):
    """Four penalties multiplied together in one CTA (NPT = 4, the layout used when the per-penalty
    split does not fit the SMs) in each lean layout (2x32 / 4x16 / 4+4 shared-memory rows per
    thread), two units, against the oracle."""
    from paper_1801_09661_b200 import oem_fit_path, oem_gram
    monkeypatch.setenv("OEM_PATH_SOLVER", "batched")
    spec = CONFIGS["cfg2"].spec.replace(n=2000 + 3 * p, p=p, nnz=min(8, p))
    bt = dg.beta(spec)
    X, y = dg.rows_host(spec, bt)
    Xd = torch.from_numpy(X).cuda()
    yd = torch.from_numpy(y).cuda()
    h = (X.shape[0] // 2) & ~1
    G0, c0, _, n0 = oem_gram(ctx, Xd[:h], yd[:h])
    G1, c1, _, n1 = oem_gram(ctx, Xd[h:], yd[h:])
    pens = [("lasso", 0.0, 1.0), ("mcp", 3.0, 1.0), ("scad", 3.7, 1.0), ("enet", 0.0, 0.5)]
    fit = oem_fit_path(ctx, torch.stack([G0, G1]), torch.stack([c0, c1]), [n0, n1], pens, nlambda=8)
    for u, (lo, hi, nn) in enumerate([(0, h, n0), (h, X.shape[0], n1)]):
        Go, co, _ = orc.gram(X[lo:hi], y[lo:hi])
        d = float(fit.d[u])
        check_d(d, Go, nn)
        for q, (fam, gamma, alpha) in enumerate(pens):
            B, it, cv = orc.oem_path(Go / nn, co / nn, d, fam, fit.lam[u, q].cpu().numpy(), gamma, alpha)
            assert np.max(np.abs(fit.beta[u, q].cpu().numpy() - B)) <= TOL_BETA, (p, u, fam)


@pytest.mark.parametrize("p,solver", [(60, "active"), (260, None), (300, "global"), (700, "lean"), (1000, None)])
def test_active_set_solver(ctx, p, solver, monkeypatch):
    """The active-set cluster solver (default for p > 256; forced at p = 60) and the solvers it
    replaced there (grid-wide at p = 300, forced; lean has no layout at p = 700, so that case
    runs the grid-wide solver too), four penalties including a group one, two units, warm starts
    from a previous path and an explicit grid, all against the oracle's own pipeline."""
    from paper_1801_09661_b200 import oem_fit_path, oem_gram
    if solver:
        monkeypatch.setenv("OEM_PATH_SOLVER", solver)
    spec = CONFIGS["cfg4"].spec.replace(n=3000 + 2 * p, p=p - p % 10, nnz=3)
    pp = spec.p
    bt = dg.beta(spec)
    X, y = dg.rows_host(spec, bt)
    Xd, yd = torch.from_numpy(X).cuda(), torch.from_numpy(y).cuda()
    h = (X.shape[0] // 2) & ~1
    G0, c0, _, n0 = oem_gram(ctx, Xd[:h], yd[:h])
    G1, c1, _, n1 = oem_gram(ctx, Xd[h:], yd[h:])
    grp = (np.arange(pp) // 10).astype(np.int32)
    pens = [("lasso", 0.0, 1.0), ("grp_lasso", 0.0, 1.0), ("mcp", 3.0, 1.0), ("enet", 0.0, 0.5)]
    G = torch.stack([G0, G1]); c = torch.stack([c0, c1])
    fit = oem_fit_path(ctx, G, c, [n0, n1], pens, nlambda=10, group=grp, ngroups=pp // 10)
    for u, (lo, hi, nn) in enumerate([(0, h, n0), (h, X.shape[0], n1)]):
        Go, co, _ = orc.gram(X[lo:hi], y[lo:hi])
        d_ref = check_d(float(fit.d[u]), Go, nn, G[u].cpu().numpy())
        for q, (fam, gamma, alpha) in enumerate(pens):
            g = grp if fam.startswith("grp") else None
            lam = orc.lambda_grid(orc.lambda_max(fam, co / nn, group=g, alpha=alpha), 10)
            assert np.max(np.abs(fit.lam[u, q].cpu().numpy() - lam) / lam) < 1e-13
            B, it, cv = orc.oem_path(Go / nn, co / nn, d_ref, fam, lam, gamma, alpha, group=g)
            assert np.max(np.abs(fit.beta[u, q].cpu().numpy() - B)) <= TOL_BETA, (p, u, fam)
            assert np.array_equal(fit.conv[u, q].cpu().numpy().astype(bool), cv)
    # warm start from the last solutions, explicit two-point grid below the path's end
    init = fit.beta[:, :, -1, :].contiguous()
    lam2 = [float(fit.lam[0, 0, -1]) * 0.7, float(fit.lam[0, 0, -1]) * 0.5]
    fit2 = oem_fit_path(ctx, G, c, [n0, n1], pens[:1], lambdas=lam2, beta_init=init[:, :1].contiguous(),
                        d_in=[float(v) for v in fit.d.cpu()])
    for u, (lo, hi, nn) in enumerate([(0, h, n0), (h, X.shape[0], n1)]):
        Go, co, _ = orc.gram(X[lo:hi], y[lo:hi])
        B, it, cv = orc.oem_path(Go / nn, co / nn, float(fit.d[u]), "lasso", lam2,
                                 beta_init=init[u, 0].cpu().numpy())
        assert np.max(np.abs(fit2.beta[u, 0].cpu().numpy() - B)) <= TOL_BETA


@pytest.mark.parametrize("screen", ["0", "1", "32"])  # off, default capacity, 32 compact rows
def test_screened_active_cfg2_full_size(ctx, screen, monkeypatch):
    """The active-set solver on cfg2 at full size (n = 1e6, p = 100; lasso, MCP, SCAD paths of 100
    lambda), with and without the screened compact iterations (OEM_SCREEN): every unit against the
    oracle's path solve on the same Gram at the GPU's d."""
    from paper_1801_09661_b200 import oem_fit_path, oem_gram
    monkeypatch.setenv("OEM_PATH_SOLVER", "active")
    monkeypatch.setenv("OEM_SCREEN", screen)
    cfg = CONFIGS["cfg2"]
    bt = dg.beta(cfg.spec)
    Xd, yd = device_rows(cfg.spec, bt)
    G, c, yy, n = oem_gram(ctx, Xd, yd)
    del Xd, yd
    fit = oem_fit_path(ctx, G, c, [n], cfg.penalties, nlambda=cfg.nlambda)
    Gh, ch = G.cpu().numpy(), c.cpu().numpy()
    d = float(fit.d[0])
    errs = []
    for q, (fam, gamma, alpha) in enumerate(cfg.penalties):
        lg = fit.lam[0, q].cpu().numpy()
        B, it, cv = orc.oem_path(Gh / n, ch / n, d, fam, lg, gamma, alpha)
        Bg = fit.beta[0, q].cpu().numpy()
        e = np.max(np.abs(Bg - B), axis=1)
        errs.append((fam, float(e.max()), int(np.argmax(e)), int(fit.iters[0, q].sum()), int(it.sum())))
    for fam, e, l, itg, ito in errs:
        assert e <= TOL_BETA, errs
        assert abs(itg - ito) <= max(2, 0.02 * ito), errs


@pytest.mark.parametrize("p,screen", [(300, "1"), (300, "0"), (600, "1"), (90, "1")])
def test_screened_every_family(ctx, p, screen, monkeypatch):
    """The screened compact iterations for every family of Table 1 on the active-set
    solver: group MCP / SCAD (the compact step's norm thresholds), the sparse group lasso, the
    elastic net with variable weights, MCP and SCAD, with non-contiguous groups and group weights,
    in 256-thread (p = 300, 90) and 512-thread (p = 600) CTAs, screening on and off: every beta
    at 1e-8, the converged flags and the iteration counts against the oracle."""
    from paper_1801_09661_b200 import oem_fit_path, oem_gram
    monkeypatch.setenv("OEM_PATH_SOLVER", "active")
    monkeypatch.setenv("OEM_SCREEN", screen)
    rng = np.random.default_rng(p + 11)
    spec = CONFIGS["cfg3"].spec.replace(n=9000, p=p, nnz=min(12, p))
    bt = dg.beta(spec)
    X, y = dg.rows_host(spec, bt)
    Xp = np.zeros((X.shape[0], p + (p & 1)))
    Xp[:, :p] = X
    G, c, yy, n = oem_gram(ctx, torch.from_numpy(Xp).cuda()[:, :p], torch.from_numpy(y).cuda())
    Go, co, _ = orc.gram(X, y)
    ng = p // 6
    grp = rng.integers(0, ng, size=p).astype(np.int32)
    grp[:ng] = np.arange(ng)
    gw = rng.uniform(0.5, 2.0, ng)
    w = rng.uniform(0.5, 1.5, p)
    L = 16
    runs = [([("grp_mcp", 3.0, 1.0), ("grp_scad", 3.7, 1.0), ("sgl", 0.0, 0.5)], dict(group=grp, ngroups=ng, grp_w=gw)),
            ([("enet", 0.0, 0.4), ("mcp", 3.0, 1.0), ("scad", 3.7, 1.0)], dict(w=w))]
    for pens, kw in runs:
        kwd = dict(kw)
        if "w" in kwd:
            kwd = dict(var_w=torch.from_numpy(kwd.pop("w")).cuda())
        fit = oem_fit_path(ctx, G, c, [n], pens, nlambda=L, **kwd)
        d = float(fit.d[0])
        for q, (fam, gamma, alpha) in enumerate(pens):
            lg = fit.lam[0, q].cpu().numpy()
            B, it, cv = orc.oem_path(Go / n, co / n, d, fam, lg, gamma, alpha, **kw)
            Bg = fit.beta[0, q].cpu().numpy()
            assert np.max(np.abs(Bg - B)) <= TOL_BETA, (fam, np.max(np.abs(Bg - B)))
            assert np.array_equal(fit.conv[0, q].cpu().numpy().astype(bool), cv), fam
            itg = fit.iters[0, q].cpu().numpy()
            assert np.max(np.abs(itg - it)) <= max(2, 0.02 * it.max()), (fam, itg - it)
