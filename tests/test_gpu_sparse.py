"""f4 sparse design (§5.8): the CSR Gram pass (oem_gram_csr) against the oracle's
plain definition over the MATERIALISED dense matrix (O1, orc.gram), and the fit from it against
the oracle's pipeline; the device CSR generator against the host dense generator (bit for bit)."""
import numpy as np
import pytest

import datagen as dg
import oracle as orc
from datagen.configs import CONFIGS, groups_of
from gpu_util import scale_err, xty_err

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")


@pytest.fixture(scope="module")
def ctx():
    from paper_1801_09661_b200 import Context
    c = Context(0)
    yield c
    c.close()


def dense_from_csr(rp, col, val, n, p):
    X = np.zeros((n, p))
    rp, col, val = rp.cpu().numpy(), col.cpu().numpy(), val.cpu().numpy()
    rows = np.repeat(np.arange(n), np.diff(rp))
    X[rows, col] = val
    return X


def csr_from_dense(X):
    n, p = X.shape
    nzr, nzc = np.nonzero(X)
    rp = np.zeros(n + 1, dtype=np.int64)
    np.add.at(rp, nzr + 1, 1)
    rp = np.cumsum(rp)
    return (torch.from_numpy(rp).cuda(), torch.from_numpy(nzc.astype(np.int32)).cuda(),
            torch.from_numpy(X[nzr, nzc].copy()).cuda())


def test_device_csr_generator_matches_host_dense():
    spec = CONFIGS["sparse"].spec.replace(n=20_011)
    bt = dg.beta(spec)
    rp, col, val, y = dg.csr_cuda(spec, bt)
    X, yh = dg.rows_host(spec, bt)
    assert np.array_equal(dense_from_csr(rp, col, val, spec.n, spec.p), X)
    assert np.array_equal(y.cpu().numpy(), yh)
    c = col.cpu().numpy()
    r = rp.cpu().numpy()
    for i in range(0, spec.n, 997):          # ascending, in-range columns within each row
        seg = c[r[i]:r[i + 1]]
        assert np.all(np.diff(seg) > 0) and (seg.size == 0 or (seg[0] >= 0 and seg[-1] < spec.p))


@pytest.mark.parametrize("n,p,d", [(100_000, 200, 0.01), (30_011, 200, 0.01), (5_003, 37, 0.2),
                                   (4_001, 300, 0.05), (2_000, 100, 0.9), (777, 1, 0.5), (3_001, 768, 0.02)])
def test_sparse_gram_parity(ctx, n, p, d):
    """The paper's example shape (n = 1e5, p = 200, density 0.01), ragged n, p = 300 and 768 (two
    and more triangle slices), density 0.9 (chunks split by the nonzero cap), p = 1."""
    from paper_1801_09661_b200 import oem_gram_csr
    spec = CONFIGS["sparse"].spec.replace(n=n, p=p, rho=d, nnz=min(15, p))
    bt = dg.beta(spec)
    rp, col, val, y = dg.csr_cuda(spec, bt)
    G, c, yy, nt = oem_gram_csr(ctx, rp, col, val, y, p)
    X, yh = dg.rows_host(spec, bt)
    Go, co, yyo = orc.gram(X, yh)
    assert nt == n
    assert scale_err(G.cpu().numpy(), Go) <= 1e-12
    assert xty_err(c.cpu().numpy(), co, Go, yyo) <= 1e-12
    assert abs(float(yy) - yyo) <= 1e-12 * yyo
    # determinism: a second call is bitwise identical
    G2, c2, yy2, _ = oem_gram_csr(ctx, rp, col, val, y, p)
    assert torch.equal(G, G2) and torch.equal(c, c2) and torch.equal(yy, yy2)


def test_sparse_gram_integer_bit_exact_and_edges(ctx):
    """Integer values: every partial sum is exact, so GPU == oracle bitwise in any order; empty
    rows, a dense row, n = 0."""
    from paper_1801_09661_b200 import oem_gram_csr
    rng = np.random.default_rng(5)
    n, p = 3001, 50
    X = rng.integers(-8, 9, size=(n, p)).astype(float) * (rng.random((n, p)) < 0.08)
    X[10] = 0.0
    X[11] = rng.integers(1, 9, size=p)
    y = rng.integers(-8, 9, size=n).astype(float)
    rp, col, val = csr_from_dense(X)
    G, c, yy, nt = oem_gram_csr(ctx, rp, col, val, torch.from_numpy(y).cuda(), p)
    Go, co, yyo = orc.gram(X, y)
    assert np.array_equal(G.cpu().numpy(), Go) and np.array_equal(c.cpu().numpy(), co)
    assert float(yy) == yyo and nt == n
    z = torch.zeros(1, dtype=torch.int64, device="cuda")
    e = torch.zeros(0, dtype=torch.int32, device="cuda")
    G0, c0, yy0, n0 = oem_gram_csr(ctx, z, e, torch.zeros(0, dtype=torch.float64, device="cuda"),
                                   torch.zeros(0, dtype=torch.float64, device="cuda"), 7)
    assert n0 == 0 and not G0.any() and not c0.any() and float(yy0) == 0.0


def test_sparse_equals_dense_path_and_fit(ctx):
    """The sparse pass and the dense tensor-core pass give the same statistics on the same data,
    and the paper's example fit (lasso + group lasso with 40 groups of 5) from the
    sparse statistics matches the oracle's pipeline on the dense matrix."""
    from paper_1801_09661_b200 import oem_fit_path, oem_gram, oem_gram_csr
    cfg = CONFIGS["sparse"].with_n(100_000)
    bt = dg.beta(cfg.spec)
    rp, col, val, y = dg.csr_cuda(cfg.spec, bt)
    Gs, cs, yys, n = oem_gram_csr(ctx, rp, col, val, y, cfg.p)
    X, yh = dg.rows_host(cfg.spec, bt)
    Gd, cd, yyd, _ = oem_gram(ctx, torch.from_numpy(X).cuda(), torch.from_numpy(yh).cuda())
    assert scale_err(Gs.cpu().numpy(), Gd.cpu().numpy()) <= 2e-12
    grp = groups_of(cfg)
    fit = oem_fit_path(ctx, Gs, cs, [n], cfg.penalties, nlambda=30, group=grp, ngroups=cfg.p // 5)
    Go, co, _ = orc.gram(X, yh)
    d_ref = orc.d_rule(Go / n)[0]
    assert abs(float(fit.d[0]) - d_ref) <= 1e-11 * d_ref
    for q, (fam, gamma, alpha) in enumerate(cfg.penalties):
        g = grp if fam.startswith("grp") else None
        lam = orc.lambda_grid(orc.lambda_max(fam, co / n, group=g), 30)
        B, it, cv = orc.oem_path(Go / n, co / n, d_ref, fam, lam, gamma, alpha, group=g)
        assert np.max(np.abs(fit.beta[0, q].cpu().numpy() - B)) <= 1e-8, fam


def test_sparse_full_size_column_sample(ctx):
    """The benched size (n = 1e7, p = 200, density 0.01, 2e7 nonzeros), in bench.py's launch
    configuration: a 24 x 24 sub-Gram (columns 0-11 and 188-199), X^T y and y^T y against the
    oracle's sums over all 1e7 rows of the materialised columns (host generator, those columns)."""
    from paper_1801_09661_b200 import oem_gram_csr
    cfg = CONFIGS["sparse"]
    bt = dg.beta(cfg.spec)
    rp, col, val, y = dg.csr_cuda(cfg.spec, bt)
    G, c, yy, n = oem_gram_csr(ctx, rp, col, val, y, cfg.p)
    del rp, col, val, y
    blocks = ((0, 12), (188, 12))
    idx = np.concatenate([np.arange(a, a + m) for a, m in blocks])
    acc = orc.GramAccumulator(idx.size)
    for r in range(0, cfg.n, 1_000_000):
        parts, yb = [], None
        for a, m in blocks:
            Xb, yv = dg.rows_host(cfg.spec, bt, r, 1_000_000, a, m, want_y=yb is None)
            parts.append(Xb)
            yb = yv if yb is None else yb
        acc.add(np.ascontiguousarray(np.hstack(parts)), yb)
    Go, co, yyo = acc.result()
    assert scale_err(G.cpu().numpy()[np.ix_(idx, idx)], Go) <= 1e-12
    assert xty_err(c.cpu().numpy()[idx], co, Go, yyo) <= 1e-12
    assert abs(float(yy) - yyo) <= 1e-12 * yyo
