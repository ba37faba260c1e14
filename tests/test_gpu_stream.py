"""GPU parity for f4, the out-of-core Gram passes (oem_gram_host / oem_gram_folds_host): X and y
stay in pinned host memory and are streamed through the tensor-core Gram kernel in row blocks
(P:L743-892 big.oem). Integer-valued data make every partial sum exact, so the streamed result
must equal the oracle bit for bit whatever the block size (ragged last blocks, folds that
straddle blocks, a nonzero global row offset)."""
import numpy as np
import pytest

import datagen as dg
import oracle as orc
from datagen.configs import CONFIGS
from gpu_util import scale_err

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")


@pytest.fixture(scope="module")
def ctx():
    from paper_1801_09661_b200 import Context
    c = Context(0)
    yield c
    c.close()


def _pinned(X, y, p):
    Xh = torch.zeros((X.shape[0], p + (p & 1)), dtype=torch.float64, pin_memory=True)
    Xh[:, :p] = torch.from_numpy(X)
    yh = torch.from_numpy(y).pin_memory()
    return Xh[:, :p], yh


@pytest.mark.parametrize("n,p,blk", [(20_011, 7, 32), (20_011, 7, 4097), (20_011, 300, 1000), (5_000, 129, 5_000),
                                     (3_001, 1001, 777)])
def test_gram_host_exact(ctx, n, p, blk):
    from paper_1801_09661_b200 import oem_gram_host
    rng = np.random.default_rng(p + blk)
    X = rng.integers(-8, 9, size=(n, p)).astype(float)
    y = rng.integers(-8, 9, size=n).astype(float)
    Xh, yh = _pinned(X, y, p)
    G, c, yy, nt = oem_gram_host(ctx, Xh, yh, block_rows=blk)
    Go, co, yyo = orc.gram(X, y)
    assert nt == n
    assert np.array_equal(G.cpu().numpy(), Go)
    assert np.array_equal(c.cpu().numpy(), co)
    assert float(yy) == yyo


@pytest.mark.parametrize("K,off,blk", [(10, 0, 1000), (7, 3, 333), (3, 11, 32)])
def test_gram_folds_host_exact(ctx, K, off, blk):
    from paper_1801_09661_b200 import oem_gram_folds_host
    n, p = 9_001, 40
    rng = np.random.default_rng(K)
    X = rng.integers(-8, 9, size=(n, p)).astype(float)
    y = rng.integers(-8, 9, size=n).astype(float)
    Xh, yh = _pinned(X, y, p)
    G, c, yy, cnt = oem_gram_folds_host(ctx, Xh, yh, K, row_offset=off, block_rows=blk)
    Gf, cf, yyf, cnto = orc.gram_folds(X, y, K, row_offset=off)
    assert list(cnt) == list(cnto)
    assert np.array_equal(G.cpu().numpy(), Gf)
    assert np.array_equal(c.cpu().numpy(), cf)
    assert np.array_equal(yy.cpu().numpy(), yyf)


def test_gram_host_float_matches_in_core(ctx):
    """cfg4-shaped rows (p = 1000) streamed in 4 ragged blocks vs the oracle at the north-star
    tolerance (R#32)."""
    from paper_1801_09661_b200 import oem_gram_host
    spec = CONFIGS["cfg4"].spec.replace(n=6_007)
    bt = dg.beta(spec)
    X, y = dg.rows_host(spec, bt)
    Xh, yh = _pinned(X, y, X.shape[1])
    G, c, yy, nt = oem_gram_host(ctx, Xh, yh, block_rows=1600)
    Go, co, yyo = orc.gram(X, y)
    assert scale_err(G.cpu().numpy(), Go) <= 1e-12


def test_stream_edge_cases(ctx):
    """n = 0 gives zero statistics; block_rows below the minimum (32) and a fold with no rows are
    reported through the status codes, never as wrong numbers; blocks of exactly one row-tile."""
    from paper_1801_09661_b200 import OemError, oem_gram_folds_host, oem_gram_host
    p = 6
    X0 = torch.zeros((0, p), dtype=torch.float64).pin_memory()
    y0 = torch.zeros(0, dtype=torch.float64).pin_memory()
    G, c, yy, nt = oem_gram_host(ctx, X0, y0, block_rows=64)
    assert nt == 0 and not G.any() and not c.any() and float(yy) == 0.0
    rng = np.random.default_rng(5)
    X = rng.integers(-8, 9, size=(100, p)).astype(float)
    y = rng.integers(-8, 9, size=100).astype(float)
    Xh, yh = _pinned(X, y, p)
    with pytest.raises(OemError) as e:
        oem_gram_host(ctx, Xh, yh, block_rows=31)
    assert e.value.status == "OEM_ERR_INVALID_ARG"
    with pytest.raises(OemError) as e:   # K = 200 > n = 100 rows: folds 100..199 are empty
        oem_gram_folds_host(ctx, Xh, yh, 200, block_rows=64)
    assert e.value.status == "OEM_ERR_EMPTY_FOLD"
    G, c, yy, nt = oem_gram_host(ctx, Xh, yh, block_rows=32)   # 4 blocks, the last one ragged
    Go, co, yyo = orc.gram(X, y)
    assert nt == 100 and np.array_equal(G.cpu().numpy(), Go) and np.array_equal(c.cpu().numpy(), co)


def test_gram_host_full_size_cfg4(ctx):
    """f4 at full size, as bench.py's e2e leg runs it: cfg4's 1e7 x 1000 design (80 GB) in pinned
    host memory streamed through the Gram kernel in 2^20-row blocks, against the oracle's sums over
    all 1e7 rows on a 32-column sample spanning four panels (gpu_util.cfg4_oracle_sample), and
    against the in-core pass over the same rows (every entry)."""
    from paper_1801_09661_b200 import oem_gram, oem_gram_host
    cfg = CONFIGS["cfg4"]
    bt = dg.beta(cfg.spec)
    from gpu_util import device_rows
    Xd, yd = device_rows(cfg.spec, bt)
    G, c, yy, nt = oem_gram(ctx, Xd, yd)
    Xh = torch.empty(Xd.shape, dtype=torch.float64, pin_memory=True)
    Xh.copy_(Xd)
    yh = yd.cpu().pin_memory()
    del Xd, yd
    torch.cuda.empty_cache()
    Gs, cs, yys, ns = oem_gram_host(ctx, Xh, yh, block_rows=1 << 20)
    assert ns == nt == cfg.n
    Gh = G.cpu().numpy()
    assert scale_err(Gs.cpu().numpy(), Gh) <= 1e-12
    d = np.sqrt(np.diag(Gh))
    assert np.max(np.abs(cs.cpu().numpy() - c.cpu().numpy()) / (d * np.sqrt(float(yy)))) <= 1e-12
    assert abs(float(yys) - float(yy)) <= 1e-12 * float(yy)
    from gpu_util import cfg4_oracle_sample, scale_err as serr, xty_err
    idx, Go, co, yyo, _, _ = cfg4_oracle_sample()
    assert serr(Gs.cpu().numpy()[np.ix_(idx, idx)], Go) <= 1e-12
    assert xty_err(cs.cpu().numpy()[idx], co, Go, yyo) <= 1e-12
    assert abs(float(yys) - yyo) <= 1e-12 * yyo
