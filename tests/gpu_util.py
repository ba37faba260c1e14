"""Helpers for the -m gpu parity tests: device-resident synthetic inputs and error metrics."""
import functools

import numpy as np

import datagen as dg


def device_rows(spec, beta_true, row0=0, nrows=None, ldx=None):
    """X (nrows x p, row-major, leading dim ldx) and y generated ON THE DEVICE by the CUDA
    generator (bit-identical to datagen.rows_host)."""
    import torch
    nrows = spec.n - row0 if nrows is None else nrows
    p = spec.p
    ldx = ldx or (p + (p & 1))
    Xs = torch.empty((max(nrows, 1), ldx), dtype=torch.float64, device="cuda")
    y = torch.empty(max(nrows, 1), dtype=torch.float64, device="cuda")
    b = torch.from_numpy(np.ascontiguousarray(beta_true, dtype=np.float64)).cuda()
    dg.rows_cuda(spec, b.data_ptr(), row0, nrows, Xs.data_ptr(), ldx, y.data_ptr(),
                 torch.cuda.current_stream().cuda_stream)
    return Xs[:nrows, :p], y[:nrows]


def scale_err(A, B):
    """DESIGN.md R#32: max |A_jk - B_jk| / sqrt(B_jj B_kk)."""
    d = np.sqrt(np.abs(np.diag(B)))
    s = np.outer(d, d)
    s[s == 0] = 1.0
    return float(np.max(np.abs(A - B) / s)) if A.size else 0.0


def xty_err(c, co, Go, yy):
    s = np.sqrt(np.abs(np.diag(Go)) * abs(yy))
    s[s == 0] = 1.0
    return float(np.max(np.abs(c - co) / s)) if c.size else 0.0


CFG4_COLUMN_BLOCKS = ((0, 8), (248, 8), (496, 8), (992, 8))


@functools.lru_cache(maxsize=1)
def cfg4_oracle_sample():
    """The oracle's sums over ALL n = 1e7 rows of cfg4 for 32 columns in four 8-column blocks
    that lie in four different 128-column panels of the two-panel Gram plan (columns 0-7, 248-255,
    496-503, 992-999), so the 32 x 32 sub-Gram holds diagonal-panel entries and every kind of
    off-diagonal panel pair. Rows come from the host generator, those columns only. Computed once
    per session (shared by the in-core and the streamed full-size tests).
    Returns (idx, G_sub, xty_sub, yty, xsum_sub, xabs_sub)."""
    import oracle as orc
    from datagen.configs import CONFIGS
    cfg = CONFIGS["cfg4"]
    bt = dg.beta(cfg.spec)
    idx = np.concatenate([np.arange(c0, c0 + m) for c0, m in CFG4_COLUMN_BLOCKS])
    acc = orc.GramAccumulator(idx.size)
    xs = np.zeros(idx.size)
    xa = np.zeros(idx.size)
    for r in range(0, cfg.n, 1_000_000):
        parts = []
        y = None
        for c0, m in CFG4_COLUMN_BLOCKS:
            X, yb = dg.rows_host(cfg.spec, bt, r, 1_000_000, c0, m, want_y=y is None)
            parts.append(X)
            y = yb if y is None else y
        X = np.ascontiguousarray(np.hstack(parts))
        acc.add(X, y)
        xs += X.sum(axis=0)
        xa += np.abs(X).sum(axis=0)
    Go, co, yyo = acc.result()
    return idx, Go, co, yyo, xs, xa
