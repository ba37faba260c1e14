"""Helpers for the -m gpu parity tests: device-resident synthetic inputs and error metrics."""
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
