"""datagen — seeded synthetic inputs shared by the oracle tests and the CUDA path.

Holds none of the method's arithmetic (see include/oem_datagen.h for the generator
specification). Host rows come from libdatagen_host.so, device rows from libdatagen_cuda.so;
the two are independent implementations of the same spec and agree bit for bit.
"""
from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_ROOT = os.path.dirname(_HERE)
HOST_SO = os.path.join(_HERE, "libdatagen_host.so")
CUDA_SO = os.path.join(_HERE, "libdatagen_cuda.so")

DG_IID, DG_AR1, DG_BLOCK, DG_SPARSE = 0, 1, 2, 3
DG_LINEAR, DG_LOGISTIC = 0, 1
DG_BETA_EXPLICIT, DG_BETA_UNIFORM, DG_BETA_NORMAL, DG_BETA_ACTIVE_GROUPS = 0, 1, 2, 3


class Spec(ctypes.Structure):
    _fields_ = [("seed", ctypes.c_uint64), ("n", ctypes.c_int64), ("p", ctypes.c_int32),
                ("design", ctypes.c_int32), ("rho", ctypes.c_double),
                ("group_size", ctypes.c_int32), ("response", ctypes.c_int32),
                ("sigma", ctypes.c_double), ("beta_kind", ctypes.c_int32),
                ("nnz", ctypes.c_int32), ("beta_lo", ctypes.c_double), ("beta_hi", ctypes.c_double)]

    def replace(self, **kw):
        s = Spec()
        ctypes.pointer(s)[0] = self
        for k, v in kw.items():
            setattr(s, k, v)
        return s


def make_spec(seed, n, p, design=DG_IID, rho=0.0, group_size=1, response=DG_LINEAR, sigma=1.0,
              beta_kind=DG_BETA_EXPLICIT, nnz=0, beta_lo=0.0, beta_hi=0.0) -> Spec:
    return Spec(seed, n, p, design, rho, group_size, response, sigma, beta_kind, nnz, beta_lo,
                beta_hi)


def build_host(force=False):
    src = os.path.join(_HERE, "datagen_host.c")
    hdr = os.path.join(_ROOT, "include", "oem_datagen.h")
    if force or not os.path.exists(HOST_SO) or os.path.getmtime(HOST_SO) < max(
            os.path.getmtime(src), os.path.getmtime(hdr)):
        subprocess.check_call(["gcc", "-O2", "-ffp-contract=off", "-fPIC", "-shared", "-o", HOST_SO,
                               src, "-lm"])
    return HOST_SO


_host = None
_cuda = None


def host():
    global _host
    if _host is None:
        build_host()
        _host = ctypes.CDLL(HOST_SO)
        P = ctypes.c_void_p
        _host.dg_beta.restype = ctypes.c_int
        _host.dg_beta.argtypes = [ctypes.POINTER(Spec), P]
        _host.dg_rows_host.restype = ctypes.c_int
        _host.dg_rows_host.argtypes = [ctypes.POINTER(Spec), P, ctypes.c_int64, ctypes.c_int64,
                                       ctypes.c_int32, ctypes.c_int32, P, ctypes.c_int64, P]
        _host.dg_ln.restype = ctypes.c_double
        _host.dg_ln.argtypes = [ctypes.c_double]
        _host.dg_exp.restype = ctypes.c_double
        _host.dg_exp.argtypes = [ctypes.c_double]
        _host.dg_sincos2pi.argtypes = [ctypes.c_double, P, P]
    return _host


def cuda():
    global _cuda
    if _cuda is None:
        if not os.path.exists(CUDA_SO):
            raise RuntimeError(f"{CUDA_SO} missing: run __graft_entry__.build()")
        _cuda = ctypes.CDLL(CUDA_SO)
        P = ctypes.c_void_p
        _cuda.dg_rows_cuda.restype = ctypes.c_int
        _cuda.dg_rows_cuda.argtypes = [ctypes.POINTER(Spec), P, ctypes.c_int64, ctypes.c_int64, P,
                                       ctypes.c_int64, P, P]
        _cuda.dg_csr_count_cuda.restype = ctypes.c_int
        _cuda.dg_csr_count_cuda.argtypes = [ctypes.POINTER(Spec), ctypes.c_int64, ctypes.c_int64, P, P]
        _cuda.dg_csr_fill_cuda.restype = ctypes.c_int
        _cuda.dg_csr_fill_cuda.argtypes = [ctypes.POINTER(Spec), P, ctypes.c_int64, ctypes.c_int64, P, P, P,
                                           P, P]
    return _cuda


def philox(ctr, key):
    c = (ctypes.c_uint32 * 4)(*ctr)
    k = (ctypes.c_uint32 * 2)(*key)
    o = (ctypes.c_uint32 * 4)()
    host().dg_philox4x32_10(c, k, o)
    return list(o)


def beta(spec: Spec, explicit=None) -> np.ndarray:
    b = np.zeros(spec.p)
    if spec.beta_kind == DG_BETA_EXPLICIT:
        if explicit is None:
            raise ValueError("explicit beta required")
        b[:] = explicit
        return b
    if host().dg_beta(ctypes.byref(spec), b.ctypes.data_as(ctypes.c_void_p)) != 0:
        raise ValueError("invalid datagen spec")
    return b


def rows_host(spec: Spec, beta_true, row0=0, nrows=None, col0=0, ncols=None, want_y=True):
    """Host rows [row0,row0+nrows) x cols [col0,col0+ncols) -> (X (nrows,ncols), y or None)."""
    nrows = spec.n - row0 if nrows is None else nrows
    ncols = spec.p - col0 if ncols is None else ncols
    X = np.empty((nrows, max(ncols, 1)))
    y = np.empty(nrows) if want_y else None
    b = np.ascontiguousarray(beta_true, dtype=np.float64)
    rc = host().dg_rows_host(ctypes.byref(spec), b.ctypes.data_as(ctypes.c_void_p), row0, nrows,
                             col0, ncols, X.ctypes.data_as(ctypes.c_void_p), max(ncols, 1),
                             None if y is None else y.ctypes.data_as(ctypes.c_void_p))
    if rc != 0:
        raise ValueError("dg_rows_host: invalid arguments")
    return X[:, :ncols], y


def rows_cuda(spec: Spec, beta_dev_ptr: int, row0: int, nrows: int, X_ptr: int, ldx: int,
              y_ptr: int, stream_ptr: int = 0) -> None:
    rc = cuda().dg_rows_cuda(ctypes.byref(spec), beta_dev_ptr, row0, nrows, X_ptr, ldx, y_ptr,
                             stream_ptr)
    if rc != 0:
        raise RuntimeError(f"dg_rows_cuda failed rc={rc}")


def csr_cuda(spec: Spec, beta_true, row0: int = 0, nrows: int | None = None, want_y: bool = True):
    """SPARSE design rows [row0, row0+nrows) generated on the current CUDA device in CSR form:
    (row_ptr int64 [nrows+1], col int32 [nnz], val float64 [nnz], y float64 [nrows] or None), torch
    tensors. The row offsets are the exclusive prefix sum of the per-row counts (torch.cumsum:
    input residency, not the method)."""
    import torch
    nrows = spec.n - row0 if nrows is None else nrows
    st = torch.cuda.current_stream().cuda_stream
    counts = torch.empty(max(nrows, 1), dtype=torch.int64, device="cuda")
    if cuda().dg_csr_count_cuda(ctypes.byref(spec), row0, nrows, counts.data_ptr(), st) != 0:
        raise RuntimeError("dg_csr_count_cuda failed")
    row_ptr = torch.zeros(nrows + 1, dtype=torch.int64, device="cuda")
    if nrows:
        torch.cumsum(counts[:nrows], 0, out=row_ptr[1:])
    nnz = int(row_ptr[-1])
    col = torch.empty(max(nnz, 1), dtype=torch.int32, device="cuda")
    val = torch.empty(max(nnz, 1), dtype=torch.float64, device="cuda")
    y = torch.empty(max(nrows, 1), dtype=torch.float64, device="cuda") if want_y else None
    b = torch.from_numpy(np.ascontiguousarray(beta_true, dtype=np.float64)).cuda()
    if cuda().dg_csr_fill_cuda(ctypes.byref(spec), b.data_ptr(), row0, nrows, row_ptr.data_ptr(), col.data_ptr(),
                               val.data_ptr(), None if y is None else y.data_ptr(), st) != 0:
        raise RuntimeError("dg_csr_fill_cuda failed")
    return row_ptr, col[:nnz], val[:nnz], (y[:nrows] if y is not None else None)
