"""Thin Python binding of liboem.so (include/oem.h): argument marshalling only.

Every step of the hot path runs in the CUDA kernels behind the C ABI; this module passes
torch-owned device pointers and sizes through ctypes and turns status codes into exceptions.
There is no CPU fallback: if liboem.so is missing or no CUDA device is present, calls fail
loudly.
"""
from __future__ import annotations

import ctypes
import os
from dataclasses import dataclass

import torch

_PKG = os.path.dirname(os.path.abspath(__file__))
LIBOEM = os.path.join(_PKG, "liboem.so")

OEM_LASSO, OEM_ENET, OEM_MCP, OEM_SCAD, OEM_GRP_LASSO, OEM_GRP_MCP, OEM_GRP_SCAD, OEM_SGL = range(8)
FAMILY = {"lasso": OEM_LASSO, "enet": OEM_ENET, "mcp": OEM_MCP, "scad": OEM_SCAD,
          "grp_lasso": OEM_GRP_LASSO, "grp_mcp": OEM_GRP_MCP, "grp_scad": OEM_GRP_SCAD,
          "sgl": OEM_SGL}   # sparse group lasso: (family, gamma unused, tau)
STATUS = ["OEM_OK", "OEM_ERR_INVALID_ARG", "OEM_ERR_DIM", "OEM_ERR_ALIGN", "OEM_ERR_EMPTY_FOLD",
          "OEM_ERR_NONFINITE", "OEM_ERR_CUDA", "OEM_ERR_NCCL", "OEM_ERR_NOMEM", "OEM_ERR_UNSUPPORTED"]

# Every symbol include/oem.h declares (checked by tests/test_abi.py).
ABI_SYMBOLS = ["oem_status_string", "oem_last_error", "oem_version", "oem_nccl_unique_id",
               "oem_ctx_create", "oem_ctx_destroy", "oem_gram", "oem_gram_folds",
               "oem_gram_weighted", "oem_fit_path", "oem_path_cfg_default", "oem_fit_logistic",
               "oem_logistic_cfg_default", "oem_cv_error", "oem_logit_grad", "oem_gram_moments", "oem_path_loss", "oem_gram_host", "oem_gram_folds_host", "oem_ctx_set_timing", "oem_ctx_stats",
               "oem_gram_csr", "oem_gram_sums", "oem_gram_folds_sums"]
_VOID = ("oem_status_string", "oem_last_error", "oem_version", "oem_path_cfg_default",
         "oem_logistic_cfg_default")


class OemError(RuntimeError):
    def __init__(self, code, detail):
        self.code = code
        self.status = STATUS[code] if 0 <= code < len(STATUS) else f"status {code}"
        super().__init__(f"{self.status}: {detail}")


class Penalty(ctypes.Structure):
    _fields_ = [("family", ctypes.c_int32), ("gamma", ctypes.c_double), ("alpha", ctypes.c_double)]


class PathCfg(ctypes.Structure):
    _fields_ = [("nlambda", ctypes.c_int32), ("lambda_min_ratio", ctypes.c_double),
                ("lambda_", ctypes.c_void_p), ("tol", ctypes.c_double), ("maxit", ctypes.c_int64),
                ("var_w", ctypes.c_void_p), ("group", ctypes.c_void_p), ("ngroups", ctypes.c_int32),
                ("grp_w", ctypes.c_void_p), ("d_squarings", ctypes.c_int32),
                ("fold_mode", ctypes.c_int32),
                ("lambda_max_override", ctypes.c_void_p), ("standardize", ctypes.c_int32),
                ("xsum", ctypes.c_void_p), ("ysum", ctypes.c_void_p), ("intercept_out", ctypes.c_void_p)]


class LogisticCfg(ctypes.Structure):
    _fields_ = [("nlambda", ctypes.c_int32), ("lambda_min_ratio", ctypes.c_double),
                ("lambda_", ctypes.c_void_p), ("tol_in", ctypes.c_double),
                ("maxit_in", ctypes.c_int64), ("tol_out", ctypes.c_double),
                ("outer_maxit", ctypes.c_int32), ("eps", ctypes.c_double),
                ("d_squarings", ctypes.c_int32), ("var_w", ctypes.c_void_p),
                ("group", ctypes.c_void_p), ("ngroups", ctypes.c_int32), ("grp_w", ctypes.c_void_p),
                ("hessian_upper_bound", ctypes.c_int32)]


class Stats(ctypes.Structure):
    _fields_ = [("launches", ctypes.c_int64), ("gram_ms", ctypes.c_double),
                ("reduce_ms", ctypes.c_double), ("allreduce_ms", ctypes.c_double),
                ("power_ms", ctypes.c_double), ("path_ms", ctypes.c_double)]

    def as_dict(self):
        return {k: getattr(self, k) for k, _ in self._fields_}


_lib = None


def lib():
    """Load liboem.so (in-tree). Raises if it has not been built: there is no fallback."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIBOEM):
            raise RuntimeError(f"{LIBOEM} not built: run `python -c 'import __graft_entry__ as g; g.build()'`")
        L = ctypes.CDLL(LIBOEM)
        P, i32, i64, d = ctypes.c_void_p, ctypes.c_int32, ctypes.c_int64, ctypes.c_double
        L.oem_status_string.restype = ctypes.c_char_p
        L.oem_status_string.argtypes = [ctypes.c_int]
        L.oem_last_error.restype = ctypes.c_char_p
        L.oem_version.restype = ctypes.c_char_p
        L.oem_nccl_unique_id.argtypes = [P]
        L.oem_ctx_create.argtypes = [ctypes.c_int, ctypes.c_int, ctypes.c_int, P, ctypes.POINTER(P)]
        L.oem_ctx_destroy.argtypes = [P]
        L.oem_gram.argtypes = [P, P, P, i64, i32, i64, P, P, P, ctypes.POINTER(i64), P]
        L.oem_gram_folds.argtypes = [P, P, P, i64, i32, i64, i64, i32, P, P, P, P, P]
        L.oem_gram_weighted.argtypes = [P, P, P, P, i64, i32, i64, d, P, P, P, P]
        L.oem_fit_path.argtypes = [P, P, P, P, i32, i32, ctypes.POINTER(Penalty), i32,
                                   ctypes.POINTER(PathCfg), P, P, P, P, P, P, P, P]
        L.oem_path_cfg_default.argtypes = [ctypes.POINTER(PathCfg)]
        L.oem_path_cfg_default.restype = None
        L.oem_logistic_cfg_default.argtypes = [ctypes.POINTER(LogisticCfg)]
        L.oem_logistic_cfg_default.restype = None
        L.oem_fit_logistic.argtypes = [P, P, P, i64, i32, i64, ctypes.POINTER(Penalty),
                                       ctypes.POINTER(LogisticCfg), P, P, P, P, P, P]
        L.oem_cv_error.argtypes = [P, P, P, P, P, i32, i32, i32, i32, P, P, P, P, P, P, P, P, P, P, P]
        L.oem_logit_grad.argtypes = [P, P, P, P, i64, i32, i64, P, P, P]
        L.oem_gram_moments.argtypes = [P, P, P, i64, i32, i64, i64, i32, P, P, P]
        L.oem_gram_host.argtypes = [P, P, P, i64, i32, i64, i64, P, P, P, ctypes.POINTER(i64), P]
        L.oem_gram_folds_host.argtypes = [P, P, P, i64, i32, i64, i64, i32, i64, P, P, P, P, P]
        L.oem_path_loss.argtypes = [P, P, P, P, P, i32, i32, i32, i32, P, P, P]
        L.oem_gram_csr.argtypes = [P, P, P, P, P, i64, i32, P, P, P, ctypes.POINTER(i64), P]
        L.oem_gram_sums.argtypes = [P, P, P, i64, i32, i64, P, P, P, P, P, ctypes.POINTER(i64), P]
        L.oem_gram_folds_sums.argtypes = [P, P, P, i64, i32, i64, i64, i32, P, P, P, P, P, P, P]
        L.oem_ctx_set_timing.argtypes = [P, ctypes.c_int]
        L.oem_ctx_stats.argtypes = [P, ctypes.POINTER(Stats), ctypes.c_int]
        for name in ABI_SYMBOLS:
            f = getattr(L, name)
            if name not in _VOID:
                f.restype = ctypes.c_int
        _lib = L
    return _lib


def _check(rc):
    if rc != 0:
        raise OemError(rc, lib().oem_last_error().decode())


def _ptr(t):
    return None if t is None else ctypes.c_void_p(t.data_ptr())


def _stream(stream):
    s = torch.cuda.current_stream() if stream is None else stream
    return ctypes.c_void_p(s.cuda_stream)


def _hold_until_done(ctx, stream, *tensors):
    """Keep host tensors alive until `stream` has passed the enqueued work that reads them (the
    f4 copies are asynchronous: a freed pinned block could be handed out again by PyTorch's
    caching host allocator while DMA still reads it). Finished entries are dropped on each call."""
    ev = torch.cuda.Event()
    ev.record(torch.cuda.current_stream() if stream is None else stream)
    ctx._inflight = [(e, t) for e, t in ctx._inflight if not e.query()] + [(ev, tensors)]


class Context:
    """One per (process, device): owns workspace and (nranks > 1) the NCCL communicator."""

    def __init__(self, device=0, nranks=1, rank=0, uid: bytes | None = None):
        if not torch.cuda.is_available():
            raise RuntimeError("liboem needs a CUDA device (no CPU fallback)")
        self.device, self.nranks, self.rank = device, nranks, rank
        self._inflight = []
        h = ctypes.c_void_p()
        buf = None if uid is None else ctypes.create_string_buffer(uid, 128)
        _check(lib().oem_ctx_create(device, nranks, rank, buf, ctypes.byref(h)))
        self.h = h

    def close(self):
        if getattr(self, "h", None):
            lib().oem_ctx_destroy(self.h)   # synchronises the device: in-flight copies are done
            self.h = None
            self._inflight = []

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def oem_nccl_unique_id() -> bytes:
    buf = ctypes.create_string_buffer(128)
    _check(lib().oem_nccl_unique_id(buf))
    return buf.raw


def _check_x(X, y):
    if X.dtype != torch.float64 or y.dtype != torch.float64 or not X.is_cuda or not y.is_cuda:
        raise TypeError("X and y must be float64 CUDA tensors")
    if X.dim() != 2 or X.stride(1) != 1:
        raise ValueError("X must be 2-D row-major (stride(1) == 1)")
    if y.dim() != 1 or y.stride(0) != 1 or y.shape[0] != X.shape[0]:
        raise ValueError("y must be contiguous with len(y) == X.shape[0]")


def oem_gram(ctx: Context, X: torch.Tensor, y: torch.Tensor, stream=None):
    """a2: raw (G = X^T X, xty = X^T y, yty, n_total), allreduced over ranks."""
    _check_x(X, y)
    n, p = X.shape
    dev = X.device
    G = torch.empty((p, p), dtype=torch.float64, device=dev)
    xty = torch.empty(p, dtype=torch.float64, device=dev)
    yty = torch.empty(1, dtype=torch.float64, device=dev)
    nt = ctypes.c_int64()
    _check(lib().oem_gram(ctx.h, _ptr(X), _ptr(y), n, p, X.stride(0), _ptr(G), _ptr(xty),
                          _ptr(yty), ctypes.byref(nt), _stream(stream)))
    return G, xty, yty, nt.value


def oem_gram_folds(ctx: Context, X, y, K: int, row_offset: int = 0, stream=None):
    """a3: K raw per-fold sums (G_k, xty_k, yty_k) and global fold counts."""
    _check_x(X, y)
    n, p = X.shape
    dev = X.device
    G = torch.empty((K, p, p), dtype=torch.float64, device=dev)
    xty = torch.empty((K, p), dtype=torch.float64, device=dev)
    yty = torch.empty(K, dtype=torch.float64, device=dev)
    counts = (ctypes.c_int64 * K)()
    _check(lib().oem_gram_folds(ctx.h, _ptr(X), _ptr(y), n, p, X.stride(0), row_offset, K, _ptr(G),
                                _ptr(xty), _ptr(yty), counts, _stream(stream)))
    return G, xty, yty, list(counts)


def oem_gram_sums(ctx: Context, X: torch.Tensor, y: torch.Tensor, stream=None):
    """a2 + f3 in one pass over [X | y | 1]: (G, xty, yty, xsum = X^T 1, ysum = 1^T y [1], n_total)."""
    _check_x(X, y)
    n, p = X.shape
    dev = X.device
    G = torch.empty((p, p), dtype=torch.float64, device=dev)
    xty = torch.empty(p, dtype=torch.float64, device=dev)
    yty = torch.empty(1, dtype=torch.float64, device=dev)
    xs = torch.empty(p, dtype=torch.float64, device=dev)
    ys = torch.empty(1, dtype=torch.float64, device=dev)
    nt = ctypes.c_int64()
    _check(lib().oem_gram_sums(ctx.h, _ptr(X), _ptr(y), n, p, X.stride(0), _ptr(G), _ptr(xty), _ptr(yty),
                               _ptr(xs), _ptr(ys), ctypes.byref(nt), _stream(stream)))
    return G, xty, yty, xs, ys, nt.value


def oem_gram_folds_sums(ctx: Context, X, y, K: int, row_offset: int = 0, stream=None):
    """a3 + f3 in one pass: (G_k, xty_k, yty_k, xsum_k [K][p], ysum_k [K], counts)."""
    _check_x(X, y)
    n, p = X.shape
    dev = X.device
    G = torch.empty((K, p, p), dtype=torch.float64, device=dev)
    xty = torch.empty((K, p), dtype=torch.float64, device=dev)
    yty = torch.empty(K, dtype=torch.float64, device=dev)
    xs = torch.empty((K, p), dtype=torch.float64, device=dev)
    ys = torch.empty(K, dtype=torch.float64, device=dev)
    counts = (ctypes.c_int64 * K)()
    _check(lib().oem_gram_folds_sums(ctx.h, _ptr(X), _ptr(y), n, p, X.stride(0), row_offset, K, _ptr(G),
                                     _ptr(xty), _ptr(yty), _ptr(xs), _ptr(ys), counts, _stream(stream)))
    return G, xty, yty, xs, ys, list(counts)


def oem_gram_weighted(ctx: Context, X, y01, beta, eps=1e-5, stream=None, scalars=True):
    """a4: raw (G_w, X^T W z, [sum w, loglik]) for the proximal-Newton step.

    scalars=False skips the sum of w and the log-likelihood (third result None)."""
    _check_x(X, y01)
    n, p = X.shape
    dev = X.device
    if beta.dtype != torch.float64 or not beta.is_cuda or beta.numel() != p:
        raise ValueError("beta must be a float64 CUDA tensor of length p")
    beta = beta.contiguous()
    Gw = torch.empty((p, p), dtype=torch.float64, device=dev)
    cw = torch.empty(p, dtype=torch.float64, device=dev)
    sc = torch.empty(2, dtype=torch.float64, device=dev) if scalars else None
    _check(lib().oem_gram_weighted(ctx.h, _ptr(X), _ptr(y01), _ptr(beta), n, p, X.stride(0), eps,
                                   _ptr(Gw), _ptr(cw), _ptr(sc), _stream(stream)))
    return Gw, cw, sc


@dataclass
class PathResult:
    beta: torch.Tensor      # [nG'][nP][L][p]
    lam: torch.Tensor       # [nG'][nP][L]
    iters: torch.Tensor     # [nG'][nP][L] int64
    conv: torch.Tensor      # [nG'][nP][L] uint8
    d: torch.Tensor         # [nG']
    intercept: torch.Tensor = None   # [nG'][nP][L] when fitted with an intercept (f3)


def oem_fit_path(ctx: Context, G, xty, counts, penalties, nlambda=100, lambda_min_ratio=1e-3,
                 lambdas=None, tol=1e-11, maxit=100000, var_w=None, group=None, ngroups=0,
                 grp_w=None, d_squarings=12, fold_mode=False, d_in=None,
                 beta_init=None, lambda_max=None, standardize=False, xsum=None, ysum=None,
                 stream=None) -> PathResult:
    """a6-a10: normalise, d, lambda grid and OEM paths for every (Gram, penalty) unit.

    G: [nG, p, p] (or [p, p]) raw sums, xty: [nG, p], counts: nG ints. penalties: list of
    (family, gamma, alpha)."""
    if G.dim() == 2:
        G = G.unsqueeze(0)
        xty = xty.unsqueeze(0)
    nG, p, _ = G.shape
    G = G.contiguous()
    xty = xty.contiguous()
    nGo = nG + 1 if fold_mode else nG
    nP = len(penalties)
    L = nlambda if lambdas is None else len(lambdas)
    pens = (Penalty * nP)(*[Penalty(FAMILY[f], float(g), float(a)) for f, g, a in penalties])
    cfg = PathCfg()
    lib().oem_path_cfg_default(ctypes.byref(cfg))
    cfg.nlambda = L
    cfg.lambda_min_ratio = lambda_min_ratio
    keep = []
    if lambdas is not None:
        lam_h = (ctypes.c_double * L)(*[float(v) for v in lambdas])
        keep.append(lam_h)
        cfg.lambda_ = ctypes.cast(lam_h, ctypes.c_void_p)
    cfg.tol = tol
    cfg.maxit = maxit
    if var_w is not None:
        var_w = var_w.to(device=G.device, dtype=torch.float64).contiguous()
        cfg.var_w = var_w.data_ptr()
    if group is not None:
        g_h = (ctypes.c_int32 * p)(*[int(v) for v in group])
        keep.append(g_h)
        cfg.group = ctypes.cast(g_h, ctypes.c_void_p)
        cfg.ngroups = int(ngroups or (max(int(v) for v in group) + 1))
    if grp_w is not None:
        gw_h = (ctypes.c_double * len(grp_w))(*[float(v) for v in grp_w])
        keep.append(gw_h)
        cfg.grp_w = ctypes.cast(gw_h, ctypes.c_void_p)
    cfg.d_squarings = d_squarings
    cfg.fold_mode = 1 if fold_mode else 0
    if lambda_max is not None:
        lm_h = ctypes.c_double(float(lambda_max))
        keep.append(lm_h)
        cfg.lambda_max_override = ctypes.cast(ctypes.pointer(lm_h), ctypes.c_void_p)
    cfg.standardize = 1 if standardize else 0
    icpt = None
    if xsum is not None or ysum is not None:
        xsum = xsum.reshape(nG, p).to(device=G.device, dtype=torch.float64).contiguous()
        ysum = ysum.reshape(nG).to(device=G.device, dtype=torch.float64).contiguous()
        keep += [xsum, ysum]
        cfg.xsum, cfg.ysum = xsum.data_ptr(), ysum.data_ptr()
        icpt = torch.empty((nGo, nP, L), dtype=torch.float64, device=G.device)
        cfg.intercept_out = icpt.data_ptr()
    cnt = (ctypes.c_int64 * nG)(*[int(c) for c in counts])
    d_h = None
    if d_in is not None:
        d_h = (ctypes.c_double * nGo)(*[float(v) for v in d_in])
    dev = G.device
    beta = torch.empty((nGo, nP, L, p), dtype=torch.float64, device=dev)
    lam = torch.empty((nGo, nP, L), dtype=torch.float64, device=dev)
    iters = torch.empty((nGo, nP, L), dtype=torch.int64, device=dev)
    conv = torch.empty((nGo, nP, L), dtype=torch.uint8, device=dev)
    d = torch.empty(nGo, dtype=torch.float64, device=dev)
    if beta_init is not None:
        beta_init = beta_init.to(device=dev, dtype=torch.float64).contiguous()
    _check(lib().oem_fit_path(ctx.h, _ptr(G), _ptr(xty), cnt, nG, p, pens, nP, ctypes.byref(cfg),
                              d_h, _ptr(beta_init), _ptr(beta), _ptr(lam), _ptr(iters), _ptr(conv),
                              _ptr(d), _stream(stream)))
    return PathResult(beta, lam, iters, conv, d, icpt)


def _check_host(X, y):
    if X.device.type != "cpu" or y.device.type != "cpu":
        raise ValueError("X and y must be host (CPU) tensors; pin them for overlapped copies")
    if X.dtype != torch.float64 or y.dtype != torch.float64:
        raise ValueError("X and y must be float64")
    if X.dim() != 2 or X.stride(1) != 1 or y.dim() != 1 or y.stride(0) != 1 or y.shape[0] != X.shape[0]:
        raise ValueError("X must be row-major [n, p] (unit column stride) and y [n] contiguous")


def oem_gram_host(ctx: Context, X, y, block_rows: int = 1 << 20, device=None, stream=None):
    """f4: the a2 Gram pass over host-resident (pinned) X, y streamed in row blocks."""
    _check_host(X, y)
    n, p = X.shape
    dev = device or torch.device("cuda", torch.cuda.current_device())
    G = torch.empty((p, p), dtype=torch.float64, device=dev)
    xty = torch.empty(p, dtype=torch.float64, device=dev)
    yty = torch.empty(1, dtype=torch.float64, device=dev)
    nt = ctypes.c_int64(0)
    _check(lib().oem_gram_host(ctx.h, X.data_ptr(), y.data_ptr(), n, p, X.stride(0), int(block_rows), _ptr(G),
                               _ptr(xty), _ptr(yty), ctypes.byref(nt), _stream(stream)))
    _hold_until_done(ctx, stream, X, y)
    return G, xty, yty, nt.value


def oem_gram_folds_host(ctx: Context, X, y, K: int, row_offset: int = 0, block_rows: int = 1 << 20, device=None,
                        stream=None):
    """f4: the a3 fold-segmented pass over host-resident (pinned) X, y streamed in row blocks."""
    _check_host(X, y)
    n, p = X.shape
    dev = device or torch.device("cuda", torch.cuda.current_device())
    G = torch.empty((K, p, p), dtype=torch.float64, device=dev)
    xty = torch.empty((K, p), dtype=torch.float64, device=dev)
    yty = torch.empty(K, dtype=torch.float64, device=dev)
    counts = (ctypes.c_int64 * K)()
    _check(lib().oem_gram_folds_host(ctx.h, X.data_ptr(), y.data_ptr(), n, p, X.stride(0), row_offset, K,
                                     int(block_rows), _ptr(G), _ptr(xty), _ptr(yty), counts, _stream(stream)))
    _hold_until_done(ctx, stream, X, y)
    return G, xty, yty, list(counts)


def oem_gram_csr(ctx: Context, row_ptr, col, val, y, p: int, stream=None):
    """f4 sparse design: the a2 statistics (G, X^T y, y^T y, n_total) of one pass over X in CSR
    form (row_ptr int64 [n+1], col int32 [nnz] ascending within rows, val float64 [nnz]) and y."""
    n = row_ptr.numel() - 1
    for t, dt in ((row_ptr, torch.int64), (col, torch.int32), (val, torch.float64), (y, torch.float64)):
        if t.dtype != dt or not t.is_cuda or not t.is_contiguous():
            raise ValueError("oem_gram_csr: row_ptr int64, col int32, val / y float64, contiguous CUDA tensors")
    if y.numel() != n or col.numel() != val.numel():
        raise ValueError("oem_gram_csr: y must have n entries and col / val the same length")
    G = torch.empty((p, p), dtype=torch.float64, device=y.device)
    xty = torch.empty(p, dtype=torch.float64, device=y.device)
    yty = torch.empty(1, dtype=torch.float64, device=y.device)
    nt = ctypes.c_int64(0)
    _check(lib().oem_gram_csr(ctx.h, _ptr(row_ptr), _ptr(col) if col.numel() else None,
                              _ptr(val) if val.numel() else None, _ptr(y), n, p, _ptr(G), _ptr(xty), _ptr(yty),
                              ctypes.byref(nt), _stream(stream)))
    return G, xty, yty, nt.value


def oem_gram_moments(ctx: Context, X, y, K: int = 1, row_offset: int = 0, stream=None):
    """f3: per-fold column sums (X^T 1 [K][p], 1^T y [K]) for the intercept / standardization."""
    _check_x(X, y)
    n, p = X.shape
    xs = torch.empty((K, p), dtype=torch.float64, device=X.device)
    ys = torch.empty(K, dtype=torch.float64, device=X.device)
    _check(lib().oem_gram_moments(ctx.h, _ptr(X), _ptr(y), n, p, X.stride(0), row_offset, K, _ptr(xs),
                                  _ptr(ys), _stream(stream)))
    return xs, ys


def oem_path_loss(ctx: Context, G, xty, yty, counts, beta, stream=None):
    """f3 compute.loss: mean squared residual of every path point from the raw unit statistics
    (G [nG][p][p], xty [nG][p], yty [nG], beta [nG][nP][L][p]) -> [nG][nP][L]."""
    if G.dim() == 2:
        G, xty, yty = G.unsqueeze(0), xty.unsqueeze(0), yty.reshape(1)
    nG, p, _ = G.shape
    nU, nP, L, pb = beta.shape
    if nU != nG or pb != p:
        raise ValueError("beta must be [nG][nP][L][p]")
    loss = torch.empty((nG, nP, L), dtype=torch.float64, device=G.device)
    cnt = (ctypes.c_int64 * nG)(*[int(c) for c in counts])
    _check(lib().oem_path_loss(ctx.h, _ptr(G.contiguous()), _ptr(xty.contiguous()), _ptr(yty.contiguous()), cnt,
                               nG, p, nP, L, _ptr(beta.contiguous()), _ptr(loss), _stream(stream)))
    return loss


@dataclass
class LogisticResult:
    beta: torch.Tensor        # [L][p]
    lam: torch.Tensor         # [L]
    outer_iters: list
    inner_iters: list
    conv: list


def oem_fit_logistic(ctx: Context, X, y01, penalty=("lasso", 0.0, 1.0), nlambda=50,
                     lambda_min_ratio=1e-3, lambdas=None, tol_in=1e-11, maxit_in=100000,
                     tol_out=1e-10, outer_maxit=100, eps=1e-5, d_squarings=12,
                     var_w=None, group=None, ngroups=0, grp_w=None, hessian_upper_bound=False,
                     stream=None) -> LogisticResult:
    """a4 + a6-a9 to convergence: proximal-Newton logistic path; with
    hessian_upper_bound=True the f1 mode (w = 1/4): Gram once, one gradient pass
    per outer step."""
    _check_x(X, y01)
    n, p = X.shape
    L = nlambda if lambdas is None else len(lambdas)
    cfg = LogisticCfg()
    lib().oem_logistic_cfg_default(ctypes.byref(cfg))
    cfg.nlambda = L
    cfg.lambda_min_ratio = lambda_min_ratio
    keep = []
    if lambdas is not None:
        lam_h = (ctypes.c_double * L)(*[float(v) for v in lambdas])
        keep.append(lam_h)
        cfg.lambda_ = ctypes.cast(lam_h, ctypes.c_void_p)
    cfg.tol_in, cfg.maxit_in, cfg.tol_out, cfg.outer_maxit = tol_in, maxit_in, tol_out, outer_maxit
    cfg.eps, cfg.d_squarings = eps, d_squarings
    if group is not None:
        g_h = (ctypes.c_int32 * p)(*[int(v) for v in group])
        keep.append(g_h)
        cfg.group = ctypes.cast(g_h, ctypes.c_void_p)
        cfg.ngroups = int(ngroups or (max(int(v) for v in group) + 1))
    if grp_w is not None:
        gw_h = (ctypes.c_double * len(grp_w))(*[float(v) for v in grp_w])
        keep.append(gw_h)
        cfg.grp_w = ctypes.cast(gw_h, ctypes.c_void_p)
    cfg.hessian_upper_bound = 1 if hessian_upper_bound else 0
    if var_w is not None:
        var_w = var_w.to(device=X.device, dtype=torch.float64).contiguous()
        cfg.var_w = var_w.data_ptr()
    f, g, a = penalty
    pen = Penalty(FAMILY[f], float(g), float(a))
    beta = torch.empty((L, p), dtype=torch.float64, device=X.device)
    lam = torch.empty(L, dtype=torch.float64, device=X.device)
    oi = (ctypes.c_int32 * L)()
    ii = (ctypes.c_int64 * L)()
    cv = (ctypes.c_uint8 * L)()
    _check(lib().oem_fit_logistic(ctx.h, _ptr(X), _ptr(y01), n, p, X.stride(0), ctypes.byref(pen),
                                  ctypes.byref(cfg), _ptr(beta), _ptr(lam), oi, ii, cv,
                                  _stream(stream)))
    return LogisticResult(beta, lam, list(oi), list(ii), [bool(v) for v in cv])


def oem_logit_grad(ctx: Context, X, y01, beta, stream=None, loglik=True):
    """f1: (X^T (y - sigma(X beta)), loglik) as raw sums in one pass over [X | y];
    loglik=False skips the log-likelihood (second result None)."""
    _check_x(X, y01)
    n, p = X.shape
    if beta.dtype != torch.float64 or not beta.is_cuda or beta.numel() != p:
        raise ValueError("beta must be a float64 CUDA tensor of length p")
    g = torch.empty(p, dtype=torch.float64, device=X.device)
    ll = torch.empty(1, dtype=torch.float64, device=X.device) if loglik else None
    _check(lib().oem_logit_grad(ctx.h, _ptr(X), _ptr(y01), _ptr(beta.contiguous()), n, p, X.stride(0),
                                _ptr(g), _ptr(ll), _stream(stream)))
    return g, ll


@dataclass
class CvResult:
    err: torch.Tensor       # [K][nP][L] held-out MSE of each complement fit on its fold
    cvm: torch.Tensor       # [nP][L]
    cvsd: torch.Tensor      # [nP][L]
    idx_min: list           # per penalty: index of lambda_min
    idx_1se: list           # per penalty: index of lambda_1se
    best: int               # penalty with the smallest min cvm


def oem_cv_error(ctx: Context, G_folds, xty_folds, yty_folds, counts, beta, intercept=None,
                 xsum_folds=None, ysum_folds=None, stream=None) -> CvResult:
    """f2: fast-CV error curve and selection from the fold sums and the fold-mode paths
    (beta: [K+1][nP][L][p] from oem_fit_path(..., fold_mode=True)); for a fit with an intercept
    pass its intercept [K+1][nP][L] and the fold column sums of oem_gram_moments."""
    K, p, _ = G_folds.shape
    nU, nP, L, pb = beta.shape
    if nU != K + 1 or pb != p:
        raise ValueError("beta must be the fold-mode path output [K+1][nP][L][p]")
    dev = G_folds.device
    err = torch.empty((K, nP, L), dtype=torch.float64, device=dev)
    cvm = torch.empty((nP, L), dtype=torch.float64, device=dev)
    cvsd = torch.empty((nP, L), dtype=torch.float64, device=dev)
    cnt = (ctypes.c_int64 * K)(*[int(c) for c in counts])
    imin = (ctypes.c_int32 * nP)()
    i1se = (ctypes.c_int32 * nP)()
    best = ctypes.c_int32()
    keep = [G_folds.contiguous(), xty_folds.contiguous(), yty_folds.contiguous(), beta.contiguous()]
    if intercept is not None:
        if xsum_folds is None or ysum_folds is None:
            raise ValueError("an intercept needs xsum_folds and ysum_folds (oem_gram_moments)")
        keep += [intercept.contiguous(), xsum_folds.reshape(K, p).contiguous(), ysum_folds.reshape(K).contiguous()]
    ptrs = [_ptr(t) for t in keep] + [None] * (7 - len(keep))
    _check(lib().oem_cv_error(ctx.h, ptrs[0], ptrs[1], ptrs[2], cnt, K, p, nP, L, ptrs[3], ptrs[5], ptrs[6],
                              ptrs[4], _ptr(err), _ptr(cvm), _ptr(cvsd), imin, i1se, ctypes.byref(best),
                              _stream(stream)))
    return CvResult(err, cvm, cvsd, list(imin), list(i1se), int(best.value))


def set_timing(ctx: Context, enable: bool = True):
    _check(lib().oem_ctx_set_timing(ctx.h, 1 if enable else 0))


def stats(ctx: Context, reset: bool = False) -> dict:
    """Accumulated device time per phase (CUDA events on the launching stream) and the number
    of kernels the context launched."""
    s = Stats()
    _check(lib().oem_ctx_stats(ctx.h, ctypes.byref(s), 1 if reset else 0))
    return s.as_dict()
