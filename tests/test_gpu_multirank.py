"""a5 cross-GPU combine through the library's own NCCL path ("computed
independently ... in parallel", P:L72-76 Gram quantities on a cluster).

1. On ONE GPU: a context created with an NCCL unique id holds a one-rank communicator, so every
   entry point takes its multi-rank branch (ncclCommInitRank, the packed-triangle allreduce, the
   int64 row-count allreduce, the fp64 n_total allreduce of the logistic driver). A one-rank sum
   is the identity: every output must equal the no-communicator context's bit for bit.
2. On >= 2 GPUs (skipped otherwise; this pool has one GPU per box): torchrun with one rank per
   GPU runs tests/mr_worker.py, which shards the rows, combines through the library's NCCL
   allreduce, checks that every rank holds bitwise-identical statistics and fits, and compares
   rank 0's combined statistics with the oracle on the whole design."""
import os
import socket
import subprocess
import sys

import numpy as np
import pytest

import datagen as dg
import oracle as orc
from datagen.configs import CONFIGS
from gpu_util import device_rows, scale_err

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def ctxs():
    from paper_1801_09661_b200 import Context, oem_nccl_unique_id
    plain = Context(0)
    nccl = Context(0, 1, 0, oem_nccl_unique_id())
    yield plain, nccl
    nccl.close()
    plain.close()


def test_one_rank_communicator_is_bitwise_identity(ctxs):
    from paper_1801_09661_b200 import (oem_fit_logistic, oem_fit_path, oem_gram, oem_gram_folds,
                                       oem_gram_moments, oem_gram_weighted, oem_logit_grad)
    plain, nccl = ctxs
    spec = CONFIGS["cfg2"].spec.replace(n=20_011, p=40, nnz=6)
    bt = dg.beta(spec)
    Xd, yd = device_rows(spec, bt)
    a = oem_gram(plain, Xd, yd)
    b = oem_gram(nccl, Xd, yd)
    assert a[3] == b[3] == spec.n
    for u, v in zip(a[:3], b[:3]):
        assert torch.equal(u, v)
    a = oem_gram_folds(plain, Xd, yd, 7, row_offset=3)
    b = oem_gram_folds(nccl, Xd, yd, 7, row_offset=3)
    assert list(a[3]) == list(b[3])
    for u, v in zip(a[:3], b[:3]):
        assert torch.equal(u, v)
    for u, v in zip(oem_gram_moments(plain, Xd, yd, 3), oem_gram_moments(nccl, Xd, yd, 3)):
        assert torch.equal(u, v)
    y01 = (yd > 0).double()
    beta = torch.linspace(-0.2, 0.2, spec.p, dtype=torch.float64, device="cuda")
    for u, v in zip(oem_gram_weighted(plain, Xd, y01, beta), oem_gram_weighted(nccl, Xd, y01, beta)):
        assert torch.equal(u, v)
    for u, v in zip(oem_logit_grad(plain, Xd, y01, beta), oem_logit_grad(nccl, Xd, y01, beta)):
        assert torch.equal(u, v)
    G, c, yy, n = oem_gram(nccl, Xd, yd)
    fa = oem_fit_path(plain, G, c, [n], [("lasso", 0, 1), ("scad", 3.7, 1)], nlambda=10)
    fb = oem_fit_path(nccl, G, c, [n], [("lasso", 0, 1), ("scad", 3.7, 1)], nlambda=10)
    assert torch.equal(fa.beta, fb.beta) and torch.equal(fa.d, fb.d)
    la = oem_fit_logistic(plain, Xd, y01, nlambda=4)
    lb = oem_fit_logistic(nccl, Xd, y01, nlambda=4)
    assert torch.equal(la.beta, lb.beta) and la.outer_iters == lb.outer_iters
    from paper_1801_09661_b200 import oem_gram_folds_sums, oem_gram_sums
    for u, v in zip(oem_gram_sums(plain, Xd, yd), oem_gram_sums(nccl, Xd, yd)):
        assert torch.equal(u, v) if torch.is_tensor(u) else u == v
    for u, v in zip(oem_gram_folds_sums(plain, Xd, yd, 7, 3), oem_gram_folds_sums(nccl, Xd, yd, 7, 3)):
        assert torch.equal(u, v) if torch.is_tensor(u) else u == v
    from paper_1801_09661_b200 import oem_gram_csr
    sspec = CONFIGS["sparse"].spec.replace(n=30_011)
    rp, col, val, ys = dg.csr_cuda(sspec, dg.beta(sspec))
    a = oem_gram_csr(plain, rp, col, val, ys, sspec.p)
    b = oem_gram_csr(nccl, rp, col, val, ys, sspec.p)
    assert a[3] == b[3] == sspec.n
    for u, v in zip(a[:3], b[:3]):
        assert torch.equal(u, v)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


@pytest.mark.skipif(not torch.cuda.is_available() or torch.cuda.device_count() < 2,
                    reason="needs >= 2 GPUs (one rank per GPU)")
def test_torchrun_row_sharded_combine():
    world = torch.cuda.device_count()
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={world}",
           "--master-addr", "127.0.0.1", "--master-port", str(_free_port()),
           os.path.join(ROOT, "tests", "mr_worker.py")]
    r = subprocess.run(cmd, cwd=ROOT, capture_output=True, text=True, timeout=900)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-3000:]
    assert "MR_WORKER_OK" in r.stdout


def test_worker_single_process_reference():
    """The worker's oracle comparison, run here at world size 1 (no communicator): the same
    sharding code with one shard must reproduce the oracle (guards the worker itself)."""
    env = dict(os.environ, WORLD_SIZE="1", RANK="0", LOCAL_RANK="0")
    r = subprocess.run([sys.executable, os.path.join(ROOT, "tests", "mr_worker.py")], cwd=ROOT,
                       capture_output=True, text=True, timeout=600, env=env)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-3000:]
    assert "MR_WORKER_OK" in r.stdout
