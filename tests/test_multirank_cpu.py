"""World-size-2 (and 3) CPU tests of the multi-GPU host logic with torch.distributed/gloo: row
sharding, fold phases from the global row offset, and the sum-combine of per-rank raw statistics
(the NCCL allreduce's job on the GPUs) reproduce the single-process statistics exactly on
integer-valued designs. Oracle arithmetic stands in for the per-rank Gram
kernels, which need a GPU."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import oracle as orc
from paper_1801_09661_b200.shard import fold_counts, row_range


def free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def design(n, p, seed=3):
    rng = np.random.default_rng(seed)
    return rng.integers(-8, 9, size=(n, p)).astype(float), rng.integers(-8, 9, size=n).astype(float)


def worker(rank, world, port, n, p, K, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        X, y = design(n, p)
        r0, r1 = row_range(n, world, rank)
        Xs, ys = X[r0:r1], y[r0:r1]
        # plain Gram: local raw sums, then the sum-combine
        G, c, yy = orc.gram(Xs, ys, nthreads=1)
        t = torch.from_numpy(np.concatenate([G.ravel(), c, [yy, r1 - r0]]))
        dist.all_reduce(t, op=dist.ReduceOp.SUM)
        # fold Grams with the global row offset as the fold phase
        Gk, ck, yyk, cnt = orc.gram_folds(Xs, ys, K, row_offset=r0, nthreads=1)
        assert list(cnt) == fold_counts(r1 - r0, r0, K)
        tf = torch.from_numpy(np.concatenate([Gk.ravel(), ck.ravel(), yyk, cnt.astype(float)]))
        dist.all_reduce(tf, op=dist.ReduceOp.SUM)
        # weighted Gram and logistic gradient (a4 / f1): per-rank raw sums combine to the
        # single-process ones (beta replicated on every rank)
        y01 = (ys > 0).astype(float)
        beta = np.linspace(-0.3, 0.2, p)
        Gw, cw, sw = orc.gram_weighted(Xs, y01, beta, nthreads=1)
        g, ll = orc.logit_grad(Xs, y01, beta)
        tw = torch.from_numpy(np.concatenate([Gw.ravel(), cw, sw, g, [ll]]))
        dist.all_reduce(tw, op=dist.ReduceOp.SUM)
        if rank == 0:
            q.put((t.numpy().copy(), tf.numpy().copy(), tw.numpy().copy()))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_sharded_combine_equals_single_process(world):
    n, p, K = 1003, 6, 10
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = free_port()
    procs = [ctx.Process(target=worker, args=(r, world, port, n, p, K, q)) for r in range(world)]
    for pr in procs:
        pr.start()
    t, tf, tw = q.get(timeout=120)
    for pr in procs:
        pr.join(timeout=120)
        assert pr.exitcode == 0
    X, y = design(n, p)
    G, c, yy = orc.gram(X, y)
    assert np.array_equal(t[: p * p].reshape(p, p), G)
    assert np.array_equal(t[p * p: p * p + p], c)
    assert t[-2] == yy and t[-1] == n
    Gk, ck, yyk, cnt = orc.gram_folds(X, y, K)
    off = 0
    assert np.array_equal(tf[off: off + K * p * p].reshape(K, p, p), Gk)
    off += K * p * p
    assert np.array_equal(tf[off: off + K * p].reshape(K, p), ck)
    off += K * p
    assert np.array_equal(tf[off: off + K], yyk)
    assert np.array_equal(tf[off + K:], cnt.astype(float))
    # combined weighted statistics equal the single-process ones (up to the order of the sums)
    y01 = (y > 0).astype(float)
    beta = np.linspace(-0.3, 0.2, p)
    Gw, cw, sw = orc.gram_weighted(X, y01, beta)
    g, ll = orc.logit_grad(X, y01, beta)
    ref = np.concatenate([Gw.ravel(), cw, sw, g, [ll]])
    assert np.allclose(tw, ref, rtol=1e-12, atol=1e-9)


def test_row_range_and_fold_counts():
    for n in (10, 1003, 10_000_000):
        for world in (1, 2, 4, 8):
            rr = [row_range(n, world, r) for r in range(world)]
            assert rr[0][0] == 0 and rr[-1][1] == n
            assert all(rr[i][1] == rr[i + 1][0] for i in range(world - 1))
            if n >= 80:
                K = 10
                tot = np.sum([fold_counts(r1 - r0, r0, K) for r0, r1 in rr], axis=0)
                assert list(tot) == [len(range(k, n, K)) for k in range(K)]
    # cfg3: n divisible by 80 -> every rank's fold phase is 0
    assert all(row_range(10_000_000, 8, r)[0] % 10 == 0 for r in range(8))
