"""One rank of the multi-GPU parity run (tests/test_gpu_multirank.py), launched by torchrun with
one rank per GPU (or directly at world size 1). Each rank generates ITS rows of the design on
its GPU, the library combines the raw statistics with its NCCL allreduce, and:
  - every rank must hold bitwise-identical combined statistics and fits (all-gathered digests);
  - rank 0 compares the combined Gram, fold Grams, weighted Gram and the paths with the oracle
    over the whole design."""
import hashlib
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))

import numpy as np  # noqa: E402
import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402

import datagen as dg  # noqa: E402
from datagen.configs import CONFIGS  # noqa: E402
from paper_1801_09661_b200 import (Context, oem, oem_fit_path, oem_gram, oem_gram_folds,  # noqa: E402
                                   oem_gram_weighted)
from paper_1801_09661_b200.shard import row_range  # noqa: E402


def digest(*ts):
    h = hashlib.sha256()
    for t in ts:
        h.update(t.detach().cpu().numpy().tobytes())
    return h.hexdigest()


def main():
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    if world > 1:
        os.environ.setdefault("NCCL_ALGO", "Ring")
        os.environ.setdefault("NCCL_PROTO", "Simple")
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        obj = [oem.oem_nccl_unique_id() if rank == 0 else None]
        dist.broadcast_object_list(obj, src=0)
        ctx = Context(local, world, rank, obj[0])
    else:
        ctx = Context(local)
    spec = CONFIGS["cfg3"].spec.replace(n=40_007, p=96, nnz=8)
    K = 10
    bt = dg.beta(spec)
    r0, r1 = row_range(spec.n, world, rank)
    nl = r1 - r0
    ldx = spec.p
    Xs = torch.empty((max(nl, 1), ldx), dtype=torch.float64, device="cuda")
    yd = torch.empty(max(nl, 1), dtype=torch.float64, device="cuda")
    btd = torch.from_numpy(bt).cuda()
    dg.rows_cuda(spec, btd.data_ptr(), r0, nl, Xs.data_ptr(), ldx, yd.data_ptr(),
                 torch.cuda.current_stream().cuda_stream)
    Xd, yd = Xs[:nl], yd[:nl]
    G, c, yy, n = oem_gram(ctx, Xd, yd)
    Gk, ck, yyk, cnt = oem_gram_folds(ctx, Xd, yd, K, row_offset=r0)
    y01 = (yd > 0).double()
    beta = torch.linspace(-0.1, 0.1, spec.p, dtype=torch.float64, device="cuda")
    Gw, cw, sw = oem_gram_weighted(ctx, Xd, y01, beta)
    fit = oem_fit_path(ctx, G, c, [n], [("lasso", 0, 1), ("mcp", 3, 1)], nlambda=12)
    cvf = oem_fit_path(ctx, Gk, ck, cnt, [("lasso", 0, 1)], nlambda=8, fold_mode=True)
    # the sparse pass over this rank's rows in CSR form (f4)
    from paper_1801_09661_b200 import oem_gram_csr
    sspec = CONFIGS["sparse"].spec.replace(n=40_007, p=96, nnz=8)
    sbt = dg.beta(sspec)
    rp, scol, sval, sy = dg.csr_cuda(sspec, sbt, r0, nl)
    Gs, cs, yys, ns = oem_gram_csr(ctx, rp, scol, sval, sy, sspec.p)
    # the one-pass column sums (ones column), whole data and per fold
    from paper_1801_09661_b200 import oem_gram_folds_sums, oem_gram_sums
    G1, c1, yy1, xs1, ys1, n1 = oem_gram_sums(ctx, Xd, yd)
    _, _, _, xsk, ysk, _ = oem_gram_folds_sums(ctx, Xd, yd, K, row_offset=r0)
    mine = digest(G, c, yy, Gk, ck, yyk, Gw, cw, sw, fit.beta, fit.d, cvf.beta, cvf.d, Gs, cs, yys, G1, xs1, ys1,
                  xsk, ysk)
    digests = [None] * world
    if world > 1:
        dist.all_gather_object(digests, mine)
    else:
        digests = [mine]
    if len(set(digests)) != 1:
        print("MR_WORKER_FAIL: ranks disagree", digests, flush=True)
        return 1
    if rank == 0:
        import oracle as orc
        from gpu_util import scale_err, xty_err
        X, y = dg.rows_host(spec, bt)
        assert n == spec.n and sum(cnt) == spec.n
        Go, co, yyo = orc.gram(X, y)
        assert scale_err(G.cpu().numpy(), Go) <= 1e-12
        assert xty_err(c.cpu().numpy(), co, Go, yyo) <= 1e-12
        Gfo, cfo, yyfo, cnto = orc.gram_folds(X, y, K)
        assert list(cnto) == list(cnt)
        for k in range(K):
            assert scale_err(Gk[k].cpu().numpy(), Gfo[k]) <= 1e-12
        Gwo, cwo, swo = orc.gram_weighted(X, (y > 0).astype(float), beta.cpu().numpy())
        assert scale_err(Gw.cpu().numpy(), Gwo) <= 1e-12
        d_ref = orc.d_rule(Go / n)[0]
        assert abs(float(fit.d[0]) - d_ref) <= 1e-11 * d_ref
        for q, (fam, gamma, alpha) in enumerate([("lasso", 0, 1), ("mcp", 3, 1)]):
            lam = orc.lambda_grid(orc.lambda_max(fam, co / n), 12)
            B, it, cv = orc.oem_path(Go / n, co / n, d_ref, fam, lam, gamma, alpha)
            assert np.max(np.abs(fit.beta[0, q].cpu().numpy() - B)) <= 1e-8
        assert n1 == spec.n and scale_err(G1.cpu().numpy(), Go) <= 1e-12
        xabs = np.abs(X).sum(axis=0)
        assert np.max(np.abs(xs1.cpu().numpy() - X.sum(axis=0)) / xabs) <= 1e-12
        assert abs(float(ys1) - y.sum()) <= 1e-12 * np.abs(y).sum()
        fold = (np.arange(spec.n)) % K
        for k in range(K):
            assert np.max(np.abs(xsk[k].cpu().numpy() - X[fold == k].sum(axis=0)) / xabs) <= 1e-12
        Xs, yh = dg.rows_host(sspec, sbt)
        Gso, cso, yyso = orc.gram(Xs, yh)
        assert ns == sspec.n and scale_err(Gs.cpu().numpy(), Gso) <= 1e-12
        assert xty_err(cs.cpu().numpy(), cso, Gso, yyso) <= 1e-12
        print(f"MR_WORKER_OK world={world} digest={mine[:16]}", flush=True)
    ctx.close()
    if world > 1:
        dist.destroy_process_group()
    return 0


if __name__ == "__main__":
    sys.exit(main())
