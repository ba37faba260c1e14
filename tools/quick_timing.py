"""Quick per-phase timings of the hot path on one config (developer tool, not the bench)."""
import argparse
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))

import numpy as np  # noqa: E402
import torch  # noqa: E402

import datagen as dg  # noqa: E402
from datagen.configs import CONFIGS, groups_of  # noqa: E402
from gpu_util import device_rows  # noqa: E402
from paper_1801_09661_b200 import Context, oem_fit_path, oem_gram, oem_gram_folds, oem_gram_weighted  # noqa: E402


def ev():
    return torch.cuda.Event(enable_timing=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--cfg", default="cfg2")
    ap.add_argument("--n", type=int, default=0)
    ap.add_argument("--p", type=int, default=0, help="override p (same design recipe)")
    ap.add_argument("--reps", type=int, default=3)
    ap.add_argument("--nofit", action="store_true")
    ap.add_argument("--plain", action="store_true", help="plain Gram pass even for folds / logistic workloads")
    ap.add_argument("--noscal", action="store_true", help="weighted pass without sum w / log-likelihood")
    a = ap.parse_args()
    cfg = CONFIGS[a.cfg]
    if a.n:
        cfg = cfg.with_n(a.n)
    if a.p:
        cfg.spec = cfg.spec.replace(p=a.p, nnz=min(cfg.spec.nnz, a.p))
    ctx = Context(0)
    bt = dg.beta(cfg.spec, cfg.explicit_beta)
    t0 = time.time()
    Xd, yd = device_rows(cfg.spec, bt)
    torch.cuda.synchronize()
    gen_s = time.time() - t0
    n, p = cfg.n, cfg.p
    flops = n * p * (p + 6) if (cfg.logistic and not a.plain) else n * p * (p + 3)
    out = {"cfg": cfg.name, "n": n, "p": p, "gen_s": gen_s}
    grp = groups_of(cfg)
    for r in range(a.reps + 1):
        e0, e1, e2 = ev(), ev(), ev()
        e0.record()
        if a.plain:
            G, c, yy, nn = oem_gram(ctx, Xd, yd)
            cnt = [nn]
        elif cfg.folds:
            G, c, yy, cnt = oem_gram_folds(ctx, Xd, yd, cfg.folds)
        elif cfg.logistic:
            G, c, sc = oem_gram_weighted(ctx, Xd, yd, torch.zeros(p, dtype=torch.float64, device="cuda"),
                                         scalars=not a.noscal)
            cnt = [n]
        else:
            G, c, yy, nn = oem_gram(ctx, Xd, yd)
            cnt = [nn]
        e1.record()
        if not a.nofit and not cfg.logistic and not a.plain:
            fit = oem_fit_path(ctx, G, c, cnt, cfg.penalties, nlambda=cfg.nlambda, fold_mode=bool(cfg.folds),
                               group=grp, ngroups=(p // cfg.group_size) if grp is not None else 0)
        e2.record()
        torch.cuda.synchronize()
        if r == 0 and a.reps > 0:
            continue
        g_ms = e0.elapsed_time(e1)
        f_ms = e1.elapsed_time(e2)
        out.setdefault("gram_ms", []).append(g_ms)
        out.setdefault("fit_ms", []).append(f_ms)
    if a.reps == 0:
        print(json.dumps(out))
        return
    out["gram_tflops"] = flops / (min(out["gram_ms"]) * 1e-3) / 1e12
    if not a.nofit and not cfg.logistic and not a.plain:
        out["iters_total"] = int(fit.iters.sum())
        out["iters_max_unit"] = int(fit.iters.sum(-1).max())
        out["us_per_iter"] = min(out["fit_ms"]) * 1e3 / max(1, out["iters_max_unit"])
        out["d"] = [float(x) for x in fit.d.cpu()]
    print(json.dumps(out))


if __name__ == "__main__":
    main()
