"""Path-solver timings of one workload with the screened compact iterations on and off
(developer tool, not the bench): the Gram(s) are formed once at the workload's size, then
oem_fit_path runs --reps times per mode; prints the path phase per fit, the iterations of the
longest unit, microseconds per iteration and the largest |beta| difference between modes.

  python tools/path_timing.py --cfg cfg4 [--n N] [--solver active] [--reps 3]
"""
import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))

import torch  # noqa: E402

import datagen as dg  # noqa: E402
from datagen.configs import CONFIGS, groups_of  # noqa: E402
from gpu_util import device_rows  # noqa: E402
from paper_1801_09661_b200 import Context, oem_fit_path, oem_gram, oem_gram_folds  # noqa: E402
from paper_1801_09661_b200.oem import set_timing, stats  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--cfg", default="cfg4")
    ap.add_argument("--n", type=int, default=0)
    ap.add_argument("--solver", default="", help="OEM_PATH_SOLVER for both modes")
    ap.add_argument("--reps", type=int, default=3)
    ap.add_argument("--modes", default="0,1", help="OEM_SCREEN values to compare")
    ap.add_argument("--pen", type=int, default=-1, help="fit only penalty #pen of the workload")
    a = ap.parse_args()
    cfg = CONFIGS[a.cfg]
    if a.n:
        cfg = cfg.with_n(a.n)
    ctx = Context(0)
    bt = dg.beta(cfg.spec, cfg.explicit_beta)
    Xd, yd = device_rows(cfg.spec, bt)
    if cfg.folds:
        G, c, _, cnt = oem_gram_folds(ctx, Xd, yd, cfg.folds)
    else:
        G, c, _, nn = oem_gram(ctx, Xd, yd)
        cnt = [nn]
    del Xd, yd
    torch.cuda.empty_cache()
    grp = groups_of(cfg)
    kw = dict(nlambda=cfg.nlambda, fold_mode=bool(cfg.folds))
    if grp is not None:
        kw.update(group=grp, ngroups=int(grp.max()) + 1)
    if a.solver:
        os.environ["OEM_PATH_SOLVER"] = a.solver
    set_timing(ctx, True)
    res = {}
    for m in a.modes.split(","):
        os.environ["OEM_SCREEN"] = m
        ms = []
        for _ in range(a.reps + 1):
            stats(ctx, reset=True)
            pens = cfg.penalties if a.pen < 0 else [cfg.penalties[a.pen]]
            fit = oem_fit_path(ctx, G, c, cnt, pens, **kw)
            torch.cuda.synchronize()
            ms.append(stats(ctx)["path_ms"])
        it = int(fit.iters.sum(-1).max())
        res[m] = {"path_ms": min(ms[1:] or ms), "iters_max_unit": it, "us_per_iter": 1e3 * min(ms[1:] or ms) / it,
                  "iters_total": int(fit.iters.sum()), "beta": fit.beta.clone(),
                  "conv_all": bool(fit.conv.all())}
    modes = list(res)
    out = {"cfg": cfg.name, "solver": a.solver or "default"}
    for m in modes:
        out[f"screen={m}"] = {k: v for k, v in res[m].items() if k != "beta"}
    if os.environ.get("PT_DUMP"):
        for m in modes:
            b = res[m]["beta"]
            out[f"dump{m}"] = [float(b[0, 0, 39, 25]), float(b[0, 1, 45, 24]),
                               [float((res[m2]["beta"] - b).abs().max()) for m2 in modes]]
    if len(modes) > 1:
        out["max_abs_dbeta"] = float((res[modes[0]]["beta"] - res[modes[1]]["beta"]).abs().max())
    print(json.dumps(out))


if __name__ == "__main__":
    main()
