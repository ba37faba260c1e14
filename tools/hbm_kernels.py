"""Bandwidth of the HBM-bound kernels against MEASURED_PEAKS.json's copy bandwidth (developer
tool; results in profiles/hbm_kernels_<round>.json):

  logit_grad  (f1)  one pass over [X | y]: 8 (p+1) bytes per row             cfg5 shape (n 5e6, p 200)
  moments     (f3)  column sums of [X | y]: 8 (p+1) bytes per row            cfg4 shape (n 1e7, p 1000)
  weighted WZ (a4)  row_weights pre-pass + WZ contraction at p = 500          (times the whole call)

CUDA events around the public API call on the current stream, best of R after a warm-up."""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))

import numpy as np  # noqa: E402
import torch  # noqa: E402

import datagen as dg  # noqa: E402
from datagen.configs import CONFIGS  # noqa: E402
from gpu_util import device_rows  # noqa: E402
from paper_1801_09661_b200 import Context, oem_gram_moments, oem_gram_weighted, oem_logit_grad  # noqa: E402

PEAK = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))["hbm_gbs"] if os.path.exists(
    os.path.join(ROOT, "MEASURED_PEAKS.json")) else 6549.8


def best_ms(fn, reps=5):
    fn()
    out = []
    for _ in range(reps):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        fn()
        b.record()
        torch.cuda.synchronize()
        out.append(a.elapsed_time(b))
    return min(out)


def main():
    ctx = Context(0)
    res = {"peak_gbs": PEAK, "peak_source": "MEASURED_PEAKS.json hbm_gbs (copy)"}
    cfg = CONFIGS["cfg5"]
    bt = dg.beta(cfg.spec)
    Xd, yd = device_rows(cfg.spec, bt)
    beta = torch.from_numpy(0.5 * bt).cuda()
    nbytes = 8.0 * cfg.n * (cfg.p + 1)
    ms = best_ms(lambda: oem_logit_grad(ctx, Xd, yd, beta))
    res["logit_grad_cfg5"] = {"n": cfg.n, "p": cfg.p, "ms": ms, "gbs": nbytes / ms / 1e6, "frac": nbytes / ms / 1e6 / PEAK}
    ms = best_ms(lambda: oem_logit_grad(ctx, Xd, yd, beta, loglik=False))
    res["logit_grad_cfg5_no_loglik"] = {"n": cfg.n, "p": cfg.p, "ms": ms, "gbs": nbytes / ms / 1e6,
                                        "frac": nbytes / ms / 1e6 / PEAK, "note": "as the upper-bound fit calls it"}
    del Xd, yd
    torch.cuda.empty_cache()
    spec = cfg.spec.replace(p=500, nnz=20)
    bt = dg.beta(spec)
    Xd, yd = device_rows(spec, bt)
    beta = torch.from_numpy(0.5 * bt).cuda()
    ms = best_ms(lambda: oem_gram_weighted(ctx, Xd, yd, beta, scalars=False))
    res["weighted_p500"] = {"n": spec.n, "p": 500, "ms": ms, "tflops": spec.n * 500 * 506 / ms / 1e9}
    del Xd, yd
    torch.cuda.empty_cache()
    cfg = CONFIGS["cfg4"]
    bt = dg.beta(cfg.spec)
    Xd, yd = device_rows(cfg.spec, bt)
    ms = best_ms(lambda: oem_gram_moments(ctx, Xd, yd, 1, 0), reps=3)
    nbytes = 8.0 * cfg.n * (cfg.p + 1)
    res["moments_cfg4"] = {"n": cfg.n, "p": cfg.p, "ms": ms, "gbs": nbytes / ms / 1e6, "frac": nbytes / ms / 1e6 / PEAK}
    print(json.dumps(res))


if __name__ == "__main__":
    main()
