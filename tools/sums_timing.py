"""Time the Gram pass with and without the ones column (developer tool, not the bench): per
config, oem_gram (or oem_gram_folds) alone, oem_gram_sums (one pass over [X | y | 1]) and the
two-pass route oem_gram + oem_gram_moments; CUDA events on the current stream, median of reps.

    python tools/sums_timing.py [--cfgs cfg2,cfg3,cfg4] [--reps 5]"""
import argparse
import json
import os
import statistics
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))

import torch  # noqa: E402

import datagen as dg  # noqa: E402
from datagen.configs import CONFIGS  # noqa: E402
from gpu_util import device_rows  # noqa: E402
from paper_1801_09661_b200 import (Context, oem_gram, oem_gram_folds, oem_gram_folds_sums, oem_gram_moments,  # noqa: E402
                                   oem_gram_sums)


def timed(fn, reps):
    ms = []
    for r in range(reps + 1):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        fn()
        e1.record()
        torch.cuda.synchronize()
        if r:
            ms.append(e0.elapsed_time(e1))
    return statistics.median(ms)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--cfgs", default="cfg2,cfg3,cfg4")
    ap.add_argument("--reps", type=int, default=5)
    a = ap.parse_args()
    ctx = Context(0)
    for name in a.cfgs.split(","):
        cfg = CONFIGS[name]
        Xd, yd = device_rows(cfg.spec, dg.beta(cfg.spec, cfg.explicit_beta))
        K = cfg.folds or 1
        if cfg.folds:
            base = timed(lambda: oem_gram_folds(ctx, Xd, yd, K), a.reps)
            one = timed(lambda: oem_gram_folds_sums(ctx, Xd, yd, K), a.reps)
            two = timed(lambda: (oem_gram_folds(ctx, Xd, yd, K), oem_gram_moments(ctx, Xd, yd, K)), a.reps)
        else:
            base = timed(lambda: oem_gram(ctx, Xd, yd), a.reps)
            one = timed(lambda: oem_gram_sums(ctx, Xd, yd), a.reps)
            two = timed(lambda: (oem_gram(ctx, Xd, yd), oem_gram_moments(ctx, Xd, yd)), a.reps)
        print(json.dumps({"cfg": name, "n": cfg.n, "p": cfg.p, "K": K, "gram_ms": base, "gram_sums_ms": one,
                          "gram_plus_moments_ms": two}), flush=True)
        del Xd, yd
        torch.cuda.empty_cache()
    ctx.close()


if __name__ == "__main__":
    main()
