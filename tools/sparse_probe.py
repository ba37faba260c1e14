"""Time the CSR Gram pass (f4) on the 'sparse' workload shape (developer tool, not the bench).

    python tools/sparse_probe.py [--n N] [--p P] [--density D] [--reps R]"""
import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import datagen as dg  # noqa: E402
from datagen.configs import CONFIGS  # noqa: E402
from paper_1801_09661_b200 import Context, oem_gram_csr  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=int, default=10_000_000)
    ap.add_argument("--p", type=int, default=200)
    ap.add_argument("--density", type=float, default=0.01)
    ap.add_argument("--reps", type=int, default=5)
    a = ap.parse_args()
    spec = CONFIGS["sparse"].spec.replace(n=a.n, p=a.p, rho=a.density)
    bt = dg.beta(spec)
    rp, col, val, y = dg.csr_cuda(spec, bt)
    ctx = Context(0)
    ms = []
    for r in range(a.reps + 1):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        oem_gram_csr(ctx, rp, col, val, y, a.p)
        e1.record()
        torch.cuda.synchronize()
        if r:
            ms.append(e0.elapsed_time(e1))
    nbytes = 8 * (a.n + 1) + 8 * a.n + 12 * col.numel()
    print(json.dumps({"n": a.n, "p": a.p, "density": a.density, "nnz": int(col.numel()), "ms": ms,
                      "gbs": nbytes / (min(ms) * 1e-3) / 1e9}))


if __name__ == "__main__":
    main()
