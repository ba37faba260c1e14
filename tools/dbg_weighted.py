"""Developer check: weighted Gram parity over small p and several beta scales (not a test)."""
import os
import sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
import numpy as np
import torch
import datagen as dg
import oracle as orc
from datagen.configs import CONFIGS
from gpu_util import device_rows, scale_err
from paper_1801_09661_b200 import Context, oem_gram_weighted

ctx = Context(0)
for p in [1, 2, 3, 5, 7, 8, 9, 16, 17, 33, 200]:
    for n in [31, 3000]:
        for sc in [0.0, 0.5, 3.0]:
            spec = CONFIGS["cfg5"].spec.replace(n=n, p=p, nnz=min(3, p))
            bt = dg.beta(spec)
            Xd, yd = device_rows(spec, bt)
            X, y = dg.rows_host(spec, bt)
            beta = sc * np.sin(np.arange(p) + 1.0)
            Gw, cw, s = oem_gram_weighted(ctx, Xd, yd, torch.from_numpy(beta).cuda())
            Go, co, so = orc.gram_weighted(X, y, beta)
            G = Gw.cpu().numpy()
            bad = not np.all(np.isfinite(G)) or not np.all(np.isfinite(cw.cpu().numpy()))
            e = scale_err(G, Go)
            ec = float(np.max(np.abs(cw.cpu().numpy() - co)) / max(1e-300, np.max(np.abs(co))))
            es = [float(abs(s[i].item() - so[i]) / max(1e-300, abs(so[i]))) for i in range(2)]
            flag = "BAD" if bad or e > 1e-12 or ec > 1e-10 or max(es) > 1e-12 else "ok"
            print(f"p={p} n={n} sc={sc} G {e:.1e} c {ec:.1e} s {es[0]:.1e} {es[1]:.1e} {flag}", flush=True)
