"""Developer check: replicate the proximal-Newton loop step by step (not a test)."""
import os
import sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np
import torch
import datagen as dg
import oracle as orc
from datagen.configs import CONFIGS
from paper_1801_09661_b200 import Context, oem_gram_weighted, oem_fit_path

ctx = Context(0)
spec = CONFIGS["cfg5"].spec.replace(n=3000, p=5, nnz=3)
bt = dg.beta(spec)
X, y = dg.rows_host(spec, bt)
Xp = np.zeros((X.shape[0], 6)); Xp[:, :5] = X
Xd = torch.from_numpy(Xp).cuda()[:, :5]
yd = torch.from_numpy(y).cuda()
beta = torch.zeros(5, dtype=torch.float64, device="cuda")
for o in range(12):
    Gw, cw, sc = oem_gram_weighted(ctx, Xd, yd, beta)
    Go, co, so = orc.gram_weighted(X, y, beta.cpu().numpy())
    print("outer", o, "beta", beta.cpu().numpy(), "Gerr", float(np.max(np.abs(Gw.cpu().numpy() - Go))),
          "cerr", float(np.max(np.abs(cw.cpu().numpy() - co))), flush=True)
    print("  eig(Gw/n)", np.linalg.eigvalsh(Go / 3000), flush=True)
    try:
        fit = oem_fit_path(ctx, Gw, cw, [3000], [("lasso", 0.0, 1.0)], lambdas=[0.0], beta_init=beta.view(1, 1, 5))
    except Exception as ex:
        print("  fit error", ex, flush=True)
        pass
        break
    print("  d", float(fit.d[0]), "iters", int(fit.iters.sum()), "conv", int(fit.conv.sum()), flush=True)
    beta = fit.beta[0, 0, 0].clone()
