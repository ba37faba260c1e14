"""Device time of the d rule (drule_kernel, phase PH_POWER) vs p and the number of squarings S
(developer tool): oem_fit_path on a synthetic Gram with one lambda, timing enabled."""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

from paper_1801_09661_b200 import Context, oem, oem_fit_path  # noqa: E402


def main():
    ctx = Context(0)
    out = []
    for p, nU in ((20, 1), (100, 1), (200, 1), (500, 1), (500, 11), (1000, 1)):
        g = torch.Generator(device="cpu").manual_seed(p)
        Z = torch.randn(4 * p, p, generator=g, dtype=torch.float64)
        G = (Z.T @ Z).cuda().expand(nU, p, p).contiguous()
        c = torch.randn(nU, p, generator=g, dtype=torch.float64).cuda()
        for S in (0, 1, 4, 12):
            for rep in range(4):
                oem.set_timing(ctx, True)
                oem.stats(ctx, reset=True)
                oem_fit_path(ctx, G, c, [4 * p] * nU, [("lasso", 0, 1)], nlambda=1, d_squarings=S)
                torch.cuda.synchronize()
                st = oem.stats(ctx, reset=True)
            out.append({"p": p, "units": nU, "S": S, "d_ms": st["power_ms"]})
            print(json.dumps(out[-1]), flush=True)


if __name__ == "__main__":
    main()
