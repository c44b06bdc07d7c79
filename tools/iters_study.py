"""Per-sample MINRES iteration counts of configs[1] level 3 vs cheap predictors (LPT scheduling study).
Writes gpurun_out/iters_l3.npz: fine/coarse iterations and field statistics per sample."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import workloads as W  # noqa: E402
from paper_2503_05533_b200 import Context, precision  # noqa: E402

cfg = W.CONFIGS["C2"]
ctx = Context(field="expcov", m=cfg["m"], sigma2=cfg["sigma2"], corr_len=cfg["corr_len"], h0_inv=cfg["h0_inv"],
              L_max=3, device=0, workspace_bytes=1 << 30)
n = 1200
r = ctx.sample_level(3, n, seed=cfg["seed"], prec_fine=precision("minres"), tol_fine=cfg["tols"][3],
                     tol_coarse=cfg["tols"][2], per_sample=True)
ps = r.per_sample
xi, a = ctx.debug_field(3, 3, n, cfg["seed"])
la = torch.log(a).cpu().numpy()
stats = {"fine": ps[:, 2], "coarse": ps[:, 3], "contrast": la.max(1) - la.min(1), "var": la.var(1),
         "mean": la.mean(1)}
N = 64
g = la.reshape(n, N, N, 2)
stats["grad2"] = ((np.diff(g, axis=1) ** 2).sum((1, 2, 3)) + (np.diff(g, axis=2) ** 2).sum((1, 2, 3)))
os.makedirs("gpurun_out", exist_ok=True)
np.savez("gpurun_out/iters_l3.npz", **stats)
for k, v in stats.items():
    if k != "fine":
        print(k, "corr with fine iters:", np.corrcoef(v, stats["fine"])[0, 1])
print("fine iters: min", ps[:, 2].min(), "mean", ps[:, 2].mean(), "max", ps[:, 2].max())
