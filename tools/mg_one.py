"""One MG-PCG (K3m-g) sample_level call on configs[4] at level L (ncu target).  python tools/mg_one.py [L] [n] [tol]"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import workloads as W  # noqa: E402
from paper_2503_05533_b200 import Context, precision  # noqa: E402

L = int(sys.argv[1]) if len(sys.argv) > 1 else 6
n = int(sys.argv[2]) if len(sys.argv) > 2 else 148
tol = float(sys.argv[3]) if len(sys.argv) > 3 else 1e-6
cfg = W.CONFIGS["C5"]
ctx = Context(field="expcov", m=cfg["m"], sigma2=cfg["sigma2"], corr_len=cfg["corr_len"], h0_inv=cfg["h0_inv"],
              L_max=cfg["L_max"], device=0, workspace_bytes=12 << 30)
mg = precision("mgcg")
r = ctx.sample_level(L, n, seed=1, prec_fine=mg, prec_coarse=mg, tol_fine=tol, tol_coarse=tol, per_sample=True)
torch.cuda.synchronize()
print("iters fine", r.per_sample[:, 2].mean(), "coarse", r.per_sample[:, 3].mean())
ctx.close()
