"""One configs[4] level-4 batch (h = 1/128 fine on K3b): python tools/k3b_one.py [n] [tol] (ncu target)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import workloads as W  # noqa: E402
from paper_2503_05533_b200 import Context, precision  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 148
tol = float(sys.argv[2]) if len(sys.argv) > 2 else 1e-8
cfg = W.CONFIGS["C5"]
ctx = Context(field=cfg["field"], m=cfg["m"], sigma2=cfg["sigma2"], corr_len=cfg["corr_len"], h0_inv=8, L_max=6,
              device=0, workspace_bytes=4 << 30)
mr = precision("minres", max_iter=300)
ctx.sample_level(4, 4, seed=1, prec_fine=mr, prec_coarse=mr, tol_fine=tol, tol_coarse=tol)
r = ctx.sample_level(4, n, seed=2, prec_fine=mr, prec_coarse=mr, tol_fine=tol, tol_coarse=tol)
print("steps", r.sums["iters_f"] / n)
ctx.close()
