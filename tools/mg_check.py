"""MG-PCG (NEXT-4) vs MINRES on configs[1]: per level, iterations, Q difference, time (device)."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import workloads as W  # noqa: E402
from paper_2503_05533_b200 import Context, precision  # noqa: E402

cfg = W.CONFIGS["C2"]
ctx = Context(field="expcov", m=cfg["m"], sigma2=cfg["sigma2"], corr_len=cfg["corr_len"], h0_inv=8, L_max=3,
              device=0, workspace_bytes=2 << 30)
for level, n in enumerate(cfg["N"]):
    tf, tc = cfg["tols"][level], cfg["tols"][level - 1] if level else cfg["tols"][0]
    res = {}
    for name in ("minres", "mgcg"):
        p = precision(name)
        ctx.sample_level(level, n, seed=1, prec_fine=p, prec_coarse=p, tol_fine=tf, tol_coarse=tc)   # warm-up
        a0, a1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        a0.record()
        r = ctx.sample_level(level, n, seed=1, first_index=n, prec_fine=p, prec_coarse=p, tol_fine=tf, tol_coarse=tc,
                             per_sample=True)
        a1.record()
        torch.cuda.synchronize()
        res[name] = (r.per_sample, a0.elapsed_time(a1))
    a, b = res["minres"][0], res["mgcg"][0]
    dq = np.max(np.abs(a[:, 0] - b[:, 0]) / np.abs(a[:, 0]))
    print(f"level {level}: minres {res['minres'][1]:.3f} ms iters {a[:, 2].mean():.1f} | mgcg {res['mgcg'][1]:.3f} ms "
          f"iters {b[:, 2].mean():.1f} max {b[:, 2].max():.0f} status {b[:, 6].max():.0f} relres {b[:, 4].max():.2e} | "
          f"max rel dQ {dq:.2e} (tol {tf:.0e})", flush=True)
ctx.close()
