"""MG-PCG (K3m-g) vs streamed MINRES (K3c) on the fine meshes of configs[4] (h = 1/128 .. 1/512):
per level, device time of one sample_level call, iterations, max relative Q difference.
  python tools/mg_fine.py [n] [tol]"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import workloads as W  # noqa: E402
from paper_2503_05533_b200 import Context, precision  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 148
tol = float(sys.argv[2]) if len(sys.argv) > 2 else 1e-6
solvers = ("mgcg",) if len(sys.argv) > 3 and sys.argv[3] == "mg" else ("mgcg", "minres")
cfg = W.CONFIGS["C5"]
ctx = Context(field="expcov", m=cfg["m"], sigma2=cfg["sigma2"], corr_len=cfg["corr_len"], h0_inv=cfg["h0_inv"],
              L_max=cfg["L_max"], device=0, workspace_bytes=12 << 30)
for level in (4, 5, 6):
    res = {}
    for name in solvers:
        p = precision(name)
        ctx.sample_level(level, 2, seed=1, prec_fine=p, prec_coarse=p, tol_fine=tol, tol_coarse=tol)   # warm-up
        a0, a1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        a0.record()
        r = ctx.sample_level(level, n, seed=1, first_index=10, prec_fine=p, prec_coarse=p, tol_fine=tol,
                             tol_coarse=tol, per_sample=True)
        a1.record()
        torch.cuda.synchronize()
        res[name] = (r.per_sample, a0.elapsed_time(a1))
    if "minres" not in res:
        b = res["mgcg"][0]
        print(f"level {level} h=1/{8 << level} n {n} tol {tol:.0e}: mgcg {res['mgcg'][1]:.1f} ms iters "
              f"{b[:, 2].mean():.1f} max {b[:, 2].max():.0f} status {b[:, 6:8].max():.0f}", flush=True)
        continue
    a, b = res["minres"][0], res["mgcg"][0]
    dq = np.max(np.abs(a[:, 0] - b[:, 0]) / np.abs(a[:, 0]))
    print(f"level {level} h=1/{8 << level} n {n} tol {tol:.0e}: minres {res['minres'][1]:.1f} ms iters "
          f"{a[:, 2].mean():.0f} | mgcg {res['mgcg'][1]:.1f} ms iters {b[:, 2].mean():.1f} max {b[:, 2].max():.0f} "
          f"status {b[:, 6:8].max():.0f} | max rel dQ {dq:.2e} | speed-up {res['minres'][1] / res['mgcg'][1]:.1f}",
          flush=True)
ctx.close()
