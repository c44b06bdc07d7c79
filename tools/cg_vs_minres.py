"""CG against MINRES on the configs[1] levels: per-level pass time (device events around the
sampling call, fine and coarse halves) and mean / max step counts, same seeds and tolerances.
  python tools/cg_vs_minres.py"""
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import workloads as W  # noqa: E402
from paper_2503_05533_b200 import Context, precision  # noqa: E402

cfg = W.CONFIGS["C2"]
ctx = Context(field="expcov", m=cfg["m"], sigma2=cfg["sigma2"], corr_len=cfg["corr_len"], h0_inv=8, L_max=3,
              device=0, workspace_bytes=2 << 30)
N = (20000, 5000, 1200, 300)
TOL = (1e-4, 1e-5, 1e-6, 1e-8)
out = {}
for l in range(4):
    row = {}
    for name in ("minres", "cg"):
        p = precision(name)
        kw = dict(prec_fine=p, prec_coarse=p, tol_fine=TOL[l], tol_coarse=TOL[l - 1] if l else TOL[l])
        ctx.sample_level(l, N[l], seed=1, **kw)
        ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
        torch.cuda.synchronize()
        ev[0].record()
        reps = 5
        for r in range(reps):
            res = ctx.sample_level(l, N[l], seed=1, first_index=r * N[l], per_sample=True, **kw)
        ev[1].record()
        torch.cuda.synchronize()
        rec = res.per_sample
        row[name] = {"ms": ev[0].elapsed_time(ev[1]) / reps, "mean_iters_f": float(rec[:, 2].mean()),
                     "max_iters_f": float(rec[:, 2].max()), "fails": int((rec[:, 6] != 0).sum())}
    row["cg_over_minres_time"] = row["cg"]["ms"] / row["minres"]["ms"]
    out[f"l{l}"] = row
    print(json.dumps({f"l{l}": row}), flush=True)
ctx.close()
