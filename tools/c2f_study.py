"""NEXT-4 coarse-to-fine initial guess on the configs[1] levels (the bench workload): per level the pass time
(device events around the sampling call, L2 flushed) and the mean fine MINRES steps, from x0 = 0 (the fine and
coarse halves concurrent) and from x0 = P x_c (MLMC_FLAG_C2F: coarse half first, then the fine half).
    python tools/c2f_study.py"""
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
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
mr = precision("minres")
out = {}
for l in (1, 2, 3):
    n, tf, tc = cfg["N"][l], cfg["tols"][l], cfg["tols"][l - 1]
    row = {}
    for name, pf in (("x0=0", mr), ("x0=Pxc", precision("minres", c2f=True))):
        ctx.sample_level(l, n, seed=5, first_index=10**6, prec_fine=pf, prec_coarse=mr, tol_fine=tf, tol_coarse=tc)
        ts, its = [], []
        for rep in range(5):
            flush.zero_()
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record()
            r = ctx.sample_level(l, n, seed=5, first_index=rep * n, prec_fine=pf, prec_coarse=mr, tol_fine=tf,
                                 tol_coarse=tc)
            b.record()
            torch.cuda.synchronize()
            ts.append(a.elapsed_time(b))
            its.append(r.sums["iters_f"] / n)
        row[name] = {"ms_median": sorted(ts)[2], "mean_fine_steps": sum(its) / len(its)}
    row["step_ratio"] = row["x0=Pxc"]["mean_fine_steps"] / row["x0=0"]["mean_fine_steps"]
    row["time_ratio"] = row["x0=Pxc"]["ms_median"] / row["x0=0"]["ms_median"]
    out[f"l{l}"] = row
    print(json.dumps({f"l{l}": row}), flush=True)
ctx.close()
