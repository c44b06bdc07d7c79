"""Level pass time (both halves, CUDA events around sample_level_async) on configs[4] levels 4 and 5 -- A/B of
the coarse-half fork next to a K3b fine half.  python tools/fork_probe.py"""
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import workloads as W  # noqa: E402
from paper_2503_05533_b200 import Context, precision  # noqa: E402

cfg = W.CONFIGS["C5"]
ctx = Context(field=cfg["field"], m=cfg["m"], sigma2=cfg["sigma2"], corr_len=cfg["corr_len"], h0_inv=8, L_max=6,
              device=0, workspace_bytes=8 << 30)
mr = precision("minres")
sums = torch.zeros(12, dtype=torch.float64, device="cuda")
out = {}
for level, n, tol in ((4, 148, 1e-8), (5, 148, 1e-8)):
    ctx.sample_level_async(level, 4, 1, 10**6, mr, mr, tol, tol, sums_out=sums)
    ms = []
    for rep in range(2):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        ctx.sample_level_async(level, n, 2, rep * n, mr, mr, tol, tol, sums_out=sums)
        e1.record()
        torch.cuda.synchronize()
        ms.append(e0.elapsed_time(e1))
    out[f"level {level} (h = 1/{8 << level})"] = min(ms)
print(json.dumps({"fork": os.environ.get("MLMC_SCHED_FORK", "1"), **out}))
ctx.close()
