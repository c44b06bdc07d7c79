"""configs[2] level 2 (h = 1/32 fine, 1/16 coarse; 100000 coupled samples, Cholesky fp16 / fp32 + fp64 IR to
1e-10) against the workspace size, which sets the samples per pass: does a smaller pass (factors of fewer
samples in flight, fewer pages touched) run faster per sample?  python tools/c3_pass_size.py"""
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import workloads as W  # noqa: E402
from paper_2503_05533_b200 import Context, precision  # noqa: E402

cfg = W.CONFIGS["C3"]
sums = torch.zeros(12, dtype=torch.float64, device="cuda")
for ws in (1, 2, 4, 8, 16, 48):
    ctx = Context(field="expcov", m=cfg["m"], sigma2=cfg["sigma2"], corr_len=cfg["corr_len"], h0_inv=cfg["h0_inv"],
                  L_max=cfg["L_max"], device=0, workspace_bytes=ws << 30)
    row = {"workspace_GB": ws}
    for uf in ("h", "s"):
        prec = precision("chol_ir", uf, "s")
        ctx.sample_level_async(2, 2000, cfg["seed"], 10**7, prec, prec, cfg["tol"], cfg["tol"], sums_out=sums)
        a0, a1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a0.record()
        ctx.sample_level_async(2, 100000, cfg["seed"], 0, prec, prec, cfg["tol"], cfg["tol"], sums_out=sums)
        a1.record()
        torch.cuda.synchronize()
        row[f"ms_{uf}"] = a0.elapsed_time(a1)
    print(json.dumps(row), flush=True)
    ctx.close()
    del ctx
    torch.cuda.empty_cache()
