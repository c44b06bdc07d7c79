"""One-time costs a user meets: process start to a finished first adaptive run, by stage (import + build check,
context (plan: KL eigenpairs), first call of every level (its KL tables, kernel attribute / occupancy set-up),
first adaptive run (policy 0 and policy 3 pilots), second run.  python tools/cold_start.py"""
import json
import os
import sys
import time

t_start = time.perf_counter()
import torch  # noqa: E402

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import workloads as W  # noqa: E402
from paper_2503_05533_b200 import Context, precision  # noqa: E402

out = {}
torch.cuda.init()
out["import_s"] = time.perf_counter() - t_start
cfg = W.CONFIGS["C5"]
t = time.perf_counter()
ctx = Context(field="expcov", m=cfg["m"], sigma2=cfg["sigma2"], corr_len=cfg["corr_len"], h0_inv=8, L_max=6, device=0,
              workspace_bytes=8 << 30)
out["context_s"] = time.perf_counter() - t
mr = precision("minres")
for l in range(7):
    torch.cuda.synchronize()
    t = time.perf_counter()
    ctx.sample_level(l, 1, seed=1, prec_fine=mr, prec_coarse=mr, tol_fine=1e-4, tol_coarse=1e-4)
    torch.cuda.synchronize()
    out[f"first_call_level{l}_s"] = time.perf_counter() - t
for pol in (0, 3):
    for k in ("first", "second"):
        t = time.perf_counter()
        r = ctx.adaptive_run(cfg["eps"], k_p=cfg["k_p"], seed=7, policy=pol)
        out[f"adaptive_p{pol}_{k}_s"] = time.perf_counter() - t
print(json.dumps({k: round(v, 4) for k, v in out.items()}))
ctx.close()
