"""Policy 3 on configs[4] at eps = 1e-5: wall time of the first adaptive run (pilots included), the choice per
mesh (mlmc_auto_choice), and a second run with the choices cached.  python tools/auto_probe.py"""
import os
import sys
import time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import workloads as W
from paper_2503_05533_b200 import Context
cfg = W.CONFIGS["C5"]
ctx = Context(field="expcov", m=cfg["m"], sigma2=cfg["sigma2"], corr_len=cfg["corr_len"], h0_inv=8, L_max=6, device=0, workspace_bytes=16 << 30)
t=time.perf_counter(); r = ctx.adaptive_run(1e-5, k_p=0.05, seed=5, policy=3, on_fail=1); t1=time.perf_counter()-t
print("first run", round(t1,3), r["L"], r["N"])
for N in (8,16,32,64,128,256,512):
    try: print(N, ctx.auto_choice(N))
    except Exception as e: print(N, "none", e)
t=time.perf_counter(); r = ctx.adaptive_run(1e-5, k_p=0.05, seed=5, policy=3, on_fail=1); print("second run (choices cached)", round(time.perf_counter()-t,3))
