"""configs[4] at small eps (SURVEY section 8(d) 'C5-small-eps'): adaptive MPML down to the finest levels
of the 7-level hierarchy (h = 1/8 .. 1/512), MINRES policy 0 (K3 on chip, K3c streamed) or policy 2
(MG-PCG on h = 1/32, 1/64).  python tools/small_eps.py [eps] [policy]"""
import json
import os
import sys
import time

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import workloads as W  # noqa: E402
from paper_2503_05533_b200 import Context, precision  # noqa: E402

eps = float(sys.argv[1]) if len(sys.argv) > 1 else 2e-5
policy = int(sys.argv[2]) if len(sys.argv) > 2 else 0
cfg = W.CONFIGS["C5"]
ctx = Context(field="expcov", m=cfg["m"], sigma2=cfg["sigma2"], corr_len=cfg["corr_len"], h0_inv=cfg["h0_inv"],
              L_max=cfg["L_max"], device=0, workspace_bytes=16 << 30)
ctx.adaptive_run(1e-3, k_p=cfg["k_p"], seed=99, policy=policy)          # warm-up (plan, kernels)
for l in range(cfg["L_max"] + 1):                                        # KL tables of every level on HBM
    p = precision("mgcg" if policy == 2 and (cfg["h0_inv"] << l) >= 32 else "minres")
    ctx.sample_level(l, 1, seed=98, prec_fine=p, prec_coarse=p, tol_fine=1e-6, tol_coarse=1e-6)
torch.cuda.synchronize()
t0 = time.perf_counter()
r = ctx.adaptive_run(eps, k_p=cfg["k_p"], N_init=100, seed=cfg["seed"], policy=policy, on_fail=1)
torch.cuda.synchronize()
el = time.perf_counter() - t0
prof = None
if len(sys.argv) > 3 and sys.argv[3] == "prof":       # per kernel class device time (events: a second run)
    ctx.profile_enable(True)
    ctx.adaptive_run(eps, k_p=cfg["k_p"], N_init=100, seed=cfg["seed"], policy=policy, on_fail=1)
    prof = [(k, n, c, round(ms, 2)) for k, n, c, ms in ctx.profile_read() if ms > 0.5]
    ctx.profile_enable(False)
print(json.dumps({"eps": eps, "policy": policy, "seconds": el, "solve_seconds": r["solve_seconds"], "L": r["L"],
                  "N": r["N"], "eps_l": r["eps"], "mean": r["mean"], "var": r["var"], "cost": r["cost"],
                  "estimate": r["estimate"], "rounds": r["rounds"], "code": r["code"], "n_fail": r["n_fail"],
                  "profile_ms": prof}))
ctx.close()
