"""Per-step latency of one MINRES system on its resources: h = 1/64 tile (one CTA per system) and h = 1/128 /
1/256 K3b (one cluster per system), one wave of equal-length solves (max_iter = 300), device time / 300.
python tools/step_latency.py"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import workloads as W  # noqa: E402
from paper_2503_05533_b200 import Context, precision  # noqa: E402

cfg = W.CONFIGS["C5"]
ctx = Context(field=cfg["field"], m=cfg["m"], sigma2=cfg["sigma2"], corr_len=cfg["corr_len"], h0_inv=8, L_max=6,
              device=0, workspace_bytes=8 << 30)
pr = precision("minres", max_iter=300)
out = {}
for level, n in ((3, 148), (3, 1), (4, 33), (4, 1), (5, 8), (5, 1)):
    N = 8 << level
    ctx.sample_level(level, 2, seed=1, prec_fine=pr, prec_coarse=pr, tol_fine=1e-14, tol_coarse=1e-14)
    ctx.profile_enable(True)
    ctx.sample_level(level, n, seed=2, prec_fine=pr, prec_coarse=pr, tol_fine=1e-14, tol_coarse=1e-14)
    prof = ctx.profile_read()
    ctx.profile_enable(False)
    ms = sum(p[3] for p in prof if p[0] == "minres" and p[1] == N)
    out[f"h=1/{N} x{n}"] = {"us_per_step": ms * 1e3 / 300}
print(json.dumps(out))
ctx.close()
