"""Per-kernel-class device time of one sample_level call (no concurrency: events are exact).
  python tools/level_profile.py [config] [level] [n] [solver]"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import workloads as W  # noqa: E402
from paper_2503_05533_b200 import Context, precision  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "C5"
level = int(sys.argv[2]) if len(sys.argv) > 2 else 0
n = int(sys.argv[3]) if len(sys.argv) > 3 else 1000000
solver = sys.argv[4] if len(sys.argv) > 4 else "minres"
cfg = W.CONFIGS[name]
ctx = Context(field=cfg["field"], m=cfg["m"], sigma2=cfg["sigma2"], corr_len=cfg["corr_len"],
              q_decay=cfg.get("q_decay", 2.0), h0_inv=cfg["h0_inv"], L_max=cfg["L_max"], device=0,
              workspace_bytes=16 << 30)
p = precision(solver)
tol = 1e-4
ctx.sample_level(level, n, seed=1, prec_fine=p, prec_coarse=p, tol_fine=tol, tol_coarse=tol)   # warm-up
ctx.profile_enable(True)
ctx.sample_level(level, n, seed=2, prec_fine=p, prec_coarse=p, tol_fine=tol, tol_coarse=tol)
st = ctx.profile_read()
ctx.profile_enable(False)
tot = sum(s[3] for s in st)
for k, N, c, ms in st:
    print(f"{name} level {level} n {n}: {k:8s} N={N:4d} launches {c:3d} {ms:9.3f} ms ({100 * ms / tot:4.1f}%)")
ctx.close()
