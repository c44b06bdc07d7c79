"""Per-sample records of configs[1] level 3 (h = 1/64 fine) with the current MINRES path, as JSON (A/B checks
of tuning variants across processes).  python tools/k3b_ab.py OUT.json"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import workloads as W  # noqa: E402
from paper_2503_05533_b200 import Context, precision  # noqa: E402

cfg = W.CONFIGS["C2"]
ctx = Context(field="expcov", m=cfg["m"], sigma2=cfg["sigma2"], corr_len=cfg["corr_len"], h0_inv=8, L_max=3, device=0,
              workspace_bytes=2 << 30)
mr = precision("minres")
r = ctx.sample_level(3, 300, seed=7, prec_fine=mr, prec_coarse=mr, tol_fine=1e-8, tol_coarse=1e-6, per_sample=True)
json.dump(r.per_sample.tolist(), open(sys.argv[1], "w"))
ctx.close()
