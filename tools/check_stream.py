"""Per-sample fine-mesh MINRES results (h = 1/128, 1/256) for an A/B between K3c (streamed) and the
three-phase global-memory kernel (MLMC_MINRES_GM=1): writes gpurun_out/stream_<tag>.npz."""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import workloads as W  # noqa: E402
from paper_2503_05533_b200 import Context, precision  # noqa: E402

tag = sys.argv[1]
cfg = W.CONFIGS["C5"]
ctx = Context(field="expcov", m=cfg["m"], sigma2=cfg["sigma2"], corr_len=cfg["corr_len"], h0_inv=cfg["h0_inv"],
              L_max=cfg["L_max"], device=0, workspace_bytes=4 << 30)
res = {}
for level, n, tol in ((4, 20, 1e-10), (5, 6, 1e-8)):
    r = ctx.sample_level(level, n, seed=5, prec_fine=precision("minres"), tol_fine=tol, tol_coarse=tol, per_sample=True)
    res[f"l{level}"] = r.per_sample
    print(tag, level, "Qf", r.per_sample[:3, 0], "iters", r.per_sample[:3, 2], "status", r.per_sample[:, 6].max())
os.makedirs("gpurun_out", exist_ok=True)
np.savez(f"gpurun_out/stream_{tag}.npz", **res)
ctx.close()
