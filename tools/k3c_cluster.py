"""Streamed MINRES (K3c) on configs[4] fine levels under the CTAs-per-system setting of MLMC_STREAM_CLUSTER
(read once per process): device time of one sample_level call and the per-sample records (saved for the
bound comparison between settings).   python tools/k3c_cluster.py <level> <n> <tol> <out.npy>"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import workloads as W  # noqa: E402
from paper_2503_05533_b200 import Context, precision  # noqa: E402

level, n, tol = int(sys.argv[1]), int(sys.argv[2]), float(sys.argv[3])
cfg = W.CONFIGS["C5"]
ctx = Context(field="expcov", m=cfg["m"], sigma2=cfg["sigma2"], corr_len=cfg["corr_len"], h0_inv=cfg["h0_inv"],
              L_max=cfg["L_max"], device=0, workspace_bytes=8 << 30)
p = precision("minres")
ctx.sample_level(level, 2, seed=1, first_index=10**6, prec_fine=p, prec_coarse=p, tol_fine=1e-3, tol_coarse=1e-3)
a0, a1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
torch.cuda.synchronize()
a0.record()
r = ctx.sample_level(level, n, seed=1, prec_fine=p, prec_coarse=p, tol_fine=tol, tol_coarse=tol, per_sample=True)
a1.record()
torch.cuda.synchronize()
ps = r.per_sample
np.save(sys.argv[4], ps)
print(f"level {level} n {n} tol {tol:.1e} cluster={os.environ.get('MLMC_STREAM_CLUSTER', 'auto')}: "
      f"{a0.elapsed_time(a1):.1f} ms; fine iters mean {ps[:, 2].mean():.0f} max {ps[:, 2].max():.0f}; "
      f"status max {ps[:, 6:8].max():.0f}", flush=True)
ctx.close()
