"""One configs[1] level through the K3 tile kernel under the variant set by MLMC_MINRES_TILE_N<N> (read once
per process): device time of the level call (median of 5) and the per-sample records saved for a bit-for-bit
comparison between variants.   python tools/k3_variant.py <level> <out.npy>"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import workloads as W  # noqa: E402
from paper_2503_05533_b200 import Context, precision  # noqa: E402

level = int(sys.argv[1])
cfg = W.CONFIGS["C2"]
ctx = Context(field="expcov", m=cfg["m"], sigma2=cfg["sigma2"], corr_len=cfg["corr_len"], h0_inv=8, L_max=3,
              device=0, workspace_bytes=2 << 30)
n = cfg["N"][level]
tf, tc = cfg["tols"][level], cfg["tols"][level - 1] if level else cfg["tols"][0]
p = precision("minres")
ctx.sample_level(level, n, seed=1, prec_fine=p, prec_coarse=p, tol_fine=tf, tol_coarse=tc)
ts = []
for rep in range(5):
    a0, a1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    a0.record()
    r = ctx.sample_level(level, n, seed=1, first_index=n, prec_fine=p, prec_coarse=p, tol_fine=tf, tol_coarse=tc,
                         per_sample=True)
    a1.record()
    torch.cuda.synchronize()
    ts.append(a0.elapsed_time(a1))
np.save(sys.argv[2], r.per_sample)
env = {k: v for k, v in os.environ.items() if k.startswith("MLMC_MINRES_TILE")}
print(f"level {level} {env}: {np.median(ts):.3f} ms (min {min(ts):.3f}) iters {r.per_sample[:, 2].mean():.1f}", flush=True)
ctx.close()
