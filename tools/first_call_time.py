"""Wall time of the first sample_level call per fine level (includes building the level's KL table on the host)."""
import time, sys, os
sys.path.insert(0, os.getcwd())
import torch
import workloads as W
from paper_2503_05533_b200 import Context, precision
cfg = W.CONFIGS["C5"]
ctx = Context(field="expcov", m=cfg["m"], sigma2=cfg["sigma2"], corr_len=cfg["corr_len"], h0_inv=8, L_max=6, device=0, workspace_bytes=4 << 30)
mg = precision("mgcg")
for l in (4, 5, 6):
    torch.cuda.synchronize(); t = time.perf_counter()
    ctx.sample_level(l, 1, seed=1, prec_fine=mg, prec_coarse=mg, tol_fine=1e-6, tol_coarse=1e-6)
    torch.cuda.synchronize(); print("first call level", l, round(time.perf_counter() - t, 3), "s", flush=True)
ctx.close()
