"""MINRES on the paper's Eq. (20) field (sigma = 2, contrast up to ~1e7): failures and iteration counts per level
and tolerance, 200 samples each -- the probe behind the default iteration cap 16 n + 1000.
python tools/_eq20_probe.py"""
import os
import sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import workloads as W
from paper_2503_05533_b200 import Context, precision
cfg = W.CONFIGS["EQ20"]
ctx = Context(field="eq20", m=cfg["m"], sigma2=cfg["sigma2"], corr_len=0.0, q_decay=cfg["q_decay"], h0_inv=cfg["h0_inv"], L_max=cfg["L_max"], device=0, workspace_bytes=2 << 30)
for l in range(5):
    for tol in (1e-6, 1e-10, 1e-12):
        r = ctx.sample_level(l, 200, seed=3, prec_fine=precision("minres"), tol_fine=tol, tol_coarse=tol, per_sample=True)
        ps = r.per_sample
        print(l, tol, "fails", r.sums["n_fail"], "iters mean/max", ps[:,2].mean(), ps[:,2].max(), "status", set(ps[:,6].tolist()), set(ps[:,7].tolist()))
