"""Run configs[2] (C3) at one level / factor format: python tools/c3_one.py LEVEL {h|s} [N_SAMPLES] (ncu target)."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import workloads as W  # noqa: E402
from paper_2503_05533_b200 import Context, precision  # noqa: E402

level, uf = int(sys.argv[1]), sys.argv[2]
n = int(sys.argv[3]) if len(sys.argv) > 3 else 100000
cfg = W.CONFIGS["C3"]
ctx = Context(field="expcov", m=cfg["m"], sigma2=cfg["sigma2"], corr_len=cfg["corr_len"], h0_inv=cfg["h0_inv"],
              L_max=cfg["L_max"], device=0, workspace_bytes=int(os.environ.get("C3_WS_GB", "4")) << 30)
sums = torch.zeros(12, dtype=torch.float64, device="cuda")
prec = precision("chol_ir", uf, "s")
ctx.sample_level_async(level, 2000, cfg["seed"], 10**7, prec, prec, cfg["tol"], cfg["tol"], sums_out=sums)
a0, a1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
a0.record()
ctx.sample_level_async(level, n, cfg["seed"], 0, prec, prec, cfg["tol"], cfg["tol"], sums_out=sums)
a1.record()
torch.cuda.synchronize()
print(f"level {level} u_f {uf}: {n} samples in {a0.elapsed_time(a1):.3f} ms; mean steps {sums[7].item() / n:.3f}")
ctx.close()
