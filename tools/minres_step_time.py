"""Per-step time of the on-chip MINRES kernels: one full wave of systems per mesh, fixed step count
(tol 1e-300 -> every system runs max_iter steps).  Prints us per step, per-SM node-steps per us and the
algorithmic FP64 rate (25 flops per unknown and step).  python tools/minres_step_time.py [steps]"""
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import workloads as W  # noqa: E402
from paper_2503_05533_b200 import Context, precision  # noqa: E402

steps = int(sys.argv[1]) if len(sys.argv) > 1 else 400
solver = sys.argv[2] if len(sys.argv) > 2 else "minres"
cfg = W.CONFIGS["C2"]
ctx = Context(field="expcov", m=cfg["m"], sigma2=cfg["sigma2"], corr_len=cfg["corr_len"], h0_inv=8, L_max=3,
              device=0, workspace_bytes=2 << 30)
pr = precision(solver, max_iter=steps)
sums = torch.zeros(12, dtype=torch.float64, device="cuda")
for level, nb in ((0, 148 * 32), (1, 148 * 4 * 3), (2, 148 * 3), (3, 148)):
    N = 8 << level
    ctx.sample_level_async(level, nb, 1, 0, pr, pr, 1e-300, 1e-300, sums_out=sums)
    ctx.profile_enable(True)
    ctx.sample_level_async(level, nb, 1, 0, pr, pr, 1e-300, 1e-300, sums_out=sums)
    prof = ctx.profile_read()
    ctx.profile_enable(False)
    ms = sum(r[3] for r in prof if r[0] == "minres" and r[1] == N)
    n = (N - 1) ** 2
    print(json.dumps({"solver": solver, "N": N, "systems": nb, "steps": steps, "us_per_step": ms * 1e3 / steps,
                      "alg_tflops": 25.0 * n * nb * steps / (ms / 1e3) / 1e12}), flush=True)
ctx.close()
