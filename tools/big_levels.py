"""Fine-mesh MINRES throughput (h = 1/128, 1/256, 1/512): one batch of systems per mesh, device-timed.

  python tools/big_levels.py [nb] [max_iter]

Prints per mesh: ms, iterations, node-iterations/s and GB/s on the algorithmic 80 B per node and
iteration -- the HBM roofline basis of the streaming levels."""
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import workloads as W  # noqa: E402
from paper_2503_05533_b200 import Context, precision  # noqa: E402

nb = int(sys.argv[1]) if len(sys.argv) > 1 else 148
mi = int(sys.argv[2]) if len(sys.argv) > 2 else 1000
cfg = W.CONFIGS["C5"]
ctx = Context(field="expcov", m=cfg["m"], sigma2=cfg["sigma2"], corr_len=cfg["corr_len"], h0_inv=cfg["h0_inv"],
              L_max=cfg["L_max"], device=0, workspace_bytes=8 << 30)
sums = torch.zeros(12, dtype=torch.float64, device="cuda")
out = {}
for level in (4, 5, 6):
    N = cfg["h0_inv"] << level
    prec = precision("minres", max_iter=mi)
    ctx.sample_level_async(level, 2, cfg["seed"], 10**6, prec, prec, 1e-14, 1e-14, sums_out=sums)   # warm-up
    ctx.profile_enable(True)
    a0, a1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a0.record()
    ctx.sample_level_async(level, nb, cfg["seed"], 0, prec, prec, 1e-14, 1e-14, sums_out=sums)  # max_iter bound
    a1.record()
    torch.cuda.synchronize()
    prof = ctx.profile_read()
    ctx.profile_enable(False)
    s = sums.cpu().numpy()
    n_f, n_c = (N - 1) ** 2, (N // 2 - 1) ** 2
    k_ms = {f"{k}_{NN}": ms for (k, NN, _, ms) in prof}
    node_it_f = s[7] * n_f
    ms_f = k_ms.get(f"minres_{N}", 0.0)
    out[f"h=1/{N}"] = {"nb": nb, "ms_total": a0.elapsed_time(a1), "kernel_ms_fine": ms_f,
                       "iters_fine_mean": s[7] / nb, "iters_coarse_mean": s[8] / nb,
                       "GBs_80B_fine": 80 * node_it_f / (ms_f / 1e3) / 1e9 if ms_f else None,
                       "kernels": k_ms}
    print(json.dumps({f"h=1/{N}": out[f"h=1/{N}"]}), flush=True)
ctx.close()
