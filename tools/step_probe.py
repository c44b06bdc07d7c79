"""Is the configs[1] step bound by level 3's longest solve or by the total work?  Times the concurrent step
(mlmc_sample_levels_async, all levels, L2 flushed, CUDA events) with level 3's sample count varied and with
single levels alone.  python tools/step_probe.py"""
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import workloads as W  # noqa: E402
from paper_2503_05533_b200 import Context, precision  # noqa: E402

cfg = W.CONFIGS["C2"]
Nl, tols, seed, m = cfg["N"], cfg["tols"], cfg["seed"], cfg["m"]
dev = torch.device("cuda", 0)
stream = torch.cuda.current_stream(dev)
ctx = Context(field="expcov", m=m, sigma2=cfg["sigma2"], corr_len=cfg["corr_len"], h0_inv=cfg["h0_inv"], L_max=3,
              device=0, workspace_bytes=2 << 30, stream=stream)
mr = precision("minres")
flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
sums = torch.zeros((4, 12), dtype=torch.float64, device=dev)


def run(levels, n, steps=20, warm=3):
    tol_f = [tols[l] for l in levels]
    tol_c = [tols[l - 1] if l else tols[0] for l in levels]
    tot = 0.0
    for i in range(warm + steps):
        first = [(i + 1000) * Nl[l] for l in levels]
        flush.zero_()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        ctx.sample_levels_async(levels, n, seed, first, [mr] * len(levels), [mr] * len(levels), tol_f, tol_c,
                                sums[:len(levels)])
        e1.record(stream)
        torch.cuda.synchronize()
        if i >= warm:
            tot += e0.elapsed_time(e1)
    return tot / steps


out = {}
out["all levels, N = (20000, 5000, 1200, 300)"] = run([0, 1, 2, 3], [20000, 5000, 1200, 300])
if os.environ.get("STEP_PROBE_QUICK") == "1":          # the full step only (tuning A/B)
    out["sums_sha"] = __import__("hashlib").sha1(sums.cpu().numpy().tobytes()).hexdigest()[:16]
    print(json.dumps(out))
    ctx.close()
    sys.exit(0)
for n3 in (148, 200, 450, 600):
    out[f"all levels, level 3 N = {n3}"] = run([0, 1, 2, 3], [20000, 5000, 1200, n3])
out["levels 0-2 only"] = run([0, 1, 2], [20000, 5000, 1200])
for l in range(4):
    out[f"level {l} alone"] = run([l], [Nl[l]])
out["level 3 alone, N = 148"] = run([3], [148])
for k, v in out.items():
    print(f"{k:45s} {v:7.3f} ms")
print(json.dumps(out))
ctx.close()
