"""Timeline of one configs[1] step (all levels concurrently) from the MINRES job trace of the tuning build
(mlmc_debug_trace): per mesh the first start / last end of its solves, and the busy SMs over time.
MLMC_TUNING=1 build; python tools/step_trace.py [out.json]"""
import ctypes as C
import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import workloads as W  # noqa: E402
from paper_2503_05533_b200 import Context, precision  # noqa: E402
from paper_2503_05533_b200 import _capi as K  # noqa: E402

cfg = W.CONFIGS["C2"]
Nl, tols, seed = cfg["N"], cfg["tols"], cfg["seed"]
dev = torch.device("cuda", 0)
stream = torch.cuda.current_stream(dev)
ctx = Context(field="expcov", m=cfg["m"], sigma2=cfg["sigma2"], corr_len=cfg["corr_len"], h0_inv=8, L_max=3, device=0,
              workspace_bytes=2 << 30, stream=stream)
mr = precision("minres")
sums = torch.zeros((4, 12), dtype=torch.float64, device=dev)
levels = [0, 1, 2, 3]
tol_c = [tols[l - 1] if l else tols[0] for l in levels]


def step(i):
    ctx.sample_levels_async(levels, Nl, seed, [(i + 77) * n for n in Nl], [mr] * 4, [mr] * 4, tols, tol_c, sums)


for i in range(3):
    step(i)
torch.cuda.synchronize()
cap = 40000
buf = torch.zeros(cap * 4, dtype=torch.int64, device=dev)
cnt = C.c_uint32()
K.check(K.lib().mlmc_debug_trace(ctx.ctx, C.c_void_p(buf.data_ptr()), cap, C.byref(cnt)), ctx.ctx)
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record(stream)
step(10)
e1.record(stream)
torch.cuda.synchronize()
K.check(K.lib().mlmc_debug_trace(ctx.ctx, None, 0, C.byref(cnt)), ctx.ctx)
n = min(cnt.value, cap)
t = buf[: 4 * n].view(n, 4).cpu().numpy().astype(np.uint64)
t0 = t[:, 0].min()
start, end = (t[:, 0] - t0) / 1e3, (t[:, 1] - t0) / 1e3            # microseconds
sm, mesh = (t[:, 2] >> np.uint64(32)).astype(int), (t[:, 2] & np.uint64(0xffffffff)).astype(int)
half = ((t[:, 3] >> np.uint64(32)) & np.uint64(1)).astype(int)          # 0 fine, 1 coarse
mesh = mesh * 10 + half                                                  # key: N * 10 + half
out = {"step_ms_events": e0.elapsed_time(e1), "records": int(n), "span_us": float(end.max()), "meshes": {}}
for N in sorted(set(mesh.tolist())):
    k = mesh == N
    d = end[k] - start[k]
    out["meshes"][f"N={N // 10} {'coarse' if N % 10 else 'fine'}"] = {"solves": int(k.sum()), "first_start_us": float(start[k].min()),
                             "last_start_us": float(start[k].max()), "last_end_us": float(end[k].max()),
                             "mean_us": float(d.mean()), "max_us": float(d.max()), "sum_ms": float(d.sum() / 1e3)}
# busy SMs over time (a solve occupies its SM from start to end; several groups of one CTA overlap)
bins = np.arange(0.0, end.max() + 25.0, 25.0)
busy = []
for b0 in bins:
    b1 = b0 + 25.0
    act = (start < b1) & (end > b0)
    busy.append(len(set(sm[act].tolist())))
out["busy_sms_per_25us"] = busy
out["mean_busy_sms"] = float(np.mean(busy))
print(json.dumps(out))
if len(sys.argv) > 1:
    json.dump({"raw": t.tolist(), **out}, open(sys.argv[1], "w"))
ctx.close()
