"""Robustness sweep: adaptive runs over configs, policies, seeds and tolerances on one GPU; every run must
return MLMC_OK or MLMC_ELMAX with an estimate in the fields' sanity range and no failed solves (on_fail = 2
escalates failed MINRES solves to MG-PCG and counts what still fails).   python tools/fuzz_adaptive.py [runs] [smallest eps]"""
import math
import os
import random
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import workloads as W  # noqa: E402
from paper_2503_05533_b200 import Context  # noqa: E402

runs = int(sys.argv[1]) if len(sys.argv) > 1 else 60
EPS_LO = float(sys.argv[2]) if len(sys.argv) > 2 else 1.5e-4
rng = random.Random(2025)
ctxs = {}
bad = 0
t0 = time.perf_counter()
for i in range(runs):
    name = rng.choice(["C2", "C4", "C5", "EQ20"])
    cfg = W.CONFIGS[name]
    if name not in ctxs:
        L_max = {"C2": 3, "C4": 5, "C5": 6, "EQ20": 4}[name]
        ctxs[name] = Context(field=cfg["field"], m=cfg["m"], sigma2=cfg["sigma2"], corr_len=cfg["corr_len"],
                             q_decay=cfg.get("q_decay", 2.0), h0_inv=cfg["h0_inv"], L_max=L_max, device=0,
                             workspace_bytes=4 << 30)
    ctx = ctxs[name]
    policy = rng.choice([0, 1, 2, 3])
    eps = 10 ** rng.uniform(math.log10(EPS_LO), math.log10(2e-3))
    k_p = rng.choice([0.05, 0.05, 0.2, 0.0])
    seed = rng.randrange(1 << 30)
    try:
        r = ctx.adaptive_run(eps, k_p=k_p, seed=seed, policy=policy, N_init=rng.choice([20, 100]), on_fail=2,
                             fixed_tol=1e-8)
        ok = r["code"] in (0, 4) and 0.02 < r["estimate"] < 0.05 and r["n_fail"] == 0
    except Exception as e:  # noqa: BLE001
        r, ok = {"error": str(e)}, False
    if not ok:
        bad += 1
        print("BAD", name, policy, f"{eps:.2e}", k_p, seed, r, flush=True)
print(f"{runs} runs, {bad} bad, {time.perf_counter() - t0:.1f} s")
for c in ctxs.values():
    c.close()
sys.exit(1 if bad else 0)
