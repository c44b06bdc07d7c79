"""C4-R / C5-R (SURVEY section 8(d) 'additional honest variants'; the estimator pin of section 8(c)):
R replicate adaptive MPML runs (seeds 0..R-1) of configs[3] / configs[4] at their eps, against a
reference Q_ref = the same GPU path at eps/5.  Reports RMSE(Q_hat - Q_ref) (must be <= eps), the mean
estimate, time per run (wall clock of mlmc_adaptive_run) and the L / N_l distribution.
  python tools/replicates.py [C4|C5] [R] [policy]"""
import json
import math
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import workloads as W  # noqa: E402
from paper_2503_05533_b200 import Context  # noqa: E402


def run(name="C4", R=100, policy=0, ref_seed=10**6):
    cfg = W.CONFIGS[name]
    ctx = Context(field=cfg["field"], m=cfg["m"], sigma2=cfg["sigma2"], corr_len=cfg["corr_len"],
                  h0_inv=cfg["h0_inv"], L_max=cfg["L_max"], device=0, workspace_bytes=8 << 30)
    eps = cfg["eps"]
    ref = ctx.adaptive_run(eps / 5, k_p=cfg["k_p"], seed=ref_seed, policy=policy, on_fail=1)
    ctx.adaptive_run(eps, k_p=cfg["k_p"], seed=ref_seed + 1, policy=policy)          # warm-up
    est, secs, Ls, Ns = [], [], [], []
    for r in range(R):
        torch.cuda.synchronize()
        t = time.perf_counter()
        a = ctx.adaptive_run(eps, k_p=cfg["k_p"], seed=r, policy=policy)
        secs.append(time.perf_counter() - t)
        est.append(a["estimate"])
        Ls.append(a["L"])
        Ns.append(a["N"])
        assert a["code"] == 0, a["code"]
    ctx.close()
    e = np.array(est)
    rmse = float(np.sqrt(np.mean((e - ref["estimate"]) ** 2)))
    return {"config": name, "eps": eps, "R": R, "policy": policy,
            "reference": {"eps": eps / 5, "estimate": ref["estimate"], "L": ref["L"], "N": ref["N"]},
            "rmse": rmse, "rmse_over_eps": rmse / eps, "mean_estimate": float(e.mean()),
            "std_estimate": float(e.std(ddof=1)), "seconds_per_run_mean": float(np.mean(secs)),
            "seconds_per_run_max": float(np.max(secs)), "L_hist": {str(L): Ls.count(L) for L in sorted(set(Ls))},
            "N0_mean": float(np.mean([n[0] for n in Ns]))}


if __name__ == "__main__":
    name = sys.argv[1] if len(sys.argv) > 1 else "C4"
    R = int(sys.argv[2]) if len(sys.argv) > 2 else 100
    policy = int(sys.argv[3]) if len(sys.argv) > 3 else 0
    res = run(name, R, policy)
    print(json.dumps(res))
