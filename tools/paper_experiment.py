"""The paper's MINRES experiment (Section 5.1) on the GPU: adaptive MPML (Algorithm 2 with
the Eq. (16) effective precisions, k_p = 0.05) against standard adaptive MLMC (the same algorithm with a
fixed MINRES tolerance of 1e-6), Eq. (20) field with s = 4, q = 2, sigma = 2, h0 = 1/8, for
TOL^2 = 8, 4, 2, 1 x 1e-6; R replicate runs per method and tolerance (the paper uses 1000).  The MSE is
taken against the paper's reference: standard MLMC at TOL^2 = 2e-8 with a direct double-precision
solver -- tests/golden/eq20_reference_tol2_2e-8.json, written by tools/oracle_reference.py from the oracle's
Algorithm 2 and binary64 banded Cholesky (a GPU standard-MLMC run with MINRES at 1e-12 is reported beside it).  Cost = the deterministic work model of the runs
(R5: MINRES iterations x unknowns, the analogue of the paper's PETSc FLOP count) and the measured GPU
time of the sampling calls.

  python tools/paper_experiment.py [R] [out.json]
  python tools/paper_experiment.py kp [R] [out.json]     # the k_p sensitivity study
"""
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


def run(R=100, tol2s=(8e-6, 4e-6, 2e-6, 1e-6), k_p=0.05, std_tol=1e-6, N_init=10, device=0, verbose=False):
    cfg = W.CONFIGS["EQ20"]
    ctx = Context(field="eq20", m=cfg["m"], sigma2=cfg["sigma2"], corr_len=0.0, q_decay=cfg["q_decay"],
                  h0_inv=cfg["h0_inv"], L_max=cfg["L_max"], device=device, workspace_bytes=2 << 30)
    ctx.adaptive_run(math.sqrt(8e-6), k_p=k_p, seed=10**7, N_init=N_init, on_fail=1)   # plan warm-up
    t0 = time.perf_counter()
    ref = ctx.adaptive_run(math.sqrt(2e-8), k_p=0.0, fixed_tol=1e-12, seed=10**8, N_init=N_init, on_fail=1)
    ref_s = time.perf_counter() - t0
    out = {"reference": {"estimate": ref["estimate"], "L": ref["L"], "N": ref["N"], "seconds": ref_s,
                         "n_fail": ref["n_fail"], "how": "standard MLMC, TOL^2 = 2e-8, MINRES tol 1e-12"},
           "R": R, "k_p": k_p, "standard_minres_tol": std_tol, "N_init": N_init, "tol2": {}}
    gold = json.load(open(os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests",
                                       "golden", "eq20_reference_tol2_2e-8.json")))
    out["reference"]["gpu_minres_1e-12"] = out["reference"].pop("estimate")
    out["reference"].update({"estimate": gold["estimate"], "L": gold["L"], "N": gold["N"], "how": gold["how"]})
    Q = gold["estimate"]
    for tol2 in tol2s:
        tol = math.sqrt(tol2)
        rows = {"mpml": [], "mlmc": []}
        for r in range(R):
            for name, kw in (("mpml", dict(k_p=k_p, seed=2 * r)),
                             ("mlmc", dict(k_p=0.0, fixed_tol=std_tol, seed=2 * r + 1))):
                torch.cuda.synchronize()
                t = time.perf_counter()
                res = ctx.adaptive_run(tol, N_init=N_init, on_fail=1, **kw)
                torch.cuda.synchronize()
                wall = time.perf_counter() - t
                cost = float(sum(n * c for n, c in zip(res["N"], res["cost"])))
                rows[name].append((res["estimate"], cost, res["solve_seconds"], wall, res["L"], res["N"], res["n_fail"]))
        entry = {}
        for name, rr in rows.items():
            est = np.array([x[0] for x in rr])
            se2 = (est - Q) ** 2
            Lmax = max(x[4] for x in rr)
            Nmean = [float(np.mean([x[5][l] if l < len(x[5]) else 0 for x in rr])) for l in range(Lmax + 1)]
            entry[name] = {"mse": float(se2.mean()), "mse_ci95": float(1.96 * se2.std(ddof=1) / math.sqrt(len(rr))),
                           "cost_model": float(np.mean([x[1] for x in rr])),
                           "gpu_solve_s": float(np.mean([x[2] for x in rr])),
                           "wall_s": float(np.mean([x[3] for x in rr])),
                           "L_hist": {str(L): int(sum(1 for x in rr if x[4] == L)) for L in range(Lmax + 1)},
                           "N_mean": Nmean, "failed_solves": int(sum(x[6] for x in rr))}
        entry["cost_ratio_mlmc_over_mpml"] = entry["mlmc"]["cost_model"] / entry["mpml"]["cost_model"]
        entry["gpu_time_ratio_mlmc_over_mpml"] = entry["mlmc"]["gpu_solve_s"] / entry["mpml"]["gpu_solve_s"]
        entry["tol2"] = tol2
        out["tol2"][f"{tol2:g}"] = entry
        if verbose:
            print(json.dumps({f"{tol2:g}": {k: entry[k] for k in ("cost_ratio_mlmc_over_mpml",
                                                                     "gpu_time_ratio_mlmc_over_mpml")} |
                              {m: {"mse": entry[m]["mse"], "ci": entry[m]["mse_ci95"]} for m in ("mpml", "mlmc")}}),
                  flush=True)
    ctx.close()
    return out


def kp_sweep(R=1000, kps=(0.05, 0.1, 0.2, 0.4), tol2=2e-6):
    """The k_p sensitivity study (the paper's MSE-vs-k_p figure): MPML at TOL^2 = 2e-6 for k_p = 0.05,
    0.1, 0.2, 0.4 against standard MLMC with the MINRES tolerance at 1e-10, R runs each."""
    out = {"tol2": tol2, "R": R, "mlmc_minres_tol": 1e-10, "k_p": {}}
    for kp in kps:
        r = run(R, tol2s=(tol2,), k_p=kp, std_tol=1e-10)
        e = r["tol2"][f"{tol2:g}"]
        out["k_p"][f"{kp:g}"] = {"mse_mpml": e["mpml"]["mse"], "mse_mpml_ci95": e["mpml"]["mse_ci95"],
                                 "mse_mlmc": e["mlmc"]["mse"], "mse_mlmc_ci95": e["mlmc"]["mse_ci95"],
                                 "N_mean_mpml": e["mpml"]["N_mean"], "N_mean_mlmc": e["mlmc"]["N_mean"],
                                 "cost_ratio": e["cost_ratio_mlmc_over_mpml"]}
        print(json.dumps({f"k_p={kp:g}": out["k_p"][f"{kp:g}"]}), flush=True)
    return out


if __name__ == "__main__":
    if len(sys.argv) > 1 and sys.argv[1] == "kp":
        R = int(sys.argv[2]) if len(sys.argv) > 2 else 1000
        res = kp_sweep(R)
        path = sys.argv[3] if len(sys.argv) > 3 else "gpurun_out/paper_kp_sweep.json"
        os.makedirs(os.path.dirname(path) or ".", exist_ok=True)
        json.dump(res, open(path, "w"), indent=1)
        sys.exit(0)
    R = int(sys.argv[1]) if len(sys.argv) > 1 else 100
    res = run(R, N_init=int(os.environ.get("N_INIT", "10")), verbose=True)
    path = sys.argv[2] if len(sys.argv) > 2 else "gpurun_out/paper_experiment.json"
    os.makedirs(os.path.dirname(path) or ".", exist_ok=True)
    json.dump(res, open(path, "w"), indent=1)
    print("reference", res["reference"])
