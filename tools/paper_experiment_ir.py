"""The paper's direct-solver experiments (Section 5.2) on the GPU: MPML with low-precision
banded Cholesky + iterative refinement (Algorithm 1, K4) against standard MLMC with a binary64
Cholesky solve, with the SAME numbers of samples and the SAME random inputs, so that the MSE
difference is the computational error alone.

  E3: Eq. (20) field s = 4, q = 2, sigma = 2, h0 = 1/8, k_p = 0.05; Table 1 right quads
       -- level 0 hhss, level 1 ssss, levels 2+ ssdd -- exactly (u_s = u_f selectable).
  E4: s = 1, sigma = 1, h0 = 1/4, k_p = 0.4; level 0 qhhh, levels 1-3 hhss, exactly.

The sample counts of run r come from a standard adaptive MLMC run (fixed MINRES tolerance 1e-10, as
in P:700 "determined by 1000 runs of the standard adaptive MLMC algorithm"); both estimators then use
those N_l with the same per-level seeds.  Cost: the bytes the solves move, counted two ways --
(a) the paper's simulated memory model, "the number of entries in all vectors and the number of
non-zeros in all sparse factorisations ... computed and stored in the process of solving", in bits
(factor n(bw+1) b_f once, and per IR step the three vectors x, r, d at their precisions); (b) K4's
algorithmic HBM bytes (the factor read by both substitutions of every solve) and
the measured GPU time of the sampling calls.

  python tools/paper_experiment_ir.py [E3|E4] [R] [out.json]
"""
import json
import math
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2503_05533_b200 import Context, precision  # noqa: E402
from paper_2503_05533_b200.api import mlmc_eps_schedule  # noqa: E402

BITS = {"q": 8, "h": 16, "s": 32, "d": 64}
SETUPS = {
    # field (Eq. (20)), h0, k_p, L_max for K4 (h >= 1/32), quads per level (paper -> implemented)
    "E3": dict(m=4, sigma2=4.0, h0_inv=8, k_p=0.05, L_cap=2,
               paper=["hhss", "ssss", "ssdd"], quads=["hhss", "ssss", "ssdd"], tol2=(8e-6, 4e-6, 2e-6, 1e-6)),
    "E4": dict(m=1, sigma2=1.0, h0_inv=4, k_p=0.4, L_cap=3,
               paper=["qhhh", "hhss", "hhss", "hhss"], quads=["qhhh", "hhss", "hhss", "hhss"], tol2=(2e-6,)),
}


def solve_bits(N, quad, steps_mean):
    """The paper's simulated memory model for one solve of the N-mesh system."""
    n, bw = (N - 1) ** 2, N - 1
    bf, bs, bu, br = (BITS[c] for c in quad)
    return n * (bw + 1) * bf + n * (bu + br + bs) * (1.0 + steps_mean)


def k4_bytes(N, quad, steps_mean):
    """K4 algorithmic HBM bytes of one solve."""
    fac = (N - 1) ** 2 * N * BITS[quad[0]] / 8
    return fac * (1 + 2 * (1 + steps_mean)) + 16 * N * N


def run(name="E3", R=200, device=0, verbose=False):
    cfg = SETUPS[name]
    L_cap = cfg["L_cap"]
    ctx = Context(field="eq20", m=cfg["m"], sigma2=cfg["sigma2"], corr_len=0.0, q_decay=2.0, h0_inv=cfg["h0_inv"],
                  L_max=L_cap, device=device, workspace_bytes=2 << 30)
    h0 = 1.0 / cfg["h0_inv"]
    std = precision("chol_ir", "d", "d")                  # binary64 Cholesky (the direct solve)
    ref = ctx.adaptive_run(math.sqrt(2e-8), k_p=0.0, fixed_tol=1e-12, seed=10**8, N_init=10, on_fail=1)
    Q = ref["estimate"]
    out = {"setup": name, "R": R, "reference": {"estimate": Q, "N": ref["N"], "L": ref["L"]},
           "quads_paper": cfg["paper"], "quads_impl": cfg["quads"], "tol2": {}}
    for tol2 in cfg["tol2"]:
        tol = math.sqrt(tol2)
        est = {"mpml": [], "mlmc": []}
        cost = {"mpml": np.zeros(L_cap + 1), "mlmc": np.zeros(L_cap + 1)}
        hbm = {"mpml": np.zeros(L_cap + 1), "mlmc": np.zeros(L_cap + 1)}
        gpu = {"mpml": 0.0, "mlmc": 0.0}
        used = 0
        for r in range(R):
            a = ctx.adaptive_run(tol, k_p=0.0, fixed_tol=1e-10, seed=7 * r + 3, N_init=10, on_fail=1)
            if a["L"] > L_cap:                        # K4 covers h >= 1/32 only
                continue
            used += 1
            L = a["L"]
            Nl = a["N"]
            eps = mlmc_eps_schedule(L, h0, cfg["k_p"])
            for meth in ("mpml", "mlmc"):
                s_total = 0.0
                for l in range(L + 1):
                    Nf = cfg["h0_inv"] << l
                    if meth == "mpml":
                        pf = precision("chol_ir", *cfg["quads"][l])
                        pc = precision("chol_ir", *cfg["quads"][l - 1]) if l else pf
                        tf, tc = eps[l], eps[l - 1] if l else eps[0]
                    else:
                        pf = pc = std
                        tf = tc = 1e-13
                    torch.cuda.synchronize()
                    t = time.perf_counter()
                    res = ctx.sample_level(l, Nl[l], seed=1000 + r, first_index=0, prec_fine=pf, prec_coarse=pc,
                                           tol_fine=tf, tol_coarse=tc)
                    gpu[meth] += time.perf_counter() - t
                    sm = res.sums
                    s_total += sm["sum_y"] / Nl[l]
                    qf = cfg["quads"][l] if meth == "mpml" else "dddd"
                    qc = (cfg["quads"][l - 1] if l else None) if meth == "mpml" else ("dddd" if l else None)
                    sf = sm["iters_f"] / Nl[l]
                    cost[meth][l] += Nl[l] * solve_bits(Nf, qf, sf)
                    hbm[meth][l] += Nl[l] * k4_bytes(Nf, qf, sf)
                    if l:
                        sc = sm["iters_c"] / Nl[l]
                        cost[meth][l] += Nl[l] * solve_bits(Nf // 2, qc, sc)
                        hbm[meth][l] += Nl[l] * k4_bytes(Nf // 2, qc, sc)
                est[meth].append(s_total)
        e = {}
        for meth in ("mpml", "mlmc"):
            se = (np.array(est[meth]) - Q) ** 2
            e[meth] = {"mse": float(se.mean()), "mse_ci95": float(1.96 * se.std(ddof=1) / math.sqrt(len(se))),
                       "memory_bits_per_level": (cost[meth] / max(used, 1)).tolist(),
                       "k4_hbm_bytes_per_level": (hbm[meth] / max(used, 1)).tolist(),
                       "gpu_seconds": gpu[meth] / max(used, 1)}
        e["runs_used"] = used
        e["mse_rel_diff"] = abs(e["mpml"]["mse"] - e["mlmc"]["mse"]) / e["mlmc"]["mse"]
        e["memory_gain_total"] = sum(e["mlmc"]["memory_bits_per_level"]) / sum(e["mpml"]["memory_bits_per_level"])
        e["memory_gain_per_level"] = [m / p if p else None for m, p in zip(e["mlmc"]["memory_bits_per_level"],
                                                                          e["mpml"]["memory_bits_per_level"])]
        e["k4_hbm_gain_total"] = sum(e["mlmc"]["k4_hbm_bytes_per_level"]) / sum(e["mpml"]["k4_hbm_bytes_per_level"])
        e["gpu_time_ratio"] = e["mlmc"]["gpu_seconds"] / e["mpml"]["gpu_seconds"]
        out["tol2"][f"{tol2:g}"] = e
        if verbose:
            print(json.dumps({f"{tol2:g}": {k: e[k] for k in ("runs_used", "mse_rel_diff", "memory_gain_total",
                                                                  "memory_gain_per_level", "k4_hbm_gain_total",
                                                                  "gpu_time_ratio")}}), flush=True)
    ctx.close()
    return out


if __name__ == "__main__":
    name = sys.argv[1] if len(sys.argv) > 1 else "E3"
    R = int(sys.argv[2]) if len(sys.argv) > 2 else 200
    res = run(name, R, verbose=True)
    path = sys.argv[3] if len(sys.argv) > 3 else f"gpurun_out/paper_experiment_{name}.json"
    os.makedirs(os.path.dirname(path) or ".", exist_ok=True)
    json.dump(res, open(path, "w"), indent=1)
