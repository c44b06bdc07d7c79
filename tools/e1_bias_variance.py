"""NEXT-1 E1 (Figure "bias/variance decay"): computational error in the variance of the
difference estimators Var[Y~_l] and in the bias |E[Q~_l - Q]| against the effective precision eps_l, on the
paper's Eq. (20) field (s = 4, q = 2, sigma = 2, h_l = 1/8 * 2^-l), MINRES stopped on the relative
residual ("relative residuals produced by MINRES are monitored").  Lemma 4.? predicts an
initial decay of at least O(eps^2) for the variance and O(eps) for the bias, until the discretisation error
dominates.

Per level l = 0..4 and eps on a half-decade grid:
  var_Y       sample variance of Y~_l = Q~_l - Q~_{l-1} (both halves to eps, R31), 10^2 samples (as the paper);
  var_err     variance of the computational error Y~_l(eps) - Y_l over the same samples (Y_l: both halves to
              1e-12 -- MINRES on chip for h >= 1/64, MG-PCG for h = 1/128, same relative-residual contract);
  bias_total  |mean Q~_l(eps) - Q_ref| with Q_ref the oracle reference (tests/golden), 10^4 samples
              (10^3 at h = 1/128);
  bias_comp   |mean(Q~_l(eps) - Q_l)| over the same samples (the computational part alone).
Fitted log-log slopes of var_err and bias_comp over the eps range where they exceed the 1e-12 solve error.
    python tools/e1_bias_variance.py [out.json]"""
import json
import math
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import workloads as W  # noqa: E402
from paper_2503_05533_b200 import Context, precision  # noqa: E402

EPS = [1e-1, 3e-2, 1e-2, 3e-3, 1e-3, 3e-4, 1e-4, 3e-5, 1e-5, 3e-6, 1e-6, 1e-7, 1e-8]


def slope(x, y, floor):
    x, y = np.asarray(x), np.asarray(y)
    m = y > floor
    if m.sum() < 3:
        return None
    return float(np.polyfit(np.log(x[m]), np.log(y[m]), 1)[0])


def main(path):
    cfg = W.CONFIGS["EQ20"]
    ctx = Context(field="eq20", m=cfg["m"], sigma2=cfg["sigma2"], corr_len=0.0, q_decay=cfg["q_decay"],
                  h0_inv=cfg["h0_inv"], L_max=4, device=0, workspace_bytes=4 << 30)
    q_ref = json.load(open(os.path.join(ROOT, "tests", "golden", "eq20_reference_tol2_2e-8.json")))["estimate"]
    mr = precision("minres")
    out = {"field": "Eq. (20), s=4, q=2, sigma=2", "Q_ref": q_ref, "eps": EPS, "levels": {}}
    for l in range(5):
        N = 8 << l
        ex = precision("mgcg") if N >= 128 else mr
        exc = precision("mgcg") if (N // 2) >= 128 else mr
        nv, nb = 100, (10000 if l <= 3 else 1000)
        # exact halves (1e-12) of the variance and bias samples
        yv = ctx.sample_level(l, nv, seed=11, prec_fine=ex, prec_coarse=exc, tol_fine=1e-12, tol_coarse=1e-12,
                              per_sample=True).per_sample
        qb = ctx.sample_level(l, nb, seed=12, prec_fine=ex, prec_coarse=exc, tol_fine=1e-12, tol_coarse=1e-12,
                              per_sample=True).per_sample[:, 0]
        Y = yv[:, 0] - yv[:, 1]
        rows = []
        for eps in EPS:
            pv = ctx.sample_level(l, nv, seed=11, prec_fine=mr, prec_coarse=mr, tol_fine=eps, tol_coarse=eps,
                                  per_sample=True).per_sample
            pb = ctx.sample_level(l, nb, seed=12, prec_fine=mr, prec_coarse=mr, tol_fine=eps, tol_coarse=eps,
                                  per_sample=True).per_sample
            Yt = pv[:, 0] - pv[:, 1]
            rows.append({"eps": eps, "var_Y": float(Yt.var()), "var_err": float((Yt - Y).var()),
                         "bias_total": float(abs(pb[:, 0].mean() - q_ref)),
                         "bias_comp": float(abs((pb[:, 0] - qb).mean())),
                         "mean_iters_fine": float(pb[:, 2].mean()), "fails": int((pb[:, 6] != 0).sum())})
        out["levels"][str(l)] = {
            "h": f"1/{N}", "samples_var": nv, "samples_bias": nb, "var_Y_exact": float(Y.var()),
            "bias_exact": float(abs(qb.mean() - q_ref)), "rows": rows,
            "slope_var_err": slope(EPS, [r["var_err"] for r in rows], 1e-24),
            "slope_bias_comp": slope(EPS, [r["bias_comp"] for r in rows], 1e-13)}
        print(json.dumps({f"l{l}": {k: out["levels"][str(l)][k] for k in ("slope_var_err", "slope_bias_comp",
                                                                             "var_Y_exact", "bias_exact")}}),
              flush=True)
    ctx.close()
    json.dump(out, open(path, "w"), indent=1)


if __name__ == "__main__":
    main(sys.argv[1] if len(sys.argv) > 1 else "gpurun_out/e1.json")
