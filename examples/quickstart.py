"""Python quickstart (the same steps as examples/quickstart.c, through the thin ctypes binding).

    python examples/quickstart.py

1. plan a 4-level hierarchy of the BASELINE field (exponential covariance, 64 KL modes, h = 1/8 .. 1/64);
2. one coupled-sample batch per level at the paper's MINRES tolerances (Eq. (16) schedule), host sums;
3. all four levels concurrently into a device tensor (the bench step, no host synchronisation);
4. the adaptive algorithm (Algorithm 2, policy 0 = MINRES everywhere) to an RMSE target;
5. the same with policy 3 (per mesh, the fastest admissible solver from pilot timings).
Needs a B200 and the built libmlmc.so (python __graft_entry__.py).
"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2503_05533_b200 import Context, precision  # noqa: E402


def main():
    ctx = Context(field="expcov", m=64, sigma2=1.0, corr_len=0.3, h0_inv=8, L_max=3, device=0,
                  workspace_bytes=1 << 30)
    for l in range(4):
        print("level", l, ctx.level_info(l))

    # 2. one batch per level: Y_l = Q_l - Q_{l-1} from the same xi, fine half at eps_l, coarse half at eps_{l-1}
    tols = [1e-4, 1e-5, 1e-6, 1e-8]
    mr = precision("minres")
    for l, n in enumerate([2000, 500, 120, 30]):
        r = ctx.sample_level(l, n, seed=1, prec_fine=mr, prec_coarse=mr, tol_fine=tols[l],
                             tol_coarse=tols[l - 1] if l else tols[0])
        s = r.sums
        mean = s["sum_y"] / s["n"]
        var = s["sum_y2"] / s["n"] - mean ** 2
        print(f"level {l}: n {int(s['n'])}  mean Y {mean:.6e}  var Y {var:.3e}  mean MINRES steps "
              f"{s['iters_f'] / s['n']:.1f}  failures {int(s['n_fail'])}")

    # 3. all levels concurrently on the device (what bench.py times); sums land in a [4, 12] float64 tensor
    sums = torch.zeros((4, 12), dtype=torch.float64, device="cuda")
    ctx.sample_levels_async([0, 1, 2, 3], [2000, 500, 120, 30], 2, [0, 0, 0, 0], [mr] * 4, [mr] * 4, tols,
                            [tols[0], tols[0], tols[1], tols[2]], sums)
    torch.cuda.synchronize()
    est = float((sums[:, 0] / sums[:, 5]).sum())
    print(f"telescoping estimate from one concurrent step: {est:.6f}")

    # 4./5. Algorithm 2 to RMSE eps
    for policy in (0, 3):
        res = ctx.adaptive_run(1e-3, k_p=0.05, seed=3, policy=policy)
        print(f"adaptive (policy {policy}): estimate {res['estimate']:.6f}, L = {res['L']}, N_l = {res['N']}, "
              f"rounds {res['rounds']}")
    ctx.close()


if __name__ == "__main__":
    main()
