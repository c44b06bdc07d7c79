"""Check every MINRES kernel variant against the oracle (iterations and QoI bound) on a few samples.

Usage: python tools/check_variants.py            (spawns one process per variant)
"""
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

CASES = {8: (0, 1e-4), 16: (1, 1e-5), 32: (2, 1e-6), 64: (3, 1e-8), 128: (4, 1e-8)}
VARIANTS = {8: [0], 16: [0], 32: [0], 64: [0, 1]}


def one(N):
    import numpy as np
    from concurrent.futures import ThreadPoolExecutor
    from oracle import core as oc
    from paper_2503_05533_b200 import Context, precision
    level, tol = CASES[N]
    ctx = Context(field="expcov", m=64, sigma2=1.0, corr_len=0.3, h0_inv=8, L_max=4, device=0,
                  workspace_bytes=1 << 30)
    mr = precision("minres", verify=True)
    n = 8 if N < 128 else 3
    ps = ctx.sample_level(level, n, seed=1, prec_fine=mr, prec_coarse=mr, tol_fine=tol, tol_coarse=tol,
                          per_sample=True).per_sample
    P = oc.OracleProblem(0, 64, 1.0, 0.3, 2.0, 8)

    def ref(k):
        xi = oc.normals(1, level, k, 64)
        o = P.solve_mesh(N, xi, oc.SOLVER_MINRES, tol=tol)
        a = P.field_triangles(N, xi)
        AB, _, b = oc.assemble(N, a)
        x, _ = oc.chol_band_solve(AB, b)
        return o["iters"], (1.0 / N) ** 2 * x.sum(), np.linalg.norm(b) * np.linalg.norm(x)

    with ThreadPoolExecutor(8) as ex:
        refs = list(ex.map(ref, range(n)))
    worst_it = max(abs(ps[k, 2] - refs[k][0]) / refs[k][0] for k in range(n))
    worst_q = max(abs(ps[k, 0] - refs[k][1]) / (tol * refs[k][2]) for k in range(n))
    print(json.dumps({"N": N, "variant": int(os.environ.get(f"MLMC_MINRES_TILE_N{N}", "0")),
                      "iters_gpu": ps[:, 2].tolist(), "iters_oracle": [r[0] for r in refs],
                      "worst_rel_iter_diff": worst_it, "worst_q_err_over_bound": worst_q,
                      "max_true_relres_over_tol": float(ps[:, 4].max() / tol)}), flush=True)


def main():
    if len(sys.argv) > 1 and sys.argv[1] == "--one":
        one(int(sys.argv[2]))
        return
    for N, vs in VARIANTS.items():
        for v in vs:
            env = dict(os.environ, **{f"MLMC_MINRES_TILE_N{N}": str(v)})
            r = subprocess.run([sys.executable, __file__, "--one", str(N)], env=env, capture_output=True, text=True)
            out = [l for l in r.stdout.splitlines() if l.startswith("{")]
            print(out[-1] if out else json.dumps({"N": N, "variant": v, "error": r.stderr[-600:]}), flush=True)


if __name__ == "__main__":
    main()
