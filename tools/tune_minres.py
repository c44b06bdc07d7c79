"""Time the MINRES kernel variants (MLMC_MINRES_TILE_N<N>) on the configs[1] workload.

Usage: python tools/tune_minres.py            (spawns one process per variant)
       python tools/tune_minres.py --one N L n (internal: time one level's solves)
Prints one JSON line per variant: mesh N, variant, ms per solve batch, node-iterations/s.
"""
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

# (mesh N, level whose FINE mesh is N, samples, tolerance) from configs[1]
CASES = {8: (0, 20000, 1e-4), 16: (1, 5000, 1e-5), 32: (2, 1200, 1e-6), 64: (3, 300, 1e-8)}
VARIANTS = {8: [0], 16: [0, 4], 32: [0, 7], 64: [0]}


def one(N):
    import torch
    import workloads as W
    from paper_2503_05533_b200 import Context, precision
    cfg = W.CONFIGS["C2"]
    level, n, tol = CASES[N]
    ctx = Context(field="expcov", m=cfg["m"], sigma2=cfg["sigma2"], corr_len=cfg["corr_len"], h0_inv=8,
                  L_max=3, device=0, workspace_bytes=2 << 30)
    mr = precision("minres")
    for _ in range(2):
        ctx.sample_level(level, n, seed=1, prec_fine=mr, prec_coarse=mr, tol_fine=tol, tol_coarse=tol * 10)
    ctx.profile_enable(True)
    reps = 5
    its = 0.0
    for r in range(reps):
        s = ctx.sample_level(level, n, seed=1, first_index=r * n, prec_fine=mr, prec_coarse=mr, tol_fine=tol,
                             tol_coarse=tol * 10).sums
        its += s["iters_f"]
    prof = ctx.profile_read()
    ms = [p for p in prof if p[0] == "minres" and p[1] == N][0]
    per = ms[3] / ms[2]
    nodes = (N - 1) ** 2
    print(json.dumps({"N": N, "variant": int(os.environ.get(f"MLMC_MINRES_TILE_N{N}", "0")),
                      "ms_per_launch": per, "node_iters_per_s": its / reps * nodes / (per / 1e3),
                      "fp64_tflops_alg": 25 * its / reps * nodes / (per / 1e3) / 1e12}), flush=True)


def main():
    if len(sys.argv) > 1 and sys.argv[1] == "--one":
        one(int(sys.argv[2]))
        return
    for N, vs in VARIANTS.items():
        for v in vs:
            env = dict(os.environ, **{f"MLMC_MINRES_TILE_N{N}": str(v)})
            r = subprocess.run([sys.executable, __file__, "--one", str(N)], env=env, capture_output=True, text=True)
            out = [l for l in r.stdout.splitlines() if l.startswith("{")]
            print(out[-1] if out else json.dumps({"N": N, "variant": v, "error": r.stderr[-400:]}), flush=True)


if __name__ == "__main__":
    main()
