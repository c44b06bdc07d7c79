"""K3b (cluster-resident MINRES) vs K3c (streamed) on the fine meshes of configs[4]: device ms of the fine-mesh
MINRES launch for a batch of equal-tolerance systems.  python tools/k3b_time.py   (spawns one process per path)
Prints JSON lines: mesh, systems, path, ms, mean steps, unknown-steps per second."""
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
CASES = [(4, 148, 1e-8), (4, 441, 1e-8), (5, 148, 1e-8), (5, 37, 1e-8)]


def one():
    import workloads as W
    from paper_2503_05533_b200 import Context, precision
    cfg = W.CONFIGS["C5"]
    ctx = Context(field=cfg["field"], m=cfg["m"], sigma2=cfg["sigma2"], corr_len=cfg["corr_len"], h0_inv=8,
                  L_max=6, device=0, workspace_bytes=16 << 30)
    mr = precision("minres")
    for level, n, tol in CASES:
        N = 8 << level
        ctx.sample_level(level, 4, seed=1, prec_fine=mr, prec_coarse=mr, tol_fine=tol, tol_coarse=tol)   # warm-up
        ctx.profile_enable(True)
        r = ctx.sample_level(level, n, seed=2, prec_fine=mr, prec_coarse=mr, tol_fine=tol, tol_coarse=tol)
        prof = ctx.profile_read()
        ctx.profile_enable(False)
        ms = sum(p[3] for p in prof if p[0] == "minres" and p[1] == N)
        steps = r.sums["iters_f"] / n
        print(json.dumps({"h": f"1/{N}", "systems": n, "path": os.environ.get("MLMC_MINRES_K3B", "1") == "0" and "K3c"
                          or "K3b", "fine_minres_ms": ms, "mean_steps": steps,
                          "unknown_steps_per_s": n * steps * (N - 1) ** 2 / (ms / 1e3)}), flush=True)
    ctx.close()


if __name__ == "__main__":
    if len(sys.argv) > 1 and sys.argv[1] == "--one":
        one()
    else:
        for v in ("1", "0"):
            env = dict(os.environ, MLMC_MINRES_K3B=v)
            r = subprocess.run([sys.executable, __file__, "--one"], env=env, capture_output=True, text=True)
            for l in r.stdout.splitlines():
                if l.startswith("{"):
                    print(l, flush=True)
            if r.returncode:
                print(json.dumps({"path": v, "error": r.stderr[-600:]}), flush=True)
