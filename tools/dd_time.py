"""K3d timing on one B200: ONE configs[4] system at h = 1/256 and 1/512, to the finest-level tolerance of
an L = 6 run (eps_6 = k_p h^2), solved (a) by K3c inside mlmc_sample_level (a 2-CTA cluster per system),
(b) by K3d on the whole GPU (G = 1, mlmc_dd_run_local: 32-step CUDA graphs), (c) by K3d as G = 2 / 4 slabs
emulated in one process (host-driven steps; per-step cost of the multi-rank schedule minus NVLink).
Device time with CUDA events.   python tools/dd_time.py"""
import json
import os
import sys
import time

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import workloads as W  # noqa: E402
from paper_2503_05533_b200 import Context, precision  # noqa: E402
from paper_2503_05533_b200.dd import SlabSolver, dd_run_fused_emulated, dd_solve_emulated  # noqa: E402


def ev_time(fn):
    s = torch.cuda.current_stream()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    a.record(s)
    r = fn()
    b.record(s)
    torch.cuda.synchronize()
    return r, a.elapsed_time(b), 1e3 * (time.perf_counter() - t0)


def main():
    cfg = W.CONFIGS["C5"]
    ctx = Context(field=cfg["field"], m=cfg["m"], sigma2=cfg["sigma2"], corr_len=cfg["corr_len"],
                  h0_inv=cfg["h0_inv"], L_max=cfg["L_max"], device=0, workspace_bytes=4 << 30)
    out = {}
    for level in (5, 6):
        N = cfg["h0_inv"] << level
        tol = cfg["k_p"] / N ** 2
        seed, k = 7, 0
        mr = precision("minres")
        ctx.sample_level(level, 1, seed=seed, first_index=99, prec_fine=mr, tol_fine=1e-3, tol_coarse=1e-3)
        r, ms, wall = ev_time(lambda: ctx.sample_level(level, 1, seed=seed, first_index=k, prec_fine=mr, tol_fine=tol,
                                                      tol_coarse=tol, per_sample=True).per_sample[0])
        row = {"tol": tol, "k3c_cluster2": {"ms_coupled_sample": ms, "iters_fine": r[2], "iters_coarse": r[3],
                                             "Q": r[0]}}
        for G in (1, 2, 4):
            eng = [SlabSolver(ctx, level, g, G) for g in range(G)]
            for e in eng:
                e.begin(seed, level, k, tol)
            if G == 1:
                res, ms, wall = ev_time(lambda: [eng[0].run_local()])
            else:
                res, ms, wall = ev_time(lambda: dd_solve_emulated(eng))
            it = res[0]["iters"]
            row[f"k3d_G{G}"] = {"ms_fine_solve": ms, "wall_ms": wall, "iters": it, "us_per_step": 1e3 * ms / max(it, 1),
                                "Q": res[0]["Q"], "status": res[0]["status"],
                                "note": "whole GPU, CUDA graphs" if G == 1 else "G slabs emulated on one GPU, host-driven"}
            for e in eng:
                e.close()
        for G in (2, 4, 8):        # the fused peer-memory exchange, all ranks in one cooperative launch
            eng = [SlabSolver(ctx, level, g, G) for g in range(G)]
            for e in eng:
                e.begin(seed, level, k, tol)
            res, ms, wall = ev_time(lambda: dd_run_fused_emulated(eng))
            row[f"k3d_fused_G{G}"] = {"ms_fine_solve": ms, "iters": res["iters"], "Q": res["Q"],
                                      "us_per_step": 1e3 * ms / max(res["iters"], 1), "status": res["status"],
                                      "note": "G slabs, exchange fused into the kernel, one cooperative launch"}
            for e in eng:
                e.close()
        out[f"h=1/{N}"] = row
    ctx.close()
    print(json.dumps(out))


if __name__ == "__main__":
    main()
