"""Small cases of every kernel family for compute-sanitizer (one tool per gpurun call, B200_PROFILING.md):
K0/K1 (rng, field), K3 tile MINRES (h = 1/8 .. 1/64), K3c streamed MINRES with 2-CTA clusters + TMA/mbarrier
(h = 1/128), K3m on-chip MG-PCG and K3m-t tiled MG-PCG with TMA (h = 1/128), K4a/K4b Cholesky + IR with the
cp.async.bulk ring (h = 1/32, fp16 and fp32 factors), K5 sums (incl. the exact fixed-point sums of an adaptive
run), K3d slab MINRES (G = 1 fused and G = 2 emulated).
    compute-sanitizer --tool racecheck python tools/sanitize_cases.py"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import workloads as W  # noqa: E402
from paper_2503_05533_b200 import Context, precision  # noqa: E402
from paper_2503_05533_b200.dd import SlabSolver, dd_solve_emulated  # noqa: E402

cfg = W.CONFIGS["C5"]
ctx = Context(field=cfg["field"], m=cfg["m"], sigma2=cfg["sigma2"], corr_len=cfg["corr_len"], h0_inv=cfg["h0_inv"],
              L_max=4, device=0, workspace_bytes=1 << 30)
mr, mg = precision("minres"), precision("mgcg")
for level, n in ((0, 40), (1, 20), (2, 6), (3, 3)):
    r = ctx.sample_level(level, n, seed=1, prec_fine=mr, tol_fine=1e-6, tol_coarse=1e-6)
    assert r.sums["n_fail"] == 0
    r = ctx.sample_level(level, n, seed=1, prec_fine=mg, prec_coarse=mg, tol_fine=1e-6, tol_coarse=1e-6)
    assert r.sums["n_fail"] == 0
print("K3 / K3m ok", flush=True)
r = ctx.sample_level(4, 2, seed=1, prec_fine=precision("minres", max_iter=60), tol_fine=1e-12, tol_coarse=1e-12)
r = ctx.sample_level(4, 2, seed=1, prec_fine=mg, prec_coarse=mg, tol_fine=1e-6, tol_coarse=1e-6)
assert r.sums["n_fail"] == 0
print("K3c / K3m-t ok", flush=True)
c3 = W.CONFIGS["C3"]
ctx3 = Context(field="expcov", m=c3["m"], sigma2=c3["sigma2"], corr_len=c3["corr_len"], h0_inv=8, L_max=2, device=0,
               workspace_bytes=1 << 30)
for uf in ("h", "s"):
    p = precision("chol_ir", uf, "s")
    for level in (0, 1, 2):
        r = ctx3.sample_level(level, 64 if level < 2 else 16, seed=2, prec_fine=p, prec_coarse=p, tol_fine=1e-10,
                              tol_coarse=1e-10)
        assert r.sums["n_fail"] == 0
print("K4 ok", flush=True)
a = ctx3.adaptive_run(3e-3, k_p=0.05, N_init=20, seed=3)
print("K5 / adaptive ok", a["L"], flush=True)
ctx3.close()
for G in (1, 2):
    eng = [SlabSolver(ctx, 4, g, G) for g in range(G)]
    for e in eng:
        e.begin(1, 4, 0, 1e-4, 40)
    res = [eng[0].run_local()] if G == 1 else dd_solve_emulated(eng, check_every=8)
    for e in eng:
        e.close()
print("K3d ok", flush=True)
ctx.close()
print("sanitize cases done")
