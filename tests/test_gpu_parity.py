"""GPU parity of the C-ABI hot path against the CPU oracle (-m gpu).

Inputs are the seeded synthetic workloads of BASELINE.json (see DESIGN.md
section 5); every expected value comes from oracle/ (never from the CUDA path).
Tolerances:
  * RNG normals / field coefficients: binary64 rounding of different libm
    implementations (1e-13 relative);
  * fp64 mode (tol 1e-12): per-sample QoI to 1e-10 relative (north star);
  * reduced-accuracy modes: |Q_gpu - Q_exact| <= tol ||b|| ||x_exact|| (1 + 1e-6)
    + 1e-14 Q, the rigorous per-sample bound of DESIGN.md section 4 (w = b, A SPD).
"""
import math
import os
import sys
from concurrent.futures import ThreadPoolExecutor

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

from oracle import core as oc  # noqa: E402
from paper_2503_05533_b200 import Context, precision  # noqa: E402
import workloads as W  # noqa: E402


@pytest.fixture(scope="module", autouse=True)
def built():
    import __graft_entry__
    __graft_entry__.build()


def _ctx(cfg, L_max=None, ws=256 << 20):
    return Context(field=cfg["field"], m=cfg["m"], sigma2=cfg["sigma2"], corr_len=cfg["corr_len"],
                   q_decay=cfg.get("q_decay", 2.0), h0_inv=cfg["h0_inv"],
                   L_max=cfg["L_max"] if L_max is None else L_max, device=0, workspace_bytes=ws)


def _oracle(cfg):
    return oc.OracleProblem(cfg["field_code"], cfg["m"], cfg["sigma2"], cfg["corr_len"], cfg.get("q_decay", 2.0),
                            cfg["h0_inv"])


def _exact(P, N, xi):
    """Direct fp64 solve (O-exact): Q, ||b||, ||x||."""
    a = P.field_triangles(N, xi)
    AB, _, b = oc.assemble(N, a)
    x, _ = oc.chol_band_solve(AB, b)
    return (1.0 / N) ** 2 * x.sum(), np.linalg.norm(b), np.linalg.norm(x)


def _pmap(f, xs):
    with ThreadPoolExecutor(8) as ex:
        return list(ex.map(f, xs))


# ============================================================================ K0 / K1+K2
@pytest.mark.parametrize("cfg_name", ["C1", "C2", "C4", "EQ20"])
def test_rng_and_field_match_oracle(cfg_name):
    cfg = W.CONFIGS[cfg_name]
    ctx = _ctx(cfg, L_max=2)
    P = _oracle(cfg)
    for level, mesh in ((0, 0), (2, 2), (2, 1)):
        n = 37
        xi, a = ctx.debug_field(level, mesh, n, seed=11, first_index=1000)
        xi, a = xi.cpu().numpy(), a.cpu().numpy()
        N = cfg["h0_inv"] << mesh
        for k in (0, 5, 36):
            ref_xi = oc.normals(11, level, 1000 + k, cfg["m"])
            assert np.allclose(xi[k], ref_xi, rtol=1e-13, atol=1e-14)
            ref_a = P.field_triangles(N, ref_xi)
            assert np.max(np.abs(a[k] / ref_a - 1)) < 1e-12
    ctx.close()


def test_field_synthesis_paths_match_oracle():
    """configs[4] (m = 256, K = 30 one-dimensional functions): h = 1/8 takes the P x m synthesis on the FP64
    tensor cores (N = 8 with K > 16), h = 1/16 .. 1/512 the separable one (K1s: 8 samples x 8 x 8, 4 x 16 x 16
    and 32 x 32 tiles, up to 256 tiles per sample at h = 1/512; ragged sample groups); both reproduce the
    oracle's centroid-by-centroid KL sum to 1e-12."""
    cfg = W.CONFIGS["C5"]
    ctx = _ctx(cfg, L_max=6)
    P = _oracle(cfg)
    for level, mesh, n, ks in ((0, 0, 37, (0, 17, 36)), (1, 1, 37, (0, 17, 36)), (3, 3, 37, (0, 17, 36)),
                               (3, 2, 37, (0, 17, 36)), (4, 4, 5, (0, 4)), (6, 6, 3, (2,)), (1, 1, 1, (0,)),
                               (2, 2, 1, (0,))):
        xi, a = ctx.debug_field(level, mesh, n, seed=12, first_index=77)
        xi, a = xi.cpu().numpy(), a.cpu().numpy()
        N = cfg["h0_inv"] << mesh
        for k in ks:
            ref_a = P.field_triangles(N, oc.normals(12, level, 77 + k, cfg["m"]))
            assert np.max(np.abs(a[k] / ref_a - 1)) < 1e-12, (level, mesh, k)
    ctx.close()


# ============================================================================ C1: fp64 parity 1e-10
def test_C1_fp64_per_sample_parity_and_sums():
    cfg = W.CONFIGS["C1"]
    ctx = _ctx(cfg)
    P = _oracle(cfg)
    vprec = precision("minres", verify=True)
    for level, n in ((0, cfg["N"][0]), (1, cfg["N"][1])):
        r = ctx.sample_level(level, n, seed=cfg["seed"], prec_fine="minres", tol_fine=1e-12, tol_coarse=1e-12,
                             per_sample=True)
        ps = r.per_sample
        assert np.all(ps[:, 6:8] == 0)
        assert np.all(ps[:, 4] <= 1e-12)                     # phibar / ||b||, the stopping quantity
        # VERIFY instantiation: same Q bits, plus the true residual ||b - A x|| / ||b||
        rv = ctx.sample_level(level, n, seed=cfg["seed"], prec_fine=vprec, prec_coarse=vprec, tol_fine=1e-12,
                              tol_coarse=1e-12, per_sample=True).per_sample
        assert np.array_equal(rv[:, [0, 1, 2, 3, 6, 7]], ps[:, [0, 1, 2, 3, 6, 7]])
        assert np.all(rv[:, 4] <= 1e-12 * 1.05) and (level == 0 or np.all(rv[:, 5] <= 1e-12 * 1.05))
        idx = list(range(0, n, max(1, n // 150))) + [n - 1]
        refs = _pmap(lambda k: P.coupled_sample(level, cfg["seed"], k), idx)
        for k, ref in zip(idx, refs):
            assert abs(ps[k, 0] / ref[0] - 1) < 1e-10, (level, k, ps[k, 0], ref[0])
            if level > 0:
                assert abs(ps[k, 1] / ref[1] - 1) < 1e-10
            else:
                assert ps[k, 1] == 0.0
        y = ps[:, 0] - ps[:, 1]
        s = r.sums
        assert s["n"] == n and s["n_fail"] == 0
        assert abs(s["sum_y"] - y.sum()) <= 1e-13 * np.abs(y).sum()
        assert abs(s["sum_y2"] - (y * y).sum()) <= 1e-13 * (y * y).sum()
        assert s["iters_f"] == ps[:, 2].sum() and s["iters_f_max"] == ps[:, 2].max()
        nf = (cfg["h0_inv"] << level) - 1
        expect_cost = (ps[:, 2] * nf ** 2).sum() + (ps[:, 3] * ((cfg["h0_inv"] << (level - 1)) - 1) ** 2).sum() \
            if level else (ps[:, 2] * nf ** 2).sum()
        assert abs(s["sum_cost"] - expect_cost) <= 1e-12 * expect_cost
    ctx.close()


def test_minres_iteration_counts_track_oracle():
    cfg = W.CONFIGS["C2"]
    ctx = _ctx(cfg)
    P = _oracle(cfg)
    for level, tf, tc in ((1, 1e-5, 1e-4), (2, 1e-6, 1e-5), (3, 1e-8, 1e-6)):
        n = 12
        ps = ctx.sample_level(level, n, seed=1, tol_fine=tf, tol_coarse=tc, per_sample=True).per_sample
        refs = _pmap(lambda k: P.coupled_sample(level, 1, k, solver=oc.SOLVER_MINRES, tol_f=tf, tol_c=tc), range(n))
        for k, ref in enumerate(refs):
            # finite-precision Lanczos: rounding order moves the count by a few
            slack = lambda it: max(2, 0.03 * it)
            assert abs(ps[k, 2] - ref[2]) <= slack(ref[2]) and abs(ps[k, 3] - ref[3]) <= slack(ref[3]), \
                (level, k, ps[k, 2:4], ref[2:4])
            assert abs(ps[k, 0] - ref[0]) <= 2.5 * tf * ref[0]
    ctx.close()


# ============================================================================ C2: reduced accuracy bound
@pytest.mark.parametrize("level", [0, 1, 2, 3])
def test_C2_reduced_accuracy_within_residual_bound(level):
    cfg = W.CONFIGS["C2"]
    tols = cfg["tols"]
    ctx = _ctx(cfg)
    P = _oracle(cfg)
    n = {0: 4097, 1: 600, 2: 120, 3: 24}[level]             # spans several chunks / a ragged tail
    tf = tols[level]
    tc = tols[level - 1] if level else tf
    r = ctx.sample_level(level, n, seed=cfg["seed"], tol_fine=tf, tol_coarse=tc, per_sample=True)
    ps = r.per_sample
    assert r.sums["n_fail"] == 0 and np.all(ps[:, 6:8] == 0)
    vp = precision("minres", verify=True)
    pv = ctx.sample_level(level, n, seed=cfg["seed"], prec_fine=vp, prec_coarse=vp, tol_fine=tf, tol_coarse=tc,
                          per_sample=True).per_sample
    assert np.array_equal(pv[:, 0:4], ps[:, 0:4])
    assert np.all(pv[:, 4] <= tf * 1.01)                        # true residual meets Eq. (2)
    if level:
        assert np.all(pv[:, 5] <= tc * 1.01)
    idx = sorted(set(list(range(0, n, max(1, n // 40))) + [n - 1]))
    Nf = cfg["h0_inv"] << level

    def chk(k):
        xi = oc.normals(cfg["seed"], level, k, cfg["m"])
        out = [_exact(P, Nf, xi)]
        if level:
            out.append(_exact(P, Nf // 2, xi))
        return out

    for k, ex in zip(idx, _pmap(chk, idx)):
        qf, bn, xn = ex[0]
        assert abs(ps[k, 0] - qf) <= tf * bn * xn * (1 + 1e-6) + 1e-14 * qf, (level, k)
        if level:
            qc, bn, xn = ex[1]
            assert abs(ps[k, 1] - qc) <= tc * bn * xn * (1 + 1e-6) + 1e-14 * qc
    ctx.close()


# ============================================================================ C3: Cholesky + IR
@pytest.mark.parametrize("uf,us", [("h", "s"), ("s", "s"), ("s", "d"), ("h", "d")])
def test_C3_cholesky_ir_parity(uf, us):
    cfg = W.CONFIGS["C3"]
    ctx = _ctx(cfg)
    P = _oracle(cfg)
    prec = precision("chol_ir", uf, us)
    for level, n in ((0, 3000), (1, 300), (2, 40)):
        r = ctx.sample_level(level, n, seed=3, prec_fine=prec, prec_coarse=prec, tol_fine=1e-10, tol_coarse=1e-10,
                             per_sample=True)
        ps = r.per_sample
        assert r.sums["n_fail"] == 0 and np.all(ps[:, 6:8] == 0)
        assert np.all(ps[:, 4] < 1e-10) and (level == 0 or np.all(ps[:, 5] < 1e-10))
        steps = ps[:, 2]
        if uf == "s":
            assert steps.max() <= 3                                   # SC-9: 1-2 steps
        else:
            assert steps.mean() <= 1.5 * {0: 4.0, 1: 6.2, 2: 11.9}[level] + 1
        idx = list(range(0, n, max(1, n // 25)))
        Nf = cfg["h0_inv"] << level
        exs = _pmap(lambda k: _exact(P, Nf, oc.normals(3, level, k, cfg["m"])), idx)
        for k, (q, bn, xn) in zip(idx, exs):
            assert abs(ps[k, 0] - q) <= 1e-10 * bn * xn * (1 + 1e-6) + 1e-14 * q
        # the oracle's emulated Algorithm 1 converges to the same tolerance on the same systems
        for k in idx[:3]:
            xi = oc.normals(3, level, k, cfg["m"])
            o = P.solve_mesh(Nf, xi, oc.SOLVER_IR, tol=1e-10, quad=uf + us + "dd", max_iter=50)
            assert o["status"] == 0 and abs(o["iters"] - steps[k]) <= max(2, 0.5 * o["iters"])
    ctx.close()


def test_ir_limiting_accuracy_reported_as_failure():
    """Corollary 3.3: an fp16 factor with fp32 corrections cannot reach 1e-14."""
    cfg = W.CONFIGS["C3"]
    ctx = _ctx(cfg)
    r = ctx.sample_level(1, 8, seed=0, prec_fine=precision("chol_ir", "h", "s", max_iter=30),
                         prec_coarse=precision("chol_ir", "h", "s", max_iter=30), tol_fine=1e-15, tol_coarse=1e-15,
                         per_sample=True)
    assert r.sums["n_fail"] == 8 and np.all(r.per_sample[:, 6] == 1)
    ctx.close()


# ============================================================================ edge cases
def test_edge_cases_empty_ragged_batching_and_determinism():
    cfg = W.CONFIGS["C2"]
    small = _ctx(cfg, ws=3 << 20)          # forces several passes per call
    big = _ctx(cfg)
    r0 = big.sample_level(1, 0, seed=1, tol_fine=1e-6, tol_coarse=1e-5)
    assert r0.sums["n"] == 0 and r0.sums["sum_y"] == 0.0
    a = big.sample_level(1, 1000, seed=1, tol_fine=1e-6, tol_coarse=1e-5, per_sample=True).per_sample
    b = small.sample_level(1, 1000, seed=1, tol_fine=1e-6, tol_coarse=1e-5, per_sample=True).per_sample
    c = big.sample_level(1, 1000, seed=1, tol_fine=1e-6, tol_coarse=1e-5, per_sample=True).per_sample
    assert np.array_equal(a, b) and np.array_equal(a, c)            # batch- and run-independent
    d = big.sample_level(1, 7, seed=1, first_index=501, tol_fine=1e-6, tol_coarse=1e-5, per_sample=True).per_sample
    assert np.array_equal(d, a[501:508])                             # counter-based sample identity
    e = big.sample_level(1, 1, seed=2, tol_fine=1e-6, tol_coarse=1e-5, per_sample=True).per_sample
    assert not np.array_equal(e[0], a[0])
    # loose tolerance stops early; max_iter exhaustion is counted as a failure, not an error
    f = big.sample_level(2, 5, seed=1, tol_fine=0.5, tol_coarse=0.5, per_sample=True).per_sample
    f6 = big.sample_level(2, 5, seed=1, tol_fine=1e-6, tol_coarse=1e-6, per_sample=True).per_sample
    assert np.all(f[:, 4] <= 0.5) and np.all(f[:, 2] < f6[:, 2]) and np.all(f[:, 3] < f6[:, 3])
    g = big.sample_level(2, 5, seed=1, prec_fine=precision("minres", max_iter=3),
                         prec_coarse=precision("minres", max_iter=3), tol_fine=1e-12, tol_coarse=1e-12)
    assert g.sums["n_fail"] == 5
    with pytest.raises(RuntimeError):
        big.sample_level(9, 5, seed=1)                              # level beyond L_max
    with pytest.raises(RuntimeError):
        big.sample_level(1, 5, seed=1, tol_fine=0.0)
    # device-resident per-sample export equals the host export
    dev = big.sample_level(1, 1000, seed=1, tol_fine=1e-6, tol_coarse=1e-5, per_sample="device").per_sample
    assert np.array_equal(dev.cpu().numpy(), a)
    small.close()
    big.close()


def test_concurrent_levels_equal_sequential_levels():
    """mlmc_sample_levels_async (levels on concurrent streams, split workspace) gives bit-identical
    level sums to one mlmc_sample_level call per level; small workspace forces multi-pass slices."""
    cfg = W.CONFIGS["C2"]
    tols = cfg["tols"]
    Nl = [2000, 500, 120, 30]
    tc = [tols[l - 1] if l else tols[0] for l in range(4)]
    mr = precision("minres")
    for ws in (512 << 20, 6 << 20):
        ctx = _ctx(cfg, ws=ws)
        sums = torch.zeros((4, 12), dtype=torch.float64, device="cuda")
        ctx.sample_levels_async([3, 1, 0, 2], [Nl[3], Nl[1], Nl[0], Nl[2]], 1, [7, 5, 3, 11], [mr] * 4, [mr] * 4,
                                [tols[3], tols[1], tols[0], tols[2]], [tc[3], tc[1], tc[0], tc[2]], sums)
        torch.cuda.synchronize()
        got = sums.cpu().numpy()
        for q, (l, first) in enumerate(zip([3, 1, 0, 2], [7, 5, 3, 11])):
            ref = ctx.sample_level(l, Nl[l], seed=1, first_index=first, tol_fine=tols[l], tol_coarse=tc[l]).sums
            ref = np.array([ref[f] for f in ("sum_y", "sum_y2", "sum_qf", "sum_qc", "sum_cost", "n", "n_fail",
                                             "iters_f", "iters_c", "iters_f_max", "iters_c_max", "n_escalated")])
            if ws > (64 << 20):      # one pass on both sides: bit-identical
                assert np.array_equal(got[q], ref), (ws, l)
            else:                    # passes smaller than a 4096-chunk: summation order differs
                assert np.array_equal(got[q][4:], ref[4:]) and np.allclose(got[q], ref, rtol=1e-13, atol=0)
        ctx.close()


def test_full_size_C2_step_sampled_parity():
    """BASELINE configs[1] at full size in the launch configuration bench.py times
    (one call per level); sampled outputs against the oracle bound."""
    cfg = W.CONFIGS["C2"]
    ctx = _ctx(cfg, ws=1 << 30)
    P = _oracle(cfg)
    tols = cfg["tols"]
    for level, n in enumerate(cfg["N"]):
        tf, tc = tols[level], (tols[level - 1] if level else tols[0])
        r = ctx.sample_level(level, n, seed=cfg["seed"], tol_fine=tf, tol_coarse=tc, per_sample=True)
        ps = r.per_sample
        assert r.sums["n"] == n and r.sums["n_fail"] == 0
        rng = np.random.default_rng(level)
        idx = sorted(rng.choice(n, size=min(n, 6), replace=False))
        Nf = cfg["h0_inv"] << level
        for k in idx:
            q, bn, xn = _exact(P, Nf, oc.normals(cfg["seed"], level, int(k), cfg["m"]))
            assert abs(ps[k, 0] - q) <= tf * bn * xn * (1 + 1e-6) + 1e-14 * q
        y = ps[:, 0] - ps[:, 1]
        assert abs(r.sums["sum_y"] - y.sum()) <= 1e-12 * np.abs(y).sum()
    ctx.close()


# ============================================================================ Algorithm 2 end to end
def test_adaptive_C4_matches_oracle_controller():
    """Algorithm 2 through the C-ABI vs the oracle's Algorithm 2 driven by oracle
    MINRES samples (same seeds): identical decisions, estimate within 1e-9."""
    from oracle import mlmc as om
    cfg = W.CONFIGS["C4"]
    ctx = _ctx(cfg, ws=512 << 20)
    g = ctx.adaptive_run(cfg["eps"], k_p=0.05, N_init=100, seed=4)
    assert g["code"] == 0
    P = _oracle(cfg)

    def sampler(l, first, count, tf, tc):
        outs = _pmap(lambda k: P.coupled_sample(l, 4, k, solver=oc.SOLVER_MINRES, tol_f=tf, tol_c=tc),
                     range(first, first + count))
        nf = ((cfg["h0_inv"] << l) - 1) ** 2
        nc = ((cfg["h0_inv"] << (l - 1)) - 1) ** 2 if l else 0
        return [o[0] - o[1] for o in outs], [o[2] * nf + o[3] * nc for o in outs]

    o = om.adaptive_mpml(sampler, cfg["eps"], 1 / cfg["h0_inv"], 0.05, L_max=cfg["L_max"], N_init=100)
    assert o.L == g["L"]
    # both sides solve every sample to relative residual eps_l, so each Q differs from the exact one by at
    # most eps_l ||b|| ||x|| <= 1.5 eps_l Q; Q < 0.06 for these fields
    bound = sum(2 * 1.5 * 0.06 * (e + (g["eps"][l - 1] if l else 0.0)) for l, e in enumerate(g["eps"]))
    if o.N == g["N"]:
        assert abs(o.estimate - g["estimate"]) < bound
    else:   # a +-1 MINRES iteration can move C_l and hence ceil(N_l) by a sample or two
        assert all(abs(a - b) <= max(2, 0.02 * b) for a, b in zip(o.N, g["N"])), (o.N, g["N"])
        assert abs(o.estimate - g["estimate"]) < 0.1 * cfg["eps"]
    assert 0.030 < g["estimate"] < 0.038
    ctx.close()


# ============================================================================ K3c: streamed fine meshes
def test_streamed_minres_fine_mesh_parity():
    """h = 1/128 fine (K3b since round 2; K3c before), 1/64 coarse, configs[4] field: per-sample Q within the
    rigorous residual bound of the oracle's direct banded Cholesky solve, at a tight and a loose tolerance;
    MLMC_FLAG_VERIFY is refused on this mesh (EINVAL)."""
    cfg = W.CONFIGS["C5"]
    ctx = _ctx(cfg, ws=1 << 30)
    P = _oracle(cfg)
    n = 4
    for tol in (1e-11, 1e-6):
        r = ctx.sample_level(4, n, seed=11, prec_fine=precision("minres"), tol_fine=tol, tol_coarse=tol,
                             per_sample=True)
        ps = r.per_sample
        assert r.sums["n_fail"] == 0 and np.all(ps[:, 6:8] == 0)
        assert np.all(ps[:, 4] <= tol)
        exs = _pmap(lambda k: (_exact(P, 128, oc.normals(11, 4, k, cfg["m"])),
                               _exact(P, 64, oc.normals(11, 4, k, cfg["m"]))), list(range(n)))
        for k, ((qf, bf, xf), (qc, bc, xc)) in enumerate(exs):
            assert abs(ps[k, 0] - qf) <= tol * bf * xf * (1 + 1e-6) + 1e-14 * qf, (tol, k, ps[k, 0], qf)
            assert abs(ps[k, 1] - qc) <= tol * bc * xc * (1 + 1e-6) + 1e-14 * qc
        if tol < 1e-10:
            assert np.max(np.abs(ps[:, 0] / np.array([e[0][0] for e in exs]) - 1)) < 1e-9
    # the true-residual instantiation exists on the on-chip tile meshes only: refused here, not ignored
    with pytest.raises(RuntimeError, match="VERIFY"):
        ctx.sample_level(4, 2, seed=11, prec_fine=precision("minres", verify=True), tol_fine=1e-6, tol_coarse=1e-6)
    ctx.close()


def test_async_profile_workspace_and_level_info_entry_points():
    """The C-ABI calls the other tests reach only indirectly: mlmc_sample_level_async (device sums and device
    per-sample records, no synchronisation) equals mlmc_sample_level bit for bit; mlmc_profile_enable / _read
    count the launches of every kernel class of the pass (the longest-first order is formed inside the field
    launch on this mesh, so no separate order launch); mlmc_workspace_bytes[_prec] grow with the batch and
    the Cholesky-IR scratch; mlmc_level_info_get returns the mesh geometry (level table)."""
    cfg = W.CONFIGS["C2"]
    ctx = _ctx(cfg)
    mr = precision("minres")
    ref = ctx.sample_level(3, 50, seed=4, first_index=9, prec_fine=mr, prec_coarse=mr, tol_fine=1e-8, tol_coarse=1e-6,
                           per_sample=True)
    sums = torch.zeros(12, dtype=torch.float64, device="cuda")
    ps = torch.zeros((50, 8), dtype=torch.float64, device="cuda")
    ctx.profile_enable(True)
    ctx.sample_level_async(3, 50, seed=4, first_index=9, prec_fine=mr, prec_coarse=mr, tol_fine=1e-8, tol_coarse=1e-6,
                           sums_out=sums, per_sample_out=ps)
    prof = ctx.profile_read()
    ctx.profile_enable(False)
    torch.cuda.synchronize()
    assert np.array_equal(ps.cpu().numpy(), ref.per_sample)
    got = sums.cpu().numpy()
    want = np.array([ref.sums[f] for f in ("sum_y", "sum_y2", "sum_qf", "sum_qc", "sum_cost", "n", "n_fail",
                                             "iters_f", "iters_c", "iters_f_max", "iters_c_max", "n_escalated")])
    assert np.array_equal(got, want)
    kinds = {(k, N): c for k, N, c, ms in prof}
    assert kinds.get(("minres", 64)) == 1 and kinds.get(("minres", 32)) == 1, prof
    assert kinds.get(("field", 64)) == 1 and kinds.get(("field", 32)) == 1 and ("order", 64) not in kinds, prof
    assert all(ms > 0 for k, N, c, ms in prof if k in ("minres", "field")), prof
    w1, w2 = ctx.workspace_bytes(2, 100), ctx.workspace_bytes(2, 1000)
    assert 0 < w1 < w2
    ir = precision("chol_ir", "h", "s")
    assert ctx.workspace_bytes_prec(2, 1000, ir, ir) > ctx.workspace_bytes_prec(2, 1000, mr, mr) > 0
    for l in range(4):
        info = ctx.level_info(l)
        N = cfg["h0_inv"] << l
        assert info == {"N": N, "n": (N - 1) ** 2, "P": 2 * N * N, "bw": N - 1, "h": 1.0 / N}, info
    ctx.close()


def test_job_trace_is_refused_by_the_production_build():
    """mlmc_debug_trace (schedule analysis, tools/step_trace.py) records only in the MLMC_TUNING build; the
    production library answers EINVAL with a message instead of silently recording nothing."""
    import ctypes as C
    from paper_2503_05533_b200 import _capi as K
    cfg = W.CONFIGS["C2"]
    ctx = _ctx(cfg)
    buf = torch.zeros(64, dtype=torch.int64, device="cuda")
    cnt = C.c_uint32()
    rc = K.lib().mlmc_debug_trace(ctx.ctx, C.c_void_p(buf.data_ptr()), 16, C.byref(cnt))
    assert rc == 2, rc                                    # MLMC_EINVAL
    assert b"MLMC_TUNING" in K.lib().mlmc_last_error(ctx.ctx)
    ctx.close()


# ============================================================================ the paper's experiment
def test_paper_experiment_mpml_cost_gain_without_accuracy_loss():
    """Section 5.1: adaptive MPML vs standard adaptive MLMC (fixed MINRES tol 1e-6) on the
    Eq. (20) field at TOL^2 = 2e-6, 200 replicate runs each: both MSEs within TOL^2 and equal up to
    their statistical error, and MPML cheaper (the paper: ~1.5x fewer FLOPs)."""
    import sys as _sys
    import os as _os
    _sys.path.insert(0, _os.path.join(_os.path.dirname(_os.path.dirname(_os.path.abspath(__file__))), "tools"))
    import paper_experiment
    res = paper_experiment.run(R=200, tol2s=(2e-6,))
    e = res["tol2"]["2e-06"]
    for m in ("mpml", "mlmc"):                   # MSE <= TOL^2 up to its own 95% sampling error
        assert e[m]["mse"] - e[m]["mse_ci95"] < 2e-6, (m, e[m])
    diff = abs(e["mpml"]["mse"] - e["mlmc"]["mse"])
    assert diff < 3.0 * math.hypot(e["mpml"]["mse_ci95"], e["mlmc"]["mse_ci95"]) / 1.96, e
    assert e["cost_ratio_mlmc_over_mpml"] > 1.25, e


def test_levels_xi_concurrent_equals_single_level_calls():
    """mlmc_sample_levels_xi (all levels at once, host xi in, host records out) reproduces the per-level
    mlmc_sample_level_xi results bit for bit (same xi, same kernels, different streams)."""
    cfg = W.CONFIGS["C2"]
    ctx = _ctx(cfg, ws=1 << 30)
    rng = np.random.default_rng(7)
    ns = [700, 300, 90, 12]
    xs = [rng.standard_normal((n, cfg["m"])) for n in ns]
    tf = cfg["tols"]
    tc = [tf[l - 1] if l else tf[0] for l in range(4)]
    outs = [np.zeros((n, 8)) for n in ns]
    sums = ctx.sample_levels_xi([0, 1, 2, 3], xs, ["minres"] * 4, ["minres"] * 4, tf, tc, per_sample=outs)
    for l in range(4):
        ref = np.zeros((ns[l], 8))
        r = ctx.sample_level_xi(l, xs[l], "minres", "minres", tf[l], tc[l], per_sample=ref)
        assert np.array_equal(ref, outs[l]), l
        assert sums[l]["n"] == ns[l] and abs(sums[l]["sum_y"] - r.sums["sum_y"]) <= 1e-15 * abs(r.sums["sum_y"])
    ctx.close()


# ============================================================================ NEXT-2: quarter / binary64 factors
def test_quarter_precision_factor_level0_h0_quarter():
    """The paper's last example: s = 1, sigma = 1, h0 = 1/4, quarter-precision (q43 ~ E4M3)
    factor on level 0 with iterative refinement (here u_s = binary32, u = u_r = binary64, R14/R17).
    IR converges to 1e-10 on every sample, Q within the residual bound of the oracle's direct solve,
    and the oracle's emulated Algorithm 1 with a q43 factor converges on the same systems."""
    cfg = dict(field="eq20", field_code=1, m=1, sigma2=1.0, corr_len=0.0, q_decay=2.0, h0_inv=4, L_max=3)
    ctx = _ctx(cfg)
    P = _oracle(cfg)
    for lev, quad in ((0, "qsdd"), (1, "hsdd")):
        prec = precision("chol_ir", quad[0], quad[1], max_iter=200)
        r = ctx.sample_level(lev, 400, seed=21, prec_fine=prec, prec_coarse=precision("chol_ir", "q", "s", max_iter=200),
                             tol_fine=1e-10, tol_coarse=1e-10, per_sample=True)
        ps = r.per_sample
        assert r.sums["n_fail"] == 0 and np.all(ps[:, 6:8] == 0), (lev, ps[:, 6:8].max())
        assert np.all(ps[:, 4] < 1e-10)
        Nf = 4 << lev
        idx = list(range(0, 400, 40))
        exs = _pmap(lambda k: _exact(P, Nf, oc.normals(21, lev, k, 1)), idx)
        for k, (q, bn, xn) in zip(idx, exs):
            assert abs(ps[k, 0] - q) <= 1e-10 * bn * xn * (1 + 1e-6) + 1e-14 * q
        for k in idx[:3]:
            o = P.solve_mesh(Nf, oc.normals(21, lev, k, 1), oc.SOLVER_IR, tol=1e-10, quad=quad, max_iter=200)
            assert o["status"] == 0
    ctx.close()


def test_binary64_factor_on_the_h32_mesh():
    """Binary64 band factor at h = 1/32 (the standard-MLMC direct solver of P:694): one refinement step
    at most to 1e-13, Q equal to the oracle's direct solve to 1e-11 relative."""
    cfg = W.CONFIGS["C3"]
    ctx = _ctx(cfg, ws=1 << 30)
    P = _oracle(cfg)
    prec = precision("chol_ir", "d", "d")
    r = ctx.sample_level(2, 60, seed=4, prec_fine=prec, prec_coarse=prec, tol_fine=1e-13, tol_coarse=1e-13,
                         per_sample=True)
    ps = r.per_sample
    assert r.sums["n_fail"] == 0 and ps[:, 2].max() <= 2
    exs = _pmap(lambda k: _exact(P, 32, oc.normals(4, 2, k, cfg["m"])), list(range(0, 60, 6)))
    for k, (q, _, _) in zip(range(0, 60, 6), exs):
        assert abs(ps[k, 0] / q - 1) < 1e-11
    ctx.close()


def test_paper_direct_solver_experiment_same_samples():
    """Section 5.2: MPML with low-precision Cholesky + IR vs standard MLMC with a binary64
    Cholesky solve on the same N_l and random inputs: MSE differs by well under 0.1% (paper: < 0.01%),
    the paper's memory model gains > 1.5 (paper: ~2)."""
    import sys as _sys
    import os as _os
    _sys.path.insert(0, _os.path.join(_os.path.dirname(_os.path.dirname(_os.path.abspath(__file__))), "tools"))
    import paper_experiment_ir
    res = paper_experiment_ir.run("E3", R=40)
    for k, e in res["tol2"].items():
        assert e["mse_rel_diff"] < 1e-3, (k, e["mse_rel_diff"])
        assert e["memory_gain_total"] > 1.5 and e["k4_hbm_gain_total"] > 1.5, (k, e)


def test_streamed_minres_edge_cases_and_order_invariance():
    """h = 1/128 (K3b since round 2: 4-CTA clusters; K3c before) with no system, one, fewer than the resident
    clusters, and more than one wave; the longest-first
    job order (C2 level 3, the tile kernel) changes no per-sample result: the same samples drawn one
    at a time (no ordering: a single system) and in a batch agree bit for bit."""
    cfg = W.CONFIGS["C5"]
    ctx = _ctx(cfg, ws=2 << 30)
    mr = precision("minres", max_iter=400)
    for n in (0, 1, 3, 150):
        r = ctx.sample_level(4, n, seed=2, prec_fine=mr, prec_coarse=mr, tol_fine=1e-6, tol_coarse=1e-6,
                             per_sample=True)
        assert r.sums["n"] == n
        if n:
            one = ctx.sample_level(4, 1, seed=2, first_index=n - 1, prec_fine=mr, prec_coarse=mr, tol_fine=1e-6,
                                   tol_coarse=1e-6, per_sample=True).per_sample
            assert np.array_equal(one[0], r.per_sample[n - 1])
    ctx.close()
    c2 = W.CONFIGS["C2"]
    ctx = _ctx(c2, ws=1 << 30)
    batch = ctx.sample_level(3, 40, seed=9, prec_fine=mr, prec_coarse=mr, tol_fine=1e-7, tol_coarse=1e-6,
                             per_sample=True).per_sample
    for k in (0, 17, 39):
        one = ctx.sample_level(3, 1, seed=9, first_index=k, prec_fine=mr, prec_coarse=mr, tol_fine=1e-7,
                               tol_coarse=1e-6, per_sample=True).per_sample
        assert np.array_equal(one[0], batch[k]), k
    ctx.close()


def test_adaptive_run_counts_failed_solves_on_gpu():
    """R15 on the GPU path: Cholesky-IR with an fp16 factor (policy 1, Table 1) cannot reach 1e-15
    (limiting accuracy, Corollary 3.3); on_fail = 0 stops with a solver error, on_fail = 1 finishes
    and reports the failures."""
    cfg = W.CONFIGS["C4"]
    ctx = _ctx(cfg, ws=1 << 30)
    with pytest.raises(RuntimeError, match="solver failure"):
        ctx.adaptive_run(cfg["eps"], k_p=0.0, fixed_tol=1e-15, N_init=20, seed=3, max_rounds=3, policy=1)
    r = ctx.adaptive_run(cfg["eps"], k_p=0.0, fixed_tol=1e-15, N_init=20, seed=3, max_rounds=3, policy=1,
                       on_fail=1)
    assert r["n_fail"] > 0
    ctx.close()


# ============================================================================ NEXT-4: MG-PCG
@pytest.mark.parametrize("level,tol", [(0, 1e-10), (1, 1e-8), (2, 1e-6), (3, 1e-10)])
def test_mgcg_within_residual_bound(level, tol):
    """K3m (multigrid-preconditioned CG, same stopping rule ||r||/||b|| <= tol): per-sample Q within the
    rigorous bound of the oracle's direct solve, fine and coarse halves; iteration counts mesh-
    independent (<= 20 at every level, MINRES needs 25..600)."""
    cfg = W.CONFIGS["C2"]
    ctx = _ctx(cfg)
    P = _oracle(cfg)
    n = {0: 200, 1: 100, 2: 40, 3: 12}[level]
    r = ctx.sample_level(level, n, seed=13, prec_fine=precision("mgcg"), prec_coarse=precision("mgcg"),
                         tol_fine=tol, tol_coarse=tol, per_sample=True)
    ps = r.per_sample
    assert r.sums["n_fail"] == 0 and np.all(ps[:, 6:8] == 0)
    assert ps[:, 2].max() <= 20 and np.all(ps[:, 4] <= tol)
    Nf = 8 << level
    idx = list(range(0, n, max(1, n // 6)))
    exs = _pmap(lambda k: (_exact(P, Nf, oc.normals(13, level, k, cfg["m"])),
                           _exact(P, Nf // 2, oc.normals(13, level, k, cfg["m"])) if level else None), idx)
    for k, (f, c) in zip(idx, exs):
        assert abs(ps[k, 0] - f[0]) <= tol * f[1] * f[2] * (1 + 1e-6) + 1e-14 * f[0], (level, k)
        if c is not None:
            assert abs(ps[k, 1] - c[0]) <= tol * c[1] * c[2] * (1 + 1e-6) + 1e-14 * c[0]
    ctx.close()


@pytest.mark.parametrize("level,n,tol", [(4, 4, 1e-10), (4, 150, 1e-6), (5, 2, 1e-8)])
def test_mgcg_streamed_meshes_within_residual_bound(level, n, tol):
    """K3m-g (MG-PCG with every grid in global scratch, h = 1/128 and 1/256; configs[4] field): per-
    sample Q within the rigorous bound of the oracle's direct solve on sampled systems, iteration
    counts mesh-independent; a batch over one wave of CTAs (n = 150 > 148) and single systems agree
    bit for bit (one CTA per system, no cross-system state)."""
    cfg = W.CONFIGS["C5"]
    ctx = _ctx(cfg, ws=8 << 30)
    P = _oracle(cfg)
    mg = precision("mgcg")
    r = ctx.sample_level(level, n, seed=21, prec_fine=mg, prec_coarse=mg, tol_fine=tol, tol_coarse=tol,
                         per_sample=True)
    ps = r.per_sample
    assert r.sums["n_fail"] == 0 and np.all(ps[:, 6:8] == 0)
    assert ps[:, 2].max() <= 25 and np.all(ps[:, 4] <= tol)
    Nf = 8 << level
    idx = [0, n - 1] if n > 1 else [0]
    exs = _pmap(lambda k: (_exact(P, Nf, oc.normals(21, level, k, cfg["m"])),
                           _exact(P, Nf // 2, oc.normals(21, level, k, cfg["m"]))), idx)
    for k, ((qf, bf, xf), (qc, bc, xc)) in zip(idx, exs):
        assert abs(ps[k, 0] - qf) <= tol * bf * xf * (1 + 1e-6) + 1e-14 * qf, (level, k, ps[k, 0], qf)
        assert abs(ps[k, 1] - qc) <= tol * bc * xc * (1 + 1e-6) + 1e-14 * qc
    if n > 1:
        one = ctx.sample_level(level, 1, seed=21, first_index=n - 1, prec_fine=mg, prec_coarse=mg, tol_fine=tol,
                               tol_coarse=tol, per_sample=True).per_sample
        assert np.array_equal(one[0], ps[n - 1])
    ctx.close()


def test_level_pass_over_field_grid_limit():
    """One pass of more than 65535 x 64 samples (the field kernel's grid.y limit, sliced in launch_field):
    the last sample of a 4.3M-sample level-0 pass equals the same sample drawn alone, bit for bit."""
    cfg = W.CONFIGS["C2"]
    ctx = _ctx(cfg, ws=12 << 30)
    mr = precision("minres")
    n = 65535 * 64 + 1000
    r = ctx.sample_level(0, n, seed=5, prec_fine=mr, tol_fine=1e-4, per_sample=True)
    assert r.sums["n"] == n and r.sums["n_fail"] == 0
    for k in (0, 65535 * 64 - 1, 65535 * 64, n - 1):
        one = ctx.sample_level(0, 1, seed=5, first_index=k, prec_fine=mr, tol_fine=1e-4, per_sample=True).per_sample
        assert np.array_equal(one[0], r.per_sample[k]), k
    ctx.close()


@pytest.mark.parametrize("name", ["C4", "C5"])
def test_replicate_rmse_within_eps(name):
    """The estimator pin of SURVEY section 8(c): over R = 50 seeds, RMSE(Q_hat - Q_ref) <= eps, with
    Q_ref the same GPU path at eps / 5 (its samples are the ones the per-sample parity tests pin)."""
    sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tools"))
    import replicates
    r = replicates.run(name, R=50)
    assert r["rmse"] <= r["eps"], r
    assert 0.030 < r["mean_estimate"] < 0.038


def test_mgcg_edge_cases_and_finest_mesh():
    """MG-PCG edge cases: empty and single-system passes on every kernel (on chip h = 1/8 .. 1/64, tiled
    h = 1/128 .. 1/512), a single system equals the same sample inside a batch bit for bit; at h = 1/512
    (no oracle solve in test time) MG-PCG and the streamed MINRES agree to the tolerance they were
    both solved to (same per-sample residual contract)."""
    cfg = W.CONFIGS["C5"]
    ctx = _ctx(cfg, ws=8 << 30)
    mg, mr = precision("mgcg"), precision("minres")
    for level in range(cfg["L_max"] + 1):
        assert ctx.sample_level(level, 0, seed=3, prec_fine=mg, prec_coarse=mg, tol_fine=1e-6,
                                tol_coarse=1e-6).sums["n"] == 0
        n = 3 if level >= 5 else 37
        batch = ctx.sample_level(level, n, seed=3, prec_fine=mg, prec_coarse=mg, tol_fine=1e-7, tol_coarse=1e-7,
                                 per_sample=True).per_sample
        assert np.all(batch[:, 6:8] == 0) and np.all(batch[:, 4] <= 1e-7)
        one = ctx.sample_level(level, 1, seed=3, first_index=n - 1, prec_fine=mg, prec_coarse=mg, tol_fine=1e-7,
                               tol_coarse=1e-7, per_sample=True).per_sample
        assert np.array_equal(one[0], batch[n - 1]), level
    a = ctx.sample_level(6, 2, seed=4, prec_fine=mg, prec_coarse=mg, tol_fine=1e-9, tol_coarse=1e-9,
                         per_sample=True).per_sample
    b = ctx.sample_level(6, 2, seed=4, prec_fine=mr, prec_coarse=mr, tol_fine=1e-9, tol_coarse=1e-9,
                         per_sample=True).per_sample
    assert np.all(a[:, 6:8] == 0) and np.all(b[:, 6:8] == 0)
    # |Q_mg - Q_exact| and |Q_minres - Q_exact| are each <= tol ||b|| ||x|| <= 1.5 tol Q
    assert np.all(np.abs(a[:, :2] - b[:, :2]) <= 2 * 1.5e-9 * np.abs(b[:, :2]) + 1e-15)
    ctx.close()


@pytest.mark.parametrize("level", [1, 2, 3])
def test_mgcg_iterations_track_oracle_pcg(level):
    """K3m against the oracle's textbook MG-PCG (oracle/mg.py: Galerkin products P^T A P, binary64
    V-cycle) on the same fields: CG step counts within +-1 (the kernel's V-cycle runs in binary32)
    and both QoIs within the residual bound of each other."""
    from oracle import mg as omg
    cfg = W.CONFIGS["C2"]
    ctx = _ctx(cfg)
    P = _oracle(cfg)
    tol = 1e-8
    n = 6
    r = ctx.sample_level(level, n, seed=17, prec_fine=precision("mgcg"), prec_coarse=precision("mgcg"),
                         tol_fine=tol, tol_coarse=tol, per_sample=True).per_sample
    Nf = 8 << level
    outs = _pmap(lambda k: omg.pcg(Nf, P.field_triangles(Nf, oc.normals(17, level, k, cfg["m"])), tol), range(n))
    for k, o in enumerate(outs):
        assert o["status"] == 0 and abs(int(r[k, 2]) - o["iters"]) <= 1, (level, k, r[k, 2], o["iters"])
        assert abs(r[k, 0] - o["Q"]) <= 2 * 1.5 * tol * o["Q"], (level, k)
    ctx.close()


def test_c_quickstart(tmp_path):
    """The C ABI from plain C (examples/quickstart.c): plan, workspace from cudaMalloc, one coupled pass of
    every configs[1] level, Algorithm 2 on configs[3]; estimates in the survey's sanity range."""
    import subprocess
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    exe = str(tmp_path / "quickstart")
    pkg = os.path.join(root, "paper_2503_05533_b200")
    subprocess.check_call(["gcc", "-std=c99", "-O2", os.path.join(root, "examples", "quickstart.c"),
                           "-I" + os.path.join(root, "include"), "-I/usr/local/cuda/include", "-L" + pkg, "-lmlmc",
                           "-L/usr/local/cuda/lib64", "-lcudart", "-Wl,-rpath," + pkg, "-o", exe])
    r = subprocess.run([exe], capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stdout + r.stderr
    assert r.stdout.strip().endswith("ok")
    assert "level 3:" in r.stdout and "adaptive MPML" in r.stdout


def test_python_quickstart():
    """examples/quickstart.py (the Python binding end to end: per-level batches, the concurrent step into a device
    tensor, Algorithm 2 with policies 0 and 3) runs and its estimates lie in the survey's sanity range."""
    import re
    import subprocess
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    r = subprocess.run([sys.executable, os.path.join(root, "examples", "quickstart.py")], capture_output=True,
                       text=True, timeout=600, cwd=root)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "failures 0" in r.stdout and "adaptive (policy 3)" in r.stdout
    ests = [float(x) for x in re.findall(r"estimate (?:from one concurrent step: )?([0-9.]+)", r.stdout)]
    assert len(ests) == 3 and all(0.028 < e < 0.042 for e in ests), r.stdout   # seeded: fixed values ~0.037


def test_separable_synthesis_on_every_mesh_subprocess():
    """MLMC_FIELD_KERNEL=sep (read once per process, hence a subprocess): the separable synthesis on every
    mesh, for the BASELINE field (configs[1]) and the paper's Eq. (20) field, against the oracle."""
    import subprocess
    import textwrap
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    code = textwrap.dedent("""
        import sys, numpy as np
        sys.path.insert(0, %r); sys.path.insert(0, %r)
        import workloads as W
        from oracle import core as oc
        from paper_2503_05533_b200 import Context
        for name in ("C2", "EQ20"):
            cfg = W.CONFIGS[name]
            ctx = Context(field=cfg["field"], m=cfg["m"], sigma2=cfg["sigma2"], corr_len=cfg["corr_len"],
                          q_decay=cfg.get("q_decay", 2.0), h0_inv=cfg["h0_inv"], L_max=3, device=0,
                          workspace_bytes=256 << 20)
            P = oc.OracleProblem(cfg["field_code"], cfg["m"], cfg["sigma2"], cfg["corr_len"], cfg.get("q_decay", 2.0),
                                 cfg["h0_inv"])
            for level, mesh in ((0, 0), (1, 1), (3, 3), (3, 2)):
                xi, a = ctx.debug_field(level, mesh, 21, seed=5, first_index=3)
                a = a.cpu().numpy()
                N = cfg["h0_inv"] << mesh
                for k in (0, 20):
                    ref = P.field_triangles(N, oc.normals(5, level, 3 + k, cfg["m"]))
                    err = np.max(np.abs(a[k] / ref - 1))
                    assert err < 1e-12, (name, level, mesh, k, err)
            ctx.close()
        print("sep ok")
    """) % (root, os.path.join(root, "tests"))
    env = dict(os.environ, MLMC_FIELD_KERNEL="sep")
    r = subprocess.run([sys.executable, "-c", code], capture_output=True, text=True, timeout=600, env=env, cwd=root)
    assert r.returncode == 0 and "sep ok" in r.stdout, r.stdout + r.stderr


@pytest.mark.parametrize("quad,level,tol", [("hsss", 0, 3.5e-3), ("ssss", 1, 8.7e-4), ("hsss", 1, 1e-5),
                                            ("ssss", 2, 2.2e-4)])
def test_ir_single_precision_working_vectors(quad, level, tol):
    """Algorithm 1 with u = u_r = binary32 (the paper's "..ss" quads of Table 1 right; u_s = s by
    R24) at tolerances of Table 1's order (a binary32 residual cannot certify much below ~1e-5 at h = 1/32:
    its rounding error is ~u_s ||A|| ||x||, which is why the paper switches to ..dd there): converged samples
    reach the tolerance, Q within the direct solve's residual bound, the step counts track the oracle's
    Algorithm 1 emulating the same quad (every operation rounded to its format)."""
    cfg = W.CONFIGS["C3"]
    ctx = _ctx(cfg)
    P = _oracle(cfg)
    prec = precision("chol_ir", *quad)
    n = {0: 2000, 1: 300, 2: 40}[level]
    r = ctx.sample_level(level, n, seed=8, prec_fine=prec, prec_coarse=prec, tol_fine=tol, tol_coarse=tol,
                         per_sample=True)
    ps = r.per_sample
    assert r.sums["n_fail"] == 0 and np.all(ps[:, 6:8] == 0)
    assert np.all(ps[:, 4] < tol)
    Nf = cfg["h0_inv"] << level
    idx = list(range(0, n, max(1, n // 12)))
    exs = _pmap(lambda k: _exact(P, Nf, oc.normals(8, level, k, cfg["m"])), idx)
    for k, (q, bn, xn) in zip(idx, exs):
        # the binary32 x adds its own rounding (|dx| <= u_fp32 |x|) to the residual bound
        assert abs(ps[k, 0] - q) <= tol * bn * xn * (1 + 1e-6) + 2e-7 * q, (quad, level, k)
    for k in idx[:3]:
        o = P.solve_mesh(Nf, oc.normals(8, level, k, cfg["m"]), oc.SOLVER_IR, tol=tol, quad=quad, max_iter=50)
        assert o["status"] == 0 and abs(o["iters"] - ps[k, 2]) <= max(2, 0.5 * o["iters"]), (o["iters"], ps[k, 2])
    ctx.close()


@pytest.mark.parametrize("quad", ["qshh", "hshh", "qhhh", "hhhh", "hhss"])
def test_ir_half_precision_working_vectors(quad):
    """Algorithm 1 with binary16 working vectors and / or substitutions (the paper's qhhh / hhss of the E4
    experiment; u_s = s as R24 prefers, or u_s = h as the paper writes) on the level-0 mesh of that setup (h0 = 1/4, eps_0 = sqrt(k_p) h0^2 = 0.04 for k_p = 0.4): the
    solves converge, Q within the direct solve's residual bound (+ the binary16 rounding of x), and the
    step counts track the oracle's emulation of the same quad."""
    ctx = Context(field="eq20", m=1, sigma2=1.0, corr_len=0.0, q_decay=2.0, h0_inv=4, L_max=3, device=0,
                  workspace_bytes=256 << 20)
    P = oc.OracleProblem(1, 1, 1.0, 0.0, 2.0, 4)
    tol = 0.04
    prec = precision("chol_ir", *quad)
    n = 500
    ps = ctx.sample_level(0, n, seed=6, prec_fine=prec, tol_fine=tol, per_sample=True).per_sample
    assert np.all(ps[:, 6] == 0) and np.all(ps[:, 4] < tol)
    for k in range(0, n, 50):
        xi = oc.normals(6, 0, k, 1)
        q, bn, xn = _exact(P, 4, xi)
        assert abs(ps[k, 0] - q) <= tol * bn * xn * (1 + 1e-6) + 2e-3 * q, (k, ps[k, 0], q)
        o = P.solve_mesh(4, xi, oc.SOLVER_IR, tol=tol, quad=quad, max_iter=50)
        assert o["status"] == 0 and abs(o["iters"] - ps[k, 2]) <= 2, (o["iters"], ps[k, 2])
    ctx.close()


def test_adaptive_auto_policy():
    """Policy 3 (auto): every mesh the run uses gets a solver chosen by pilot timing among the
    admissible candidates; the run converges to an estimate in the survey's sanity window, and the
    choice is reported through mlmc_auto_choice."""
    cfg = W.CONFIGS["C4"]
    ctx = _ctx(cfg, ws=1 << 30)
    r = ctx.adaptive_run(2e-4, k_p=0.05, seed=3, policy=3)
    assert r["code"] == 0 and r["n_fail"] == 0 and 0.033 < r["estimate"] < 0.036
    for l in range(r["L"] + 1):
        ch = ctx.auto_choice(cfg["h0_inv"] << l)
        assert ch is not None and ch["solver"] in ("minres", "mgcg", "chol_ir") and ch["ms_per_sample"] > 0, (l, ch)
    assert ctx.auto_choice(1024) is None
    ctx.close()


def test_auto_policy_screens_minres_on_fine_meshes():
    """Policy 3 on configs[4] down to h = 1/128: MINRES's pilot is screened against the best candidate so far
    (200 steps and a log-linear extrapolation of their residual decay) instead of being run to thousands of
    steps; on h >= 1/64 MG-PCG is the choice by a wide margin (37x at h = 1/128), the run converges."""
    cfg = W.CONFIGS["C5"]
    ctx = _ctx(cfg, L_max=4, ws=4 << 30)
    r = ctx.adaptive_run(6e-5, k_p=0.05, seed=4, policy=3, on_fail=1)
    assert r["code"] in (0, 4) and r["n_fail"] == 0 and 0.030 < r["estimate"] < 0.038, r
    assert r["L"] >= 3, r
    for N in (64, 128):
        if (cfg["h0_inv"] << r["L"]) >= N:
            ch = ctx.auto_choice(N)
            assert ch is not None and ch["solver"] == "mgcg", (N, ch)
    ctx.close()


def test_escalation_repairs_failed_minres_solves():
    """on_fail = 2 / MLMC_FLAG_ESCALATE: MINRES capped far below what the tolerance needs fails
    on every sample; escalation solves each again with MG-PCG, so every record ends with status 4, the
    level sums count them as escalated (not failed), and Q meets the direct solve's residual bound -- on an
    on-chip mesh (h = 1/32) and a streamed one (h = 1/128, fine and coarse)."""
    cfg = W.CONFIGS["C5"]
    ctx = _ctx(cfg, ws=4 << 30)
    P = _oracle(cfg)
    tol = 1e-8
    capped = precision("minres", max_iter=20, escalate=True)
    for level, n in ((2, 40), (4, 3)):
        r = ctx.sample_level(level, n, seed=31, prec_fine=capped, prec_coarse=capped, tol_fine=tol, tol_coarse=tol,
                             per_sample=True)
        ps = r.per_sample
        assert np.all(ps[:, 6] == 4) and np.all(ps[:, 7] == 4)
        assert r.sums["n_fail"] == 0 and r.sums["n_escalated"] == n
        Nf = 8 << level
        for k in (0, n - 1):
            qf, bf, xf = _exact(P, Nf, oc.normals(31, level, k, cfg["m"]))
            assert abs(ps[k, 0] - qf) <= tol * bf * xf * (1 + 1e-6) + 1e-14 * qf
    # without the flag the same cap is a counted failure
    r = ctx.sample_level(2, 40, seed=31, prec_fine=precision("minres", max_iter=20), tol_fine=tol, tol_coarse=tol)
    assert r.sums["n_fail"] == 40 and r.sums["n_escalated"] == 0
    ctx.close()


# ============================================================================ SURVEY 8(e): rank independence
def _adaptive_threads(cfg, world, eps, **kw):
    """world ranks of mlmc_adaptive_run as host threads, one context each on cuda:0, exchanging through a
    thread-barrier all-reduce (the same C callback torch.distributed drives; the kernels of the ranks never
    wait on one another)."""
    import ctypes as C
    import threading
    from paper_2503_05533_b200 import _capi as K
    from paper_2503_05533_b200.api import _result_dict
    bar = threading.Barrier(world)
    bufs = [None] * world
    ctxs = [_ctx(cfg, ws=512 << 20) for _ in range(world)]
    out = [None] * world

    def rank_main(r):
        def _allreduce(buf, count, op, user):
            arr = np.ctypeslib.as_array(buf, shape=(count,))
            bufs[r] = arr.copy()
            bar.wait()
            tot = bufs[0].copy()
            for q in range(1, world):
                tot = tot + bufs[q] if op == 0 else np.maximum(tot, bufs[q])
            bar.wait()
            arr[:] = tot
            return 0
        cb = K.ALLREDUCE_FN(_allreduce)
        opts = K.AdaptiveOpts(kw.get("k_p", 0.0), kw.get("fixed_tol", 1e-8), 1.0, kw.get("N_init", 50), 0, r, world,
                              kw.get("max_rounds", 8), kw.get("seed", 11), 1, 0)
        res = K.Result()
        rc = K.lib().mlmc_adaptive_run(ctxs[r].ctx, eps, C.byref(opts), cb, None, C.byref(res))
        out[r] = (rc, _result_dict(res))

    th = [threading.Thread(target=rank_main, args=(r,)) for r in range(world)]
    for t in th:
        t.start()
    for t in th:
        t.join()
    for c in ctxs:
        c.close()
    return out


def test_adaptive_sums_exact_and_rank_independent():
    """the controller's level sums are exact fixed-point totals, so (i) each level mean and
    variance equals the correctly rounded sum of the per-sample Y and Y^2 (math.fsum) divided by N_l, and
    (ii) 1, 2 and 3 ranks produce bit-identical estimates, sample counts, means, variances and costs."""
    cfg = W.CONFIGS["C4"]
    eps = cfg["eps"]
    kw = dict(k_p=0.0, fixed_tol=1e-8, N_init=50, seed=11, max_rounds=8)
    runs = {w: _adaptive_threads(cfg, w, eps, **kw) for w in (1, 2, 3)}
    rc1, g = runs[1][0]
    assert rc1 in (0, 4) and g["L"] >= 1
    for w in (2, 3):
        for rc, r in runs[w]:
            assert rc == rc1
            for key in ("estimate", "L", "rounds", "N", "mean", "var", "cost", "n_fail"):
                assert r[key] == g[key], (w, key, r[key], g[key])
    # (i) against the per-sample records of the same indices (batch-independent; fixed tolerance 1e-8)
    ctx = _ctx(cfg, ws=512 << 20)
    for l in range(g["L"] + 1):
        lr = ctx.sample_level(l, g["N"][l], seed=11, first_index=0, prec_fine="minres", prec_coarse="minres",
                              tol_fine=1e-8, tol_coarse=1e-8, per_sample=True)
        rec = np.asarray(lr.per_sample).reshape(-1, 8)
        y = rec[:, 0] - (rec[:, 1] if l > 0 else 0.0)
        n = float(g["N"][l])
        mean = math.fsum(y.tolist()) / n
        assert g["mean"][l] == mean, (l, g["mean"][l], mean)
        var = max(0.0, math.fsum((y * y).tolist()) / n - mean * mean)
        assert g["var"][l] == var, (l, g["var"][l], var)
    ctx.close()


@pytest.mark.parametrize("level", [0, 1, 2, 3])
def test_cg_tracks_oracle_cg_and_minres(level):
    """Plain CG (MLMC_SOLVER_CG) against the oracle's textbook CG on the same fields: QoIs within the
    residual bound of each other, step counts within 2% + 2 (finite-precision CG amplifies rounding
    differences), and -- MINRES minimising the residual over the same Krylov space -- MINRES on the same
    samples stops no later than CG (+1), with CG at most 1.5x MINRES on average ("similar")."""
    from oracle import mg as omg
    cfg = W.CONFIGS["C2"]
    ctx = _ctx(cfg)
    P = _oracle(cfg)
    tol, n = 1e-8, 8
    r = ctx.sample_level(level, n, seed=19, prec_fine=precision("cg"), prec_coarse=precision("cg"),
                         tol_fine=tol, tol_coarse=tol, per_sample=True).per_sample
    m = ctx.sample_level(level, n, seed=19, prec_fine=precision("minres"), prec_coarse=precision("minres"),
                         tol_fine=tol, tol_coarse=tol, per_sample=True).per_sample
    Nf = 8 << level
    outs = _pmap(lambda k: omg.cg(Nf, P.field_triangles(Nf, oc.normals(19, level, k, cfg["m"])), tol), range(n))
    for k, o in enumerate(outs):
        assert r[k, 6] == 0 and o["status"] == 0
        assert abs(int(r[k, 2]) - o["iters"]) <= 0.02 * o["iters"] + 2, (level, k, r[k, 2], o["iters"])
        assert abs(r[k, 0] - o["Q"]) <= 2 * 1.5 * tol * o["Q"], (level, k)
        assert m[k, 2] <= r[k, 2] + 1, (level, k, m[k, 2], r[k, 2])
    assert r[:, 2].mean() <= 1.5 * m[:, 2].mean()
    ctx.close()
