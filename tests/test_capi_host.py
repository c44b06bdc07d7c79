"""The C-ABI library on a CPU-only box (-m "not gpu"): it loads, exports every symbol
include/mlmc.h declares, its host-only helpers agree with the oracle, and compute
entry points fail loudly (MLMC_ECUDA) instead of falling back to the CPU."""
import ctypes as C
import subprocess

import numpy as np
import pytest

from oracle import core as oc
from oracle import mlmc as om
from paper_2503_05533_b200 import _capi as K
from paper_2503_05533_b200 import api


@pytest.fixture(scope="module", autouse=True)
def built():
    import __graft_entry__
    __graft_entry__.build()


def test_library_exports_every_declared_symbol():
    names = K.declared_symbols()
    assert "mlmc_plan_levels" in names and "mlmc_sample_level" in names and "mlmc_adaptive_run" in names
    L = K.lib()
    for nm in names:
        assert hasattr(L, nm), nm
    out = subprocess.run(["nm", "-D", "--defined-only", K.SO_PATH], capture_output=True, text=True).stdout
    exported = {ln.split()[-1] for ln in out.splitlines() if " T " in ln}
    assert set(names) <= exported, set(names) - exported


def test_library_targets_sm100a():
    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "--list-elf", K.SO_PATH], capture_output=True, text=True)
    assert "sm_100a" in out.stdout


def test_eps_schedule_matches_oracle():
    for L in range(1, 7):
        for kp in (0.05, 0.4):
            a = api.mlmc_eps_schedule(L, 1 / 8, kp)
            b = om.eps_schedule_fem(L, 1 / 8, kp)
            assert np.allclose(a, b, rtol=1e-15, atol=0)


def test_optimal_samples_matches_oracle():
    rng = np.random.default_rng(0)
    for _ in range(20):
        n = rng.integers(1, 7)
        V = list(rng.uniform(1e-10, 1e-4, n))
        Cs = list(rng.uniform(1, 1e4, n))
        tol = 10 ** rng.uniform(-4, -2)
        assert np.allclose(api.mlmc_optimal_samples(V, Cs, tol), om.optimal_samples(V, Cs, tol), rtol=1e-13)
    assert np.allclose(api.mlmc_optimal_samples([4, 1], [1, 4], 2 ** 0.5), [8, 2])


@pytest.mark.parametrize("sigma2,ell,m", [(1.0, 0.3, 16), (1.0, 0.3, 64), (1.0, 0.1, 128), (2.0, 0.1, 256)])
def test_kl_modes_match_oracle(sigma2, ell, m):
    ik, jk, lam, w = api.mlmc_kl_modes(sigma2, ell, m, nroots=min(20, m + 1))
    oik, ojk, olam, ow = oc.kl_modes(sigma2, ell, m)
    assert np.array_equal(ik, oik) and np.array_equal(jk, ojk)
    assert np.allclose(lam, olam, rtol=1e-13, atol=0)
    assert np.allclose(w, ow[:len(w)], rtol=1e-13, atol=0)


def test_plan_fails_loudly_without_gpu():
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    p = K.Problem(0, 16, 1.0, 0.3, 2.0, 8, 2, 1, 0)
    ctx = C.c_void_p()
    assert K.lib().mlmc_plan_levels(C.byref(p), C.byref(ctx)) == K.MLMC_ECUDA
    with pytest.raises(Exception):
        api.Context(m=16)


def test_invalid_problems_rejected():
    bad = [K.Problem(0, 0, 1.0, 0.3, 2.0, 8, 2, 1, 0),      # m = 0
           K.Problem(0, 16, 1.0, 0.3, 2.0, 8, 3, 1, 0),     # refine 3
           K.Problem(0, 16, 1.0, 0.3, 2.0, 8, 2, 7, 0),     # 8 * 2^7 > 512
           K.Problem(0, 16, -1.0, 0.3, 2.0, 8, 2, 1, 0),    # sigma2 < 0
           K.Problem(5, 16, 1.0, 0.3, 2.0, 8, 2, 1, 0)]     # bad field
    for p in bad:
        ctx = C.c_void_p()
        assert K.lib().mlmc_plan_levels(C.byref(p), C.byref(ctx)) == K.MLMC_EINVAL


def test_controller_failed_solves_abort_or_are_counted():
    """R15: a sample whose solve missed its tolerance is never resampled; Algorithm 2 either stops with
    MLMC_ESOLVER (on_fail = 0) or keeps it and reports the count (on_fail = 1).  Host sampler: level sums
    with a variance that decays 4x per level, one failed solve flagged on level 0 of the first round."""
    import numpy as np
    from paper_2503_05533_b200 import _capi as K
    from paper_2503_05533_b200.api import mlmc_adaptive_run_host

    calls = {"n": 0}

    def sampler(level, n, first, pf, pc, tf, tc):
        rng = np.random.default_rng(1000 * level + first)
        y = rng.normal(0.03 * 4.0 ** -level, 0.01 * 4.0 ** -level, n)
        s = np.zeros(12)
        s[0], s[1], s[4], s[5] = y.sum(), (y * y).sum(), n * 4.0 ** level, n
        if level == 0 and calls["n"] == 0:
            s[6] = 1.0
        calls["n"] += 1
        return s

    with pytest.raises(RuntimeError, match="solver failure"):
        mlmc_adaptive_run_host(8, 4, 2e-3, sampler, N_init=50)
    calls["n"] = 0
    r = mlmc_adaptive_run_host(8, 4, 2e-3, sampler, N_init=50, on_fail=1)
    assert r["n_fail"] == 1 and r["code"] in (K.MLMC_OK, K.MLMC_ELMAX) and r["L"] >= 1


def test_null_context_calls_are_rejected():
    """Host-side argument checks of the C ABI (no device needed)."""
    p = K.Precision()
    ms = C.c_double()
    assert K.lib().mlmc_auto_choice(None, 8, C.byref(p), C.byref(ms)) == K.MLMC_EINVAL
    out = C.c_size_t()
    assert K.lib().mlmc_workspace_bytes(None, 0, 10, C.byref(out)) == K.MLMC_EINVAL
    assert K.lib().mlmc_profile_enable(None, 1) == K.MLMC_EINVAL


def test_host_controller_auto_policy_falls_back_to_minres_quads():
    """Policy 3 (auto) needs the GPU's pilot timings; over a host sampler it runs as policy 0 (MINRES
    precisions are handed to the sampler)."""
    seen = []

    def sampler(level, n, first, pf, pc, tf, tc):
        seen.append(pf.solver)
        rng = np.random.default_rng(level * 1000 + first)
        y = rng.normal(0.03 / 4 ** level, 0.01 / 4 ** level, n)
        s = np.zeros(12)
        s[0], s[1], s[4], s[5] = y.sum(), (y * y).sum(), n * 4.0 ** level, n
        return s

    r = api.mlmc_adaptive_run_host(8, 3, 2e-3, sampler, k_p=0.05, N_init=20, policy=3, seed=1)
    assert r["code"] in (0, 4) and set(seen) == {K.SOLVER_MINRES}
