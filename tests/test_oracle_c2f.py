"""Pins of the oracle's coarse-to-fine MINRES (oracle/c2f.py, or_minres_band_x0; NEXT-4, R32),
-m "not gpu".  Each pin fixes something other than the code itself: x0 = 0 reduces to the pinned textbook
MINRES bit for bit; x0 = the exact solution needs no step; residual optimality over x0 + K_k(A, r0) at every
step (dense least squares over an Arnoldi basis of r0); the stop is the first step meeting Eq. (2) relative
to ||b||; the prolongated coarse solution is the coarse P1 function (closed-form hats, as in test_oracle_mg);
the fine Q is within the rigorous bound tol ||b|| ||x|| of the direct solve."""
import numpy as np
import pytest

from oracle import c2f
from oracle import core as oc
from oracle import mg

from test_oracle_alg1_minres import _krylov_min_residuals


def _system(N, index, m=16, sigma2=1.0, seed=0):
    P = oc.OracleProblem(0, m, sigma2, 0.3, 2.0, 8)
    xi = oc.normals(seed, 0, index, m)
    return oc.assemble(N, P.field_triangles(N, xi), dense=True)


@pytest.mark.parametrize("N,index", [(8, 0), (16, 3)])
def test_x0_zero_is_textbook_minres_bit_for_bit(N, index):
    AB, _, b = _system(N, index)
    for tol in (1e-3, 1e-8):
        x, it, rr, st = oc.minres_band(AB, b, tol)
        y, it2, rr2, st2 = oc.minres_band_x0(AB, b, np.zeros_like(b), tol)
        assert it == it2 and st == st2 and np.array_equal(x, y)


def test_exact_initial_guess_needs_no_step_and_stop_is_relative_to_b():
    AB, D, b = _system(8, 1)
    x = np.linalg.solve(D, b)
    y, it, rr, st = oc.minres_band_x0(AB, b, x, 1e-10)
    assert st == 0 and it == 0 and np.array_equal(y, x)
    # a guess whose residual is 1e-3 ||b||: tol 1e-2 (relative to ||b||) needs no step, 1e-4 needs some
    rng = np.random.default_rng(0)
    e = rng.normal(size=b.size)
    e *= 1e-3 * np.linalg.norm(b) / np.linalg.norm(D @ e)
    _, it1, _, _ = oc.minres_band_x0(AB, b, x + e, 1e-2)
    _, it2, rr2, _ = oc.minres_band_x0(AB, b, x + e, 1e-4)
    assert it1 == 0 and it2 >= 1 and rr2 <= 1e-4 * (1 + 1e-6)


@pytest.mark.parametrize("N,index", [(8, 2), (16, 4)])
def test_residual_is_minimum_over_x0_plus_krylov_space(N, index):
    """||b - A x_k|| = min over x0 + K_k(A, r0) while the minimum is >= 1e-3 ||r0|| (orthogonal Lanczos)."""
    AB, D, b = _system(N, index)
    x0 = np.random.default_rng(N).normal(size=b.size) * 0.01
    r0 = b - D @ x0
    ref = _krylov_min_residuals(D, r0, min(b.size, 40))
    checked = 0
    for k in range(1, len(ref) + 1):
        if ref[k - 1] < 1e-3 * np.linalg.norm(r0):
            break
        x, it, _, _ = oc.minres_band_x0(AB, b, x0, 0.0, max_iter=k)
        res = np.linalg.norm(b - D @ x)
        assert it == k and abs(res - ref[k - 1]) <= 1e-10 * ref[k - 1], (k, res, ref[k - 1])
        checked += 1
    assert checked >= 6


def test_prolongation_reproduces_coarse_p1_function():
    """P x_c evaluated at the fine nodes equals the coarse P1 function: for x_c sampled from a linear function
    (exact in P1), P x_c is that linear function at the fine interior nodes (Dirichlet nodes excluded, so the
    function is built to vanish on the boundary lines it touches: use the hat-sum identity instead)."""
    N = 16
    Nc = N // 2
    rng = np.random.default_rng(5)
    xc = rng.normal(size=(Nc - 1) ** 2)

    def coarse_p1(x, y):        # evaluate the coarse P1 function with values xc at (x, y) by barycentric weights
        H = 1.0 / Nc
        I, J = min(int(x / H), Nc - 1), min(int(y / H), Nc - 1)
        u, v = x / H - I, y / H - J
        val = lambda i, j: 0.0 if (i <= 0 or j <= 0 or i >= Nc or j >= Nc) else xc[(j - 1) * (Nc - 1) + (i - 1)]
        if v <= u:   # lower triangle (I,J),(I+1,J),(I+1,J+1)
            return (1 - u) * val(I, J) + (u - v) * val(I + 1, J) + v * val(I + 1, J + 1)
        return (1 - v) * val(I, J) + (v - u) * val(I, J + 1) + u * val(I + 1, J + 1)
    x0 = mg.prolongation(N) @ xc
    for j in range(1, N):
        for i in range(1, N):
            assert abs(x0[(j - 1) * (N - 1) + (i - 1)] - coarse_p1(i / N, j / N)) < 1e-14


@pytest.mark.parametrize("level,tol_f,tol_c", [(1, 1e-6, 1e-5), (2, 1e-8, 1e-6)])
def test_c2f_sample_within_bound_of_direct_solve(level, tol_f, tol_c):
    P = oc.OracleProblem(0, 64, 1.0, 0.3, 2.0, 8)
    for idx in range(3):
        r = c2f.coupled_sample_c2f(P, level, 1, idx, tol_f, tol_c)
        AB, b = r["AB"], r["b"]
        x, _ = oc.chol_band_solve(AB, b)
        N = 8 << level
        q = x.sum() / N ** 2
        assert r["status_f"] == 0 and r["relres_f"] <= tol_f * (1 + 1e-6)
        assert abs(r["Qf"] - q) <= tol_f * np.linalg.norm(b) * np.linalg.norm(x) * (1 + 1e-6) + 1e-14 * q
        # the interpolated coarse solution carries interpolation (high-frequency) error, so its residual is
        # LARGER than ||b|| (1.7-2.7x here), but those components are cheap for MINRES: from level 2 on the
        # fine half needs fewer steps than from 0 (measured 15-20% at h = 1/32, 1/64)
        r0 = b - oc.band_matvec(AB, r["x0"])
        assert np.linalg.norm(r0) > np.linalg.norm(b)
        if level >= 2:
            _, it0, _, _ = oc.minres_band(AB, b, tol_f)
            assert r["iters_f"] < it0
