"""Two-sided pins of the oracle's Algorithm 1 precision emulation and of its MINRES
(-m "not gpu"; VERDICT r01 "What's weak #1").

* Algorithm 1: the factor (step 1) and the substitutions (steps 2
  and 7) are reproduced BIT FOR BIT by a banded Cholesky written here in
  NumPy float16 / float32 scalar arithmetic (IEEE binary16 / binary32 operations,
  each correctly rounded -- NumPy evaluates binary16 through binary32, and double
  rounding 24 -> 11 bits is innocuous because 24 >= 2*11 + 2).  That fixes the
  rounding of every operation, not only convergence.  The refinement step counts on
  the configs[2] field are held between lower and upper bounds from SURVEY SC-9
  (an independent numpy session: fp16 means 3.9 / 6.2 / 11.9 at h = 1/8, 1/16, 1/32,
  fp32 1 / 1 / 2), and a mutant oracle that keeps the factor in binary64 is shown
  to fail the lower bound.
* MINRES: MINRES is defined by residual optimality -- x_k minimises
  ||b - A x|| over the Krylov space K_k(A, b) (x0 = 0).  At every step k the
  oracle's true residual must equal that minimum, computed here by a dense least
  squares over an Arnoldi basis (full reorthogonalisation, numpy/LAPACK); and the
  oracle's stopping step at tol must be the first k where the minimum drops to
  tol ||b||.  This fixes the step count exactly (an off-by-one stop fails).
"""
import os
import re
import subprocess

import numpy as np
import pytest

from oracle import core as oc

C3 = dict(m=64, sigma2=1.0, corr_len=0.3, seed=2)   # configs[2] (BASELINE.json, workloads.C3)


def _c3_system(N, index, level=0, seed=C3["seed"], dense=False, P=None):
    P = P or oc.OracleProblem(0, C3["m"], C3["sigma2"], C3["corr_len"], 2.0, 8)
    xi = oc.normals(seed, level, index, C3["m"])
    return oc.assemble(N, P.field_triangles(N, xi), dense=dense)


# ----------------------------------------------------------------------------- NumPy IEEE re-implementation
def np_chol_band(AB, dt):
    """Band Cholesky in dtype dt arithmetic: L(i,j) = (A(i,j) - sum_k L(i,k)L(j,k)) / L(j,j),
    L(j,j) = sqrt(.), k ascending; every product, difference, quotient, root rounded to dt."""
    n, bwp1 = AB.shape
    bw = bwp1 - 1
    L = np.zeros((n, bwp1), dt)
    for j in range(n):
        for i in range(j, min(n, j + bw + 1)):
            s = dt(AB[i, i - j])
            for k in range(max(0, i - bw), j):
                s = dt(s - dt(L[i, i - k] * L[j, j - k]))
            if i == j:
                if not s > 0:
                    raise np.linalg.LinAlgError("pivot")
                L[j, 0] = dt(np.sqrt(s))
            else:
                L[i, i - j] = dt(s / L[j, 0])
    return L


def np_band_solve(L, rhs, dt):
    """L y = rhs then L^T x = y, in dt arithmetic (row-oriented, d ascending)."""
    n, bwp1 = L.shape
    bw = bwp1 - 1
    Lc = L.astype(dt)
    y = np.zeros(n, dt)
    x = np.zeros(n, dt)
    for i in range(n):
        s = dt(rhs[i])
        for d in range(1, min(bw, i) + 1):
            s = dt(s - dt(Lc[i, d] * y[i - d]))
        y[i] = dt(s / Lc[i, 0])
    for i in range(n - 1, -1, -1):
        s = y[i]
        for d in range(1, bw + 1):
            if i + d >= n:
                break
            s = dt(s - dt(Lc[i + d, d] * x[i + d]))
        x[i] = dt(s / Lc[i, 0])
    return x


DT = {"h": np.float16, "s": np.float32}


@pytest.mark.parametrize("fmt", ["h", "s"])
@pytest.mark.parametrize("N,index", [(4, 0), (4, 1), (8, 0), (8, 3), (8, 7)])
def test_rounded_factor_and_substitution_bit_exact(fmt, N, index):
    """Algorithm 1 steps 1, 2 in the oracle == IEEE dt arithmetic, every bit."""
    AB, _, b = _c3_system(N, index)
    with np.errstate(all="ignore"):
        Lref = np_chol_band(AB, DT[fmt])
    L, st = oc.chol_band_rounded(AB, fmt)
    assert st == 0
    assert np.array_equal(L, Lref.astype(np.float64)), np.max(np.abs(L - Lref))
    for sfmt in (("h", "s") if fmt == "h" else ("s",)):   # u_s at least as precise as u_f (every paper quad)
        x = oc.band_solve_rounded(L, b, sfmt)
        with np.errstate(all="ignore"):
            xref = np_band_solve(L, b, DT[sfmt])
        assert np.array_equal(x, xref.astype(np.float64))
    # a correction solve with a residual-like right-hand side (step 7)
    r = np.random.default_rng(N + index).normal(size=b.size) * 1e-6
    assert np.array_equal(oc.band_solve_rounded(L, r, "s"), np_band_solve(L, r, np.float32).astype(np.float64))


def test_rounded_factor_bit_exact_high_contrast_and_subnormal_range():
    """Large-contrast coefficients (sigma^2 = 4 field) and a tiny right-hand side whose
    fp16 substitution runs through the subnormal range."""
    P = oc.OracleProblem(0, 64, 4.0, 0.3, 2.0, 8)
    AB, _, b = _c3_system(8, 11, P=P)
    with np.errstate(all="ignore"):
        Lref = np_chol_band(AB, np.float16)
    L, st = oc.chol_band_rounded(AB, "h")
    assert st == 0 and np.array_equal(L, Lref.astype(np.float64))
    tiny = b * 1e-5                                       # ~1.6e-7: binary16 subnormals (< 6.1e-5)
    with np.errstate(all="ignore"):
        xr = np_band_solve(L, tiny, np.float16)
    assert np.array_equal(oc.band_solve_rounded(L, tiny, "h"), xr.astype(np.float64))
    assert np.any((np.abs(xr) < 6.1e-5) & (xr != 0))


def test_ir_loop_matches_numpy_algorithm1():
    """The whole of Algorithm 1 for quad hsdd: x0 by fp16-factor / fp32 substitution,
    binary64 residual and update, stop at ||r||/||b|| < tol -- same step count, same x to 1e-13."""
    for N, idx in ((8, 0), (8, 5), (16, 2)):
        AB, D, b = _c3_system(N, idx, dense=True)
        with np.errstate(all="ignore"):
            L = np_chol_band(AB, np.float16).astype(np.float64)
            x = np_band_solve(L, b, np.float32).astype(np.float64)
        steps = 0
        while True:
            r = b - D @ x
            if np.linalg.norm(r) / np.linalg.norm(b) < 1e-10:
                break
            with np.errstate(all="ignore"):
                x = x + np_band_solve(L, r, np.float32).astype(np.float64)
            steps += 1
        xo, so, rr, st = oc.ir_band(AB, b, "hsdd", 1e-10)
        assert st == 0 and so == steps, (N, idx, so, steps)
        assert np.allclose(xo, x, rtol=1e-13, atol=0)


# ----------------------------------------------------------------------------- SC-9 step-count window
def _mean_steps(N, quad, count, tol=1e-10):
    P = oc.OracleProblem(0, C3["m"], C3["sigma2"], C3["corr_len"], 2.0, 8)
    steps = []
    for k in range(count):
        AB, _, b = _c3_system(N, k, P=P)
        _, s, _, st = oc.ir_band(AB, b, quad, tol)
        assert st == 0
        steps.append(s)
    return float(np.mean(steps)), steps


@pytest.mark.parametrize("N,count,lo,hi", [(8, 24, 3.0, 5.0), (16, 12, 4.5, 8.0), (32, 6, 9.0, 15.0)])
def test_fp16_factor_step_counts_bounded_both_sides(N, count, lo, hi):
    """SC-9: fp16 factor + fp32 substitution to 1e-10 needs 3.9 / 6.2 / 11.9 steps on average
    (max 19).  Lower AND upper bounds: a factor computed in a wider format converges in 1-2."""
    mean, steps = _mean_steps(N, "hsdd", count)
    assert lo <= mean <= hi, (mean, steps)
    assert max(steps) <= 19 + 4


@pytest.mark.parametrize("N,count,hi", [(8, 12, 1.5), (16, 8, 1.5), (32, 4, 2.5)])
def test_fp32_factor_step_counts_bounded_both_sides(N, count, hi):
    """SC-9: fp32 factor needs 1 / 1 / 2 steps; never 0 (x0 from a binary32 factor is not 1e-10 accurate)."""
    mean, steps = _mean_steps(N, "ssdd", count)
    assert min(steps) >= 1 and mean <= hi, steps


def test_mutant_binary64_factor_fails_the_lower_bound(tmp_path):
    """Mutation check: an oracle whose step 1 silently keeps the factor in binary64 (u_f rounding
    dropped) must fail the fp16 lower bound above -- so the pin is two-sided, not decorative."""
    src = open(os.path.join(os.path.dirname(oc.__file__), "oracle.c")).read()
    mut, n = re.subn(r"(OR_EXPORT int or_chol_band_rounded\(int n, int bw, const double\* AB, double\* L, int )ff\) \{",
                     r"\1ff_unused) { int ff = 3;", src)
    assert n == 1
    (tmp_path / "mut.c").write_text(mut)
    so = str(tmp_path / "libmut.so")
    subprocess.check_call(["gcc", "-O2", "-std=c11", "-shared", "-fPIC", "-o", so, str(tmp_path / "mut.c"), "-lm"])
    import ctypes as C
    lib = C.CDLL(so)
    dp = np.ctypeslib.ndpointer(dtype=np.float64, flags="C_CONTIGUOUS")
    ip = np.ctypeslib.ndpointer(dtype=np.int32, flags="C_CONTIGUOUS")
    lib.or_ir_band.argtypes = [C.c_int, C.c_int, dp, dp, ip, C.c_double, C.c_int, dp,
                               C.POINTER(C.c_int), C.POINTER(C.c_double)]
    P = oc.OracleProblem(0, C3["m"], C3["sigma2"], C3["corr_len"], 2.0, 8)
    steps = []
    for k in range(24):
        AB, _, b = _c3_system(8, k, P=P)
        x = np.zeros(b.size)
        it, rr = C.c_int(), C.c_double()
        st = lib.or_ir_band(49, 7, np.ascontiguousarray(AB).ravel(), b, np.array([1, 2, 3, 3], np.int32),
                            1e-10, 50, x, C.byref(it), C.byref(rr))
        assert st == 0
        steps.append(it.value)
    assert np.mean(steps) < 3.0          # the mutant is caught by test_fp16_factor_step_counts_bounded_both_sides


# ----------------------------------------------------------------------------- MINRES residual optimality
def _krylov_min_residuals(A, b, kmax):
    """min_{x in K_k(A,b)} ||b - A x|| for k = 1..kmax via an Arnoldi basis with full
    reorthogonalisation (twice-iterated Gram-Schmidt) and numpy lstsq."""
    n = b.size
    V = np.zeros((n, kmax))
    v = b / np.linalg.norm(b)
    out = []
    for k in range(kmax):
        V[:, k] = v
        Vk = V[:, :k + 1]
        y, *_ = np.linalg.lstsq(A @ Vk, b, rcond=None)
        out.append(np.linalg.norm(b - A @ (Vk @ y)))
        w = A @ v
        for _ in range(2):
            w = w - Vk @ (Vk.T @ w)
        nw = np.linalg.norm(w)
        if nw < 1e-14 * np.linalg.norm(A @ v):
            break
        v = w / nw
    return np.array(out)


@pytest.mark.parametrize("N,index,sigma2,m", [(4, 0, 1.0, 16), (4, 2, 4.0, 16), (8, 0, 1.0, 16), (8, 9, 4.0, 16),
                                              (16, 3, 1.0, 64)])
def test_minres_residual_is_krylov_minimum_at_every_step(N, index, sigma2, m):
    """P:100-102 (MINRES): ||b - A x_k|| = min over x0 + K_k(A, b), x0 = 0, at every step k, to 1e-10
    relative while the minimum is >= 1e-3 ||b|| (binary64 Lanczos still orthogonal: Paige's analysis,
    P:104 -- later, lost orthogonality only delays convergence); and never below the minimum."""
    P = oc.OracleProblem(0, m, sigma2, 0.3, 2.0, 8)
    xi = oc.normals(0, 0, index, m)
    AB, D, b = oc.assemble(N, P.field_triangles(N, xi), dense=True)
    ref = _krylov_min_residuals(D, b, min(b.size, 60))
    bn = np.linalg.norm(b)
    checked = 0
    for k in range(1, len(ref) + 1):
        if ref[k - 1] < 1e-6 * bn:
            break
        x, it, _, st = oc.minres_band(AB, b, 0.0, max_iter=k)
        assert it == k
        res = np.linalg.norm(b - D @ x)
        assert res >= ref[k - 1] * (1 - 1e-9), (k, res, ref[k - 1])      # optimality cannot be beaten
        if ref[k - 1] >= 1e-3 * bn or b.size <= 9:
            assert abs(res - ref[k - 1]) <= 1e-10 * ref[k - 1], (k, res, ref[k - 1])
            checked += 1
    assert checked >= min(b.size - 1, 8)


@pytest.mark.parametrize("N,index,sigma2", [(8, 1, 1.0), (8, 6, 4.0), (16, 3, 1.0), (32, 0, 1.0)])
def test_minres_stopping_step_is_first_step_meeting_eq2(N, index, sigma2):
    """Eq. (2) with C = 1: the oracle stops at the FIRST k whose iterate x_k has
    relative residual <= tol -- x_{k-1} (run with max_iter = k-1) does not meet it, x_k does (up
    to the gap between the recurrence phibar_k and the true residual, ~1e-6 relative here; steps
    that sit that close to tol are skipped).  An off-by-one stop fails this."""
    P = oc.OracleProblem(0, 64, sigma2, 0.3, 2.0, 8)
    xi = oc.normals(1, 0, index, 64)
    AB, D, b = oc.assemble(N, P.field_triangles(N, xi), dense=(N <= 16))
    bn = np.linalg.norm(b)

    def true_rel(x):
        return np.linalg.norm(b - oc.band_matvec(AB, x)) / bn

    checked = 0
    for tol in (1e-2, 1e-3, 1e-4, 1e-6, 1e-8):
        x, it, rr, st = oc.minres_band(AB, b, tol)
        assert st == 0 and it >= 1
        xp, itp, _, _ = oc.minres_band(AB, b, 0.0, max_iter=it - 1) if it > 1 else (np.zeros_like(b), 0, 1, 0)
        r_k, r_km1 = true_rel(x), true_rel(xp)
        if abs(r_k / tol - 1) < 1e-5 or abs(r_km1 / tol - 1) < 1e-5:
            continue
        assert r_k <= tol and r_km1 > tol, (tol, it, r_k, r_km1)
        checked += 1
    assert checked >= 4
