"""Pins of the CPU oracle against things other than itself (-m "not gpu").

Each test names what fixes the expected value: a published KAT, the paper's
printed numbers (P:n = /root/reference/PAPER.md line n), a closed form, an
invariant, or a brute-force / library computation on a different code path.
"""
import math
import os

import numpy as np
import pytest
from scipy import integrate, stats

from oracle import core as oc
from oracle import mlmc as om

GOLDEN = os.path.join(os.path.dirname(__file__), "golden")


# ============================================================================ RNG
def test_philox_kat_vectors():
    """Philox4x32-10 known-answer vectors (Salmon et al., Random123 KAT file)."""
    assert list(oc.philox([0, 0, 0, 0], [0, 0])) == [0x6627E8D5, 0xE169C58D, 0xBC57AC4C, 0x9B00DBD8]
    assert list(oc.philox([0xFFFFFFFF] * 4, [0xFFFFFFFF] * 2)) == [0x408F276D, 0x41C83B0E, 0xA20BC7C6, 0x6D5451FD]
    assert list(oc.philox([0x243F6A88, 0x85A308D3, 0x13198A2E, 0x03707344], [0xA4093822, 0x299F31D0])) == \
        [0xD16CFE09, 0x94FDCCEB, 0x5001E420, 0x24126EA1]


def test_normals_are_standard_normal():
    """omega_j ~ N(0, sigma^2): KS test + moments on 40k draws."""
    xs = np.concatenate([oc.normals(7, 2, k, 64) for k in range(625)])
    assert abs(xs.mean()) < 0.02 and abs(xs.var() - 1.0) < 0.03
    assert stats.kstest(xs, "norm").pvalue > 1e-3
    # counter structure: different level / index / seed give different streams
    a, b, c, d = (oc.normals(0, 0, 0, 8), oc.normals(0, 1, 0, 8), oc.normals(0, 0, 1, 8), oc.normals(1, 0, 0, 8))
    assert not np.allclose(a, b) and not np.allclose(a, c) and not np.allclose(a, d)
    # prefix property: the first m draws do not depend on m
    assert np.array_equal(oc.normals(3, 1, 5, 16), oc.normals(3, 1, 5, 64)[:16])


# ============================================================================ KL (BASELINE field, R11)
@pytest.mark.parametrize("ell", [0.3, 0.1])
def test_kl_1d_roots_interlace_and_solve(ell):
    c = 1.0 / ell
    w = oc.kl_roots(ell, 30)
    for k, wk in enumerate(w, start=1):
        assert (k - 1) * math.pi < wk < k * math.pi            # one root per ((k-1)pi, k pi)
        f = (wk * wk - c * c) * math.sin(wk) - 2 * c * wk * math.cos(wk)
        assert abs(f) < 1e-10 * (wk * wk + c * c)


@pytest.mark.parametrize("ell", [0.3, 0.1])
def test_kl_1d_eigen_relation_by_quadrature(ell):
    """theta_k e_k(x) = int_0^1 exp(-|x-y|/l) e_k(y) dy and int e_k e_j = delta_kj
    (adaptive quadrature, split at the kink y = x)."""
    c = 1.0 / ell
    w = oc.kl_roots(ell, 6)
    for k in range(6):
        th = oc.kl_theta(ell, w[k])
        for x in (0.0, 0.137, 0.5, 0.93, 1.0):
            f = lambda y: math.exp(-c * abs(x - y)) * oc.kl_efun(ell, w[k], y)
            lhs = integrate.quad(f, 0, x, epsabs=1e-13, epsrel=1e-13)[0] + \
                integrate.quad(f, x, 1, epsabs=1e-13, epsrel=1e-13)[0]
            assert abs(lhs - th * oc.kl_efun(ell, w[k], x)) < 1e-10
        for j in range(6):
            g = integrate.quad(lambda y: oc.kl_efun(ell, w[k], y) * oc.kl_efun(ell, w[j], y), 0, 1,
                               epsabs=1e-13, epsrel=1e-13, limit=200)[0]
            assert abs(g - (1.0 if j == k else 0.0)) < 1e-10
        assert oc.kl_efun(ell, w[k], 0.0) > 0                   # sign convention e_k(0) = N_k > 0


def test_kl_1d_trace_and_printed_values():
    """Mercer trace: sum_k theta_k = int_0^1 C(x,x) dx = 1 (remaining tail ~ 2c/(pi^2 K))."""
    ell = 0.3
    c = 1 / ell
    w = oc.kl_roots(ell, 3000)
    th = np.array([oc.kl_theta(ell, x) for x in w])
    tail = sum(2 * c / ((k * math.pi) ** 2) for k in range(3001, 400000))
    assert abs(th.sum() + tail - 1.0) < 2e-5
    assert np.all(np.diff(th) < 0)
    # regression hints (SURVEY SC-5, independent scipy/Nystrom session): theta_1..3, w_1, N_1
    assert np.allclose(th[:3], [0.436249, 0.216812, 0.106997], atol=1e-6)
    assert abs(w[0] - 2.0422278101) < 1e-9
    assert abs(oc.kl_norm(ell, w[0]) - 0.6164772242) < 1e-9


def test_kl_2d_modes_ties_and_variance_fraction():
    ik, jk, lam, w1d = oc.kl_modes(1.0, 0.3, 16)
    th = [oc.kl_theta(0.3, x) for x in w1d]
    for k in range(16):
        assert lam[k] == 1.0 * (th[ik[k] - 1] * th[jk[k] - 1])
    assert np.all(np.diff(lam) <= 0)
    assert lam[1] == lam[2] and (ik[1], jk[1]) == (1, 2) and (ik[2], jk[2]) == (2, 1)   # exact tie, R11 order
    assert (ik[15], jk[15]) == (1, 6)                            # its tie partner (6,1) is cut off
    assert np.allclose(lam[:4], [0.190312864, 0.094584119, 0.094584119, 0.047007624], atol=1e-9)
    # captured variance fraction sum(lam)/(sigma^2 |D|) (trace of the 2D kernel = sigma^2 |D| = 1)
    assert abs(lam.sum() - 0.698) < 1e-3
    _, _, lam256, _ = oc.kl_modes(2.0, 0.1, 256)
    assert abs(lam256.sum() / 2.0 - 0.796) < 1e-3


# ============================================================================ assembly (R10)
def _laplacian_5pt(N):
    n = (N - 1) ** 2
    A = np.zeros((n, n))
    for j in range(1, N):
        for i in range(1, N):
            p = (j - 1) * (N - 1) + i - 1
            A[p, p] = 4
            for di, dj in ((1, 0), (-1, 0), (0, 1), (0, -1)):
                if 1 <= i + di < N and 1 <= j + dj < N:
                    A[p, (j + dj - 1) * (N - 1) + i + di - 1] = -1
    return A


def test_assembly_constant_coefficient_is_5pt_laplacian():
    for N in (2, 3, 4, 8, 16):
        _, D, b = oc.assemble(N, np.ones(2 * N * N), dense=True)
        assert np.array_equal(D, _laplacian_5pt(N))
        assert np.allclose(b, (1.0 / N) ** 2, rtol=1e-15, atol=0)     # b_i = int phi_i = h^2
    _, D, b = oc.assemble(2, np.ones(8), dense=True)
    assert D.tolist() == [[4.0]] and abs(b[0] - 0.25) < 1e-16
    P = oc.OracleProblem(0, 16, 1.0, 0.3, 2.0, 8)
    assert abs(P.solve_mesh(2, np.zeros(16), oc.SOLVER_DIRECT)["Q"] - 1 / 64) < 1e-17


def test_assembly_random_coefficient_equals_conductance_form():
    """P1 on the SW-NE triangulation = 5-point stencil with edge conductance the
    mean of the two triangles sharing the edge (derived by hand; the oracle
    assembles element by element)."""
    rng = np.random.default_rng(0)
    for N in (3, 4, 7):
        a = np.exp(rng.normal(size=2 * N * N))
        AB, D, b = oc.assemble(N, a, dense=True)
        aL = lambda i, j: a[2 * (j * N + i)]
        aU = lambda i, j: a[2 * (j * N + i) + 1]
        n = (N - 1) ** 2
        E = np.zeros((n, n))
        idx = lambda i, j: (j - 1) * (N - 1) + i - 1 if (0 < i < N and 0 < j < N) else -1
        for j in range(1, N):
            for i in range(1, N):
                p = idx(i, j)
                cE = 0.5 * (aL(i, j) + aU(i, j - 1))
                cW = 0.5 * (aL(i - 1, j) + aU(i - 1, j - 1))
                cN = 0.5 * (aU(i, j) + aL(i - 1, j))
                cS = 0.5 * (aU(i, j - 1) + aL(i - 1, j - 1))
                E[p, p] = cE + cW + cN + cS
                for q, cc in ((idx(i + 1, j), cE), (idx(i - 1, j), cW), (idx(i, j + 1), cN), (idx(i, j - 1), cS)):
                    if q >= 0:
                        E[p, q] = -cc
        assert np.max(np.abs(D - E)) < 1e-14 * np.max(np.abs(E))
        assert np.array_equal(D, D.T)
        assert np.all(np.linalg.eigvalsh(D) > 0)
        # band storage agrees with the dense matrix
        bw = N - 1
        for p in range(n):
            for d in range(bw + 1):
                if p - d >= 0:
                    assert AB[p, d] == D[p, p - d]


def _exact_poisson_qoi(terms=4001):
    """int_D u for -Lap u = 1 on the unit square, u = 0 on the boundary:
    sum over odd j,k of 64 / (pi^6 j^2 k^2 (j^2 + k^2))."""
    j = np.arange(1, terms, 2, dtype=np.float64)
    J, K = np.meshgrid(j, j)
    return float(np.sum(64.0 / (math.pi ** 6 * J ** 2 * K ** 2 * (J ** 2 + K ** 2))))


def test_discretisation_error_is_O_h2_against_fourier_series():
    exact = _exact_poisson_qoi()
    assert abs(exact - 0.0351442537) < 1e-10
    P = oc.OracleProblem(0, 16, 1.0, 0.3, 2.0, 8)
    Q = [P.solve_mesh(N, np.zeros(16), oc.SOLVER_DIRECT)["Q"] for N in (8, 16, 32, 64)]
    err = [exact - q for q in Q]
    assert all(e > 0 for e in err)
    ratios = [err[i] / err[i + 1] for i in range(3)]
    assert all(3.8 < r < 4.1 for r in ratios), ratios
    assert np.allclose(Q, [0.033423031078, 0.034702752314, 0.035033019542, 0.035116381629], atol=2e-12)


def test_manufactured_solution_O_h2():
    """a == 1, u = sin(pi x) sin(pi y), f = 2 pi^2 u: nodal max error and |Q_h - 4/pi^2|
    fall ~4x per halving of h; a == c scales the discrete solution by exactly 1/c."""
    errs, qerrs = [], []
    for N in (8, 16, 32, 64):
        AB, _, b = oc.assemble(N, np.ones(2 * N * N), f_kind=1)
        x, _ = oc.chol_band_solve(AB, b)
        h = 1.0 / N
        g = np.arange(1, N) * h
        X, Y = np.meshgrid(g, g)
        u = (np.sin(math.pi * X) * np.sin(math.pi * Y)).ravel()
        errs.append(np.max(np.abs(x - u)))
        qerrs.append(abs(h * h * x.sum() - 4 / math.pi ** 2))
        AB3, _, b3 = oc.assemble(N, 3.0 * np.ones(2 * N * N), f_kind=1)
        x3, _ = oc.chol_band_solve(AB3, b3)
        assert np.allclose(x3 * 3.0, x, rtol=1e-12, atol=0)
    for e in (errs, qerrs):
        r = [e[i] / e[i + 1] for i in range(3)]
        assert all(3.5 < v < 4.5 for v in r), r


def test_condition_number_closed_form_and_slope():
    """kappa_2(A(0)) = (4 - 2cos(pi h(N-1)) ... ) closed form of the 5-point Laplacian;
    Lemma 3.2: kappa_2 <= c h^-2 -> log-log slope ~2."""
    ks = []
    for N in (8, 16, 32):
        _, D, _ = oc.assemble(N, np.ones(2 * N * N), dense=True)
        ev = np.linalg.eigvalsh(D)
        h = 1.0 / N
        lmin = 8 * math.sin(math.pi * h / 2) ** 2
        lmax = 8 * math.cos(math.pi * h / 2) ** 2
        assert abs(ev[0] - lmin) < 1e-12 and abs(ev[-1] - lmax) < 1e-12
        ks.append(ev[-1] / ev[0])
    assert np.allclose(ks, [25.27, 103.09, 414.35], atol=0.01)
    slope = np.polyfit(np.log([1 / 8, 1 / 16, 1 / 32]), np.log(ks), 1)[0]
    assert -2.1 < slope < -1.9


# ============================================================================ solvers
def _random_system(N, seed=0, ell=0.3, m=16):
    P = oc.OracleProblem(0, m, 1.0, ell, 2.0, 8)
    xi = oc.normals(seed, 0, 0, m)
    a = P.field_triangles(N, xi)
    return oc.assemble(N, a, dense=True)


@pytest.mark.parametrize("N", [4, 8, 16])
def test_direct_solvers_agree_with_lapack(N):
    AB, D, b = _random_system(N, seed=N)
    xb, _ = oc.chol_band_solve(AB, b)
    xd, Ld = oc.chol_dense_solve(D, b)
    ref = np.linalg.solve(D, b)
    assert np.allclose(xb, ref, rtol=1e-12, atol=0)
    assert np.allclose(xd, ref, rtol=1e-12, atol=0)
    assert np.allclose(Ld @ Ld.T, D, rtol=0, atol=1e-13 * np.abs(D).max())
    assert np.max(np.abs(oc.band_matvec(AB, ref) - D @ ref)) < 1e-14 * np.abs(D).max() * np.abs(ref).max()


def test_minres_special_cases():
    AB = np.zeros((5, 2)); AB[:, 0] = 1.0
    b = np.arange(1.0, 6.0)
    x, it, rr, st = oc.minres_band(AB, b, 1e-6)
    assert st == 0 and it == 1 and np.allclose(x, b, rtol=1e-15)
    AB = np.array([[1.0, 0.0], [2.0, 0.0]])
    x, it, rr, st = oc.minres_band(AB, np.array([1.0, 2.0]), 1e-12)
    assert st == 0 and it <= 2 and np.allclose(x, [1, 1], rtol=1e-12)


@pytest.mark.parametrize("N", [8, 16])
def test_minres_relative_residual_criterion(N):
    """Eq. (2) with C = 1: the true relative residual meets tol;
    iteration count monotone in tol; at tol 1e-12 Q matches the direct solve to 1e-10."""
    AB, D, b = _random_system(N, seed=3)
    ref = np.linalg.solve(D, b)
    prev = 0
    for tol in (3.5e-3, 1e-4, 1e-6, 1e-8, 1e-12):
        x, it, rr, st = oc.minres_band(AB, b, tol)
        assert st == 0
        true_rr = np.linalg.norm(b - D @ x) / np.linalg.norm(b)
        assert abs(true_rr - rr) < 1e-14 and true_rr <= tol * (1 + 1e-6)
        assert it >= prev
        prev = it
        # per-sample QoI bound (w = b, A SPD): |Q(x) - Q(x*)| = |x*^T r| <= ||x*|| ||r||
        h2 = 1.0 / N ** 2
        assert abs(h2 * (x.sum() - ref.sum())) <= np.linalg.norm(ref) * np.linalg.norm(b - D @ x) * (1 + 1e-8) + 1e-18
    assert abs(x.sum() - ref.sum()) / ref.sum() < 1e-10


def test_minres_true_residual_nonincreasing_on_random_spd():
    rng = np.random.default_rng(1)
    for trial in range(20):
        n, bw = 30, 3
        M = rng.normal(size=(n, n))
        D = M @ M.T + n * np.eye(n)
        D = np.tril(np.triu(D, -bw), bw)        # banded SPD (diag dominant)
        D = D + np.eye(n) * np.abs(D).sum(1).max()
        AB = np.zeros((n, bw + 1))
        for i in range(n):
            for d in range(bw + 1):
                if i - d >= 0:
                    AB[i, d] = D[i, i - d]
        b = rng.normal(size=n)
        last = np.inf
        for k in range(1, 12):
            x, it, rr, st = oc.minres_band(AB, b, 0.0, max_iter=k)
            assert rr <= last * (1 + 1e-12) + 1e-15
            last = rr
        x, it, rr, st = oc.minres_band(AB, b, 1e-12)
        assert np.allclose(x, np.linalg.solve(D, b), rtol=1e-9, atol=1e-12)


# ============================================================================ precision emulation
def test_round_matches_ieee_conversions():
    rng = np.random.default_rng(2)
    xs = np.concatenate([rng.normal(size=20000) * 10.0 ** rng.integers(-9, 6, 20000),
                         [6.1e-5, 5.96e-8, 2.98e-8, 65504.0, 65519.0, 1 + 2 ** -11, 1 + 3 * 2 ** -11]])
    for x in xs:
        h = oc.round_to(x, "h")
        ref = float(np.float16(x))
        assert h == ref or (math.isinf(ref) and math.isinf(h)), (x, h, ref)
        assert oc.round_to(x, "s") == float(np.float32(x))
        assert oc.round_to(x, "d") == x
    assert math.isinf(oc.round_to(65520.0, "h"))


def test_round_standard_model_and_q43():
    """fl(x) = x(1+nu), |nu| <= u in the normal range; q43 u = 2^-4."""
    rng = np.random.default_rng(3)
    for fmt, u, lo, hi in (("h", 2 ** -11, 6.2e-5, 6e4), ("s", 2 ** -24, 1.2e-38, 1e38), ("q", 2 ** -4, 0.016, 240)):
        xs = np.exp(rng.uniform(math.log(lo), math.log(hi), 5000)) * rng.choice([-1, 1], 5000)
        r = np.array([oc.round_to(x, fmt) for x in xs])
        assert np.all(np.abs(r - xs) <= u * np.abs(xs))
        assert np.all(np.array([oc.round_to(v, fmt) for v in r]) == r)          # idempotent
        s = np.sort(xs)
        rs = np.array([oc.round_to(v, fmt) for v in s])
        assert np.all(np.diff(rs) >= 0)                                            # monotone
    assert oc.round_to(1.0 + 2 ** -5, "q") == 1.0
    assert oc.round_to(1.0 + 2 ** -4, "q") == 1.0        # tie -> even significand
    assert oc.round_to(1.0 + 3 * 2 ** -4, "q") == 1.25   # tie -> even
    assert oc.round_to(240.0, "q") == 240.0 and math.isinf(oc.round_to(250.0, "q"))


# ============================================================================ Algorithm 1
@pytest.mark.parametrize("N,quad,tol", [(8, "hhss", 3.49e-3), (16, "ssss", 8.7e-4), (32, "ssdd", 2.2e-4),
                                        (8, "hsdd", 1e-10), (16, "ssdd", 1e-10), (16, "hsdd", 1e-10)])
def test_ir_converges_to_tolerance(N, quad, tol):
    AB, D, b = _random_system(N, seed=5, m=64)
    x, steps, rr, st = oc.ir_band(AB, b, quad, tol)
    assert st == 0, (st, steps, rr)
    true_rr = np.linalg.norm(b - D @ x) / np.linalg.norm(b)
    assert true_rr <= tol * (1 + 1e-3)
    if quad[0] == "s" and tol == 1e-10:
        assert steps <= 3                     # SC-9: fp32 factor needs 1-2 steps
    if quad[0] == "h" and tol == 1e-10:
        assert steps <= 30


def test_ir_limiting_accuracy_and_monotone_steps():
    """Corollary 3.3: the residual stalls at ~u ||b||: hhss cannot reach 1e-12."""
    AB, D, b = _random_system(16, seed=6)
    x, steps, rr, st = oc.ir_band(AB, b, "hhss", 1e-12, i_max=50)
    assert st == 1 and steps == 50
    prev = -1
    for tol in (1e-2, 1e-4, 1e-6, 1e-8, 1e-10):
        _, s, _, st = oc.ir_band(AB, b, "hsdd", tol)
        assert st == 0 and s >= prev
        prev = s
    _, s, _, st = oc.ir_band(AB, b, "dddd", 1e-12)
    assert st == 0 and s <= 1


# ============================================================================ schedule / estimators / Algorithm 2
def _golden_table1():
    rows = {}
    for line in open(os.path.join(GOLDEN, "table1_eps.txt")):
        if line.startswith("#") or not line.strip():
            continue
        v = line.split()
        rows[int(v[0])] = [float(t) for t in v[1:]]
    return rows


def test_eps_schedule_reproduces_table1():
    """Eq. (16) at k_p = 0.05, h0 = 1/8 against Table 1, printed to 2
    significant digits: agree within one unit of the last printed digit (the
    paper truncates 1.95e-4 to 1.9e-4)."""
    for L, printed in _golden_table1().items():
        eps = om.eps_schedule_fem(L, 1 / 8, 0.05)
        assert len(eps) == len(printed) == L + 1
        for e, p in zip(eps, printed):
            unit = 10 ** (math.floor(math.log10(p)) - 1)
            assert abs(e - p) <= unit * 1.0001, (L, e, p)
    # the general form Eq. (15) with Lemma 4.5's rates is Eq. (16)
    for L in range(1, 7):
        assert np.allclose(om.eps_schedule_general(L, 1 / 8, 2, 0.05, 2, 1, 4, 2),
                           om.eps_schedule_fem(L, 1 / 8, 0.05), rtol=1e-14)
    # schedule safety (inequalities after Eq. (15))
    eps = om.eps_schedule_fem(5, 1 / 8, 0.05)
    for l, e in enumerate(eps):
        assert e ** 2 <= 0.05 * (1 / 8 / 2 ** l) ** 4 * (1 + 1e-12)
    assert eps[-1] <= 0.05 * (1 / 8 / 32) ** 2 * (1 + 1e-12)


def test_optimal_samples_and_cost_formulas():
    N = om.optimal_samples([4, 1], [1, 4], math.sqrt(2))
    assert np.allclose(N, [8, 2])
    N2 = om.optimal_samples([8, 2], [1, 4], math.sqrt(2))
    assert np.allclose(N2, [2 * v for v in N])                     # homogeneous in V
    V, Cs, TOL = [3e-5, 2e-6, 3e-8], [1.0, 5.0, 30.0], 1e-3
    N = om.optimal_samples(V, Cs, TOL)
    assert abs(sum(v / n for v, n in zip(V, N)) - TOL ** 2 / 2) < 1e-18   # variance constraint is tight
    assert om.predicted_gain(0.25, 2, 4, 2) == 0.625               # "at least a factor of 1.6"
    assert abs(om.predicted_gain(0.5, 2, 4, 2) - 0.75) < 1e-15
    assert abs(om.finite_L_cost_ratio(0.25, 2, 4, 2, 200) - 0.625) < 1e-12
    with pytest.raises(ValueError):
        om.predicted_gain(0.25, 2, 2, 4)


def test_estimators_use_1_over_N():
    rng = np.random.default_rng(4)
    Y = list(rng.normal(size=37))
    assert abs(om.level_var(Y) - np.var(Y, ddof=0)) < 1e-15
    assert abs(om.level_mean(Y) - np.mean(Y)) < 1e-15
    assert om.mlmc_estimate([1.0, 0.5, 0.25]) == 1.75


def test_algorithm2_synthetic_levels():
    """Algorithm 2 on synthetic levels with known mean/variance decay
    (E[Y_l] = 0.03 * 4^-l, V[Y_l] = 1e-5 * 16^-l, C_l = 4^l)."""
    rng = np.random.default_rng(5)

    def sampler(l, first, count, tf, tc):
        mu, sd = 0.03 * 4.0 ** -l, math.sqrt(1e-5 * 16.0 ** -l)
        return list(rng.normal(mu, sd, count)), [4.0 ** l] * count

    for TOL in (1e-3, 3e-4):
        res = om.adaptive_mpml(sampler, TOL, 1 / 8, 0.05, L_max=8, N_init=100)
        assert res.code == 0
        assert abs(res.means[-1]) <= 3 / math.sqrt(2) * TOL
        assert sum(v / n for v, n in zip(res.variances, res.N)) <= TOL ** 2 / 2
        assert abs(res.estimate - 0.03 * sum(4.0 ** -l for l in range(res.L + 1))) < 5 * TOL
    # L_max reached with the bias test failing -> code 4 (R2)
    res = om.adaptive_mpml(sampler, 1e-5, 1 / 8, 0.05, L_max=2, N_init=50)
    assert res.code == 4 and res.L == 2


def test_algorithm2_deterministic_field_stops_at_L1():
    """omega pinned to 0 (zero variance): terminates at L = 1 with N = N_init and
    the estimate Q_1(0) (the telescoping sum)."""
    P = oc.OracleProblem(0, 16, 1.0, 0.3, 2.0, 8)
    q = {N: P.solve_mesh(N, np.zeros(16), oc.SOLVER_DIRECT)["Q"] for N in (8, 16)}

    def sampler(l, first, count, tf, tc):
        y = q[16] - q[8] if l == 1 else q[8]
        return [y] * count, [1.0] * count

    res = om.adaptive_mpml(sampler, 1e-2, 1 / 8, 0.05, L_max=4, N_init=100)
    assert res.code == 0 and res.L == 1 and res.N == [100, 100]
    assert abs(res.estimate - q[16]) < 1e-15


# ============================================================================ worked examples (SC-12/15)
def test_worked_example_qois():
    """Regression hints from an independent scipy implementation (SURVEY SC-12,
    SC-15); conventions R10, R11.  Tolerance 1e-9 relative (that session used
    Brent roots with xtol ~ 2e-12)."""
    P = oc.OracleProblem(0, 16, 1.0, 0.3, 2.0, 8)
    cases = [(np.eye(16)[0], 0.022691784995, 0.023698363769),
             (np.ones(16) / 4.0, 0.029050894284, 0.030214832769),
             (np.array([(-1.0) ** k for k in range(16)]), 0.021293703254, 0.022412473280)]
    for xi, q8, q16 in cases:
        assert abs(P.solve_mesh(8, xi, 0)["Q"] / q8 - 1) < 1e-9
        assert abs(P.solve_mesh(16, xi, 0)["Q"] / q16 - 1) < 1e-9
    P20 = oc.OracleProblem(1, 4, 4.0, 0.0, 2.0, 8)   # Eq. (20): s = 4, q = 2, sigma = 2
    for xi, vals in (([1, 0, 0, 0], (0.028698442814, 0.031055248935, 0.031701820214)),
                     ([1, 1, 1, 1], (0.028117869376, 0.030172536354, 0.030738751883)),
                     ([1, -1, 1, -1], (0.028120529977, 0.031269046318, 0.032240469316))):
        for N, v in zip((8, 16, 32), vals):
            assert abs(P20.solve_mesh(N, np.array(xi, float), 0)["Q"] - v) < 2e-12


def test_coupled_sample_structure():
    P = oc.OracleProblem(0, 16, 1.0, 0.3, 2.0, 8)
    out0 = P.coupled_sample(0, 0, 5)
    assert out0[1] == 0.0 and out0[6] == 0
    out1 = P.coupled_sample(1, 0, 5)
    xi = oc.normals(0, 1, 5, 16)
    assert out1[0] == P.solve_mesh(16, xi, 0)["Q"] and out1[1] == P.solve_mesh(8, xi, 0)["Q"]
    m = P.coupled_sample(2, 0, 3, solver=oc.SOLVER_MINRES, tol_f=1e-8, tol_c=1e-6)
    d = P.coupled_sample(2, 0, 3)
    assert m[4] <= 1e-8 * (1 + 1e-6) and m[5] <= 1e-6 * (1 + 1e-6)
    assert abs(m[0] - d[0]) < 1e-6 and abs(m[1] - d[1]) < 1e-4
