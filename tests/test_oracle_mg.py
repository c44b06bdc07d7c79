"""Pins of the oracle's multigrid-preconditioned CG (``oracle/mg.py``, NEXT-4) against mathematics
(-m "not gpu"): the Galerkin identity of nested P1 spaces, the structure the red-black smoother relies
on, the symmetry / definiteness that CG needs, a textbook direct solve, and mesh independence."""
import numpy as np
import pytest
import scipy.sparse.linalg as spla

from oracle import mg


def _lognormal_triangles(N, seed, sigma=1.0):
    rng = np.random.default_rng(seed)
    return np.exp(sigma * rng.standard_normal(2 * N * N))


def _coarse_average(N, a):
    """Coefficient of each triangle of the 2h mesh = mean of the four h triangles inside it (the
    rule the kernels use; derived here from the triangle vertex lists, not from the kernels)."""
    Nc = N // 2
    ac = np.zeros(2 * Nc * Nc)

    def t(i, j, upper):
        return 2 * (j * N + i) + (1 if upper else 0)

    for J in range(Nc):
        for I in range(Nc):
            i, j = 2 * I, 2 * J
            # lower {(I,J), (I+1,J), (I+1,J+1)}: fine L(i,j), L(i+1,j), U(i+1,j), L(i+1,j+1)
            ac[2 * (J * Nc + I)] = 0.25 * (a[t(i, j, 0)] + a[t(i + 1, j, 0)] + a[t(i + 1, j, 1)] + a[t(i + 1, j + 1, 0)])
            # upper {(I,J), (I+1,J+1), (I,J+1)}: fine U(i,j), L(i,j+1), U(i,j+1), U(i+1,j+1)
            ac[2 * (J * Nc + I) + 1] = 0.25 * (a[t(i, j, 1)] + a[t(i, j + 1, 0)] + a[t(i, j + 1, 1)] + a[t(i + 1, j + 1, 1)])
    return ac


def test_prolongation_reproduces_coarse_p1_functions():
    """P maps the nodal values of a coarse P1 function to the nodal values of the same function on
    the fine mesh: check with the hat functions' closed form (a piecewise-linear function that is
    linear on every coarse SW-NE triangle is evaluated exactly at the fine nodes)."""
    N = 16
    Nc = N // 2
    rng = np.random.default_rng(0)
    uc = rng.standard_normal((Nc - 1) ** 2)
    U = np.zeros((Nc + 1, Nc + 1))                       # U[J, I], Dirichlet ring 0
    for J in range(1, Nc):
        for I in range(1, Nc):
            U[J, I] = uc[mg.interior_index(Nc, I, J)]

    def eval_p1(x, y):                                   # x, y in coarse index units
        I, J = min(int(np.floor(x)), Nc - 1), min(int(np.floor(y)), Nc - 1)
        s, t = x - I, y - J
        if s >= t:                                       # lower triangle (I,J),(I+1,J),(I+1,J+1)
            return U[J, I] + s * (U[J, I + 1] - U[J, I]) + t * (U[J + 1, I + 1] - U[J, I + 1])
        return U[J, I] + t * (U[J + 1, I] - U[J, I]) + s * (U[J + 1, I + 1] - U[J + 1, I])

    uf = mg.prolongation(N) @ uc
    ref = np.array([eval_p1(i / 2, j / 2) for j in range(1, N) for i in range(1, N)])
    assert np.max(np.abs(uf - ref)) < 1e-14


@pytest.mark.parametrize("N", [4, 8, 16, 32])
def test_galerkin_product_equals_coarse_assembly_with_averaged_coefficients(N):
    """P^T A_h P (sparse products) == the P1 stiffness of the 2h mesh whose triangle coefficients are
    the means of their four sub-triangles (coarse hats are linear on every coarse triangle and the
    four sub-triangles have equal area) -- the identity that makes every level a 5-point operator."""
    a = _lognormal_triangles(N, N)
    A, _ = mg.stiffness(N, a)
    P = mg.prolongation(N)
    Ag = (P.T @ A @ P).toarray()
    Ac, _ = mg.stiffness(N // 2, _coarse_average(N, a))
    assert np.max(np.abs(Ag - Ac.toarray())) <= 1e-13 * np.max(np.abs(Ac.toarray()))


@pytest.mark.parametrize("N", [8, 16])
def test_every_level_is_five_point_and_colours_decouple(N):
    """The Galerkin operators couple a node only to its E/W/N/S neighbours (the SW-NE coupling of
    P1 on right triangles is zero; the sparse products leave it at rounding level), so red and black
    unknowns are decoupled inside a colour."""
    levels, _ = mg.hierarchy(N, _lognormal_triangles(N, 3))
    for Nl, A, _ in levels:
        D = A.toarray()
        eps = 1e-14 * np.max(np.abs(D))
        red, black = mg.colours(Nl)
        for idx in (red, black):
            B = D[np.ix_(idx, idx)]
            assert np.max(np.abs(B - np.diag(np.diag(B))), initial=0.0) <= eps
        for p in range(D.shape[0]):
            i, j = p % (Nl - 1) + 1, p // (Nl - 1) + 1
            for q in np.nonzero(np.abs(D[p]) > eps)[0]:
                k, l = q % (Nl - 1) + 1, q // (Nl - 1) + 1
                assert abs(i - k) + abs(j - l) <= 1


def test_vcycle_is_symmetric_positive_definite():
    """M^-1 (one V(1,1) cycle with the symmetric red/black order) is SPD, as CG requires."""
    N = 8
    levels, _ = mg.hierarchy(N, _lognormal_triangles(N, 5, sigma=1.5))
    n = (N - 1) ** 2
    M = np.column_stack([mg.vcycle(levels, 0, e) for e in np.eye(n)])
    assert np.max(np.abs(M - M.T)) < 1e-12 * np.max(np.abs(M))
    assert np.min(np.linalg.eigvalsh(0.5 * (M + M.T))) > 0.0


@pytest.mark.parametrize("N", [8, 16, 32, 64])
def test_pcg_matches_direct_solve_and_is_mesh_independent(N):
    """PCG at tol 1e-10: Q within the residual bound of the direct solve (textbook sparse LU on a
    different code path), true residual consistent with the recurrence one, and iteration counts
    bounded independently of h (a = 1: <= 14; i.i.d. lognormal triangles, sigma = 1: <= 22 -- measured
    7/12/13/13 and 11/16/18/20 at h = 1/8 .. 1/64, against MINRES's O(1/h))."""
    for a, cap in ((np.ones(2 * N * N), 14), (_lognormal_triangles(N, 11), 22)):
        r = mg.pcg(N, a, 1e-10)
        assert r["status"] == 0 and r["iters"] <= cap, (N, r["iters"])
        A, b = mg.stiffness(N, a)
        x = spla.spsolve(A.tocsc(), b)
        Qx = x.sum() / N ** 2
        # Q = b^T x (b = h^2 1): |b^T (x~ - x)| = |x^T r| <= tol ||b|| ||x||
        assert abs(r["Q"] - Qx) <= 1e-10 * np.linalg.norm(b) * np.linalg.norm(x) * (1 + 1e-6) + 1e-16
        assert r["relres_true"] <= 1e-9


def test_pcg_constant_coefficient_reference_values():
    """a = 1: the MG-PCG QoI equals the closed-form-pinned discrete values of DESIGN.md section 4
    (Q_h(a = 1) at h = 1/8 .. 1/64, themselves pinned against the Fourier series)."""
    ref = {8: 0.033423031078, 16: 0.034702752314, 32: 0.035033019542, 64: 0.035116381629}
    for N, q in ref.items():
        assert abs(mg.pcg(N, np.ones(2 * N * N), 1e-12)["Q"] - q) < 1e-11


# ---------------------------------------------------------------------------- plain CG
def test_cg_converges_in_as_many_steps_as_distinct_excited_eigenvalues():
    """a = 1, N = 4: A is the 5-point Laplacian (9 unknowns) and b = h^2 1 has components only along the
    eigenvectors sin(i pi x) sin(j pi y) with i, j odd -- (1,1), (1,3), (3,1), (3,3) -- whose eigenvalues
    4 - 2cos(i pi/4) - 2cos(j pi/4) take 3 distinct values, so exact CG terminates at step 3."""
    r = mg.cg(4, np.ones(32), 1e-12)
    assert r["status"] == 0 and r["iters"] == 3
    assert r["relres_true"] < 1e-13


def test_cg_matches_library_cg_and_direct_solve():
    """Iterates of the textbook CG against scipy's CG (an independent implementation, same stopping rule on
    the recurrence residual) and the solution against a sparse direct solve."""
    N, tol = 16, 1e-10
    a = _lognormal_triangles(N, 3)
    r = mg.cg(N, a, tol)
    A, b = mg.stiffness(N, a)
    its = []
    xs, info = spla.cg(A, b, rtol=tol, atol=0.0, maxiter=10000, callback=lambda xk: its.append(1))
    assert info == 0 and abs(len(its) - r["iters"]) <= 1
    xd = spla.spsolve(A.tocsc(), b)
    assert np.linalg.norm(r["x"] - xd) <= 1e-8 * np.linalg.norm(xd)
    Qd = (1.0 / N) ** 2 * xd.sum()
    assert abs(r["Q"] - Qd) <= tol * np.linalg.norm(b) * np.linalg.norm(xd) * (1 + 1e-6)


def test_minres_needs_no_more_steps_than_cg():
    """For SPD A, MINRES minimises ||b - A x|| over the same Krylov space CG works in, so at a given
    residual tolerance it stops no later than CG (one step of slack for rounding)."""
    from oracle import core as oc
    for seed, N in ((5, 8), (6, 16)):
        a = _lognormal_triangles(N, seed)
        r = mg.cg(N, a, 1e-8)
        AB, _, b = oc.assemble(N, a)
        _, m_iters, _, st = oc.minres_band(AB, b, 1e-8)
        assert st == 0 and m_iters <= r["iters"] + 1
