"""Multigrid-preconditioned CG (NEXT-4 of SURVEY section 8(f); the paper's "optimal solver") --
TEST INFRASTRUCTURE ONLY (see ``oracle/__init__.py``).

Textbook definitions in binary64, written so that a reader can check them one by one:

* ``prolongation(N)``: P1 interpolation from the nested mesh of spacing 2h = 2/N (its SW-NE
  triangles, P:611 / reading R10) to the mesh of spacing h, on the interior unknowns (the Dirichlet
  nodes are dropped).  A fine node that is a coarse node takes its value; a fine node at the
  midpoint of a coarse horizontal, vertical or SW-NE diagonal edge takes the mean of the edge's ends.
* ``hierarchy(N, a)``: A_h from the oracle's generic element assembly (``core.assemble``), then the
  Galerkin products A_{2h} = P^T A_h P as sparse matrix products -- the textbook definition, *not*
  the coefficient-averaging shortcut the CUDA kernels use (the tests compare the two).
* ``vcycle``: red-black Gauss-Seidel (red = (i + j) even), red then black before the coarse
  correction and black then red after, the single unknown of the 1/2-mesh solved exactly, u = 0 at
  the start of every level.
* ``pcg``: conjugate gradients from x0 = 0 preconditioned by one V-cycle, stopped at the first k with
  ||r_k||_2 / ||b||_2 <= tol, r_k the CG recurrence residual (reading R30).
* ``cg``: plain conjugate gradients (Hestenes-Stiefel) from x0 = 0 with the same stopping rule -- the
  Krylov solver the paper names beside MINRES for the SPD systems (NEXT-4).

Every step is plain numpy / scipy.sparse (a library sparse product and matrix-vector product); no
blocking or fusion.
"""
from __future__ import annotations

import numpy as np
import scipy.sparse as sp

from . import core


def interior_index(N: int, i: int, j: int) -> int:
    """Unknown of node (i, j), 1 <= i, j <= N - 1 (the oracle's assembly order)."""
    return (j - 1) * (N - 1) + (i - 1)


def prolongation(N: int) -> sp.csr_matrix:
    """P1 interpolation N/2 -> N on the interior unknowns: sparse ((N-1)^2 x (N/2-1)^2)."""
    Nc = N // 2
    rows, cols, vals = [], [], []

    def add(r, I, J, w):
        if 1 <= I <= Nc - 1 and 1 <= J <= Nc - 1:          # coarse Dirichlet nodes carry 0
            rows.append(r)
            cols.append(interior_index(Nc, I, J))
            vals.append(w)

    for j in range(1, N):
        for i in range(1, N):
            r = interior_index(N, i, j)
            I, J = i // 2, j // 2
            if i % 2 == 0 and j % 2 == 0:
                add(r, I, J, 1.0)                             # a coarse node
            elif i % 2 == 1 and j % 2 == 0:
                add(r, I, J, 0.5)                             # midpoint of a horizontal coarse edge
                add(r, I + 1, J, 0.5)
            elif i % 2 == 0 and j % 2 == 1:
                add(r, I, J, 0.5)                             # midpoint of a vertical coarse edge
                add(r, I, J + 1, 0.5)
            else:
                add(r, I, J, 0.5)                             # midpoint of the SW-NE diagonal
                add(r, I + 1, J + 1, 0.5)
    return sp.csr_matrix((vals, (rows, cols)), shape=((N - 1) ** 2, (Nc - 1) ** 2))


def stiffness(N: int, a_tri) -> tuple[sp.csr_matrix, np.ndarray]:
    """A_h (sparse, symmetric) and b from the oracle's element assembly (lower band -> full)."""
    AB, _, b = core.assemble(N, a_tri)
    n, bwp1 = AB.shape
    rows, cols, vals = [], [], []
    for d in range(bwp1):
        p = np.arange(d, n)
        v = AB[d:, d]
        nz = v != 0.0
        rows.append(p[nz])
        cols.append(p[nz] - d)
        vals.append(v[nz])
        if d:
            rows.append(p[nz] - d)
            cols.append(p[nz])
            vals.append(v[nz])
    A = sp.csr_matrix((np.concatenate(vals), (np.concatenate(rows), np.concatenate(cols))), shape=(n, n))
    return A, b


def hierarchy(N: int, a_tri):
    """[(N_l, A_l, P_l)] for N_l = N, N/2, ..., 2 (P_l maps level l+1 to l; None on the last level), b."""
    A, b = stiffness(N, a_tri)
    levels = []
    Nl = N
    while True:
        if Nl == 2:
            levels.append((Nl, A, None))
            break
        P = prolongation(Nl)
        levels.append((Nl, A, P))
        A = (P.T @ A @ P).tocsr()                             # Galerkin coarse operator
        Nl //= 2
    return levels, b


def colours(N: int) -> tuple[np.ndarray, np.ndarray]:
    """Unknown indices of the red ((i + j) even) and black nodes."""
    red, black = [], []
    for j in range(1, N):
        for i in range(1, N):
            (red if (i + j) % 2 == 0 else black).append(interior_index(N, i, j))
    return np.array(red, dtype=np.int64), np.array(black, dtype=np.int64)


def gs_colour(A: sp.csr_matrix, u: np.ndarray, f: np.ndarray, idx: np.ndarray) -> None:
    """Gauss-Seidel update of the unknowns idx (one colour; no couplings inside a colour, which
    ``tests/test_oracle_mg.py`` checks): u_p = (f_p - sum_{q != p} A_pq u_q) / A_pp."""
    d = A.diagonal()[idx]
    u[idx] = (f[idx] - (A[idx] @ u) + d * u[idx]) / d


def vcycle(levels, l: int, f: np.ndarray) -> np.ndarray:
    """V(1,1) from u = 0 on level l: M_l^-1 f."""
    N, A, P = levels[l]
    if N == 2:
        return f / A.diagonal()
    red, black = colours(N)
    u = np.zeros_like(f)
    gs_colour(A, u, f, red)
    gs_colour(A, u, f, black)
    r = f - A @ u
    u += P @ vcycle(levels, l + 1, P.T @ r)
    gs_colour(A, u, f, black)
    gs_colour(A, u, f, red)
    return u


def pcg(N: int, a_tri, tol: float, max_iter: int = 1000) -> dict:
    """MG-preconditioned CG from x0 = 0; Q = h^2 1^T x."""
    levels, b = hierarchy(N, a_tri)
    A = levels[0][1]
    x = np.zeros_like(b)
    r = b.copy()
    z = vcycle(levels, 0, r)
    p = z.copy()
    rz = r @ z
    bnorm = np.linalg.norm(b)
    it, status = 0, 1
    while it < max_iter:
        q = A @ p
        alpha = rz / (p @ q)
        x += alpha * p
        r -= alpha * q
        it += 1
        if np.linalg.norm(r) <= tol * bnorm:
            status = 0
            break
        z = vcycle(levels, 0, r)
        rz_new = r @ z
        p = z + (rz_new / rz) * p
        rz = rz_new
    h = 1.0 / N
    return {"Q": h * h * x.sum(), "iters": it, "status": status, "x": x,
            "relres_true": np.linalg.norm(b - A @ x) / bnorm}


def cg(N: int, a_tri, tol: float, max_iter: int = 100000) -> dict:
    """Unpreconditioned CG from x0 = 0; stop at the first k with ||r_k|| / ||b|| <= tol (R30);
    Q = h^2 1^T x."""
    A, b = stiffness(N, a_tri)
    x = np.zeros_like(b)
    r = b.copy()
    p = r.copy()
    rr = r @ r
    bnorm = np.sqrt(rr)
    it, status = 0, 1
    if bnorm == 0.0:
        status = 0
    while status == 1 and it < max_iter:
        q = A @ p
        alpha = rr / (p @ q)
        x += alpha * p
        r -= alpha * q
        it += 1
        rr_new = r @ r
        if np.sqrt(rr_new) <= tol * bnorm:
            status = 0
            break
        p = r + (rr_new / rr) * p
        rr = rr_new
    h = 1.0 / N
    return {"Q": h * h * x.sum(), "iters": it, "status": status, "x": x,
            "relres_true": np.linalg.norm(b - A @ x) / bnorm}
