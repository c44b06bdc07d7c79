"""Coarse-to-fine initial guess for the fine half of a coupled sample (NEXT-4 of SURVEY section 8(f); the
paper's remark that the solver may start from any initial guess under the relative-residual criterion,
P:97-102; reading R32) -- TEST INFRASTRUCTURE ONLY (see ``oracle/__init__.py``).

Step by step: the coarse half (mesh h_{l-1}) is solved by textbook MINRES from 0 to tol_c
(``core.minres_band``); its solution is interpolated to the fine mesh with the P1 prolongation of
``oracle/mg.py`` (pinned against the closed-form coarse hat functions); the fine half is solved by MINRES
from that x0 (``core.minres_band_x0``: Paige-Saunders on A e = b - A x0, stopped at phibar_k <= tol_f ||b||).
"""
from __future__ import annotations

import numpy as np

from . import core
from . import mg


def coupled_sample_c2f(P: core.OracleProblem, level: int, seed: int, index: int, tol_f: float, tol_c: float,
                       max_iter: int = 100000) -> dict:
    if level < 1:
        raise ValueError("coarse-to-fine needs level >= 1")
    xi = core.normals(seed, level, index, P.m)
    Nf = P.h0_inv << level
    Nc = Nf // 2
    ABc, _, bc = core.assemble(Nc, P.field_triangles(Nc, xi))
    xc, itc, rrc, stc = core.minres_band(ABc, bc, tol_c, max_iter)
    x0 = mg.prolongation(Nf) @ xc
    ABf, _, bf = core.assemble(Nf, P.field_triangles(Nf, xi))
    xf, itf, rrf, stf = core.minres_band_x0(ABf, bf, x0, tol_f, max_iter)
    return {"Qf": xf.sum() / Nf ** 2, "Qc": xc.sum() / Nc ** 2, "iters_f": itf, "iters_c": itc, "relres_f": rrf,
            "relres_c": rrc, "status_f": stf, "status_c": stc, "x0": x0, "xf": xf, "AB": ABf, "b": bf}
