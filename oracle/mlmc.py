"""MLMC / MPML estimators and Algorithm 2 -- TEST INFRASTRUCTURE ONLY.

Written step by step from the paper (P:n = /root/reference/PAPER.md line n) in
its own order and notation, in plain Python floats (binary64).  Readings where
the paper is silent or garbled are DESIGN.md section 3's R1..R24.
"""
from __future__ import annotations

import math
from dataclasses import dataclass, field
from typing import Callable, List, Sequence


# ----------------------------------------------------------------------------- Eq. (14)-(16)
def eps_schedule_general(L: int, h0: float, m: int, k_p: float, alpha1: float, alpha2: float,
                         beta1: float, beta2: float) -> List[float]:
    """Eq. (15): eps_l = (k_p h_l^beta1)^(1/beta2) for l < L and
    eps_L = min{(k_p h_L^beta1)^(1/beta2), (k_p h_L^alpha1)^(1/alpha2)}; h_l = h0 m^-l."""
    h = [h0 * m ** (-l) for l in range(L + 1)]
    eps = [(k_p * h[l] ** beta1) ** (1.0 / beta2) for l in range(L)]
    eps.append(min((k_p * h[L] ** beta1) ** (1.0 / beta2), (k_p * h[L] ** alpha1) ** (1.0 / alpha2)))
    return eps


def eps_schedule_fem(L: int, h0: float, k_p: float, m: int = 2) -> List[float]:
    """Eq. (16): eps_l = sqrt(k_p) h_l^2 (l < L), eps_L = k_p h_L^2."""
    h = [h0 * m ** (-l) for l in range(L + 1)]
    return [math.sqrt(k_p) * h[l] ** 2 for l in range(L)] + [k_p * h[L] ** 2]


# ----------------------------------------------------------------------------- Eq. (3), (4)
def level_mean(Y: Sequence[float]) -> float:
    """hat Y_l = (1/N_l) sum_k Y_l^(k)."""
    return sum(Y) / len(Y)


def level_var(Y: Sequence[float]) -> float:
    """s_l^2 = (1/N_l) sum_k (Y_l^(k) - hat Y_l)^2 (Eq. (4)) -- 1/N_l, not 1/(N_l-1)."""
    mu = level_mean(Y)
    return sum((y - mu) ** 2 for y in Y) / len(Y)


def mlmc_estimate(level_means: Sequence[float]) -> float:
    """Eq. (3): hat Q = sum_l hat Y_l."""
    return sum(level_means)


# ----------------------------------------------------------------------------- Algorithm 2 step 7
def optimal_samples(V: Sequence[float], Cst: Sequence[float], TOL: float) -> List[float]:
    """N_l = sqrt(V_l / C_l) (2 / TOL^2) sum_k sqrt(V_k C_k), real-valued."""
    S = sum(math.sqrt(v * c) for v, c in zip(V, Cst))
    return [math.sqrt(v / c) * 2.0 / TOL ** 2 * S for v, c in zip(V, Cst)]


def predicted_gain(q: float, m: float, beta: float, gamma: float) -> float:
    """Corollary 4.4: C_MPML / C_ML <= q + m^((gamma-beta)/2) (1-q)."""
    if not beta > gamma:
        raise ValueError("Corollary 4.4 needs beta > gamma")
    return q + m ** ((gamma - beta) / 2.0) * (1.0 - q)


def finite_L_cost_ratio(q: float, m: float, beta: float, gamma: float, L: int) -> float:
    """The finite-L bound displayed at P:419."""
    r = m ** ((gamma - beta) / 2.0)
    return q * (1 - r) / (1 - r ** L) + r * (1 - r ** (L - 1)) / (1 - r ** L)


# ----------------------------------------------------------------------------- Algorithm 2
@dataclass
class LevelState:
    Y: List[float] = field(default_factory=list)   # all coupled differences drawn so far
    cost: List[float] = field(default_factory=list)
    eps_used: List[float] = field(default_factory=list)


@dataclass
class AdaptiveResult:
    estimate: float
    L: int
    N: List[int]
    means: List[float]
    variances: List[float]
    costs: List[float]
    eps_last: List[float]
    rounds: int
    code: int               # 0 ok, 4 L_max reached with the bias test failing (R2)


def adaptive_mpml(sampler: Callable[[int, int, int, float, float], tuple],
                  TOL: float, h0: float, k_p: float | None, L_max: int, N_init: int = 100,
                  m: int = 2, alpha: float = 2.0, r: float = 1.0, fixed_tol: float = 1e-10,
                  max_rounds: int = 100) -> AdaptiveResult:
    """Algorithm 2, with readings R1-R6, R8, R20, R21, R23.

    ``sampler(level, first_index, count, tol_fine, tol_coarse)`` returns two lists
    (Y values, per-sample costs) for global sample indices
    [first_index, first_index + count) of that level.  ``k_p=None`` is standard
    MLMC (Algorithm 2 without step 2): every solve at ``fixed_tol``.
    """
    L = 1                                                       # REQUIRE: L = 1
    st = [LevelState(), LevelState()]
    N_target = [float(N_init), float(N_init)]                   # N_0 = N_1 = N_init
    code, rounds, eps = 0, 0, []
    bias_c = (r * m ** alpha - 1.0) / math.sqrt(2.0)            # R1
    while L <= L_max and rounds < max_rounds:                   # WHILE L <= L_max
        rounds += 1
        # step 2: eps_l via Eq. (16) for the current L (R20: computed samples are kept)
        if k_p is None:
            eps = [fixed_tol] * (L + 1)
        else:
            eps = eps_schedule_fem(L, h0, k_p, m)
        for l in range(L + 1):                                  # FOR l = 0..L
            dN = max(0, math.ceil(N_target[l]) - len(st[l].Y))  # R3
            if dN > 0:                                          # step 4 (R8: coarse half at eps_{l-1})
                Y, c = sampler(l, len(st[l].Y), dN, eps[l], eps[l - 1] if l > 0 else 0.0)
                st[l].Y.extend(Y)
                st[l].cost.extend(c)
                st[l].eps_used.extend([eps[l]] * dN)
        means = [level_mean(s.Y) for s in st]                   # step 5
        V = [level_var(s.Y) for s in st]
        Cst = [sum(s.cost) / len(s.cost) for s in st]           # R5, R21
        Nopt = optimal_samples(V, Cst, TOL)                     # step 7 (R4)
        N_target = [max(float(len(s.Y)), n) for s, n in zip(st, Nopt)]   # R3: N_l never decreases
        bias_fail = abs(means[L]) > bias_c * TOL                # step 8
        # step 12's variance test uses the N_l drawn so far (R25): with the updated
        # targets of step 7 it would hold with equality by construction.
        var_ok = sum(v / len(s.Y) for v, s in zip(V, st)) <= TOL ** 2 / 2.0
        if not bias_fail and var_ok:                            # steps 12-13 (R2: stop here)
            return AdaptiveResult(mlmc_estimate(means), L, [len(s.Y) for s in st], means, V, Cst,
                                  eps, rounds, 0)
        if bias_fail:
            if L == L_max:                                      # R2: cannot refine further
                code = 4
                if var_ok:
                    break
                continue
            L += 1                                              # steps 9-10
            st.append(LevelState())
            N_target.append(float(N_init))
    means = [level_mean(s.Y) for s in st]
    V = [level_var(s.Y) for s in st]
    Cst = [sum(s.cost) / len(s.cost) for s in st]
    return AdaptiveResult(mlmc_estimate(means), L, [len(s.Y) for s in st], means, V, Cst, eps,
                          rounds, code if code else 4)
