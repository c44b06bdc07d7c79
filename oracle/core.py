"""ctypes binding of ``oracle.c`` -- TEST INFRASTRUCTURE ONLY (see ``oracle/__init__.py``).

Marshalling only; every number is computed in ``oracle.c``.  The shared library
is built by :func:`build` with plain ``gcc -O2`` (no ``-march=native``: the
binary travels to the GPU box, whose host CPU may differ).
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess
import threading

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "oracle.c")
_SO = os.path.join(_HERE, "liboracle.so")
_lock = threading.Lock()
_lib = None

FMT = {"q": 0, "h": 1, "s": 2, "d": 3}
SOLVER_DIRECT, SOLVER_MINRES, SOLVER_IR = 0, 1, 2


def build(force: bool = False) -> str:
    """Compile oracle.c -> liboracle.so (gcc, binary64, no fast-math)."""
    if force or not os.path.exists(_SO) or os.path.getmtime(_SO) < os.path.getmtime(_SRC):
        subprocess.check_call(["gcc", "-O2", "-std=c11", "-fno-fast-math", "-shared", "-fPIC",
                               "-o", _SO, _SRC, "-lm"])
    return _SO


class Problem(C.Structure):
    _fields_ = [("field", C.c_int), ("m", C.c_int), ("sigma2", C.c_double),
                ("corr_len", C.c_double), ("q_decay", C.c_double), ("h0_inv", C.c_int),
                ("ik", C.POINTER(C.c_int)), ("jk", C.POINTER(C.c_int)),
                ("lam", C.POINTER(C.c_double)), ("w1d", C.POINTER(C.c_double)),
                ("K_used", C.c_int)]


def lib():
    global _lib
    with _lock:
        if _lib is None:
            L = C.CDLL(build())
            dp = np.ctypeslib.ndpointer(dtype=np.float64, flags="C_CONTIGUOUS")
            ip = np.ctypeslib.ndpointer(dtype=np.int32, flags="C_CONTIGUOUS")
            up = np.ctypeslib.ndpointer(dtype=np.uint32, flags="C_CONTIGUOUS")
            L.or_philox4x32_10.argtypes = [up, up, up]
            L.or_normals.argtypes = [C.c_uint64, C.c_int, C.c_uint64, C.c_int, dp]
            L.or_kl_roots_1d.argtypes = [C.c_double, C.c_int, dp]
            L.or_kl_theta.argtypes = [C.c_double, C.c_double]
            L.or_kl_theta.restype = C.c_double
            L.or_kl_norm.argtypes = [C.c_double, C.c_double]
            L.or_kl_norm.restype = C.c_double
            L.or_kl_efun.argtypes = [C.c_double, C.c_double, C.c_double]
            L.or_kl_efun.restype = C.c_double
            L.or_kl_modes.argtypes = [C.c_double, C.c_double, C.c_int, ip, ip, dp, dp]
            L.or_centroid.argtypes = [C.c_int, C.c_int, C.POINTER(C.c_double), C.POINTER(C.c_double)]
            L.or_problem_init.argtypes = [C.POINTER(Problem)]
            L.or_problem_free.argtypes = [C.POINTER(Problem)]
            L.or_field_triangles.argtypes = [C.POINTER(Problem), C.c_int, dp, dp]
            L.or_assemble.argtypes = [C.c_int, dp, C.c_int, C.c_void_p, C.c_void_p, dp]
            L.or_band_matvec.argtypes = [C.c_int, C.c_int, dp, dp, dp]
            L.or_chol_band.argtypes = [C.c_int, C.c_int, dp, dp]
            L.or_chol_band_solve.argtypes = [C.c_int, C.c_int, dp, dp, dp]
            L.or_chol_dense.argtypes = [C.c_int, dp, dp]
            L.or_chol_dense_solve.argtypes = [C.c_int, dp, dp, dp]
            L.or_minres_band.argtypes = [C.c_int, C.c_int, dp, dp, C.c_double, C.c_int, dp,
                                         C.POINTER(C.c_int), C.POINTER(C.c_double)]
            L.or_minres_band_x0.argtypes = [C.c_int, C.c_int, dp, dp, dp, C.c_double, C.c_int, dp,
                                            C.POINTER(C.c_int), C.POINTER(C.c_double)]
            L.or_round.argtypes = [C.c_double, C.c_int]
            L.or_round.restype = C.c_double
            L.or_chol_band_rounded.argtypes = [C.c_int, C.c_int, dp, dp, C.c_int]
            L.or_band_solve_rounded.argtypes = [C.c_int, C.c_int, dp, dp, dp, C.c_int]
            L.or_ir_band.argtypes = [C.c_int, C.c_int, dp, dp, ip, C.c_double, C.c_int, dp,
                                     C.POINTER(C.c_int), C.POINTER(C.c_double)]
            L.or_solve_level_mesh.argtypes = [C.POINTER(Problem), C.c_int, dp, C.c_int, ip,
                                              C.c_double, C.c_int, dp]
            L.or_coupled_sample.argtypes = [C.POINTER(Problem), C.c_int, C.c_uint64, C.c_uint64,
                                            C.c_int, ip, ip, C.c_double, C.c_double, C.c_int, dp]
            _lib = L
    return _lib


# ----------------------------------------------------------------------------- RNG
def philox(ctr, key):
    out = np.zeros(4, np.uint32)
    lib().or_philox4x32_10(np.asarray(ctr, np.uint32), np.asarray(key, np.uint32), out)
    return out


def normals(seed: int, level: int, index: int, m: int) -> np.ndarray:
    xi = np.zeros(m, np.float64)
    lib().or_normals(seed, level, index, m, xi)
    return xi


# ----------------------------------------------------------------------------- KL
def kl_roots(corr_len: float, K: int) -> np.ndarray:
    w = np.zeros(K, np.float64)
    if lib().or_kl_roots_1d(corr_len, K, w) != 0:
        raise RuntimeError("root scan failed")
    return w


def kl_theta(corr_len, w):
    return lib().or_kl_theta(corr_len, w)


def kl_norm(corr_len, w):
    return lib().or_kl_norm(corr_len, w)


def kl_efun(corr_len, w, x):
    return lib().or_kl_efun(corr_len, w, x)


def kl_modes(sigma2: float, corr_len: float, m: int):
    ik = np.zeros(m, np.int32)
    jk = np.zeros(m, np.int32)
    lam = np.zeros(m, np.float64)
    w1d = np.zeros(m + 1, np.float64)
    if lib().or_kl_modes(sigma2, corr_len, m, ik, jk, lam, w1d) != 0:
        raise RuntimeError("kl_modes failed")
    return ik, jk, lam, w1d


def centroid(N: int, t: int):
    a, b = C.c_double(), C.c_double()
    lib().or_centroid(N, t, C.byref(a), C.byref(b))
    return a.value, b.value


# ----------------------------------------------------------------------------- problem
class OracleProblem:
    """A field definition with its KL modes precomputed once (or_problem_init)."""

    def __init__(self, field: int = 0, m: int = 16, sigma2: float = 1.0, corr_len: float = 0.3,
                 q_decay: float = 2.0, h0_inv: int = 8):
        self.p = Problem(field, m, sigma2, corr_len, q_decay, h0_inv, None, None, None, None, 0)
        if lib().or_problem_init(C.byref(self.p)) != 0:
            raise RuntimeError("or_problem_init failed")
        self.m = m
        self.h0_inv = h0_inv

    def __del__(self):
        try:
            lib().or_problem_free(C.byref(self.p))
        except Exception:
            pass

    def field_triangles(self, N: int, xi) -> np.ndarray:
        a = np.zeros(2 * N * N, np.float64)
        if lib().or_field_triangles(C.byref(self.p), N, np.ascontiguousarray(xi, np.float64), a) != 0:
            raise RuntimeError("field failed")
        return a

    def solve_mesh(self, N: int, xi, solver: int, tol: float = 0.0, quad="dddd", max_iter: int = 100000):
        out = np.zeros(4, np.float64)
        q = np.array([FMT[c] for c in quad], np.int32)
        lib().or_solve_level_mesh(C.byref(self.p), N, np.ascontiguousarray(xi, np.float64), solver, q,
                                  tol, max_iter, out)
        return {"Q": out[0], "iters": int(out[1]), "relres": out[2], "status": int(out[3])}

    def coupled_sample(self, level: int, seed: int, index: int, solver: int = SOLVER_DIRECT,
                       tol_f: float = 0.0, tol_c: float = 0.0, quad_f="dddd", quad_c="dddd",
                       max_iter: int = 100000) -> np.ndarray:
        """[Qf, Qc, iters_f, iters_c, relres_f, relres_c, status_f, status_c]."""
        out = np.zeros(8, np.float64)
        qf = np.array([FMT[c] for c in quad_f], np.int32)
        qc = np.array([FMT[c] for c in quad_c], np.int32)
        lib().or_coupled_sample(C.byref(self.p), level, seed, index, solver, qf, qc, tol_f, tol_c,
                                max_iter, out)
        return out


# ----------------------------------------------------------------------------- assembly / solvers
def assemble(N: int, a_tri, f_kind: int = 0, dense: bool = False):
    n, bw = (N - 1) ** 2, N - 1
    AB = np.zeros(n * (bw + 1), np.float64)
    b = np.zeros(n, np.float64)
    D = np.zeros(n * n, np.float64) if dense else None
    rc = lib().or_assemble(N, np.ascontiguousarray(a_tri, np.float64), f_kind, AB.ctypes.data,
                           D.ctypes.data if dense else None, b)
    if rc != 0:
        raise RuntimeError("assembly failed")
    return AB.reshape(n, bw + 1), (D.reshape(n, n) if dense else None), b


def band_matvec(AB, x):
    n, bwp1 = AB.shape
    y = np.zeros(n, np.float64)
    lib().or_band_matvec(n, bwp1 - 1, np.ascontiguousarray(AB).ravel(), np.ascontiguousarray(x, np.float64), y)
    return y


def chol_band_solve(AB, b):
    n, bwp1 = AB.shape
    L = np.zeros(n * bwp1, np.float64)
    if lib().or_chol_band(n, bwp1 - 1, np.ascontiguousarray(AB).ravel(), L) != 0:
        raise np.linalg.LinAlgError("non-positive pivot")
    x = np.zeros(n, np.float64)
    lib().or_chol_band_solve(n, bwp1 - 1, L, np.ascontiguousarray(b, np.float64), x)
    return x, L.reshape(n, bwp1)


def chol_dense_solve(A, b):
    n = A.shape[0]
    L = np.zeros(n * n, np.float64)
    if lib().or_chol_dense(n, np.ascontiguousarray(A, np.float64).ravel(), L) != 0:
        raise np.linalg.LinAlgError("non-positive pivot")
    x = np.zeros(n, np.float64)
    lib().or_chol_dense_solve(n, L, np.ascontiguousarray(b, np.float64), x)
    return x, L.reshape(n, n)


def minres_band(AB, b, tol: float, max_iter: int = 100000):
    n, bwp1 = AB.shape
    x = np.zeros(n, np.float64)
    it, rr = C.c_int(), C.c_double()
    st = lib().or_minres_band(n, bwp1 - 1, np.ascontiguousarray(AB).ravel(), np.ascontiguousarray(b, np.float64),
                              tol, max_iter, x, C.byref(it), C.byref(rr))
    return x, it.value, rr.value, st


def minres_band_x0(AB, b, x0, tol: float, max_iter: int = 100000):
    """MINRES from the initial guess x0 (or_minres_band_x0): stops at phibar_k <= tol ||b||."""
    n, bwp1 = AB.shape
    x = np.zeros(n, np.float64)
    it, rr = C.c_int(), C.c_double()
    st = lib().or_minres_band_x0(n, bwp1 - 1, np.ascontiguousarray(AB).ravel(), np.ascontiguousarray(b, np.float64),
                                 np.ascontiguousarray(x0, np.float64), tol, max_iter, x, C.byref(it), C.byref(rr))
    return x, it.value, rr.value, st


def round_to(x: float, fmt: str) -> float:
    return lib().or_round(float(x), FMT[fmt])


def chol_band_rounded(AB, fmt: str):
    """Algorithm 1 step 1: the band factor with every operation rounded to ``fmt``."""
    n, bwp1 = AB.shape
    L = np.zeros(n * bwp1, np.float64)
    st = lib().or_chol_band_rounded(n, bwp1 - 1, np.ascontiguousarray(AB).ravel(), L, FMT[fmt])
    return L.reshape(n, bwp1), st


def band_solve_rounded(L, rhs, fmt: str):
    """Algorithm 1 steps 2 / 7: forward + backward substitution rounded to ``fmt``."""
    n, bwp1 = L.shape
    x = np.zeros(n, np.float64)
    lib().or_band_solve_rounded(n, bwp1 - 1, np.ascontiguousarray(L).ravel(),
                                np.ascontiguousarray(rhs, np.float64), x, FMT[fmt])
    return x


def ir_band(AB, b, quad: str, tol: float, i_max: int = 50):
    n, bwp1 = AB.shape
    x = np.zeros(n, np.float64)
    it, rr = C.c_int(), C.c_double()
    q = np.array([FMT[c] for c in quad], np.int32)
    st = lib().or_ir_band(n, bwp1 - 1, np.ascontiguousarray(AB).ravel(), np.ascontiguousarray(b, np.float64),
                          q, tol, i_max, x, C.byref(it), C.byref(rr))
    return x, it.value, rr.value, st
