"""ctypes declarations of include/mlmc.h (argument marshalling only).

Loading fails loudly if ``libmlmc.so`` is missing: there is no CPU fallback.
"""
from __future__ import annotations

import ctypes as C
import os
import re

HERE = os.path.dirname(os.path.abspath(__file__))
SO_PATH = os.path.join(HERE, "libmlmc.so")
HEADER = os.path.join(os.path.dirname(HERE), "include", "mlmc.h")

MLMC_OK, MLMC_EINVAL, MLMC_ESOLVER, MLMC_ELMAX, MLMC_ECUDA, MLMC_ENOMEM = 0, 2, 3, 4, 5, 6
MLMC_MAX_LEVELS, MLMC_SUMS_LEN, MLMC_SAMPLE_LEN = 16, 12, 8
FIELD_EXPCOV_KL, FIELD_PAPER_EQ20 = 0, 1
FMT = {"q": 0, "h": 1, "s": 2, "d": 3}
SOLVER_MINRES, SOLVER_CHOL_IR, SOLVER_MGCG, SOLVER_CG = 0, 1, 2, 3
FLAG_VERIFY = 1
FLAG_ESCALATE = 2
FLAG_C2F = 4


class Problem(C.Structure):
    _fields_ = [("field", C.c_int32), ("m", C.c_int32), ("sigma2", C.c_double), ("corr_len", C.c_double),
                ("q_decay", C.c_double), ("h0_inv", C.c_int32), ("refine", C.c_int32), ("L_max", C.c_int32),
                ("device", C.c_int32)]


class Precision(C.Structure):
    _fields_ = [("solver", C.c_int32), ("u_f", C.c_int32), ("u_s", C.c_int32), ("u", C.c_int32),
                ("u_r", C.c_int32), ("max_iter", C.c_int32), ("flags", C.c_int32)]


class LevelSums(C.Structure):
    _fields_ = [(n, C.c_double) for n in ("sum_y", "sum_y2", "sum_qf", "sum_qc", "sum_cost", "n", "n_fail",
                                          "iters_f", "iters_c", "iters_f_max", "iters_c_max", "n_escalated")]


class LevelInfo(C.Structure):
    _fields_ = [("N", C.c_int32), ("n", C.c_int32), ("P", C.c_int32), ("bw", C.c_int32), ("h", C.c_double)]


class AdaptiveOpts(C.Structure):
    _fields_ = [("k_p", C.c_double), ("fixed_tol", C.c_double), ("r_bias", C.c_double), ("N_init", C.c_int32),
                ("policy", C.c_int32), ("rank", C.c_int32), ("world", C.c_int32), ("max_rounds", C.c_int32),
                ("seed", C.c_uint64), ("on_fail", C.c_int32), ("reserved0", C.c_int32)]


class Result(C.Structure):
    _fields_ = [("estimate", C.c_double), ("L", C.c_int32), ("rounds", C.c_int32), ("code", C.c_int32),
                ("n_fail", C.c_int32), ("N", C.c_uint64 * MLMC_MAX_LEVELS), ("eps", C.c_double * MLMC_MAX_LEVELS),
                ("mean", C.c_double * MLMC_MAX_LEVELS), ("var", C.c_double * MLMC_MAX_LEVELS),
                ("cost", C.c_double * MLMC_MAX_LEVELS), ("solve_seconds", C.c_double)]


class DDLayout(C.Structure):
    _fields_ = [(n, C.c_int32) for n in ("N", "rank", "world", "j0", "j1", "rows", "pitch", "tiles")] + \
               [("bytes", C.c_uint64), ("plane_off", C.c_uint64 * 5), ("sums_off", C.c_uint64),
                ("state_off", C.c_uint64), ("partials_off", C.c_uint64), ("counter_off", C.c_uint64),
                ("rpart_off", C.c_uint64), ("xi_off", C.c_uint64), ("a_off", C.c_uint64)]


class KernelStat(C.Structure):
    _fields_ = [("kind", C.c_int32), ("N", C.c_int32), ("launches", C.c_uint64), ("ms", C.c_double)]


KERNEL_KINDS = {0: "rng", 1: "field", 2: "minres", 3: "chol_ir", 4: "sums", 5: "order"}

ALLREDUCE_FN = C.CFUNCTYPE(C.c_int, C.POINTER(C.c_double), C.c_int, C.c_int, C.c_void_p)
LEVEL_SAMPLER_FN = C.CFUNCTYPE(C.c_int, C.c_int, C.c_uint64, C.c_uint64, C.POINTER(Precision),
                               C.POINTER(Precision), C.c_double, C.c_double, C.POINTER(C.c_double), C.c_void_p)

_lib = None


def declared_symbols() -> list:
    """Every function name declared in include/mlmc.h."""
    txt = open(HEADER).read()
    txt = re.sub(r"/\*.*?\*/", "", txt, flags=re.S)
    names = re.findall(r"\b(mlmc_[a-z_0-9]+)\s*\(", txt)
    return sorted(set(n for n in names if not n.endswith("_fn")))


def lib():
    """Load libmlmc.so (raises if it has not been built: no fallback)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(SO_PATH):
        raise ImportError(f"{SO_PATH} is missing: run `python -c 'import __graft_entry__ as g; g.build()'` "
                          "(there is no CPU fallback)")
    L = C.CDLL(SO_PATH)
    vp, dp = C.c_void_p, C.POINTER(C.c_double)
    L.mlmc_plan_levels.argtypes = [C.POINTER(Problem), C.POINTER(vp)]
    L.mlmc_destroy.argtypes = [vp]
    L.mlmc_destroy.restype = None
    L.mlmc_strerror.argtypes = [C.c_int]
    L.mlmc_strerror.restype = C.c_char_p
    L.mlmc_last_error.argtypes = [vp]
    L.mlmc_last_error.restype = C.c_char_p
    L.mlmc_level_info_get.argtypes = [vp, C.c_int, C.POINTER(LevelInfo)]
    L.mlmc_workspace_bytes.argtypes = [vp, C.c_int, C.c_uint64, C.POINTER(C.c_size_t)]
    L.mlmc_workspace_bytes_prec.argtypes = [vp, C.c_int, C.c_uint64, C.POINTER(Precision), C.POINTER(Precision),
                                            C.POINTER(C.c_size_t)]
    L.mlmc_bind_workspace.argtypes = [vp, vp, C.c_size_t, vp]
    L.mlmc_sample_level.argtypes = [vp, C.c_int, C.c_uint64, C.c_uint64, C.c_uint64, C.POINTER(Precision),
                                    C.POINTER(Precision), C.c_double, C.c_double, C.POINTER(LevelSums), vp]
    L.mlmc_sample_level_async.argtypes = [vp, C.c_int, C.c_uint64, C.c_uint64, C.c_uint64, C.POINTER(Precision),
                                          C.POINTER(Precision), C.c_double, C.c_double, vp, vp]
    L.mlmc_adaptive_run.argtypes = [vp, C.c_double, C.POINTER(AdaptiveOpts), ALLREDUCE_FN, vp, C.POINTER(Result)]
    L.mlmc_auto_choice.argtypes = [vp, C.c_int, C.POINTER(Precision), dp]
    L.mlmc_auto_choice_set.argtypes = [vp, C.c_int, C.c_int, C.POINTER(Precision)]
    L.mlmc_eps_schedule.argtypes = [C.c_int, C.c_double, C.c_double, dp]
    L.mlmc_optimal_samples.argtypes = [C.c_int, dp, dp, C.c_double, dp]
    L.mlmc_kl_modes.argtypes = [C.c_double, C.c_double, C.c_int, C.POINTER(C.c_int32), C.POINTER(C.c_int32), dp, dp,
                                C.c_int]
    L.mlmc_debug_field.argtypes = [vp, C.c_int, C.c_int, C.c_uint64, C.c_uint64, C.c_uint64, vp, vp]
    L.mlmc_debug_trace.argtypes = [vp, vp, C.c_uint32, C.POINTER(C.c_uint32)]
    L.mlmc_sample_level_xi.argtypes = [vp, C.c_int, C.c_uint64, vp, C.POINTER(Precision), C.POINTER(Precision),
                                       C.c_double, C.c_double, C.POINTER(LevelSums), vp]
    L.mlmc_sample_levels_xi.argtypes = [vp, C.c_int, C.POINTER(C.c_int), C.POINTER(C.c_uint64), C.POINTER(vp),
                                        C.POINTER(Precision), C.POINTER(Precision), dp, dp, C.POINTER(LevelSums),
                                        C.POINTER(vp)]
    L.mlmc_sample_levels_async.argtypes = [vp, C.c_int, C.POINTER(C.c_int), C.POINTER(C.c_uint64), C.c_uint64,
                                           C.POINTER(C.c_uint64), C.POINTER(Precision), C.POINTER(Precision), dp, dp,
                                           vp]
    L.mlmc_adaptive_run_host.argtypes = [C.c_int, C.c_int, C.c_double, C.POINTER(AdaptiveOpts), LEVEL_SAMPLER_FN, vp,
                                         ALLREDUCE_FN, vp, C.POINTER(Result)]
    L.mlmc_profile_enable.argtypes = [vp, C.c_int]
    L.mlmc_profile_read.argtypes = [vp, C.POINTER(KernelStat), C.c_int, C.POINTER(C.c_int)]
    L.mlmc_dd_layout_get.argtypes = [C.c_int, C.c_int, C.c_int, C.c_int, C.POINTER(DDLayout)]
    L.mlmc_dd_exchange_rows.argtypes = [C.POINTER(DDLayout), C.c_int, C.POINTER(C.c_int64)]
    L.mlmc_dd_create.argtypes = [vp, C.c_int, C.c_int, C.c_int, vp, C.c_size_t, C.POINTER(vp)]
    L.mlmc_dd_begin.argtypes = [vp, C.c_uint64, C.c_int, C.c_uint64, C.c_double, C.c_int]
    L.mlmc_dd_pass.argtypes = [vp]
    L.mlmc_dd_scalar.argtypes = [vp]
    L.mlmc_dd_result.argtypes = [vp, dp]
    L.mlmc_dd_run_local.argtypes = [vp, dp]
    L.mlmc_dd_run_peer.argtypes = [vp, C.POINTER(vp), dp]
    L.mlmc_dd_run_emulated.argtypes = [C.POINTER(vp), C.c_int, dp]
    L.mlmc_dd_ipc_handle.argtypes = [vp, C.c_char_p, C.POINTER(C.c_uint64)]
    L.mlmc_dd_ipc_open.argtypes = [vp, C.c_char_p, C.c_uint64, C.POINTER(vp), C.POINTER(vp)]
    L.mlmc_dd_ipc_close.argtypes = [vp, vp]
    L.mlmc_dd_destroy.argtypes = [vp]
    L.mlmc_dd_destroy.restype = None
    _lib = L
    return L


def check(rc: int, ctx=None):
    if rc != MLMC_OK:
        msg = lib().mlmc_last_error(ctx).decode() if ctx is not None else ""
        raise RuntimeError(f"mlmc error {rc} ({lib().mlmc_strerror(rc).decode()}): {msg}")
