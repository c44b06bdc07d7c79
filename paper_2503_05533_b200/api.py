"""Thin Python binding of the MPML C-ABI (include/mlmc.h).

Argument marshalling only: every step of the hot path runs in libmlmc.so's
sm_100a kernels.  PyTorch supplies device memory (the workspace), the CUDA
stream and, for multi-rank runs, the torch.distributed process group that
carries the per-round all-reduce of the level sums.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass
from typing import Optional

import numpy as np

from . import _capi as K

__all__ = ["Context", "precision", "mlmc_plan_levels", "mlmc_sample_level", "mlmc_sample_level_async",
           "mlmc_adaptive_run", "mlmc_eps_schedule", "mlmc_optimal_samples", "mlmc_kl_modes",
           "mlmc_debug_field", "mlmc_workspace_bytes", "SUM_FIELDS"]

SUM_FIELDS = ("sum_y", "sum_y2", "sum_qf", "sum_qc", "sum_cost", "n", "n_fail", "iters_f", "iters_c",
              "iters_f_max", "iters_c_max", "n_escalated")


def precision(solver: str = "minres", u_f: str = "s", u_s: str = "s", u: str = "d", u_r: str = "d",
              max_iter: int = 0, verify: bool = False, escalate: bool = False, c2f: bool = False) -> K.Precision:
    """MINRES (all binary64) or Cholesky-IR with Algorithm 1's quad.
    verify=True (MINRES): also carry x_k and report the true residual; escalate=True (MINRES, IR): a failed solve
    is solved again by MG-PCG (status 4 when that converges); c2f=True (on prec_fine, MINRES): the fine half starts
    from the P1 interpolation of the coarse half's solution (MLMC_FLAG_C2F, NEXT-4)."""
    s = {"minres": K.SOLVER_MINRES, "chol_ir": K.SOLVER_CHOL_IR, "ir": K.SOLVER_CHOL_IR, "mgcg": K.SOLVER_MGCG, "cg": K.SOLVER_CG}[solver]
    flags = (K.FLAG_VERIFY if verify else 0) | (K.FLAG_ESCALATE if escalate else 0) | (K.FLAG_C2F if c2f else 0)
    return K.Precision(s, K.FMT[u_f], K.FMT[u_s], K.FMT[u], K.FMT[u_r], max_iter, flags)


def _as_prec(p) -> K.Precision:
    if p is None:
        return precision("minres")
    if isinstance(p, K.Precision):
        return p
    if isinstance(p, str):
        if p in ("minres", "mgcg"):
            return precision(p)
        # quad string like "hsdd": Cholesky-IR (u_f, u_s, u, u_r)
        return precision("chol_ir", p[0], p[1], p[2], p[3])
    raise TypeError(p)


@dataclass
class LevelResult:
    sums: dict
    per_sample: Optional[np.ndarray]


class Context:
    """One mlmc_ctx on one device: plan + borrowed torch workspace + stream."""

    def __init__(self, field: str = "expcov", m: int = 16, sigma2: float = 1.0, corr_len: float = 0.3,
                 q_decay: float = 2.0, h0_inv: int = 8, L_max: int = 1, device: int = 0,
                 workspace_bytes: int = 1 << 30, stream=None):
        import torch
        self._torch = torch
        L = K.lib()
        f = {"expcov": K.FIELD_EXPCOV_KL, "eq20": K.FIELD_PAPER_EQ20}[field]
        self.problem = K.Problem(f, m, sigma2, corr_len, q_decay, h0_inv, 2, L_max, device)
        ctx = C.c_void_p()
        K.check(L.mlmc_plan_levels(C.byref(self.problem), C.byref(ctx)))
        self.ctx = ctx
        self.device = torch.device("cuda", device)
        self.m = m
        self.L_max = L_max
        self.h0_inv = h0_inv
        self.ws = torch.empty(int(workspace_bytes), dtype=torch.uint8, device=self.device)
        self.stream = stream if stream is not None else torch.cuda.current_stream(self.device)
        K.check(L.mlmc_bind_workspace(ctx, C.c_void_p(self.ws.data_ptr()), C.c_size_t(self.ws.numel()),
                                      C.c_void_p(self.stream.cuda_stream)), ctx)
        self._sums_dev = torch.zeros(K.MLMC_SUMS_LEN, dtype=torch.float64, device=self.device)

    def close(self):
        if getattr(self, "ctx", None):
            K.lib().mlmc_destroy(self.ctx)
            self.ctx = None

    __del__ = close

    def level_info(self, level: int) -> dict:
        li = K.LevelInfo()
        K.check(K.lib().mlmc_level_info_get(self.ctx, level, C.byref(li)), self.ctx)
        return {"N": li.N, "n": li.n, "P": li.P, "bw": li.bw, "h": li.h}

    def workspace_bytes(self, level: int, batch: int) -> int:
        out = C.c_size_t()
        K.check(K.lib().mlmc_workspace_bytes(self.ctx, level, batch, C.byref(out)), self.ctx)
        return out.value

    def workspace_bytes_prec(self, level: int, batch: int, prec_fine="minres", prec_coarse=None) -> int:
        """mlmc_workspace_bytes_prec: includes the Cholesky-IR factor scratch of the given precisions."""
        pf = _as_prec(prec_fine)
        pc = _as_prec(prec_coarse if prec_coarse is not None else prec_fine)
        out = C.c_size_t()
        K.check(K.lib().mlmc_workspace_bytes_prec(self.ctx, level, batch, C.byref(pf), C.byref(pc), C.byref(out)),
                self.ctx)
        return out.value

    # ------------------------------------------------------------------ hot path
    def sample_level(self, level: int, n: int, seed: int, first_index: int = 0, prec_fine="minres",
                     prec_coarse=None, tol_fine: float = 1e-8, tol_coarse: Optional[float] = None,
                     per_sample=False) -> LevelResult:
        """mlmc_sample_level: host sums (+ optional per-sample records, host numpy or device tensor)."""
        pf = _as_prec(prec_fine)
        pc = _as_prec(prec_coarse if prec_coarse is not None else prec_fine)
        tc = tol_coarse if tol_coarse is not None else tol_fine
        sums = K.LevelSums()
        ps = None
        ptr = None
        if per_sample is True or per_sample == "host":
            ps = np.zeros((n, K.MLMC_SAMPLE_LEN), np.float64)
            ptr = C.c_void_p(ps.ctypes.data) if n else None
        elif per_sample == "device":
            ps = self._torch.zeros((n, K.MLMC_SAMPLE_LEN), dtype=self._torch.float64, device=self.device)
            ptr = C.c_void_p(ps.data_ptr()) if n else None
        rc = K.lib().mlmc_sample_level(self.ctx, level, n, seed, first_index, C.byref(pf), C.byref(pc), tol_fine, tc,
                                       C.byref(sums), ptr)
        K.check(rc, self.ctx)
        return LevelResult({f: getattr(sums, f) for f in SUM_FIELDS}, ps)

    def sample_level_async(self, level: int, n: int, seed: int, first_index: int = 0, prec_fine="minres",
                           prec_coarse=None, tol_fine: float = 1e-8, tol_coarse: Optional[float] = None,
                           sums_out=None, per_sample_out=None):
        """mlmc_sample_level_async: enqueue on the bound stream; sums land in a device tensor."""
        pf = _as_prec(prec_fine)
        pc = _as_prec(prec_coarse if prec_coarse is not None else prec_fine)
        tc = tol_coarse if tol_coarse is not None else tol_fine
        out = sums_out if sums_out is not None else self._sums_dev
        rc = K.lib().mlmc_sample_level_async(self.ctx, level, n, seed, first_index, C.byref(pf), C.byref(pc),
                                             tol_fine, tc, C.c_void_p(out.data_ptr()),
                                             C.c_void_p(per_sample_out.data_ptr()) if per_sample_out is not None
                                             else None)
        K.check(rc, self.ctx)
        return out

    def sample_levels_async(self, levels, n, seed: int, first_index, prec_fine, prec_coarse, tol_fine, tol_coarse,
                            sums_out):
        """mlmc_sample_levels_async: all listed levels concurrently; sums_out is a device tensor
        [len(levels), 12] (row q = levels[q])."""
        k = len(levels)
        pf = (K.Precision * k)(*[_as_prec(p) for p in prec_fine])
        pc = (K.Precision * k)(*[_as_prec(p) for p in prec_coarse])
        rc = K.lib().mlmc_sample_levels_async(self.ctx, k, (C.c_int * k)(*levels), (C.c_uint64 * k)(*n), seed,
                                              (C.c_uint64 * k)(*first_index), pf, pc, (C.c_double * k)(*tol_fine),
                                              (C.c_double * k)(*tol_coarse), C.c_void_p(sums_out.data_ptr()))
        K.check(rc, self.ctx)
        return sums_out

    def sample_level_xi(self, level: int, xi, prec_fine="minres", prec_coarse=None, tol_fine: float = 1e-8,
                        tol_coarse: Optional[float] = None, per_sample=None) -> LevelResult:
        """mlmc_sample_level_xi: caller-supplied standard normals xi [n, m] (host numpy / pinned torch
        tensor, or a device tensor) instead of the Philox draw.  per_sample: None, a host buffer
        (numpy / pinned tensor, [n, 8] float64) or a device tensor, filled in place."""
        pf = _as_prec(prec_fine)
        pc = _as_prec(prec_coarse if prec_coarse is not None else prec_fine)
        tc = tol_coarse if tol_coarse is not None else tol_fine
        n = int(xi.shape[0])
        xptr = xi.ctypes.data if isinstance(xi, np.ndarray) else xi.data_ptr()
        pptr = None
        if per_sample is not None:
            pptr = per_sample.ctypes.data if isinstance(per_sample, np.ndarray) else per_sample.data_ptr()
        sums = K.LevelSums()
        K.check(K.lib().mlmc_sample_level_xi(self.ctx, level, n, C.c_void_p(xptr), C.byref(pf), C.byref(pc),
                                             tol_fine, tc, C.byref(sums), C.c_void_p(pptr) if pptr else None),
                self.ctx)
        return LevelResult({f: getattr(sums, f) for f in SUM_FIELDS}, per_sample)

    def sample_levels_xi(self, levels, xis, prec_fine, prec_coarse, tol_fine, tol_coarse, per_sample=None) -> list:
        """mlmc_sample_levels_xi: all listed levels concurrently from caller-supplied normals xis[q] [n_q, m]
        (host numpy / pinned tensors or device tensors); per_sample: None or a list of host / device
        [n_q, 8] float64 buffers filled in place.  Returns one sums dict per entry."""
        k = len(levels)
        ptr = lambda a: a.ctypes.data if isinstance(a, np.ndarray) else a.data_ptr()
        xs = (C.c_void_p * k)(*[ptr(x) for x in xis])
        ps = (C.c_void_p * k)(*[ptr(p) if p is not None else None for p in (per_sample or [None] * k)])
        pf = (K.Precision * k)(*[_as_prec(p) for p in prec_fine])
        pc = (K.Precision * k)(*[_as_prec(p) for p in prec_coarse])
        sums = (K.LevelSums * k)()
        rc = K.lib().mlmc_sample_levels_xi(self.ctx, k, (C.c_int * k)(*levels),
                                           (C.c_uint64 * k)(*[int(x.shape[0]) for x in xis]), xs, pf, pc,
                                           (C.c_double * k)(*tol_fine), (C.c_double * k)(*tol_coarse), sums, ps)
        K.check(rc, self.ctx)
        return [{f: getattr(sums[q], f) for f in SUM_FIELDS} for q in range(k)]

    def profile_enable(self, on: bool = True):
        K.check(K.lib().mlmc_profile_enable(self.ctx, 1 if on else 0), self.ctx)

    def profile_read(self) -> list:
        """[(kind, N, launches, ms)] per kernel class since profile_enable (synchronises the stream)."""
        arr = (K.KernelStat * 64)()
        cnt = C.c_int()
        K.check(K.lib().mlmc_profile_read(self.ctx, arr, 64, C.byref(cnt)), self.ctx)
        return [(K.KERNEL_KINDS.get(s.kind, str(s.kind)), s.N, s.launches, s.ms) for s in arr[:min(cnt.value, 64)]]

    def debug_field(self, level: int, mesh_level: int, n: int, seed: int, first_index: int = 0):
        """mlmc_debug_field: (xi [n, m], a [n, 2N^2]) device tensors."""
        t = self._torch
        N = self.h0_inv << mesh_level
        xi = t.zeros((max(n, 1), self.m), dtype=t.float64, device=self.device)
        a = t.zeros((max(n, 1), 2 * N * N), dtype=t.float64, device=self.device)
        K.check(K.lib().mlmc_debug_field(self.ctx, level, mesh_level, n, seed, first_index,
                                         C.c_void_p(xi.data_ptr()), C.c_void_p(a.data_ptr())), self.ctx)
        return xi[:n], a[:n]

    def auto_choice(self, N: int):
        """mlmc_auto_choice: the solver / precision policy 3 chose for mesh N (= 1/h), or None."""
        p = K.Precision()
        ms = C.c_double()
        if K.lib().mlmc_auto_choice(self.ctx, N, C.byref(p), C.byref(ms)) != K.MLMC_OK:
            return None
        fmt = "qhsd"
        name = {K.SOLVER_MINRES: "minres", K.SOLVER_CHOL_IR: "chol_ir", K.SOLVER_MGCG: "mgcg", K.SOLVER_CG: "cg"}[p.solver]
        quad = "".join(fmt[v] for v in (p.u_f, p.u_s, p.u, p.u_r)) if p.solver == K.SOLVER_CHOL_IR else None
        return {"solver": name, "quad": quad, "ms_per_sample": ms.value}

    def auto_choice_set(self, N: int, tol_class: int, prec) -> None:
        """mlmc_auto_choice_set: record policy 3's choice for mesh N and tolerance class (0: tol >= 1e-3,
        1: >= 1e-5, 2: below) so that a run reproduces recorded decisions without pilot timings."""
        p = _as_prec(prec)
        K.check(K.lib().mlmc_auto_choice_set(self.ctx, N, tol_class, C.byref(p)), self.ctx)

    def adaptive_run(self, eps: float, k_p: float = 0.05, N_init: int = 100, policy: int = 0, seed: int = 0,
                     fixed_tol: float = 1e-10, r_bias: float = 1.0, max_rounds: int = 100, group=None,
                     on_fail: int = 0) -> dict:
        """mlmc_adaptive_run (Algorithm 2).  With a torch.distributed group the per-round level sums are
        all-reduced through it (NCCL on GPU tensors, gloo on CPU tensors); group=None runs locally."""
        rank, world, cb = _allreduce_callback(group, self.device)
        opts = K.AdaptiveOpts(k_p, fixed_tol, r_bias, N_init, policy, rank, world, max_rounds, seed, on_fail, 0)
        res = K.Result()
        rc = K.lib().mlmc_adaptive_run(self.ctx, eps, C.byref(opts), cb, None, C.byref(res))
        if rc not in (K.MLMC_OK, K.MLMC_ELMAX):
            K.check(rc, self.ctx)
        return _result_dict(res)


def _result_dict(res) -> dict:
    L = res.L
    return {"estimate": res.estimate, "L": L, "rounds": res.rounds, "code": res.code, "n_fail": res.n_fail,
            "N": list(res.N[:L + 1]), "eps": list(res.eps[:L + 1]), "mean": list(res.mean[:L + 1]),
            "var": list(res.var[:L + 1]), "cost": list(res.cost[:L + 1]), "solve_seconds": res.solve_seconds}


def _allreduce_callback(group, device):
    """(rank, world, mlmc_allreduce_fn) for the torch.distributed group; group=None is a local run (world 1)
    even when a default process group exists -- a multi-rank run names its group explicitly, so that a call
    made by one rank alone (e.g. rank 0's extra measurements in bench.py) never waits on the others.  NCCL
    groups reduce a tensor on `device`, others (gloo) on the CPU."""
    import torch as t
    if group is None:
        return 0, 1, K.ALLREDUCE_FN(0)
    import torch.distributed as dist
    rank, world = dist.get_rank(group), dist.get_world_size(group)
    dev = device if dist.get_backend(group) == "nccl" else t.device("cpu")

    # persistent staging: one pinned host buffer and one buffer on the collective's device, grown on demand, so a
    # round's exchange is two copies and ONE all-reduce (the controller sends everything in one SUM call)
    bufs = {}

    def _staging(count):
        if bufs.get("n", 0) < count:
            n = max(count, 2 * bufs.get("n", 0), 256)
            pin = dev.type == "cuda"
            bufs["h"] = t.empty(n, dtype=t.float64, pin_memory=pin)
            bufs["d"] = t.empty(n, dtype=t.float64, device=dev) if pin else bufs["h"]
            bufs["n"] = n
        return bufs["h"][:count], bufs["d"][:count]

    def _allreduce(buf, count, op, user):
        try:
            arr = np.ctypeslib.as_array(buf, shape=(count,))
            h, d = _staging(count)
            h.numpy()[:] = arr
            if d is not h:
                d.copy_(h, non_blocking=True)
            dist.all_reduce(d, op=dist.ReduceOp.SUM if op == 0 else dist.ReduceOp.MAX, group=group)
            if d is not h:
                h.copy_(d)
            arr[:] = h.numpy()
            return 0
        except Exception:  # noqa: BLE001 -- reported to the C side as a failure
            return 1

    return rank, world, K.ALLREDUCE_FN(_allreduce)


def mlmc_adaptive_run_host(h0_inv: int, L_max: int, eps: float, sampler, k_p: float = 0.05, N_init: int = 100,
                           policy: int = 0, seed: int = 0, fixed_tol: float = 1e-10, r_bias: float = 1.0,
                           max_rounds: int = 100, group=None, on_fail: int = 0) -> dict:
    """The library's Algorithm 2 over a host sampler (no GPU): ``sampler(level, n, first_index, prec_fine,
    prec_coarse, tol_fine, tol_coarse) -> 12 level sums``.  Used by the CPU tests of the controller and
    of the multi-rank exchange (gloo)."""
    rank, world, cb = _allreduce_callback(group, None)

    def _cb(level, n, first, pf, pc, tf, tc, sums, user):
        try:
            out = sampler(level, int(n), int(first), pf.contents, pc.contents, tf, tc)
            for k in range(K.MLMC_SUMS_LEN):
                sums[k] = float(out[k])
            return 0
        except Exception:  # noqa: BLE001
            import traceback
            traceback.print_exc()
            return 1

    scb = K.LEVEL_SAMPLER_FN(_cb)
    opts = K.AdaptiveOpts(k_p, fixed_tol, r_bias, N_init, policy, rank, world, max_rounds, seed, on_fail, 0)
    res = K.Result()
    rc = K.lib().mlmc_adaptive_run_host(h0_inv, L_max, eps, C.byref(opts), scb, None, cb, None, C.byref(res))
    if rc not in (K.MLMC_OK, K.MLMC_ELMAX):
        K.check(rc)
    return _result_dict(res)


# ---------------------------------------------------------------------- C-ABI names
def mlmc_plan_levels(**problem) -> Context:
    return Context(**problem)


def mlmc_sample_level(ctx: Context, *a, **k) -> LevelResult:
    return ctx.sample_level(*a, **k)


def mlmc_sample_level_async(ctx: Context, *a, **k):
    return ctx.sample_level_async(*a, **k)


def mlmc_adaptive_run(ctx: Context, eps: float, **k) -> dict:
    return ctx.adaptive_run(eps, **k)


def mlmc_debug_field(ctx: Context, *a, **k):
    return ctx.debug_field(*a, **k)


def mlmc_workspace_bytes(ctx: Context, level: int, batch: int) -> int:
    return ctx.workspace_bytes(level, batch)


def mlmc_eps_schedule(L: int, h0: float, k_p: float) -> list:
    out = (C.c_double * (L + 1))()
    K.check(K.lib().mlmc_eps_schedule(L, h0, k_p, out))
    return list(out)


def mlmc_optimal_samples(V, Cst, tol: float) -> list:
    n = len(V)
    v = (C.c_double * n)(*V)
    c = (C.c_double * n)(*Cst)
    out = (C.c_double * n)()
    K.check(K.lib().mlmc_optimal_samples(n, v, c, tol, out))
    return list(out)


def mlmc_kl_modes(sigma2: float, corr_len: float, m: int, nroots: int = 0):
    ik = (C.c_int32 * m)()
    jk = (C.c_int32 * m)()
    lam = (C.c_double * m)()
    w = (C.c_double * max(nroots, 1))()
    K.check(K.lib().mlmc_kl_modes(sigma2, corr_len, m, ik, jk, lam, w, nroots))
    return np.array(ik), np.array(jk), np.array(lam), np.array(w[:nroots])
