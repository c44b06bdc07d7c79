"""K3d binding and host driver: MINRES of ONE sample over row slabs (include/mlmc.h "K3d"; SURVEY 8(f)
NEXT-3).  Argument marshalling and the exchange schedule only -- every step of the solve runs in
libmlmc.so (dd_pass_kernel, dd_scalar_kernel); torch.distributed carries the per-step all-reduce of three
doubles and the one-row halo exchange with each neighbour (NCCL over NVLink on GPUs).

    lay = layout(N, m, rank, world)          # host: partition + workspace layout (mlmc_dd_layout_get)
    s = SlabSolver(ctx, mesh_level, rank, world); s.begin(seed, level, index, tol)
    Q, iters, relres, status = dd_solve(s, group)          # world ranks, one slab each
    Q, ... = s.run_local()                                  # world = 1: whole GPU on one system
"""
from __future__ import annotations

import ctypes as C

from . import _capi as K


def layout(N: int, m: int, rank: int, world: int) -> K.DDLayout:
    lay = K.DDLayout()
    K.check(K.lib().mlmc_dd_layout_get(N, m, rank, world, C.byref(lay)))
    return lay


def exchange_rows(lay: K.DDLayout, step: int) -> list:
    """Byte offsets [send to rank-1, receive from rank-1, send to rank+1, receive from rank+1] (-1: none)."""
    offs = (C.c_int64 * 4)()
    K.check(K.lib().mlmc_dd_exchange_rows(C.byref(lay), step, offs))
    return list(offs)


class SlabSolver:
    """One rank's slab of one system on the device (mlmc_dd_*); the workspace is a torch tensor."""

    def __init__(self, ctx, mesh_level: int, rank: int = 0, world: int = 1):
        import torch
        self.ctx = ctx
        N = ctx.h0_inv << mesh_level
        self.lay = layout(N, ctx.m, rank, world)
        self.rank, self.world = rank, world
        self.ws = torch.zeros(int(self.lay.bytes), dtype=torch.uint8, device=ctx.device)
        dd = C.c_void_p()
        K.check(K.lib().mlmc_dd_create(ctx.ctx, mesh_level, rank, world, C.c_void_p(self.ws.data_ptr()),
                                       C.c_size_t(self.ws.numel()), C.byref(dd)), ctx.ctx)
        self.dd = dd
        self.sums = self.ws[self.lay.sums_off:self.lay.sums_off + 24].view(torch.float64)

    def row(self, off: int):
        return self.ws[off:off + 8 * self.lay.pitch].view(self._dtype())

    def _dtype(self):
        import torch
        return torch.float64

    def begin(self, seed: int, level: int, index: int, tol: float, max_iter: int = 0):
        K.check(K.lib().mlmc_dd_begin(self.dd, seed, level, index, tol, max_iter), self.ctx.ctx)

    def pass_(self):
        K.check(K.lib().mlmc_dd_pass(self.dd), self.ctx.ctx)

    def scalar(self):
        K.check(K.lib().mlmc_dd_scalar(self.dd), self.ctx.ctx)

    def exchange_offsets(self, step: int) -> list:
        return exchange_rows(self.lay, step)

    def result(self) -> dict:
        out = (C.c_double * 5)()
        K.check(K.lib().mlmc_dd_result(self.dd, out), self.ctx.ctx)
        return {"Q": out[0], "iters": int(out[1]), "relres": out[2], "status": int(out[3]), "done": bool(out[4])}

    def done(self) -> bool:
        return self.result()["done"]

    def run_local(self) -> dict:
        out = (C.c_double * 5)()
        K.check(K.lib().mlmc_dd_run_local(self.dd, out), self.ctx.ctx)
        return {"Q": out[0], "iters": int(out[1]), "relres": out[2], "status": int(out[3]), "done": bool(out[4])}

    def run_peer(self, peer_ptrs) -> dict:
        """mlmc_dd_run_peer: this rank's part of the fused-exchange solve; peer_ptrs[q] = rank q's workspace as
        mapped on this device (every rank calls it after every rank's begin())."""
        arr = (C.c_void_p * len(peer_ptrs))(*[C.c_void_p(int(p)) for p in peer_ptrs])
        out = (C.c_double * 5)()
        K.check(K.lib().mlmc_dd_run_peer(self.dd, arr, out), self.ctx.ctx)
        return {"Q": out[0], "iters": int(out[1]), "relres": out[2], "status": int(out[3]), "done": bool(out[4])}

    def ipc_handle(self):
        """(64-byte CUDA IPC handle of this workspace's allocation, byte offset of the workspace in it)."""
        h = C.create_string_buffer(64)
        off = C.c_uint64()
        K.check(K.lib().mlmc_dd_ipc_handle(self.dd, h, C.byref(off)), self.ctx.ctx)
        return h.raw, off.value

    def ipc_open(self, handle: bytes, offset: int):
        """A peer's workspace mapped on this device: (pointer, mapping base for ipc_close)."""
        ptr, base = C.c_void_p(), C.c_void_p()
        K.check(K.lib().mlmc_dd_ipc_open(self.ctx.ctx, handle, offset, C.byref(ptr), C.byref(base)), self.ctx.ctx)
        return ptr.value, base.value

    def ipc_close(self, base: int):
        K.check(K.lib().mlmc_dd_ipc_close(self.ctx.ctx, C.c_void_p(base)), self.ctx.ctx)

    def close(self):
        if getattr(self, "dd", None):
            K.lib().mlmc_dd_destroy(self.dd)
            self.dd = None

    __del__ = close


def dd_solve(engine, group=None, check_every: int = 32, max_steps: int = 10 ** 7) -> dict:
    """One rank's side of a slab-decomposed solve: per MINRES step pass -> all-reduce(SUM) of the three
    partial sums + one-row halo exchange with each neighbour -> scalar step.  Every rank decides `done` from
    identical reduced sums at the same step, so all leave the loop together.  `engine` is a SlabSolver (or any
    object with its interface: pass_, scalar, sums, row, exchange_offsets, result, rank, world)."""
    import torch.distributed as dist
    world, rank = engine.world, engine.rank
    # NCCL moves the device rows and sums directly (NVLink); a CPU backend (gloo: tests, or several processes
    # sharing one GPU) goes through host staging copies of the same rows
    staged = world > 1 and dist.get_backend(group) != "nccl" and engine.sums.device.type == "cuda"
    if staged:
        import torch
        h_sums = torch.empty(3, dtype=torch.float64)
        h_rows = [torch.empty(engine.lay.pitch, dtype=torch.float64) for _ in range(4)]
    for step in range(max_steps):
        engine.pass_()
        if world > 1:
            o = engine.exchange_offsets(step)
            if staged:
                h_sums.copy_(engine.sums)
                dist.all_reduce(h_sums, group=group)
                engine.sums.copy_(h_sums)
                send = {0: o[0], 2: o[2]}
                for q, off in send.items():
                    if off >= 0:
                        h_rows[q].copy_(engine.row(off))
                bufs = {q: h_rows[q] for q in range(4)}
            else:
                dist.all_reduce(engine.sums, group=group)
                bufs = {q: engine.row(o[q]) if o[q] >= 0 else None for q in range(4)}
            ops = []
            if o[0] >= 0:
                ops.append(dist.P2POp(dist.isend, bufs[0], rank - 1, group))
                ops.append(dist.P2POp(dist.irecv, bufs[1], rank - 1, group))
            if o[2] >= 0:
                ops.append(dist.P2POp(dist.isend, bufs[2], rank + 1, group))
                ops.append(dist.P2POp(dist.irecv, bufs[3], rank + 1, group))
            for r in dist.batch_isend_irecv(ops):
                r.wait()
            if staged:
                for q in (1, 3):
                    if o[q] >= 0:
                        engine.row(o[q]).copy_(h_rows[q])
        engine.scalar()
        if (step + 1) % check_every == 0 and engine.done():
            break
    return engine.result()


def dd_solve_peer(engine, group=None) -> dict:
    """One rank of the fused-exchange solve on a multi-GPU node (one process per GPU, every rank calls it after its
    begin()): the workspaces are peer-mapped with CUDA IPC (handles exchanged over torch.distributed), then ONE
    kernel per rank runs the whole solve, the ranks exchanging halo rows and partial sums through NVLink stores
    and system-scope flags (mlmc_dd_run_peer).  Ranks must sit on distinct GPUs: they wait on one another inside
    the kernel (on one GPU use dd_run_fused_emulated)."""
    import torch.distributed as dist
    world, rank = engine.world, engine.rank
    mine = engine.ipc_handle()
    allh = [None] * world
    dist.all_gather_object(allh, mine, group=group)
    ptrs, bases = [], []
    for q in range(world):
        if q == rank:
            ptrs.append(engine.ws.data_ptr())
        else:
            p, b = engine.ipc_open(*allh[q])
            ptrs.append(p)
            bases.append(b)
    engine.result()                            # this rank's begin() (planes, zeroed counters) is on the GPU ...
    dist.barrier(group=group)                  # ... on every rank, before any rank's kernel stores into it
    try:
        return engine.run_peer(ptrs)
    finally:
        dist.barrier(group=group)              # nobody unmaps while a peer may still store into it
        for b in bases:
            engine.ipc_close(b)


def dd_run_fused_emulated(engines: list) -> dict:
    """All ranks of one solve (SlabSolvers of one ctx, engines[q] = rank q) in ONE cooperative launch of the
    fused-exchange kernel (mlmc_dd_run_emulated): the peer-memory exchange of a multi-GPU run, on one GPU."""
    arr = (C.c_void_p * len(engines))(*[e.dd for e in engines])
    out = (C.c_double * 5)()
    K.check(K.lib().mlmc_dd_run_emulated(arr, len(engines), out), engines[0].ctx.ctx)
    return {"Q": out[0], "iters": int(out[1]), "relres": out[2], "status": int(out[3]), "done": bool(out[4])}


def dd_solve_emulated(engines: list, check_every: int = 32, max_steps: int = 10 ** 7) -> dict:
    """All ranks of one solve in one process (e.g. G slabs on one GPU): the all-reduce is the sum of the
    ranks' partials in rank order, the halo rows are copied between the slabs' workspaces.  Same kernels and
    exchange schedule as dd_solve; no launch waits on another (the host orders them)."""
    G = len(engines)
    for step in range(max_steps):
        for e in engines:
            e.pass_()
        if G > 1:
            tot = engines[0].sums.clone()
            for e in engines[1:]:
                tot += e.sums
            for e in engines:
                e.sums.copy_(tot)
            offs = [e.exchange_offsets(step) for e in engines]
            for g in range(G - 1):          # rank g <-> rank g+1
                engines[g + 1].row(offs[g + 1][1]).copy_(engines[g].row(offs[g][2]))
                engines[g].row(offs[g][3]).copy_(engines[g + 1].row(offs[g + 1][0]))
        for e in engines:
            e.scalar()
        if (step + 1) % check_every == 0 and engines[0].done():
            break
    return [e.result() for e in engines]
