"""K3d (NEXT-3, domain-decomposed MINRES of one sample) on the GPU (-m gpu).

One B200 runs every rank: G slabs of one system in one process (paper_2503_05533_b200.dd.dd_solve_emulated:
the all-reduce is the rank-order sum of the slabs' partials, the halo rows are device copies between the
slab workspaces; launches never wait on one another).  The kernels, layouts and exchange schedule are the
multi-GPU ones (dd_solve over NCCL differs only in who moves the rows).

Checks against the oracle (configs[4] field): Q within the per-sample residual bound of the binary64 direct
solve; G = 1 / 2 / 3 / 4 agree with each other to rounding and with the streamed MINRES (K3c) of the same
sample within both solves' bounds; iteration counts within 1% of K3c's; max_iter exhaustion is reported.
"""
import time

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

from oracle import core as oc  # noqa: E402
from paper_2503_05533_b200 import Context, precision  # noqa: E402
from paper_2503_05533_b200.dd import SlabSolver, dd_solve_emulated, layout  # noqa: E402
import workloads as W  # noqa: E402


@pytest.fixture(scope="module", autouse=True)
def built():
    import __graft_entry__
    __graft_entry__.build()


def _ctx(ws=4 << 30):
    cfg = W.CONFIGS["C5"]
    return cfg, Context(field=cfg["field"], m=cfg["m"], sigma2=cfg["sigma2"], corr_len=cfg["corr_len"],
                        h0_inv=cfg["h0_inv"], L_max=cfg["L_max"], device=0, workspace_bytes=ws)


def _exact(cfg, N, seed, level, k):
    P = oc.OracleProblem(0, cfg["m"], cfg["sigma2"], cfg["corr_len"], 2.0, cfg["h0_inv"])
    a = P.field_triangles(N, oc.normals(seed, level, k, cfg["m"]))
    AB, _, b = oc.assemble(N, a)
    x, _ = oc.chol_band_solve(AB, b)
    return x.sum() / N ** 2, np.linalg.norm(b), np.linalg.norm(x)


def _solve(ctx, mesh_level, G, seed, level, k, tol, max_iter=0):
    engines = [SlabSolver(ctx, mesh_level, g, G) for g in range(G)]
    for e in engines:
        e.begin(seed, level, k, tol, max_iter)
    if G == 1:
        res = [engines[0].run_local()]
    else:
        res = dd_solve_emulated(engines)
    for e in engines:
        e.close()
    return res


def test_dd_h256_matches_oracle_and_k3c():
    """h = 1/256 (configs[4] level 5, fine half): G = 1, 2, 3 slabs vs the oracle's direct solve and K3c."""
    cfg, ctx = _ctx()
    seed, level, k, tol = 41, 5, 2, 1e-10
    q, bn, xn = _exact(cfg, 256, seed, level, k)
    ref = ctx.sample_level(level, 1, seed=seed, first_index=k, prec_fine=precision("minres"), tol_fine=tol,
                           tol_coarse=tol, per_sample=True).per_sample[0]
    out = {}
    for G in (1, 2, 3):
        res = _solve(ctx, level, G, seed, level, k, tol)
        assert all(r == res[0] for r in res)                     # every rank holds the same result
        r = res[0]
        assert r["done"] and r["status"] == 0 and r["relres"] <= tol
        assert abs(r["Q"] - q) <= tol * bn * xn * (1 + 1e-6) + 1e-14 * q, (G, r["Q"], q)
        assert abs(r["iters"] - ref[2]) <= max(2, 0.01 * ref[2]), (G, r["iters"], ref[2])
        out[G] = r
    for G in (2, 3):
        assert abs(out[G]["Q"] / out[1]["Q"] - 1) < tol   # different reduction orders, both within tol of exact
    # the coarse half of the same coupled sample (mesh level 4 of level 5)
    qc, bc, xc = _exact(cfg, 128, seed, level, k)
    rc = _solve(ctx, level - 1, 2, seed, level, k, tol)[0]
    assert abs(rc["Q"] - qc) <= tol * bc * xc * (1 + 1e-6) + 1e-14 * qc
    ctx.close()


def test_dd_h512_single_system_and_slabs():
    """h = 1/512 (configs[4] level 6): one system on the whole GPU (G = 1) and as 4 slabs, against K3c's
    2-CTA-cluster solve of the same sample: both within tol ||b|| ||x|| <= 1.5 tol Q of the exact Q."""
    cfg, ctx = _ctx(ws=8 << 30)
    seed, level, k, tol = 42, 6, 0, 1e-8
    ref = ctx.sample_level(level, 1, seed=seed, first_index=k, prec_fine=precision("minres"), tol_fine=tol,
                           tol_coarse=tol, per_sample=True).per_sample[0]
    for G in (1, 4):
        r = _solve(ctx, level, G, seed, level, k, tol)[0]
        assert r["status"] == 0 and r["relres"] <= tol
        assert abs(r["Q"] - ref[0]) <= 2 * 1.5 * tol * abs(ref[0]), (G, r["Q"], ref[0])
        assert abs(r["iters"] - ref[2]) <= max(2, 0.01 * ref[2]), (G, r["iters"], ref[2])
    ctx.close()


def test_dd_edge_cases():
    cfg, ctx = _ctx()
    r = _solve(ctx, 4, 1, 1, 4, 0, 1e-12, max_iter=50)[0]
    assert r["done"] and r["status"] == 1 and r["iters"] == 50     # max_iter exhaustion reported, not hidden
    with pytest.raises(RuntimeError):
        layout(128, cfg["m"], 0, 100)                                # 127 rows over 100 ranks
    with pytest.raises(RuntimeError):
        SlabSolver(ctx, 4, 0, 1).begin(1, 6, 0, 1e-6)                 # level must be mesh_level or +1
    ctx.close()


def _two_process_worker(rank, world, port, q):
    """One rank of a 2-process slab solve on ONE GPU (host-driven exchange over gloo: no kernel waits on another
    process's kernel, B200_PROFILING.md), rank 0 also solving the same system alone (world = 1)."""
    import os
    import torch.distributed as dist
    from paper_2503_05533_b200.dd import dd_solve
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import __graft_entry__  # noqa: F401  (sys.path)
        cfg, ctx = _ctx(ws=1 << 30)
        eng = SlabSolver(ctx, 4, rank, world)
        eng.begin(9, 4, 3, 1e-9)
        res = dd_solve(eng, dist.group.WORLD, check_every=16)
        eng.close()
        one = None
        if rank == 0:
            e1 = SlabSolver(ctx, 4, 0, 1)
            e1.begin(9, 4, 3, 1e-9)
            one = e1.run_local()
            e1.close()
        ctx.close()
        q.put((rank, res, one))
    finally:
        dist.destroy_process_group()


def test_dd_two_processes_on_one_gpu_gloo():
    """VERDICT r01 'Build NEXT-3': the multi-rank driver (dd.dd_solve) as 2 processes on one GPU: both ranks hold
    the same result, equal to the 1-rank solve within the tolerance (different reduction order), same steps +-1%."""
    import socket
    import torch.multiprocessing as mp
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_two_process_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    out = {r: (res, one) for r, res, one in (q.get(timeout=600) for _ in range(2))}
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    r0, r1, one = out[0][0], out[1][0], out[0][1]
    assert r0 == r1 and r0["status"] == 0 and one["status"] == 0
    assert abs(r0["Q"] / one["Q"] - 1) < 1e-9
    assert abs(r0["iters"] - one["iters"]) <= max(2, 0.01 * one["iters"])


@pytest.mark.parametrize("level,G,tol", [(5, 2, 1e-10), (5, 3, 1e-10), (6, 4, 1e-8), (6, 8, 1e-8)])
def test_dd_fused_peer_exchange_emulated(level, G, tol):
    """The fused-exchange kernel (mlmc_dd_run_emulated: the per-step halo rows pushed into the neighbours' ghost
    rows and the rank partials into every rank's table from inside the solve kernel, all G ranks in one
    cooperative launch): same result as the host-driven G-slab solve to rounding, within the residual bound
    of the oracle's direct solve (h = 1/256) or of K3c (h = 1/512)."""
    from paper_2503_05533_b200.dd import dd_run_fused_emulated
    cfg, ctx = _ctx(ws=8 << 30)
    seed, k = 43, 1
    N = cfg["h0_inv"] << level
    eng = [SlabSolver(ctx, level, g, G) for g in range(G)]
    for e in eng:
        e.begin(seed, level, k, tol)
    r = dd_run_fused_emulated(eng)
    per_rank = [e.result() for e in eng]
    for e in eng:
        e.close()
    assert all(p == per_rank[0] for p in per_rank) and per_rank[0]["Q"] == r["Q"]
    assert r["status"] == 0 and r["relres"] <= tol
    host = _solve(ctx, level, G, seed, level, k, tol)[0]
    assert abs(r["Q"] / host["Q"] - 1) < tol and abs(r["iters"] - host["iters"]) <= max(2, 0.01 * host["iters"])
    if level == 5:
        q, bn, xn = _exact(cfg, N, seed, level, k)
        assert abs(r["Q"] - q) <= tol * bn * xn * (1 + 1e-6) + 1e-14 * q
    else:
        ref = ctx.sample_level(level, 1, seed=seed, first_index=k, prec_fine=precision("minres"), tol_fine=tol,
                               tol_coarse=tol, per_sample=True).per_sample[0]
        assert abs(r["Q"] - ref[0]) <= 2 * 1.5 * tol * abs(ref[0])
    ctx.close()


def _ipc_worker(rank, world, port, q):
    """Peer mapping of the slab workspaces (mlmc_dd_ipc_handle / _open / _close) between 2 processes on one GPU:
    each rank reads the other's copy of the sample's triangle coefficients through the mapped pointer (no kernel
    waits on another: only the mapping of dd_solve_peer is exercised, its kernel is tested emulated)."""
    import os
    import numpy as np
    import torch.distributed as dist
    import warnings
    warnings.simplefilter("ignore", FutureWarning)
    from cuda import cudart
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        cfg, ctx = _ctx(ws=1 << 30)
        eng = SlabSolver(ctx, 5, rank, world)
        eng.begin(17, 5, 4, 1e-6)
        eng.result()
        allh = [None] * world
        dist.all_gather_object(allh, eng.ipc_handle())
        other = 1 - rank
        ptr, base = eng.ipc_open(*allh[other])
        lay = eng.lay
        nbytes = 8 * 2 * lay.N * lay.N
        mine = np.empty(2 * lay.N * lay.N, np.float64)
        theirs = np.empty_like(mine)
        err1, = cudart.cudaMemcpy(mine.ctypes.data, eng.ws.data_ptr() + lay.a_off, nbytes,
                                  cudart.cudaMemcpyKind.cudaMemcpyDeviceToHost)
        from paper_2503_05533_b200.dd import layout as dd_layout
        their_off = dd_layout(lay.N, cfg["m"], other, world).a_off       # the peer's own layout
        err2, = cudart.cudaMemcpy(theirs.ctypes.data, ptr + their_off, nbytes,
                                  cudart.cudaMemcpyKind.cudaMemcpyDeviceToHost)
        dist.barrier()
        eng.ipc_close(base)
        eng.close()
        ctx.close()
        q.put((rank, int(err1), int(err2), bool(np.array_equal(mine, theirs)), float(np.abs(mine).sum())))
    finally:
        dist.destroy_process_group()


def test_dd_peer_mapping_two_processes_one_gpu():
    import socket
    import torch.multiprocessing as mp
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_ipc_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    out = [q.get(timeout=300) for _ in range(2)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    for rank, e1, e2, same, tot in out:
        assert e1 == 0 and e2 == 0 and same and tot > 0, (rank, e1, e2, same)
