"""K3d (NEXT-3) multi-rank logic on CPU (-m "not gpu"): ONE sample's MINRES split into row slabs over
world size 1, 2 and 3 with torch.distributed gloo, through the product's host driver
(paper_2503_05533_b200.dd.dd_solve) and the C-ABI's host-only partition / exchange-row functions
(mlmc_dd_layout_get, mlmc_dd_exchange_rows).  The device kernels are replaced by a NumPy emulation
written here (TEST CODE: the same per-node arithmetic as dd_pass_kernel / dd_scalar_kernel, so the
driver's all-reduce and halo schedule are exercised exactly as on GPUs).

Checks: every rank returns the same Q and iteration count; Q within the per-sample residual bound of the
oracle's direct solve (tol ||b|| ||x|| + 1e-14 Q); iteration count within 2 of the oracle's textbook
MINRES; the 2- and 3-rank solves equal the 1-rank solve to rounding (1e-12 relative); the
ghost rows each rank computes locally equal its neighbour's owned rows bit for bit.
"""
import math
import os
import socket

import numpy as np
import pytest
import torch
import torch.multiprocessing as mp

from oracle import core as oc

CASE = dict(m=16, sigma2=1.0, corr_len=0.3, N=32, seed=3, index=5, tol=1e-9)


class NumpySlab:
    """CPU stand-in for SlabSolver (test-only): same workspace layout (from the C-ABI), same arithmetic."""

    def __init__(self, N, m, rank, world):
        from paper_2503_05533_b200 import dd
        self.dd = dd
        self.lay = dd.layout(N, m, rank, world)
        self.rank, self.world, self.N = rank, world, N
        self.ws = torch.zeros(int(self.lay.bytes), dtype=torch.uint8)
        self.sums = self.ws[self.lay.sums_off:self.lay.sums_off + 24].view(torch.float64)
        L = self.lay
        self.planes = [self.ws[L.plane_off[q]:L.plane_off[q] + 8 * L.rows * L.pitch].view(torch.float64)
                       .view(L.rows, L.pitch).numpy() for q in range(5)]
        self.st = None

    def row(self, off):
        return self.ws[off:off + 8 * self.lay.pitch].view(torch.float64)

    def exchange_offsets(self, step):
        return self.dd.exchange_rows(self.lay, step)

    def begin(self, a, tol, max_iter=100000):
        L, N = self.lay, self.N
        C, h2 = N - 1, 1.0 / N ** 2
        P0, P1, P2, CE, CN = self.planes
        for r in range(L.rows):
            j = L.j0 - 2 + r
            for c in range(L.pitch):
                i = c - 1
                inside = 1 <= i <= C and 1 <= j <= C
                P0[r, c] = 0.0
                P1[r, c] = h2 if inside else 0.0
                P2[r, c] = 0.0
                CE[r, c] = 0.5 * (a[2 * (j * N + i)] + a[2 * ((j - 1) * N + i) + 1]) if (0 <= i < N and 1 <= j < N) else 0.0
                CN[r, c] = 0.5 * (a[2 * (j * N + i) + 1] + a[2 * (j * N + i - 1)]) if (1 <= i < N and 0 <= j < N) else 0.0
        self.st = dict(tol=tol, max_iter=max_iter, k=0, step=0, status=1, done=False, cs=-1.0, sn=0.0, ct=0.0,
                       c1=1.0, c0=0.0, dbar=0.0, epsln=0.0, phibar=0.0, s1q=0.0, s2q=0.0, Xq=0.0, beta1=0.0,
                       inv_beta1=0.0, tol_b=0.0, invb_prev=0.0, alpha_prev=0.0, sigma_prev=0.0, Q=0.0, relres=1.0)

    def pass_(self):
        s, L, N = self.st, self.lay, self.N
        if s["done"]:
            return
        C = N - 1
        Pj = self.planes[(s["step"] + 1) % 3]
        Pp = self.planes[s["step"] % 3]
        Pn = self.planes[(s["step"] + 2) % 3]
        CE, CN = self.planes[3], self.planes[4]
        r = lambda j: j - (L.j0 - 2)

        def Ap(P, j, i):
            ce, cw, cn, cs = CE[r(j), i + 1], CE[r(j), i], CN[r(j), i + 1], CN[r(j) - 1, i + 1]
            d = (ce + cw) + (cn + cs)
            return d * P[r(j), i + 1] - ce * P[r(j), i + 2] - cw * P[r(j), i] - cn * P[r(j) + 1, i + 1] \
                - cs * P[r(j) - 1, i + 1]
        new = {}
        for j in range(max(L.j0 - 1, 1), min(L.j1, C) + 1):
            for i in range(1, C + 1):
                new[(j, i)] = s["ct"] * Ap(Pj, j, i) + (s["c1"] * Pj[r(j), i + 1] + s["c0"] * Pp[r(j), i + 1])
        for (j, i), v in new.items():
            Pn[r(j), i + 1] = v
        sa = sb = sc = 0.0
        for j in range(L.j0, L.j1):
            for i in range(1, C + 1):
                pv = Pn[r(j), i + 1]
                sa += pv * Ap(Pn, j, i)
                sb += pv * pv
                sc += pv
        self.sums[:3] = torch.tensor([sa, sb, sc], dtype=torch.float64)

    def scalar(self):
        s = self.st
        if s["done"]:
            return
        sa, bb, sc = (float(v) for v in self.sums[:3])
        invb = 1.0 / math.sqrt(bb) if bb > 0 else 0.0
        beta, alpha, sigma = bb * invb, sa * invb * invb, sc * invb
        k = s["k"]
        if k > 0:
            oldeps = s["epsln"]
            delta = s["cs"] * s["dbar"] + s["sn"] * s["alpha_prev"]
            gbar = s["sn"] * s["dbar"] - s["cs"] * s["alpha_prev"]
            s["epsln"] = s["sn"] * beta
            s["dbar"] = -s["cs"] * beta
            invg = 1.0 / math.sqrt(gbar * gbar + bb)
            s["cs"], s["sn"] = gbar * invg, beta * invg
            phi = s["cs"] * s["phibar"]
            s["phibar"] = s["sn"] * s["phibar"]
            sq = (s["sigma_prev"] - oldeps * s["s2q"] - delta * s["s1q"]) * invg
            s["s2q"], s["s1q"] = s["s1q"], sq
            s["Xq"] += phi * sq
        else:
            s["beta1"], s["inv_beta1"], s["tol_b"], s["phibar"] = beta, invb, s["tol"] * beta, beta
        done = False
        if k == 0:
            done = s["beta1"] == 0.0
        elif s["phibar"] <= s["tol_b"]:
            s["status"], done = 0, True
        elif k >= s["max_iter"]:
            done = True
        if done:
            s["done"], s["Q"], s["relres"] = True, s["Xq"] / self.N ** 2, s["phibar"] * s["inv_beta1"]
        else:
            s["ct"], s["c1"] = invb, -alpha * invb
            s["c0"] = 0.0 if k == 0 else -beta * s["invb_prev"]
            s["invb_prev"], s["alpha_prev"], s["sigma_prev"] = invb, alpha, sigma
            s["k"], s["step"] = k + 1, s["step"] + 1

    def done(self):
        return self.st["done"]

    def result(self):
        s = self.st
        return {"Q": s["Q"], "iters": s["k"], "relres": s["relres"], "status": s["status"], "done": s["done"]}


def _coeffs():
    P = oc.OracleProblem(0, CASE["m"], CASE["sigma2"], CASE["corr_len"], 2.0, 8)
    xi = oc.normals(CASE["seed"], 2, CASE["index"], CASE["m"])
    return P.field_triangles(CASE["N"], xi)


def _worker(rank, world, port, q):
    import torch.distributed as dist
    from paper_2503_05533_b200.dd import dd_solve
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        e = NumpySlab(CASE["N"], CASE["m"], rank, world)
        e.begin(_coeffs(), CASE["tol"])
        res = dd_solve(e, dist.group.WORLD, check_every=4)
        # the halo rows j0-1 / j1 formed locally vs the neighbour's owned rows, last p_{j+1} plane
        L = e.lay
        Pn = e.planes[(e.st["step"] + 2) % 3]       # p_{j+1} of the last pass (done: step not advanced)
        r = lambda j: j - (L.j0 - 2)
        mine = {"lo_halo": Pn[r(L.j0 - 1)].copy() if rank > 0 else None,
                "hi_halo": Pn[r(L.j1)].copy() if rank + 1 < world else None,
                "first": Pn[r(L.j0)].copy(), "last": Pn[r(L.j1 - 1)].copy()}
        q.put((rank, res, mine))
    finally:
        dist.destroy_process_group()


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


@pytest.fixture(scope="module", autouse=True)
def built():
    import __graft_entry__
    __graft_entry__.build()


def _run(world):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    out = [q.get(timeout=600) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    return {r: (res, mine) for r, res, mine in out}


def test_partition_and_exchange_rows_host_functions():
    """mlmc_dd_layout_get splits rows 1..N-1 evenly (>= 2 rows per rank; otherwise EINVAL) and
    mlmc_dd_exchange_rows pairs every send with the neighbour's receive of the same global row."""
    from paper_2503_05533_b200 import dd
    N = 64
    for world in (1, 2, 3, 5, 31):
        lays = [dd.layout(N, 16, r, world) for r in range(world)]
        assert lays[0].j0 == 1 and lays[-1].j1 == N and all(a.j1 == b.j0 for a, b in zip(lays, lays[1:]))
        assert all(L.j1 - L.j0 >= 2 for L in lays)
        for step in (0, 1, 2, 7):
            offs = [dd.exchange_rows(L, step) for L in lays]
            for g in range(world - 1):
                a, b = lays[g], lays[g + 1]
                plane = (step + 2) % 3
                row_of = lambda L, off: (off - L.plane_off[plane]) // (8 * L.pitch) + L.j0 - 2
                assert row_of(a, offs[g][2]) == row_of(b, offs[g + 1][1]) == a.j1 - 2     # a -> b
                assert row_of(b, offs[g + 1][0]) == row_of(a, offs[g][3]) == b.j0 + 1     # b -> a
            assert offs[0][0] == offs[0][1] == -1 and offs[-1][2] == offs[-1][3] == -1
    with pytest.raises(RuntimeError):
        dd.layout(N, 16, 0, 40)                     # 63 rows over 40 ranks: a slab of 1 row


def test_slab_minres_two_and_three_ranks_gloo():
    N, tol = CASE["N"], CASE["tol"]
    a = _coeffs()
    AB, _, b = oc.assemble(N, a)
    x, _ = oc.chol_band_solve(AB, b)
    q_exact, bn, xn = x.sum() / N ** 2, np.linalg.norm(b), np.linalg.norm(x)
    _, it_or, _, _ = oc.minres_band(AB, b, tol)
    one = NumpySlab(N, CASE["m"], 0, 1)
    one.begin(a, tol)
    from paper_2503_05533_b200.dd import dd_solve
    r1 = dd_solve(one, None, check_every=4)
    assert r1["status"] == 0 and abs(r1["Q"] - q_exact) <= tol * bn * xn * (1 + 1e-6) + 1e-14 * q_exact
    assert abs(r1["iters"] - it_or) <= 2, (r1["iters"], it_or)
    for world in (2, 3):
        out = _run(world)
        res = [out[r][0] for r in range(world)]
        assert all(r["Q"] == res[0]["Q"] and r["iters"] == res[0]["iters"] for r in res)
        assert res[0]["status"] == 0 and abs(res[0]["iters"] - r1["iters"]) <= 1
        assert abs(res[0]["Q"] / r1["Q"] - 1) < 1e-12
        for g in range(world - 1):
            assert np.array_equal(out[g][1]["hi_halo"], out[g + 1][1]["first"])
            assert np.array_equal(out[g + 1][1]["lo_halo"], out[g][1]["last"])
