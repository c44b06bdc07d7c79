"""Multi-rank Algorithm 2 on CPU (-m "not gpu"): the library's controller
(mlmc_adaptive_run_host, the same code mlmc_adaptive_run runs over the GPU)
with world size 2 over torch.distributed gloo, each rank drawing its slice of
every level's new sample indices through an oracle-backed host sampler.

Checks: both ranks return identical results; the 2-rank run takes the same
decisions (L, N_l) as the 1-rank run and as the oracle's own Algorithm 2 on
the same samples; the estimate agrees to rounding (the rank partial sums are
added in a different order).
"""
import math
import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp

from oracle import core as oc
from oracle import mlmc as om

CFG = dict(m=16, sigma2=1.0, corr_len=0.3, h0_inv=8, L_max=3, eps=6e-4, k_p=0.05, seed=9, N_init=40)


def _sampler_factory():
    P = oc.OracleProblem(0, CFG["m"], CFG["sigma2"], CFG["corr_len"], 2.0, CFG["h0_inv"])

    def sampler(level, n, first, pf, pc, tf, tc):
        s = np.zeros(12)
        nf = ((CFG["h0_inv"] << level) - 1) ** 2
        nc = ((CFG["h0_inv"] << (level - 1)) - 1) ** 2 if level else 0
        for k in range(first, first + n):
            o = P.coupled_sample(level, CFG["seed"], k, solver=oc.SOLVER_MINRES, tol_f=tf, tol_c=tc)
            y = o[0] - o[1]
            s[0] += y
            s[1] += y * y
            s[2] += o[0]
            s[3] += o[1]
            s[4] += o[2] * nf + o[3] * nc          # R5 cost model (MINRES: iterations x unknowns)
            s[5] += 1
            s[6] += (o[6] != 0) or (o[7] != 0)
            s[7] += o[2]
            s[8] += o[3]
            s[9] = max(s[9], o[2])
            s[10] = max(s[10], o[3])
        return s
    return sampler


def _run(group=None):
    from paper_2503_05533_b200.api import mlmc_adaptive_run_host
    return mlmc_adaptive_run_host(CFG["h0_inv"], CFG["L_max"], CFG["eps"], _sampler_factory(), k_p=CFG["k_p"],
                                  N_init=CFG["N_init"], seed=CFG["seed"], group=group)


def _worker(rank, world, port, q):
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        q.put((rank, _run(dist.group.WORLD)))
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


def test_controller_two_ranks_gloo_matches_one_rank_and_oracle():
    single = _run(None)
    assert single["code"] == 0 and single["L"] >= 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=600) for _ in range(2))
    for p in procs:
        p.join(timeout=60)
    for r in res.values():
        r.pop("solve_seconds")
    assert res[0] == res[1]                                           # every rank took the same decisions
    two = res[0]
    assert two["L"] == single["L"] and two["N"] == single["N"] and two["rounds"] == single["rounds"]
    assert abs(two["estimate"] - single["estimate"]) <= 1e-13 * abs(single["estimate"])
    # the oracle's Algorithm 2 over the same samples
    smp = _sampler_factory()

    def osampler(l, first, count, tf, tc):
        P = oc.OracleProblem(0, CFG["m"], CFG["sigma2"], CFG["corr_len"], 2.0, CFG["h0_inv"])
        nf = ((CFG["h0_inv"] << l) - 1) ** 2
        nc = ((CFG["h0_inv"] << (l - 1)) - 1) ** 2 if l else 0
        outs = [P.coupled_sample(l, CFG["seed"], k, solver=oc.SOLVER_MINRES, tol_f=tf, tol_c=tc)
                for k in range(first, first + count)]
        return [o[0] - o[1] for o in outs], [o[2] * nf + o[3] * nc for o in outs]

    o = om.adaptive_mpml(osampler, CFG["eps"], 1 / CFG["h0_inv"], CFG["k_p"], L_max=CFG["L_max"],
                         N_init=CFG["N_init"])
    assert o.L == single["L"] and o.N == single["N"]
    assert abs(o.estimate - single["estimate"]) <= 1e-12 * abs(o.estimate)
    del smp


def test_controller_standard_mlmc_mode_and_lmax():
    """k_p <= 0 is standard MLMC (fixed solver accuracy on every level); an eps too small for
    L_max returns MLMC_ELMAX (R2) with the estimate filled."""
    from paper_2503_05533_b200.api import mlmc_adaptive_run_host
    seen = []
    base = _sampler_factory()

    def sampler(level, n, first, pf, pc, tf, tc):
        seen.append((tf, tc))
        return base(level, n, first, pf, pc, tf, tc)

    r = mlmc_adaptive_run_host(CFG["h0_inv"], 2, 3e-3, sampler, k_p=0.0, fixed_tol=1e-9, N_init=20, seed=1)
    assert all(tf == 1e-9 and tc == 1e-9 for tf, tc in seen)
    assert r["code"] in (0, 4)
    r = mlmc_adaptive_run_host(CFG["h0_inv"], 1, 2e-4, base, k_p=0.05, N_init=20, max_rounds=3)
    assert r["code"] == 4 and r["L"] == 1 and math.isfinite(r["estimate"])


def _worker_local_on_one_rank(rank, world, port, q):
    """A default process group exists, but only rank 0 runs an adaptive run with group=None: it must stay
    local (world 1) instead of all-reducing through the default group while rank 1 waits in a barrier."""
    import datetime
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world, timeout=datetime.timedelta(seconds=60))
    try:
        r = _run(None) if rank == 0 else None
        dist.barrier()
        q.put((rank, r))
    finally:
        dist.destroy_process_group()


def test_group_none_is_local_even_with_a_default_group():
    single = _run(None)
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker_local_on_one_rank, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=240) for _ in range(2))
    for p in procs:
        p.join(timeout=60)
    r0 = res[0]
    r0.pop("solve_seconds")
    single.pop("solve_seconds")
    assert res[1] is None and r0 == single


# ---------------------------------------------------------------------------- exact level sums
def _dyadic_sampler(level, n, first, pf, pc, tf, tc):
    """Synthetic coupled differences that are dyadic rationals (multiples of 2^-(2l+12), about a third of
    them negative), so every rank's double partial sums are exact whatever its slice: the exchange of the
    exact fixed-point sums (32-bit pieces, carries, two's complement) must then reproduce the 1-rank run
    bit for bit."""
    k = np.arange(first, first + n, dtype=np.int64)
    noise = ((k * 2654435761 + 97 * level) % 2001 - 1000).astype(np.float64)
    y = (2.0 ** (-2 * level - 4)) + noise * 2.0 ** (-2 * level - 12)
    s = np.zeros(12)
    s[0] = y.sum()
    s[1] = (y * y).sum()
    s[2] = s[0]
    s[4] = float(n) * 100.0 * 4 ** level
    s[5] = n
    s[7] = 10.0 * n
    s[9] = 10.0
    return s


def _run_dyadic(group=None):
    from paper_2503_05533_b200.api import mlmc_adaptive_run_host
    return mlmc_adaptive_run_host(8, 4, 1e-3, _dyadic_sampler, k_p=0.05, N_init=40, seed=1, group=group)


def _worker_dyadic(rank, world, port, q):
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        q.put((rank, _run_dyadic(dist.group.WORLD)))
    finally:
        dist.destroy_process_group()


def test_exact_sum_exchange_two_ranks_bit_identical():
    from fractions import Fraction
    single = _run_dyadic(None)
    assert single["code"] == 0 and single["L"] == 3
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker_dyadic, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=600) for _ in range(2))
    for p in procs:
        p.join(timeout=60)
    single.pop("solve_seconds")
    for r in res.values():
        r.pop("solve_seconds")
        assert r == single                                           # bit-identical, every field
    # the level means are the exact sums over all drawn samples, rounded once
    for l in range(single["L"] + 1):
        n = single["N"][l]
        y = _dyadic_sampler(l, n, 0, None, None, 0, 0)[0]
        k = np.arange(0, n, dtype=np.int64)
        noise = ((k * 2654435761 + 97 * l) % 2001 - 1000)
        exact = sum((Fraction(1, 2 ** (2 * l + 4)) + Fraction(int(v), 2 ** (2 * l + 12)) for v in noise), Fraction(0))
        assert single["mean"][l] == float(exact / n) and y == float(exact)


# ---------------------------------------------------------------------------- a rank-local failure
def _worker_fail(rank, world, port, q):
    """Rank 1's sampler raises in the second round: both ranks must leave mlmc_adaptive_run_host with an
    error (the failure travels in the round's single all-reduce) instead of rank 0 waiting forever."""
    import datetime
    import torch.distributed as dist
    from paper_2503_05533_b200.api import mlmc_adaptive_run_host
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world, timeout=datetime.timedelta(seconds=60))
    calls = {"n": 0}

    def sampler(level, n, first, pf, pc, tf, tc):
        calls["n"] += 1
        if rank == 1 and calls["n"] > 2:
            raise RuntimeError("injected rank-local failure")
        return _dyadic_sampler(level, n, first, pf, pc, tf, tc)
    try:
        try:
            mlmc_adaptive_run_host(8, 4, 1e-3, sampler, k_p=0.05, N_init=40, seed=1, group=dist.group.WORLD)
            q.put((rank, "no error"))
        except RuntimeError as e:
            q.put((rank, str(e)))
    finally:
        dist.destroy_process_group()


def test_rank_local_sampler_failure_stops_every_rank():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker_fail, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=120) for _ in range(2))
    for p in procs:
        p.join(timeout=60)
    assert res[0] != "no error" and res[1] != "no error", res


def test_round_log_json_lines(tmp_path, monkeypatch):
    """MLMC_ROUND_LOG: one JSON line per adaptive round (the controller's trace), consistent with the result."""
    import json
    path = tmp_path / "rounds.jsonl"
    monkeypatch.setenv("MLMC_ROUND_LOG", str(path))
    r = _run_dyadic(None)
    lines = [json.loads(x) for x in path.read_text().splitlines()]
    assert len(lines) == r["rounds"] and [x["round"] for x in lines] == list(range(1, r["rounds"] + 1))
    last = lines[-1]
    assert last["L"] == r["L"] and [lv["N"] for lv in last["levels"]] == r["N"]
    assert all(abs(lv["mean"] - m) <= 1e-15 * abs(m) for lv, m in zip(last["levels"], r["mean"]))
    assert last["var_ok"] and not last["bias_fail"]
