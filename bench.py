#!/usr/bin/env python
"""bench.py -- one JSON line for the MPML hot path on B200 (contract in DESIGN.md section 8).

Step = one pass of the whole hot path over BASELINE.json configs[1] (C2): for
each level l = 0..3 of h = 1/8..1/64, N_l = (20000, 5000, 1200, 300) coupled
samples: Philox normals -> KL field (m = 64) on both meshes -> P1 assembly ->
fp64 MINRES to the level tolerance (1e-4, 1e-5, 1e-6, 1e-8; coarse half at
tol_{l-1}) -> QoI -> level sums; with N > 1 ranks each rank draws its own
index range (weak scaling) and the level sums are all-reduced over NCCL once
per step (the method's only exchange).

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]

--impl reference times the CPU oracle (oracle/, plain C) on a bounded sample of
the same workload on this box's host cores (rank 0 only).
"""
from __future__ import annotations

import argparse
import json
import math
import os
import subprocess
import sys
import tempfile
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import workloads as W  # noqa: E402

METRIC = "coupled level samples/sec per level and time-to-eps at 1/2/4/8 B200; HBM GB/s vs peak"
UNIT = "coupled samples/s"
# algorithmic fp64 flops of one MINRES iteration per unknown: SURVEY section 8(d)'s count (5-point matvec 13,
# two dots 4, Lanczos / w / x updates 11); the kernel's own one-reduction form needs 25
FLOPS_PER_NODE_ITER = 28.0


def _measured_alu_peaks() -> dict:
    """ALU peaks measured on this pool by tools/peak_alu.cu (profiles/r02_peaks.json, committed with its clock
    record); MEASURED_PEAKS.json has no FP64/FP32 entries.  Fallback only if the file is missing: the guide's unit
    counts (148 SMs x 64 FP64 / 128 FP32 FMA per clock x 2 x 1.965 GHz)."""
    try:
        d = json.load(open(os.path.join(ROOT, "profiles", "r02_peaks.json")))
        return {"fp64": float(d["fp64_fma_tflops"]), "fp32": float(d["fp32_fma_tflops"]),
                "source": "measured: DFMA / FFMA microbenchmark tools/peak_alu.cu at "
                          f"{d['clocks']['sm_mhz']:.0f} MHz (profiles/r02_peaks.json)"}
    except Exception:
        return {"fp64": 148 * 64 * 2 * 1.965e9 / 1e12, "fp32": 148 * 128 * 2 * 1.965e9 / 1e12,
                "source": "derived (profiles/r02_peaks.json missing): unit counts x 1.965 GHz"}


ALU = _measured_alu_peaks()
FP64_PEAK_TFLOPS = ALU["fp64"]
FP32_PEAK_TFLOPS = ALU["fp32"]


def _measured_hbm_gbs() -> float:
    """MEASURED_PEAKS.json (driver-written, copy bandwidth); else the profiling guide's B200 fallback."""
    try:
        return float(json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))["hbm_gbs"])
    except Exception:
        return 6650.0                    # B200_PROFILING.md fallback (6.65 TB/s), used only without the file


HBM_PEAK_GBS = _measured_hbm_gbs()


def _dbg(msg):
    """BENCH_DEBUG=1: rank-tagged progress on stderr (multi-rank debugging)."""
    if os.environ.get("BENCH_DEBUG"):
        print(f"[rank {os.environ.get('RANK', '0')}] {msg}", file=sys.stderr, flush=True)


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-extras", action="store_true", help="skip cpu_baseline / e2e / time-to-eps")
    return ap.parse_args()


# ----------------------------------------------------------------------------- clocks
class ClockSampler:
    """SM clock and clock-event reasons sampled every ~2 ms by NVML on a background thread between
    start() and stop() -- the timed region is tens of milliseconds, far below nvidia-smi's polling
    period.  Falls back to one nvidia-smi reading if NVML is unavailable."""
    REASONS = (("hw_slowdown", "nvmlClocksEventReasonHwSlowdown"),
               ("hw_thermal_slowdown", "nvmlClocksEventReasonHwThermalSlowdown"),
               ("sw_thermal_slowdown", "nvmlClocksEventReasonSwThermalSlowdown"),
               ("sw_power_cap", "nvmlClocksEventReasonSwPowerCap"))

    def __init__(self, index: int):
        self.index = index
        self.rows = []
        self.ev = threading.Event()
        self.th = None
        try:
            import pynvml
            pynvml.nvmlInit()
            self.nv = pynvml
            self.h = pynvml.nvmlDeviceGetHandleByIndex(index)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM)
            get = getattr(pynvml, "nvmlDeviceGetCurrentClocksEventReasons", None) or \
                pynvml.nvmlDeviceGetCurrentClocksThrottleReasons
            self.get_reasons = lambda: get(self.h)
        except Exception:
            self.nv = None

    def _loop(self):
        nv = self.nv
        while not self.ev.is_set():
            try:
                self.rows.append((nv.nvmlDeviceGetClockInfo(self.h, nv.NVML_CLOCK_SM), self.get_reasons()))
            except Exception:
                pass
            time.sleep(0.002)

    def start(self):
        if self.nv:
            self.rows = []
            self.ev.clear()
            self.th = threading.Thread(target=self._loop, daemon=True)
            self.th.start()

    def stop(self) -> dict:
        if not self.nv:
            return self._smi_once()
        self.ev.set()
        if self.th:
            self.th.join()
        if not self.rows:
            return {"sm_mhz": None, "sm_max_mhz": self.max_mhz, "reasons": [], "samples": 0, "source": "nvml"}
        sm = sorted(r[0] for r in self.rows)
        reasons = sorted({name for _, mask in self.rows for name, const in self.REASONS
                          if mask & getattr(self.nv, const, 0)})
        return {"sm_mhz": sm[len(sm) // 2], "sm_min_mhz": sm[0], "sm_max_mhz": self.max_mhz, "reasons": reasons,
                "samples": len(self.rows), "source": "nvml, every 2 ms during the timed steps"}

    def _smi_once(self) -> dict:
        try:
            out = subprocess.run(["nvidia-smi", "-i", str(self.index), "--query-gpu=clocks.sm,clocks.max.sm",
                                  "--format=csv,noheader,nounits"], capture_output=True, text=True).stdout
            a, b = [int(x) for x in out.strip().split(",")[:2]]
            return {"sm_mhz": a, "sm_max_mhz": b, "reasons": [], "samples": 1, "source": "nvidia-smi (no NVML)"}
        except Exception:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["clock query unavailable"], "samples": 0}


# ----------------------------------------------------------------------------- oracle timing
def _cpu_model() -> str:
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


def ref_counts(div: int) -> dict:
    """A bounded sample of the configs[1] step with the same level mix: N_l / div samples per level (>= 1)."""
    return {l: max(1, n // div) for l, n in enumerate(W.CONFIGS["C2"]["N"])}


def oracle_step(counts: dict, seed: int, threads: int, first: int = 10_000_000) -> float:
    """Wall seconds for the oracle (oracle/oracle.c: KL field, element-by-element assembly, textbook MINRES to the
    same tolerances, coarse half at tol_{l-1}) on counts[l] coupled samples of each configs[1] level, all levels'
    samples in one pool of `threads` host threads, longest (finest) first."""
    from concurrent.futures import ThreadPoolExecutor
    from oracle import core as oc
    cfg = W.CONFIGS["C2"]
    P = oc.OracleProblem(0, cfg["m"], cfg["sigma2"], cfg["corr_len"], 2.0, cfg["h0_inv"])
    tols = cfg["tols"]
    tasks = [(l, first + k) for l in sorted(counts, reverse=True) for k in range(counts[l])]

    def one(t):
        l, k = t
        return P.coupled_sample(l, seed, k, solver=oc.SOLVER_MINRES, tol_f=tols[l], tol_c=tols[l - 1] if l else tols[0])
    t0 = time.perf_counter()
    if threads == 1:
        for t in tasks:
            one(t)
    else:
        with ThreadPoolExecutor(threads) as ex:
            list(ex.map(one, tasks))
    return time.perf_counter() - t0


def cpu_baseline(seed: int) -> dict:
    """The oracle as it stands on this box's host cores (rank 0, N = 1): all cores on 1/20 of the configs[1] step
    and one core on 1/100 of it (same level mix), coupled samples per second."""
    from oracle import core as oc
    oc.build()
    threads = os.cpu_count() or 1
    c_all, c_one = ref_counts(20), ref_counts(100)
    t_all = oracle_step(c_all, seed, threads)
    t_one = oracle_step(c_one, seed, 1, first=20_000_000)
    n_all, n_one = sum(c_all.values()), sum(c_one.values())
    return {"value": n_all / t_all, "unit": UNIT, "cores": threads, "kind": "oracle",
            "sample": f"{'/'.join(str(c_all[l]) for l in sorted(c_all))} coupled samples of levels 0..3 "
                      "(1/20 of the configs[1] step, same mix) through the oracle's KL field, element-by-element "
                      "assembly and textbook MINRES at the same tolerances, on all host threads",
            "seconds": t_all,
            "single_thread": {"value": n_one / t_one, "seconds": t_one,
                              "sample": f"{'/'.join(str(c_one[l]) for l in sorted(c_one))} (1/100 of the step)"},
            "cpu_model": _cpu_model()}


def run_reference(args):
    """--impl reference: the CPU oracle, as it stands, on this box's host cores; rank 0 only.  A step is a bounded
    sample of the configs[1] step (1/20 of each level's count, same level mix), wall-timed; value = coupled samples
    per second over the K timed steps.  Same metric, unit and config as our arm."""
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    if rank != 0:
        return
    from oracle import core as oc
    oc.build()
    threads = os.cpu_count() or 1
    cfg = W.CONFIGS["C2"]
    counts = ref_counts(20)
    per_step = sum(counts.values())
    for i in range(args.warmup):
        oracle_step(counts, cfg["seed"], threads, first=30_000_000 + i * per_step)
    walls = [oracle_step(counts, cfg["seed"], threads, first=40_000_000 + i * per_step) for i in range(args.steps)]
    wall = sum(walls)
    value = per_step * args.steps / wall
    sample = (f"per step: {'/'.join(str(counts[l]) for l in sorted(counts))} coupled samples of levels 0..3 "
              "(1/20 of the configs[1] step, same level mix), wall-timed")
    line = {"impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * wall / args.steps,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": c2_config(world, "nccl"),
            "engine": f"CPU oracle (oracle/oracle.c), textbook MINRES, {threads} host threads ({_cpu_model()})",
            "cpu_baseline": {"value": value, "unit": UNIT, "cores": threads, "kind": "oracle", "sample": sample,
                             "cpu_model": _cpu_model()},
            "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
            "wall_s": wall}
    print(json.dumps(line), flush=True)


C2_CONFIG = {"workload": "configs[1] (C2): 4-level MLMC h=1/8..1/64, KL m=64 (var 1, corr 0.3), "
                         "N=(20000,5000,1200,300) per GPU, fp64 MINRES tols 1e-4/1e-5/1e-6/1e-8",
             "l2": "flushed between timed steps (256 MiB write)"}


def c2_config(world: int, backend: str) -> dict:
    return {**C2_CONFIG, "parallelism": f"samples sharded, {world} rank(s), "
                                        f"{'NCCL' if backend == 'nccl' else backend} all-reduce of level sums"}


# ----------------------------------------------------------------------------- our arm
def run_ours(args):
    import numpy as np
    import torch
    import torch.distributed as dist

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if args.gpus != world and world == 1 and args.gpus > 1:
        print(json.dumps({"error": "--gpus > 1 must be launched with torch.distributed.run"}))
        sys.exit(2)
    # BENCH_DIST_BACKEND=gloo with more ranks than GPUs exercises the multi-rank logic (sharding, all-reduce,
    # max over ranks) on one GPU; its numbers are not scaling results.  The driver's runs use NCCL.
    backend = os.environ.get("BENCH_DIST_BACKEND", "nccl")
    local = local % max(1, torch.cuda.device_count())
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        if backend == "nccl":
            dist.init_process_group("nccl", device_id=dev)
        else:
            dist.init_process_group(backend)

    import __graft_entry__
    if rank == 0 or world == 1:
        __graft_entry__.build()
    if world > 1:
        dist.barrier()
    from paper_2503_05533_b200 import Context, precision

    cfg = W.CONFIGS["C2"]
    Nl, tols, seed, m = cfg["N"], cfg["tols"], cfg["seed"], cfg["m"]
    L = len(Nl)
    stream = torch.cuda.current_stream(dev)
    ctx = Context(field="expcov", m=m, sigma2=cfg["sigma2"], corr_len=cfg["corr_len"], h0_inv=cfg["h0_inv"],
                  L_max=L - 1, device=local, workspace_bytes=2 << 30, stream=stream)
    minres = precision("minres")
    sums = torch.zeros((L, 12), dtype=torch.float64, device=dev)
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)     # > 126 MB L2

    levels = list(range(L))
    tol_c = [tols[l - 1] if l else tols[0] for l in levels]

    def step(i):
        """One pass of the whole hot path: all levels concurrently (mlmc_sample_levels_async) + exchange."""
        first = [(i * world + rank) * Nl[l] for l in levels]
        ctx.sample_levels_async(levels, Nl, seed, first, [minres] * L, [minres] * L, tols, tol_c, sums)
        if world > 1:
            dist.all_reduce(sums)

    _dbg("context ready")
    clocks = ClockSampler(local)
    for i in range(args.warmup):
        step(10_000 + i)
    _dbg("warm-up done")
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    ctx.profile_enable(False)             # reset the per-kernel table: launch counts only (no event overhead)
    clocks.start()
    total_ms = 0.0
    iters_f = [0.0] * L
    iters_max = [[0.0, 0.0] for _ in range(L)]
    iters_c = [0.0] * L
    for i in range(args.steps):
        flush.zero_()                                                   # L2 flush between timed steps
        e0 = torch.cuda.Event(enable_timing=True)
        e_end = torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        step(i)
        e_end.record(stream)                                            # after the NCCL all-reduce (N > 1)
        torch.cuda.synchronize()
        total_ms += e0.elapsed_time(e_end)
        s = sums.cpu().numpy()
        for l in range(L):
            iters_f[l] += s[l, 7] / world
            iters_c[l] += s[l, 8] / world
            iters_max[l] = [max(iters_max[l][0], s[l, 9]), max(iters_max[l][1], s[l, 10])]
    torch.cuda.synchronize()
    clk = clocks.stop()
    if world > 1:
        t = torch.tensor([total_ms], dtype=torch.float64, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        total_ms = float(t.item())
        dist.barrier()
    torch.cuda.synchronize()
    gpu_launches = int(sum(r[2] for r in ctx.profile_read()))

    # per-level throughput: each level alone (same launch path: its fine and coarse solves concurrently), CUDA
    # events, L2 flushed before each; then the same passes with the library's per-launch events (the solves
    # serialised: clean per-kernel times for the roofline and the kernel table)
    def level_pass(profiled):
        ctx.profile_enable(profiled)
        ms_l = [0.0] * L
        for l in levels:
            for i in range(args.steps):
                flush.zero_()
                a0 = torch.cuda.Event(enable_timing=True)
                a1 = torch.cuda.Event(enable_timing=True)
                a0.record(stream)
                ctx.sample_level_async(l, Nl[l], seed, (50_000 + i * world + rank) * Nl[l], minres, minres, tols[l],
                                       tol_c[l], sums_out=sums[l])
                a1.record(stream)
                torch.cuda.synchronize()
                ms_l[l] += a0.elapsed_time(a1)
        pr = ctx.profile_read() if profiled else None
        ctx.profile_enable(False)
        return ms_l, pr
    level_ms, _ = level_pass(False)
    prof_level_ms, prof = level_pass(True)
    per_level_total_ms = sum(prof_level_ms)

    n_step = sum(Nl)
    value = world * n_step * args.steps / (total_ms / 1e3)
    ms_per_step = total_ms / args.steps
    per_level = {f"l{l}": {"h": f"1/{cfg['h0_inv'] << l}", "N": Nl[l], "tol_fine": tols[l],
                           "samples_per_s": world * Nl[l] * args.steps / (level_ms[l] / 1e3),
                           "ms_alone": level_ms[l] / args.steps,
                           "mean_iters_fine": iters_f[l] / (Nl[l] * args.steps),
                           "mean_iters_coarse": iters_c[l] / (Nl[l] * args.steps) if l else 0.0,
                           # (the step's all-reduce adds the per-rank maxima: reported at N = 1 only)
                           "max_iters_fine": iters_max[l][0] if world == 1 else None,
                           "max_iters_coarse": (iters_max[l][1] if l else 0.0) if world == 1 else None}
                 for l in range(L)}

    # ---- roofline of the dominant kernel (largest device time in the timed region)
    kern = sorted(prof, key=lambda r: -r[3])
    top = kern[0]
    n_of = lambda N: (N - 1) ** 2
    work = 0.0                                                          # node-iterations of this kernel class
    if top[0] == "minres":
        for l in range(L):
            if (cfg["h0_inv"] << l) == top[1]:
                work += iters_f[l] * n_of(top[1])
            if l and (cfg["h0_inv"] << (l - 1)) == top[1]:
                work += iters_c[l] * n_of(top[1])
    flops_per_launch = FLOPS_PER_NODE_ITER * work / max(top[2], 1)
    ms_per_launch = top[3] / max(top[2], 1)
    achieved = flops_per_launch / (ms_per_launch / 1e3) / 1e12
    traffic = None
    tf = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    if os.path.exists(tf):
        try:
            traffic = json.load(open(tf)).get(f"{top[0]}_N{top[1]}")
        except Exception:
            traffic = None
    roofline = {"kernel": f"{top[0]} N={top[1]}", "bound": "alu", "achieved": achieved, "peak": FP64_PEAK_TFLOPS,
                "unit": "TFLOP/s", "frac": achieved / FP64_PEAK_TFLOPS, "traffic": traffic,
                "peak_source": ALU["source"],
                "flops_basis": f"{FLOPS_PER_NODE_ITER:.0f} flops per unknown per MINRES iteration (SURVEY 8(d)) x "
                               "unknowns x iterations of the kernel's launches",
                "share_of_level_pass": top[3] / per_level_total_ms,
                "timing": "library CUDA events around each launch during the per-level pass (levels one at a time)",
                "launches": top[2], "ms_per_launch": ms_per_launch}
    kernels = [{"kernel": f"{k}", "N": N, "launches": n, "ms_total": ms, "share": ms / per_level_total_ms}
               for (k, N, n, ms) in kern]

    line = {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms_per_step, "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": c2_config(world, backend),
            "per_level": per_level, "roofline": roofline, "kernels": kernels, "gpu_launches": gpu_launches,
            "clocks": clk}

    _dbg("timed steps and level pass done")
    if not args.no_extras:
        line["c2_step_with_mgpcg"] = mg_leg(ctx, cfg, args, world, rank, torch, dist, stream)
        line["c2_step_coarse_to_fine"] = c2f_step_leg(ctx, cfg, args, world, rank, torch, dist, stream)
        _dbg("mg leg done")
        line["e2e"] = e2e_leg(ctx, cfg, args, world, rank, torch, np, dist)
        _dbg("e2e leg done")
        line["time_to_eps"] = adaptive_leg(args, world, rank, local, torch, dist)
        _dbg("adaptive leg done")
        line["c1_fp64"] = c1_leg(local, torch)
        _dbg("c1 leg done")
        line["c3_cholesky_ir"] = c3_leg(local, torch)
        _dbg("c3 leg done")
        line["fine_meshes"] = fine_leg(local, torch)
        _dbg("fine leg done")
        if rank == 0:
            line["fine_single_system"] = dd_leg(local, torch)
            line["c2_level3_coarse_to_fine"] = c2f_leg(local, torch)
        _dbg("dd / c2f legs done")
        if rank == 0:
            line["paper_mpml_vs_mlmc"] = paper_leg(local)
        if rank == 0 and world == 1:
            line["cpu_baseline"] = cpu_baseline(seed)
    ctx.close()
    if rank == 0:
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()


def e2e_leg(ctx, cfg, args, world, rank, torch, np, dist):
    """Same metric through the public C-ABI call with HOST buffers: pinned host xi in,
    per-sample records + level sums out, copies inside the timed region."""
    Nl, tols, m = cfg["N"], cfg["tols"], cfg["m"]
    rng = np.random.default_rng(1000 + rank)
    xs = [torch.from_numpy(rng.standard_normal((n, m))).pin_memory() for n in Nl]
    outs = [torch.zeros((n, 8), dtype=torch.float64).pin_memory() for n in Nl]
    from paper_2503_05533_b200 import precision
    mr = precision("minres")

    L = len(Nl)
    tol_c = [tols[l - 1] if l else tols[0] for l in range(L)]

    def step():
        # one call: every level's host xi copied in and records copied out on the level's own stream
        ctx.sample_levels_xi(list(range(L)), xs, [mr] * L, [mr] * L, tols, tol_c, per_sample=outs)
    for _ in range(max(1, args.warmup)):
        step()
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(args.steps):
        step()
    torch.cuda.synchronize()
    el = time.perf_counter() - t0
    if world > 1:
        t = torch.tensor([el], dtype=torch.float64, device=torch.device("cuda", torch.cuda.current_device()))
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        el = float(t.item())
    return {"value": world * sum(Nl) * args.steps / el, "unit": UNIT,
            "h2d_bytes_per_step": int(sum(Nl) * m * 8), "d2h_bytes_per_step": int(sum(Nl) * 8 * 8 + len(Nl) * 96),
            "api": "mlmc_sample_levels_xi (all levels concurrently; host pinned xi in, host per-sample records + "
                   "level sums out)",
            "clock": "host wall clock around the synchronous calls, max over ranks"}


def c1_leg(local, torch):
    """configs[0] (C1): both levels (h = 1/8, 1/16; N = 2000, 500 coupled samples) solved in binary64 to
    relative residual 1e-12 -- the parity configuration -- with MINRES and with the binary64 banded
    Cholesky (+ IR, u_s = binary64); device time of one sample_level call per level (median of 5)."""
    from paper_2503_05533_b200 import Context, precision
    cfg = W.CONFIGS["C1"]
    ctx = Context(field="expcov", m=cfg["m"], sigma2=cfg["sigma2"], corr_len=cfg["corr_len"], h0_inv=cfg["h0_inv"],
                  L_max=cfg["L_max"], device=local, workspace_bytes=1 << 30)
    stream = torch.cuda.current_stream()
    sums = torch.zeros(12, dtype=torch.float64, device=torch.device("cuda", local))
    out = {}
    for name, prec in (("minres", precision("minres")), ("chol_fp64", precision("chol_ir", "d", "d"))):
        for l, n in enumerate(cfg["N"]):
            ctx.sample_level_async(l, n, cfg["seed"], 10**7, prec, prec, cfg["tol"], cfg["tol"], sums_out=sums)
            ts = []
            for rep in range(5):
                a0, a1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                a0.record(stream)
                ctx.sample_level_async(l, n, cfg["seed"], 0, prec, prec, cfg["tol"], cfg["tol"], sums_out=sums)
                a1.record(stream)
                torch.cuda.synchronize()
                ts.append(a0.elapsed_time(a1))
            s = sums.cpu().numpy()
            ms = sorted(ts)[2]
            out[f"l{l}_{name}"] = {"h": f"1/{cfg['h0_inv'] << l}", "samples": n, "ms": ms,
                                   "samples_per_s": n / (ms / 1e3), "mean_steps_fine": s[7] / n,
                                   "failures": s[6]}
    ctx.close()
    return out


def c3_leg(local, torch):
    """configs[2]: 100000 coupled samples per level, h = 1/8, 1/16, 1/32, banded Cholesky in fp16 / fp32
    with fp64 iterative refinement to 1e-10 (substitutions in fp32); device-timed per level.  K4 is HBM-bound:
    its roofline line counts the algorithmic factor bytes -- the band factor
    n(bw+1) b_f written once and read by every substitution (2 per solve: x0 and each correction) -- plus the
    coefficient read, over the library's per-launch CUDA-event time of the Cholesky-IR kernels."""
    import numpy as np
    from paper_2503_05533_b200 import Context, precision
    cfg = W.CONFIGS["C3"]
    ctx, ws_gb = None, 0
    for ws_gb in (48, 16, 4):          # one pass of 100k samples needs ~32 GB (fp32 factors); smaller: more passes
        try:
            ctx = Context(field="expcov", m=cfg["m"], sigma2=cfg["sigma2"], corr_len=cfg["corr_len"],
                          h0_inv=cfg["h0_inv"], L_max=cfg["L_max"], device=local, workspace_bytes=ws_gb << 30)
            break
        except torch.cuda.OutOfMemoryError:
            torch.cuda.empty_cache()
    stream = torch.cuda.current_stream()
    sums = torch.zeros(12, dtype=torch.float64, device=torch.device("cuda", local))
    out = {}
    for uf in ("h", "s"):
        prec = precision("chol_ir", uf, "s")
        bf = 2 if uf == "h" else 4
        for l, n in enumerate(cfg["N"]):
            ctx.sample_level_async(l, 2000, cfg["seed"], 10**7, prec, prec, cfg["tol"], cfg["tol"], sums_out=sums)
            # the level's time (fine and coarse solves concurrent), then the per-kernel times (serialised)
            a0, a1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a0.record(stream)
            ctx.sample_level_async(l, n, cfg["seed"], 0, prec, prec, cfg["tol"], cfg["tol"], sums_out=sums)
            a1.record(stream)
            torch.cuda.synchronize()
            ms = a0.elapsed_time(a1)
            ctx.profile_enable(True)
            ctx.sample_level_async(l, n, cfg["seed"], 0, prec, prec, cfg["tol"], cfg["tol"], sums_out=sums)
            torch.cuda.synchronize()
            prof = ctx.profile_read()
            ctx.profile_enable(False)
            s = sums.cpu().numpy()
            Nf, Nc = cfg["h0_inv"] << l, (cfg["h0_inv"] << (l - 1)) if l else 0
            k_ms = sum(r[3] for r in prof if r[0] == "chol_ir")

            def solve_bytes(N, steps_sum):
                fac = (N - 1) ** 2 * N * bf                      # band factor n (bw + 1) b_f
                return n * fac * 3 + fac * 2 * steps_sum + n * 16 * N * N

            def solve_flops(N, steps_sum):
                # n bw^2 per factorisation, 4 n bw per substitution pair (x0 and every correction),
                # 10 n per binary64 residual (one per pair)
                nn, bw = (N - 1) ** 2, N - 1
                return n * (nn * bw * bw + 4 * nn * bw + 10 * nn) + steps_sum * (4 * nn * bw + 10 * nn)

            stream_bytes = solve_bytes(Nf, s[7]) + (solve_bytes(Nc, s[8]) if l else 0.0)
            flops = solve_flops(Nf, s[7]) + (solve_flops(Nc, s[8]) if l else 0.0)
            # the HBM bytes the method itself needs once the factor is on chip: the triangle
            # coefficients of both meshes read, the per-sample record written
            alg = n * (16 * Nf * Nf + (16 * Nc * Nc if l else 0) + 64)
            tflops = flops / (k_ms / 1e3) / 1e12 if k_ms > 0 else 0.0
            gbs = stream_bytes / (k_ms / 1e3) / 1e9 if k_ms > 0 else 0.0
            key = f"chol_ir_N{Nf}_{'fp16' if uf == 'h' else 'fp32'}_bytes_per_sample"
            # IR-step histogram of the fine solves: a separate untimed pass over
            # the same samples with per-sample records
            ps = ctx.sample_level(l, n, cfg["seed"], 0, prec, prec, cfg["tol"], cfg["tol"], per_sample=True).per_sample
            steps, counts = np.unique(ps[:, 2].astype(int), return_counts=True)
            out[f"l{l}_{'fp16' if uf == 'h' else 'fp32'}"] = {
                "h": f"1/{Nf}", "samples": n, "ms": ms, "samples_per_s": n / (ms / 1e3),
                "mean_ir_steps_fine": s[7] / n, "max_ir_steps_fine": s[9], "failures": s[6],
                "ir_steps_histogram_fine": {str(int(a)): int(b) for a, b in zip(steps, counts)},
                "k4_ms": k_ms,
                "k4_roofline": {"bound": "alu", "achieved": tflops, "peak": FP32_PEAK_TFLOPS, "unit": "TFLOP/s",
                                "frac": tflops / FP32_PEAK_TFLOPS, "peak_source": ALU["source"] + " (FFMA)",
                                "flops_basis": "SURVEY 8(d): n bw^2 per factorisation + 4 n bw per substitution "
                                               "pair + 10 n per residual, fine + coarse"},
                "k4_algorithmic_bytes_per_sample": alg / n,
                "k4_dram_bytes_per_sample_ncu": _ncu_traffic(key),
                "k4_factor_stream_GBs": gbs, "k4_factor_stream_hbm_frac": gbs / HBM_PEAK_GBS,
                "workspace_GB": ws_gb}
    ctx.close()
    return out


def _ncu_traffic(key):
    """dram__bytes_read.sum + dram__bytes_write.sum of one launch / sample from a committed ncu capture
    (profiles/ncu_traffic.json, written from the round's ncu reports), or None."""
    try:
        return json.load(open(os.path.join(ROOT, "profiles", "ncu_traffic.json"))).get(key)
    except Exception:
        return None


def dd_leg(local, torch):
    """NEXT-3 / the fine-level critical path: ONE configs[4] system at h = 1/512 to the finest tolerance of an L = 6
    run (eps_6 = k_p h^2), fine half only -- by K3c in a 2-CTA cluster (what mlmc_sample_level does per sample)
    and by K3d on the whole GPU (mlmc_dd_run_local, one slab).  Device time, CUDA events."""
    from paper_2503_05533_b200 import Context, precision
    from paper_2503_05533_b200.dd import SlabSolver
    cfg = W.CONFIGS["C5"]
    ctx = Context(field="expcov", m=cfg["m"], sigma2=cfg["sigma2"], corr_len=cfg["corr_len"], h0_inv=cfg["h0_inv"],
                  L_max=cfg["L_max"], device=local, workspace_bytes=2 << 30)
    N, level = 512, 6
    tol = cfg["k_p"] / N ** 2
    stream = torch.cuda.current_stream()

    def timed(fn):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(stream)
        r = fn()
        b.record(stream)
        torch.cuda.synchronize()
        return r, a.elapsed_time(b)
    mr = precision("minres")
    ctx.sample_level(level, 1, 7, first_index=99, prec_fine=mr, tol_fine=1e-3, tol_coarse=1e-3)
    ctx.profile_enable(True)
    r, ms = timed(lambda: ctx.sample_level(level, 1, 7, first_index=0, prec_fine=mr, tol_fine=tol, tol_coarse=tol,
                                           per_sample=True).per_sample[0])
    prof = ctx.profile_read()
    ctx.profile_enable(False)
    k3c_ms = sum(p[3] for p in prof if p[0] == "minres" and p[1] == N)
    eng = SlabSolver(ctx, level, 0, 1)
    eng.begin(7, level, 0, tol)
    d, dms = timed(eng.run_local)
    eng.close()
    ctx.close()
    return {"h": "1/512", "tol": tol, "k3c_cluster2": {"ms_fine_kernel": k3c_ms, "iters": r[2], "Q": r[0]},
            "k3d_whole_gpu": {"ms": dms, "iters": d["iters"], "us_per_step": 1e3 * dms / max(d["iters"], 1),
                              "Q": d["Q"]},
            "speedup": k3c_ms / dms if dms > 0 else None}


def c2f_leg(local, torch):
    """NEXT-4 coarse-to-fine x0 on the configs[1] level-3 pass (300 coupled samples, tol 1e-8 / 1e-6): device
    time of the pass and mean fine MINRES steps from x0 = 0 and from the P1 interpolation of the coarse solution."""
    from paper_2503_05533_b200 import Context, precision
    cfg = W.CONFIGS["C2"]
    ctx = Context(field="expcov", m=cfg["m"], sigma2=cfg["sigma2"], corr_len=cfg["corr_len"], h0_inv=8, L_max=3,
                  device=local, workspace_bytes=1 << 30)
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=torch.device("cuda", local))
    mr = precision("minres")
    out = {}
    for name, pf in (("x0=0", mr), ("x0=Pxc", precision("minres", c2f=True))):
        ctx.sample_level(3, 300, 5, first_index=10**6, prec_fine=pf, prec_coarse=mr, tol_fine=1e-8, tol_coarse=1e-6)
        ts, its = [], []
        for rep in range(5):
            flush.zero_()
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record()
            r = ctx.sample_level(3, 300, 5, first_index=300 * rep, prec_fine=pf, prec_coarse=mr, tol_fine=1e-8,
                                 tol_coarse=1e-6)
            b.record()
            torch.cuda.synchronize()
            ts.append(a.elapsed_time(b))
            its.append(r.sums["iters_f"] / 300)
        out[name] = {"ms_median": sorted(ts)[2], "mean_fine_steps": sum(its) / len(its)}
    ctx.close()
    return out


def fine_leg(local, torch):
    """MINRES on the fine meshes of configs[4]: K3b (h = 1/128 on 4-CTA clusters, 1/256 on 16-CTA clusters, every
    row on chip) and K3c (h = 1/512, streamed): one batch of 148 systems per mesh, 300 MINRES steps each
    (max_iter; the finest levels need thousands -- the rate per step is what the roofline measures).  K3b is
    FP64-ALU work on chip (28 flops per unknown and step); K3c moves p_j, p_{j-1}, cE, cN in and
    p_{j+1} out once per step: 40 algorithmic bytes per unknown and step.  The kernel time
    is the library's per-launch CUDA-event time."""
    from paper_2503_05533_b200 import Context, precision
    cfg = W.CONFIGS["C5"]
    ctx = Context(field="expcov", m=cfg["m"], sigma2=cfg["sigma2"], corr_len=cfg["corr_len"], h0_inv=cfg["h0_inv"],
                  L_max=cfg["L_max"], device=local, workspace_bytes=8 << 30)
    sums = torch.zeros(12, dtype=torch.float64, device=torch.device("cuda", local))
    nb, steps = 148, 300
    prec = precision("minres", max_iter=steps)
    out = {}
    for level in (4, 5, 6):
        N = cfg["h0_inv"] << level
        ctx.sample_level_async(level, 2, cfg["seed"], 10**6, prec, prec, 1e-14, 1e-14, sums_out=sums)
        ctx.profile_enable(True)
        ctx.sample_level_async(level, nb, cfg["seed"], 0, prec, prec, 1e-14, 1e-14, sums_out=sums)
        prof = ctx.profile_read()
        ctx.profile_enable(False)
        s = sums.cpu().numpy()
        k_ms = sum(r[3] for r in prof if r[0] == "minres" and r[1] == N)
        node_steps = s[7] * (N - 1) ** 2
        row = {"systems": nb, "minres_steps_each": s[7] / nb, "kernel_ms": k_ms,
               "unknown_steps_per_s": node_steps / (k_ms / 1e3)}
        if N <= 256:                                                   # K3b: on chip, FP64 ALU
            tf = FLOPS_PER_NODE_ITER * node_steps / (k_ms / 1e3) / 1e12
            row.update({"kernel": "K3b minres cluster", "achieved_TFLOPs_28": tf, "fp64_frac": tf / FP64_PEAK_TFLOPS,
                        "bound": "alu"})
        else:                                                          # K3c: streamed, HBM
            gbs = 40.0 * node_steps / (k_ms / 1e3) / 1e9
            row.update({"kernel": "K3c minres stream", "achieved_GBs_40B": gbs, "hbm_frac": gbs / HBM_PEAK_GBS,
                        "bound": "hbm"})
        out[f"h=1/{N}"] = row
    # K3m-t, the temporally blocked MG-PCG on the same meshes (NEXT-4): a real solve to 1e-6, 148 systems.
    # Algorithmic bytes per fine unknown and CG step: 106 on the fine level (passes C 44, A 37, B 25) + 37
    # for the coarser levels' plain V-cycle passes = 143 B (ncu measured 147).
    mg = precision("mgcg")
    for level in (5, 6):
        N = cfg["h0_inv"] << level
        ctx.sample_level_async(level, 2, cfg["seed"], 10**6, mg, mg, 1e-6, 1e-6, sums_out=sums)
        ctx.profile_enable(True)
        ctx.sample_level_async(level, nb, cfg["seed"], 0, mg, mg, 1e-6, 1e-6, sums_out=sums)
        prof = ctx.profile_read()
        ctx.profile_enable(False)
        s = sums.cpu().numpy()
        k_ms = sum(r[3] for r in prof if r[0] == "minres" and r[1] == N)
        node_steps = s[7] * (N - 1) ** 2
        gbs = 143.0 * node_steps / (k_ms / 1e3) / 1e9
        out[f"mgpcg h=1/{N}"] = {"systems": nb, "cg_steps_mean": s[7] / nb, "kernel_ms": k_ms,
                                 "unknown_steps_per_s": node_steps / (k_ms / 1e3), "achieved_GBs_143B": gbs,
                                 "hbm_frac": gbs / HBM_PEAK_GBS, "bound": "hbm"}
    ctx.close()
    return out


def c2f_step_leg(ctx, cfg, args, world, rank, torch, dist, stream):
    """The same configs[1] step (MINRES, same tolerances) with the NEXT-4 coarse-to-fine initial guess on levels
    1-3 (MLMC_FLAG_C2F: each level's coarse half first, its fine half from P x_c; R32).  Device-timed like the
    headline, L2 flushed between steps."""
    from paper_2503_05533_b200 import precision
    Nl, tols, seed = cfg["N"], cfg["tols"], cfg["seed"]
    L = len(Nl)
    dev = torch.device("cuda", torch.cuda.current_device())
    pf = [precision("minres", c2f=(l > 0)) for l in range(L)]
    pc = [precision("minres") for _ in range(L)]
    tol_c = [tols[l - 1] if l else tols[0] for l in range(L)]
    sums = torch.zeros((L, 12), dtype=torch.float64, device=dev)
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)

    def step(i):
        first = [(i * world + rank) * Nl[l] for l in range(L)]
        ctx.sample_levels_async(list(range(L)), Nl, seed, first, pf, pc, tols, tol_c, sums)
        if world > 1:
            dist.all_reduce(sums)
    for i in range(args.warmup):
        step(40_000 + i)
    torch.cuda.synchronize()
    total, its = 0.0, [0.0] * L
    for i in range(args.steps):
        flush.zero_()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        step(i)
        e1.record(stream)
        torch.cuda.synchronize()
        total += e0.elapsed_time(e1)
        s = sums.cpu().numpy()
        for l in range(L):
            its[l] += s[l, 7] / world
    if world > 1:
        t = torch.tensor([total], dtype=torch.float64, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        total = float(t.item())
    return {"solver": "MINRES, fine halves of levels 1-3 from the P1 interpolation of the coarse solution",
            "ms_per_step": total / args.steps, "value": world * sum(Nl) * args.steps / (total / 1e3), "unit": UNIT,
            "mean_iters_fine": [its[l] / (Nl[l] * args.steps) for l in range(L)]}


def mg_leg(ctx, cfg, args, world, rank, torch, dist, stream):
    """The same configs[1] step with the NEXT-4 solver where it pays: multigrid-preconditioned CG (K3m;
    same relative-residual tolerances, same per-sample accuracy contract) on the h <= 1/32 meshes,
    MINRES on h = 1/8, 1/16.  Not the headline (the configuration names MINRES); device-timed like it."""
    from paper_2503_05533_b200 import precision
    Nl, tols, seed = cfg["N"], cfg["tols"], cfg["seed"]
    L = len(Nl)
    dev = torch.device("cuda", torch.cuda.current_device())
    pick = lambda N: precision("mgcg") if N >= 32 else precision("minres")
    pf = [pick(cfg["h0_inv"] << l) for l in range(L)]
    pc = [pick(cfg["h0_inv"] << (l - 1)) if l else precision("minres") for l in range(L)]
    tol_c = [tols[l - 1] if l else tols[0] for l in range(L)]
    sums = torch.zeros((L, 12), dtype=torch.float64, device=dev)
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)

    def step(i):
        first = [(i * world + rank) * Nl[l] for l in range(L)]
        ctx.sample_levels_async(list(range(L)), Nl, seed, first, pf, pc, tols, tol_c, sums)
        if world > 1:
            dist.all_reduce(sums)
    for i in range(args.warmup):
        step(20_000 + i)
    torch.cuda.synchronize()
    total, its = 0.0, [0.0] * L
    for i in range(args.steps):
        flush.zero_()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        step(30_000 + i)
        e1.record(stream)
        torch.cuda.synchronize()
        total += e0.elapsed_time(e1)
        s = sums.cpu().numpy()
        for l in range(L):
            its[l] += s[l, 7] / world
    if world > 1:
        t = torch.tensor([total], dtype=torch.float64, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        total = float(t.item())
    return {"solver": "MG-PCG (h <= 1/32) + MINRES (h >= 1/16), same tolerances",
            "ms_per_step": total / args.steps, "value": world * sum(Nl) * args.steps / (total / 1e3), "unit": UNIT,
            "mean_iters_fine": [its[l] / (Nl[l] * args.steps) for l in range(L)]}


def paper_leg(local):
    """The paper's own experiment (Section 5.1): adaptive MPML vs standard adaptive MLMC (fixed
    MINRES tolerance 1e-6) on the Eq. (20) field, R = 100 replicate runs per method and TOL^2 (the paper:
    1000; tools/paper_experiment.py runs those, profiles/r01e_paper_experiment.md).  Reports the modelled
    cost ratio (the paper's FLOP count analogue, ~1.5 there), the GPU solve-time ratio and both MSEs."""
    sys.path.insert(0, os.path.join(ROOT, "tools"))
    import paper_experiment
    t0 = time.perf_counter()
    res = paper_experiment.run(R=100, device=local)
    out = {"R": res["R"], "reference_Q": res["reference"]["estimate"], "seconds": time.perf_counter() - t0}
    for k, e in res["tol2"].items():
        out[f"TOL2={k}"] = {"cost_ratio_mlmc_over_mpml": e["cost_ratio_mlmc_over_mpml"],
                            "gpu_time_ratio_mlmc_over_mpml": e["gpu_time_ratio_mlmc_over_mpml"],
                            "mse_mpml": e["mpml"]["mse"], "mse_mlmc": e["mlmc"]["mse"]}
    return out


def adaptive_leg(args, world, rank, local, torch, dist):
    """Time-to-eps of Algorithm 2 for configs[3] (C4) and configs[4] (C5), wall clock, max over ranks: policy 0
    (the paper's MINRES at eps_l) and policy 3 (auto: the solver / precision per mesh from pilot timings,
    SURVEY A14; the timed run reuses the choice the untimed first run made)."""
    from paper_2503_05533_b200 import Context
    out = {}
    for name in ("C4", "C5"):
        cfg = W.CONFIGS[name]
        ctx = Context(field="expcov", m=cfg["m"], sigma2=cfg["sigma2"], corr_len=cfg["corr_len"],
                      h0_inv=cfg["h0_inv"], L_max=cfg["L_max"], device=local, workspace_bytes=1 << 30)
        for l in range(4):                                   # plan warm-up: Phi_l uploaded before timing
            ctx.sample_level(l, 1, cfg["seed"] + 99, tol_fine=1e-2, tol_coarse=1e-2)
        if world > 1:
            dist.barrier()
        grp = dist.group.WORLD if world > 1 else None
        for policy, key in ((0, name), (3, f"{name}_auto")):
            # an untimed run first (other seed): policy 3's pilots run once per mesh and tolerance class and the
            # timed run reuses the choice; for policy 0 it is the warm-up of the run's launch path
            ctx.adaptive_run(cfg["eps"], k_p=cfg["k_p"], N_init=100, seed=cfg["seed"] + 1, policy=policy, group=grp)
            if world > 1:
                dist.barrier()
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            r = ctx.adaptive_run(cfg["eps"], k_p=cfg["k_p"], N_init=100, seed=cfg["seed"], policy=policy, group=grp)
            torch.cuda.synchronize()
            el = time.perf_counter() - t0
            if world > 1:
                t = torch.tensor([el], dtype=torch.float64, device=torch.device("cuda", local))
                dist.all_reduce(t, op=dist.ReduceOp.MAX)
                el = float(t.item())
            out[key] = {"eps": cfg["eps"], "policy": policy, "seconds": el, "L": r["L"], "N": r["N"],
                        "rounds": r["rounds"], "estimate": r["estimate"], "code": r["code"]}
            if policy == 3:
                out[key]["choice"] = {str(cfg["h0_inv"] << l): ctx.auto_choice(cfg["h0_inv"] << l)
                                      for l in range(r["L"] + 1)}
        ctx.close()
    return out


def main():
    args = parse()
    if args.impl == "reference":
        run_reference(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
