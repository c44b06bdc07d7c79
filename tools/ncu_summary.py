"""Summarise ncu output for profiles/ (run here, on the CPU box, after a gpurun ncu pass).

  python tools/ncu_summary.py launches <launches.csv>          per-kernel launch list (count, time, share)
  python tools/ncu_summary.py full <prof.ncu-rep>              key counters of every captured launch
  python tools/ncu_summary.py traffic <prof.ncu-rep> <out.json>  dram bytes per launch, keyed like bench.py

The launch list is cold-cache and serialised (one kernel at a time under ncu):
compare SHARES with bench.py's per-kernel table, not absolute times.
"""
import csv
import io
import json
import re
import subprocess
import sys
from collections import defaultdict


def short(name: str) -> str:
    m = re.search(r"(\w+_kernel)(<[^>]*>)?", name)
    if not m:
        return name[:60]
    tpl = (m.group(2) or "").replace("(int)", "").replace("(bool)", "")
    return m.group(1) + tpl


def launches(path):
    txt = open(path).read().splitlines()
    body = [l for l in txt if l.startswith('"')]
    rows = list(csv.DictReader(io.StringIO("\n".join(body))))
    agg = defaultdict(lambda: [0, 0.0])
    for r in rows:
        if r.get("Metric Name") != "gpu__time_duration.sum":
            continue
        scale = {"ns": 1e-3, "us": 1.0, "usecond": 1.0, "ms": 1e3, "msecond": 1e3, "nsecond": 1e-3}[r["Metric Unit"]]
        k = short(r["Kernel Name"])
        agg[k][0] += 1
        agg[k][1] += float(r["Metric Value"].replace(",", "")) * scale
    ours = {k: v for k, v in agg.items() if not k.startswith(("vectorized_elementwise", "elementwise", "at::"))
            and "FillFunctor" not in k}
    tot = sum(v[1] for v in ours.values())
    print("| kernel | launches | total us | share of our kernels |")
    print("|---|---|---|---|")
    for k, v in sorted(ours.items(), key=lambda x: -x[1][1]):
        print(f"| `{k}` | {v[0]} | {v[1]:.1f} | {100 * v[1] / tot:.1f}% |")
    other = {k: v for k, v in agg.items() if k not in ours}
    if other:
        print(f"\n(torch kernels in the capture, not ours: {sum(v[0] for v in other.values())} launches, "
              f"{sum(v[1] for v in other.values()):.1f} us -- the L2 flush / sums zeroing)")


def raw(path):
    """The raw page of an ncu report (or of its CSV export `ncu -i rep --page raw --csv > rep.raw.csv`, made on
    the GPU box so that the large .ncu-rep need not travel back)."""
    if path.endswith(".csv"):
        out = open(path).read()
    else:
        out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    r = list(csv.reader(io.StringIO(out)))
    return r[0], r[1], r[2:]


KEYS = [
    ("gpu__time_duration.sum", "duration"),
    ("launch__grid_size", "grid"),
    ("launch__block_size", "block"),
    ("launch__registers_per_thread", "regs/thread"),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "achieved occupancy %"),
    ("sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active", "FP64 pipe % (active)"),
    ("sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_elapsed", "FP64 pipe % (elapsed)"),
    ("sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active", "LSU pipe % (active)"),
    ("sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active", "FMA pipe % (active)"),
    ("sm__pipe_fp16_cycles_active.avg.pct_of_peak_sustained_active", "FP16 pipe % (active)"),
    ("smsp__issue_active.avg.pct_of_peak_sustained_active", "issue slots busy %"),
    ("smsp__inst_executed.sum", "warp instructions"),
    ("l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum", "smem bank conflicts"),
    ("dram__bytes_read.sum", "DRAM read"),
    ("dram__bytes_write.sum", "DRAM write"),
    ("sass__inst_executed_local_loads", "local loads (spills)"),
]
STALLS = ["short_scoreboard", "wait", "math_pipe_throttle", "mio_throttle", "not_selected", "barrier",
          "dispatch_stall", "branch_resolving", "long_scoreboard", "lg_throttle", "no_instruction"]


def full(path):
    h, u, rows = raw(path)
    idx = {n: j for j, n in enumerate(h)}
    names = [short(r[idx["Kernel Name"]]) for r in rows]
    print("| counter | " + " | ".join(f"#{i} `{n}`" for i, n in enumerate(names)) + " |")
    print("|---|" + "---|" * len(rows))
    for key, label in KEYS:
        if key in idx:
            j = idx[key]
            print(f"| {label} ({u[j]}) | " + " | ".join(r[j] for r in rows) + " |")
    for s in STALLS:
        key = f"smsp__average_warps_issue_stalled_{s}_per_issue_active.ratio"
        if key in idx:
            j = idx[key]
            print(f"| stall {s} (warps per issue) | " + " | ".join(r[j] for r in rows) + " |")


def traffic(path, out):
    h, u, rows = raw(path)
    idx = {n: j for j, n in enumerate(h)}
    unit = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
    res = {}
    for r in rows:
        m = re.search(r"minres_strip_kernel<\(?i?n?t?\)?(\d+)", r[idx["Kernel Name"]])
        nm = re.search(r"<(?:\(int\))?(\d+)", r[idx["Kernel Name"]])
        key = f"minres_N{nm.group(1)}" if "minres" in r[idx["Kernel Name"]] and nm else short(r[idx["Kernel Name"]])
        b = sum(float(r[idx[k]].replace(",", "")) * unit[u[idx[k]]] for k in ("dram__bytes_read.sum", "dram__bytes_write.sum"))
        res.setdefault(key, b)
    json.dump(res, open(out, "w"), indent=1)
    print(json.dumps(res))


if __name__ == "__main__":
    {"launches": lambda: launches(sys.argv[2]), "full": lambda: full(sys.argv[2]),
     "traffic": lambda: traffic(sys.argv[2], sys.argv[3])}[sys.argv[1]]()
