"""Opcode histogram (executed warp instructions and stall samples) of one kernel in an ncu report.
Usage: python tools/sass_hist.py <rep> <kernel-regex> [launch-skip]"""
import csv, io, subprocess, sys
from collections import defaultdict
rep, kre = sys.argv[1], sys.argv[2]
skip = sys.argv[3] if len(sys.argv) > 3 else "0"
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass", "-k", "regex:" + kre,
                      "--launch-skip", skip, "--launch-count", "1"], capture_output=True, text=True).stdout
r = list(csv.reader(io.StringIO(out)))
h = r[1]; rows = r[2:]
si = h.index("Warp Stall Sampling (All Samples)"); ie = h.index("Instructions Executed"); src = h.index("Source")
num = lambda s: int(s) if s.strip().isdigit() else 0
rows = [x for x in rows if len(x) > si and x[0].startswith("0x")]
tot = sum(num(x[si]) for x in rows) or 1
ex = defaultdict(int); st = defaultdict(int)
for x in rows:
    t = x[src].split()
    if not t: continue
    op = t[1] if t[0].startswith("@") and len(t) > 1 else t[0]
    op = op.split(".")[0]
    ex[op] += num(x[ie]); st[op] += num(x[si])
te = sum(ex.values()) or 1
print(f"{r[0][1][:100]}\ntotal stall samples {tot}, executed warp instrs {te}, static instrs {len(rows)}")
for op in sorted(ex, key=lambda o: -ex[o])[:28]:
    print(f"{op:10s} exec {100 * ex[op] / te:5.1f}%  stall-samples {100 * st[op] / tot:5.1f}%")
