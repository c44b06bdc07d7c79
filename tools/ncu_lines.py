"""Per-source-line instruction and stall-sample shares of one ncu report (needs -lineinfo + --import-source).

  python tools/ncu_lines.py <report.ncu-rep> [top=30] [file-substring]
"""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 30
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"] + (["--launch-skip", sys.argv[3], "--launch-count", "1"] if len(sys.argv) > 3 else []),
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
hi = next(i for i, r in enumerate(rows) if r and r[0] == "Line No")
h = rows[hi]
ie, iss = h.index("Instructions Executed"), h.index("Warp Stall Sampling (All Samples)")
fname = rows[0][1] if rows and rows[0] and rows[0][0] == "File Path" else ""
data = []
cur_file = fname
for r in rows[hi + 1:]:
    if r and r[0] == "File Path":
        cur_file = r[1]
        continue
    if r and r[0] and r[0].isdigit():
        try:
            data.append((int(r[ie] or 0), int(r[iss] or 0), cur_file.split("/")[-1], r[0], r[1].strip()[:100]))
        except ValueError:
            pass
tot = sum(d[0] for d in data) or 1
tots = sum(d[1] for d in data) or 1
print(f"total warp instructions {tot:.4g}, stall samples {tots}")
for d in sorted(data, key=lambda x: -x[1])[:top]:
    print(f"{d[0] / tot * 100:5.1f}% inst {d[1] / tots * 100:5.1f}% stall  {d[2]}:{d[3]}: {d[4]}")
