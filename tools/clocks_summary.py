"""Summarise an `nvidia-smi --query-gpu=... --format=csv -lms N` log (the recipe's clocks line):
median SM clock over the samples under load (power above idle), max clock, reasons seen."""
import csv
import json
import statistics
import sys


def summarise(path):
    rows = []
    with open(path) as f:
        rd = csv.reader(f)
        hdr = next(rd, None)
        for r in rd:
            if len(r) < 9:
                continue
            try:
                sm = float(r[1].split()[0])
                mx = float(r[2].split()[0])
                pw = float(r[3].split()[0])
            except ValueError:
                continue
            rows.append((sm, mx, pw, [x.strip() for x in r[5:9]]))
    if not rows:
        return {"samples": 0}
    names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
    idle = min(p for _, _, p, _ in rows)
    load = [r for r in rows if r[2] > idle + 50] or rows
    reasons = sorted({names[i] for _, _, _, fl in load for i, v in enumerate(fl) if v.lower() == "active"})
    return {"samples": len(rows), "samples_under_load": len(load),
            "sm_mhz": statistics.median(r[0] for r in load), "sm_max_mhz": max(r[1] for r in rows),
            "power_w_max": max(r[2] for r in rows), "reasons": reasons}


if __name__ == "__main__":
    print(json.dumps(summarise(sys.argv[1])))
