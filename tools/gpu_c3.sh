#!/bin/bash
# K4 (Cholesky-IR) pass: build, the IR parity tests, then the configs[2] timing leg of bench.py.
mkdir -p gpurun_out
python __graft_entry__.py > gpurun_out/build.log 2>&1 || { tail -30 gpurun_out/build.log; exit 1; }
timeout 600 python -m pytest tests -m gpu -x -q -k "C3 or ir_ or smoke or edge" > gpurun_out/pytest_c3.log 2>&1; echo "pytest rc=$?"
tail -15 gpurun_out/pytest_c3.log
timeout 600 python -c "
import json, torch, bench
print(json.dumps(bench.c3_leg(0, torch), indent=1))" > gpurun_out/c3.json 2>&1; echo "c3 rc=$?"
cat gpurun_out/c3.json | head -80
