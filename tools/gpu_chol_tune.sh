#!/bin/bash
# K4 tuning pass: configs[2] level 2 (h = 1/32) for every ring-depth / CTA-shape variant, then the IR tests.
mkdir -p gpurun_out
python __graft_entry__.py > gpurun_out/build.log 2>&1 || { tail -30 gpurun_out/build.log; exit 1; }
for uf in h s; do for v in 0 1 2 3 4; do
  MLMC_CHOL_VARIANT=$v timeout 300 python tools/c3_one.py 2 $uf 100000 2>&1 | sed "s/^/v$v /"
done; done | tee gpurun_out/chol_tune.log
timeout 600 python -m pytest tests -m gpu -x -q -k "C3 or ir_ or edge" > gpurun_out/pytest_c3.log 2>&1; echo "pytest rc=$?"
tail -3 gpurun_out/pytest_c3.log
