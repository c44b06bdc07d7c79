#!/bin/bash
# A/B of the longest-first MINRES job order (MLMC_ORDER) on the bench step, then the GPU tests.
mkdir -p gpurun_out
python __graft_entry__.py > gpurun_out/build.log 2>&1 || { tail -30 gpurun_out/build.log; exit 1; }
for o in 0 1 0 1; do
  MLMC_ORDER=$o timeout 300 python bench.py --steps 10 --warmup 3 --no-extras 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print('order=$o', round(d['ms_per_step'],4), 'ms/step', {k: round(v['ms_alone'],3) for k,v in d['per_level'].items()}, 'frac', round(d['roofline']['frac'],3))"
done | tee gpurun_out/order_ab.log
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/pytest_gpu.log
